#!/bin/bash
timeout 300 python tools/lz_debug.py > gpurun_out/lz_debug.log 2>&1; echo "debug rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_lanczos_batch -c 1 -f -o gpurun_out/lz_ncu python tools/lz_probe.py 296 > gpurun_out/lz_ncu.log 2>&1; echo "ncu rc=$?"
