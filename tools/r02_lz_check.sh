#!/bin/bash
# batched block-Lanczos: probe, GPU tests, a short c2lz bench line
timeout 300 python tools/lz_probe.py 1024 > gpurun_out/lz_probe.json 2>&1; echo "probe rc=$?"
timeout 900 python -m pytest tests/test_gpu_lanczos.py -x -q > gpurun_out/lz_tests.log 2>&1; echo "lz tests rc=$?"
timeout 600 python bench.py --config c2lz --steps 10 --warmup 3 --cpu-frames 32 > gpurun_out/lz_bench.json 2> gpurun_out/lz_bench.err; echo "lz bench rc=$?"
