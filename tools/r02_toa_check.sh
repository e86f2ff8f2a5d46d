#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_temporal.py tests/test_gpu_toa.py -x -q > gpurun_out/toa_tests.log 2>&1; echo "toa tests rc=$?"
timeout 600 python -m pytest tests/test_gpu_pipeline.py -x -q > gpurun_out/pipe_tests.log 2>&1; echo "pipe tests rc=$?"
timeout 600 python bench.py --config toa --steps 50 --warmup 5 --cpu-frames 32 > gpurun_out/toa_bench.json 2> gpurun_out/toa_bench.err; echo "toa bench rc=$?"
timeout 300 python tools/temporal_bench.py > gpurun_out/temporal_bench.json 2>&1; echo "temporal bench rc=$?"
