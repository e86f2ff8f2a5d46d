#!/bin/bash
# fp16-plane covariance: GPU tests touching multi-tile frames + one full ncu capture of the f16 cov kernel (c4).
timeout 900 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_stress.py tests/test_gpu_host.py tests/test_gpu_facade.py -x -q > gpurun_out/f16b_tests.log 2>&1
echo tests rc=$?; tail -1 gpurun_out/f16b_tests.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cov_tc_kernel -s 2 -c 1 \
  -o gpurun_out/r02t_cov_f16 -f python bench.py --config c4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_r02t_cov_f16.log 2>&1
echo ncu rc=$?
