#!/bin/bash
# fp32 Jacobi tolerance: pipeline parity (pytest) + warp eigen-work time for each setting
for fl in "-DFM_JACOBI_TOL32=1e-6f" "-DFM_JACOBI_TOL32=1e-5f" "-DFM_JACOBI_TOL32=1e-4f"; do
  FM_NVCC_FLAGS="$fl" python -c "import sys; sys.path.insert(0,'.'); from paper_1911_07434_b200 import build; build.build(force=True)" > /dev/null 2>&1
  python -m pytest tests/test_gpu_pipeline.py -q -x 2>&1 | tail -1 | sed "s/^/[$fl] /"
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_small_warp -c 1 --csv --log-file gpurun_out/ll_tol.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --subbatches 1 > /dev/null 2>&1
  python tools/launch_summary.py gpurun_out/ll_tol.csv | head -1
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_small_warp -c 1 --csv --log-file gpurun_out/ll_tol3.csv python bench.py --config c3 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --subbatches 1 > /dev/null 2>&1
  python tools/launch_summary.py gpurun_out/ll_tol3.csv | head -1
done
