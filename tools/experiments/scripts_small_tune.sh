#!/bin/bash
# small-matrix kernel tuning: warps per CTA (eigen-work / Cholesky) and register caps (solve / basis)
run() {
  FM_NVCC_FLAGS="$1" python -c "import sys; sys.path.insert(0,'.'); from paper_1911_07434_b200 import build; build.build(force=True)" > /dev/null 2>&1
  ncu --metrics gpu__time_duration.sum --clock-control none -s 30 -c 12 --csv --log-file gpurun_out/ll_st.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --subbatches 1 > /dev/null 2>&1
  echo "== $1"; python tools/launch_summary.py gpurun_out/ll_st.csv | grep -E "cholpiv|rows_solve|small_warp|basis_ct" | sort | uniq
}
run ""
run "-DFM_SMALL_WARPS=4 -DFM_PIV_WARPS=4"
run "-DFM_SMALL_WARPS=2 -DFM_PIV_WARPS=2"
run "-DFM_SOLVE_MINB=6 -DFM_BASIS_MINB=6"
run "-DFM_SOLVE_MINB=8 -DFM_BASIS_MINB=8"
