#!/bin/bash
# Co-residency experiment: covariance with fewer registers / a smaller smem ring so the fp64 kernels of
# another sub-batch can share its SMs. Prints ms/step of c2 for each setting.
run() {  # label, env...
  local label=$1; shift
  for ns in 2 4 8; do
    env "$@" python bench.py --steps 100 --warmup 10 --no-e2e --no-cpu-baseline --subbatches $ns 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$label', 'nsub', $ns, round(d['ms_per_step'],4), 'cov_alone', round(d['stages_alone_ms']['covariance'],4))"
  done
}
run default FM_X=0
run conv4 FM_COV_CONV4=1
FM_NVCC_FLAGS="-DFM_COV_MAXNREG=72" python -c "import sys; sys.path.insert(0,'.'); from paper_1911_07434_b200 import build; build.build(force=True)" >/dev/null 2>&1 || echo build failed
run cap72_conv4_r88 FM_COV_CONV4=1
run cap72_conv4_r44 FM_COV_CONV4=1 FM_COV_RING=4,2,4,4
run cap72_conv4_r62 FM_COV_CONV4=1 FM_COV_RING=4,2,6,2
run cap72_conv4_r33 FM_COV_CONV4=1 FM_COV_RING=4,2,3,3
