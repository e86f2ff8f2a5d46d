#!/bin/bash
# A/B of a compile-time variant: build default and with FLAGS, run the c2 bench line (covariance alone + step)
# for each. usage: tools/ab_build.sh "-DFM_X" [runs]
flags=$1; runs=${2:-2}
build() { FM_NVCC_FLAGS="$1" python -c "
import importlib.util
spec = importlib.util.spec_from_file_location('_b', 'paper_1911_07434_b200/build.py')
m = importlib.util.module_from_spec(spec); spec.loader.exec_module(m); m.build(force=True)" > /dev/null 2>&1; }
line() { python bench.py --steps 300 --warmup 10 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); a=d['stages_alone_ms']
print('$2', 'fps', round(d['value']), 'ms', round(d['ms_per_step'],4), 'cov_alone', round(a['covariance'],4), 'sub', round(a['subspace'],4))"; }
for v in A B; do
  if [ $v = A ]; then build ""; else build "$flags"; fi
  for i in $(seq $runs); do line x $v; done
done
