#!/bin/bash
# A/B of the fp16-plane covariance (FM_COV_F16) on the multi-tile configs: alternating builds, 3 runs each.
build() { FM_NVCC_FLAGS="$1" python -c "
import importlib.util
spec = importlib.util.spec_from_file_location('_b', 'paper_1911_07434_b200/build.py')
m = importlib.util.module_from_spec(spec); spec.loader.exec_module(m); m.build(force=True)" > /dev/null 2>&1; }
for rep in 1 2 3; do
for f in 0 1; do
  build "-DFM_COV_F16=$f"
  for cfg in c4 $EXTRA; do
  python bench.py --config $cfg --steps 20 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); a=d['stages_alone_ms']; print('f16 $f $cfg fps', round(d['value']), 'ms', round(d['ms_per_step'],3), 'cov', round(a['covariance'],3))"
  done
done; done
build ""
