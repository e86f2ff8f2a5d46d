#!/bin/bash
# Ring depth of the hi-plane-only range-finder products (FM_HI_STAGES): c2 step and subspace stage per setting.
build() { FM_NVCC_FLAGS="$1" python -c "
import importlib.util
spec = importlib.util.spec_from_file_location('_b', 'paper_1911_07434_b200/build.py')
m = importlib.util.module_from_spec(spec); spec.loader.exec_module(m); m.build(force=True)" > /dev/null 2>&1; }
for hs in 4 5 6 8; do
  build "-DFM_HI_STAGES=$hs"
  for i in 1 2; do
  python bench.py --steps 300 --warmup 10 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); a=d['stages_alone_ms']; print('hi_stages $hs fps', round(d['value']), 'ms', round(d['ms_per_step'],4), 'sub', round(a['subspace'],4))"
  done
done
