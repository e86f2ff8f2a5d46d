#!/bin/bash
# p = 32 eigen-work: two warps per frame (default) vs one (FM_SMALL_ONE_WARP=1), configs c3 / c3n / c4
for c in c3 c3n c4; do
  case $c in c4) st=20;; *) st=100;; esac
  for env in "FM_X=0" "FM_SMALL_ONE_WARP=1"; do
    env $env python bench.py --config $c --steps $st --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c $env', round(d['ms_per_step'],4), round(d['value']), {k: round(v,4) for k,v in d['stages_alone_ms'].items()})"
  done
done
