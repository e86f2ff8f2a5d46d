#!/bin/bash
for c in c3 c4; do
  for v in 0 1; do
    if [ $v = 1 ]; then export FM_FUSED_FINAL=1; else unset FM_FUSED_FINAL; fi
    timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c fused=$v', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stages_alone_ms'].items()})"
  done
done
