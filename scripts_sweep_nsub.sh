#!/bin/bash
for n in 1 2 4 8; do
  python bench.py --steps 100 --warmup 10 --no-cpu-baseline --no-e2e --subbatches $n 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($n, round(d['value']), round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['stages_ms_per_step'].items()})"
done
