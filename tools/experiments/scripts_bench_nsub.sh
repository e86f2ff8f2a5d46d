#!/bin/bash
# ms/step and stage times at nsub = 1 and 4 (no e2e / cpu legs)
for ns in 1 4; do
  python bench.py --steps 50 --warmup 10 --no-e2e --no-cpu-baseline --subbatches $ns 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('nsub', $ns, round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['stages_ms_per_step'].items()})"
done
