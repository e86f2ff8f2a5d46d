#!/bin/bash
# ms/step of c2 vs number of concurrent sub-batches
for ns in 1 2 3 4 6 8; do
  python bench.py --steps 100 --warmup 10 --no-e2e --no-cpu-baseline --subbatches $ns 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('nsub', $ns, round(d['ms_per_step'],4))"
done
