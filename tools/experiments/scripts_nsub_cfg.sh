#!/bin/bash
# ms/step with 1 vs 2 concurrent sub-batches for the batched configs
for c in c2 c3 c5 c3n; do for ns in 1 2; do
  python bench.py --config $c --steps 100 --warmup 10 --no-e2e --no-cpu-baseline --subbatches $ns 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c nsub $ns', round(d['ms_per_step'],4))"
done; done
