#!/bin/bash
# c2 ms/step vs persistent tensor-core kernel width (FM_TC_PAIRS) and sub-batches
for pairs in 74 66 60 52; do
  for ns in 1 2 3; do
    FM_TC_PAIRS=$pairs python bench.py --steps 60 --warmup 5 --no-e2e --no-cpu-baseline --subbatches $ns 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pairs', $pairs, 'nsub', $ns, round(d['ms_per_step'],4))"
  done
done
