#!/bin/bash
# c2 ms/step vs covariance grid width (FM_COV_PAIRS) and sub-batch count: SMs left free for the other
# sub-batch's latency-bound kernels
for cp in 74 66 60 52; do for ns in 2 3 4; do
  FM_COV_PAIRS=$cp python bench.py --steps 100 --warmup 10 --no-e2e --no-cpu-baseline --subbatches $ns 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pairs', $cp, 'nsub', $ns, round(d['ms_per_step'],4), round(d['stages_alone_ms']['covariance'],4))"
done; done
