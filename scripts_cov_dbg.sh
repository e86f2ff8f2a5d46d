#!/bin/bash
# covariance-stage time (sub-batch = whole batch) under the FM_COV_DBG experiment switches
A="--steps 20 --warmup 5 --no-e2e --no-cpu-baseline --subbatches 1"
for d in 0 1 2 4 5 3 7; do
  FM_NO_FUSE_C0=1 FM_COV_DBG=$d python bench.py $A 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('dbg=$d cov_ms', round(d['stages_ms_per_step']['covariance'],4))"
done
