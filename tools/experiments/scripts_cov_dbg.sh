#!/bin/bash
# covariance kernel time (whole batch, one launch) under the FM_COV_DBG experiment switches
A="--steps 20 --warmup 5 --no-e2e --no-cpu-baseline --subbatches 1"
for d in 0 2 4 6; do
  FM_COV_DBG=$d python bench.py $A 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('dbg=$d cov_ms', round(d['stages_alone_ms']['covariance'],4))"
done
