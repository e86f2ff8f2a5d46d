#!/bin/bash
# covariance kernel time (stages_alone, one launch per batch) vs TMA / operand ring depths (FM_COV_RING)
for r in 3,3,6,6 4,2,6,6 4,2,8,4 3,3,8,4; do
  for c in c2 c4; do
    FM_COV_RING=$r python bench.py --config $c --no-cpu-baseline --no-e2e --steps 20 --roof-steps 10 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('ring $r $c', round(d['ms_per_step'],4), 'cov_alone', round(d['stages_alone_ms']['covariance'],4))"
  done
done
