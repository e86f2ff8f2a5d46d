#!/bin/bash
# c2 covariance time vs the single-tile ring split (FM_COV_RING=gS,gO,dS,dO; 16 KB per staging stage, 8 KB per
# operand stage, 160 KB in all) with four converter warps
for r in 4,2,8,4 4,2,9,2 4,2,7,6 4,2,6,8 4,2,5,10; do
  FM_COV_RING=$r python bench.py --config c2 --no-cpu-baseline --no-e2e --steps 100 --roof-steps 10 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('ring $r', round(d['ms_per_step'],4), 'cov_alone', round(d['stages_alone_ms']['covariance'],4))"
done
