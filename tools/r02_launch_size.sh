#!/bin/bash
# Does a larger launch (more frames per kernel launch) raise c2 throughput at N = 1?  1024 frames per global batch,
# coalesce 1 / 2 / 4 consecutive batches per launch, depth 2 / 3.
line() { python bench.py --steps 240 --warmup 12 --no-e2e --no-cpu-baseline "$@" 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('frames/s', round(d['value']), 'ms/batch', round(d['ms_per_step'],4), 'coalesce', d['config'].get('coalesce'), 'depth', d['batches_in_flight'], 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'])"; }
for co in 1 2 4 1 2; do
  for dp in 2 3; do echo -n "coalesce $co depth $dp: "; line --coalesce $co --depth $dp; done
done
