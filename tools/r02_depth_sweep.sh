#!/bin/bash
# Batches in flight at 1024 frames per launch (default 3): is a deeper pipeline worth its memory?
line() { python bench.py --steps 300 --warmup 12 --no-e2e --no-cpu-baseline "$@" 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('frames/s', round(d['value']), 'ms/batch', round(d['ms_per_step'],4), 'depth', d['batches_in_flight'], 'graphs', d['cuda_graphs'], 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'])"; }
for rep in 1 2; do
  for dp in 3 4 5 6; do echo -n "depth $dp: "; line --depth $dp; done
  echo -n "depth 3 graphs on: "; line --depth 3 --graphs on
  echo -n "depth 4 graphs on: "; line --depth 4 --graphs on
done
