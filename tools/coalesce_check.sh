#!/bin/bash
# Per-GPU throughput of strong-scaling shards (1024 / G frames per global batch) with and without shard coalescing,
# measured on one GPU (no inter-rank waits involved): G = 8 -> 128-frame shards, G = 4 -> 256, G = 2 -> 512.
line() { python bench.py --steps 240 --warmup 10 --no-e2e --no-cpu-baseline "$@" 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('frames/s', round(d['value']), 'ms/batch', round(d['ms_per_step'],4), 'coalesce', d['config']['coalesce'], 'depth', d['batches_in_flight'], 'clk', d['clocks']['sm_mhz'])"; }
for fr in 128 256 512; do
  for co in 1 0; do echo -n "shard $fr coalesce-arg $co: "; line --frames $fr --coalesce $co; done
done
