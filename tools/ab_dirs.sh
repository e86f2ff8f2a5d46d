#!/bin/bash
# A/B of two source trees on one box: ab_variants/A (a previous commit, built) vs the working tree.
# usage: tools/ab_dirs.sh [runs] [extra bench args]
runs=${1:-3}; shift
root=$(pwd)
line() { python bench.py --steps 300 --warmup 10 --no-e2e --no-cpu-baseline "$@" 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); a=d['stages_alone_ms']
print('fps', round(d['value']), 'ms', round(d['ms_per_step'],4), 'clk', d['clocks']['sm_mhz'], {k: round(v,4) for k,v in a.items()})"; }
for i in $(seq $runs); do
  echo -n "A "; (cd ab_variants/A && line "$@")
  echo -n "B "; (cd "$root" && line "$@")
done
