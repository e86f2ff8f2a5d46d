#!/bin/bash
# usage: scripts_ncu_list.sh <out.csv> [bench args]  -- per-launch device times of one bench step
out=$1; shift
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline "$@" > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 45 -c 15 --csv --log-file "$out" \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline "$@" > gpurun_out/ncu.log 2>&1
echo "ncu rc=$?"
