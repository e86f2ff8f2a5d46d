#!/bin/bash
# One-step launch lists (depth 1, stream launches) of the other configs.
for c in "$@"; do
  B="python bench.py --config $c --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --depth 1 --graphs off"
  $B > gpurun_out/cfgl_${c}_plain.log 2>&1 || { echo "$c plain failed"; continue; }
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      -s 40 -c 60 --csv --log-file gpurun_out/cfgl_${c}_launches.csv $B > gpurun_out/cfgl_${c}_ncu.log 2>&1
  echo "$c ncu rc=$?"
done
