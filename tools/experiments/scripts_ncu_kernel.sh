#!/bin/bash
# usage: scripts_ncu_kernel.sh <kernel-regex> <out-name> [bench args]: ncu --set full of one launch (after a clean run)
k=$1; o=$2; shift 2
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline "$@" > gpurun_out/plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --set full --clock-control none --import-source on -k "regex:$k" -s 1 -c 1 -f -o "gpurun_out/$o" \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline "$@" > gpurun_out/ncu_$o.log 2>&1
echo "ncu rc=$?"
