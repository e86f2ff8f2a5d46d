#!/bin/bash
# HEAD profile refresh: one-step launch list with DRAM bytes (depth 1, stream launches) and the launch list of the
# default pipelined command (depth 3), each after the same command exited 0 without ncu.
tag=${1:-r02z}
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --depth 1 --graphs off"
$B > gpurun_out/${tag}_plain.log 2>&1; echo "plain rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -s 45 -c 40 --csv --log-file gpurun_out/${tag}_step_launches.csv $B > gpurun_out/${tag}_ncu_step.log 2>&1
echo "step ncu rc=$?"
D="python bench.py --steps 6 --warmup 3 --no-e2e --no-cpu-baseline"
$D > gpurun_out/${tag}_plain_default.log 2>&1; echo "plain default rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/${tag}_default_launches.csv $D > gpurun_out/${tag}_ncu_default.log 2>&1
echo "default ncu rc=$?"
