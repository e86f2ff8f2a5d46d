#!/bin/bash
# GPU check of the current tree: gpu tests, smoke, default bench line, one-step launch list.
# usage: tools/r02_gpu_check.sh <tag>
tag=${1:-r02}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_gputest.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo "bench rc=$?"
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --depth 1 --graphs off > gpurun_out/${tag}_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 45 -c 20 --csv --log-file gpurun_out/${tag}_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --depth 1 --graphs off > gpurun_out/${tag}_ncu.log 2>&1
echo "ncu rc=$?"
