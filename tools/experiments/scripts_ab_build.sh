#!/bin/bash
# A/B two builds in one GPU session: scripts_ab_build.sh "<nvcc flags A>" "<nvcc flags B>" [kernel regex]
kr=${3:-rmul_planes}
for fl in "$1" "$2"; do
  FM_NVCC_FLAGS="$fl" python -c "import sys; sys.path.insert(0,'.'); from paper_1911_07434_b200 import build; build.build(force=True)" > /dev/null 2>&1
  python bench.py --steps 300 --warmup 10 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('[$fl]', round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['stages_alone_ms'].items()})"
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:$kr -c 6 --csv --log-file gpurun_out/ll_ab.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --subbatches 1 > /dev/null 2>&1
  python tools/launch_summary.py gpurun_out/ll_ab.csv
done
