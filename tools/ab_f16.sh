#!/bin/bash
# c4 covariance from fp16 planes: step time, stage time, launch list of one step, c4 parity.
python bench.py --config c4 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); a=d['stages_alone_ms']; print('c4', round(d['value']), round(d['ms_per_step'],3), 'cov', round(a['covariance'],3))"
echo rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/c4f16b_launches.csv \
  python bench.py --config c4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/c4f16b_launches.csv')) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
for r in rows[1:]:
    if 'cov' in r[ki] or 'planes' in r[ki] or 'rescue' in r[ki]: print(r[ki][:60], r[vi])
PY
timeout 600 python tools/parity_sweep.py c4 c4_persource30dB 2>&1 | cut -c1-200 | tail -3
