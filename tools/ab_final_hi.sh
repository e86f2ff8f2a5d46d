#!/bin/bash
# Final (Nystrom-input) product on R's hi plane only (FM_FINAL_HI_ONLY=1): parity on c2 / c2 stress cases and the c2 step.
build() { FM_NVCC_FLAGS="$1" python -c "
import importlib.util
spec = importlib.util.spec_from_file_location('_b', 'paper_1911_07434_b200/build.py')
m = importlib.util.module_from_spec(spec); spec.loader.exec_module(m); m.build(force=True)" > /dev/null 2>&1; }
build "-DFM_FINAL_HI_ONLY=1"
timeout 900 python tools/parity_sweep.py c2 c2_persource30dB c2_persource40dB c2_scale2^-20 c4 > gpurun_out/final_hi_parity.jsonl 2> gpurun_out/final_hi_parity.err
echo parity rc=$?
python -c "
import json
for l in open('gpurun_out/final_hi_parity.jsonl'):
    d=json.loads(l); print(d['case'], 'worst', round(d['worst_db'],5), 'p99', round(d['p99_db'],5), 'mism', d['n_mismatch'], 'status', d['status_values'])"
python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); a=d['stages_alone_ms']; print('c2', round(d['value']), round(d['ms_per_step'],4), a)"
build ""
