#!/bin/bash
# Threads per frame of the long-grid peak picking (FM_PEAKS_LONG_NT, L > 8192): c4 step and stage times.
build() { FM_NVCC_FLAGS="$1" python -c "
import importlib.util
spec = importlib.util.spec_from_file_location('_b', 'paper_1911_07434_b200/build.py')
m = importlib.util.module_from_spec(spec); spec.loader.exec_module(m); m.build(force=True)" > /dev/null 2>&1; }
for nt in 128 256 512 1024; do
  build "-DFM_PEAKS_LONG_NT=$nt"
  python bench.py --config c4 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); a=d['stages_alone_ms']; print('nt $nt fps', round(d['value']), 'ms', round(d['ms_per_step'],3), 'spec_peaks', round(a['spectrum_peaks'],4))"
done
