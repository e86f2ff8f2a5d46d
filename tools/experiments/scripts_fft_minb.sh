#!/bin/bash
# k_autocorr_fft time vs its minimum-blocks-per-SM launch bound (register cap)
for nb in 2 3 4; do
  FM_NVCC_FLAGS="-DFM_FFT_MINB=$nb" python -c "import sys; sys.path.insert(0,'.'); from paper_1911_07434_b200 import build; build.build(force=True)" > /dev/null 2>&1
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_autocorr -c 2 --csv --log-file gpurun_out/ll_fft$nb.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --subbatches 1 > /dev/null 2>&1
  python tools/launch_summary.py gpurun_out/ll_fft$nb.csv | head -1 | sed "s/^/minb $nb: /"
done
