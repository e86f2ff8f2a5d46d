#!/bin/bash
# c2 ms/step with the Gram epilogue (default) vs the separate Gram kernels (FM_NO_GRAM_EPI=1)
for env in "FM_X=0" "FM_NO_GRAM_EPI=1"; do
  env $env python bench.py --steps 200 --warmup 10 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$env', round(d['ms_per_step'],4), d['stages_alone_ms'], d.get('parity_sample'))"
done
