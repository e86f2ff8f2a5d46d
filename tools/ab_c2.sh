#!/bin/bash
# quick A/B of the c2 step: device stages (one batch at a time) and the default bench number
python tools/run_batches.py c2 3 >/dev/null 2>&1
python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --depth 1 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('depth1', round(d['value']), round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['stages_alone_ms'].items()})"
python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('default', round(d['value']), round(d['ms_per_step'],4), 'depth', d['batches_in_flight'])"
