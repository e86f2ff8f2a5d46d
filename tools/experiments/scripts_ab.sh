#!/bin/bash
# A/B: c2 ms/step with the default build vs an env switch. usage: scripts_ab.sh "ENV=1" [steps]
st=${2:-300}
for env in "FM_X=0" "$1"; do
  env $env python bench.py --steps $st --warmup 10 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$env', round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['stages_alone_ms'].items()})"
done
