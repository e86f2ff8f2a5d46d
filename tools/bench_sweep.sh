#!/bin/bash
# Shard-size / batches-in-flight / graph sweep at N = 1 (proxies for the strong split at N = 2, 4, 8: 512, 256, 128
# frames per GPU). One line per setting.
for fr in ${FRAMES:-128 256 512 1024}; do
  for dp in ${DEPTHS:-1 2 3 4}; do
    for gr in ${GRAPHS:-off on}; do
      python bench.py --frames $fr --depth $dp --graphs $gr --steps ${STEPS:-100} --warmup 10 --no-e2e --no-cpu-baseline 2>/dev/null |
        python -c "import json,sys;d=json.loads(sys.stdin.read());print('frames',$fr,'depth',$dp,'graphs','$gr','fps',round(d['value']),'ms',round(d['ms_per_step'],4))"
    done
  done
done
