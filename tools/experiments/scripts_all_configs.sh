#!/bin/bash
# one bench line per BASELINE config (short runs) + the reference arm
for c in c1 c2 c3 c4 c5 c3n; do
  case $c in c5) st=5;; c4) st=20;; *) st=50;; esac
  timeout 600 python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline > gpurun_out/cfg_$c.json 2> gpurun_out/cfg_$c.err
  echo "$c rc=$?"
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ref_c2.json 2> gpurun_out/ref_c2.err; echo "ref rc=$?"
