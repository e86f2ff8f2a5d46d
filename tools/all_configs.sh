#!/bin/bash
# One bench line per config (device-resident value, e2e, covariance roofline; CPU legs skipped) -> one JSONL file.
# usage: tools/all_configs.sh <out.jsonl>
out=${1:-gpurun_out/all_configs.jsonl}
: > $out
for c in c1 c2 c3 c4 c5 c3n c2lz toa; do
  case $c in c4) st=20;; c2lz) st=10;; *) st=100;; esac
  timeout 900 python bench.py --config $c --steps $st --warmup 5 --no-cpu-baseline 2> gpurun_out/cfg_$c.err | tail -1 >> $out
  echo "$c rc=$?"
done
