#!/bin/bash
# Bench lines of the other configs from the current build (short runs; CPU legs off except where noted).
for c in c1 c3 c3n c4 c5 c2lz toa; do
  timeout 600 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1
done
timeout 900 python bench.py --config c5 --exact-jacobi --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1
