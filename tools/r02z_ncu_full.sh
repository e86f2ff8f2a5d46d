#!/bin/bash
# ncu --set full of the final kernels (one launch each over 1024 c2 frames), after the same command ran clean.
tag=${1:-r02z}
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --subbatches 1 --depth 1 --graphs off"
$B > gpurun_out/${tag}_full_plain.log 2>&1; echo "plain rc=$?"
for k in cov_tc_kernel rmul_planes_kernel k_small_warp k_spectrum_tc; do
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$k" -s 2 -c 1 -f -o gpurun_out/${tag}_${k} \
      $B > gpurun_out/ncu_${tag}_${k}.log 2>&1
  echo "ncu $k rc=$?"
done
