#!/bin/bash
# Round-2 profile set: one-step launch list with DRAM bytes, and ncu --set full of the top kernels (each capture
# after its own command exited 0 without ncu). usage: tools/r02_profile.sh <tag>
tag=${1:-r02h}
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --depth 1 --graphs off"
$B > gpurun_out/${tag}_plain.log 2>&1; echo "plain rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -s 45 -c 40 --csv --log-file gpurun_out/${tag}_step_launches.csv $B > gpurun_out/${tag}_ncu_step.log 2>&1
echo "step ncu rc=$?"
for k in cov_tc_kernel rmul_planes_kernel k_spectrum_tc k_small_warp k_autocorr_fft k_peaks_rounds k_cholpiv_warp; do
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$k" -s 2 -c 1 -f -o gpurun_out/${tag}_${k} \
      python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --subbatches 1 --depth 1 --graphs off \
      > gpurun_out/ncu_${tag}_${k}.log 2>&1
  echo "ncu $k rc=$?"
done
