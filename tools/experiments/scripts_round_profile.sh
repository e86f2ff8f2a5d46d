#!/bin/bash
# Full bench line + launch list + ncu --set full of the dominant kernels (each after a clean run).
# usage: scripts_round_profile.sh <tag>
tag=$1
python bench.py > gpurun_out/bench_${tag}.json 2> gpurun_out/bench_${tag}.err; echo "bench rc=$?"
./scripts_ncu_list.sh gpurun_out/launches_${tag}.csv --subbatches 1
for k in cov_tc_kernel rmul_planes_kernel k_spectrum_i8 k_small_warp k_peaks_rounds k_autocorr_fft; do
  ncu --set full --clock-control none --import-source on -k "regex:$k" -s 1 -c 1 -f -o gpurun_out/${tag}_${k} \
      python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --subbatches 1 > gpurun_out/ncu_${tag}_${k}.log 2>&1
  echo "ncu $k rc=$?"
done
