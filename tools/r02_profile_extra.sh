#!/bin/bash
# Extra round-2 evidence: c2 one-step launch list with DRAM bytes (final kernels), ncu --set full of the temporal-mode
# covariance and the half-mode spectrum (ToA config) and of the batched block-Lanczos kernel.
tag=${1:-r02q}
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --depth 1 --graphs off"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -s 45 -c 40 --csv --log-file gpurun_out/${tag}_step_launches.csv $B > /dev/null 2>&1; echo "step rc=$?"
T="python bench.py --config toa --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --depth 1 --graphs off --subbatches 1"
for k in cov_tc_kernel k_spectrum_tc rmul_tc_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$k" -s 1 -c 1 -f -o gpurun_out/${tag}_toa_${k} $T > /dev/null 2>&1
  echo "toa $k rc=$?"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_lanczos_batch -c 1 -f -o gpurun_out/${tag}_lanczos python tools/lz_probe.py 296 > /dev/null 2>&1
echo "lanczos rc=$?"
