build() { FM_NVCC_FLAGS="$1" python -c "
import importlib.util
spec = importlib.util.spec_from_file_location('_b', 'paper_1911_07434_b200/build.py')
m = importlib.util.module_from_spec(spec); spec.loader.exec_module(m); m.build(force=True)" > /dev/null 2>&1; }
for v in "" "-DFM_COV_SPLIT_GEN"; do
  build "$v"
  for i in 1 2; do echo "[$v]"; python tools/temporal_bench.py; done
  python bench.py --config c4 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); a=d['stages_alone_ms']; print('c4', round(d['value']), 'ms', round(d['ms_per_step'],3), 'cov', round(a['covariance'],3))"
done
FM_NVCC_FLAGS=-DFM_COV_SPLIT_GEN timeout 600 python -m pytest tests/test_gpu_temporal.py tests/test_gpu_toa.py -x -q 2>&1 | tail -1
