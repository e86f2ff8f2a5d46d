build() { FM_NVCC_FLAGS="$1" python -c "
import importlib.util
spec = importlib.util.spec_from_file_location('_b', 'paper_1911_07434_b200/build.py')
m = importlib.util.module_from_spec(spec); spec.loader.exec_module(m); m.build(force=True)" > /dev/null 2>&1; }
for v in 0 6 12 20; do
  build "-DFM_RESERVE_PAIRS=$v"
  for d in 3 5; do
  python bench.py --steps 300 --warmup 10 --no-e2e --no-cpu-baseline --depth $d 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); a=d['stages_alone_ms']; print('reserve $v depth $d fps', round(d['value']), 'ms', round(d['ms_per_step'],4), 'cov', round(a['covariance'],4), 'sub', round(a['subspace'],4))"
  done
done
