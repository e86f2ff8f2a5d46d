"""Precision sweep: GPU pipeline vs the fp64 oracle on many frames of one BASELINE config, for each setting
of an experiment switch (env var toggled between runs in one process; "-" = one run with the defaults).
Prints per setting: worst spectrum
dB error (within 40 dB of max), 99th percentile, frames whose peak cells differ."""
import json
import os as _os
for _v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
    _os.environ.setdefault(_v, "1")  # one BLAS thread per oracle worker (the pool uses every core)
import os
import sys
from concurrent.futures import ProcessPoolExecutor

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from oracle import fastmusic_oracle as O  # noqa: E402
from tests.gpu_helpers import run_gpu  # noqa: E402

CFG = None


def _ref(args):
    i, f, xi = args
    cfg = O.baseline_configs()[CFG]
    est, p_ref, pk = O.run_frame(cfg, xi, f, O.baseline_grid(cfg.grid_size))
    return i, p_ref, pk.cells


def main():
    global CFG
    import paper_1911_07434_b200 as fm
    CFG = sys.argv[1] if len(sys.argv) > 1 else "c2"
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 256
    f0 = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    var = sys.argv[4] if len(sys.argv) > 4 else "FM_RMUL_HI_ONLY"
    cfg = O.baseline_configs()[CFG]
    frames = list(range(f0, f0 + n))
    x, _, _ = O.generate_batch(cfg.base_seed, frames, cfg.spec)
    with ProcessPoolExecutor(max_workers=os.cpu_count()) as ex:
        refs = sorted(ex.map(_ref, [(i, f, x[i]) for i, f in enumerate(frames)], chunksize=4))
    for val in (("0", "1") if var != "-" else ("-",)):
        if var != "-":
            os.environ[var] = val
        res = run_gpu(fm, O, cfg, x, frames, basis=False)
        errs, mism = [], []
        for i, p_ref, cells in refs:
            errs.append(O.spectrum_db_error(res["spectrum"][i].astype(np.float64), p_ref))
            c = [int(v) for v in res["peak_cells"][i][: int(res["peak_count"][i])]]
            if c != cells:
                mism.append(frames[i])
        e = np.array(errs)
        print(json.dumps({"config": CFG, "frames": n, "f0": f0, var: val, "worst_db": float(e.max()),
                          "p99_db": float(np.percentile(e, 99)), "median_db": float(np.median(e)),
                          "peak_mismatch_frames": mism[:20], "n_mismatch": len(mism)}), flush=True)


if __name__ == "__main__":
    main()
