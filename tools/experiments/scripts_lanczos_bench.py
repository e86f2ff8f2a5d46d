"""block_lanczos_subspace on BASELINE c2 frames (M=256, K=8, block=16): GPU fp64 facade (wall clock and the
CUDA-event cost_seconds) against the oracle restatement on one host core. Prints one JSON line."""
import json
import os
import sys
import time

import numpy as np

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import paper_1911_07434_b200 as fm  # noqa: E402
from oracle import fastmusic_oracle as O  # noqa: E402


def main():
    cfg = O.baseline_configs()["c2"]
    frames = list(range(8))
    x, _, _ = O.generate_batch(cfg.base_seed, frames, cfg.spec)
    covs = [O.spatial_covariance(x[i].astype(np.complex128)) for i in range(len(frames))]
    fm.block_lanczos_subspace(covs[0], 8, 16, 100)  # warm-up (context, module load)
    t0 = time.perf_counter()
    costs, errs = [], []
    for s in covs:
        est = fm.block_lanczos_subspace(s, 8, 16, 100)
        costs.append(est.cost_seconds)
    gpu_wall = (time.perf_counter() - t0) / len(covs)
    t0 = time.perf_counter()
    for s, c in zip(covs, costs):
        ref = O.block_lanczos_subspace(s, 8, 16, 100)
    cpu = (time.perf_counter() - t0) / len(covs)
    for s in covs[:2]:
        a = fm.block_lanczos_subspace(s, 8, 16, 100)
        b = O.block_lanczos_subspace(s, 8, 16, 100)
        errs.append(O.projector_error(a.basis, b.basis))
    print(json.dumps({"what": "block_lanczos_subspace c2 (M=256, K=8, block=16)", "frames": len(covs),
                      "gpu_wall_ms_per_call": gpu_wall * 1e3, "gpu_cost_ms_median": float(np.median(costs)) * 1e3,
                      "oracle_cpu_ms_per_call_1core": cpu * 1e3, "max_projector_err_vs_oracle": max(errs)}))


if __name__ == "__main__":
    main()
