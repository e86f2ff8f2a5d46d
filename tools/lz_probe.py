"""Batched block-Lanczos probe: time fm_block_lanczos_batch on c2 covariances (from the plan's export) and print
the Krylov-iteration / Jacobi-sweep statistics. Usage: python tools/lz_probe.py [frames]"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1911_07434_b200 as fm  # noqa: E402


def main():
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    M, N, K = 256, 512, 8
    x = np.empty((B, M, N), np.complex64)
    fm.generate_frames(M, N, K, 2, 0, B, out=x, theta_lo_deg=-60.0, theta_hi_deg=60.0, min_sep_deg=3.0,
                       snr_lo_db=10.0, snr_hi_db=30.0)
    xd = torch.from_numpy(x.view(np.float32)).cuda()
    plan = fm.BatchPlan(M, N, K, "lanczos", p=0, t=200, grid_size=3601, max_frames=B)
    out = plan.outputs(B, spectrum=False, covariance=True)
    plan.run(B, xd, None, None, out)
    torch.cuda.synchronize()
    r = out["covariance"]
    for _ in range(2):
        fm.block_lanczos_batch(torch.view_as_complex(r), K, K, 200)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    b, e, st, it = fm.block_lanczos_batch(torch.view_as_complex(r), K, K, 200)
    e1.record()
    torch.cuda.synchronize()
    it = it.cpu().numpy()
    print(json.dumps({"frames": B, "ms": e0.elapsed_time(e1), "status_ok": int((st.cpu().numpy() == 0).sum()),
                      "krylov_iters": np.bincount(it // 10000).tolist(),
                      "sweeps_mean": float((it % 10000).mean()), "sweeps_max": int((it % 10000).max())}))


if __name__ == "__main__":
    main()
