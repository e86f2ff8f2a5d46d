"""A/B the host path's chunk count on one box: c2 shape, 1024 frames from pinned host memory."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import paper_1911_07434_b200 as fm  # noqa: E402

B, M, N, K, P = 1024, 256, 512, 8, 16
x = torch.empty((B, M, N), dtype=torch.complex64).pin_memory()
xn = x.numpy()
fm.generate_frames(M, N, K, 5, 0, B, out=xn)
seeds = np.array([fm.derive(9, f) for f in range(B)], np.uint64)
plan = fm.BatchPlan(M, N, K, "fast2", p=P, t=2, grid_size=3601, max_frames=B)
# pure copy speed for reference
xd = torch.empty((B, M, N), dtype=torch.complex64, device="cuda")
for _ in range(2):
    xd.copy_(x, non_blocking=True)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5):
    xd.copy_(x, non_blocking=True)
torch.cuda.synchronize()
print(f"plain H2D {xn.nbytes * 5 / (time.perf_counter() - t0) / 1e9:.1f} GB/s")
for rnd in range(2):
    for ch in ["1", "2", "4", "8"]:
        os.environ["FM_HOST_CHUNKS"] = ch
        plan.estimate_host(xn, seeds)
        t0 = time.perf_counter()
        for _ in range(5):
            plan.estimate_host(xn, seeds)
        el = (time.perf_counter() - t0) / 5
        print(f"round {rnd} chunks {ch}: {el * 1e3:.2f} ms/step  {B / el:.0f} frames/s")
