"""Gram warps of the plane product kernel at c2: per-frame wait at the tile-full barrier and Gram compute cycles
(CTA 0, last product launch of a run)."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import paper_1911_07434_b200 as fm  # noqa: E402
from paper_1911_07434_b200 import _capi  # noqa: E402

M, N, K, P, B = 256, 512, 8, 16, 1024
x, _, _ = fm.generate_frames(M, N, K, 2, 0, B)
seeds = np.array([fm.derive(fm.derive(2, f), 4) for f in range(B)], np.uint64)
om = torch.from_numpy(fm.draw_omega_batch(seeds, M, P)).cuda()
xd = torch.from_numpy(x.view(np.float32)).cuda()
dbg = torch.zeros(64, dtype=torch.int64, device="cuda")
lib = ctypes.CDLL(_capi.LIB_PATH)
lib.fm_debug_set_gram_buffer(ctypes.c_void_p(dbg.data_ptr()))
plan = fm.BatchPlan(M, N, K, "fast2", p=P, t=2, grid_size=3601, max_frames=B)
plan.set_concurrency(1)
out = plan.outputs(B)
for _ in range(2):
    plan.run(B, xd, om, None, out)
torch.cuda.synchronize()
d = dbg.cpu().numpy().reshape(32, 2)[:14]
print("per frame (wait, gram) cycles:", d.tolist())
lib.fm_debug_set_gram_buffer(ctypes.c_void_p(0))
