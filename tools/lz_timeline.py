"""Per-phase clock64 totals of block 0 of the batched block-Lanczos kernel (library built with
FM_NVCC_FLAGS=-DFM_LZ_TIMELINE): W = S Q, strip, extend + copy, tridiagonalise, bisection, Gram-Schmidt passes,
orthonormal_range, final Jacobi. python tools/lz_timeline.py"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1911_07434_b200 as fm  # noqa: E402

lib = ctypes.CDLL(os.path.join(ROOT, "paper_1911_07434_b200", "libfastmusic_b200.so"))
M, N, K, B = 256, 512, 8, 148
x = np.empty((B, M, N), np.complex64)
fm.generate_frames(M, N, K, 2, 0, B, out=x, theta_lo_deg=-60.0, theta_hi_deg=60.0, min_sep_deg=3.0,
                   snr_lo_db=10.0, snr_hi_db=30.0)
plan = fm.BatchPlan(M, N, K, "lanczos", p=0, t=200, grid_size=3601, max_frames=B)
out = plan.outputs(B, spectrum=False, covariance=True)
plan.run(B, torch.from_numpy(x.view(np.float32)).cuda(), None, None, out)
torch.cuda.synchronize()
r = torch.view_as_complex(out["covariance"])
lib.fm_debug_lz_timeline(None, 1)
b, e, st, it = fm.block_lanczos_batch(r, K, K, 200)
torch.cuda.synchronize()
buf = (ctypes.c_longlong * 16)()
lib.fm_debug_lz_timeline(buf, 0)
names = ["W=SQ", "strip", "extend+copy", "tridiag", "bisect", "gram-schmidt", "orth_range", "final_jacobi", "exit"]
tot = sum(buf[i] for i in range(9))
print("frame 0 iterations", int(it[0].item()) // 10000, "total cycles", tot)
for i, n in enumerate(names):
    print(f"{n:14s} {buf[i]:10d}  {100.0 * buf[i] / max(tot, 1):5.1f} %")
