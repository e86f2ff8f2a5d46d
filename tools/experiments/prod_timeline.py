"""Per-tile timeline of CTA 0 of a range-finder product kernel (debug hook fm_debug_set_prod_buffer):
slots 0 producer first-stage issue, 1 MMA accumulator acquired, 2 MMA last commit, 3 epilogue acc ready,
4 epilogue Gram-tile free, 5 epilogue tile handed over. sel = LO + 2 GM (1: G+hi, 2: ... )."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1911_07434_b200 as fm  # noqa: E402
from paper_1911_07434_b200._capi import LIB  # noqa: E402
from bench import CONFIGS  # noqa: E402

sel = int(sys.argv[1]) if len(sys.argv) > 1 else 2
c = CONFIGS["c2"]
B, M, N, K, P, L = c["frames"], c["m"], c["n"], c["k"], c["p"], c["L"]
x = np.empty((B, M, N), np.complex64)
fm.generate_frames(M, N, K, c["seed"], 0, B, out=x, **c["scene"])
seeds = np.array([fm.derive(fm.derive(c["seed"], f), 4) for f in range(B)], np.uint64)
om = torch.from_numpy(fm.draw_omega_batch(seeds, M, P)).cuda()
xd = torch.from_numpy(x.view(np.float32)).cuda()
plan = fm.BatchPlan(M, N, K, "fast2", p=P, t=c["t"], grid_size=L, max_frames=B)
out = plan.outputs(B, spectrum=True)
plan.run(B, xd, om, None, out)
dbg = torch.zeros(8 * 64, dtype=torch.int64, device="cuda")
LIB.fm_debug_set_prod_buffer.argtypes = [C.c_void_p, C.c_int32]
LIB.fm_debug_set_prod_buffer(dbg.data_ptr(), sel)
plan.run(B, xd, om, None, out)
torch.cuda.synchronize()
LIB.fm_debug_set_prod_buffer(None, -1)
d = dbg.cpu().numpy().reshape(64, 8)
t0 = d[0, 0]
for t in range(16):
    r = d[t]
    if r[1] == 0:
        break
    print(t, " ".join(f"{(v - t0) / 1000:7.2f}" if v else "      -" for v in r[:6]),
          f" | mma {(r[2] - r[1]) / 1000:5.2f}k  epi {(r[5] - r[3]) / 1000:5.2f}k  gram-wait {(r[4] - r[3]) / 1000:5.2f}k")

# Gram warp 0 of CTA 0: (wait for the tile, compute) cycles per frame
g = torch.zeros(2 * 64, dtype=torch.int64, device="cuda")
LIB.fm_debug_set_gram_buffer.argtypes = [C.c_void_p]
LIB.fm_debug_set_gram_buffer(g.data_ptr())
plan.run(B, xd, om, None, out)
torch.cuda.synchronize()
LIB.fm_debug_set_gram_buffer(None)
gg = g.cpu().numpy().reshape(64, 2)
print("gram (last product launch) wait/compute k-cycles:", [(round(a / 1000, 1), round(b / 1000, 1)) for a, b in gg[:14]])
