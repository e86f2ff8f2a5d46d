import os, sys, ctypes, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import paper_1911_07434_b200 as fm
from paper_1911_07434_b200 import _capi
M, N, K, P = 256, 512, 8, 32
B = 148 * 3
x, _, _ = fm.generate_frames(M, N, K, 2, 0, B)
seeds = np.array([fm.derive(fm.derive(2, f), 3) for f in range(B)], np.uint64)
ix = torch.from_numpy(fm.draw_indices_batch(seeds, M, P)).cuda()
xd = torch.from_numpy(x.view(np.float32)).cuda()
dbg = torch.zeros(B * 4, dtype=torch.int32, device="cuda")
lib = ctypes.CDLL(_capi.LIB_PATH); lib.fm_debug_set_phase_buffer(ctypes.c_void_p(dbg.data_ptr()))
plan = fm.BatchPlan(M, N, K, "fast1", p=P, grid_size=3601, max_frames=B); plan.set_concurrency(1)
out = plan.outputs(B)
for _ in range(2): plan.run(B, xd, None, ix, out)
torch.cuda.synchronize()
d = dbg.cpu().numpy().reshape(B, 4)
print("p=32 small_warp phases (chol+Y, jacobi, T) cycles + sweeps: median", np.median(d, axis=0), "max", d.max(axis=0))
lib.fm_debug_set_phase_buffer(ctypes.c_void_p(0))
