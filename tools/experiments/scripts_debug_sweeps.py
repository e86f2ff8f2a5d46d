import os, sys, ctypes, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import paper_1911_07434_b200 as fm
from paper_1911_07434_b200 import _capi
M, N, K, P, B = 256, 512, 8, 16, 256
x, _, _ = fm.generate_frames(M, N, K, 2, 0, B)
seeds = np.array([fm.derive(fm.derive(2, f), 4) for f in range(B)], np.uint64)
om = torch.from_numpy(fm.draw_omega_batch(seeds, M, P)).cuda()
xd = torch.from_numpy(x.view(np.float32)).cuda()
dbg = torch.zeros(B, dtype=torch.int32, device="cuda")
lib = ctypes.CDLL(_capi.LIB_PATH); lib.fm_debug_set_sweep_buffer(ctypes.c_void_p(dbg.data_ptr()))
plan = fm.BatchPlan(M, N, K, "fast2", p=P, t=2, grid_size=3601, max_frames=B)
out = plan.outputs(B)
plan.run(B, xd, om, None, out); torch.cuda.synchronize()
d = dbg.cpu().numpy()
print("sweeps", np.bincount(d))
