import ctypes, sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import paper_1911_07434_b200 as fm
from paper_1911_07434_b200 import _capi
M, N, K, P, B = 256, 512, 8, 16, 1024
x, _, _ = fm.generate_frames(M, N, K, 2, 0, B)
seeds = np.array([fm.derive(fm.derive(2, f), 4) for f in range(B)], np.uint64)
om = torch.from_numpy(fm.draw_omega_batch(seeds, M, P)).cuda()
plan = fm.BatchPlan(M, N, K, "fast2", p=P, t=2, grid_size=3601, max_frames=B); plan.set_concurrency(1)
out = plan.outputs(B)
dbg = torch.zeros(B * 4, dtype=torch.int64, device="cuda")
lib = ctypes.CDLL(_capi.LIB_PATH); lib.fm_debug_set_peak_buffer(ctypes.c_void_p(dbg.data_ptr()))
for _ in range(2): plan.run(B, torch.from_numpy(x.view(np.float32)).cuda(), om, None, out)
torch.cuda.synchronize()
d = dbg.cpu().numpy().reshape(B, 4)
print("peaks phases (load, detect, greedy) cycles, nc: median", np.median(d, axis=0), "max", d.max(axis=0))
lib.fm_debug_set_peak_buffer(ctypes.c_void_p(0))
