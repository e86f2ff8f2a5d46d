"""Exact method (certified subspace iteration): residual/gap ratios on c5 frames + timing."""
import ctypes, os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import paper_1911_07434_b200 as fm
from paper_1911_07434_b200 import _capi
M, N, K, B = 256, 512, 8, 512
x, _, _ = fm.generate_frames(M, N, K, 2, 0, B, snr_lo_db=20.0, snr_hi_db=20.0)
xd = torch.from_numpy(x.view(np.float32)).cuda()
lib = ctypes.CDLL(_capi.LIB_PATH)
ratio = torch.zeros(B, dtype=torch.float64, device="cuda")
lib.fm_debug_set_exact_ratio_buffer(ctypes.c_void_p(ratio.data_ptr()))
plan = fm.BatchPlan(M, N, K, "exact", grid_size=3601, max_frames=B)
out = plan.outputs(B)
plan.run(B, xd, None, None, out)
torch.cuda.synchronize()
r = ratio.cpu().numpy()
print("ratio quantiles", np.quantile(r, [0, 0.5, 0.9, 0.99, 1.0]), "over tol 1e-3:", int((r > 1e-3).sum()))
t0 = time.perf_counter()
for _ in range(5):
    plan.run(B, xd, None, None, out)
torch.cuda.synchronize()
print("exact ms per 512 frames", (time.perf_counter() - t0) / 5 * 1e3, "status", np.unique(out["status"].cpu().numpy()))
lib.fm_debug_set_exact_ratio_buffer(ctypes.c_void_p(0))
# independent check of the certification on a few frames (numpy, fp64)
out2 = plan.outputs(B, basis=True, covariance=True)
lib.fm_debug_set_exact_ratio_buffer(ctypes.c_void_p(ratio.data_ptr()))
plan.run(B, xd, None, None, out2)
torch.cuda.synchronize()
lib.fm_debug_set_exact_ratio_buffer(ctypes.c_void_p(0))
r = ratio.cpu().numpy()
R = out2["covariance"].cpu().numpy(); R = R[..., 0] + 1j * R[..., 1]
b = out2["basis"].cpu().numpy(); U = (b[..., 0] + 1j * b[..., 1]).transpose(0, 2, 1)
lam = out2["eigenvalues"].cpu().numpy()
for f in [0, 1, 2, 3, 100, 300]:
    res = np.linalg.norm(R[f].astype(np.complex128) @ U[f] - U[f] * lam[f], axis=0).max()
    w = np.linalg.eigvalsh(R[f].astype(np.complex128))[::-1]
    print(f, "kernel ratio", r[f], "numpy residual", res, "gap", w[K - 1] - w[K], "lam", lam[f][:2], "eigvalsh", w[:2])
