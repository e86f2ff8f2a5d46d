import numpy as np, torch, sys
sys.path.insert(0, "/root/repo")
import paper_1911_07434_b200 as fm
M, N, K, P, B = 256, 512, 8, 16, 64
x, _, _ = fm.generate_frames(M, N, K, 2, 0, B)
seeds = np.array([fm.derive(fm.derive(2, f), 4) for f in range(B)], np.uint64)
om = torch.from_numpy(fm.draw_omega_batch(seeds, M, P)).cuda()
plan = fm.BatchPlan(M, N, K, "fast2", p=P, t=2, grid_size=3601, max_frames=B)
out = plan.outputs(B)
plan.run(B, torch.from_numpy(x.view(np.float32)).cuda(), om, None, out)
s = out["spectrum"].cpu().numpy().astype(np.float64)
nc = [int(((v[1:-1] > v[:-2]) & (v[1:-1] > v[2:])).sum()) for v in s]
print("local maxima per frame: min/median/max", min(nc), int(np.median(nc)), max(nc))
