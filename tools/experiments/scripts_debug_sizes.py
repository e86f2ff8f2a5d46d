import os, sys, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import paper_1911_07434_b200 as fm
M, N, K, P = 256, 512, 8, 16
for arg in sys.argv[1:]:
    f0, B = [int(v) for v in arg.split(":")]
    x, _, _ = fm.generate_frames(M, N, K, 2, f0, B)
    seeds = np.array([fm.derive(fm.derive(2, f0 + f), 4) for f in range(B)], np.uint64)
    om = torch.from_numpy(fm.draw_omega_batch(seeds, M, P)).cuda()
    xd = torch.from_numpy(x.view(np.float32)).cuda()
    plan = fm.BatchPlan(M, N, K, "fast2", p=P, t=2, grid_size=3601, max_frames=B)
    out = plan.outputs(B)
    torch.cuda.synchronize()
    try:
        plan.run(B, xd, om, None, out)
        torch.cuda.synchronize()
        st = out["status"].cpu().numpy()
        print(arg, "ok", np.unique(st, return_counts=True), flush=True)
    except Exception as e:
        print(arg, "FAIL", e, flush=True)
        break
    plan.close()
