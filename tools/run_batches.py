"""Run `batches` back-to-back fm_run_batch calls of a BASELINE config on one stream (one batch in flight):
the workload for ncu launch lists (`ncu --metrics gpu__time_duration.sum -s <skip> -c <count>`) and captures.
  python tools/run_batches.py [config] [batches] [frames]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1911_07434_b200 as fm  # noqa: E402
from bench import CONFIGS  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
batches = int(sys.argv[2]) if len(sys.argv) > 2 else 3
c = dict(CONFIGS[name])
B = int(sys.argv[3]) if len(sys.argv) > 3 else c["frames"]
M, N, K, P, L = c["m"], c["n"], c["k"], c["p"], c["L"]
x = np.empty((B, M, N), np.complex64)
fm.generate_frames(M, N, K, c["seed"], 0, B, out=x, **c["scene"])
seeds = np.array([fm.derive(fm.derive(c["seed"], f), 4 if c["method"] == "fast2" else 3) for f in range(B)], np.uint64)
om = torch.from_numpy(fm.draw_omega_batch(seeds, M, P)).cuda() if c["method"] == "fast2" else None
ix = torch.from_numpy(fm.draw_indices_batch(seeds, M, P)).cuda() if c["method"] == "fast1" else None
if c["method"] == "fast1_norm2":
    om = torch.from_numpy(fm.draw_uniforms_batch(seeds, M)).cuda()
xd = torch.from_numpy(x.view(np.float32)).cuda()
plan = fm.BatchPlan(M, N, K, c["method"], p=P, t=c["t"], grid_size=L, max_frames=B)
out = plan.outputs(B, spectrum=True)
s = torch.cuda.Stream()
for _ in range(batches):
    plan.run(B, xd, om, ix, out, stream=s)
torch.cuda.synchronize()
print("launches per batch", plan.launches_per_batch(), "status nonzero", int((out["status"] != 0).sum()))
