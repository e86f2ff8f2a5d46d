import os, sys
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_1911_07434_b200 as fm
from oracle import fastmusic_oracle as O
cfg = O.baseline_configs()["c2"]
x, _, _ = O.generate_batch(cfg.base_seed, [0], cfg.spec)
s = O.spatial_covariance(x[0].astype(np.complex128))
for _ in range(2):
    est = fm.block_lanczos_subspace(s, 8, 16, 100)
print("cost", est.cost_seconds)
