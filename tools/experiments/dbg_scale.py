import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
import paper_1911_07434_b200 as fm
from oracle import fastmusic_oracle as O
from tests.gpu_helpers import run_gpu
cfgs = O.baseline_configs()
cfg = cfgs["c2"]
frames = list(range(int(sys.argv[2]) if len(sys.argv) > 2 else 4))
x, _, _ = O.generate_batch(cfg.base_seed, frames, cfg.spec)
xs = (x * np.float32(2.0 ** int(sys.argv[1]))).astype(np.complex64)
try:
    res = run_gpu(fm, O, cfg, xs, frames)
    print("status", res["status"][:8], "cells", res["peak_cells"][0])
except Exception as e:
    print("ERR", e, fm._capi.last_error() if hasattr(fm, "_capi") else "")
