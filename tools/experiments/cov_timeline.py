"""Per-tile clock64 timeline of the covariance kernel's CTA 0 (library built with
FM_NVCC_FLAGS=-DFM_COV_TIMELINE): MMA start / last commit, epilogue acc_full / after s_f / drain done,
converter first / last stage, and per tile the cycles the converter waited on TMA (stage_full) and on the MMA
(op_empty), and the MMA waited on operands (op_full).
  python tools/experiments/cov_timeline.py"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.argv = [sys.argv[0], "c2", "1"]
lib = ctypes.CDLL(os.path.join(ROOT, "paper_1911_07434_b200", "libfastmusic_b200.so"))
import runpy  # noqa: E402

runpy.run_path(os.path.join(ROOT, "tools", "run_batches.py"), run_name="__main__")  # warm
lib.fm_debug_cov_timeline(None, 1)
runpy.run_path(os.path.join(ROOT, "tools", "run_batches.py"), run_name="__main__")
torch.cuda.synchronize()
buf = (ctypes.c_longlong * 256)()
lib.fm_debug_cov_timeline(buf, 0)
tl = np.array(buf[:], dtype=np.int64).reshape(16, 16)
# run_batches ran one batch after the zeroing: stamps belong to its launch; times relative to tile 0 MMA start
t0 = tl[0, 0]
names = ["mma_start", "mma_end", "epi_accfull", "epi_sf", "epi_drained", "conv_first", "conv_last"]
print("tile " + " ".join(f"{n:>11}" for n in names) + "  conv_wait_tma conv_wait_mma mma_wait_op")
for i in range(14):
    r = tl[i]
    print(f"{i:4d} " + " ".join(f"{(r[j] - t0):11d}" for j in range(7)) + f"  {r[7]:13d} {r[8]:13d} {r[9]:11d}")
d = tl[1:13]
print("per-tile means: mma span", int(np.mean(d[:, 1] - d[:, 0])), " drain (accfull->drained)",
      int(np.mean(d[:, 4] - d[:, 2])), " s_f part", int(np.mean(d[:, 3] - d[:, 2])),
      " period", int(np.mean(np.diff(tl[1:13, 0]))))
