"""Debug: fm_block_lanczos_batch vs the facade vs the oracle on small gapped matrices."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1911_07434_b200 as fm  # noqa: E402
from oracle import fastmusic_oracle as O  # noqa: E402
from tests.test_gpu_facade import gapped_spectrum, proj_err, psd_with_spectrum  # noqa: E402

m = 40
s = psd_with_spectrum(fm, gapped_spectrum(m, 4, 0.3), 80)
s64 = s.astype(np.complex64)
st = torch.from_numpy(np.stack([s64])).cuda()
b, e, stt, it = fm.block_lanczos_batch(st, 4, 4, 200)
torch.cuda.synchronize()
ref = O.block_lanczos_subspace(s64.astype(np.complex128), 4, 4, 200)
g = b[0].cpu().numpy()
print("strides", b.stride(), b.shape, g.shape, g.dtype)
print("conj", proj_err(np.conj(g), ref.basis), "plain", proj_err(g, ref.basis))
print("orth", np.max(np.abs(g.conj().T @ g - np.eye(4))))
print("resid", np.linalg.norm(s64 @ g - g * e[0].cpu().numpy()[None, :]))
print("resid conjS", np.linalg.norm(s64.conj() @ g - g * e[0].cpu().numpy()[None, :]))
raw = torch.view_as_complex(torch.empty(0)) if False else None
