"""Check the device Ritz-value path (tridiagonalisation + Sturm multisection, lanczos_batch.cu) against numpy."""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = C.CDLL(os.path.join(ROOT, "paper_1911_07434_b200", "libfastmusic_b200.so"))
rng = np.random.default_rng(1)
for n in (2, 3, 8, 16, 40, 72):
    x = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    h = np.asfortranarray(x + x.conj().T)
    if n == 40:
        h = np.asfortranarray(np.diag(np.linspace(100, 1, n)).astype(complex) + 1e-3 * h)
    kk = min(8, n)
    out = np.zeros(kk)
    st = lib.fm_debug_ritz_values(h.ctypes.data_as(C.c_void_p), n, kk, out.ctypes.data_as(C.c_void_p))
    ref = np.sort(np.linalg.eigvalsh(h))[::-1][:kk]
    print(n, st, np.max(np.abs(out - ref) / np.abs(ref).max()), out[:3], ref[:3])
