"""Check the tensor-core range-finder product (rmul_tc.cu) on the GPU.

Runs fm_debug_rmul_tc on random Hermitian R and random V / Omega, once with the raw fp32 R
as the tf32 A_hi operand and once with an explicit truncation pass (FM_RMUL_TRUNC_A=1, in a
subprocess), and compares both against an fp64 numpy product. Prints max relative errors and
whether the two modes agree bitwise (they do iff the tensor core truncates fp32 -> tf32).
"""
import ctypes
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(m, p, frames, real, seed, out_path):
    import torch
    from paper_1911_07434_b200 import _capi
    lib = ctypes.CDLL(_capi.LIB_PATH)
    rng = np.random.default_rng(seed)
    x = (rng.standard_normal((frames, m, 2 * m)) + 1j * rng.standard_normal((frames, m, 2 * m))).astype(np.complex64)
    r = (x @ x.conj().transpose(0, 2, 1) / (2 * m)).astype(np.complex64)
    rd = torch.from_numpy(r.view(np.float32).copy()).cuda()
    if real:
        om = rng.standard_normal((frames, m, p)).astype(np.float32)
        vd = torch.from_numpy(om).cuda()
        ref = np.einsum("fij,fjc->fic", r.astype(np.complex128), om.astype(np.float64))
        args = (ctypes.c_void_p(rd.data_ptr()), ctypes.c_void_p(vd.data_ptr()), None)
    else:
        v = (rng.standard_normal((frames, p, m)) + 1j * rng.standard_normal((frames, p, m))).astype(np.complex64)
        vd = torch.from_numpy(v.view(np.float32).copy()).cuda()
        ref = np.einsum("fij,fcj->fic", r.astype(np.complex128), v.astype(np.complex128))
        args = (ctypes.c_void_p(rd.data_ptr()), None, ctypes.c_void_p(vd.data_ptr()))
    cd = torch.zeros(frames * p * m * 2, dtype=torch.float32, device="cuda")
    lib.fm_debug_rmul_tc.restype = ctypes.c_int32
    lib.fm_debug_rmul_tc.argtypes = [ctypes.c_void_p] * 4 + [ctypes.c_int64] * 3
    st = lib.fm_debug_rmul_tc(*args, ctypes.c_void_p(cd.data_ptr()), frames, m, p)
    assert st == 0, st
    c = cd.cpu().numpy().view(np.complex64).reshape(frames, p, m).transpose(0, 2, 1)
    np.save(out_path, c)
    err = np.abs(c - ref).max() / np.abs(ref).max()
    return err


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--child":
        m, p, frames, real, seed = map(int, sys.argv[2:7])
        print(run(m, p, frames, bool(real), seed, sys.argv[7]))
        sys.exit(0)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    for (m, p, frames, real) in [(256, 16, 8, 0), (256, 16, 8, 1), (64, 8, 4, 0), (300, 12, 3, 0), (1024, 32, 2, 0),
                                 (520, 32, 2, 1)]:
        outs, errs = [], []
        for trunc in (0, 1):
            path = f"/tmp/rmul_{m}_{p}_{real}_{trunc}.npy"
            env = dict(os.environ, FM_RMUL_TRUNC_A=str(trunc))
            r = subprocess.run([sys.executable, __file__, "--child", str(m), str(p), str(frames), str(real), "7", path],
                               env=env, capture_output=True, text=True)
            if r.returncode != 0:
                print("FAIL", m, p, real, trunc, r.stderr[-2000:])
                sys.exit(1)
            errs.append(float(r.stdout.strip().splitlines()[-1]))
            outs.append(np.load(path))
        print(f"m={m} p={p} real={real}: rel err raw={errs[0]:.3e} trunc={errs[1]:.3e} "
              f"bitwise_equal={np.array_equal(outs[0], outs[1])}")
