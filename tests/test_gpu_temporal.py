"""Temporal covariance (SURVEY.md §8(f)4, R/src/scene.cpp:140-153,161-163: T = Y^H Y / M, N x N):
the fp64 single-matrix entry against the oracle to rounding, and the batched tensor-core entry (covariance
kernel on X^H) against the oracle under the same precision contract as the spatial covariance."""
import numpy as np
import pytest

from paper_1911_07434_b200 import _capi

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("m,n", [(5, 7), (16, 3), (64, 200), (1, 4), (9, 1)])
def test_temporal_covariance_fp64(fm, oracle, m, n):
    z = fm.normals(m * 100 + n, 2 * m * n).reshape(m, n, 2)
    y = z[..., 0] + 1j * z[..., 1]
    got = fm.temporal_covariance(y)
    ref = oracle.temporal_covariance(y)
    assert got.shape == (n, n)
    assert np.max(np.abs(got - ref)) <= 1e-12 * np.max(np.abs(ref))
    assert np.array_equal(got, got.conj().T)
    assert np.all(np.diag(got).imag == 0.0)
    # T = Y^H Y / M is the spatial covariance of Y^H (scaled by its own column count, M)
    assert np.max(np.abs(got - fm.spatial_covariance(y.conj().T))) <= 1e-13 * np.max(np.abs(ref))


def test_temporal_covariance_validation(fm):
    with pytest.raises(ValueError):
        fm.temporal_covariance(np.zeros((0, 3)))
    y = np.ones((3, 3), complex)
    y[1, 1] = np.inf
    with pytest.raises(ValueError, match="non-finite"):
        fm.temporal_covariance(y)


# c2 frames (N = 512 -> off-diagonal tiles), odd M (padded snapshot), odd N (generic-store epilogue),
# N < M, N > 256 with few snapshots
@pytest.mark.parametrize("m,n", [(256, 512), (37, 64), (64, 101), (100, 30), (8, 300), (1, 40)])
def test_temporal_covariance_batch(fm, oracle, m, n):
    import torch
    frames = 3
    x, _, _ = fm.generate_frames(m, n, 1 if m < 3 else 2, 51, 0, frames)
    xd = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    t, st = fm.temporal_covariance_batch(xd)
    torch.cuda.synchronize()
    t = t.cpu().numpy()
    assert np.all(st.cpu().numpy() == 0)
    for f in range(frames):
        ref = oracle.temporal_covariance(x[f].astype(np.complex128))
        got = t[f].astype(np.complex128)
        rel = np.linalg.norm(got - ref) / np.linalg.norm(ref)
        # fp16 operands, fp32 accumulation: same bound as the spatial covariance (tests/test_gpu_pipeline.py)
        assert rel < (2e-4 if m >= 16 else 1e-3), (m, n, f, rel)
        assert np.all(np.diag(got).imag == 0.0)
        assert np.max(np.abs(got - got.conj().T)) <= 1e-6 * np.abs(ref).max()


def test_temporal_covariance_batch_flags(fm, oracle):
    """Out-of-fp16-range frames (x 1e5, x 2^-30) are recomputed with a power-of-two prescale (cov_tc.cu rescue
    pass) and match the fp64 covariance; only frames beyond the complex64 range (2^+-50) are flagged RANGE."""
    import torch
    m, n = 32, 48
    x, _, _ = fm.generate_frames(m, n, 2, 52, 0, 5)
    x[1, 3, 5] = complex(np.nan, 0)
    x[2] *= np.float32(1e5)      # |x| ~ 1e5 overflows the fp16 operand range unscaled
    x[3] *= np.float32(2.0 ** -30)  # fp16 subnormal / zero unscaled
    x[4] *= np.float32(2.0 ** 60)   # R would overflow complex64
    t, st = fm.temporal_covariance_batch(torch.from_numpy(x).cuda())
    torch.cuda.synchronize()
    st = st.cpu().numpy()
    t = t.cpu().numpy()
    assert st[0] == 0 and st[2] == 0 and st[3] == 0
    assert st[1] & _capi.FRAME_NONFINITE
    assert st[4] & _capi.FRAME_RANGE
    for f in (0, 2, 3):
        ref = oracle.temporal_covariance(x[f].astype(np.complex128))
        rel = np.linalg.norm(t[f].astype(np.complex128) - ref) / np.linalg.norm(ref)
        assert rel < 2e-4, (f, rel)
