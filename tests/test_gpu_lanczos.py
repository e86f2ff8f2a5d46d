"""Block-Lanczos subspace (SURVEY.md §8(f)3, R/src/estimators.cpp:154-222) through the library (fp64 on the
GPU): the reference's own test cases (R/tests/test_estimators.cpp:207-242, 380-395, 466-487) with their
tolerances, and parity against the oracle restatement on random gapped / covariance matrices."""
import numpy as np
import pytest

from tests.test_gpu_facade import gapped_spectrum, proj_err, psd_with_spectrum

pytestmark = pytest.mark.gpu


def test_dominant_diagonal_converges_immediately(fm):
    d = np.diag([10.0, 1.0, 0.1, 0.01, 0.001, 0.0001]).astype(complex)
    est = fm.block_lanczos_subspace(d, 1, 1, 50)
    e1 = np.zeros(6, complex)
    e1[0] = 1.0
    assert np.linalg.norm(e1 - est.basis @ (est.basis.conj().T @ e1)) < 1e-8
    assert abs(est.eigenvalues[0] - 10.0) <= 1e-10 * 10.0
    assert est.method == "lanczos"


def test_matches_exact_on_gapped_matrix(fm):
    s = psd_with_spectrum(fm, gapped_spectrum(30, 4, 0.3), 29)
    est = fm.block_lanczos_subspace(s, 4, 4, 100)
    ex = fm.exact_signal_subspace(s, 4)
    assert proj_err(est.basis, ex.basis) < 1e-8
    assert np.allclose(est.eigenvalues, ex.eigenvalues, rtol=1e-8)
    assert np.max(np.abs(est.basis.conj().T @ est.basis - np.eye(4))) < 1e-8
    assert est.cost_seconds > 0.0


def test_iteration_cap_raises_with_last_change(fm):
    v = 1.0 - 1e-4 * np.arange(40)
    s = psd_with_spectrum(fm, v, 31)
    with pytest.raises(fm.NonConvergenceError) as ei:
        fm.block_lanczos_subspace(s, 3, 3, 2)
    assert ei.value.residual >= 0.0
    with pytest.raises(ValueError):
        fm.block_lanczos_subspace(s, 3, 2, 10)
    with pytest.raises(ValueError):
        fm.block_lanczos_subspace(s, 0, 2, 10)
    with pytest.raises(ValueError):
        fm.block_lanczos_subspace(s, 3, 3, 0)


def test_exact_ritz_pairs_when_krylov_space_exhausts(fm):
    sp = np.zeros(20)
    sp[:3] = [4.0, 2.0, 1.0]
    s = psd_with_spectrum(fm, sp, 53)
    est = fm.block_lanczos_subspace(s, 2, 3, 50)
    assert proj_err(est.basis, fm.exact_signal_subspace(s, 2).basis) < 1e-8
    assert abs(est.eigenvalues[0] - 4.0) <= 4e-9 and abs(est.eigenvalues[1] - 2.0) <= 2e-9
    s4 = psd_with_spectrum(fm, [3.0, 2.0, 1.0, 0.5], 54)
    est4 = fm.block_lanczos_subspace(s4, 2, 4, 50)  # block = M: the basis fills the space at once
    assert proj_err(est4.basis, fm.exact_signal_subspace(s4, 2).basis) < 1e-9


@pytest.mark.parametrize("m,k,block,gap,seed", [(30, 4, 4, 0.3, 61), (64, 3, 8, 0.5, 62), (128, 8, 16, 0.2, 63),
                                                 (48, 5, 5, 0.7, 64)])
def test_parity_with_oracle(fm, oracle, m, k, block, gap, seed):
    s = psd_with_spectrum(fm, gapped_spectrum(m, k, gap), seed)
    got = fm.block_lanczos_subspace(s, k, block, 200)
    ref = oracle.block_lanczos_subspace(s, k, block, 200)
    assert proj_err(got.basis, ref.basis) < 1e-8
    assert np.allclose(got.eigenvalues, ref.eigenvalues, rtol=1e-9)


def test_on_a_c2_covariance(fm, oracle):
    """A BASELINE c2 frame: the converged subspace equals the exact top-K (the paper's accurate baseline)."""
    cfg = oracle.baseline_configs()["c2"]
    x, _, _ = oracle.generate_batch(cfg.base_seed, [0], cfg.spec)
    s = oracle.spatial_covariance(x[0].astype(np.complex128))
    est = fm.block_lanczos_subspace(s, 8, 16, 100)
    ex = oracle.exact_signal_subspace(s, 8)
    assert proj_err(est.basis, ex.basis) < 1e-8
    assert np.allclose(est.eigenvalues, ex.eigenvalues, rtol=1e-9)


def test_deterministic(fm):
    s = psd_with_spectrum(fm, gapped_spectrum(40, 3, 0.4), 65)
    a = fm.block_lanczos_subspace(s, 3, 4, 100)
    b = fm.block_lanczos_subspace(s, 3, 4, 100)
    assert np.array_equal(a.basis, b.basis) and np.array_equal(a.eigenvalues, b.eigenvalues)


# ---------------------------------------------------------------- batched plan method (lanczos_batch.cu)
def test_batch_lanczos_c2_frames(fm, oracle):
    """FM_METHOD_LANCZOS on c2 frames (block = K, cap 200): identical peak cells and spectra within 0.05 dB of
    the oracle's block_lanczos_subspace on the fp64 covariance, Ritz values to the covariance precision."""
    from tests.gpu_helpers import compare_frames, run_gpu
    cfg = oracle.baseline_configs()["c2lz"]
    frames = list(range(24))
    x, _, _ = oracle.generate_batch(cfg.base_seed, frames, cfg.spec)
    res = run_gpu(fm, oracle, cfg, x, frames)
    assert np.all(res["status"] == 0), res["status"]
    worst, mism = compare_frames(oracle, cfg, x, frames, res)
    assert not mism, mism
    assert worst <= 0.05, worst
    for i in range(4):
        s = oracle.spatial_covariance(x[i])
        ref = oracle.block_lanczos_subspace(s, 8, 8, 200)
        assert np.allclose(res["eigenvalues"][i], ref.eigenvalues, rtol=2e-4)
        b = res["basis_c"][i]
        assert np.max(np.abs(b.conj().T @ b - np.eye(8))) < 1e-9


def test_batch_lanczos_matches_facade_on_exported_covariance(fm, oracle):
    """The batch method on the plan's complex64 R equals the fp64 facade (same device loop) run on that R."""
    from tests.gpu_helpers import run_gpu
    cfg = oracle.baseline_configs()["c2lz"]
    frames = [3, 7]
    x, _, _ = oracle.generate_batch(cfg.base_seed, frames, cfg.spec)
    res = run_gpu(fm, oracle, cfg, x, frames, covariance=True)
    for i in range(len(frames)):
        r = res["cov_c"][i].astype(np.complex128)
        est = fm.block_lanczos_subspace(r, 8, 8, 200)
        # the facade symmetrises 0.5 (R + R^H) as HermitianMatrix does; the batch reads R's lower triangle
        # (conj of its columns), and the two triangles of the tensor-core R differ at complex64 rounding
        assert proj_err(est.basis, res["basis_c"][i]) < 1e-7
        assert np.allclose(est.eigenvalues, res["eigenvalues"][i], rtol=1e-7)


@pytest.mark.parametrize("m,k,block", [(64, 3, 3), (48, 2, 5), (128, 4, 6)])
def test_batch_lanczos_shapes(fm, oracle, m, k, block):
    """Other shapes and blocks through the plan (fp16-free complex64 R path) against the oracle."""
    from tests.gpu_helpers import compare_frames, run_gpu
    spec = oracle.SceneSpec(m, 2 * m, k, -60.0, 60.0, 6.0, 15.0, 25.0)
    cfg = oracle.PathConfig("lz", "lanczos", spec, 6, 1801, p=block, t=200, base_seed=7)
    frames = list(range(6))
    x, _, _ = oracle.generate_batch(cfg.base_seed, frames, spec)
    res = run_gpu(fm, oracle, cfg, x, frames)
    assert np.all(res["status"] == 0), res["status"]
    worst, mism = compare_frames(oracle, cfg, x, frames, res)
    assert not mism, mism
    assert worst <= 0.05, worst


def test_batch_lanczos_capacity(fm, oracle):
    """A block-16 Krylov basis outgrows the device loop's 72 columns: the batch flags the frame NOCONV, the
    facade finishes it with the host-driven loop and still matches the oracle."""
    import torch
    s = psd_with_spectrum(fm, gapped_spectrum(128, 4, 0.05), 71)
    b, e, st, it = fm.block_lanczos_batch(torch.from_numpy(s[None].astype(np.complex64)).cuda(), 4, 16, 200)
    torch.cuda.synchronize()
    assert st.cpu().numpy()[0] & 2
    got = fm.block_lanczos_subspace(s, 4, 16, 200)
    ref = oracle.block_lanczos_subspace(s, 4, 16, 200)
    assert proj_err(got.basis, ref.basis) < 1e-8


def test_batch_lanczos_iteration_cap_flags_noconv(fm, oracle):
    from tests.gpu_helpers import run_gpu
    cfg = oracle.baseline_configs()["c2lz"]
    cfg = oracle.PathConfig("lzcap", "lanczos", cfg.spec, 2, 3601, p=0, t=2, base_seed=2)
    x, _, _ = oracle.generate_batch(cfg.base_seed, [0, 1], cfg.spec)
    res = run_gpu(fm, oracle, cfg, x, [0, 1])
    assert np.all(res["status"] & 2), res["status"]  # FM_FRAME_NOCONV


def test_block_lanczos_batch_entry(fm, oracle):
    """fm_block_lanczos_batch on device matrices: gapped spectra of several sizes against the oracle."""
    import torch
    frames = []
    for i in range(6):
        frames.append(psd_with_spectrum(fm, gapped_spectrum(40, 4, 0.3 + 0.05 * i), 80 + i))
    s = torch.from_numpy(np.stack(frames).astype(np.complex64)).cuda()
    b, e, st, it = fm.block_lanczos_batch(s, 4, 4, 200)
    torch.cuda.synchronize()
    assert np.all(st.cpu().numpy() == 0)
    for i in range(6):
        ref = oracle.block_lanczos_subspace(frames[i].astype(np.complex64).astype(np.complex128), 4, 4, 200)
        assert proj_err(b[i].cpu().numpy(), ref.basis) < 1e-7
        assert np.allclose(e[i].cpu().numpy(), ref.eigenvalues, rtol=1e-7)
    assert np.all(it.cpu().numpy() // 10000 >= 3)
