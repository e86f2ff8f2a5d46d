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
