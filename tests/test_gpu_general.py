"""Facade entry points beyond the shared-memory kernels' sizes (general.cu): the reference API accepts any M,
K < M and K <= p <= M (R/src/estimators.cpp:73-139, 154-222), so exact_signal_subspace at M > 384 (the massive-array
shape of BASELINE config 4, M = 1024), fast_music_1/2 with p > 64 and block-Lanczos at M > 384 / block > 64 must
run -- on the GPU, in fp64 -- and agree with the oracle restatement to the facade's fp64 tolerances."""
import numpy as np
import pytest

from tests.test_gpu_facade import gapped_spectrum, proj_err, psd_with_spectrum

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("m,k,seed", [(400, 5, 71), (1024, 16, 72)])
def test_exact_large_m_matches_full_decomposition(fm, m, k, seed):
    s = psd_with_spectrum(fm, gapped_spectrum(m, k, 0.5), seed)
    est = fm.exact_signal_subspace(s, k)
    w, v = np.linalg.eigh(s)
    assert proj_err(est.basis, v[:, ::-1][:, :k]) < 1e-9
    assert np.allclose(est.eigenvalues, w[::-1][:k], rtol=1e-10)
    assert np.max(np.abs(est.basis.conj().T @ est.basis - np.eye(k))) < 1e-10


def test_exact_large_m_covariance_vs_oracle(fm, oracle):
    """A c4-shaped covariance (M = 1024 ULA, 16 sources) through the facade vs the oracle's exact subspace:
    identical spectrum to fp64 precision."""
    rng = np.random.default_rng(73)
    m, n, k = 1024, 2048, 16
    th = np.deg2rad(np.sort(rng.uniform(-70, 70, k)))
    a = np.exp(1j * np.pi * np.outer(np.arange(m), np.sin(th)))
    sig = (rng.normal(size=(k, n)) + 1j * rng.normal(size=(k, n))) / np.sqrt(2)
    y = a @ sig + 0.1 * (rng.normal(size=(m, n)) + 1j * rng.normal(size=(m, n))) / np.sqrt(2)
    s = fm.hermitian(y @ y.conj().T / n)
    est = fm.exact_signal_subspace(s, k)
    ref = oracle.exact_signal_subspace(s, k)
    assert proj_err(est.basis, ref.basis) < 1e-9
    assert np.allclose(est.eigenvalues, ref.eigenvalues, rtol=1e-10)


def test_exact_large_m_indefinite_signed_order(fm):
    rng = np.random.default_rng(74)
    m = 400
    ev = np.concatenate([[5.0, 3.0], rng.uniform(-4.0, 1.0, m - 2)])
    s = psd_with_spectrum(fm, ev, 75)
    est = fm.exact_signal_subspace(s, 3)
    top = np.sort(ev)[::-1][:3]
    assert np.allclose(est.eigenvalues, top, rtol=1e-10)


@pytest.mark.parametrize("m,k,p,t,seed", [(200, 6, 80, 2, 81), (300, 40, 96, 1, 82)])
def test_fast2_large_p_vs_oracle(fm, oracle, m, k, p, t, seed):
    s = psd_with_spectrum(fm, gapped_spectrum(m, k, 0.3), seed)
    est = fm.fast_music_2(s, k, fm.Fast2Params(p, t, seed))
    ref = oracle.fast_music_2(s, k, p, t, seed)
    assert proj_err(est.basis, ref.basis) < 1e-8
    assert np.allclose(est.eigenvalues, ref.eigenvalues, rtol=1e-8)


def test_fast1_large_p_vs_oracle(fm, oracle):
    s = psd_with_spectrum(fm, gapped_spectrum(160, 5, 0.3), 83)
    est = fm.fast_music_1(s, 5, fm.Fast1Params(100, 84))
    ref = oracle.fast_music_1(s, 5, 100, 84)
    assert proj_err(est.basis, ref.basis) < 1e-8
    assert np.allclose(est.eigenvalues, ref.eigenvalues, rtol=1e-8)


def test_fast1_large_p_singular_block_truncates(fm):
    """R/tests/test_estimators.cpp:117-126 at p > 64: S(I, I) of rank 2, pinv truncates."""
    ev = np.zeros(120)
    ev[:2] = [3.0, 1.0]
    s = psd_with_spectrum(fm, ev, 85)
    est = fm.fast_music_1(s, 2, fm.Fast1Params(80, 3))
    assert proj_err(est.basis, fm.exact_signal_subspace(s, 2).basis) < 1e-7


@pytest.mark.parametrize("m,k,block,seed", [(512, 4, 8, 91), (200, 3, 80, 92)])
def test_lanczos_beyond_shared_memory_sizes_vs_oracle(fm, oracle, m, k, block, seed):
    s = psd_with_spectrum(fm, gapped_spectrum(m, k, 0.3), seed)
    est = fm.block_lanczos_subspace(s, k, block, 100)
    ref = oracle.block_lanczos_subspace(s, k, block, 100)
    assert proj_err(est.basis, ref.basis) < 1e-8
    assert np.allclose(est.eigenvalues, ref.eigenvalues, rtol=1e-9)
