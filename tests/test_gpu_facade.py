"""The reference's own unit tests (R/tests/test_estimators.cpp, test_spectrum.cpp,
test_scene.cpp, acceptance.cpp criterion 1) re-run through the reference-named API,
executed on the GPU in fp64 (fm_z_* entry points), with the reference tolerances."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def random_unitary(fm, n, seed):
    from oracle import fastmusic_oracle as O  # checker-side construction of test inputs
    return O.qr_orthonormal(fm.gaussian_matrix_real(n, n, seed) + 1j * fm.gaussian_matrix_real(n, n, seed + 1))


def psd_with_spectrum(fm, ev, seed):
    q = random_unitary(fm, len(ev), seed)
    return fm.hermitian((q * np.asarray(ev)) @ q.conj().T)


def gapped_spectrum(n, k, gap):
    v = np.empty(n)
    for i in range(k):
        v[i] = 2.0 - 0.5 * i / max(k, 1)
    for i in range(k, n):
        v[i] = v[k - 1] * gap * 0.9 ** (i - k)
    return v


def proj_err(a, b):
    return float(np.linalg.norm(a @ a.conj().T - b @ b.conj().T, 2))


def test_covariance_cases(fm):
    s = fm.spatial_covariance(np.eye(2))
    assert np.linalg.norm(s - 0.5 * np.eye(2)) < 1e-15
    rng = np.random.default_rng(9)
    y = rng.normal(size=(6, 10)) + 1j * rng.normal(size=(6, 10))
    ref = sum(np.outer(y[:, n], y[:, n].conj()) for n in range(10)) / 10
    assert np.linalg.norm(s := fm.spatial_covariance(y)) > 0
    assert np.linalg.norm(s - ref) < 1e-12 * np.linalg.norm(ref)
    x = rng.normal(size=3) + 1j * rng.normal(size=3)
    s2 = fm.spatial_covariance(np.outer(x, np.ones(7)))
    assert np.linalg.norm(s2 - np.outer(x, x.conj())) < 1e-12 * np.linalg.norm(x) ** 2


def test_exact_diagonal_and_validation(fm):
    d = np.diag([3.0, 2.0, 1.0]).astype(complex)
    est = fm.exact_signal_subspace(d, 2)
    assert np.allclose(est.eigenvalues, [3.0, 2.0])
    assert abs(abs(est.basis[0, 0]) - 1) < 1e-12 and abs(abs(est.basis[1, 1]) - 1) < 1e-12
    assert est.method == "exact" and est.cost_seconds >= 0.0
    with pytest.raises(ValueError):
        fm.exact_signal_subspace(d, 3)


@pytest.mark.parametrize("m", [1, 2, 7, 64, 65, 130, 300])
def test_hermitian_eig_full_decomposition(fm, m):
    """R/src/linalg.cpp:77-89: eigenvalues descending (signed), column i pairs with eigenvalue i, orthonormal
    eigenvectors; against numpy's eigh on an indefinite Hermitian matrix (shared-memory Jacobi for M <= 64, the
    global-memory Jacobi beyond)."""
    rng = np.random.default_rng(100 + m)
    a = rng.standard_normal((m, m)) + 1j * rng.standard_normal((m, m))
    s = 0.5 * (a + a.conj().T)
    r = fm.hermitian_eig(s)
    w = np.linalg.eigvalsh(s)[::-1]
    scale = max(1.0, np.abs(w).max())
    assert r.eigenvalues.shape == (m,) and r.eigenvectors.shape == (m, m)
    assert np.all(np.diff(r.eigenvalues) <= 1e-12 * scale)
    assert np.abs(r.eigenvalues - w).max() < 1e-10 * scale
    v = r.eigenvectors
    assert np.abs(v.conj().T @ v - np.eye(m)).max() < 1e-10
    assert np.abs(s @ v - v * r.eigenvalues[None, :]).max() < 1e-9 * scale


def test_hermitian_eig_matches_exact_signal_subspace(fm):
    s = psd_with_spectrum(fm, gapped_spectrum(12, 4, 0.4), 5)
    full = fm.hermitian_eig(s)
    est = fm.exact_signal_subspace(s, 4)
    assert np.allclose(full.eigenvalues[:4], est.eigenvalues, rtol=1e-12)
    assert proj_err(full.eigenvectors[:, :4], est.basis) < 1e-10
    with pytest.raises(ValueError):
        fm.hermitian_eig(np.full((3, 3), np.nan, complex))
    with pytest.raises(ValueError):
        fm.hermitian_eig(np.zeros((2, 3), complex))


def test_exact_projector_vs_full_decomposition(fm):
    s = psd_with_spectrum(fm, gapped_spectrum(10, 3, 0.4), 3)
    est = fm.exact_signal_subspace(s, 3)
    w, v = np.linalg.eigh(s)
    assert proj_err(est.basis, v[:, ::-1][:, :3]) < 1e-9
    assert np.allclose(est.eigenvalues, w[::-1][:3], rtol=1e-10)


def test_exact_indefinite_signed_order(fm):
    a = np.array([[1.0, 2.0], [2.0, 1.0]], complex)  # eigenvalues 3, -1
    est = fm.exact_signal_subspace(a, 1)
    assert abs(est.eigenvalues[0] - 3.0) < 1e-12


def test_fast1_full_sampling_reproduces_exact(fm):
    s = psd_with_spectrum(fm, gapped_spectrum(24, 4, 0.3), 7)
    ex = fm.exact_signal_subspace(s, 4)
    f1 = fm.fast_music_1(s, 4, fm.Fast1Params(24, 1))
    assert proj_err(f1.basis, ex.basis) < 1e-8 and f1.method == "fast1"


def test_fast1_determinism_and_validation(fm):
    s = psd_with_spectrum(fm, gapped_spectrum(16, 3, 0.3), 9)
    a = fm.fast_music_1(s, 3, fm.Fast1Params(6, 42))
    b = fm.fast_music_1(s, 3, fm.Fast1Params(6, 42))
    assert np.array_equal(a.basis, b.basis)
    with pytest.raises(ValueError):
        fm.fast_music_1(s, 3, fm.Fast1Params(2, 0))
    with pytest.raises(ValueError):
        fm.fast_music_1(s, 3, fm.Fast1Params(17, 0))


def test_fast1_singular_block_truncates(fm):
    ev = np.zeros(12)
    ev[:2] = [3.0, 1.0]
    s = psd_with_spectrum(fm, ev, 11)
    est = fm.fast_music_1(s, 2, fm.Fast1Params(6, 3))
    assert proj_err(est.basis, fm.exact_signal_subspace(s, 2).basis) < 1e-7


def test_fast2_exact_rank_capture(fm):
    ev = np.zeros(20)
    ev[:3] = [5.0, 2.5, 1.0]
    s = psd_with_spectrum(fm, ev, 13)
    est = fm.fast_music_2(s, 3, fm.Fast2Params(3, 1, 17))
    assert proj_err(est.basis, fm.exact_signal_subspace(s, 3).basis) < 1e-8 and est.method == "fast2"


def test_fast2_power_iterations_geometric(fm):
    gap = 0.3
    s = psd_with_spectrum(fm, gapped_spectrum(50, 3, gap), 15)
    ex = fm.exact_signal_subspace(s, 3)
    assert proj_err(fm.fast_music_2(s, 3, fm.Fast2Params(6, 10, 4)).basis, ex.basis) < 1e-6
    med = []
    for t in (1, 2, 3):
        errs = sorted(proj_err(fm.fast_music_2(s, 3, fm.Fast2Params(6, t, seed)).basis, ex.basis) for seed in range(50))
        med.append(errs[25])
    assert med[1] <= gap * med[0] * 1.10 and med[2] <= gap * med[1] * 1.10


def test_fast2_determinism_validation_and_redraw_exhaustion(fm):
    s = psd_with_spectrum(fm, gapped_spectrum(16, 3, 0.2), 19)
    a = fm.fast_music_2(s, 3, fm.Fast2Params(5, 2, 7))
    b = fm.fast_music_2(s, 3, fm.Fast2Params(5, 2, 7))
    assert np.array_equal(a.basis, b.basis)
    for p, t in ((2, 2), (5, 0), (5, 21)):
        with pytest.raises(ValueError):
            fm.fast_music_2(s, 3, fm.Fast2Params(p, t, 0))
    ev = np.zeros(16)
    ev[:2] = [2.0, 1.0]
    with pytest.raises(fm.RankDeficiencyError):
        fm.fast_music_2(psd_with_spectrum(fm, ev, 47), 2, fm.Fast2Params(4, 2, 5))


def test_acceptance_criterion1(fm):
    """R/tests/acceptance.cpp:66-103: 50 random gapped PSD matrices up to 64x64."""
    from oracle import fastmusic_oracle as O
    rng_shapes = O.below_stream(0xC1, 57, 1)  # first draw only used for M below (restated loop)
    worst1 = worst2 = 0.0
    r = np.random.default_rng(0xC1)
    for trial in range(50):
        m = int(8 + r.integers(0, 57))
        k = int(1 + r.integers(0, max(1, min(6, m // 4))))
        ev = np.array([2.0 - i / (2 * k) for i in range(k)] + [0.0] * (m - k))
        for i in range(k, m):
            ev[i] = 0.3 * ev[k - 1] * 0.85 ** (i - k)
        q = random_unitary(fm, m, 1000 + trial)
        s = fm.hermitian((q * ev) @ q.conj().T)
        ex = fm.exact_signal_subspace(s, k)
        worst1 = max(worst1, proj_err(fm.fast_music_1(s, k, fm.Fast1Params(m, 2000 + trial)).basis, ex.basis))
        evk = ev.copy()
        evk[k:] = 0.0
        sk = fm.hermitian((q * evk) @ q.conj().T)
        f2 = fm.fast_music_2(sk, k, fm.Fast2Params(k, 1, 3000 + trial))
        worst2 = max(worst2, proj_err(f2.basis, fm.exact_signal_subspace(sk, k).basis))
    assert worst1 <= 1e-8 and worst2 <= 1e-8, (worst1, worst2)
    assert rng_shapes.size == 1


def test_spectrum_cases(fm):
    est = fm.SubspaceEstimate(np.zeros((8, 0), complex), np.zeros(0))
    p = fm.music_spectrum(est, fm.AngleGrid(64), 0.002, 0.004)
    assert np.allclose(p.values, 1 / 8, rtol=1e-12)
    with pytest.raises(ValueError):
        fm.music_spectrum(fm.SubspaceEstimate(2.0 * np.eye(8, 2, dtype=complex), np.zeros(2)), fm.AngleGrid(32),
                          0.002, 0.004)
    s = fm.hermitian(fm.gaussian_matrix_real(12, 12, 3) @ fm.gaussian_matrix_real(12, 12, 3).T)
    e4 = fm.exact_signal_subspace(s, 4)
    p = fm.music_spectrum(e4, fm.AngleGrid(721), 0.002, 0.004)
    assert p.values.min() > 0.0
    q = random_unitary(fm, 4, 9)
    p2 = fm.music_spectrum(fm.SubspaceEstimate(e4.basis @ q, e4.eigenvalues), fm.AngleGrid(721), 0.002, 0.004)
    assert np.max(np.abs(p.values - p2.values)) < 1e-10 * p.values.max()


def test_spectrum_matches_oracle_on_random_bases(fm, oracle):
    for seed, (m, k, L) in enumerate([(16, 2, 181), (64, 3, 1801), (256, 8, 3601)]):
        s = psd_with_spectrum(fm, gapped_spectrum(m, k, 0.05), 100 + seed)
        est = fm.exact_signal_subspace(s, k)
        grid = fm.baseline_grid(L)
        got = fm.music_spectrum(est, grid, 0.5, 1.0).values
        ref = oracle.music_spectrum(est.basis, oracle.baseline_grid(L))
        assert np.max(np.abs(got - ref) / ref) < 1e-9


def test_peak_rules(fm):
    def spec(vals):
        return fm.PseudoSpectrum(fm.AngleGrid(len(vals)), np.array(vals, float))
    pk = fm.extract_peaks(spec([0.1, 0.2, 1.0, 0.2, 0.1]), 1, 1)
    assert pk.cells == [2] and pk.heights == [1.0] and not pk.shortfall and abs(pk.baseline - 0.1) < 1e-15
    pk = fm.extract_peaks(spec([0.1, 1.0, 0.1, 0.05, 0.1, 1.0, 0.1]), 2, 2)
    assert pk.cells == [1, 5] and pk.angles[0] < pk.angles[1]
    assert fm.extract_peaks(spec([0.1, 0.5, 0.5, 0.5, 0.1]), 1, 1).cells == [1]
    pk = fm.extract_peaks(spec([0.1, 0.2, 1.0, 0.2, 0.1]), 3, 1)
    assert pk.shortfall and len(pk.cells) == 1
    v = [0.1, 0.9, 0.2, 0.3, 0.8, 0.1, 0.4, 0.2]
    assert fm.extract_peaks(spec(v), 3, 1).cells == fm.extract_peaks(spec([37.5 * a for a in v]), 3, 1).cells
    with pytest.raises(ValueError):
        fm.extract_peaks(spec(v), 0, 1)


def test_peaks_match_oracle_random(fm, oracle):
    rng = np.random.default_rng(5)
    for _ in range(100):
        n = int(rng.integers(3, 300))
        v = rng.integers(0, 6, size=n).astype(float) if rng.random() < 0.5 else rng.random(n)
        k, sep = int(rng.integers(1, 9)), int(rng.integers(0, 5))
        got = fm.extract_peaks(fm.PseudoSpectrum(fm.AngleGrid(max(n, 2)), v), k, sep)
        ref = oracle.extract_peaks(v, k, sep)
        assert got.cells == ref.cells and got.heights == ref.heights
        assert got.baseline == ref.baseline and got.shortfall == ref.shortfall


def _peaks_equal(fm, oracle, v, k, sep, tag=None):
    got = fm.extract_peaks(fm.PseudoSpectrum(fm.AngleGrid(max(len(v), 2)), np.asarray(v, float)), k, sep)
    ref = oracle.extract_peaks(np.asarray(v, float), k, sep)
    assert got.cells == ref.cells and got.heights == ref.heights, tag
    assert got.baseline == ref.baseline and got.shortfall == ref.shortfall, tag


def test_peaks_negative_and_db_scale_spectra(fm, oracle):
    """any finite spectrum, e.g. a dB-scale one with every value below -1 (the argmax starts at
    -inf; the baseline keeps the reference's 0 start, R/src/spectrum.cpp:150-164)."""
    rng = np.random.default_rng(31)
    for _ in range(60):
        n = int(rng.integers(3, 500))
        v = rng.random(n)
        mode = rng.integers(0, 3)
        if mode == 0:
            v = 10.0 * np.log10(v * 1e-3)          # all < -30 dB
        elif mode == 1:
            v = -1.0 - 5.0 * v                      # all below -1
        else:
            v = rng.integers(-6, 0, size=n).astype(float)  # negative plateaus
        _peaks_equal(fm, oracle, v, int(rng.integers(1, 12)), int(rng.integers(0, 5)), (n, mode))


def test_peaks_global_workspace_long_grids_large_k(fm, oracle):
    """Grids whose peak workspace does not fit shared memory (L = 30001, 60001) and K beyond 64 run the same
    kernel over a global workspace: identical to the reference's sort + greedy walk."""
    rng = np.random.default_rng(13)
    for n, k, sep in ((30001, 16, 3), (60001, 100, 2), (30001, 300, 0), (4001, 500, 1)):
        for ints in (False, True):
            v = rng.integers(0, 4, size=n).astype(float) if ints else rng.random(n)
            _peaks_equal(fm, oracle, v, k, sep, (n, k, sep, ints))


def test_peaks_rounds_long_grids_wide_bands(fm, oracle):
    """K-round argmax peak kernel (the batch path's default) on long grids with many maxima, wide
    separation bands, large K and plateau-heavy integer data: identical to the reference's sort + greedy walk."""
    rng = np.random.default_rng(21)
    for n, k, sep in ((3601, 8, 3), (18001, 16, 3), (3601, 64, 40), (1801, 33, 0), (5000, 20, 150), (2, 1, 1), (3, 4, 1)):
        for ints in (False, True):
            v = rng.integers(0, 4, size=n).astype(float) if ints else rng.random(n)
            got = fm.extract_peaks(fm.PseudoSpectrum(fm.AngleGrid(n), v), k, sep)
            ref = oracle.extract_peaks(v, k, sep)
            assert got.cells == ref.cells and got.heights == ref.heights, (n, k, sep, ints)
            assert got.baseline == ref.baseline and got.shortfall == ref.shortfall, (n, k, sep, ints)
