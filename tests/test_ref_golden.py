"""The oracle restatement against the REFERENCE's own code: golden vectors produced by the reference's
R/src/{scene,linalg,estimators,spectrum}.cpp compiled here in place (oracle/_ref, Eigen-API shim over LAPACK;
tests/golden/make_ref_golden.py), plus live comparisons when that library is present (this dev container).
Peaks are index work: bit-exact. Estimators / spectra: fp64 agreement (decomposition internals differ only by
LAPACK vs Eigen rounding and unitary freedom)."""
import numpy as np
import pytest

from tests.ref_golden import est_cases, frame_cases, load, peak_cases

G = load()


def test_golden_peaks_oracle_bit_exact(oracle):
    n = 0
    for v, k, sep, cells, heights, base, sf in peak_cases(G):
        ps = oracle.extract_peaks(v, k, sep)
        assert ps.cells == cells and ps.heights == heights and ps.baseline == base and ps.shortfall == sf, (len(v), k, sep)
        n += 1
    assert n >= 400


def test_golden_estimators_oracle(oracle):
    for name, s, method, k, p, t, seed, st, proj, eig in est_cases(G):
        assert st == 0, name
        if method == "exact":
            est = oracle.exact_signal_subspace(s, k)
        elif method == "fast1":
            est = oracle.fast_music_1(s, k, p, seed)
        else:
            est = oracle.fast_music_2(s, k, p, t, seed)
        b = est.basis
        assert np.linalg.norm(b @ b.conj().T - proj, 2) < 1e-9, name
        assert np.allclose(est.eigenvalues, eig, rtol=1e-9, atol=1e-12), name
    st, col = (int(v) for v in G["est_zero_fast2_status_column"])
    assert st == 2 and col == 0  # RankDeficiencyError after the redraws, column 0
    with pytest.raises(oracle.RankDeficiencyError):
        oracle.fast_music_2(np.zeros((8, 8), complex), 2, 3, 1, 5)


def test_golden_frames_oracle(oracle):
    """Whole path on BASELINE frames, reference grid [0, pi]: covariance -> estimator -> spectrum -> peaks."""
    cfgs = oracle.baseline_configs()
    for cname, f, spec, cells, eig in frame_cases(G):
        cfg = cfgs[cname]
        x, _, _ = oracle.generate_batch(cfg.base_seed, [f], cfg.spec)
        grid = oracle.AngleGrid(cfg.grid_size)  # [0, pi]: the reference's AngleGrid
        est, p, pk = oracle.run_frame(cfg, x[0], f, grid)
        assert np.max(np.abs(p - spec) / spec) < 1e-8, (cname, f)
        assert pk.cells == cells, (cname, f)
        assert np.allclose(est.eigenvalues, eig, rtol=1e-9), (cname, f)


def test_golden_steering(oracle):
    i = 0
    while f"steer_{i}" in G:
        th, m = G[f"steer_{i}_args"]
        assert np.array_equal(oracle.steering_vector(float(th), int(m)), G[f"steer_{i}"])
        i += 1


def _ref():
    from oracle import ref_lib
    if not ref_lib.available():
        pytest.skip("oracle/_ref/libref_fastmusic.so not built (reference tree absent)")
    return ref_lib


def test_live_reference_peaks(oracle):
    R = _ref()
    rng = np.random.default_rng(77)
    for t in range(3000):
        n = int(rng.integers(1, 120))
        v = (rng.integers(-3, 4, n).astype(float) if t % 3 == 0 else rng.standard_normal(n) if t % 3 == 1
             else np.round(rng.random(n), 2))
        k, sep = int(rng.integers(1, 10)), int(rng.integers(0, 5))
        c, h, b, sf = R.extract_peaks(v, k, sep)
        ps = oracle.extract_peaks(v, k, sep)
        assert (c, h, b, sf) == (ps.cells, ps.heights, ps.baseline, ps.shortfall), (n, k, sep)


def test_live_reference_estimators(oracle):
    R = _ref()
    rng = np.random.default_rng(78)
    for t in range(12):
        m = int(rng.integers(8, 48))
        y = rng.standard_normal((m, 2 * m)) + 1j * rng.standard_normal((m, 2 * m))
        s_ref = R.spatial_covariance(y)
        s = oracle.spatial_covariance(y)
        assert np.linalg.norm(s - s_ref) <= 1e-14 * np.linalg.norm(s)
        k = int(rng.integers(1, 4))
        p = int(rng.integers(k, min(m, 12) + 1))
        seed = int(rng.integers(0, 2**63))
        st, b, e, _ = R.fast_music_2(s_ref, k, p, 2, seed)
        assert st == 0
        est = oracle.fast_music_2(s, k, p, 2, seed)
        assert oracle.projector_error(est.basis, b) < 1e-9
        b1, e1 = R.fast_music_1(s_ref, k, p, seed)
        est1 = oracle.fast_music_1(s, k, p, seed)
        assert oracle.projector_error(est1.basis, b1) < 1e-9
        bx, ex = R.exact_signal_subspace(s_ref, k)
        assert oracle.projector_error(oracle.exact_signal_subspace(s, k).basis, bx) < 1e-9
        spec = R.music_spectrum(b, 721)
        assert np.max(np.abs(oracle.music_spectrum(b, oracle.AngleGrid(721)) - spec) / spec) < 1e-9


def test_live_reference_run_frame_matches_port(oracle):
    """The CPU reference arm of bench.py (oracle/_ref ref_run_frame: the reference's covariance -> estimator ->
    music_spectrum on AngleGrid(L) = [0, pi] -> extract_peaks) agrees with the port on the same grid."""
    from oracle import ref_lib
    if not ref_lib.available():
        pytest.skip("oracle/_ref/libref_fastmusic.so not built (reference tree absent)")
    cfg = oracle.baseline_configs()["c1"]
    x, _, _ = oracle.generate_batch(cfg.base_seed, [0], cfg.spec)
    seed = oracle.derive(oracle.frame_seed(cfg.base_seed, 0), 4)
    st, cells, spec = ref_lib.run_frame(x[0], cfg.spec.k, "fast2", cfg.p, cfg.t, seed, cfg.grid_size, spectrum=True)
    assert st == 0
    grid = oracle.AngleGrid(cfg.grid_size)
    est, p, pk = oracle.run_frame(cfg, x[0], 0, grid)
    assert np.max(np.abs(p - spec) / spec) < 1e-8
    # [0, pi] is mirror-symmetric in sin(theta): theta and pi - theta peaks tie to rounding, either may rank first
    fold = lambda cs: sorted(min(c, cfg.grid_size - 1 - c) for c in cs)  # noqa: E731
    assert fold(cells) == fold(pk.cells)
    for method in ("exact", "lanczos"):
        st, c2, _ = ref_lib.run_frame(x[0], cfg.spec.k, method, 0, 200, 0, cfg.grid_size)
        assert st == 0 and len(c2) == cfg.spec.k
