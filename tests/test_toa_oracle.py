"""ToA path oracle against the REFERENCE's own code: golden vectors from tests/golden/toa_golden.npz
(temporal_covariance -> fast_music_2 on T -> music_spectrum at d = lambda / 2, which is the beat spectrum at
w = -pi sin(theta) -> extract_peaks, all compiled from R/src here), plus live checks when oracle/_ref exists."""
import os

import numpy as np
import pytest

G = dict(np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "toa_golden.npz")))


def _cases():
    for i in range(int(G["toa_count"][0])):
        m, n, k, p, t, L, seed = (int(v) for v in G[f"toa_{i}_args"])
        yield i, m, n, k, p, t, L, seed


def test_golden_toa_path_oracle(oracle):
    for i, m, n, k, p, t, L, seed in _cases():
        x = G[f"toa_{i}_x"]
        tm = oracle.temporal_covariance(x)
        assert np.linalg.norm(tm - G[f"toa_{i}_t"]) <= 1e-14 * np.linalg.norm(tm), i
        est = oracle.fast_music_2(tm, k, p, t, seed)
        b = est.basis
        assert np.linalg.norm(b @ b.conj().T - G[f"toa_{i}_projector"], 2) < 1e-9, i
        assert np.allclose(est.eigenvalues, G[f"toa_{i}_eig"], rtol=1e-9, atol=1e-12), i
        th = oracle.AngleGrid(L).thetas()
        w = -(oracle.KPI * np.sin(th))  # the reference's step 2 pi (1/2) sin(theta) / 1 = pi sin(theta) = -w
        p_or = oracle.toa_spectrum(b, w)
        ref = G[f"toa_{i}_spectrum"]
        assert np.max(np.abs(p_or - ref) / ref) < 1e-9, i
        assert oracle.extract_peaks(ref, k, 3).cells == [int(c) for c in G[f"toa_{i}_cells"]]


def test_toa_frames_locate_beats(oracle):
    """Seeded beat frames: the oracle ToA path puts its K peaks on the true beat phases (to the grid cell and the
    finite-N bias), on the config's grid [0, pi]."""
    cfg = oracle.ToaConfig()
    spec = oracle.ToaSpec(m=64, n=128, k=4, min_sep=0.15)
    cfg = oracle.ToaConfig(spec=spec, p=8, grid_size=1801)
    w = oracle.beat_grid(cfg.grid_size, cfg.w0, cfg.w1)
    for f in range(3):
        x, wt = oracle.generate_toa_frame(oracle.frame_seed(cfg.base_seed, f), spec)
        _, p, pk = oracle.run_toa_frame(cfg, x, f)
        assert not pk.shortfall
        assert np.max(np.abs(np.sort(w[pk.cells]) - wt)) < 0.01, (f, w[pk.cells], wt)


def test_live_reference_temporal_covariance(oracle):
    from oracle import ref_lib
    if not ref_lib.available():
        pytest.skip("oracle/_ref/libref_fastmusic.so not built (reference tree absent)")
    rng = np.random.default_rng(5)
    for m, n in ((3, 7), (12, 5), (30, 41), (1, 6)):
        y = rng.standard_normal((m, n)) + 1j * rng.standard_normal((m, n))
        ref = ref_lib.temporal_covariance(y)
        got = oracle.temporal_covariance(y)
        assert np.linalg.norm(got - ref) <= 1e-14 * np.linalg.norm(ref)
        assert np.array_equal(ref, ref.conj().T)
