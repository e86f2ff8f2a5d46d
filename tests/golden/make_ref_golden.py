"""Generate tests/golden/ref_golden.npz from the REFERENCE's own code compiled here (oracle/_ref/libref_fastmusic.so:
R/src/{scene,linalg,estimators,spectrum}.cpp built in place against oracle/eigen_shim; see oracle/ref_lib.py).
Runs only where /root/reference was present at build time; the fixtures it writes are committed and checked by
tests/test_ref_golden.py (oracle restatement, CPU) and tests/test_gpu_ref_golden.py (GPU facade and batch paths).

  make -C oracle && python tests/golden/make_ref_golden.py

Contents (arrays prefixed by case name):
  peaks_*      extract_peaks (R/src/spectrum.cpp:97-188) on random / plateau / negative / long spectra
  est_*        exact / fast_music_1 / fast_music_2 on the reference's own unit-test matrices and a c1 frame
  frame_*      whole path on BASELINE frames (generator DESIGN.md §3, bit-pinned RNG): reference covariance ->
               estimator -> music_spectrum on the reference grid AngleGrid(L) = [0, pi] -> extract_peaks
  steer_*      steering_vector (R/src/scene.cpp:72-82)
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import fastmusic_oracle as O  # noqa: E402
from oracle import ref_lib as R  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ref_golden.npz")


def psd_with_spectrum(spec, seed):
    """Hermitian PSD matrix with the given spectrum and a seeded random unitary (the reference tests' fixture
    pattern, R/tests/test_estimators.cpp:20-44; our own seeded unitary)."""
    rng = np.random.default_rng(seed)
    n = len(spec)
    z = rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))
    q, _ = np.linalg.qr(z)
    s = (q * np.asarray(spec, float)) @ q.conj().T
    return 0.5 * (s + s.conj().T)


def gapped_spectrum(m, k, gap):
    v = np.empty(m)
    v[:k] = 1.0 + np.arange(k)[::-1] * 0.1
    v[k:] = gap * np.linspace(1.0, 0.1, m - k)
    return v


def main():
    if not R.available():
        raise SystemExit("oracle/_ref/libref_fastmusic.so missing: run `make -C oracle` where /root/reference exists")
    g = {}
    rng = np.random.default_rng(2024)
    # ---------------- peaks
    cases = []
    for t in range(400):
        n = int(rng.integers(1, 200))
        kind = t % 5
        if kind == 0:
            v = rng.random(n)
        elif kind == 1:
            v = rng.integers(0, 5, n).astype(float)          # plateau-heavy
        elif kind == 2:
            v = 10.0 * np.log10(rng.random(n) * 1e-3)       # dB scale, all negative
        elif kind == 3:
            v = rng.integers(-6, 0, n).astype(float)          # negative plateaus
        else:
            v = np.cumsum(rng.standard_normal(n))
        cases.append((v, int(rng.integers(1, 12)), int(rng.integers(0, 6))))
    for n, k, sep in ((3601, 8, 3), (18001, 16, 3), (3601, 100, 1), (30001, 40, 2)):
        cases.append((rng.random(n), k, sep))
        cases.append((rng.integers(0, 4, n).astype(float), k, sep))
    for i, (v, k, sep) in enumerate(cases):
        c, h, b, sf = R.extract_peaks(v, k, sep)
        g[f"peaks_{i}_values"] = v
        g[f"peaks_{i}_args"] = np.array([k, sep], np.int64)
        g[f"peaks_{i}_cells"] = np.array(c, np.int64)
        g[f"peaks_{i}_heights"] = np.array(h, np.float64)
        g[f"peaks_{i}_baseline_shortfall"] = np.array([b, float(sf)])
    g["peaks_count"] = np.array([len(cases)])
    # ---------------- estimators on the reference unit-test matrices
    ests = [
        ("exact_gapped", psd_with_spectrum(gapped_spectrum(24, 4, 0.3), 7), "exact", 4, 0, 0, 0),
        ("fast1_full", psd_with_spectrum(gapped_spectrum(24, 4, 0.3), 7), "fast1", 4, 24, 0, 1),
        ("fast1_rank2", psd_with_spectrum([3.0, 1.0] + [0.0] * 10, 11), "fast1", 2, 6, 0, 3),
        ("fast2_rank3", psd_with_spectrum([5.0, 2.5, 1.0] + [0.0] * 17, 13), "fast2", 3, 3, 1, 17),
        ("fast2_deep", psd_with_spectrum(gapped_spectrum(50, 3, 0.3), 15), "fast2", 3, 6, 10, 4),
        ("fast2_gapped", psd_with_spectrum(gapped_spectrum(16, 3, 0.2), 19), "fast2", 3, 5, 2, 7),
    ]
    names = []
    for name, s, method, k, p, t, seed in ests:
        if method == "exact":
            b, e = R.exact_signal_subspace(s, k)
            st = 0
        elif method == "fast1":
            b, e = R.fast_music_1(s, k, p, seed)
            st = 0
        else:
            st, b, e, _ = R.fast_music_2(s, k, p, t, seed)
        g[f"est_{name}_s"] = s
        g[f"est_{name}_args"] = np.array([k, p, t, seed, st], np.int64)
        g[f"est_{name}_method"] = np.array([{"exact": 0, "fast1": 1, "fast2": 2}[method]], np.int64)
        g[f"est_{name}_projector"] = b @ b.conj().T
        g[f"est_{name}_eig"] = e
        names.append(name)
    g["est_names"] = np.array(names)
    # all-zero covariance: fast2 exhausts its redraws (RankDeficiencyError, R/src/estimators.cpp:114-137)
    st, _, _, col = R.fast_music_2(np.zeros((8, 8), complex), 2, 3, 1, 5)
    g["est_zero_fast2_status_column"] = np.array([st, col], np.int64)
    # ---------------- whole path on BASELINE frames, reference grid [0, pi]
    cfgs = O.baseline_configs()
    frames = [("c1", 0), ("c2", 0), ("c2", 1), ("c3", 2), ("c5", 3)]
    fnames = []
    for cname, f in frames:
        cfg = cfgs[cname]
        x, _, _ = O.generate_batch(cfg.base_seed, [f], cfg.spec)
        s = R.spatial_covariance(x[0].astype(np.complex128))
        fin = O.frame_inputs(cfg, f)
        k = cfg.spec.k
        if cfg.method == "fast2":
            st, b, e, _ = R.fast_music_2(s, k, cfg.p, cfg.t, fin["seed"])
        elif cfg.method == "fast1":
            b, e = R.fast_music_1(s, k, cfg.p, fin["seed"])
        else:
            b, e = R.exact_signal_subspace(s, k)
        spec = R.music_spectrum(b, cfg.grid_size)
        c, h, base, sf = R.extract_peaks(spec, k, cfg.min_sep_cells)
        tag = f"{cname}_{f}"
        g[f"frame_{tag}_spectrum"] = spec
        g[f"frame_{tag}_cells"] = np.array(c, np.int64)
        g[f"frame_{tag}_eig"] = e
        g[f"frame_{tag}_cov_diag"] = np.real(np.diag(s))
        fnames.append(tag)
    g["frame_names"] = np.array(fnames)
    # ---------------- steering vectors
    for i, (th, m) in enumerate(((0.0, 8), (np.pi / 2, 9), (0.37, 64), (-1.2, 256), (3.0, 33))):
        g[f"steer_{i}"] = R.steering_vector(th, m)
        g[f"steer_{i}_args"] = np.array([th, m])
    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT}: {len(cases)} peak cases, {len(names)} estimator cases, {len(fnames)} frames")


if __name__ == "__main__":
    main()
