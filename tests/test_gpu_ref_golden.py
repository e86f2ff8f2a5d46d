"""GPU paths against the REFERENCE's own code: golden vectors from R/src/{scene,linalg,estimators,spectrum}.cpp
compiled here in place (tests/golden/make_ref_golden.py; oracle/_ref is not needed on the GPU box).

* fm_z_extract_peaks (the batch path's peak kernel) — bit-exact on every golden case, incl. dB-scale / negative
  spectra, plateaus, K up to 300 and grids whose workspace leaves shared memory (L = 30001).
* fp64 facade estimators — the reference's own tolerance (projector error 1e-8, R/tests/test_estimators.cpp).
* whole path on BASELINE frames on the reference grid AngleGrid(L) = [0, pi]: the fp64 facade chain
  (covariance -> estimator -> spectrum -> peaks) to fp64 agreement, and the batched complex64 pipeline
  (fm_run_batch with a [0, pi] plan grid) under the BASELINE gate (identical peaks, 0.05 dB within 40 dB).
"""
import numpy as np
import pytest

from tests.ref_golden import est_cases, frame_cases, load, peak_cases

pytestmark = pytest.mark.gpu
G = load()


def test_gpu_peaks_bit_exact_vs_reference(fm):
    for v, k, sep, cells, heights, base, sf in peak_cases(G):
        ps = fm.extract_peaks(fm.PseudoSpectrum(fm.AngleGrid(max(len(v), 2)), v), k, sep)
        assert ps.cells == cells and ps.heights == heights, (len(v), k, sep)
        assert ps.baseline == base and ps.shortfall == sf, (len(v), k, sep)


def test_gpu_facade_estimators_vs_reference(fm):
    for name, s, method, k, p, t, seed, st, proj, eig in est_cases(G):
        if method == "exact":
            est = fm.exact_signal_subspace(s, k)
        elif method == "fast1":
            est = fm.fast_music_1(s, k, fm.Fast1Params(p, seed))
        else:
            est = fm.fast_music_2(s, k, fm.Fast2Params(p, t, seed))
        b = est.basis
        assert np.linalg.norm(b @ b.conj().T - proj, 2) < 1e-8, name
        assert np.allclose(est.eigenvalues, eig, rtol=1e-8, atol=1e-10), name
    with pytest.raises(fm.RankDeficiencyError):
        fm.fast_music_2(np.zeros((8, 8), complex), 2, fm.Fast2Params(3, 1, 5))


def test_gpu_facade_frames_vs_reference(fm, oracle):
    cfgs = oracle.baseline_configs()
    for cname, f, spec, cells, eig in frame_cases(G):
        cfg = cfgs[cname]
        x, _, _ = oracle.generate_batch(cfg.base_seed, [f], cfg.spec)
        s = fm.spatial_covariance(x[0])
        seed = oracle.frame_inputs(cfg, f).get("seed", 0)
        if cfg.method == "fast2":
            est = fm.fast_music_2(s, cfg.spec.k, fm.Fast2Params(cfg.p, cfg.t, seed))
        elif cfg.method == "fast1":
            est = fm.fast_music_1(s, cfg.spec.k, fm.Fast1Params(cfg.p, seed))
        else:
            est = fm.exact_signal_subspace(s, cfg.spec.k)
        grid = fm.AngleGrid(cfg.grid_size)  # [0, pi]
        p = fm.music_spectrum(est, grid, 0.5, 1.0)
        assert np.max(np.abs(p.values - spec) / spec) < 1e-7, (cname, f)
        assert fm.extract_peaks(p, cfg.spec.k, cfg.min_sep_cells).cells == cells, (cname, f)


def test_gpu_batch_frames_vs_reference(fm, oracle):
    import torch
    from tests.gpu_helpers import draws
    cfgs = oracle.baseline_configs()
    for cname, f, spec, cells, eig in frame_cases(G):
        cfg = cfgs[cname]
        x, _, _ = oracle.generate_batch(cfg.base_seed, [f], cfg.spec)
        sp = cfg.spec
        plan = fm.BatchPlan(sp.m, sp.n, sp.k, cfg.method, p=cfg.p, t=cfg.t, grid_size=cfg.grid_size, theta0=0.0,
                            theta1=oracle.KPI, min_sep_cells=cfg.min_sep_cells, max_frames=1)
        om, ix = draws(fm, oracle, cfg, [f])
        out = plan.outputs(1, spectrum=True, basis=True)
        plan.run(1, torch.from_numpy(np.ascontiguousarray(x).view(np.float32)).cuda(),
                 torch.from_numpy(om).cuda() if om is not None else None,
                 torch.from_numpy(ix).cuda() if ix is not None else None, out)
        torch.cuda.synchronize()
        res = {k: v.cpu().numpy() for k, v in out.items()}
        plan.close()
        assert res["status"][0] == 0, (cname, f)
        n = int(res["peak_count"][0])
        assert [int(c) for c in res["peak_cells"][0][:n]] == cells, (cname, f)
        assert oracle.spectrum_db_error(res["spectrum"][0].astype(np.float64), spec) <= 0.05, (cname, f)
        assert np.allclose(res["eigenvalues"][0], eig, rtol=1e-3), (cname, f)
