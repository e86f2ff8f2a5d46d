"""Stress parity of the batched complex64 path in the regimes where it could diverge from the fp64 reference
(VERDICT r1 "what's weak" #2): input scale, high per-source SNR (ill-conditioned sketches), and singular
Nystrom blocks (N < p, exactly low-rank covariance). Every frame must come back with status 0 and, on the
host path, after the first draw (attempts = 1), with the oracle's peak cells and spectra within 0.05 dB.

* Scale: MUSIC is scale-free and the reference is fp64; the covariance converter rescales out-of-range frames
  by a power of two (cov_tc.cu rescue pass), so X * 2^-20 .. X * 2^12 give the unscaled answer.
* Per-source SNR (sigma^2 = 10^(-SNR/10)): = the reference convention at SNR + 10 log10 K.
  kappa(C) ~ 1e5..1e7 here; the rank rule runs at the fp64 Gram's resolution (fm_common.cuh cholqr_rank) and a
  near-singular H goes to the exact-algebra fallback (final_fallback.cu) instead of failing the frame.
* fast1 with N < p, and the exactly-rank-2 case of R/tests/test_estimators.cpp:117-126: S(I, I) is singular;
  the reference truncates in pseudo_inverse (R/src/linalg.cpp:143-163) and so does the batch path.
"""
import math

import numpy as np
import pytest

from tests.gpu_helpers import compare_frames, compare_frames_parallel, draws, plan_for, run_gpu

pytestmark = pytest.mark.gpu

DB_TOL = 0.05


@pytest.fixture(scope="module")
def cfgs(oracle):
    return oracle.baseline_configs()


def _per_source(oracle, cfg, snr_db, frames, grid=None):
    """cfg with fixed per-source SNR (sigma^2 = 10^(-SNR/10)) = reference convention at SNR + 10 log10 K."""
    sp = cfg.spec
    tot = snr_db + 10.0 * math.log10(sp.k)
    spec = oracle.SceneSpec(sp.m, sp.n, sp.k, sp.theta_lo_deg, sp.theta_hi_deg, sp.min_sep_deg, tot, tot)
    return oracle.PathConfig(f"{cfg.name}_ps{int(snr_db)}", cfg.method, spec, frames, grid or cfg.grid_size,
                             p=cfg.p, t=cfg.t, base_seed=cfg.base_seed + 100 + int(snr_db))


def _host(fm, cfg, x, frames):
    """fm_estimate_batch_host on pinned host X (redraw policy included)."""
    import torch
    nf = len(frames)
    plan = plan_for(fm, cfg, nf)
    pinned = torch.empty((nf, cfg.spec.m, cfg.spec.n), dtype=torch.complex64).pin_memory().numpy()
    pinned[:] = x
    seeds = np.array([fm.derive(fm.derive(cfg.base_seed, f), 4 if cfg.method == "fast2" else 3) for f in frames],
                     np.uint64)
    spec = np.empty((nf, cfg.grid_size), np.float32)
    res = plan.estimate_host(pinned, seeds, spectrum=spec)
    plan.close()
    return res


@pytest.mark.parametrize("scale_log2", [-20, -12, 12])
def test_scaled_frames_match_unscaled(fm, oracle, cfgs, scale_log2):
    cfg = cfgs["c2"]
    frames = list(range(48))
    x, _, _ = oracle.generate_batch(cfg.base_seed, frames, cfg.spec)
    xs = (x * np.float32(2.0 ** scale_log2)).astype(np.complex64)
    res = run_gpu(fm, oracle, cfg, xs, frames)
    assert np.all(res["status"] == 0), res["status"]
    worst, mism = compare_frames(oracle, cfg, xs, frames[:12], {k: v[:12] for k, v in res.items()})
    assert not mism, mism
    assert worst <= DB_TOL, worst
    base = run_gpu(fm, oracle, cfg, x, frames)
    assert np.array_equal(res["peak_cells"], base["peak_cells"])
    # power-of-two prescale: the covariance differs from the unscaled one only by the exact factor 2^(2s)
    db = [oracle.spectrum_db_error(res["spectrum"][i].astype(np.float64), base["spectrum"][i].astype(np.float64))
          for i in range(len(frames))]
    assert max(db) < 1e-3, max(db)
    host = _host(fm, cfg, xs, frames)
    assert np.all(host["status"] == 0) and np.all(host["attempts"] == 1)
    assert np.array_equal(host["peak_cells"], res["peak_cells"])


def test_out_of_range_frames_flagged(fm, oracle, cfgs):
    """Beyond 2^+-50 the complex64 covariance itself would under/overflow: those frames (and only they) are
    flagged FM_FRAME_RANGE; non-finite frames FM_FRAME_NONFINITE."""
    from paper_1911_07434_b200 import _capi
    cfg = cfgs["c2"]
    frames = list(range(6))
    x, _, _ = oracle.generate_batch(cfg.base_seed, frames, cfg.spec)
    x = x.copy()
    x[1] *= np.float32(2.0 ** -70)
    x[3] *= np.float32(2.0 ** 60)
    x[4, 7, 9] = np.nan
    res = run_gpu(fm, oracle, cfg, x, frames)
    assert res["status"][1] & _capi.FRAME_RANGE and res["status"][3] & _capi.FRAME_RANGE
    assert res["status"][4] & _capi.FRAME_NONFINITE
    for f in (0, 2, 5):
        assert res["status"][f] == 0


@pytest.mark.parametrize("snr_db", [30.0, 40.0])
def test_per_source_snr_c2_all_frames(fm, oracle, cfgs, snr_db):
    cfg = _per_source(oracle, cfgs["c2"], snr_db, 1024)
    frames = list(range(1024))
    x, _, _ = oracle.generate_batch(cfg.base_seed, frames, cfg.spec)
    res = run_gpu(fm, oracle, cfg, x, frames, basis=False)
    assert np.all(res["status"] == 0), np.flatnonzero(res["status"])
    worst, mism, _ = compare_frames_parallel(cfg, x, frames, res)
    assert not mism, mism[:5]
    assert worst <= DB_TOL, worst
    host = _host(fm, cfg, x, frames)
    assert np.all(host["status"] == 0) and np.all(host["attempts"] == 1)
    assert np.array_equal(host["peak_cells"], res["peak_cells"])


def test_per_source_snr_c4(fm, oracle, cfgs):
    cfg = _per_source(oracle, cfgs["c4"], 30.0, 4)
    frames = list(range(4))
    x, _, _ = oracle.generate_batch(cfg.base_seed, frames, cfg.spec)
    res = run_gpu(fm, oracle, cfg, x, frames, basis=False)
    assert np.all(res["status"] == 0), res["status"]
    worst, mism, _ = compare_frames_parallel(cfg, x, frames, res, procs=4)
    assert not mism, mism
    assert worst <= DB_TOL, worst


def test_fast1_fewer_snapshots_than_columns(fm, oracle):
    """fast1, M = 64, N = 12 < p = 16: rank(R) = 12, every S(I, I) is singular (reference: truncating pinv)."""
    spec = oracle.SceneSpec(64, 12, 3, -60.0, 60.0, 4.0, 15.0, 25.0)
    cfg = oracle.PathConfig("fast1_n12", "fast1", spec, 16, 721, p=16, base_seed=41)
    frames = list(range(16))
    x, _, _ = oracle.generate_batch(cfg.base_seed, frames, cfg.spec)
    res = run_gpu(fm, oracle, cfg, x, frames)
    assert np.all(res["status"] == 0), res["status"]
    worst, mism = compare_frames(oracle, cfg, x, frames, res)
    assert not mism, mism
    assert worst <= DB_TOL, worst


def test_fast1_exactly_rank_two_block(fm, oracle):
    """R/tests/test_estimators.cpp:117-126 in batch form: S = Q diag(3, 1, 0, ..) Q^H (M = 12) given as
    X = Q(:, :2) diag(sqrt(6), sqrt(2)) with N = 2 (S = X X^H / 2), fast1 p = 6, seed 3, K = 2: the result must
    be the exact signal subspace (projector error at the fp16-operand level)."""
    import torch
    rng = np.random.default_rng(11)
    z = rng.standard_normal((12, 12)) + 1j * rng.standard_normal((12, 12))
    q, _ = np.linalg.qr(z)
    xf = (q[:, :2] * np.array([math.sqrt(6.0), math.sqrt(2.0)])).astype(np.complex64)
    s = xf.astype(np.complex128) @ xf.astype(np.complex128).conj().T / 2.0
    exact = oracle.exact_signal_subspace(s, 2)
    frames = 3
    x = np.stack([xf] * frames)
    plan = fm.BatchPlan(12, 2, 2, "fast1", p=6, grid_size=721, max_frames=frames)
    idx = np.stack([oracle.sample_without_replacement(3, 12, 6)] * frames).astype(np.int32)
    xd = torch.from_numpy(np.ascontiguousarray(x).view(np.float32)).cuda()
    out = plan.outputs(frames, spectrum=True, basis=True)
    plan.run(frames, xd, None, torch.from_numpy(idx).cuda(), out)
    torch.cuda.synchronize()
    res = {k: v.cpu().numpy() for k, v in out.items()}
    plan.close()
    assert np.all(res["status"] == 0), res["status"]
    ref = oracle.fast_music_1(s, 2, 6, 3)
    grid = oracle.baseline_grid(721)
    p_ref = oracle.music_spectrum(ref.basis, grid)
    for f in range(frames):
        u = (res["basis"][f][..., 0] + 1j * res["basis"][f][..., 1]).T
        assert oracle.projector_error(u, exact.basis) < 5e-3
        assert oracle.spectrum_db_error(res["spectrum"][f].astype(np.float64), p_ref) <= DB_TOL
    assert oracle.projector_error(ref.basis, exact.basis) < 1e-7  # the reference's own tolerance
