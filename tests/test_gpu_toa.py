"""ToA path on the GPU (FM_PLAN_TEMPORAL): T = X^H X / M by the tensor-core covariance kernel reading
X in its stored order, the batched fast_music_2 on T (dimension N), the beat spectrum exp(-j w n) and the peaks,
against the fp64 oracle (tests/test_toa_oracle.py pins it to the reference's own code): identical peak cells and
spectra within 0.05 dB wherever the oracle spectrum is within 40 dB of its maximum."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _run_toa(fm, oracle, cfg, x, frames, covariance=False):
    import torch
    sp = cfg.spec
    nf = len(frames)
    plan = fm.BatchPlan(sp.m, sp.n, sp.k, cfg.method, p=cfg.p, t=cfg.t, grid_size=cfg.grid_size, theta0=cfg.w0,
                        theta1=cfg.w1, min_sep_cells=cfg.min_sep_cells, max_frames=nf, temporal=True)
    seeds = [fm.derive(oracle.frame_seed(cfg.base_seed, f), 4) for f in frames]
    om = torch.from_numpy(fm.draw_omega_batch(seeds, sp.n, cfg.p)).cuda()
    xd = torch.from_numpy(np.ascontiguousarray(x).view(np.float32)).cuda()
    out = plan.outputs(nf, spectrum=True, covariance=covariance)
    plan.run(nf, xd, om, None, out)
    torch.cuda.synchronize()
    res = {k: v.cpu().numpy() for k, v in out.items()}
    plan.close()
    return res


def _compare(oracle, cfg, x, frames, res):
    w = oracle.beat_grid(cfg.grid_size, cfg.w0, cfg.w1)
    bm = oracle.beat_steering_matrix(w, cfg.spec.n)
    worst, mism = 0.0, []
    for i, f in enumerate(frames):
        _, p_ref, pk = oracle.run_toa_frame(cfg, x[i], f, b_mat=bm)
        worst = max(worst, oracle.spectrum_db_error(res["spectrum"][i].astype(np.float64), p_ref))
        n = int(res["peak_count"][i])
        cells = [int(c) for c in res["peak_cells"][i][:n]]
        if cells != pk.cells:
            mism.append((f, cells, pk.cells))
    return worst, mism


def test_toa_full_shape(fm, oracle):
    """The bench's ToA workload shape (M = 256 antennas, N = 512 samples -> T is 512 x 512), 8 frames."""
    cfg = oracle.ToaConfig()
    frames = list(range(8))
    x, _ = oracle.generate_toa_batch(cfg.base_seed, frames, cfg.spec)
    res = _run_toa(fm, oracle, cfg, x, frames)
    assert np.all(res["status"] == 0), res["status"]
    worst, mism = _compare(oracle, cfg, x, frames, res)
    assert not mism, mism
    assert worst <= 0.05, worst


@pytest.mark.parametrize("m,n,k,p", [(64, 128, 4, 8), (48, 200, 3, 12), (33, 77, 2, 6), (300, 96, 5, 16)])
def test_toa_shapes(fm, oracle, m, n, k, p):
    """T on the fp16-plane path (N <= 256), odd N (padded rows, generic-store epilogue), odd M, M > N."""
    spec = oracle.ToaSpec(m=m, n=n, k=k, min_sep=0.3)
    cfg = oracle.ToaConfig(spec=spec, p=p, grid_size=1801, frames=6)
    frames = list(range(6))
    x, _ = oracle.generate_toa_batch(cfg.base_seed, frames, spec)
    res = _run_toa(fm, oracle, cfg, x, frames, covariance=True)
    assert np.all(res["status"] == 0), res["status"]
    c = res["covariance"]
    for i in range(len(frames)):
        ref = oracle.temporal_covariance(x[i])
        got = c[i][..., 0] + 1j * c[i][..., 1]
        assert np.linalg.norm(got - ref) / np.linalg.norm(ref) < 2e-4, i
    worst, mism = _compare(oracle, cfg, x, frames, res)
    assert not mism, mism
    assert worst <= 0.05, worst


def test_toa_plan_validation(fm):
    """K and p are checked against N (the dimension of T), not M."""
    with pytest.raises(ValueError):
        fm.BatchPlan(8, 16, 16, "fast2", p=16, t=1, temporal=True)  # K < N violated
    plan = fm.BatchPlan(4, 64, 8, "fast2", p=16, t=1, temporal=True)  # K > M is fine: T is 64 x 64
    plan.close()
