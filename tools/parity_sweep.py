"""Parity sweep: the batched GPU path vs the fp64 oracle on whole batches (every frame), for the BASELINE configs
and the stress regimes of tests/test_gpu_stress.py. One JSON line per case:

  config, frames, worst / p99 / median spectrum error (dB, where the oracle is within 40 dB of its max), frames
  with different peak cells, per-frame status counts, and the near-tie margin of the oracle spectra:
  for every selected peak, min over its neighbours of (P_peak - P_neighbour) / P_peak, and the rank margin
  (h_K - h_{K+1}) / h_K between the last selected peak and the best rejected candidate. A peak mismatch on a
  frame whose margin is below ~1e-5 is a tie the fp32-vs-fp64 difference may legitimately flip.

  python tools/parity_sweep.py [case ...] > profiles/rNN_parity_sweep.jsonl
"""
import json
import math
import os as _os

for _v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
    _os.environ.setdefault(_v, "1")  # one BLAS thread per oracle worker (the pool uses every core)
import os  # noqa: E402
import sys  # noqa: E402
from concurrent.futures import ProcessPoolExecutor  # noqa: E402

import numpy as np  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import fastmusic_oracle as O  # noqa: E402
from tests.gpu_helpers import run_gpu  # noqa: E402

_A = {}


def _amat(cfg):
    key = (cfg.spec.m, cfg.grid_size)
    if key not in _A:
        _A[key] = O.steering_matrix(O.baseline_grid(cfg.grid_size), cfg.spec.m)
    return _A[key]


def _margins(p, cells, k):
    """(min neighbour margin over the selected peaks, rank margin K vs K+1)."""
    nb = 1.0
    for c in cells:
        for d in (-1, 1):
            if 0 <= c + d < p.size:
                nb = min(nb, (p[c] - p[c + d]) / p[c])
    cands = sorted((float(h) for _, h in O.local_maxima(p)), reverse=True)
    rank = 1.0
    if len(cands) > k and cands[k - 1] > 0:
        rank = (cands[k - 1] - cands[k]) / cands[k - 1]
    return nb, rank


def _ref(args):
    cfg, i, f, xi = args
    est, p_ref, pk = O.run_frame(cfg, xi, f, O.baseline_grid(cfg.grid_size), _amat(cfg))
    nb, rank = _margins(p_ref, pk.cells, cfg.spec.k)
    return i, p_ref, pk.cells, nb, rank


def per_source(cfg, snr_db, frames=None):
    sp = cfg.spec
    tot = snr_db + 10.0 * math.log10(sp.k)
    spec = O.SceneSpec(sp.m, sp.n, sp.k, sp.theta_lo_deg, sp.theta_hi_deg, sp.min_sep_deg, tot, tot)
    return O.PathConfig(f"{cfg.name}_persource{int(snr_db)}dB", cfg.method, spec, frames or cfg.frames,
                        cfg.grid_size, p=cfg.p, t=cfg.t, base_seed=cfg.base_seed + 100 + int(snr_db))


def cases():
    c = O.baseline_configs()
    out = {name: (c[name], 1.0) for name in ("c1", "c2", "c3", "c4", "c5", "c3n", "c2lz")}
    for s in (-20, -12, 12):
        cfg = c["c2"]
        out[f"c2_scale2^{s}"] = (cfg, 2.0 ** s)
    out["c2_persource30dB"] = (per_source(c["c2"], 30.0), 1.0)
    out["c2_persource40dB"] = (per_source(c["c2"], 40.0), 1.0)
    out["c4_persource30dB"] = (per_source(c["c4"], 30.0, 64), 1.0)
    spec = O.SceneSpec(64, 12, 3, -60.0, 60.0, 4.0, 15.0, 25.0)
    out["fast1_M64_N12_p16"] = (O.PathConfig("fast1_n12", "fast1", spec, 256, 721, p=16, base_seed=41), 1.0)
    return out


def run_case(fm, name, cfg, scale):
    frames = list(range(cfg.frames))
    x, _, _ = O.generate_batch(cfg.base_seed, frames, cfg.spec)
    if scale != 1.0:
        x = (x * np.float32(scale)).astype(np.complex64)
    res = run_gpu(fm, O, cfg, x, frames, basis=False)
    workers = min(os.cpu_count() or 1, 48 if cfg.spec.m <= 256 else 8)  # c4's steering table is 295 MB / worker
    with ProcessPoolExecutor(max_workers=workers) as ex:
        refs = sorted(ex.map(_ref, [(cfg, i, f, x[i]) for i, f in enumerate(frames)], chunksize=2))
    errs, mism, nbm, rkm = [], [], [], []
    for i, p_ref, cells, nb, rank in refs:
        errs.append(O.spectrum_db_error(res["spectrum"][i].astype(np.float64), p_ref))
        nbm.append(nb)
        rkm.append(rank)
        got = [int(v) for v in res["peak_cells"][i][: int(res["peak_count"][i])]]
        if got != cells:
            mism.append({"frame": frames[i], "gpu": got, "oracle": cells, "nb_margin": nb, "rank_margin": rank})
    e = np.array(errs)
    st = res["status"]
    return {"case": name, "config": cfg.name, "method": cfg.method, "frames": len(frames), "scale": scale,
            "worst_db": float(e.max()), "p99_db": float(np.percentile(e, 99)), "median_db": float(np.median(e)),
            "n_mismatch": len(mism), "mismatches": mism[:10], "status_nonzero": int(np.count_nonzero(st)),
            "status_values": sorted({int(v) for v in st}),
            "min_neighbour_margin": float(np.min(nbm)), "min_rank_margin": float(np.min(rkm)),
            "gate": {"db": 0.05, "pass": bool(e.max() <= 0.05 and not mism and not np.count_nonzero(st))}}


_B = {}


def _toa_ref(args):
    cfg, i, f, xi = args
    if "b" not in _B:
        _B["b"] = O.beat_steering_matrix(O.beat_grid(cfg.grid_size, cfg.w0, cfg.w1), cfg.spec.n)
    est, p_ref, pk = O.run_toa_frame(cfg, xi, f, _B["b"])
    nb, rank = _margins(p_ref, pk.cells, cfg.spec.k)
    return i, p_ref, pk.cells, nb, rank


def run_toa_case(fm):
    """The ToA path (FM_PLAN_TEMPORAL) on a whole 1024-frame batch of seeded beat frames vs the oracle."""
    import torch
    cfg = O.ToaConfig()
    frames = list(range(cfg.frames))
    x, _ = O.generate_toa_batch(cfg.base_seed, frames, cfg.spec)
    sp = cfg.spec
    plan = fm.BatchPlan(sp.m, sp.n, sp.k, "fast2", p=cfg.p, t=cfg.t, grid_size=cfg.grid_size, theta0=cfg.w0,
                        theta1=cfg.w1, min_sep_cells=cfg.min_sep_cells, max_frames=len(frames), temporal=True)
    om = torch.from_numpy(fm.draw_omega_batch([fm.derive(O.frame_seed(cfg.base_seed, f), 4) for f in frames],
                                              sp.n, cfg.p)).cuda()
    out = plan.outputs(len(frames), spectrum=True)
    plan.run(len(frames), torch.from_numpy(np.ascontiguousarray(x).view(np.float32)).cuda(), om, None, out)
    torch.cuda.synchronize()
    res = {k: v.cpu().numpy() for k, v in out.items()}
    with ProcessPoolExecutor(max_workers=min(os.cpu_count() or 1, 16)) as ex:
        refs = sorted(ex.map(_toa_ref, [(cfg, i, f, x[i]) for i, f in enumerate(frames)], chunksize=4))
    errs, mism, nbm, rkm = [], [], [], []
    for i, p_ref, cells, nb, rank in refs:
        errs.append(O.spectrum_db_error(res["spectrum"][i].astype(np.float64), p_ref))
        nbm.append(nb)
        rkm.append(rank)
        got = [int(v) for v in res["peak_cells"][i][: int(res["peak_count"][i])]]
        if got != cells:
            mism.append({"frame": frames[i], "gpu": got, "oracle": cells, "nb_margin": nb, "rank_margin": rank})
    e = np.array(errs)
    st = res["status"]
    return {"case": "toa", "config": "toa", "method": "fast2 on T = X^H X / M", "frames": len(frames), "scale": 1.0,
            "worst_db": float(e.max()), "p99_db": float(np.percentile(e, 99)), "median_db": float(np.median(e)),
            "n_mismatch": len(mism), "mismatches": mism[:10], "status_nonzero": int(np.count_nonzero(st)),
            "status_values": sorted({int(v) for v in st}),
            "min_neighbour_margin": float(np.min(nbm)), "min_rank_margin": float(np.min(rkm)),
            "gate": {"db": 0.05, "pass": bool(e.max() <= 0.05 and not mism and not np.count_nonzero(st))}}


def main():
    import paper_1911_07434_b200 as fm
    all_cases = cases()
    names = sys.argv[1:] or list(all_cases) + ["toa"]
    for n in names:
        if n == "toa":
            print(json.dumps(run_toa_case(fm)), flush=True)
            continue
        cfg, scale = all_cases[n]
        print(json.dumps(run_case(fm, n, cfg, scale)), flush=True)


if __name__ == "__main__":
    main()
