"""Shared helpers for the GPU parity tests (oracle = checker only)."""
import numpy as np


def plan_for(fm, cfg, frames):
    sp = cfg.spec
    return fm.BatchPlan(sp.m, sp.n, sp.k, cfg.method, p=cfg.p, t=cfg.t, grid_size=cfg.grid_size,
                        min_sep_cells=cfg.min_sep_cells, max_frames=frames)


def draws(fm, oracle, cfg, frames):
    fseeds = [oracle.frame_seed(cfg.base_seed, f) for f in frames]
    if cfg.method == "fast2":
        return fm.draw_omega_batch([fm.derive(s, 4) for s in fseeds], cfg.spec.m, cfg.p), None
    if cfg.method == "fast1":
        return None, fm.draw_indices_batch([fm.derive(s, 3) for s in fseeds], cfg.spec.m, cfg.p)
    if cfg.method == "fast1_norm2":  # uniforms travel in the omega slot
        return fm.draw_uniforms_batch([fm.derive(s, 3) for s in fseeds], cfg.spec.m), None
    return None, None


def run_gpu(fm, oracle, cfg, x, frames, basis=True, covariance=False):
    import torch
    nf = len(frames)
    plan = plan_for(fm, cfg, nf)
    om, ix = draws(fm, oracle, cfg, frames)
    xd = torch.from_numpy(np.ascontiguousarray(x).view(np.float32)).cuda()
    omd = torch.from_numpy(om).cuda() if om is not None else None
    ixd = torch.from_numpy(ix).cuda() if ix is not None else None
    out = plan.outputs(nf, spectrum=True, basis=basis, covariance=covariance)
    plan.run(nf, xd, omd, ixd, out)
    torch.cuda.synchronize()
    res = {k: v.cpu().numpy() for k, v in out.items()}
    if basis:
        b = res["basis"]
        res["basis_c"] = (b[..., 0] + 1j * b[..., 1]).transpose(0, 2, 1)  # [f, M, K]
    if covariance:
        c = res["covariance"]
        res["cov_c"] = c[..., 0] + 1j * c[..., 1]
    plan.close()
    return res


def tie_margins(oracle, p, cells, k):
    """how close the oracle spectrum is to a tie. Returns (min over the selected peaks of
    (P_peak - P_neighbour) / P_peak, (h_K - h_{K+1}) / h_K between the last selected and the best rejected
    local maximum). A mismatch with a margin below ~1e-5 is a tie the fp32 spectrum may legitimately flip."""
    p = np.asarray(p, dtype=np.float64)
    nb = 1.0
    for c in cells:
        for d in (-1, 1):
            if 0 <= c + d < p.size and p[c] > 0:
                nb = min(nb, float((p[c] - p[c + d]) / p[c]))
    cands = sorted((float(h) for _, h in oracle.local_maxima(p)), reverse=True)
    rank = 1.0
    if len(cands) > k and cands[k - 1] > 0:
        rank = (cands[k - 1] - cands[k]) / cands[k - 1]
    return nb, rank


def compare_frames(oracle, cfg, x, frames, res, grid=None, a_mat=None, db_tol=0.05):
    """(worst spectrum error in dB, mismatches). Each mismatch is (frame, gpu cells, oracle cells,
    {"nb_margin", "rank_margin", "near_tie"}): near-ties are reported, never silently dropped."""
    grid = grid or oracle.baseline_grid(cfg.grid_size)
    worst = 0.0
    mismatched = []
    for i, f in enumerate(frames):
        est, p_ref, pk = oracle.run_frame(cfg, x[i], f, grid, a_mat)
        p_gpu = res["spectrum"][i].astype(np.float64)
        worst = max(worst, oracle.spectrum_db_error(p_gpu, p_ref))
        n = int(res["peak_count"][i])
        cells = [int(c) for c in res["peak_cells"][i][:n]]
        if cells != pk.cells:
            nb, rank = tie_margins(oracle, p_ref, pk.cells, cfg.spec.k)
            mismatched.append((f, cells, pk.cells,
                               {"nb_margin": nb, "rank_margin": rank, "near_tie": min(nb, rank) < 1e-5}))
    return worst, mismatched


def _oracle_job(args):
    from oracle import fastmusic_oracle as O
    cfg, xf, f, p_gpu, cells = args
    est, p_ref, pk = O.run_frame(cfg, xf, f)
    db = O.spectrum_db_error(p_gpu, p_ref)
    same = cells == pk.cells
    tie = None
    if not same:
        nb, rank = tie_margins(O, p_ref, pk.cells, cfg.spec.k)
        tie = {"nb_margin": nb, "rank_margin": rank, "near_tie": min(nb, rank) < 1e-5}
    return f, db, same, pk.cells, tie


def compare_frames_parallel(cfg, x, frames, res, procs=None):
    """compare_frames over many frames with a process pool (the fp64 oracle is the slow side).
    Returns (worst dB, [(frame, gpu cells, oracle cells)] mismatches, per-frame dB list)."""
    import concurrent.futures as cf
    import multiprocessing as mp
    import os
    jobs = []
    for i, f in enumerate(frames):
        n = int(res["peak_count"][i])
        jobs.append((cfg, x[i], f, res["spectrum"][i].astype(np.float64), [int(c) for c in res["peak_cells"][i][:n]]))
    procs = procs or min(32, os.cpu_count() or 1)
    worst, mism, dbs = 0.0, [], []
    with cf.ProcessPoolExecutor(procs, mp_context=mp.get_context("fork")) as ex:
        for (f, db, same, ref_cells, tie), job in zip(ex.map(_oracle_job, jobs, chunksize=4), jobs):
            worst = max(worst, db)
            dbs.append(db)
            if not same:
                mism.append((f, job[4], ref_cells, tie))
    return worst, mism, dbs
