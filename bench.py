#!/usr/bin/env python
"""Fast-MUSIC B200 benchmark (driver contract).

Workload (BASELINE.json configs[1]): batches of 1024 frames per GPU,
ULA M=256, N=512 snapshots, K=8 sources, random-projection Fast-MUSIC p=16, t=2,
3601-point grid over [-90, 90] deg, complex64, synthetic seeded frames (no dataset).
A step = one pass of the hot path (covariance -> range finder -> Nystrom -> spectrum ->
peaks) over one batch already resident in HBM; X is 1 GiB per batch (> 126 MB L2), so no
L2 flush is needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c2]

Multi-GPU (torchrun, one process per GPU): frames are sharded (rank r owns frames
[r*B, (r+1)*B) of the stream, weak scaling); after each step the peak records are
all-gathered over NCCL (the path's only collective). Timing: CUDA events on the launching
stream, barrier + synchronize on both sides, max over ranks.
"""
from __future__ import annotations

import os

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")  # CPU baseline: one BLAS thread per worker
os.environ.setdefault("OMP_NUM_THREADS", "1")

import argparse  # noqa: E402
import json  # noqa: E402
import statistics  # noqa: E402
import subprocess  # noqa: E402
import sys  # noqa: E402
import time  # noqa: E402

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Fast-MUSIC frames/sec (M=256, 3601-pt grid); % of tensor/HBM roofline"

CONFIGS = {
    # name: (M, N, K, method, p, t, L, frames per GPU, base_seed, scene kwargs)
    "c1": dict(m=64, n=200, k=3, method="fast2", p=8, t=1, L=1801, frames=1, seed=1,
               scene=dict(fixed_angles_deg=(-20.0, 5.0, 31.0), snr_lo_db=20.0, snr_hi_db=20.0)),
    "c2": dict(m=256, n=512, k=8, method="fast2", p=16, t=2, L=3601, frames=1024, seed=2,
               scene=dict(theta_lo_deg=-60.0, theta_hi_deg=60.0, min_sep_deg=3.0, snr_lo_db=10.0, snr_hi_db=30.0)),
    "c3": dict(m=256, n=512, k=8, method="fast1", p=32, t=1, L=3601, frames=1024, seed=2,
               scene=dict(theta_lo_deg=-60.0, theta_hi_deg=60.0, min_sep_deg=3.0, snr_lo_db=10.0, snr_hi_db=30.0)),
    "c4": dict(m=1024, n=2048, k=16, method="fast2", p=32, t=2, L=18001, frames=256, seed=4,
               scene=dict(theta_lo_deg=-70.0, theta_hi_deg=70.0, min_sep_deg=1.0, snr_lo_db=20.0, snr_hi_db=20.0)),
    "c5": dict(m=256, n=512, k=8, method="exact", p=0, t=1, L=3601, frames=512, seed=2,
               scene=dict(theta_lo_deg=-60.0, theta_hi_deg=60.0, min_sep_deg=3.0, snr_lo_db=20.0, snr_hi_db=20.0)),
    # extension: config 3 with BASELINE's norm^2-weighted column sampling (not in the reference)
    "c3n": dict(m=256, n=512, k=8, method="fast1_norm2", p=32, t=1, L=3601, frames=1024, seed=2,
                scene=dict(theta_lo_deg=-60.0, theta_hi_deg=60.0, min_sep_deg=3.0, snr_lo_db=10.0, snr_hi_db=30.0)),
}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["hbm_gbs"], p["bf16_tflops"], p.get("bf16_tflops_sustained"), "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback"


def algorithmic(cfg):
    """SURVEY.md §8d per-frame work (real flops, complex MAC = 8) and bytes."""
    m, n, k, p, t, L = cfg["m"], cfg["n"], cfg["k"], cfg["p"], cfg["t"], cfg["L"]
    w_cov = 4.0 * m * (m + 1) * n
    if cfg["method"] == "fast2":
        w_rf = 4.0 * m * m * p + 8.0 * t * m * m * p
        q = 8.0 * m * n + 4.0 * m * p + 4.0 * L + 8.0 * k
    elif cfg["method"] == "fast1":
        w_rf = 0.0
        q = 8.0 * m * n + 8.0 * p + 4.0 * L + 8.0 * k
    elif cfg["method"] == "fast1_norm2":  # sampled sketch (a gather), one product R V
        w_rf = 8.0 * m * m * p
        q = 8.0 * m * n + 4.0 * m + 4.0 * L + 8.0 * k
    else:
        w_rf = 0.0
        q = 8.0 * m * n + 4.0 * L + 8.0 * k
    w_spec = 8.0 * k * m * L
    return {"w_cov": w_cov, "w_rf": w_rf, "w_spec": w_spec, "w_frame": w_cov + w_rf + w_spec, "q_frame": q}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-i", str(self.gpu), "-lms", "50"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        time.sleep(0.15)
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.proc:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = []
        for line in (self.out or "").splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        loaded = [s for s in sm if mx and s > 0.5 * max(mx)] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ----------------------------------------------------------------------------- CPU baseline
_W = {}


def _worker_init(cfg_name):
    from oracle import fastmusic_oracle as O
    cfg = O.baseline_configs()[cfg_name]
    grid = O.baseline_grid(cfg.grid_size)
    _W.update(O=O, cfg=cfg, grid=grid, A=O.steering_matrix(grid, cfg.spec.m))


def _worker_frame(args):
    f, x = args
    O, cfg = _W["O"], _W["cfg"]
    t0 = time.perf_counter()
    est, spec, pk = O.run_frame(cfg, x, f, _W["grid"], _W["A"])
    return f, pk.cells, spec.astype("float32"), time.perf_counter() - t0


def cpu_reference_run(cfg_name, xs, frames, cores, pool=None):
    """The oracle port (fp64 restatement of the reference path) over `frames`, one frame per
    worker at a time (R/src/bench.cpp:59-86 pattern); returns (wall_s, results)."""
    import multiprocessing as mp
    own = pool is None
    if own:
        pool = mp.get_context("fork").Pool(cores, initializer=_worker_init, initargs=(cfg_name,))
    t0 = time.perf_counter()
    res = pool.map(_worker_frame, [(f, xs[i]) for i, f in enumerate(frames)], chunksize=1)
    wall = time.perf_counter() - t0
    if own:
        pool.close()
        pool.join()
    return wall, res


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import multiprocessing as mp

    import numpy as np

    from oracle import fastmusic_oracle as O
    cfgd = CONFIGS[args.config]
    cfg = O.baseline_configs()[args.config]
    cores = os.cpu_count() or 1
    per_step = max(1, min(cfgd["frames"], cores))
    nsamp = per_step * 4
    xs, _, _ = O.generate_batch(cfg.base_seed, range(nsamp), cfg.spec)
    pool = mp.get_context("fork").Pool(cores, initializer=_worker_init, initargs=(args.config,))
    times = []
    for i in range(args.warmup + args.steps):
        sl = [(i * per_step + j) % nsamp for j in range(per_step)]
        wall, _ = cpu_reference_run(args.config, xs[sl], sl, cores, pool)
        if i >= args.warmup:
            times.append(wall)
    pool.close()
    pool.join()
    total = sum(times)
    value = per_step * len(times) / total
    line = {
        "metric": METRIC, "value": value, "unit": "frames/s", "impl": "reference", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / len(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128",
        "data": "synthetic (seeded BASELINE frame model, DESIGN.md §3)",
        "config": config_dict(args.config, cfgd, 1),
        "cpu_baseline": {"value": value, "unit": "frames/s", "cores": cores, "kind": "port",
                         "sample": f"{per_step} frames per step (one per core) of {args.config}; oracle fp64 "
                                   f"restatement of the reference path (numpy/scipy LAPACK, 1 BLAS thread/worker)"},
        "e2e": {"value": value, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def config_dict(name, cfgd, world):
    return {"workload": f"{name}: fast-MUSIC {cfgd['method']} M={cfgd['m']} N={cfgd['n']} K={cfgd['k']} "
                        f"p={cfgd['p']} t={cfgd['t']} L={cfgd['L']}",
            "frames_per_gpu": cfgd["frames"], "global_frames_per_step": cfgd["frames"] * world,
            "grid": "[-90, 90] deg", "l2": "inputs larger than L2 (X = %.2f GiB per GPU step)" %
            (cfgd["frames"] * cfgd["m"] * cfgd["n"] * 8 / 2**30),
            "parallelism": f"frames sharded over {world} GPU(s), NCCL all-gather of peak records"}


# ----------------------------------------------------------------------------- ours
def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1911_07434_b200 as fm
    from paper_1911_07434_b200.shard import gather_records, pack_records, shard_range

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    cfgd = CONFIGS[args.config]
    B, M, N, K, P, L = cfgd["frames"], cfgd["m"], cfgd["n"], cfgd["k"], cfgd["p"], cfgd["L"]
    if args.frames:
        B = args.frames
        cfgd = dict(cfgd, frames=B)
    f0, _ = shard_range(rank, world, B)
    # synthetic input for this rank's frames, generated on the host (pinned), staged once
    xh = torch.empty((B, M, N, 2), dtype=torch.float32, pin_memory=True)
    xnp = xh.numpy().view(np.complex64).reshape(B, M, N)
    fm.generate_frames(M, N, K, cfgd["seed"], f0, B, out=xnp, **cfgd["scene"])
    fseeds = np.array([fm.derive(cfgd["seed"], f0 + f) for f in range(B)], np.uint64)
    tag = 4 if cfgd["method"] == "fast2" else 3
    dseeds = np.array([fm.derive(int(s), tag) for s in fseeds], np.uint64)
    omega = idx = None
    if cfgd["method"] == "fast2":
        omega = torch.from_numpy(fm.draw_omega_batch(dseeds, M, P)).to(dev)
    elif cfgd["method"] == "fast1":
        idx = torch.from_numpy(fm.draw_indices_batch(dseeds, M, P)).to(dev)
    elif cfgd["method"] == "fast1_norm2":  # uniforms of the weighted sampler travel in the omega slot
        omega = torch.from_numpy(fm.draw_uniforms_batch(dseeds, M)).to(dev)
    xd = xh.to(dev)
    plan = fm.BatchPlan(M, N, K, cfgd["method"], p=P, t=cfgd["t"], grid_size=L, max_frames=B, device=local)
    # same rule as the library's automatic choice (capi.cu auto_subbatches): one sub-batch on the p <= 16 plane path
    plane_gram = cfgd["method"] in ("fast2", "fast1_norm2") and M <= 256 and P <= 16
    nsub = args.subbatches if args.subbatches > 0 else (1 if plane_gram or B < 512 else 2)
    plan.set_concurrency(nsub)
    fsub = (B + nsub - 1) // nsub  # frames in sub-batch 0 (the one the stage events time)
    out = plan.outputs(B, spectrum=True)
    stream = torch.cuda.Stream(device=dev)
    gather = None
    rec = torch.empty((B, K + 2), dtype=torch.int32, device=dev)
    if world > 1:
        gather = torch.empty((world, B, K + 2), dtype=torch.int32, device=dev)

    def step():
        plan.run(B, xd, omega, idx, out, stream=stream)
        if world > 1:
            with torch.cuda.stream(stream):
                pack_records(out["peak_cells"], out["peak_count"], out["status"], out=rec)
                gather_records(rec, world, out=gather)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    status = out["status"].cpu().numpy()
    counts = out["peak_count"].cpu().numpy()

    # ---------------- timed region
    plan.set_profiling(True)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    stage_sum, runs = plan.stage_times_ms()
    plan.set_profiling(False)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = world * B * args.steps / (ms_max / 1e3)

    # ---------------- e2e through the reference-facing host-buffer C-ABI call
    e2e = None
    if not args.no_e2e:
        draw = None if cfgd["method"] == "exact" else dseeds
        res = plan.estimate_host(xnp, draw)  # warm-up (allocates staging)
        e2e_steps = max(1, min(args.e2e_steps, args.steps))
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            res = plan.estimate_host(xnp, draw)
        el = time.perf_counter() - t0
        te = torch.tensor([el], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        h2d = B * M * N * 8 + (B * M * P * 4 if cfgd["method"] == "fast2" else B * P * 4 if cfgd["method"] == "fast1"
                               else B * M * 4 if cfgd["method"] == "fast1_norm2" else 0)
        d2h = B * K * 4 + B * 4 + B * 4
        e2e = {"value": world * B * e2e_steps / float(te.item()), "unit": "frames/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "steps": e2e_steps, "path": "fm_estimate_batch_host (pinned host X, "
                                                                  "host draws of Omega, redraw check, D2H peaks)"}
        same = np.array_equal(res["peak_cells"], out["peak_cells"].cpu().numpy())
        e2e["peaks_match_device_run"] = bool(same)

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    # ---------------- roofline of the dominant kernel, timed alone: one sub-batch (the whole
    # batch in one launch per kernel), CUDA events on the plan's launch stream around each stage
    hbm, bf16, bf16_sus, src = load_peaks()
    alg = algorithmic(cfgd)
    stage_ms = {k: v / max(runs, 1) for k, v in stage_sum.items()}  # sub-batch 0 (fsub frames), in-step
    plan.set_concurrency(1)
    plan.set_profiling(True)
    for _ in range(args.roof_steps):
        plan.run(B, xd, omega, idx, out, stream=stream)
    torch.cuda.synchronize()
    alone_sum, alone_runs = plan.stage_times_ms()
    plan.set_profiling(False)
    plan.set_concurrency(nsub)
    alone_ms = {k: v / max(alone_runs, 1) for k, v in alone_sum.items()}  # all B frames, one launch per kernel
    prof = {}
    try:
        with open(os.path.join(ROOT, "profiles", f"ncu_summary_{args.config}.json")) as f:
            prof = json.load(f)
    except Exception:
        pass
    bytes_launch = B * (8.0 * M * N + 8.0 * M * M)  # algorithmic: X read once + R (complex64) written once
    achieved = bytes_launch / (alone_ms["covariance"] / 1e3) / 1e9
    cov_prof = prof.get("cov_tc_kernel", {})
    roof = {"bound": "hbm", "kernel": "fmk::cov::cov_tc_kernel (tcgen05 cta_group::2 + TMA)", "achieved": achieved,
            "peak": hbm, "unit": "GB/s", "frac": achieved / hbm, "peak_source": src,
            "bytes_per_launch": bytes_launch, "launch_ms": alone_ms["covariance"],
            "share_of_step": alone_ms["covariance"] / sum(alone_ms.values()),
            "traffic": (cov_prof["dram_bytes"] * B / cov_prof["frames"]) if "dram_bytes" in cov_prof else None,
            "traffic_source": cov_prof.get("source")}
    p_tf32 = bf16 / 2.0
    t_roof_ms = max(B * alg["q_frame"] / (hbm * 1e9), B * alg["w_frame"] / (p_tf32 * 1e12)) * 1e3
    line = {
        "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": ms_max / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "c64",
        "data": "synthetic (seeded BASELINE frame model, DESIGN.md §3)",
        "config": config_dict(args.config, cfgd, world),
        "roofline": roof,
        "roofline_path": {"t_roof_ms_per_step": t_roof_ms, "t_meas_ms_per_step": ms_max / args.steps,
                          "frac": t_roof_ms / (ms_max / args.steps),
                          "def": "SURVEY.md §8d: max(B*Q/HBM, B*W/P_TF32), P_TF32 = measured bf16/2, 1xTF32 strict"},
        "stages_ms_per_step": stage_ms,
        "stages_note": f"CUDA-event durations of sub-batch 0 ({fsub} of {B} frames); {nsub} sub-batches run "
                       f"concurrently on plan-owned streams",
        "stages_alone_ms": alone_ms,
        "stages_alone_note": f"all {B} frames in one launch per kernel (concurrency 1), {args.roof_steps} runs",
        "subbatches": nsub,
        "gpu_launches": args.steps * plan.launches_per_batch() * nsub,
        "clocks": clk.summary(),
        "e2e": e2e,
        "frames_ok": int((status == 0).sum()), "frames_full_peaks": int((counts == K).sum()),
    }
    if world == 1 and not args.no_cpu_baseline:
        cores = os.cpu_count() or 1
        ns = min(B, max(cores, args.cpu_frames))
        frames = list(range(ns))
        import multiprocessing as mp
        pool = mp.get_context("fork").Pool(cores, initializer=_worker_init, initargs=(args.config,))
        cpu_reference_run(args.config, xnp[:cores], list(range(min(cores, ns))), cores, pool)  # warm the workers
        wall, res = cpu_reference_run(args.config, xnp[:ns], frames, cores, pool)
        pool.close()
        pool.join()
        gp = out["peak_cells"].cpu().numpy()
        gs = out["spectrum"].cpu().numpy()
        from oracle import fastmusic_oracle as O
        same = sum(1 for f, cells, spec, _ in res if list(gp[f][:len(cells)]) == cells)
        dbs = [O.spectrum_db_error(gs[f].astype("float64"), spec.astype("float64")) for f, _, spec, _ in res]
        line["cpu_baseline"] = {"value": ns / wall, "unit": "frames/s", "cores": cores, "kind": "port",
                                "sample": f"first {ns} frames of the {args.config} batch, oracle fp64 restatement "
                                          f"(numpy/scipy), one frame per worker process, pool warmed on "
                                          f"{min(cores, ns)} frames first"}
        line["parity_sample"] = {"frames": ns, "peaks_identical": same, "max_db_err_vs_port": max(dbs)}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--frames", type=int, default=0, help="override frames per GPU")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--subbatches", type=int, default=0, help="concurrent sub-batches per step (0 = auto)")
    ap.add_argument("--roof-steps", type=int, default=10, help="runs of the isolated roofline measurement")
    ap.add_argument("--cpu-frames", type=int, default=64)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
