#!/usr/bin/env python
"""Fast-MUSIC B200 benchmark (driver contract).

Workload (BASELINE.json configs[1]): batches of 1024 frames per GPU,
ULA M=256, N=512 snapshots, K=8 sources, random-projection Fast-MUSIC p=16, t=2,
3601-point grid over [-90, 90] deg, complex64, synthetic seeded frames (no dataset).
A step = one pass of the hot path (covariance -> range finder -> Nystrom -> spectrum ->
peaks) over one batch already resident in HBM; X is 1 GiB per batch (> 126 MB L2), so no
L2 flush is needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c2]

Multi-GPU (one process per GPU; `--gpus N` launches the N ranks itself through torch.distributed.run when
WORLD_SIZE is unset): --scaling strong (default) splits every global batch of B frames into
contiguous ranges [g B/G, (g+1) B/G); --scaling weak gives every GPU B frames. Small shards keep several
batches in flight (--depth, paper_1911_07434_b200/shard.py FrameStream). After each batch the peak
records are all-gathered over NCCL (the path's only collective); at N > 1 a weak-scaling companion number is
measured in the same run. Timing: CUDA events bracketing every plan stream, barrier + synchronize on both sides,
max over ranks.
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
    # SURVEY §8(f)3 block-Lanczos (the paper's accurate baseline; block = K, iteration cap 200) on the c2 frames
    "c2lz": dict(m=256, n=512, k=8, method="lanczos", p=0, t=200, L=3601, frames=1024, seed=2,
                 scene=dict(theta_lo_deg=-60.0, theta_hi_deg=60.0, min_sep_deg=3.0, snr_lo_db=10.0, snr_hi_db=30.0)),
    # SURVEY §8(f)4 ToA path: fast2 on the temporal covariance T = X^H X / M (512 x 512) of seeded beat-signal
    # frames (M = 256 antennas, N = 512 samples, K = 8 beats in [0.2, 2.9] rad/sample), beat grid [0, pi]
    "toa": dict(m=256, n=512, k=8, method="fast2", p=16, t=2, L=3601, frames=1024, seed=6, temporal=True,
                w0=0.0, w1=3.14159265358979323846, scene=None),
}


def dim_of(cfgd):
    """Dimension of the covariance the subspace is estimated on: M (spatial) or N (ToA path, T = X^H X / M)."""
    return cfgd["n"] if cfgd.get("temporal") else cfgd["m"]


def beat_frames(m, n, k, seed, f0, frames, device):
    """Seeded beat-signal frames for the ToA config, generated on the device (input data only): X(a, s) =
    sum_k exp(j (phi_k + pi a sin(theta_k) + w_k s)) + noise at 20 dB (sigma^2 = K / 100), beat phases w_k drawn
    in [0.2, 2.9] rad/sample with >= 0.05 separation. Returns a float32 view [frames, M, N, 2] on `device`."""
    import torch
    g = torch.Generator(device="cpu").manual_seed(int(seed) * 1000003 + int(f0))
    ws = torch.empty((frames, k), dtype=torch.float64)
    for f in range(frames):
        w = []
        while len(w) < k:
            c = 0.2 + 2.7 * float(torch.rand((), generator=g, dtype=torch.float64))
            if all(abs(c - x) >= 0.05 for x in w):
                w.append(c)
        ws[f] = torch.tensor(sorted(w), dtype=torch.float64)
    th = (torch.rand((frames, k), generator=g, dtype=torch.float64) * 2.0 - 1.0) * (torch.pi / 3.0)
    ph = torch.rand((frames, k), generator=g, dtype=torch.float64) * (2.0 * torch.pi)
    ws, th, ph = ws.to(device), th.to(device), ph.to(device)
    a = torch.arange(m, dtype=torch.float64, device=device)
    sidx = torch.arange(n, dtype=torch.float64, device=device)
    x = torch.empty((frames, m, n), dtype=torch.complex64, device=device)
    gd = torch.Generator(device=device).manual_seed(int(seed) * 7919 + int(f0))
    sig = (k / 100.0) ** 0.5
    for f0c in range(0, frames, 64):
        f1 = min(frames, f0c + 64)
        ang = (ph[f0c:f1, :, None, None] + torch.pi * torch.sin(th[f0c:f1, :, None, None]) * a[None, None, :, None]
               + ws[f0c:f1, :, None, None] * sidx[None, None, None, :])
        xs = torch.polar(torch.ones_like(ang), ang).sum(1)
        nz = torch.randn((f1 - f0c, m, n, 2), generator=gd, dtype=torch.float64, device=device) * (sig / 2 ** 0.5)
        x[f0c:f1] = (xs + torch.complex(nz[..., 0], nz[..., 1])).to(torch.complex64)
    return torch.view_as_real(x)


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
    x_bytes = 8.0 * m * n
    if cfg.get("temporal"):  # ToA path: the N x N covariance T over M "snapshots"
        m, n = n, m
    w_cov = 4.0 * m * (m + 1) * n
    if cfg["method"] == "fast2":
        w_rf = 4.0 * m * m * p + 8.0 * t * m * m * p
        q = x_bytes + 4.0 * m * p + 4.0 * L + 8.0 * k
    elif cfg["method"] == "fast1":
        w_rf = 0.0
        q = x_bytes + 8.0 * p + 4.0 * L + 8.0 * k
    elif cfg["method"] == "fast1_norm2":  # sampled sketch (a gather), one product R V
        w_rf = 8.0 * m * m * p
        q = x_bytes + 4.0 * m + 4.0 * L + 8.0 * k
    else:
        w_rf = 0.0
        q = x_bytes + 4.0 * L + 8.0 * k
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
    if cfg_name == "toa":
        cfg = O.ToaConfig()
        _W.update(O=O, cfg=cfg, toa=True,
                  A=O.beat_steering_matrix(O.beat_grid(cfg.grid_size, cfg.w0, cfg.w1), cfg.spec.n))
        return
    cfg = O.baseline_configs()[cfg_name]
    grid = O.baseline_grid(cfg.grid_size)
    _W.update(O=O, cfg=cfg, grid=grid, A=O.steering_matrix(grid, cfg.spec.m), toa=False)


def _worker_frame(args):
    f, x = args
    O, cfg = _W["O"], _W["cfg"]
    t0 = time.perf_counter()
    if _W["toa"]:
        est, spec, pk = O.run_toa_frame(cfg, x, f, _W["A"])
    else:
        est, spec, pk = O.run_frame(cfg, x, f, _W["grid"], _W["A"])
    return f, pk.cells, spec.astype("float32"), time.perf_counter() - t0


def _ref_available(cfg_name):
    """The reference's own path compiled here (oracle/_ref/libref_fastmusic.so: R/src/{scene,linalg,estimators,
    spectrum}.cpp against the Eigen-API shim over OpenBLAS) covers every config but the norm^2-sampling extension."""
    try:
        from oracle import ref_lib
    except Exception:
        return False
    return ref_lib.available() and CONFIGS[cfg_name]["method"] in ("fast2", "fast1", "exact", "lanczos")


def _ref_worker_init(cfg_name):
    from oracle import fastmusic_oracle as O
    from oracle import ref_lib
    _W.update(O=O, R=ref_lib, cfgd=CONFIGS[cfg_name])


def _ref_worker_frame(args):
    f, x = args
    O, R, c = _W["O"], _W["R"], _W["cfgd"]
    fs = O.frame_seed(c["seed"], f)
    seed = O.derive(fs, 4 if c["method"] == "fast2" else 3) if c["method"] in ("fast2", "fast1") else 0
    t0 = time.perf_counter()
    st, cells, _ = R.run_frame(x, c["k"], c["method"], c["p"], c["t"], seed, c["L"], 3, bool(c.get("temporal")))
    return f, cells, st, time.perf_counter() - t0


def cpu_ref_run(cfg_name, xs, frames, cores, pool):
    """The reference's own compiled path over `frames`, one frame per worker at a time (R/src/bench.cpp:59-86
    pattern, one BLAS thread per worker); returns (wall_s, results). Grid: the reference's AngleGrid(L) = [0, pi]
    (R/src/spectrum.cpp:18-28) -- the same L points and work as the GPU arm's [-90, 90] deg grid."""
    t0 = time.perf_counter()
    res = pool.map(_ref_worker_frame, [(f, xs[i]) for i, f in enumerate(frames)], chunksize=1)
    return time.perf_counter() - t0, res


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
    cores = os.cpu_count() or 1
    per_step = max(1, min(cfgd["frames"], cores))
    nsamp = per_step * 4
    if cfgd.get("temporal"):
        xs, _ = O.generate_toa_batch(cfgd["seed"], range(nsamp), O.ToaConfig().spec)
    else:
        cfg = O.baseline_configs()[args.config]
        xs, _, _ = O.generate_batch(cfg.base_seed, range(nsamp), cfg.spec)
    use_ref = _ref_available(args.config)
    pool = mp.get_context("fork").Pool(cores, initializer=_ref_worker_init if use_ref else _worker_init,
                                       initargs=(args.config,))
    times = []
    for i in range(args.warmup + args.steps):
        sl = [(i * per_step + j) % nsamp for j in range(per_step)]
        if use_ref:
            wall, _ = cpu_ref_run(args.config, xs[sl], sl, cores, pool)
        else:
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
        "cpu_baseline": {"value": value, "unit": "frames/s", "cores": cores, "kind": "reference" if use_ref else "port",
                         "cpu_model": cpu_model(),
                         "sample": (f"{per_step} frames per step (one per core) of {args.config}; " +
                                    ("the reference's own R/src/{scene,linalg,estimators,spectrum}.cpp compiled here "
                                     "(oracle/_ref, Eigen-API shim over OpenBLAS, 1 BLAS thread per worker), "
                                     "AngleGrid(L) = [0, pi]" if use_ref else
                                     "oracle fp64 restatement of the reference path (numpy/scipy LAPACK, 1 BLAS "
                                     "thread/worker)"))},
        "e2e": {"value": value, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def config_dict(name, cfgd, world, mode="strong", per_gpu=None, depth=1, coalesce=1):
    per_gpu = cfgd["frames"] if per_gpu is None else per_gpu
    gfr = cfgd["frames"] if mode == "strong" else cfgd["frames"] * world
    xb = per_gpu * cfgd["m"] * cfgd["n"] * 8
    l2 = ("inputs larger than L2 (X = %.2f GiB per GPU step)" % (xb / 2**30) if xb > 3 * 126 * 2**20 else
          "X = %.0f MB per GPU step; consecutive steps cycle through >= 3 x L2 of distinct X copies" % (xb / 1e6))
    return {"workload": f"{name}: fast-MUSIC {cfgd['method']} M={cfgd['m']} N={cfgd['n']} K={cfgd['k']} "
                        f"p={cfgd['p']} t={cfgd['t']} L={cfgd['L']}",
            "frames_per_gpu": per_gpu, "global_frames_per_step": gfr,
            "grid": "beat phase [0, pi] rad/sample (ToA path on T = X^H X / M)" if cfgd.get("temporal")
            else "[-90, 90] deg", "l2": l2,
            "parallelism": (f"{mode} scaling: frames of each {gfr}-frame batch sharded over {world} GPU(s) "
                            f"[g B/G, (g+1) B/G), NCCL all-gather of peak records" if mode == "strong" else
                            f"weak scaling: {per_gpu} frames per GPU, NCCL all-gather of peak records"),
            "coalesce": coalesce,
            "coalesce_note": "each launch runs this GPU's shards of `coalesce` consecutive global batches together"
                             " (frames are independent; the timed region still covers exactly `steps` global batches)"}


# ----------------------------------------------------------------------------- ours
def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1911_07434_b200 as fm
    from paper_1911_07434_b200.shard import FrameStream, shard_range, unshard_records

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # FM_BENCH_DRYRUN_GLOO=1: rehearse the N > 1 control flow on a box with fewer GPUs than ranks (every rank on a
    # visible device, gloo instead of NCCL). Its line is marked "dryrun" and is not a measurement.
    dry = world > 1 and os.environ.get("FM_BENCH_DRYRUN_GLOO") == "1"
    if dry:
        local %= torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if dry:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    cfgd = CONFIGS[args.config]
    if args.frames:
        cfgd = dict(cfgd, frames=args.frames)
    B, M, N, K, P, L = cfgd["frames"], cfgd["m"], cfgd["n"], cfgd["k"], cfgd["p"], cfgd["L"]
    mode = args.scaling
    f0, n = shard_range(rank, world, B, mode)
    nmax = max(shard_range(g, world, B, mode)[1] for g in range(world))
    gfr = B if mode == "strong" else B * world  # global frames per step
    # synthetic input for this rank's frames, generated on the host (pinned), staged once
    xh = torch.empty((n, M, N, 2), dtype=torch.float32, pin_memory=True)
    xnp = xh.numpy().view(np.complex64).reshape(n, M, N)
    D = dim_of(cfgd)  # dimension of the covariance (M, or N on the ToA path)
    if cfgd.get("temporal"):
        xh.copy_(beat_frames(M, N, K, cfgd["seed"], f0, n, dev).cpu())
    else:
        fm.generate_frames(M, N, K, cfgd["seed"], f0, n, out=xnp, **cfgd["scene"])
    fseeds = np.array([fm.derive(cfgd["seed"], f0 + f) for f in range(n)], np.uint64)
    tag = 4 if cfgd["method"] == "fast2" else 3
    dseeds = np.array([fm.derive(int(s), tag) for s in fseeds], np.uint64)
    omega = idx = None
    if cfgd["method"] == "fast2":
        omega = torch.from_numpy(fm.draw_omega_batch(dseeds, D, P)).to(dev)
    elif cfgd["method"] == "fast1":
        idx = torch.from_numpy(fm.draw_indices_batch(dseeds, D, P)).to(dev)
    elif cfgd["method"] == "fast1_norm2":  # uniforms of the weighted sampler travel in the omega slot
        omega = torch.from_numpy(fm.draw_uniforms_batch(dseeds, D)).to(dev)
    xd = xh.to(dev)
    # batches in flight: small shards leave too little work per kernel to hide ramps and tails
    # (measured at N = 1, c2, tools/bench_sweep.sh: 1024 frames 0.954 / 1.075 / 1.105 M frames/s at depth 1 / 2 / 3;
    # 128-frame shards 0.37 / 0.54 / 0.65 / 0.71 M at depth 1 .. 4)
    # Shard coalescing (SURVEY H6, strong scaling): a GPU's shard of one global batch shrinks to 1024 / G frames
    # (128 at G = 8), too few to fill 148 SMs; one launch therefore carries its shards of `co` consecutive global
    # batches (>= 512 frames). Frames are independent, so only the launch granularity changes.
    co = args.coalesce if args.coalesce > 0 else (max(1, -(-512 // n)) if mode == "strong" else 1)
    nl = co * n  # frames per launch
    depth = args.depth if args.depth > 0 else (3 if nl >= 512 else 4 if nl >= 256 else 6)

    # CUDA-graph replay of whole batches: small shards are otherwise bound by the host's launch rate
    graphs = args.graphs == "on" or (args.graphs == "auto" and depth <= 2)

    def make_plan(i):
        grid = dict(theta0=cfgd["w0"], theta1=cfgd["w1"], temporal=True) if cfgd.get("temporal") else {}
        p = fm.BatchPlan(M, N, K, cfgd["method"], p=P, t=cfgd["t"], grid_size=L, max_frames=nl, device=local,
                         exact_jacobi=args.exact_jacobi, **grid)
        if args.subbatches > 0:
            p.set_concurrency(args.subbatches)
        p.set_graphs(graphs)
        return p

    streams = [torch.cuda.Stream(device=dev) for _ in range(depth)]
    fs = FrameStream(make_plan, nl, co * nmax, K, world, depth, streams, dev, spectrum=True)
    plan0 = fs.plans[0]
    main_s = torch.cuda.current_stream(dev)

    # L2 hygiene: steps cycle through enough copies of X that every step reads its input from HBM (> 3x L2 in all)
    nbuf = max(depth, -(-3 * 126 * 2**20 // (nl * M * N * 8)))
    xl = xd if co == 1 else xd.repeat(co, 1, 1, 1)
    xs = [xl] + [xl.clone() for _ in range(nbuf - 1)]
    om_l = omega if (omega is None or co == 1) else omega.repeat(co, *([1] * (omega.dim() - 1)))
    ix_l = idx if (idx is None or co == 1) else idx.repeat(co, *([1] * (idx.dim() - 1)))
    ctr = [0]

    def run_steps(count):  # `count` global batches: count // co full launches, then one partial launch
        gathered = None
        full, rem = divmod(count, co)
        for i in range(full + (1 if rem else 0)):
            fr = nl if i < full else rem * n
            _, gathered = fs.step(xs[ctr[0] % nbuf], om_l, ix_l, frames=fr)
            ctr[0] += 1
        return gathered

    run_steps((max(3, args.warmup) + depth) * co)
    torch.cuda.synchronize()
    out0 = fs.output(0)
    status = out0["status"].cpu().numpy()
    counts = out0["peak_count"].cpu().numpy()

    # ---------------- timed region: barrier + synchronize, events on the main stream bracketing every plan stream
    # (per-stage events only without graphs: a profiled batch is enqueued kernel by kernel)
    plan0.set_profiling(not graphs)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        e0.record(main_s)
        for s in streams:
            s.wait_event(e0)
        gathered = run_steps(args.steps)
        for s in streams:
            ev = torch.cuda.Event()
            ev.record(s)
            main_s.wait_event(ev)
        e1.record(main_s)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    stage_sum, runs = plan0.stage_times_ms()
    plan0.set_profiling(False)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = gfr * args.steps / (ms_max / 1e3)
    recs = unshard_records(gathered[:, :nmax], world, B, mode) if world > 1 else None  # first batch of the launch

    # ---------------- weak-scaling companion (N > 1, strong default): B frames per rank, same timing rules
    weak = None
    if world > 1 and mode == "strong" and not args.no_weak:
        xw = torch.empty((B, M, N, 2), dtype=torch.float32, device=dev)
        xw.view(-1)[: xd.numel()].copy_(xd.view(-1))
        reps = (B + n - 1) // n
        for r in range(1, reps):
            lo = r * n
            hi = min(B, lo + n)
            xw[lo:hi].copy_(xd[: hi - lo])
        omw = omega.repeat(reps, 1, 1)[:B].contiguous() if omega is not None else None
        ixw = idx.repeat(reps, 1)[:B].contiguous() if idx is not None else None
        fw = FrameStream(lambda i: fm.BatchPlan(
            M, N, K, cfgd["method"], p=P, t=cfgd["t"], grid_size=L, max_frames=B, device=local,
            **(dict(theta0=cfgd["w0"], theta1=cfgd["w1"], temporal=True) if cfgd.get("temporal") else {})),
            B, B, K, world, 1, [streams[0]], dev)
        for _ in range(3):
            fw.step(xw, omw, ixw)
        dist.barrier()
        torch.cuda.synchronize()
        w0 = torch.cuda.Event(enable_timing=True)
        w1 = torch.cuda.Event(enable_timing=True)
        w0.record(streams[0])
        for _ in range(args.steps):
            fw.step(xw, omw, ixw)
        w1.record(streams[0])
        torch.cuda.synchronize()
        dist.barrier()
        tw = torch.tensor([w0.elapsed_time(w1)], dtype=torch.float64, device=dev)
        dist.all_reduce(tw, op=dist.ReduceOp.MAX)
        weak = {"value": world * B * args.steps / (float(tw.item()) / 1e3), "unit": "frames/s",
                "frames_per_gpu": B, "global_frames_per_step": world * B, "ms_per_step": float(tw.item()) / args.steps}
        fw.close()
        del xw

    # ---------------- e2e through the reference-facing host-buffer C-ABI call (this rank's shard)
    e2e = None
    if not args.no_e2e:
        draw = None if cfgd["method"] == "exact" else dseeds
        res = plan0.estimate_host(xnp, draw)  # warm-up (allocates staging)
        e2e_steps = max(1, min(args.e2e_steps, args.steps))
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            res = plan0.estimate_host(xnp, draw)
        el = time.perf_counter() - t0
        te = torch.tensor([el], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        h2d = n * M * N * 8 + (n * M * P * 4 if cfgd["method"] == "fast2" else n * P * 4 if cfgd["method"] == "fast1"
                               else n * M * 4 if cfgd["method"] == "fast1_norm2" else 0)
        d2h = n * K * 4 + n * 4 + n * 4
        e2e = {"value": gfr * e2e_steps / float(te.item()), "unit": "frames/s", "h2d_bytes_per_step": h2d * world,
               "d2h_bytes_per_step": d2h * world, "steps": e2e_steps,
               "path": "fm_estimate_batch_host (pinned host X, host draws of Omega, redraw check, D2H peaks)"}
        same = np.array_equal(res["peak_cells"], out0["peak_cells"][:n].cpu().numpy())
        e2e["peaks_match_device_run"] = bool(same)

    if rank != 0:
        fs.close()
        if world > 1:
            dist.destroy_process_group()
        return 0

    # ---------------- roofline of the dominant kernel, timed alone: one sub-batch (the whole shard in one launch
    # per kernel), CUDA events on the plan's launch stream around each stage
    hbm, bf16, bf16_sus, src = load_peaks()
    alg = algorithmic(cfgd)
    stage_ms = {k: v / max(runs, 1) for k, v in stage_sum.items()}
    plan0.set_concurrency(1)
    plan0.set_profiling(True)
    out_r = fs.output(0)
    for _ in range(args.roof_steps):
        plan0.run(n, xd, omega, idx, out_r, stream=streams[0])
    torch.cuda.synchronize()
    alone_sum, alone_runs = plan0.stage_times_ms()
    plan0.set_profiling(False)
    alone_ms = {k: v / max(alone_runs, 1) for k, v in alone_sum.items()}  # all n frames, one launch per kernel
    prof = {}
    try:
        with open(os.path.join(ROOT, "profiles", f"ncu_summary_{args.config}.json")) as f:
            prof = json.load(f)
    except Exception:
        pass
    x_bytes = n * 8.0 * M * N                  # SURVEY §8(d) algorithmic bytes of the covariance: X read once
    r_bytes = n * 8.0 * D * D                  # + R (or T) written once (complex64, or its two fp16 planes)
    cov_ms = alone_ms["covariance"]
    cov_prof = prof.get("cov_tc_kernel", {})
    roof = {"bound": "hbm", "kernel": "fmk::cov::cov_tc_kernel (tcgen05 cta_group::2 + TMA)",
            "achieved": x_bytes / (cov_ms / 1e3) / 1e9, "peak": hbm, "unit": "GB/s",
            "frac": x_bytes / (cov_ms / 1e3) / 1e9 / hbm, "peak_source": src,
            "bytes_def": "SURVEY §8(d): X read (8 M N per frame) only",
            "bytes_per_launch": x_bytes, "launch_ms": cov_ms,
            "frac_incl_r_write": (x_bytes + r_bytes) / (cov_ms / 1e3) / 1e9 / hbm,
            "share_of_step": cov_ms / sum(alone_ms.values()),
            "traffic": (cov_prof["dram_bytes"] * n / cov_prof["frames"]) if "dram_bytes" in cov_prof else None,
            "traffic_source": cov_prof.get("source")}
    step_prof = prof.get("step", {})
    p_tf32 = bf16 / 2.0
    t_roof_ms = max(gfr * alg["q_frame"] / world / (hbm * 1e9), gfr * alg["w_frame"] / world / (p_tf32 * 1e12)) * 1e3
    # "the builder should measure TF32 ... peaks": cuBLAS TF32 8192^3 on this pool's B200s
    # (tools/measure_peaks_extra.py -> profiles/measured_peaks_extra.json), reported beside the strict figure
    extra = {}
    try:
        with open(os.path.join(ROOT, "profiles", "measured_peaks_extra.json")) as f:
            extra = json.load(f)
    except Exception:
        pass

    def path_frac(p_tf):
        if not p_tf:
            return None
        t = max(gfr * alg["q_frame"] / world / (hbm * 1e9), gfr * alg["w_frame"] / world / (p_tf * 1e12)) * 1e3
        return t / (ms_max / args.steps)
    line = {
        "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": ms_max / args.steps, "higher_is_better": True,
        "scaling": mode, "vs_baseline": None, "dtype": "c64",
        "data": "synthetic (seeded BASELINE frame model, DESIGN.md §3)",
        "config": config_dict(args.config, cfgd, world, mode, n, depth, co),
        "roofline": roof,
        "roofline_path": {"t_roof_ms_per_step": t_roof_ms, "t_meas_ms_per_step": ms_max / args.steps,
                          "frac": t_roof_ms / (ms_max / args.steps),
                          "def": "SURVEY.md §8d: max(B*Q/HBM, B*W/P_TF32) per GPU, P_TF32 = measured bf16/2, "
                                 "1xTF32 strict",
                          "frac_measured_tf32": path_frac(extra.get("tf32_tflops")),
                          "frac_measured_tf32_sustained": path_frac(extra.get("tf32_tflops_sustained")),
                          "measured_tf32_tflops": [extra.get("tf32_tflops"), extra.get("tf32_tflops_sustained")],
                          "measured_tf32_source": "profiles/measured_peaks_extra.json (cuBLAS TF32 8192^3, burst / "
                                                  "sustained)" if extra else None,
                          "dram_bytes_per_frame_ncu": step_prof.get("dram_bytes_per_frame"),
                          "algorithmic_bytes_per_frame": alg["q_frame"],
                          "dram_over_algorithmic": (step_prof["dram_bytes_per_frame"] / alg["q_frame"])
                          if "dram_bytes_per_frame" in step_prof else None,
                          "dram_source": step_prof.get("source")},
        "stages_ms_per_step": stage_ms if not graphs else None,
        "stages_note": f"CUDA-event durations in plan 0's stream ({n} frames per batch, {depth} batch(es) in flight)"
                       if not graphs else "not recorded in-step: batches replayed from CUDA graphs",
        "cuda_graphs": graphs,
        "exact_solver": ("jacobi (every frame)" if args.exact_jacobi else "certified subspace iteration + Jacobi for "
                         "uncertified frames") if cfgd["method"] == "exact" else None,
        "stages_alone_ms": alone_ms,
        "stages_alone_note": f"all {n} frames in one launch per kernel (concurrency 1), {args.roof_steps} runs",
        "batches_in_flight": depth,
        "gpu_launches": -(-args.steps // co) * (plan0.launches_per_batch() + 1),  # launches x (+ the record pack)
        "clocks": clk.summary(),
        "e2e": e2e,
        "frames_ok": int((status == 0).sum()), "frames_full_peaks": int((counts == K).sum()),
    }
    if dry:
        line["dryrun"] = "gloo, ranks share GPUs: control-flow rehearsal, not a measurement"
    if weak is not None:
        line["weak_scaling"] = weak
    if recs is not None:
        line["gathered_records"] = {"frames": int(recs.shape[0]), "ok": int((recs[:, K + 1] == 0).sum().item())}
    if world == 1 and not args.no_cpu_baseline:
        cores = os.cpu_count() or 1
        ns = min(n, max(cores, args.cpu_frames))
        frames = list(range(ns))
        import multiprocessing as mp
        use_ref = _ref_available(args.config)
        ref_wall = None
        if use_ref:  # timed: the reference's own compiled path; parity: the oracle port on the same frames
            rpool = mp.get_context("fork").Pool(cores, initializer=_ref_worker_init, initargs=(args.config,))
            cpu_ref_run(args.config, xnp[:cores], list(range(min(cores, ns))), cores, rpool)  # warm the workers
            ref_wall, _ = cpu_ref_run(args.config, xnp[:ns], frames, cores, rpool)
            rpool.close()
            rpool.join()
            ns_par = min(ns, max(cores, 16))
        else:
            ns_par = ns
        pool = mp.get_context("fork").Pool(cores, initializer=_worker_init, initargs=(args.config,))
        cpu_reference_run(args.config, xnp[:cores], list(range(min(cores, ns_par))), cores, pool)  # warm the workers
        wall, res = cpu_reference_run(args.config, xnp[:ns_par], list(range(ns_par)), cores, pool)
        pool.close()
        pool.join()
        gp = out0["peak_cells"].cpu().numpy()
        gs = out0["spectrum"].cpu().numpy()
        from oracle import fastmusic_oracle as O
        same = sum(1 for f, cells, spec, _ in res if list(gp[f][:len(cells)]) == cells)
        dbs = [O.spectrum_db_error(gs[f].astype("float64"), spec.astype("float64")) for f, _, spec, _ in res]
        if use_ref:
            line["cpu_baseline"] = {"value": ns / ref_wall, "unit": "frames/s", "cores": cores, "kind": "reference",
                                    "cpu_model": cpu_model(),
                                    "sample": f"first {ns} frames of the {args.config} batch through the reference's "
                                              f"own R/src/{{scene,linalg,estimators,spectrum}}.cpp compiled here "
                                              f"(oracle/_ref, Eigen-API shim over OpenBLAS), one frame per worker "
                                              f"process, 1 BLAS thread each, AngleGrid(L) = [0, pi]; pool warmed "
                                              f"on {min(cores, ns)} frames first",
                                    "port_value": ns_par / wall}
        else:
            line["cpu_baseline"] = {"value": ns / wall, "unit": "frames/s", "cores": cores, "kind": "port",
                                    "cpu_model": cpu_model(),
                                    "sample": f"first {ns} frames of the {args.config} batch, oracle fp64 restatement "
                                              f"(numpy/scipy), one frame per worker process, pool warmed on "
                                              f"{min(cores, ns)} frames first"}
        line["parity_sample"] = {"frames": ns_par, "peaks_identical": same, "max_db_err_vs_port": max(dbs)}
    print(json.dumps(line), flush=True)
    fs.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    import platform
    return platform.processor() or "unknown"


def spawn_ranks(args) -> int:
    """`--gpus N` without torchrun: launch N ranks (one process per GPU) through torch.distributed.run."""
    import socket

    import torch
    have = torch.cuda.device_count()
    if have < args.gpus and os.environ.get("FM_BENCH_DRYRUN_GLOO") != "1":
        print(json.dumps({"error": f"--gpus {args.gpus} but only {have} CUDA device(s) visible"}), flush=True)
        return 2
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


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
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="strong: each global batch's frames split over the GPUs (SURVEY §8e); weak: a batch per GPU")
    ap.add_argument("--depth", type=int, default=0, help="batches in flight per GPU (0 = auto)")
    ap.add_argument("--coalesce", type=int, default=0,
                    help="global batches per launch on each GPU (0 = auto: shards of >= 512 frames per launch)")
    ap.add_argument("--exact-jacobi", action="store_true",
                    help="exact method (c5): the full Jacobi eigensolver on every frame (no certified iteration)")
    ap.add_argument("--graphs", default="auto", choices=["auto", "on", "off"],
                    help="replay batches from CUDA graphs (auto: when at most 2 batches are in flight)")
    ap.add_argument("--no-weak", action="store_true", help="skip the weak-scaling companion measurement (N > 1)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    ws = os.environ.get("WORLD_SIZE")
    if ws is None and args.gpus > 1:
        return spawn_ranks(args)
    if ws is not None and int(ws) != args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} but WORLD_SIZE={ws}"}), flush=True)
        return 2
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
