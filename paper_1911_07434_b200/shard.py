"""Frames across GPUs: sharding, batches in flight, and the peak-record all-gather.

The reference's only parallelism is a pool of independent frames (R/src/bench.cpp:59-86). Frames need no data
exchange, so the B200 path shards them: rank g of G owns the contiguous range [g B / G, (g + 1) B / G) of every
global batch of B frames (strong scaling, §8e), or B frames of its own (weak scaling). The only collective is
the gather of fixed-size per-frame peak records {K cells, count, status} after each batch: one
all_gather_into_tensor over NCCL (GPU) or gloo (CPU tests), B (K + 2) 4 bytes in all (40 KB at c2).

H6: a strong split leaves 1024 / 8 = 128 frames per GPU per batch, too little work to hide each
kernel's ramp and tail. ``FrameStream`` therefore keeps ``depth`` consecutive batches in flight, each on its own
plan (workspace) and stream, so one batch's tails overlap the next one's kernels; the records of batch i are
gathered on batch i's stream.
"""
from __future__ import annotations


def shard_range(rank: int, world: int, total: int, mode: str = "strong") -> tuple[int, int]:
    """(first global frame, frame count) of `rank`. strong: `total` frames per batch split into contiguous
    near-equal ranges [g total / G, (g + 1) total / G); weak: `total` frames per rank at rank * total."""
    if world < 1 or not (0 <= rank < world) or total < 0:
        raise ValueError("shard_range: need 0 <= rank < world and total >= 0")
    if mode == "weak":
        return rank * total, total
    if mode != "strong":
        raise ValueError("shard_range: mode is 'strong' or 'weak'")
    base, rem = divmod(total, world)
    return rank * base + min(rank, rem), base + (1 if rank < rem else 0)


def pack_records(peak_cells, peak_count, status, out=None):
    """[B, K+2] int32 record per frame: K cells, count, status (device or host tensors)."""
    import torch
    b, k = peak_cells.shape
    rec = out if out is not None else torch.empty((b, k + 2), dtype=torch.int32, device=peak_cells.device)
    if rec.is_cuda and rec.is_contiguous() and all(t.is_contiguous() for t in (peak_cells, peak_count, status)):
        from . import _capi  # one kernel (fm_pack_peak_records) on the current stream
        st = _capi.LIB.fm_pack_peak_records(_capi.ptr(peak_cells), _capi.ptr(peak_count), _capi.ptr(status), b, k,
                                            _capi.ptr(rec), torch.cuda.current_stream(rec.device).cuda_stream)
        if st != 0:
            raise RuntimeError(_capi.last_error())
        return rec
    rec[:, :k].copy_(peak_cells)
    rec[:, k].copy_(peak_count)
    rec[:, k + 1].copy_(status)
    return rec


def gather_records(rec, world: int, out=None, group=None):
    """All-gather every rank's [B, K+2] records into [world, B, K+2] (rank-major = frame order). Ranks with
    fewer frames (strong split of a batch that does not divide evenly) pad their records with -1 rows."""
    import torch
    import torch.distributed as dist
    if world == 1:
        return rec.unsqueeze(0)
    g = out if out is not None else torch.empty((world,) + tuple(rec.shape), dtype=rec.dtype, device=rec.device)
    if rec.is_cuda and dist.get_backend(group) == "gloo":
        # dry runs of the N > 1 flow on a one-GPU box (bench.py FM_BENCH_DRYRUN_GLOO): gloo has no CUDA all-gather,
        # so the 40 KB of records take a host round trip; never the measured path (NCCL gathers in place)
        h = torch.empty((world,) + tuple(rec.shape), dtype=rec.dtype)
        dist.all_gather_into_tensor(h.view(-1, rec.shape[1]), rec.cpu().contiguous(), group=group)
        g.copy_(h)
        return g
    dist.all_gather_into_tensor(g.view(-1, rec.shape[1]), rec.contiguous(), group=group)
    return g


def unshard_records(gathered, world: int, total: int, mode: str = "strong"):
    """[world, Bmax, K+2] gathered records -> [global frames, K+2] in global frame order."""
    import torch
    rows = []
    for g in range(world):
        _, n = shard_range(g, world, total, mode)
        rows.append(gathered[g, :n])
    return torch.cat(rows, 0)


def unshard_coalesced(gathered, world: int, total: int, co: int, mode: str = "strong"):
    """Records of a coalesced launch (each rank ran its shards of `co` consecutive global batches back to back:
    rank g's rows [i n_g, (i + 1) n_g) belong to batch i) -> list of `co` [global frames, K+2] arrays."""
    import torch
    out = []
    for i in range(co):
        rows = []
        for g in range(world):
            _, n = shard_range(g, world, total, mode)
            rows.append(gathered[g, i * n:(i + 1) * n])
        out.append(torch.cat(rows, 0))
    return out


class FrameStream:
    """One rank's part of a stream of global batches: `depth` plans / streams used round-robin, so up to `depth`
    batches are in flight; step() enqueues the batch (plan.run), packs its peak records and all-gathers them on
    the same stream, and returns the gathered [world, Bmax, K+2] tensor (valid once that stream is done).

    plan_factory(i) -> object with run(frames, x, omega, indices, out, stream) and outputs(frames, spectrum)
    (paper_1911_07434_b200.BatchPlan, or a stub in the CPU tests); streams: one per plan (torch.cuda.Stream, or
    None on the CPU)."""

    def __init__(self, plan_factory, frames: int, frames_max: int, k: int, world: int, depth: int = 1,
                 streams=None, device=None, spectrum: bool = False):
        import torch
        self.frames, self.frames_max, self.k, self.world = frames, frames_max, k, world
        self.depth = max(1, depth)
        self.plans = [plan_factory(i) for i in range(self.depth)]
        self.streams = streams if streams is not None else [None] * self.depth
        self.outs = [p.outputs(frames, spectrum=spectrum) for p in self.plans]
        self.recs = [torch.full((frames_max, k + 2), -1, dtype=torch.int32, device=device) for _ in range(self.depth)]
        self.gath = [torch.empty((world, frames_max, k + 2), dtype=torch.int32, device=device)
                     for _ in range(self.depth)] if world > 1 else [None] * self.depth
        self.i = 0

    def step(self, x, omega=None, indices=None, frames=None):
        """frames (<= the stream's frames): a shorter launch over the first `frames` frames (records beyond them
        keep the previous contents)."""
        import contextlib

        import torch
        nf = self.frames if frames is None else frames
        if not 0 < nf <= self.frames:
            raise ValueError("FrameStream.step: 0 < frames <= stream frames")
        d = self.i % self.depth
        self.i += 1
        plan, out, s = self.plans[d], self.outs[d], self.streams[d]
        plan.run(nf, x, omega, indices, out, stream=s)
        ctx = torch.cuda.stream(s) if s is not None else contextlib.nullcontext()
        with ctx:
            pack_records(out["peak_cells"][:nf], out["peak_count"][:nf], out["status"][:nf], out=self.recs[d][:nf])
            g = gather_records(self.recs[d], self.world, out=self.gath[d])
        return d, g

    def output(self, d: int):
        return self.outs[d]

    def close(self):
        for p in self.plans:
            if hasattr(p, "close"):
                p.close()
