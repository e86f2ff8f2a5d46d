"""N>1 path on CPU: world_size-2 gloo process groups running bench.py's multi-GPU step logic
(paper_1911_07434_b200/shard.py: strong / weak frame sharding, FrameStream with batches in flight, peak-record
pack -> all-gather -> unshard) with a stub plan in place of the CUDA pipeline."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


class StubPlan:
    """Stands in for BatchPlan: frame f of the shard gets cells (gid * 10 + j), count K, status gid % 3, where gid is
    the global frame index carried in x[f, 0] (plus 1000 * the batch counter so in-flight batches differ)."""

    def __init__(self, k):
        self.k = k

    def outputs(self, frames, spectrum=False):
        return {"peak_cells": torch.empty((frames, self.k), dtype=torch.int32),
                "peak_count": torch.empty((frames,), dtype=torch.int32),
                "status": torch.empty((frames,), dtype=torch.int32)}

    def run(self, frames, x, omega, indices, out, stream=None):
        gid = x[:frames, 0].to(torch.int32)
        out["peak_cells"][:frames].copy_(gid[:, None] * 10 + torch.arange(self.k, dtype=torch.int32)[None, :])
        out["peak_count"][:frames].fill_(self.k)
        out["status"][:frames].copy_(gid % 3)


def _worker(rank, world, port, total, k, mode, depth, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1911_07434_b200 import derive
        from paper_1911_07434_b200.shard import FrameStream, shard_range, unshard_records
        f0, n = shard_range(rank, world, total, mode)
        nmax = max(shard_range(g, world, total, mode)[1] for g in range(world))
        fs = FrameStream(lambda i: StubPlan(k), n, nmax, k, world, depth)
        got = []
        for b in range(3):  # three batches through `depth` plans round-robin
            x = torch.tensor([[1000 * b + f0 + f] for f in range(n)], dtype=torch.float64)
            _, g = fs.step(x)
            got.append(unshard_records(g, world, total, mode).numpy().copy())
        # per-frame draw seeds depend only on the global frame index (shard-invariant)
        seeds = [derive(derive(2, f0 + f), 4) for f in range(n)]
        q.put((rank, got, seeds, f0, n))
    finally:
        dist.destroy_process_group()


def _worker_coalesced(rank, world, port, total, k, co, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1911_07434_b200.shard import FrameStream, shard_range, unshard_coalesced
        f0, n = shard_range(rank, world, total)
        nmax = max(shard_range(g, world, total)[1] for g in range(world))
        fs = FrameStream(lambda i: StubPlan(k), co * n, co * nmax, k, world, 2)
        got = []
        for launch, nb in enumerate((co, 1)):  # one full launch of `co` global batches, then a partial one
            b0 = launch * co
            x = torch.tensor([[1000 * (b0 + i) + f0 + f] for i in range(co) for f in range(n)], dtype=torch.float64)
            _, g = fs.step(x, frames=nb * n)
            got.append([r.numpy().copy() for r in unshard_coalesced(g, world, total, nb)])
        q.put((rank, got))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("total,co", [(5, 2), (8, 3)])
def test_frame_stream_coalesced_world2(total, co):
    """Shard coalescing (bench.py --coalesce): each rank runs its shards of `co` consecutive global batches in one
    launch; the gathered records unshard per batch into global frame order (uneven strong splits included)."""
    world, k = 2, 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_coalesced, args=(r, world, port, total, k, co, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, got in out:
        batches = [b for launch in got for b in launch]
        ids = list(range(co)) + [co]
        assert len(batches) == co + 1
        for b, recs in zip(ids, batches):
            gid = np.arange(total) + 1000 * b
            expect = np.concatenate([gid[:, None] * 10 + np.arange(k)[None, :], np.full((total, 1), k),
                                     (gid % 3)[:, None]], 1).astype(np.int32)
            assert np.array_equal(recs, expect), (rank, b)


@pytest.mark.parametrize("mode,total,depth", [("strong", 5, 2), ("strong", 8, 1), ("weak", 3, 2)])
def test_frame_stream_world2(mode, total, depth):
    world, k = 2, 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, total, k, mode, depth, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from paper_1911_07434_b200 import derive
    gframes = total if mode == "strong" else total * world
    for rank, got, seeds, f0, n in out:
        assert len(got) == 3
        for b, recs in enumerate(got):
            gid = np.arange(gframes) + 1000 * b
            expect = np.concatenate([gid[:, None] * 10 + np.arange(k)[None, :], np.full((gframes, 1), k),
                                     (gid % 3)[:, None]], 1).astype(np.int32)
            assert recs.shape == (gframes, k + 2)
            assert np.array_equal(recs, expect), (rank, b)
        assert seeds == [derive(derive(2, f0 + f), 4) for f in range(n)]
    # strong: the shards tile the batch contiguously
    if mode == "strong":
        spans = sorted((f0, n) for _, _, _, f0, n in out)
        assert spans[0][0] == 0 and spans[0][0] + spans[0][1] == spans[1][0] and sum(s[1] for s in spans) == total


def test_shard_range_validation():
    from paper_1911_07434_b200.shard import shard_range
    assert shard_range(3, 8, 1024) == (384, 128)
    assert shard_range(3, 8, 128, "weak") == (384, 128)
    assert [shard_range(g, 3, 10) for g in range(3)] == [(0, 4), (4, 3), (7, 3)]
    with pytest.raises(ValueError):
        shard_range(8, 8, 1)
    with pytest.raises(ValueError):
        shard_range(0, 2, 4, "diagonal")


def test_bench_refuses_mismatched_world(tmp_path):
    """bench.py --gpus N under a launcher with WORLD_SIZE != N exits non-zero instead of silently running N = 1."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--impl", "reference"],
                       env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 2 and "WORLD_SIZE" in r.stdout
