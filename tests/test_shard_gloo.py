"""N>1 path on CPU: world_size-2 gloo process group exercising the frame sharding and the
peak-record all-gather used by bench.py's multi-GPU run."""
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


def _worker(rank, world, port, frames, k, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1911_07434_b200 import derive
        from paper_1911_07434_b200.shard import gather_records, pack_records, shard_range
        f0, nf = shard_range(rank, world, frames)
        # per-frame draw seeds depend only on the global frame index (shard-invariant)
        seeds = [derive(derive(2, f0 + f), 4) for f in range(nf)]
        cells = torch.tensor([[(f0 + f) * 10 + j for j in range(k)] for f in range(nf)], dtype=torch.int32)
        count = torch.full((nf,), k, dtype=torch.int32)
        status = torch.tensor([(f0 + f) % 3 for f in range(nf)], dtype=torch.int32)
        g = gather_records(pack_records(cells, count, status), world)
        q.put((rank, g.numpy().copy(), seeds))
    finally:
        dist.destroy_process_group()


def test_sharded_gather_world2():
    world, frames, k = 2, 5, 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, frames, k, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from paper_1911_07434_b200 import derive
    expect = np.array([[f * 10 + j for j in range(k)] + [k, f % 3] for f in range(world * frames)], np.int32)
    for rank, g, seeds in out:
        assert g.shape == (world, frames, k + 2)
        assert np.array_equal(g.reshape(-1, k + 2), expect)
        assert seeds == [derive(derive(2, rank * frames + f), 4) for f in range(frames)]


def test_shard_range_validation():
    from paper_1911_07434_b200.shard import shard_range
    assert shard_range(3, 8, 128) == (384, 128)
    with pytest.raises(ValueError):
        shard_range(8, 8, 1)
