"""Frame sharding across GPUs and the peak-record all-gather.

Frames are independent, so rank r of W owns the contiguous frame range [r*B, (r+1)*B) of the
global stream (weak scaling, no data-path collective). The only collective is the gather of
the fixed-size per-frame peak records {K cells, count, status} after each batch — one
all_gather_into_tensor over NCCL (GPU) or gloo (CPU tests), ~B*(K+2)*4 bytes per rank.
"""
from __future__ import annotations


def shard_range(rank: int, world: int, frames_per_rank: int) -> tuple[int, int]:
    """Global index of this rank's first frame and its frame count."""
    if world < 1 or not (0 <= rank < world) or frames_per_rank < 0:
        raise ValueError("shard_range: need 0 <= rank < world and frames_per_rank >= 0")
    return rank * frames_per_rank, frames_per_rank


def pack_records(peak_cells, peak_count, status, out=None):
    """[B, K+2] int32 record per frame: K cells, count, status (device or host tensors)."""
    import torch
    b, k = peak_cells.shape
    rec = out if out is not None else torch.empty((b, k + 2), dtype=torch.int32, device=peak_cells.device)
    rec[:, :k].copy_(peak_cells)
    rec[:, k].copy_(peak_count)
    rec[:, k + 1].copy_(status)
    return rec


def gather_records(rec, world: int, out=None, group=None):
    """All-gather every rank's [B, K+2] records into [world, B, K+2] (rank-major = frame order)."""
    import torch
    import torch.distributed as dist
    if world == 1:
        return rec.unsqueeze(0)
    g = out if out is not None else torch.empty((world,) + tuple(rec.shape), dtype=rec.dtype, device=rec.device)
    dist.all_gather_into_tensor(g.view(-1, rec.shape[1]), rec.contiguous(), group=group)
    return g
