"""Multi-GPU execution of the VGG16 stack (BASELINE config 4).

The path shards naturally: images are independent and the transformed
filters are read-only, so rank r of N takes images [r*B/N, (r+1)*B/N), runs
all 13 layers locally, and the ranks meet exactly once, in one all-gather of
the final (B/N, 7, 7, 512) int8 maps.  No collective sits on
the hot path.  Timing is the max over ranks of device-measured elapsed time.

Backend-agnostic (NCCL on the GPU box, gloo for the CPU tests).
"""

from __future__ import annotations

import os


def dist_env() -> tuple[int, int, int]:
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard_range(batch: int, world: int, rank: int) -> tuple[int, int]:
    """(first image, image count) of this rank; the batch must divide evenly
    so every rank's shard has the same shape (required by all_gather)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    if batch % world:
        raise ValueError(f"batch {batch} is not divisible by {world} ranks")
    per = batch // world
    return rank * per, per


def gather_maps(local, world: int, out=None, force: bool = False):
    """All-gather equal-shaped per-rank tensors along dim 0 (rank order).
    ``force`` runs the collective even for a single rank (a one-GPU check of
    the NCCL path)."""
    import torch
    import torch.distributed as dist

    if world == 1 and not force:
        return local
    if out is None:
        out = torch.empty((local.shape[0] * world, *local.shape[1:]), dtype=local.dtype, device=local.device)
    if dist.get_backend() == "nccl":
        dist.all_gather_into_tensor(out, local.contiguous())
    else:
        parts = list(out.chunk(world, dim=0))
        dist.all_gather(parts, local.contiguous())
        if parts[0].data_ptr() != out.data_ptr():
            torch.cat(parts, out=out)
    return out


def max_over_ranks(seconds: float, world: int, device=None, force: bool = False) -> float:
    import torch
    import torch.distributed as dist

    if world == 1 and not force:
        return seconds
    t = torch.tensor([seconds], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
