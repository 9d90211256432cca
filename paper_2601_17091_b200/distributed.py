"""Series-sharded multi-GPU execution (one process per GPU).

The reference models multi-device execution as contiguous near-equal row
shards run in isolation and concatenated in order
(/root/reference/pkg/src/gridrocket/engine.py:123-134, 336-364).  Here each
rank of a torch.distributed job owns shard ``plan_shards(N, world)[rank]``,
transforms it on its own GPU with the replicated bank — no collective on the
hot path — and, only when a consumer needs the whole feature matrix (the
downstream ridge fit), gathers the row blocks with one all-gather (NCCL over
NVLink on GPUs, gloo on CPU).
"""

import numpy as np

from .engine import plan_shards


def shard_of(n_series: int, world: int, rank: int):
    """(start, count) of this rank's rows (plan_shards, engine.py:123-134)."""
    return plan_shards(n_series, world)[rank]


def gather_rows(local, n_series: int, group=None):
    """All-gather near-equal row shards into the full (n_series, F) matrix.

    ``local`` is this rank's (count, F) block as a torch tensor on the
    process group's device.  Shards differ by at most one row, so every
    rank pads to the largest shard, one all_gather_into_tensor moves the
    blocks, and the padding is dropped in rank order — the result equals an
    ordered concatenation of the shards (engine.py:357-361).
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    shards = plan_shards(n_series, world)
    width = local.shape[1]
    biggest = max(c for _, c in shards)
    padded = torch.zeros((biggest, width), dtype=local.dtype, device=local.device)
    padded[: local.shape[0]] = local
    full = torch.empty((world * biggest, width), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(full, padded, group=group)
    parts = [full[r * biggest : r * biggest + c] for r, (_, c) in enumerate(shards)]
    return torch.cat(parts, dim=0)


def sharded_transform(values, bank, transform_fn, group=None):
    """Run ``transform_fn(rows) -> (count, F) array`` on this rank's shard of
    ``values`` and return (start, features) — the per-rank half of
    transform_sharded without any collective."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    start, count = shard_of(values.shape[0], world, rank)
    rows = np.asarray(values)[start : start + count]
    return start, transform_fn(rows)
