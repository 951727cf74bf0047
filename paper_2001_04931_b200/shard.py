"""Multi-GPU sharding of independent MPC instances.

One process per GPU.  Instances are split into contiguous ranges, solved
with no collective inside the solve (each instance's selection is local to
its own population), and the per-instance results are gathered once per
control step.  This mirrors the reference harness's process-level parallelism
over independent tasks (K/bench.py:688-705), with results independent of the
number of ranks because every instance keeps its own RNG counters.
"""

from __future__ import annotations

import numpy as np


def instance_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """(first, count) of the contiguous instance block owned by `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("invalid rank / world size")
    per = (total + world - 1) // world
    first = min(total, rank * per)
    return first, max(0, min(per, total - first))


def gather_instances(local: np.ndarray, total: int, group=None) -> np.ndarray:
    """All-gather per-instance rows (local block of shape (count, ...)) into a
    (total, ...) array on every rank, in instance order."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    first, count = instance_range(total, rank, world)
    assert local.shape[0] == count
    per = (total + world - 1) // world
    row_shape = local.shape[1:]
    buf = np.zeros((per,) + row_shape, dtype=local.dtype)
    buf[:count] = local
    t = torch.from_numpy(buf)
    if dist.get_backend(group) == "nccl":
        t = t.cuda()
    outs = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(outs, t, group=group)
    full = np.concatenate([o.cpu().numpy() for o in outs])[:total]
    return full
