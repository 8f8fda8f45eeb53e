"""Ensemble sharding across GPUs (BASELINE configs[4]; paper future work,
PAPER.md:749, :761).

Independent realisations are the only data-parallel axis of this workload: a
single DEM does not shard (drainage basins cross any stripe), so
members are split over ranks in contiguous balanced ranges -- the same rule
the reference uses to split sources over workers (``partition_sources``,
proj/src/scheduler.cpp:396-406) -- and batched into one device context per
rank.  The only collective is the per-step reduction of per-member
statistics (mean / max / min / sum of h), a few KB over NCCL.
"""
from __future__ import annotations

from typing import List, Tuple

import numpy as np


def member_bounds(members: int, world: int) -> List[int]:
    """bounds[w] = members * w // world (scheduler.cpp:403-404)."""
    if world < 1:
        raise ValueError("world must be >= 1")
    return [members * w // world for w in range(world + 1)]


def member_ids(members: int, world: int, rank: int) -> List[int]:
    b = member_bounds(members, world)
    return list(range(b[rank], b[rank + 1]))


def member_params(i: int) -> Tuple[int, float, float]:
    """(seed, K, m) of ensemble member i."""
    return 1000 + i, 1e-6 * (1 + i % 8), 0.35 + 0.05 * (i // 8)


def reduce_member_stats(local, ids: List[int], members: int, group=None):
    """Assemble the [members, 4] table {mean, max, min, sum} of h on every rank.

    ``local`` is this rank's [len(ids), 4] tensor (any torch device); rows of
    other ranks' members are filled by three all-reduces (SUM for mean/sum,
    MAX, MIN) -- every member is owned by exactly one rank, so the sums are
    exact copies, not floating-point reductions."""
    import torch
    import torch.distributed as dist

    dev = local.device
    s = torch.zeros(members, 2, dtype=torch.float64, device=dev)
    mx = torch.full((members,), -float("inf"), dtype=torch.float64, device=dev)
    mn = torch.full((members,), float("inf"), dtype=torch.float64, device=dev)
    idx = torch.tensor(ids, dtype=torch.long, device=dev)
    if len(ids):
        s[idx, 0] = local[:, 0]
        s[idx, 1] = local[:, 3]
        mx[idx] = local[:, 1]
        mn[idx] = local[:, 2]
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(s, group=group)
        dist.all_reduce(mx, op=dist.ReduceOp.MAX, group=group)
        dist.all_reduce(mn, op=dist.ReduceOp.MIN, group=group)
    return torch.stack([s[:, 0], mx, mn, s[:, 1]], dim=1)


def numpy_member_stats(h: np.ndarray) -> np.ndarray:
    """Reference statistics of a [M, H, W] stack (for tests)."""
    flat = h.reshape(h.shape[0], -1)
    return np.stack([flat.mean(1), flat.max(1), flat.min(1), flat.sum(1)], axis=1)
