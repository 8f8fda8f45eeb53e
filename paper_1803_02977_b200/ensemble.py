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


def nccl_unique_id() -> bytes:
    """ncclGetUniqueId through the library (libnccl.so.2 loaded at run time)."""
    import ctypes as C

    from . import _abi

    buf = C.create_string_buffer(128)
    rc = _abi.lib().lemgpu_nccl_unique_id(buf, 128)
    if rc != 0:
        raise RuntimeError(_abi.lib().lemgpu_error_message(None).decode())
    return buf.raw


class DeviceEnsemble:
    """One rank's shard of an ensemble of ``members`` realisations (configs[4]):
    its member range (the reference's partition rule), batched into ONE device
    context (lemgpu_create_ensemble_shard), with the per-member statistics
    computed inside every (or every stats_interval-th) step's CUDA graph and --
    for world > 1 -- all-reduced by ONE ncclAllReduce captured in that graph.  torch.distributed is
    only the rendezvous that carries the NCCL id; the per-step data path is
    C++/CUDA/NCCL on the context's stream."""

    def __init__(self, width: int, height: int, members: int, params=None, member_fn=member_params,
                 device: int = 0, rank: int = 0, world: int = 1, options=None, group=None, use_nccl: bool = True,
                 stats_interval: int = 1):
        import ctypes as C

        from . import _abi
        from .lem import DeviceContext, SimParams, make_options

        params = params or SimParams()
        self.members, self.rank, self.world = int(members), int(rank), int(world)
        self.ids = member_ids(self.members, self.world, self.rank)
        table = [member_fn(i) for i in range(self.members)]
        self.seeds = [t[0] for t in table]
        L = _abi.lib()
        arr = (_abi.lemgpu_member * self.members)(*[_abi.lemgpu_member(float(t[1]), float(t[2])) for t in table])
        p = params.to_abi(8)
        opts = make_options(options)
        h = C.c_void_p()
        rc = L.lemgpu_create_ensemble_shard(device, int(width), int(height), self.members, self.world, self.rank,
                                            C.byref(p), arr, int(stats_interval),
                                            C.byref(opts) if opts is not None else None, C.byref(h))
        if rc != _abi.OK:
            raise RuntimeError(L.lemgpu_error_message(None).decode())
        # wrap the raw handle in a DeviceContext (same ownership rules)
        ctx = DeviceContext.__new__(DeviceContext)
        ctx.width, ctx.height, ctx.members, ctx.connectivity = int(width), int(height), len(self.ids), 8
        ctx._h, ctx._L = h, L
        ctx.n = ctx.width * ctx.height * ctx.members
        ctx.stats_total = self.members
        self.ctx = ctx
        if self.world > 1 and use_nccl:
            import torch.distributed as dist

            obj = [nccl_unique_id() if self.rank == 0 else None]
            dist.broadcast_object_list(obj, src=0, group=group)
            ctx.stats_comm_init(obj[0], self.world, self.rank)

    def generate_terrain(self):
        self.ctx.generate_terrain([self.seeds[i] for i in self.ids])

    def table(self) -> np.ndarray:
        """[members, 4] {mean, max, min, sum} of h after the last step that computed them (all ranks' members)."""
        return self.ctx.stats_table()

    def close(self):
        self.ctx.close()


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
