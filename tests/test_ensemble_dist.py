"""Multi-process (gloo, world_size 2, CPU) checks of the ensemble sharding and
the per-step statistics reduction used by bench.py at N > 1."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1803_02977_b200 import ensemble


def test_member_partition_matches_reference_rule():
    # partition_sources (scheduler.cpp:396-406): contiguous, balanced, complete
    for M in (1, 7, 64):
        for world in (1, 2, 3, 4, 8):
            b = ensemble.member_bounds(M, world)
            assert b[0] == 0 and b[-1] == M
            ids = [i for r in range(world) for i in ensemble.member_ids(M, world, r)]
            assert ids == list(range(M))
            sizes = [b[r + 1] - b[r] for r in range(world)]
            assert max(sizes) - min(sizes) <= 1
    assert ensemble.member_params(0) == (1000, 1e-6, 0.35)
    assert ensemble.member_params(63)[1:] == (8e-6, 0.35 + 0.05 * 7)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, M, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(0)
    h = rng.random((M, 6, 5))  # every rank builds the same synthetic stack
    full = ensemble.numpy_member_stats(h)
    ids = ensemble.member_ids(M, world, rank)
    local = torch.from_numpy(full[ids].copy())
    table = ensemble.reduce_member_stats(local, ids, M)
    out[rank] = float(np.abs(table.numpy() - full).max())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("M", [5, 64])
def test_stats_allreduce_gloo_world2(M):
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), M, out), nprocs=world, join=True)
    assert sorted(out.keys()) == [0, 1]
    assert all(v == 0.0 for v in out.values())


def test_shard_members_c_abi_matches_python_rule():
    """lemgpu_shard_members (the C-ABI the product ensemble entry uses) and the
    Python rule agree for every (members, world, rank)."""
    import ctypes as C

    from paper_1803_02977_b200 import _abi

    L = _abi.lib()
    for M in (1, 5, 64, 100):
        for world in (1, 2, 3, 4, 8):
            for rank in range(world):
                f, c = C.c_uint32(), C.c_uint32()
                assert L.lemgpu_shard_members(M, world, rank, C.byref(f), C.byref(c)) == 0
                ids = ensemble.member_ids(M, world, rank)
                assert (f.value, c.value) == ((ids[0] if ids else f.value), len(ids))
    assert L.lemgpu_shard_members(4, 2, 2, C.byref(C.c_uint32()), C.byref(C.c_uint32())) != 0
