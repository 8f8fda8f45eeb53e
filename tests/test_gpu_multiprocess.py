"""Two ranks on the box's one GPU (-m gpu): the sharded ensemble product path
end to end in separate processes -- lemgpu_create_ensemble_shard per rank
(contiguous balanced member ranges, per-member K and m), the per-member
statistics computed in each rank's step graph, the table assembled across
ranks.  NCCL refuses two ranks on one device (ncclCommInitRank: invalid usage,
tools/two_ranks_probe.py), so the cross-rank assembly of the table goes
through gloo here; the NCCL all-reduce captured in the step graph is tested
with one rank in test_gpu_parity.py."""
import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _stats(hh):
    """{mean, max, min, sum} per member, the reference's summation order (row-major)."""
    out = np.zeros((hh.shape[0], 4))
    for i, h in enumerate(hh):
        s = 0.0
        for v in h.ravel():
            s += v
        out[i] = (s / h.size, h.max(), h.min(), s)
    return out


def _worker(rank, world, port, w, h, M, steps, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    import torch
    import torch.distributed as dist

    from _oracle import Oracle, make_params
    from paper_1803_02977_b200 import ensemble

    dist.init_process_group("gloo", rank=rank, world_size=world)
    ora = Oracle.get()
    ens = ensemble.DeviceEnsemble(w, h, M, device=0, rank=rank, world=world, use_nccl=False)
    ens.generate_terrain()
    refs = [ora.terrain(w, h, ensemble.member_params(i)[0]) for i in range(M)]
    bad = []
    for s in range(steps):
        want = _stats(np.stack(refs))  # the statistics of the elevation the step reads
        ens.ctx.step(1)
        for i in range(M):
            _, K, m = ensemble.member_params(i)
            ora.step(refs[i], params=make_params(K=K, m_exp=m), want_donor=False)
        g = ens.ctx.download()
        for j, i in enumerate(ens.ids):
            if not np.array_equal(g[j].view(np.uint64), refs[i].view(np.uint64)):
                bad.append(f"step {s} member {i}: elevation differs")
        t = torch.from_numpy(ens.table().copy())
        local_rows = int((np.abs(t.numpy()).sum(axis=1) > 0).sum())
        if local_rows != len(ens.ids):
            bad.append(f"step {s}: {local_rows} local table rows for {len(ens.ids)} members")
        dist.all_reduce(t)  # rows are disjoint between the ranks: an exact gather
        tt = t.numpy()
        if not (np.array_equal(tt[:, 1], want[:, 1]) and np.array_equal(tt[:, 2], want[:, 2])
                and np.allclose(tt[:, 3], want[:, 3], rtol=1e-13)):
            bad.append(f"step {s}: assembled statistics differ")
    out[rank] = {"ids": list(ens.ids), "bad": bad}
    ens.close()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_ensemble_shards_two_processes_one_gpu():
    import torch.multiprocessing as mp

    w, h, M, world = 72, 50, 7, 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), w, h, M, 3, out), nprocs=world, join=True)
    assert sorted(out.keys()) == [0, 1]
    assert out[0]["ids"] + out[1]["ids"] == list(range(M))  # partition_sources' contiguous ranges
    assert out[0]["bad"] == [] and out[1]["bad"] == [], (out[0]["bad"], out[1]["bad"])
