"""Probe: two ranks sharing one GPU, each with its DeviceEnsemble shard and the
NCCL all-reduce of the member statistics in its step graph (does NCCL accept
two ranks on one device here?).  torchrun --nproc-per-node 2 tools/two_ranks_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch.distributed as dist

from paper_1803_02977_b200 import ensemble

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo")
ens = ensemble.DeviceEnsemble(96, 80, 6, device=0, rank=rank, world=world)
ens.generate_terrain()
ens.ctx.step(2)
t = ens.table()
print(rank, "members", ens.ids, "table rows nonzero", int((np.abs(t).sum(axis=1) > 0).sum()), flush=True)
ens.close()
dist.destroy_process_group()
