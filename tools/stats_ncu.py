"""Run a few eager ens64 steps with or without fused stats (for ncu)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1803_02977_b200 as lem  # noqa: E402
from paper_1803_02977_b200 import ensemble  # noqa: E402

stats = sys.argv[1] == "1"
M = 64
ctx = lem.DeviceContext(2000, 2000, lem.SimParams(), 8, members=M,
                        per_member=[ensemble.member_params(i)[1:] for i in range(M)], options={"eager": 1, "pipe": -1})
if stats:
    ctx.stats_enable()
ctx.generate_terrain([1000 + i for i in range(M)])
ctx.step(3)
