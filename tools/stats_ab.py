"""A/B: ens64 (64 x 2000^2) step time: baseline, after a graph rebuild, with the fused member statistics."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1803_02977_b200 as lem  # noqa: E402
from paper_1803_02977_b200 import ensemble  # noqa: E402

w = h = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
M = int(sys.argv[1]) if len(sys.argv) > 1 else 64
km = [ensemble.member_params(i)[1:] for i in range(M)]
for mode in ("base", "stats", "stats10", "base", "stats", "stats10"):
    ctx = lem.DeviceContext(w, h, lem.SimParams(), 8, members=M, per_member=km)
    if mode == "stats":
        ctx.stats_enable()
    elif mode == "stats10":
        ctx.stats_enable(interval=10)
    elif mode == "rebuilt":
        ctx.tile_capture(True)
        ctx.tile_capture(False)
    ctx.generate_terrain([1000 + i for i in range(M)])
    ctx.step(3)
    ctx.kernel_timing(True)
    t0 = time.perf_counter()
    ctx.step(10)
    dt = (time.perf_counter() - t0) / 10
    kt = ctx.kernel_times()
    n = max(kt["launches"], 1)
    print(f"{mode}: wall {dt*1e3:.3f} ms/step, events {kt['step']/n:.3f}, k_recv span {kt['recv_donor']/n:.3f}, "
          f"k_tiles span {kt['tiles']/n:.3f}, bands {ctx.pipeline_bands()}")
    ctx.close()
