"""Per-barrier timeline of k_flow at a given size (debug / optimisation aid)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1803_02977_b200 as lem  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
ctx = lem.DeviceContext(n, n, lem.SimParams())
ctx.generate_terrain([42])
for _ in range(4):
    d = ctx.step(1)[0]
tl = ctx.debug_timeline()
print(f"{n}^2 nlevels={d.nlevels} phases(ms)=" + ", ".join(f"{k}:{v*1e3:.3f}" for k, v in d.timings.items()))
print("timeline (ms):", " ".join(f"{t:.3f}" for t in tl))
print("deltas   (ms):", " ".join(f"{b-a:.3f}" for a, b in zip(tl, tl[1:])))
g = ctx.download_graph(rec=False, dnum=False, order=False, A=False)
lv = g["levels"]
print("level sizes:", [int(lv[i + 1] - lv[i]) for i in range(len(lv) - 1)])
