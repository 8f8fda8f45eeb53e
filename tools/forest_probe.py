"""Timeline of k_esc_forest on an epsilon-filled DEM (debug / optimisation aid).
Usage: python tools/forest_probe.py N [steps] [knob=value ...]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1803_02977_b200 as lem  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
opts = dict(kv.split("=") for kv in sys.argv[3:])
opts = {k: int(v) for k, v in opts.items()} or None
ctx = lem.DeviceContext(n, n, lem.SimParams(), options=opts)
ctx.generate_terrain([42])
ctx.fill(mode=2, epsilon=1e-8)
for _ in range(steps):
    d = ctx.step(1)[0]
tl = ctx.debug_timeline()
print(f"{n}^2 filled nlevels={d.nlevels} escaped={d.escaped_cells} misses={d.lut_misses} kernel_ms={[round(x*1e3,3) for x in d.kernel_seconds]}")
print("timeline (ms):", " ".join(f"{t:.3f}" for t in tl))
print("deltas   (ms):", " ".join(f"{b-a:.3f}" for a, b in zip(tl, tl[1:])))
import ctypes as C
import numpy as np
buf = np.zeros(3 * 4096, np.uint32)
ctx._check(ctx._L.lemgpu_debug_copy(ctx._h, 5, buf.ctypes.data, buf.nbytes))
st = buf[4096:4096 + 8 * 148].reshape(148, 8).astype(np.int64)
top = np.argsort(-(st[:, 4] + st[:, 7]))[:6]
print("CTA: levels cells acc_threads - acc_kcyc - - ero_kcyc")
for b in top:
    print(b, list(st[b]), f"acc {st[b,4]*1024/1.965e3/max(st[b,0],1):.3f} us/level, ero {st[b,7]*1024/1.965e3/max(st[b,0],1):.3f} us/level")
