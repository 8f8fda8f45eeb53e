"""Odd-sized raster (no TMA: odd W; tiles straddling every edge) at scale:
one step against the oracle, then the device step time."""
import sys, time
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np
import paper_1803_02977_b200 as lem
from _oracle import Oracle
w, h = int(sys.argv[1]), int(sys.argv[2])
o = Oracle.get()
e = o.terrain(w, h, 7)
ctx = lem.DeviceContext(w, h, lem.SimParams(), 8)
ctx.upload(e)
d = ctx.step(1)[0]
t = time.time(); r = o.step(e, want_donor=False); t = time.time() - t
ok = np.array_equal(ctx.download().view(np.uint64), e.view(np.uint64)) and d.newton_iters == r["newton_iters"] and d.nlevels == r["nlevels"]
print(f"{w}x{h}: bit-exact {ok}, oracle step {t:.1f} s", flush=True)
ctx.kernel_timing(True); ctx.step_async(10); ctx.sync(); kt = ctx.kernel_times()
print("ms/step", {k: round(v / kt['launches'], 3) for k, v in kt.items() if k != 'launches'}, "cell-steps/s %.3e" % (w * h / (kt['step'] / kt['launches'] / 1e3)))
