"""Deep-plan regime (every tree escapes its tile; long drainage chains):
a tilted plane + small noise.  Checks a few steps against the oracle and
times the device step.  usage: python tools/deep_probe.py W H steps"""
import sys, time
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np
import paper_1803_02977_b200 as lem
from _oracle import Oracle

w, h, n = (int(x) for x in sys.argv[1:4])
rng = np.random.default_rng(5)
x = np.arange(w)[None, :].astype(np.float64)
y = np.arange(h)[:, None].astype(np.float64)
e = 0.05 * x + 0.01 * y + 1e-3 * rng.random((h, w))
o = Oracle.get()
ctx = lem.DeviceContext(w, h, lem.SimParams(), 8)
ctx.upload(e)
for s in range(n):
    d = ctx.step(1)[0]
    r = o.step(e, want_donor=False)
    ok = np.array_equal(ctx.download().view(np.uint64), e.view(np.uint64)) and d.newton_iters == r["newton_iters"]
    print(f"step {s}: nlevels {d.nlevels} (oracle {r['nlevels']}), escaped trees {d.escaped_trees}, bit-exact {ok}", flush=True)
ctx.kernel_timing(True)
ctx.step_async(5)
ctx.sync()
kt = ctx.kernel_times()
print("ms/step", {k: round(v / kt['launches'], 3) for k, v in kt.items() if k != 'launches'})
