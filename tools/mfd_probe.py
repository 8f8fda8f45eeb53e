"""MFD tile passes: passes per step and step time (device events) at a few sizes."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_1803_02977_b200 as lem

for n in [int(x) for x in (sys.argv[1:] or ["1000", "4000", "10000"])]:
    ctx = lem.DeviceContext(n, n, lem.SimParams(), 8)
    ctx.generate_terrain([42])
    ctx.set_routing(lem.Routing.kMfd, 1.0)
    for s in range(int(__import__("os").environ.get("PROBE_STEPS", "6"))):
        t = time.time()
        d = ctx.step(1)[0]
        dt = time.time() - t
        print(n, "step", s, "passes", d.mfd_passes, "wall ms %.2f" % (dt * 1e3), "nlev", d.nlevels, "esc", d.escaped_cells, flush=True)
    ctx.close()
