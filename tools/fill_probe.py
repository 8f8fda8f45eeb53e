"""Time lemgpu_fill (device Priority-Flood) against the reference's
lem::priority_flood_fill on the host, same terrain."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from paper_1803_02977_b200 import lem
from _oracle import RefLib
ref = RefLib.get() if RefLib.available() else None
for n in [int(x) for x in (sys.argv[1:] or ["1000", "4000", "10000"])]:
    for mode in (1, 2):
        ctx = lem.DeviceContext(n, n, lem.SimParams(), 8)
        ctx.generate_terrain([42])
        e = ctx.download() if ref is not None and n <= 4000 else None
        t0 = time.perf_counter()
        ctx.fill(mode=mode)
        tg = time.perf_counter() - t0
        line = f"{n}^2 mode {mode}: device fill {tg * 1e3:.1f} ms"
        if e is not None:
            t0 = time.perf_counter()
            f = ref.fill(e, mode)
            tc = time.perf_counter() - t0
            same = np.array_equal(f.view(np.uint64), ctx.download().view(np.uint64))
            line += f", reference priority_flood_fill {tc * 1e3:.0f} ms, identical={same}"
        print(line, flush=True)
        ctx.close()
