"""configs[3]: sweep of square random-noise DEMs on one B200 (device-resident
cell-steps/s per size).  Prints one JSON object.

usage: python tools/sweep.py [sizes...]"""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1803_02977_b200 as lem  # noqa: E402


def run(n, steps):
    ctx = lem.DeviceContext(n, n, lem.SimParams(), 8)
    ctx.generate_terrain([42])
    ctx.step_async(3)
    ctx.sync()
    ctx.kernel_timing(True)
    ctx.step_async(steps)
    d = ctx.sync()
    kt = ctx.kernel_times()
    ctx.kernel_timing(False)
    ms = kt["step"] / max(kt["launches"], 1)
    ctx.close()
    return {"size": n, "ms_per_step": ms, "cell_steps_per_s": n * n / (ms / 1e3), "nlevels": d[-1].nlevels,
            "escaped_trees": d[-1].escaped_trees,
            "k_tiles_ms": kt["tiles"] / kt["launches"], "k_recv_ms": kt["recv_donor"] / kt["launches"]}


sizes = [int(x) for x in sys.argv[1:]] or [500, 1000, 2000, 2500, 4000, 5000, 8000, 10000, 16000, 20000]
out = []
for n in sizes:
    r = run(n, 20 if n >= 8000 else 50)
    out.append(r)
    print(json.dumps(r), file=sys.stderr, flush=True)
# piecewise scaling exponents of time vs N (the paper's 0.33/0.16/0.42/0.92)
for a, b in zip(out, out[1:]):
    b["exponent_vs_prev"] = float(np.log(b["ms_per_step"] / a["ms_per_step"]) / np.log((b["size"] / a["size"]) ** 2))
print(json.dumps({"sweep": out, "data": "synthetic random-noise DEMs, seed 42, defaults, D8, n=1"}))
