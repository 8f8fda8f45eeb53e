"""configs[3]: sweep of square random-noise DEMs on one B200 (device-resident
cell-steps/s per size), with the unmodified reference's
rb_private_queues on all host cores beside it (--cpu) and the piecewise scaling
exponents of time vs cells over the paper's regions (A 0.33
up to 400², B 0.16 to 1000², C 0.42 to 2500², D 0.92 to 16000², RB+GPU on a
P100).  Prints one JSON object.

usage: python tools/sweep.py [--cpu] [sizes...]"""
import json
import os
import sys
import time
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


def run_cpu(n):
    """The reference's own step (oracle/_ref, test infrastructure: the CPU baseline only)."""
    sys.path.insert(0, str(ROOT / "tests"))
    from _oracle import RefLib  # noqa: E402

    if not RefLib.available():
        return None
    ref = RefLib.get()
    threads = len(os.sched_getaffinity(0))
    est = 3e-8 * n * n * 16 / threads
    steps = int(max(2, min(20, 8.0 // max(est, 1e-4))))
    secs, _ = ref.bench(n, n, steps, warmup=1, strategy="rb_private_queues", workers=threads)
    t = float(np.median(secs))
    return {"cpu_ms_per_step": t * 1e3, "cpu_cell_steps_per_s": n * n / t, "cpu_threads": threads,
            "cpu_steps": steps}


def exponents(rows, key):
    """time ~ cells^x between consecutive sizes and over the paper's regions."""
    by = {r["size"]: r[key] for r in rows if r.get(key)}
    regions = {"A (to 400^2)": (100, 400), "B (400^2-1000^2)": (400, 1000), "C (1000^2-2500^2)": (1000, 2500),
               "D (2500^2-16000^2)": (2500, 16000)}
    out = {}
    for name, (a, b) in regions.items():
        if a in by and b in by:
            out[name] = float(np.log(by[b] / by[a]) / np.log((b / a) ** 2))
    return out


args = [x for x in sys.argv[1:] if x != "--cpu"]
cpu = "--cpu" in sys.argv[1:]
sizes = [int(x) for x in args] or [100, 200, 400, 500, 1000, 2000, 2500, 4000, 5000, 8000, 10000, 16000, 20000]
out = []
for n in sizes:
    r = run(n, 20 if n >= 8000 else 50)
    if cpu:
        r.update(run_cpu(n) or {})
    out.append(r)
    print(json.dumps(r), file=sys.stderr, flush=True)
for a, b in zip(out, out[1:]):
    b["exponent_vs_prev"] = float(np.log(b["ms_per_step"] / a["ms_per_step"]) / np.log((b["size"] / a["size"]) ** 2))
res = {"sweep": out, "data": "synthetic random-noise DEMs, seed 42, defaults, D8, n=1",
       "gpu_region_exponents": exponents(out, "ms_per_step"),
       "paper_rb_gpu_p100_region_exponents": {"A": 0.33, "B": 0.16, "C": 0.42, "D": 0.92}}
if cpu:
    res["cpu_region_exponents"] = exponents(out, "cpu_ms_per_step")
    res["cpu"] = "the unmodified reference (oracle/_ref), lem::strategy_step(rb_private_queues), all host threads"
print(json.dumps(res))
