"""Where the end-to-end (host raster) step's time goes: raw PCIe copies of the
raster alone and overlapped, and lemgpu_step_host at several band counts."""
import os, sys, time
import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1803_02977_b200 import lem  # noqa: E402

N = 10000
nbytes = N * N * 8
hp = torch.empty(N * N, dtype=torch.float64).pin_memory()
hq = torch.empty(N * N, dtype=torch.float64).pin_memory()
d1 = torch.empty(N * N, dtype=torch.float64, device="cuda")
d2 = torch.empty(N * N, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best * 1e3


print("h2d ms", round(timed(lambda: d1.copy_(hp, non_blocking=True)), 2))
print("d2h ms", round(timed(lambda: hq.copy_(d2, non_blocking=True)), 2))


def both():
    with torch.cuda.stream(s1):
        d1.copy_(hp, non_blocking=True)
    with torch.cuda.stream(s2):
        hq.copy_(d2, non_blocking=True)


print("h2d+d2h concurrent ms", round(timed(both), 2))
del d1, d2, hq
torch.cuda.empty_cache()
for bands in [1, 4, 8, 16, 32, 64]:
    ctx = lem.DeviceContext(N, N, lem.SimParams(), 8, options={"host_bands": bands})
    ctx.generate_terrain([42])
    host = hp.numpy().reshape(N, N)
    ctx.download(host)
    ctx.step_host(host)
    ts = []
    for _ in range(4):
        t0 = time.perf_counter()
        d = ctx.step_host(host)
        ts.append(time.perf_counter() - t0)
    print("bands", bands, "ms/step", round(1e3 * min(ts), 2), "escaped trees", d.escaped_trees)
    del ctx
