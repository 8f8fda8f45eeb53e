"""10000^2 step time (device events) for pipeline knobs: bands, k_tiles CTAs per band, chained receivers."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1803_02977_b200 import lem  # noqa: E402

def run(opts, steps=30):
    ctx = lem.DeviceContext(10000, 10000, lem.SimParams(), 8, options=opts)
    ctx.generate_terrain([42])
    ctx.step_async(5); ctx.sync()
    ctx.kernel_timing(True)
    ctx.step_async(steps); ctx.sync()
    kt = ctx.kernel_times()
    ctx.close()
    return kt["step"] / kt["launches"]

nsm = 148
for name, o in [("default", {}), ("pipe off", {"pipe": -1}), ("pipe 12", {"pipe": 12}), ("pipe 48", {"pipe": 48}),
                ("pipe 24 tiles 5/SM", {"pipe_tile_grid": 5 * nsm}), ("pipe 24 tiles 3/SM", {"pipe_tile_grid": 3 * nsm}),
                ("pipe 24 unchained", {"pipe_unchained": 1}), ("default", {})]:
    print(f"{name:22s} {run(o):.4f} ms/step", flush=True)
