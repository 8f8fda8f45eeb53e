"""Small steps under every schedule knob, for compute-sanitizer (memcheck /
racecheck / synccheck / initcheck): `compute-sanitizer --tool X python tools/sanitize_run.py`.
Each case also checks its result against the CPU oracle (bit-exact)."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import paper_1803_02977_b200 as lem  # noqa: E402
from _oracle import Oracle, make_params  # noqa: E402

ora = Oracle.get()


def ramp(w, h, seed):
    rng = np.random.default_rng(seed)
    x = np.arange(w)[None, :].astype(np.float64)
    y = np.arange(h)[:, None].astype(np.float64)
    return 0.05 * x + 0.01 * y + 1e-3 * rng.random((h, w))


CASES = [
    ("tiles", {}, {}, "noise", 130, 97),
    ("tiles-eager", {"eager": 1}, {}, "noise", 130, 97),
    ("all-escape", {"force_escape": 1}, {}, "noise", 130, 97),
    ("half-escape", {"force_escape": 2}, {}, "noise", 130, 97),
    ("all-escape-coop", {"force_escape": 1, "no_esc_small": 1}, {}, "noise", 100, 80),
    ("all-escape-deep", {"force_escape": 1, "force_deep": 1}, {}, "noise", 100, 80),
    ("global", {"global_path": 1}, {}, "noise", 100, 80),
    ("global-eager", {"global_path": 1, "eager": 1}, {}, "noise", 100, 80),
    ("deep-ramp", {}, {}, "ramp", 200, 150),
    ("deep-ramp-nonarrow", {"no_narrow": 1}, {}, "ramp", 200, 150),
    ("no-tma", {"no_tma": 1}, {}, "noise", 131, 70),
    ("n2", {}, {"n_exp": 2.0}, "noise", 100, 80),
    ("fp-area", {}, {"dx": 0.1, "dy": 0.3}, "noise", 100, 80),
    ("few-tile-ctas", {"tile_grid": 3}, {}, "noise", 200, 120),
    ("pipelined", {}, {}, "noise", 64, 8300),
    ("forest", {"force_escape": 1, "no_esc_small": 1, "esc_forest": 1}, {}, "noise", 130, 97),
    ("forest-half-n2", {"force_escape": 2, "no_esc_small": 1, "esc_forest": 1}, {"n_exp": 2.0}, "noise", 100, 80),
    ("forest-ramp", {}, {}, "ramp", 200, 150),
    ("mfd", {}, {}, "noise", 130, 97),
    ("mfd-eager-e13", {"eager": 1}, {}, "noise", 100, 80),
    ("mfd-escape", {"force_escape": 1}, {}, "noise", 130, 97),
    ("mfd-escape-coop", {"force_escape": 2, "no_esc_small": 1}, {}, "noise", 100, 80),
    ("mfd-ramp", {}, {}, "ramp", 200, 150),
    ("mfd-levels", {"mfd_levels": 1}, {}, "noise", 100, 80),
]
only = sys.argv[1:] or None
if only == ["list"]:
    print(" ".join(c[0] for c in CASES) + " tail")
    sys.exit(0)
for name, opts, kw, terrain, w, h in CASES:
    if only and name not in only:
        continue
    if __import__("os").environ.get("SAN_EAGER"):  # racecheck: eager launches (see profiles/sanitizer_r02)
        opts = dict(opts, eager=1)
    ctx = lem.DeviceContext(w, h, lem.SimParams(**kw), 8, options=opts)
    mfd = name.startswith("mfd")
    ex = 1.3 if name.endswith("e13") else 1.0
    if mfd:
        ctx.set_routing(lem.Routing.kMfd, ex)
    e = ora.terrain(w, h, 7) if terrain == "noise" else ramp(w, h, 7)
    ctx.upload(e)
    p = make_params(**kw)
    for s in range(2):
        d = ctx.step(1)[0]
        if mfd:
            o = ora.step_mfd(e, exponent=ex, params=p)
            m = ctx.download_mfd()  # the area of the step and the plan rebuilt for the export
            assert np.array_equal(m["A"].view(np.uint64), o["A"].view(np.uint64)), f"{name}: MFD area differs"
            assert np.array_equal(m["order"], o["mfd_order"]), f"{name}: MFD plan differs"
        else:
            ora.step(e, params=p, want_donor=False)
        ok = np.array_equal(ctx.download().view(np.uint64), e.view(np.uint64))
        assert ok, f"{name}: step {s} differs from the oracle"
    print(f"{name}: ok (nlevels {d.nlevels})", flush=True)
    ctx.close()
if only and "tail" not in only:
    sys.exit(0)
# host step (banded), fill, ensemble with statistics
M, w, h = 3, 96, 70
ctx = lem.DeviceContext(w, h, lem.SimParams(), 8, members=M, options={"host_bands": 5})
host = np.stack([ora.terrain(w, h, s) for s in (1, 2, 3)])
lem._abi.lib().lemgpu_host_register(host.ctypes.data, host.nbytes)
ctx.step_host(host)
lem._abi.lib().lemgpu_host_unregister(host.ctypes.data)
ctx.stats_enable()
ctx.step(2)
ctx.fill(mode=2)
ctx.step(1)
ctx.close()
print("host-banded + stats + fill: ok", flush=True)
