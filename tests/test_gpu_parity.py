"""Parity of the sm_100a path (through the C-ABI) with the pinned CPU oracle.

Bar: rec, dnum, donor slots, order, levels, A bit-exact;
newton_iters and interior_noflow exact; h bit-exact for every n, every cell
area and every drainage area: pow is the device restatement of the host glibc
pow (glibc_pow.cuh), so the stated 1e-9 tolerance for n != 1 is met with 0."""
import json

import numpy as np
import pytest

import paper_1803_02977_b200 as lem
from _oracle import NOFLOW, Oracle, RefLib, fnv1a64, make_params

pytestmark = pytest.mark.gpu

ARRAYS = ("rec", "dnum", "donor", "order", "levels", "A")


def sim_params(**kw):
    return lem.SimParams(**kw)


def device_ctx(w, h, conn=8, options=None, **kw):
    return lem.DeviceContext(w, h, sim_params(**kw), conn, options=options)


def compare_step(ctx, oracle_out, h_gpu, h_orc, exact_h=True, tag=""):
    g = ctx.download_graph(donor=True)
    for k in ARRAYS:
        assert np.array_equal(g[k], oracle_out[k]), f"{tag}: {k} differs"
    assert g["nlevels"] == oracle_out["nlevels"], tag
    if exact_h:
        bad = np.nonzero(h_gpu.view(np.uint64).ravel() != h_orc.view(np.uint64).ravel())[0]
        assert bad.size == 0, f"{tag}: h differs at {bad[:5]} gpu={h_gpu.ravel()[bad[:3]]} cpu={h_orc.ravel()[bad[:3]]}"
    else:
        rel = np.abs(h_gpu - h_orc) / np.maximum(np.abs(h_orc), 1e-300)
        assert rel.max() <= 1e-9, f"{tag}: max rel {rel.max()}"


@pytest.mark.parametrize("path", sorted((__import__("pathlib").Path(__file__).parent / "golden").glob("small_*.npz")),
                         ids=lambda p: p.stem)
def test_small_golden(path):
    g = np.load(path)
    kw = json.loads(str(g["params"]))
    w, h, conn = int(g["w"]), int(g["h"]), int(g["conn"])
    ctx = device_ctx(w, h, conn, **kw)
    ctx.upload(g["h0"])
    d = ctx.step(1)[0]
    out = ctx.download()
    gr = ctx.download_graph(donor=True)
    for k in ARRAYS:
        assert np.array_equal(gr[k], g[k]), k
    assert np.array_equal(out.view(np.uint64), g["h1"].view(np.uint64))
    assert d.newton_iters == int(g["newton_iters"])
    assert d.interior_noflow == int(g["interior_noflow"])
    assert d.lut_misses == 0 or "m_exp" in kw or "dx" in kw


@pytest.mark.parametrize("w,h,seed,conn,kw", [
    (64, 64, 1, 8, {}),
    (100, 77, 2, 8, {}),
    (3, 3, 3, 8, {}),
    (5, 200, 4, 8, {}),
    (257, 129, 5, 8, {}),
    (131, 70, 6, 4, {}),
    (90, 61, 7, 8, {"dx": 0.5, "dy": 2.0}),
    (120, 80, 8, 8, {"m_exp": 0.35, "K": 5e-6}),
    (80, 80, 9, 8, {"K": 0.0}),
    (1024, 33, 10, 8, {}),
])
def test_multistep_vs_oracle(oracle, w, h, seed, conn, kw):
    p = make_params(**kw)
    ctx = device_ctx(w, h, conn, **kw)
    e = oracle.terrain(w, h, seed)
    ctx.upload(e)
    for s in range(8):
        d = ctx.step(1)[0]
        o = oracle.step(e, conn=conn, params=p)
        hg = ctx.download()
        compare_step(ctx, o, hg, e, tag=f"{w}x{h} step {s}")
        assert d.newton_iters == o["newton_iters"]
        assert d.interior_noflow == o["interior_noflow"]
        assert d.nlevels == o["nlevels"]


def test_terrain_generation_bit_exact(oracle):
    for (w, h, seed) in [(1000, 1000, 42), (37, 11, 7), (5, 5, 0)]:
        assert np.array_equal(lem.generate_terrain(w, h, seed), oracle.terrain(w, h, seed))


def test_anchor_1000(golden_dir):
    a = json.loads((golden_dir / "anchors.json").read_text())["1000"]
    ctx = device_ctx(1000, 1000)
    ctx.generate_terrain([42])
    assert fnv1a64(ctx.download()) == a["terrain"]
    d1 = ctx.step(1)[0]
    g = ctx.download_graph()
    st = a["step1"]
    assert fnv1a64(g["rec"]) == st["rec"]
    assert fnv1a64(g["dnum"]) == st["dnum"]
    assert fnv1a64(g["order"]) == st["order"]
    assert fnv1a64(g["A"]) == st["A"]
    assert g["levels"].tolist() == st["levels"]
    assert fnv1a64(ctx.download()) == st["h"]
    assert d1.newton_iters == st["newton_iters"] and d1.interior_noflow == st["interior_noflow"]
    ds = ctx.step(119)
    s120 = a["step120"]
    assert fnv1a64(ctx.download()) == s120["h"]
    assert d1.newton_iters + sum(d.newton_iters for d in ds) == s120["newton_total"]
    assert all(d.lut_misses == 0 for d in ds)


def test_anchor_10000(golden_dir):
    anchors = json.loads((golden_dir / "anchors.json").read_text())
    if "10000" not in anchors:
        pytest.skip("10000^2 anchors not generated")
    a = anchors["10000"]
    ctx = device_ctx(10000, 10000)
    ctx.generate_terrain([42])
    assert fnv1a64(ctx.download()) == a["terrain"]
    d1 = ctx.step(1)[0]
    g = ctx.download_graph()
    st = a["step1"]
    for k in ("rec", "dnum", "order", "A"):
        assert fnv1a64(g[k]) == st[k], k
    assert g["levels"].tolist() == st["levels"]
    assert fnv1a64(ctx.download()) == st["h"]
    assert d1.newton_iters == st["newton_iters"] and d1.interior_noflow == st["interior_noflow"]
    if "step120" in a:
        ds = ctx.step(119)
        assert fnv1a64(ctx.download()) == a["step120"]["h"]
        assert d1.newton_iters + sum(d.newton_iters for d in ds) == a["step120"]["newton_total"]


def test_10000_properties():
    """Size-independent checks at the headline size."""
    n = 10000
    ctx = device_ctx(n, n)
    ctx.generate_terrain([7])
    h0 = ctx.download()
    ctx.step(1)
    h1 = ctx.download()
    g = ctx.download_graph()
    N = n * n
    rec, order, levels, A = g["rec"], g["order"], g["levels"], g["A"]
    # order is a permutation of all cells
    seen = np.zeros(N, np.uint8)
    seen[order] = 1
    assert seen.all()
    # level-0 is exactly the NoFlow cells, ascending (traversal.cpp:27-29)
    l0 = order[: levels[1]]
    assert np.array_equal(l0, np.nonzero(rec == NOFLOW)[0].astype(np.uint32))
    # every cell sits one level below its receiver
    lvl = np.empty(N, np.int32)
    for l in range(g["nlevels"]):
        lvl[order[levels[l]:levels[l + 1]]] = l
    has = rec != NOFLOW
    assert (lvl[has] == lvl[rec[has]] + 1).all()
    # exact mass conservation (acceptance.cpp:113-129)
    assert A[~has].sum() == float(N)
    # perimeter fixed, interior never below its receiver
    hh0, hh1 = h0.reshape(n, n), h1.reshape(n, n)
    assert np.array_equal(hh0[0], hh1[0]) and np.array_equal(hh0[:, 0], hh1[:, 0])
    flat = h1.ravel()
    assert (flat[has] >= flat[rec[has]]).all()


def test_10000_step_vs_reference_cpu():
    """One full 10000^2 step against the unmodified reference on this host."""
    if not RefLib.available():
        pytest.skip("oracle/_ref/liblemref.so not present")
    ref = RefLib.get()
    n = 10000
    e = ref.terrain(n, n, 42)
    ctx = device_ctx(n, n)
    ctx.upload(e)
    d = ctx.step(1)[0]
    hg = ctx.download()
    rc, newton, _ = ref.run(e, 1, strategy="rb_private_queues", workers=ref.max_threads())
    assert rc == 0
    assert np.array_equal(hg.view(np.uint64), e.view(np.uint64))
    assert d.newton_iters == newton


def test_ensemble_members_match_independent_runs(oracle):
    w, h, M = 67, 45, 5
    members = [(1e-6 * (1 + i % 8), 0.35 + 0.05 * i) for i in range(M)]
    seeds = [1000 + i for i in range(M)]
    ctx = lem.DeviceContext(w, h, lem.SimParams(), 8, members=M, per_member=members)
    ctx.generate_terrain(seeds)
    refs = [oracle.terrain(w, h, s) for s in seeds]
    for step in range(6):
        ds = ctx.step(1)
        tot = 0
        for i in range(M):
            o = oracle.step(refs[i], params=make_params(K=members[i][0], m_exp=members[i][1]))
            tot += o["newton_iters"]
        hg = ctx.download()
        for i in range(M):
            assert np.array_equal(hg[i].view(np.uint64), refs[i].view(np.uint64)), (step, i)
        assert ds[0].newton_iters == tot


def test_member_stats():
    import torch

    w, h, M = 200, 150, 3
    ctx = lem.DeviceContext(w, h, lem.SimParams(), 8, members=M)
    ctx.generate_terrain([1, 2, 3])
    ctx.step(3)
    out = torch.empty(4 * M, dtype=torch.float64, device="cuda")
    ctx.member_stats_device(out.data_ptr())
    torch.cuda.synchronize()
    hh = ctx.download().reshape(M, -1)
    s = out.cpu().numpy().reshape(M, 4)
    assert np.allclose(s[:, 0], hh.mean(1), rtol=1e-12)
    assert (s[:, 1] == hh.max(1)).all() and (s[:, 2] == hh.min(1)).all()


def test_n2_bit_exact_120_steps(oracle):
    """n = 2 (Newton with pow(diff, 2)): bit-identical to the oracle at every
    one of 120 steps -- the drift after 120 steps is 0 (north_star asks for it
    to be reported; tools/drift_n2.py reports it at configs[2]'s 4000^2)."""
    w = h = 200
    p = make_params(n_exp=2.0)
    ctx = device_ctx(w, h, n_exp=2.0)
    e = oracle.terrain(w, h, 42)
    ctx.upload(e)
    d = ctx.step(1)[0]
    o = oracle.step(e, params=p)
    hg = ctx.download()
    compare_step(ctx, o, hg, e, tag="n=2 step 1")
    assert d.newton_iters == o["newton_iters"]
    ds = ctx.step(119)
    rc, newton, _ = oracle.run(e, 119, params=p)
    assert np.array_equal(ctx.download().view(np.uint64), e.view(np.uint64))
    assert sum(x.newton_iters for x in ds) == newton


def test_device_pow_matches_host_libm():
    """The device restatement of glibc pow == the host libm's ::pow bit for bit
    on 6e5 inputs (drainage areas^m, Newton differences^2 and ^(n-1), random
    bit patterns), in the variant the context detected.  y = 2 goes through
    the n = 2 Newton fast path (glibc_pow_sq_dev): 2e5 more x over 2^-80 ..
    2^80, ~3 % of them 1/64 .. 1/32 ulp from a rounding midpoint of x^2."""
    import ctypes

    L = lem._abi.lib()
    variant = L.lemgpu_pow_variant(None)
    assert variant in (0, 1), "neither glibc pow restatement matches this host's libm"
    libm = ctypes.CDLL("libm.so.6")
    libm.pow.restype = ctypes.c_double
    libm.pow.argtypes = [ctypes.c_double, ctypes.c_double]
    rng = np.random.default_rng(5)
    n = 100000
    xs = [rng.integers(1, 70_000_000, n).astype(np.float64),
          np.ldexp(0.5 + rng.random(n), -rng.integers(0, 60, n)),
          np.ldexp(0.5 + rng.random(n), -rng.integers(0, 80, n)),
          rng.integers(0, 2**63, n, dtype=np.int64).view(np.float64),
          np.ldexp(0.5 + rng.random(2 * n), rng.integers(-80, 80, 2 * n))]
    ys = [0.25 + 0.6 * rng.random(n), np.full(n, 2.0), -0.9 + 2.8 * rng.random(n),
          rng.integers(0, 2**63, n, dtype=np.int64).view(np.float64), np.full(2 * n, 2.0)]
    x = np.ascontiguousarray(np.concatenate(xs))
    y = np.ascontiguousarray(np.concatenate(ys))
    got = np.empty_like(x)
    assert L.lemgpu_debug_pow(0, variant, x.ctypes.data, y.ctypes.data, got.ctypes.data, x.size) == 0
    want = np.array([libm.pow(a, b) for a, b in zip(x.tolist(), y.tolist())])
    same = (got.view(np.uint64) == want.view(np.uint64)) | (np.isnan(got) & np.isnan(want))
    bad = np.nonzero(~same)[0]
    assert bad.size == 0, f"{bad.size} mismatches, e.g. pow({x[bad[0]]!r}, {y[bad[0]]!r})"


def test_convergence_error_surfaces_cell():
    ctx = device_ctx(40, 40, max_newton_iters=1)
    ctx.generate_terrain([5])
    with pytest.raises(lem.ConvergenceError) as ei:
        ctx.step(1)
    c = ei.value.cell()
    assert 0 < c < 1600 and "did not converge" in str(ei.value)
    # the context stays usable after the error is reported
    ctx2 = device_ctx(40, 40)
    ctx2.generate_terrain([5])
    ctx2.step(2)


def test_nonfinite_input_rejected():
    ctx = device_ctx(16, 16)
    e = np.zeros((16, 16))
    e[3, 4] = np.nan
    with pytest.raises(lem.ConfigError, match="non-finite value at cell 52"):
        ctx.upload(e)


def test_strategy_step_and_run_simulation_dropin(oracle):
    w, h = 48, 40
    e = oracle.terrain(w, h, 11)
    g = lem.GridGraph(w, h)
    ws = lem.SimWorkspace()
    mine = e.copy()
    for _ in range(4):
        d = lem.strategy_step(mine, g, lem.SimParams(), lem.StepSetup(), lem.Strategy(), ws)
        o = oracle.step(e)
        assert np.array_equal(mine.view(np.uint64), e.view(np.uint64))
        assert d.newton_iters == o["newton_iters"]
    cfg = lem.RunConfig(width=w, height=h, seed=11, timesteps=10)
    res = lem.run_simulation(cfg)
    e2 = oracle.terrain(w, h, 11)
    rc, newton, _ = oracle.run(e2, 10)
    assert np.array_equal(res.elevation.view(np.uint64), e2.view(np.uint64))
    assert res.newton_iters == newton
    seen = []
    lem.run_simulation(oracle.terrain(w, h, 11), cfg, on_step=lambda s, r, d: seen.append((s, float(r.sum()))))
    assert [s for s, _ in seen] == list(range(1, 11))


def test_cpp_dropin_through_reference_api():
    """The reference's own C++ API (run_simulation / strategy_step / SimWorkspace)
    driving the rb_gpu shim, byte-compared with the reference strategies."""
    import subprocess
    from pathlib import Path

    exe = Path(__file__).resolve().parents[1] / "oracle" / "_ref" / "test_dropin"
    if not exe.exists():
        pytest.skip("oracle/_ref/test_dropin not built (needs /root/reference at build time)")
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "0 failure(s)" in out.stdout


@pytest.mark.parametrize("w,h,seed,kw", [(300, 200, 21, {}), (64, 64, 22, {"n_exp": 2.0}), (90, 61, 23, {"dx": 0.5})])
def test_per_level_sweeps_match_chunked(oracle, monkeypatch, w, h, seed, kw):
    """The deep-plan schedule (one kernel per level, global scratch) forced on a
    shallow plan gives the same bits as the chunked schedule and the oracle."""
    deep = device_ctx(w, h, options={"force_deep": 1}, **kw)
    chunked = device_ctx(w, h, **kw)
    e = oracle.terrain(w, h, seed)
    deep.upload(e)
    chunked.upload(e)
    p = make_params(**kw)
    for _ in range(5):
        dd = deep.step(1)[0]
        dc = chunked.step(1)[0]
        o = oracle.step(e, params=p)
        hd, hc = deep.download(), chunked.download()
        assert np.array_equal(hd.view(np.uint64), hc.view(np.uint64))
        assert dd.newton_iters == dc.newton_iters
        compare_step(deep, o, hd, e, tag="deep")


def _ramp(w, h, seed):
    """Tilted plane + noise: long drainage chains (deep plans, trees that leave any tile)."""
    rng = np.random.default_rng(seed)
    x = np.arange(w)[None, :].astype(np.float64)
    y = np.arange(h)[:, None].astype(np.float64)
    return 0.05 * x + 0.01 * y + 1e-3 * rng.random((h, w))


@pytest.mark.parametrize("env", [{}, {"LEMGPU_FORCE_ESCAPE": "1"}, {"LEMGPU_FORCE_ESCAPE": "2"},
                                 {"LEMGPU_PATH": "global"}, {"LEMGPU_FORCE_ESCAPE": "1", "LEMGPU_FORCE_DEEP": "1"},
                                 {"LEMGPU_FORCE_ESCAPE": "1", "LEMGPU_ESC_SMALL": "0", "LEMGPU_ESC_FOREST": "-1"},
                                 {"LEMGPU_FORCE_ESCAPE": "1", "LEMGPU_ESC_SMALL": "0", "LEMGPU_ESC_FOREST": "1"},
                                 {"LEMGPU_FORCE_ESCAPE": "2", "LEMGPU_ESC_SMALL": "0", "LEMGPU_ESC_FOREST": "1"}],
                         ids=["tiles", "all-escape", "half-escape", "global", "all-escape-deep", "all-escape-coop",
                              "all-escape-forest", "half-escape-forest"])
@pytest.mark.parametrize("w,h,seed,kw,terrain", [
    (300, 200, 31, {}, "noise"), (130, 97, 32, {"n_exp": 2.0}, "noise"), (77, 65, 33, {"dx": 0.5}, "noise"),
    (129, 70, 34, {}, "ramp"), (90, 61, 35, {}, "ramp"), (400, 12, 36, {}, "ramp"), (61, 40, 37, {"n_exp": 2.0}, "ramp"),
])
def test_schedules_agree_with_oracle(oracle, monkeypatch, env, w, h, seed, kw, terrain):
    """Every schedule -- trees finished inside their tile (k_tiles), trees that
    escape to the global level path (all of them, or every odd-rooted one; in
    k_esc_small's shared memory when they fit, <= 6144 cells and <= 256 levels,
    else -- or with LEMGPU_ESC_SMALL=0 -- in the cooperative level-path
    kernels or k_esc_forest's pointer-jumped, per-tree sweeps), the global path
    alone, and its per-level sweeps -- gives the oracle's bits."""
    ctx = device_ctx(w, h, options=env, **kw)
    e = oracle.terrain(w, h, seed) if terrain == "noise" else _ramp(w, h, seed)
    ctx.upload(e)
    p = make_params(**kw)
    for s in range(4):
        d = ctx.step(1)[0]
        o = oracle.step(e, params=p)
        hg = ctx.download()
        compare_step(ctx, o, hg, e, tag=f"{env} step {s}")
        assert d.newton_iters == o["newton_iters"]
        assert d.interior_noflow == o["interior_noflow"]
        assert d.nlevels == o["nlevels"]


def test_failed_step_leaves_elevation_unchanged(oracle):
    """A step that raises (ConvergenceError) leaves the device elevation as it
    was before that step (steps read one ping-pong buffer and write the other)."""
    ctx = device_ctx(64, 48, max_newton_iters=1)
    e = oracle.terrain(64, 48, 3)
    ctx.upload(e)
    with pytest.raises(lem.ConvergenceError):
        ctx.step(3)
    assert np.array_equal(ctx.download().view(np.uint64), e.view(np.uint64))


@pytest.mark.parametrize("opts", [{"esc_forest": -1}, {"esc_forest": -1, "no_narrow": 1}, None],
                         ids=["narrow-runs", "grid-only", "forest"])
def test_deep_plan_1000(oracle, monkeypatch, opts):
    """A 1000^2 tilted plane: ~1000 levels, every tree escapes its tile.  The
    escape path's level kernels (cooperative level expansion and deep sweeps:
    runs of narrow levels on one CTA, or every level grid-wide) and, by
    default, k_esc_forest (levels by pointer jumping, trees split between
    CTAs) give the oracle's bits; the export still rebuilds the reference's
    own TraversalPlan."""
    e = _ramp(1000, 1000, 5)
    ctx = device_ctx(1000, 1000, options=opts)
    ctx.upload(e)
    for s in range(2):
        d = ctx.step(1)[0]
        o = oracle.step(e, want_donor=False)
        assert d.nlevels == o["nlevels"] > 900
        assert d.newton_iters == o["newton_iters"]
        assert np.array_equal(ctx.download().view(np.uint64), e.view(np.uint64)), f"step {s}"
    g = ctx.download_graph()
    assert np.array_equal(g["order"], o["order"]) and np.array_equal(g["levels"], o["levels"])


@pytest.mark.parametrize("env", [{}, {"LEMGPU_FORCE_ESCAPE": "2"}, {"LEMGPU_PATH": "global"}], ids=["tiles", "half-escape", "global"])
def test_inexact_cell_area(oracle, monkeypatch, env):
    """dx*dy with a full significand: the drainage area is the reference's FP
    sum in slot order (bit-exact) and pow(A, m) is evaluated on the device by
    the glibc restatement (lut misses) -- elevations bit-exact."""
    kw = {"dx": 0.1, "dy": 0.3}
    ctx = device_ctx(100, 80, options=env, **kw)
    e = oracle.terrain(100, 80, 17)
    ctx.upload(e)
    p = make_params(**kw)
    for s in range(3):
        d = ctx.step(1)[0]
        o = oracle.step(e, params=p)
        hg = ctx.download()
        compare_step(ctx, o, hg, e, tag=f"{env} step {s}")
        assert d.lut_misses > 0 and d.newton_iters == o["newton_iters"]


def _host_register(a):
    return lem._abi.lib().lemgpu_host_register(a.ctypes.data, a.nbytes) == 0


@pytest.mark.parametrize("env", [{}, {"LEMGPU_FORCE_ESCAPE": "2"},
                                 {"LEMGPU_FORCE_ESCAPE": "1", "LEMGPU_ESC_SMALL": "0", "LEMGPU_ESC_FOREST": "-1"},
                                 {"LEMGPU_FORCE_ESCAPE": "1", "LEMGPU_ESC_SMALL": "0"},
                                 {"LEMGPU_FORCE_ESCAPE": "2", "LEMGPU_PATCH_CAP": "64"}],
                         ids=["tiles", "half-escape", "all-escape-coop", "all-escape-forest", "patch-overflow"])
@pytest.mark.parametrize("w,h,terrain", [(300, 250, "noise"), (200, 170, "ramp"), (131, 97, "noise")])
def test_step_host_banded(oracle, monkeypatch, env, w, h, terrain):
    """lemgpu_step_host (the strategy_step drop-in) on pinned host memory: the
    raster goes up and comes down band by band, overlapped with the compute,
    and the escaped trees' cells are patched in afterwards (or, past the patch
    capacity, the whole raster comes down again) -- the oracle's bits."""
    ctx = device_ctx(w, h, options={"LEMGPU_HOST_BANDS": 4, **env})
    e = oracle.terrain(w, h, 41) if terrain == "noise" else _ramp(w, h, 41)
    host = e.copy()
    assert _host_register(host)
    try:
        for s in range(3):
            d = ctx.step_host(host)
            o = oracle.step(e, want_donor=False)
            bad = np.nonzero(host.view(np.uint64) != e.view(np.uint64))
            assert bad[0].size == 0, f"step {s}: {bad[0].size} cells differ, first {list(zip(*bad))[:3]}"
            assert d.nlevels == o["nlevels"] and d.newton_iters == o["newton_iters"]
    finally:
        lem._abi.lib().lemgpu_host_unregister(host.ctypes.data)


def test_step_host_pageable_and_failure(oracle):
    """Pageable host memory takes the plain copy-step-copy path (same bits); a
    failing banded step leaves the pinned host raster as it was."""
    e = oracle.terrain(150, 120, 43)
    ctx = device_ctx(150, 120)
    host = e.copy()
    ctx.step_host(host)
    oracle.step(e, want_donor=False)
    assert np.array_equal(host.view(np.uint64), e.view(np.uint64))
    bad_ctx = device_ctx(150, 120, max_newton_iters=1)
    pinned = e.copy()
    assert _host_register(pinned)
    try:
        with pytest.raises(lem.ConvergenceError):
            bad_ctx.step_host(pinned)
        assert np.array_equal(pinned.view(np.uint64), e.view(np.uint64))
    finally:
        lem._abi.lib().lemgpu_host_unregister(pinned.ctypes.data)


@pytest.mark.parametrize("mode", [1, 2], ids=["exact", "epsilon"])
def test_fill_matches_oracle(oracle, golden_dir, mode):
    """lemgpu_fill (tile relaxation to the flood's fixed point) is bit-identical
    to lem::priority_flood_fill: the reference fixtures, the 20 seeds of
    acceptance.cpp:228-249, odd and stacked (ensemble) rasters, 1000^2."""
    for path in sorted(golden_dir.glob("fill_*.npz")):
        g = np.load(path)
        if int(g["mode"]) != mode:
            continue
        f = lem.priority_flood_fill(g["h0"], lem.FillOptions(lem.FillMode(mode), float(g["eps"])))
        assert np.array_equal(f.view(np.uint64), g["f"].view(np.uint64)), path.name
    for seed in range(1, 21):
        e = oracle.terrain(100, 100, seed)
        f = lem.priority_flood_fill(e, lem.FillOptions(lem.FillMode(mode)))
        assert np.array_equal(f.view(np.uint64), oracle.fill(e, mode).view(np.uint64)), seed
    for w, h, seed in [(1000, 1000, 42), (131, 517, 5), (65, 33, 6)]:
        e = oracle.terrain(w, h, seed)
        f = lem.priority_flood_fill(e, lem.FillOptions(lem.FillMode(mode)))
        assert np.array_equal(f.view(np.uint64), oracle.fill(e, mode).view(np.uint64)), (w, h)
    # ensemble: every member filled on its own
    M, w, h = 3, 90, 70
    ctx = lem.DeviceContext(w, h, sim_params(), 8, members=M)
    ctx.generate_terrain([11, 12, 13])
    ctx.fill(mode=mode)
    out = ctx.download()
    for m, seed in enumerate([11, 12, 13]):
        want = oracle.fill(oracle.terrain(w, h, seed), mode)
        assert np.array_equal(out[m].view(np.uint64), want.view(np.uint64)), m


def test_filled_terrain_drains_and_steps(oracle):
    """After the epsilon fill no interior cell is a pit (acceptance.cpp:235-242),
    and the deep plan that follows steps bit-identically to the oracle."""
    cfg = lem.RunConfig(width=200, height=150, seed=3, timesteps=0,
                        fill=lem.FillOptions(lem.FillMode.kEpsilonAscending))
    filled = lem.run_simulation(cfg).elevation
    want = oracle.fill(oracle.terrain(200, 150, 3), 2)
    assert np.array_equal(filled.view(np.uint64), want.view(np.uint64))
    ctx = device_ctx(200, 150)
    ctx.upload(filled)
    e = filled.copy()
    for s in range(3):
        d = ctx.step(1)[0]
        o = oracle.step(e, want_donor=False)
        if s == 0:
            assert d.interior_noflow == 0 and o["interior_noflow"] == 0
        assert d.nlevels == o["nlevels"] and d.newton_iters == o["newton_iters"]
        assert np.array_equal(ctx.download().view(np.uint64), e.view(np.uint64)), s
    with pytest.raises(lem.ConfigError):
        ctx.fill(mode=2, epsilon=0.0)


def test_step_host_banded_ensemble(oracle, monkeypatch):
    """The banded host step on a stacked ensemble (bands cut across member
    boundaries): every member equals its own oracle run."""
    M, w, h = 3, 96, 70
    ctx = lem.DeviceContext(w, h, lem.SimParams(), 8, members=M, options={"host_bands": 5})
    seeds = [21, 22, 23]
    host = np.stack([oracle.terrain(w, h, s) for s in seeds])
    want = [host[m].copy() for m in range(M)]
    assert _host_register(host)
    try:
        for s in range(3):
            ctx.step_host(host)
            for m in range(M):
                oracle.step(want[m], want_donor=False)
                assert np.array_equal(host[m].view(np.uint64), want[m].view(np.uint64)), (s, m)
    finally:
        lem._abi.lib().lemgpu_host_unregister(host.ctypes.data)


@pytest.mark.parametrize("seed", range(4))
def test_random_configurations(oracle, monkeypatch, seed):
    """Randomised shapes (3..260 x 3..200, odd and even widths), D4/D8, n = 1/2,
    spacings, ensembles of 1-3 members and schedule knobs: every step of every
    member against the oracle, bit-exact."""
    rng = np.random.default_rng(1000 + seed)
    for case in range(10):
        w, h = int(rng.integers(3, 261)), int(rng.integers(3, 201))
        conn = int(rng.choice([4, 8]))
        n_exp = float(rng.choice([1.0, 1.0, 2.0]))
        dx = float(rng.choice([1.0, 1.0, 0.5, 2.0]))
        M = int(rng.integers(1, 4))
        env = [{}, {"LEMGPU_FORCE_ESCAPE": "2"}, {"LEMGPU_FORCE_ESCAPE": "1"}, {"LEMGPU_TILE_GRID": "3"},
               {"LEMGPU_NO_TMA": "1"}, {"LEMGPU_ESC_SMALL": "0", "LEMGPU_FORCE_ESCAPE": "1", "LEMGPU_ESC_FOREST": "-1"},
               {"LEMGPU_ESC_SMALL": "0", "LEMGPU_FORCE_ESCAPE": "2", "LEMGPU_ESC_FOREST": "1"}][int(rng.integers(0, 7))]
        kw = {"n_exp": n_exp, "dx": dx}
        ctx = lem.DeviceContext(w, h, sim_params(**kw), conn, members=M, options=env)
        seeds = [int(x) for x in rng.integers(1, 10**6, size=M)]
        ctx.generate_terrain(seeds)
        es = [oracle.terrain(w, h, s) for s in seeds]
        p = make_params(**kw)
        tag = f"case {case}: {w}x{h} conn={conn} n={n_exp} dx={dx} M={M} env={env}"
        for s in range(2):
            ctx.step(1)
            g = ctx.download().reshape(M, h, w)
            for m in range(M):
                oracle.step(es[m], conn=conn, params=p, want_donor=False)
                assert np.array_equal(g[m].view(np.uint64), es[m].view(np.uint64)), f"{tag} step {s} member {m}"
        ctx.close()


def test_pipelined_graph_tall_rasters(oracle):
    """Rasters of >= 256 tile rows take the pipelined graph (receiver bands
    chained, k_tiles of band b after the receivers of band b+1): a tall single
    raster and a stacked ensemble, every member bit-exact against the oracle."""
    w, h = 150, 8300  # 260 tile rows
    ctx = device_ctx(w, h)
    assert ctx.pipeline_bands() > 1 and ctx.kernels_per_step() > 2 * ctx.pipeline_bands()
    e = oracle.terrain(w, h, 51)
    ctx.upload(e)
    for s in range(2):
        d = ctx.step(1)[0]
        o = oracle.step(e, want_donor=False)
        assert np.array_equal(ctx.download().view(np.uint64), e.view(np.uint64)), s
        assert d.newton_iters == o["newton_iters"] and d.nlevels == o["nlevels"]
    M, w, h = 8, 96, 1100  # 275 stacked tile rows
    ens = lem.DeviceContext(w, h, sim_params(), 8, members=M)
    assert ens.pipeline_bands() > 1
    seeds = list(range(60, 60 + M))
    ens.generate_terrain(seeds)
    want = [oracle.terrain(w, h, sd) for sd in seeds]
    for s in range(2):
        ens.step(1)
        g = ens.download().reshape(M, h, w)
        for m in range(M):
            oracle.step(want[m], want_donor=False)
            assert np.array_equal(g[m].view(np.uint64), want[m].view(np.uint64)), (s, m)


@pytest.mark.parametrize("w,h,seed,kw,terrain", [
    (300, 200, 71, {}, "noise"), (257, 131, 72, {"dx": 0.5, "dy": 0.25}, "noise"), (130, 97, 73, {"n_exp": 2.0}, "noise"),
    (129, 70, 74, {}, "ramp"), (1000, 1000, 42, {}, "noise"),
])
def test_tile_pass_levels_and_area_direct(oracle, w, h, seed, kw, terrain):
    """The tile pass's own level lists and drainage areas (captured inside
    k_tiles from shared memory, not rebuilt by the export path) equal the
    reference's TraversalPlan levels and accumulation for every cell it
    finishes; the cells it leaves are exactly those of the escaped trees."""
    ctx = device_ctx(w, h, **kw)
    ctx.tile_capture(True)
    e = oracle.terrain(w, h, seed) if terrain == "noise" else _ramp(w, h, seed)
    ctx.upload(e)
    p = make_params(**kw)
    for s in range(2):
        d = ctx.step(1)[0]
        o = oracle.step(e, params=p, want_donor=False)
        lv, A = ctx.tile_levels()
        olv = np.empty(w * h, np.int32)
        for L in range(o["nlevels"]):
            olv[o["order"][o["levels"][L]:o["levels"][L + 1]]] = L
        done = lv != 0xFF
        assert done.sum() == w * h - d.escaped_cells, (done.sum(), d.escaped_cells)
        assert np.array_equal(lv[done].astype(np.int32), olv[done]), f"step {s}: tile levels differ"
        assert np.array_equal(A[done].view(np.uint64), o["A"][done].view(np.uint64)), f"step {s}: tile areas differ"
        if s == 0 and terrain == "noise":
            assert done.mean() > 0.9  # random noise: nearly every tree stays inside its tile
    ctx.tile_capture(False)


def _np_stats(hh):
    flat = hh.reshape(hh.shape[0], -1)
    return np.stack([flat.mean(1), flat.max(1), flat.min(1), flat.sum(1)], axis=1)


@pytest.mark.parametrize("w,h,M,interval", [(67, 45, 5, 1), (90, 20, 4, 1), (96, 1100, 8, 1), (64, 40, 3, 3)],
                         ids=["small", "short-members", "tall-pipelined", "every-3rd-step"])
def test_ensemble_stats_in_step_graph(oracle, w, h, M, interval):
    """lemgpu_stats_enable: every interval-th step's graph computes the {mean,
    max, min, sum} of each member's elevation as the step starts --
    deterministic, equal to numpy's statistics of that state; rows of other
    ranks stay 0."""
    members = [(1e-6 * (1 + i % 8), 0.35 + 0.05 * (i % 8)) for i in range(M)]

    def run():
        ctx = lem.DeviceContext(w, h, lem.SimParams(), 8, members=M, per_member=members)
        ctx.stats_enable(member_offset=2, members_total=M + 3, interval=interval)
        ctx.generate_terrain(range(500, 500 + M))
        out = []
        last = np.zeros((M + 3, 4))
        for s in range(6):
            before = ctx.download().reshape(M, h, w)
            ctx.step(1)
            t = ctx.stats_table()
            if (s + 1) % interval == 0:
                assert (t[:2] == 0).all() and (t[2 + M:] == 0).all()
                want = _np_stats(before)
                got = t[2:2 + M]
                assert np.array_equal(got[:, 1], want[:, 1]) and np.array_equal(got[:, 2], want[:, 2])
                assert np.allclose(got[:, 3], want[:, 3], rtol=1e-13) and np.allclose(got[:, 0], want[:, 0], rtol=1e-13)
            else:
                assert np.array_equal(t, last)  # not recomputed on this step
            last = t.copy()
            out.append(t)
        return out

    a, b = run(), run()
    for x, y in zip(a, b):
        assert np.array_equal(x.view(np.uint64), y.view(np.uint64))  # deterministic


def test_ensemble_shard_with_nccl_allreduce_in_graph(oracle):
    """The product ensemble entry (lemgpu_create_ensemble_shard + an NCCL
    communicator): the step graph ends with one ncclAllReduce of the table,
    captured as a child graph.  One rank here (the box has one GPU); the
    members are bit-exact against their oracle runs and the table is the
    gathered statistics."""
    from paper_1803_02977_b200 import ensemble

    w, h, M = 80, 60, 6
    ens = ensemble.DeviceEnsemble(w, h, M)
    ens.ctx.stats_comm_init(ensemble.nccl_unique_id(), 1, 0)
    ens.generate_terrain()
    refs = [oracle.terrain(w, h, ensemble.member_params(i)[0]) for i in range(M)]
    for s in range(3):
        want = _np_stats(np.stack(refs))
        ens.ctx.step(1)
        for i in range(M):
            _, K, m = ensemble.member_params(i)
            oracle.step(refs[i], params=make_params(K=K, m_exp=m), want_donor=False)
        t = ens.table()
        assert np.array_equal(t[:, 1], want[:, 1]) and np.allclose(t[:, 3], want[:, 3], rtol=1e-13)
        g = ens.ctx.download()
        for i in range(M):
            assert np.array_equal(g[i].view(np.uint64), refs[i].view(np.uint64)), (s, i)
    ens.close()


# ---- MFD routing: StepSetup::routing = kMfd -------------------------------

# MFD schedules: the area by tile passes + the D8 tile path (default), with
# every tree escaping to k_esc_small or to the cooperative escape kernels,
# eagerly launched (the pass loop on the host), and the level-synchronous
# plan + global level path (mfd_levels)
MFD_PATHS = {"tiles": None, "tiles-escape": {"force_escape": 1}, "tiles-escape-coop": {"force_escape": 2, "no_esc_small": 1},
             "tiles-eager": {"eager": 1}, "levels": {"mfd_levels": 1}}


def _mfd_ctx(w, h, ex, conn=8, members=1, options=None, **kw):
    ctx = lem.DeviceContext(w, h, sim_params(**kw), conn, members=members, options=options)
    ctx.set_routing(lem.Routing.kMfd, ex)
    return ctx


@pytest.mark.parametrize("path", sorted(MFD_PATHS))
def test_mfd_golden(oracle, golden_dir, path):
    """Every mfd_*.npz fixture (made by the unmodified reference's simulate_step
    with Routing::kMfd): h after the step, Newton iterations, the MFD drainage
    area and the MFD plan, bit for bit -- on every MFD schedule."""
    opts = MFD_PATHS[path]
    for path in sorted(golden_dir.glob("mfd_*.npz")):
        g = np.load(path)
        kw = json.loads(str(g["params"]))
        ctx = _mfd_ctx(int(g["w"]), int(g["h"]), float(g["exponent"]), int(g["conn"]), options=opts, **kw)
        ctx.upload(g["h0"])
        d = ctx.step(1)[0]
        assert np.array_equal(ctx.download().view(np.uint64), g["h1"].view(np.uint64)), path.name
        assert d.newton_iters == int(g["newton_iters"]), path.name
        m = ctx.download_mfd()
        assert np.array_equal(m["A"].view(np.uint64), g["A"].view(np.uint64)), path.name
        assert np.array_equal(m["order"], g["mfd_order"]) and np.array_equal(m["levels"], g["mfd_levels"]), path.name
        ctx.close()


@pytest.mark.parametrize("w,h,seed,conn,ex,kw,terrain", [
    (300, 200, 51, 8, 1.0, {}, "noise"), (257, 131, 52, 8, 1.3, {"m_exp": 0.4}, "noise"),
    (130, 97, 53, 4, 1.0, {}, "noise"), (77, 65, 54, 8, 2.0, {"dx": 0.5, "dy": 2.0}, "noise"),
    (120, 90, 55, 8, 1.0, {"n_exp": 2.0}, "noise"), (200, 150, 56, 8, 1.0, {}, "ramp"),
    (400, 12, 57, 8, 0.7, {}, "ramp"), (3, 3, 58, 8, 1.0, {}, "noise"),
])
@pytest.mark.parametrize("path", sorted(MFD_PATHS))
def test_mfd_steps_vs_oracle(oracle, w, h, seed, conn, ex, kw, terrain, path):
    """4 MFD steps per shape (odd widths, D4, anisotropic spacing, exponents
    0.7-2, n = 2, deep ramps): h, A and the MFD plan against the oracle each
    step, on every MFD schedule; the tile passes converge (mfd_passes > 0)."""
    ctx = _mfd_ctx(w, h, ex, conn, options=MFD_PATHS[path], **kw)
    e = oracle.terrain(w, h, seed) if terrain == "noise" else _ramp(w, h, seed)
    ctx.upload(e)
    p = make_params(**kw)
    for s in range(4):
        d = ctx.step(1)[0]
        o = oracle.step_mfd(e, exponent=ex, conn=conn, params=p)
        assert o["status"] == 0
        assert np.array_equal(ctx.download().view(np.uint64), e.view(np.uint64)), f"step {s}"
        assert d.newton_iters == o["newton_iters"] and d.interior_noflow == o["interior_noflow"]
        assert d.nlevels == o["nlevels"]  # the D8 plan's levels (the erosion's)
        assert (d.mfd_passes > 0) == (path != "levels")
        m = ctx.download_mfd()
        assert np.array_equal(m["A"].view(np.uint64), o["A"].view(np.uint64)), f"step {s}"
        assert np.array_equal(m["order"], o["mfd_order"]) and np.array_equal(m["levels"], o["mfd_levels"])


@pytest.mark.parametrize("path", ["tiles", "levels"])
def test_mfd_ensemble_members(oracle, path):
    """A stacked ensemble under MFD routing: every member equals its own oracle run."""
    M, w, h = 3, 90, 70
    ctx = _mfd_ctx(w, h, 1.0, members=M, options=MFD_PATHS[path])
    seeds = [61, 62, 63]
    ctx.generate_terrain(seeds)
    es = [oracle.terrain(w, h, sd) for sd in seeds]
    for s in range(3):
        ctx.step(1)
        g = ctx.download().reshape(M, h, w)
        for m in range(M):
            oracle.step_mfd(es[m])
            assert np.array_equal(g[m].view(np.uint64), es[m].view(np.uint64)), (s, m)


def test_mfd_1000_vs_reference():
    """configs[0]'s 1000^2 DEM under MFD routing: one step against the reference's
    simulate_step (A and the MFD plan too), then 5 more against its rb_par_all."""
    from _oracle import RefLib

    if not RefLib.available():
        pytest.skip("oracle/_ref/liblemref.so not present")
    ref = RefLib.get()
    n = 1000
    e = ref.terrain(n, n, 42)
    ctx = _mfd_ctx(n, n, 1.0)
    ctx.upload(e)
    d = ctx.step(1)[0]
    r = ref.step_mfd(e)
    assert r["status"] == 0
    assert np.array_equal(ctx.download().view(np.uint64), e.view(np.uint64))
    assert d.newton_iters == r["newton_iters"]
    m = ctx.download_mfd()
    assert np.array_equal(m["A"].view(np.uint64), r["A"].view(np.uint64))
    assert np.array_equal(m["order"], r["mfd_order"]) and np.array_equal(m["levels"], r["mfd_levels"])
    ds = ctx.step(5)
    rc, newton, _ = ref.run(e, 5, strategy="rb_par_all", workers=ref.max_threads(), routing=1)
    assert rc == 0
    assert np.array_equal(ctx.download().view(np.uint64), e.view(np.uint64))
    assert sum(x.newton_iters for x in ds) == newton


def test_mfd_routing_switch_and_dropin(oracle):
    """strategy_step with StepSetup(routing=kMfd) through the Python drop-in,
    then back to D8 on the same workspace: both against the oracle."""
    w, h = 96, 80
    e = oracle.terrain(w, h, 7)
    ref_e = e.copy()
    g = lem.GridGraph(w, h)
    ws = lem.SimWorkspace()
    for routing in (lem.Routing.kMfd, lem.Routing.kD8, lem.Routing.kMfd):
        lem.strategy_step(e, g, lem.SimParams(), lem.StepSetup(routing=routing), lem.Strategy(), ws)
        if routing == lem.Routing.kMfd:
            oracle.step_mfd(ref_e)
        else:
            oracle.step(ref_e, want_donor=False)
        assert np.array_equal(e.view(np.uint64), ref_e.view(np.uint64)), routing


@pytest.mark.parametrize("mode", [1, 2], ids=["exact", "epsilon"])
def test_mfd_filled_dem_vs_oracle(oracle, mode):
    """MFD routing on a Priority-Flood-filled DEM (flats / epsilon ramps: long
    descending chains that cross many tile edges, many tile passes): h, A and
    the MFD plan against the oracle for 3 steps."""
    w, h = 160, 120
    e = oracle.fill(oracle.terrain(w, h, 71), mode)
    ctx = _mfd_ctx(w, h, 1.0)
    ctx.upload(e)
    for s in range(3):
        d = ctx.step(1)[0]
        o = oracle.step_mfd(e)
        assert o["status"] == 0
        assert np.array_equal(ctx.download().view(np.uint64), e.view(np.uint64)), s
        assert d.newton_iters == o["newton_iters"]
        m = ctx.download_mfd()
        assert np.array_equal(m["A"].view(np.uint64), o["A"].view(np.uint64)), s
        assert np.array_equal(m["order"], o["mfd_order"]) and np.array_equal(m["levels"], o["mfd_levels"])
    assert d.mfd_passes >= 2


@pytest.mark.parametrize("clocks", [0, 1], ids=["off", "on"])
def test_phase_clock_option(oracle, clocks):
    """lemgpu_options::phase_clocks: on, lemgpu_diag.seconds holds lem::Phase
    seconds that add up to the step's device time (every phase of a tile-path
    step charged); off (the production default), they are 0 -- and the
    elevations are the oracle's either way."""
    w, h = 300, 200
    ctx = device_ctx(w, h, options={"phase_clocks": clocks})
    e = oracle.terrain(w, h, 81)
    ctx.upload(e)
    for _ in range(2):
        d = ctx.step(1)[0]
        oracle.step(e, want_donor=False)
    assert np.array_equal(ctx.download().view(np.uint64), e.view(np.uint64))
    if clocks:
        assert all(x >= 0.0 for x in d.seconds) and sum(d.seconds) > 0.0
        assert d.seconds[0] > 0.0 and d.seconds[2] > 0.0 and d.seconds[5] > 0.0  # receivers, order, erosion
    else:
        assert all(x == 0.0 for x in d.seconds)
