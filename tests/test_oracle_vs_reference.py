"""Pins the C oracle against outputs of the REAL reference: the committed
golden fixtures (tests/golden/, made by tests/golden/make_golden.py from
oracle/_ref/liblemref.so) and, when the reference library is present, live
side-by-side runs on random inputs."""
import json

import numpy as np
import pytest

from _oracle import RefLib, fnv1a64, make_params

ARRAYS = ("rec", "dnum", "donor", "order", "levels", "A")


def _small_cases(golden_dir):
    return sorted(golden_dir.glob("small_*.npz"))


def test_small_golden_fixtures(oracle, golden_dir):
    cases = _small_cases(golden_dir)
    assert len(cases) >= 8
    for path in cases:
        g = np.load(path)
        kw = json.loads(str(g["params"]))
        e = g["h0"].copy()
        s = oracle.step(e, conn=int(g["conn"]), params=make_params(**kw))
        assert s["status"] == 0, path.name
        for k in ARRAYS:
            assert np.array_equal(s[k], g[k]), (path.name, k)
        assert np.array_equal(e.view(np.uint64), g["h1"].view(np.uint64)), path.name
        assert s["newton_iters"] == int(g["newton_iters"]) and s["interior_noflow"] == int(g["interior_noflow"])


def test_anchor_1000_step1(oracle, golden_dir):
    a = json.loads((golden_dir / "anchors.json").read_text())["1000"]
    e = oracle.terrain(1000, 1000, 42)
    assert fnv1a64(e) == a["terrain"]
    s = oracle.step(e)
    st = a["step1"]
    assert fnv1a64(s["rec"]) == st["rec"]
    assert fnv1a64(s["dnum"]) == st["dnum"]
    assert fnv1a64(s["order"]) == st["order"]
    assert fnv1a64(s["A"]) == st["A"]
    assert fnv1a64(e) == st["h"]
    assert s["levels"].tolist() == st["levels"]
    assert s["interior_noflow"] == st["interior_noflow"] and s["newton_iters"] == st["newton_iters"]


@pytest.mark.slow
def test_anchor_1000_step120(oracle, golden_dir):
    a = json.loads((golden_dir / "anchors.json").read_text())["1000"]["step120"]
    e = oracle.terrain(1000, 1000, 42)
    rc, newton, _ = oracle.run(e, 120)
    assert rc == 0
    assert fnv1a64(e) == a["h"] and newton == a["newton_total"]


@pytest.mark.skipif(not RefLib.available(), reason="oracle/_ref not built (no /root/reference here)")
@pytest.mark.parametrize("w,h,seed,conn,kw", [
    (23, 19, 101, 8, {}),
    (31, 7, 102, 4, {}),
    (40, 33, 103, 8, {"dx": 0.25, "dy": 3.0, "m_exp": 0.7}),
    (26, 26, 104, 8, {"n_exp": 1.5}),
    (26, 26, 105, 8, {"n_exp": 0.7, "K": 1e-4}),
])
def test_live_vs_reference(oracle, w, h, seed, conn, kw):
    ref = RefLib.get()
    p = make_params(**kw)
    e_o = oracle.terrain(w, h, seed)
    e_r = ref.terrain(w, h, seed)
    assert np.array_equal(e_o, e_r)
    for _ in range(5):
        so = oracle.step(e_o, conn=conn, params=p)
        sr = ref.step(e_r, conn=conn, params=p)
        assert so["status"] == sr["status"] == 0
        for k in ARRAYS:
            assert np.array_equal(so[k], sr[k]), k
        assert np.array_equal(e_o.view(np.uint64), e_r.view(np.uint64))
        assert so["newton_iters"] == sr["newton_iters"]


def test_fill_golden_fixtures(oracle, golden_dir):
    """The oracle's Priority-Flood restatement reproduces lem::priority_flood_fill
    (fixtures from the real reference, both modes, two epsilons)."""
    cases = sorted(golden_dir.glob("fill_*.npz"))
    assert len(cases) >= 8
    for path in cases:
        g = np.load(path)
        f = oracle.fill(g["h0"], int(g["mode"]), float(g["eps"]))
        assert np.array_equal(f.view(np.uint64), g["f"].view(np.uint64)), path.name


@pytest.mark.skipif(not RefLib.available(), reason="reference library not built")
@pytest.mark.parametrize("mode", [1, 2])
def test_fill_vs_reference_live(oracle, mode):
    """acceptance.cpp:228-249's 20 seeds at 100^2, plus a larger raster."""
    ref = RefLib.get()
    for seed in range(1, 21):
        e = ref.terrain(100, 100, seed)
        assert np.array_equal(oracle.fill(e, mode).view(np.uint64), ref.fill(e, mode).view(np.uint64)), seed
    e = ref.terrain(400, 300, 77)
    assert np.array_equal(oracle.fill(e, mode).view(np.uint64), ref.fill(e, mode).view(np.uint64))


def test_mfd_golden_fixtures(oracle, golden_dir):
    """The oracle's MFD restatement (compute_mfd / generate_mfd_order /
    accumulate_mfd, src/mfd.cpp:33-132, inside simulate_step with
    Routing::kMfd) against fixtures made by the unmodified reference: h,
    the MFD drainage area and the MFD plan bit for bit."""
    cases = sorted(golden_dir.glob("mfd_*.npz"))
    assert len(cases) >= 7
    for path in cases:
        g = np.load(path)
        kw = json.loads(str(g["params"]))
        e = g["h0"].copy()
        s = oracle.step_mfd(e, exponent=float(g["exponent"]), conn=int(g["conn"]), params=make_params(**kw))
        assert s["status"] == 0, path.name
        assert np.array_equal(s["A"].view(np.uint64), g["A"].view(np.uint64)), path.name
        assert np.array_equal(s["mfd_order"], g["mfd_order"]) and np.array_equal(s["mfd_levels"], g["mfd_levels"])
        assert np.array_equal(e.view(np.uint64), g["h1"].view(np.uint64)), path.name
        assert s["newton_iters"] == int(g["newton_iters"]), path.name


@pytest.mark.skipif(not RefLib.available(), reason="reference library not built")
@pytest.mark.parametrize("w,h,seed,conn,ex,kw", [
    (90, 70, 21, 8, 1.0, {}), (61, 47, 22, 8, 1.3, {"m_exp": 0.4}), (50, 50, 23, 4, 1.0, {}),
    (40, 64, 24, 8, 0.7, {"dx": 2.0, "dy": 0.5}), (120, 33, 25, 8, 1.0, {"n_exp": 2.0}),
])
def test_mfd_live_vs_reference(oracle, w, h, seed, conn, ex, kw):
    ref = RefLib.get()
    p = make_params(**kw)
    e1 = ref.terrain(w, h, seed)
    e2 = e1.copy()
    for _ in range(3):
        r = ref.step_mfd(e1, exponent=ex, conn=conn, params=p)
        o = oracle.step_mfd(e2, exponent=ex, conn=conn, params=p)
        assert r["status"] == o["status"] == 0
        assert np.array_equal(r["A"].view(np.uint64), o["A"].view(np.uint64))
        assert np.array_equal(r["mfd_order"], o["mfd_order"]) and np.array_equal(r["mfd_levels"], o["mfd_levels"])
        assert np.array_equal(e1.view(np.uint64), e2.view(np.uint64))
        assert r["newton_iters"] == o["newton_iters"]
