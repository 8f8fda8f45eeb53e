"""Pins the C oracle (oracle/lem_oracle.c) to the reference's own known-answer
tests and fixtures, before it is trusted as the GPU checker.

Each test cites the reference test it replays (paths under proj/tests/).
"""
import ctypes as C

import numpy as np
import pytest

from _oracle import NOFLOW, make_params

# ---------------------------------------------------------------- fixtures.hpp
# Ten-node worked example (fixtures.hpp:50-84, Table 1).
TEN_ADJ = [
    [(1, 1), (2, 1), (3, 2)],
    [(0, 1), (2, 1), (4, 1), (5, 1)],
    [(0, 1), (1, 1), (3, 2), (5, 1), (6, 1)],
    [(0, 2), (2, 2), (6, 1), (8, 1)],
    [(1, 1), (5, 1), (7, 1)],
    [(1, 1), (2, 1), (4, 1), (6, 1), (7, 1)],
    [(2, 1), (3, 1), (5, 1), (7, 1), (8, 1)],
    [(4, 1), (5, 1), (6, 1), (8, 3), (9, 1)],
    [(3, 1), (6, 1), (7, 3), (9, 2)],
    [(7, 1), (8, 2)],
]
TEN_ELEV = [3, 2, 3, 4, 1, 2, 3, 2, 4, 3]
TEN_REC = [1, 4, 1, 6, NOFLOW, 4, 5, 4, 6, 7]
TEN_DNUM = [0, 2, 0, 0, 3, 1, 2, 1, 0, 0]
TEN_QUEUE = [4, 1, 5, 7, 0, 2, 6, 9, 3, 8]
TEN_LEVELS = [0, 1, 4, 8, 10]
TEN_ACCUM = [1, 3, 1, 1, 10, 4, 3, 2, 1, 1]


def _ten_node(oracle):
    n, dmax = 10, 5
    off = np.zeros(n + 1, np.uint32)
    nbr, dist = [], []
    for c, lst in enumerate(TEN_ADJ):
        for j, d in lst:
            nbr.append(j)
            dist.append(float(d))
        off[c + 1] = len(nbr)
    nbr = np.array(nbr, np.uint32)
    dist = np.array(dist, np.float64)
    bnd = np.zeros(n, np.uint8)
    elev = np.array(TEN_ELEV, np.float64)
    rec = np.empty(n, np.uint32)
    oracle.L.lo_receivers_explicit(n, off.ctypes.data, nbr.ctypes.data, dist.ctypes.data, bnd.ctypes.data,
                                   elev.ctypes.data, rec.ctypes.data)
    donor = np.empty(n * dmax, np.uint32)
    dnum = np.empty(n, np.uint8)
    oracle.L.lo_donors_explicit(n, dmax, off.ctypes.data, nbr.ctypes.data, rec.ctypes.data, donor.ctypes.data,
                                dnum.ctypes.data)
    return rec, donor, dnum, dmax


def test_ten_node_receivers_donors(oracle):
    # test_flow_graph.cpp:40-59, acceptance.cpp:52-82
    rec, donor, dnum, dmax = _ten_node(oracle)
    assert rec.tolist() == TEN_REC
    assert dnum.tolist() == TEN_DNUM
    assert set(donor[dmax * 4: dmax * 4 + dnum[4]].tolist()) == {1, 5, 7}
    assert set(donor[dmax * 6: dmax * 6 + dnum[6]].tolist()) == {3, 8}


def test_ten_node_queue_and_accum(oracle):
    # test_traversal.cpp:32-39, test_accumulation.cpp:27-41
    rec, donor, dnum, dmax = _ten_node(oracle)
    order = np.empty(10, np.uint32)
    levels = np.empty(12, np.uint32)
    nl = C.c_uint32(0)
    rc = oracle.L.lo_generate_queue(10, rec.ctypes.data, donor.ctypes.data, dnum.ctypes.data, dmax,
                                    order.ctypes.data, levels.ctypes.data, C.byref(nl))
    assert rc == 0
    assert order.tolist() == TEN_QUEUE
    assert levels[: nl.value + 1].tolist() == TEN_LEVELS
    assert nl.value == 4
    A = np.empty(10, np.float64)
    oracle.L.lo_accumulate(10, order.ctypes.data, donor.ctypes.data, dnum.ctypes.data, dmax, 1.0, A.ctypes.data)
    assert A.tolist() == TEN_ACCUM


def test_cycle_raises_structure_error(oracle):
    # test_traversal.cpp:131-142
    rec = np.array([1, 0, NOFLOW], np.uint32)
    donor = np.full(6, NOFLOW, np.uint32)
    dnum = np.zeros(3, np.uint8)
    donor[0], dnum[0], donor[2], dnum[1] = 1, 1, 0, 1
    order = np.empty(3, np.uint32)
    levels = np.empty(5, np.uint32)
    nl = C.c_uint32(0)
    assert oracle.L.lo_generate_queue(3, rec.ctypes.data, donor.ctypes.data, dnum.ctypes.data, 2,
                                      order.ctypes.data, levels.ctypes.data, C.byref(nl)) == 2


def test_all_noflow_single_level(oracle):
    # test_traversal.cpp:50-60
    n = 12
    rec = np.full(n, NOFLOW, np.uint32)
    donor = np.full(n * 8, NOFLOW, np.uint32)
    dnum = np.zeros(n, np.uint8)
    order = np.empty(n, np.uint32)
    levels = np.empty(n + 2, np.uint32)
    nl = C.c_uint32(0)
    assert oracle.L.lo_generate_queue(n, rec.ctypes.data, donor.ctypes.data, dnum.ctypes.data, 8,
                                      order.ctypes.data, levels.ctypes.data, C.byref(nl)) == 0
    assert order.tolist() == list(range(n))
    assert levels[: nl.value + 1].tolist() == [0, n]


# ------------------------------------------------------------- raster cases
def test_pit_tiebreak_ramp_perimeter(oracle):
    # test_flow_graph.cpp:17-38, :115-123
    r = np.full((3, 3), 9.0)
    r[1, 1] = 5.0
    assert oracle.step(r.copy())["rec"][4] == NOFLOW
    t = np.full((3, 3), 5.0)
    t[0, 1] = 4.0  # north of centre
    t[1, 0] = 4.0  # west of centre
    assert oracle.step(t.copy())["rec"][4] == 1  # north wins (first in stencil order)
    ramp = np.add.outer(np.arange(4.0), np.arange(4.0))  # elev(x,y) = x + y
    rec = oracle.step(ramp.copy())["rec"]
    assert rec[1 * 4 + 1] == 0 and rec[2 * 4 + 2] == 5 and rec[1 * 4 + 2] == 1
    e = oracle.terrain(12, 9, 3)
    rec = oracle.step(e.copy())["rec"].reshape(9, 12)
    assert (rec[0] == NOFLOW).all() and (rec[-1] == NOFLOW).all()
    assert (rec[:, 0] == NOFLOW).all() and (rec[:, -1] == NOFLOW).all()


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_donors_invert_receivers(oracle, seed):
    # test_flow_graph.cpp:71-100
    s = oracle.step(oracle.terrain(50, 50, seed))
    rec, donor, dnum = s["rec"], s["donor"], s["dnum"]
    filled = 0
    for c in range(2500):
        for k in range(dnum[c]):
            assert rec[donor[8 * c + k]] == c
            filled += 1
    assert filled == int((rec != NOFLOW).sum())


@pytest.mark.parametrize("seed", [4, 9, 1377])
def test_queue_is_dependency_respecting_permutation(oracle, seed):
    # test_traversal.cpp:62-77
    s = oracle.step(oracle.terrain(30, 30, seed))
    order, rec, levels = s["order"], s["rec"], s["levels"]
    assert sorted(order.tolist()) == list(range(900))
    lvl = np.empty(900, np.int64)
    for l in range(s["nlevels"]):
        lvl[order[levels[l]:levels[l + 1]]] = l
    has = rec != NOFLOW
    assert (lvl[np.nonzero(has)[0]] > lvl[rec[has]]).all()


def test_mass_conservation_and_chain_oracle(oracle):
    # acceptance.cpp:113-129, test_accumulation.cpp:54-83, oracles.hpp:22-40
    for seed in range(1, 51):
        s = oracle.step(oracle.terrain(50, 50, seed))
        rec, A = s["rec"], s["A"]
        assert A[rec == NOFLOW].sum() == 2500.0
        if seed <= 3:
            chain = np.zeros(2500)
            for c in range(2500):
                x = c
                while True:
                    chain[x] += 1.0
                    if rec[x] == NOFLOW:
                        break
                    x = rec[x]
            assert (chain == A).all()


def _u01(oracle, k):
    return (oracle.L.lo_splitmix64(k) >> 11) * 2.0 ** -53


def test_newton_known_answers(oracle):
    # test_erosion.cpp:31-50, :96-122; acceptance.cpp:132-157
    h, it, ok = oracle.newton(2.0, 1.0, 1.0, 1.0, 1e-6, 100)
    assert ok and abs(h - 1.5) <= 1.5e-15 and it == 2
    for i in range(1000):
        hn = 10.0 * _u01(oracle, 3 * i)
        h0 = hn + 5.0 * _u01(oracle, 3 * i + 1)
        F = 50.0 * _u01(oracle, 3 * i + 2)
        h, it, ok = oracle.newton(h0, hn, F, 1.0, 1e-6, 100)
        assert ok and abs(h - (h0 + F * hn) / (1.0 + F)) <= 1e-6
    h, it, ok = oracle.newton(7.25, 1.0, 0.0, 1.0, 1e-6, 100)
    assert h == 7.25 and it == 1
    h, it, ok = oracle.newton(2.0, 1.0, 10.0, 0.5, 1e-6, 100)
    assert ok and h >= 1.0
    h, it, ok = oracle.newton(2.0, 1.0, 1.0, 2.0, 1e-12, 100)
    assert ok and abs(h - 1.6180339887) <= 1.7e-9


def test_newton_n2_vs_bisection(oracle):
    # test_erosion.cpp:52-65 with oracles.hpp:45-57
    def bisect(h0, hn, F, n, tol=1e-13):
        lo, hi = hn, h0
        while hi - lo > tol:
            mid = 0.5 * (lo + hi)
            if mid - h0 + F * (mid - hn) ** n > 0:
                hi = mid
            else:
                lo = mid
        return 0.5 * (lo + hi)

    for i in range(100):
        hn = 5.0 * _u01(oracle, 7 * i)
        h0 = hn + 0.1 + 3.0 * _u01(oracle, 7 * i + 1)
        F = 0.01 + 20.0 * _u01(oracle, 7 * i + 2)
        h, it, ok = oracle.newton(h0, hn, F, 2.0, 1e-12, 100)
        assert ok and abs(h - bisect(h0, hn, F, 2.0)) <= 1e-9


def test_convergence_error_carries_cell(oracle):
    # test_erosion.cpp:124-144: max_newton_iters=1 forces a failure
    e = oracle.terrain(20, 20, 5)
    s = oracle.step(e, params=make_params(max_newton_iters=1))
    assert s["status"] == 3 and s["err_cell"] != NOFLOW
    assert s["rec"][s["err_cell"]] != NOFLOW  # a cell that was being eroded


def test_k_zero_is_uplift_only(oracle):
    # test_erosion.cpp:96-114, test_simulation.cpp:17-28: K=0 costs one iteration per cell
    e = oracle.terrain(12, 12, 5)
    e0 = e.copy()
    s = oracle.step(e, params=make_params(K=0.0))
    interior = np.zeros((12, 12), bool)
    interior[1:-1, 1:-1] = True
    assert (e[~interior] == e0[~interior]).all()
    assert (e[interior] == e0[interior] + 2.0).all()
    eroded = int((s["rec"] != NOFLOW).sum())
    assert s["newton_iters"] == eroded


def test_terrain_splitmix_canary(oracle):
    # test_terrain_io.cpp:62-72 style: pure function of (seed, i), fixed stream
    a = oracle.terrain(7, 5, 42)
    assert a.min() >= 0.0 and a.max() < 1.0
    z = oracle.L.lo_splitmix64(42)
    assert a.ravel()[0] == (z >> 11) * 2.0 ** -53


# ---- MFD (proj/tests/test_mfd.cpp, acceptance.cpp:283-327) -------------------

def _mfd(oracle, r, exponent=1.0):
    import ctypes as C
    h, w = r.shape
    n = w * h
    nbh = _nbh(oracle, 8)
    recs = np.empty(n * 8, np.uint32)
    alpha = np.empty(n * 8, np.float64)
    rnum = np.empty(n, np.uint8)
    oracle.L.lo_compute_mfd.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_double, C.c_void_p,
                                        C.c_void_p, C.c_void_p]
    oracle.L.lo_compute_mfd(np.ascontiguousarray(r).ctypes.data, w, h, C.addressof(nbh), exponent,
                            recs.ctypes.data, alpha.ctypes.data, rnum.ctypes.data)
    return recs.reshape(n, 8), alpha.reshape(n, 8), rnum


def _nbh(oracle, conn, dx=1.0, dy=1.0):
    import ctypes as C

    class lo_nbh(C.Structure):
        _fields_ = [("connectivity", C.c_int), ("ox", C.c_int * 8), ("oy", C.c_int * 8), ("dist", C.c_double * 8),
                    ("dx", C.c_double), ("dy", C.c_double)]

    nb = lo_nbh()
    oracle.L.lo_make_nbh.argtypes = [C.c_int, C.c_double, C.c_double, C.c_void_p]
    assert oracle.L.lo_make_nbh(conn, dx, dy, C.addressof(nb)) == 0
    return nb


def test_mfd_single_downslope_neighbor(oracle):
    """test_mfd.cpp 'single downslope neighbor gets the whole weight'."""
    r = np.full((3, 3), 5.0)
    r[1, 1] = 3.0
    r[0, 1] = 1.0
    recs, alpha, rnum = _mfd(oracle, r)
    assert rnum[4] == 1 and recs[4, 0] == 1 and alpha[4, 0] == 1.0


def test_mfd_two_cardinals_split(oracle):
    """test_mfd.cpp 'two downslope cardinals split 1/3 and 2/3 at exponent 1' (1/5, 4/5 at 2)."""
    r = np.full((3, 3), 9.0)
    r[1, 1] = 2.0
    r[0, 1] = 1.0  # north, slope 1
    r[1, 0] = 0.0  # west, slope 2
    recs, alpha, rnum = _mfd(oracle, r, 1.0)
    assert rnum[4] == 2 and recs[4, 0] == 1 and recs[4, 1] == 3  # stencil order: (0,-1) before (-1,0)
    assert abs(alpha[4, 0] - 1 / 3) < 1e-15 and abs(alpha[4, 1] - 2 / 3) < 1e-15
    recs, alpha, rnum = _mfd(oracle, r, 2.0)
    assert abs(alpha[4, 0] - 0.2) < 1e-15 and abs(alpha[4, 1] - 0.8) < 1e-15


def test_mfd_pits_and_perimeter_have_no_receivers(oracle):
    r = np.full((5, 5), 4.0)
    r[2, 2] = 1.0
    recs, alpha, rnum = _mfd(oracle, r)
    assert rnum[12] == 0
    per = np.ones((5, 5), bool)
    per[1:-1, 1:-1] = False
    assert (rnum[per.ravel()] == 0).all()


def test_mfd_weights_sum_to_one_receivers_lower(oracle):
    r = oracle.terrain(30, 30, 21)
    recs, alpha, rnum = _mfd(oracle, r, 1.1)
    e = r.ravel()
    for c in range(900):
        k = rnum[c]
        assert all(e[recs[c, i]] < e[c] for i in range(k))
        if k:
            assert abs(alpha[c, :k].sum() - 1.0) < 1e-12


def test_mfd_plan_is_a_level_order_and_mass_conserving(oracle):
    """acceptance.cpp:283-300 criterion 8 (first half): every cell sits strictly
    above all of its receivers in the MFD level order; the MFD drainage area
    reaching level 0 is the whole raster's area."""
    for seed in range(1, 6):
        e = oracle.terrain(50, 50, seed)
        r0 = e.copy()
        s = oracle.step_mfd(e)
        assert s["status"] == 0
        lvl = np.empty(2500, np.int64)
        lv = s["mfd_levels"]
        for l in range(len(lv) - 1):
            lvl[s["mfd_order"][lv[l]:lv[l + 1]]] = l
        recs, alpha, rnum = _mfd(oracle, r0)
        for c in range(2500):
            for i in range(rnum[c]):
                assert lvl[c] > lvl[recs[c, i]], (seed, c)
        sinks = s["mfd_order"][lv[0]:lv[1]]
        assert abs(s["A"][sinks].sum() - 2500.0) < 1e-8
