"""ctypes access to the parity checkers (TEST INFRASTRUCTURE).

* ``Oracle``  -- our plain-C restatement, oracle/liblemoracle.so
* ``RefLib``  -- the unmodified reference library compiled from its own
  sources (oracle/_ref/liblemref.so, see oracle/Makefile)

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg use
this module.  Nothing in the product imports it.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
ORACLE_SO = ROOT / "oracle" / "liblemoracle.so"
REF_SO = ROOT / "oracle" / "_ref" / "liblemref.so"
NOFLOW = 0xFFFFFFFF


class lo_params(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("K", "m_exp", "n_exp", "uplift_rate", "dt", "epsilon", "dx", "dy")] + [
        ("max_newton_iters", C.c_int)
    ]


class lo_step_out(C.Structure):
    _fields_ = [
        ("rec", C.c_void_p), ("donor", C.c_void_p), ("dnum", C.c_void_p), ("order", C.c_void_p),
        ("levels", C.c_void_p), ("nlevels", C.c_uint32), ("A", C.c_void_p),
        ("newton_iters", C.c_uint64), ("interior_noflow", C.c_uint32), ("err_cell", C.c_uint32),
    ]


def make_params(K=2e-6, m_exp=0.5, n_exp=1.0, uplift_rate=2e-3, dt=1000.0, epsilon=1e-6, dx=1.0, dy=1.0,
                max_newton_iters=100):
    return lo_params(K, m_exp, n_exp, uplift_rate, dt, epsilon, dx, dy, max_newton_iters)


def fnv1a64(a: np.ndarray) -> str:
    """FNV-1a-64 over raw little-endian bytes (SURVEY 8(c) golden anchors)."""
    b = np.ascontiguousarray(a).view(np.uint8).ravel()
    h = np.uint64(1469598103934665603)
    prime = np.uint64(1099511628211)
    # vectorise in chunks: FNV is sequential, so do it in C when available
    lib = Oracle.maybe()
    if lib is not None:
        return "%016x" % lib.L.lo_fnv1a64(b.ctypes.data, b.size)
    with np.errstate(over="ignore"):
        for x in b.tolist():
            h = (h ^ np.uint64(x)) * prime
    return "%016x" % int(h)


def _p(a):
    return a.ctypes.data if a is not None else None


class Oracle:
    _inst = None

    def __init__(self):
        L = C.CDLL(str(ORACLE_SO))
        L.lo_fnv1a64.restype = C.c_uint64
        L.lo_fnv1a64.argtypes = [C.c_void_p, C.c_size_t]
        L.lo_splitmix64.restype = C.c_uint64
        L.lo_splitmix64.argtypes = [C.c_uint64]
        L.lo_generate_terrain.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, C.c_void_p]
        L.lo_step.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.POINTER(lo_params), C.POINTER(lo_step_out)]
        L.lo_run.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.POINTER(lo_params), C.c_uint32,
                             C.POINTER(C.c_uint64), C.POINTER(C.c_uint32)]
        L.lo_newton.restype = C.c_double
        L.lo_newton.argtypes = [C.c_double] * 5 + [C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.lo_fill.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_double, C.c_void_p]
        L.lo_generate_queue.argtypes = [C.c_size_t, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p,
                                        C.c_void_p, C.POINTER(C.c_uint32)]
        L.lo_accumulate.argtypes = [C.c_size_t, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_double, C.c_void_p]
        L.lo_receivers_explicit.argtypes = [C.c_size_t, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                            C.c_void_p, C.c_void_p]
        L.lo_donors_explicit.argtypes = [C.c_size_t, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                         C.c_void_p]
        L.lo_step_mfd.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.POINTER(lo_params), C.c_double,
                                  C.POINTER(lo_step_out), C.c_void_p, C.c_void_p, C.POINTER(C.c_uint32)]
        self.L = L

    @classmethod
    def get(cls) -> "Oracle":
        if cls._inst is None:
            cls._inst = Oracle()
        return cls._inst

    @classmethod
    def maybe(cls):
        try:
            return cls.get()
        except OSError:
            return None

    def fill(self, elev: np.ndarray, mode: int, eps: float = 1e-8) -> np.ndarray:
        """Priority-Flood fill (depressions.cpp:26-68); mode 1 exact, 2 epsilon ascending."""
        h, w = elev.shape
        e = np.ascontiguousarray(elev, np.float64)
        out = np.empty_like(e)
        self.L.lo_fill(e.ctypes.data, w, h, mode, eps, out.ctypes.data)
        return out

    def terrain(self, w, h, seed):
        out = np.empty((h, w), np.float64)
        self.L.lo_generate_terrain(w, h, seed, out.ctypes.data)
        return out

    def step(self, elev: np.ndarray, conn=8, params=None, want_donor=True):
        """One reference step (src/simulation.cpp:68-89) on elev (modified in place)."""
        h, w = elev.shape
        n = w * h
        p = params or make_params()
        out = {
            "rec": np.empty(n, np.uint32), "donor": np.empty(n * conn, np.uint32) if want_donor else None,
            "dnum": np.empty(n, np.uint8), "order": np.empty(n, np.uint32), "levels": np.empty(n + 2, np.uint32),
            "A": np.empty(n, np.float64),
        }
        so = lo_step_out(_p(out["rec"]), _p(out["donor"]), _p(out["dnum"]), _p(out["order"]), _p(out["levels"]), 0,
                         _p(out["A"]), 0, 0, NOFLOW)
        rc = self.L.lo_step(elev.ctypes.data, w, h, conn, C.byref(p), C.byref(so))
        out["status"] = rc
        out["nlevels"] = so.nlevels
        out["levels"] = out["levels"][: so.nlevels + 1].copy()
        out["newton_iters"] = so.newton_iters
        out["interior_noflow"] = so.interior_noflow
        out["err_cell"] = so.err_cell
        return out

    def step_mfd(self, elev: np.ndarray, exponent=1.0, conn=8, params=None):
        """One reference step with StepSetup::routing = kMfd (simulation.cpp:31-89):
        A is the MFD drainage area; mfd_order / mfd_levels the MFD plan."""
        h, w = elev.shape
        n = w * h
        p = params or make_params()
        out = {"rec": np.empty(n, np.uint32), "order": np.empty(n, np.uint32), "levels": np.empty(n + 2, np.uint32),
               "A": np.empty(n, np.float64), "mfd_order": np.empty(n, np.uint32),
               "mfd_levels": np.empty(n + 2, np.uint32)}
        so = lo_step_out(_p(out["rec"]), None, None, _p(out["order"]), _p(out["levels"]), 0, _p(out["A"]), 0, 0, NOFLOW)
        mnl = C.c_uint32(0)
        rc = self.L.lo_step_mfd(elev.ctypes.data, w, h, conn, C.byref(p), exponent, C.byref(so),
                                _p(out["mfd_order"]), _p(out["mfd_levels"]), C.byref(mnl))
        out.update(status=rc, nlevels=so.nlevels, newton_iters=so.newton_iters, interior_noflow=so.interior_noflow,
                   err_cell=so.err_cell, mfd_nlevels=mnl.value)
        out["levels"] = out["levels"][: so.nlevels + 1].copy()
        out["mfd_levels"] = out["mfd_levels"][: mnl.value + 1].copy()
        return out

    def run(self, elev: np.ndarray, steps: int, conn=8, params=None):
        h, w = elev.shape
        p = params or make_params()
        nt = C.c_uint64(0)
        ec = C.c_uint32(NOFLOW)
        rc = self.L.lo_run(elev.ctypes.data, w, h, conn, C.byref(p), steps, C.byref(nt), C.byref(ec))
        return rc, nt.value, ec.value

    def newton(self, h0, hn, F, n, eps, maxit):
        it, conv = C.c_int(0), C.c_int(0)
        hh = self.L.lo_newton(h0, hn, F, n, eps, maxit, C.byref(it), C.byref(conv))
        return hh, it.value, bool(conv.value)


class RefLib:
    """The unmodified reference (oracle/_ref/liblemref.so)."""

    _inst = None

    def __init__(self):
        L = C.CDLL(str(REF_SO))
        L.lr_last_error.restype = C.c_char_p
        L.lr_max_threads.restype = C.c_int
        L.lr_generate_terrain.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, C.c_void_p]
        L.lr_simulate_step.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(lo_params), C.c_void_p] + [C.c_void_p] * 5 + [
            C.POINTER(C.c_uint32), C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]
        L.lr_run.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(lo_params), C.c_char_p, C.c_uint32, C.c_uint32,
                             C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(C.c_uint32)]
        L.lr_fill.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_double, C.c_void_p]
        L.lr_bench.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(lo_params), C.c_char_p, C.c_uint32, C.c_uint64,
                               C.c_uint32, C.c_uint32, C.c_void_p, C.POINTER(C.c_uint64), C.c_int, C.c_double]
        L.lr_bench_routing.argtypes = L.lr_bench.argtypes + [C.c_int, C.c_double]
        L.lr_simulate_step_mfd.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(lo_params), C.c_double, C.c_void_p,
                                           C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_uint32),
                                           C.POINTER(C.c_uint64), C.POINTER(C.c_uint32)]
        L.lr_run_routing.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(lo_params), C.c_char_p, C.c_uint32,
                                     C.c_uint32, C.c_int, C.c_double, C.c_void_p, C.POINTER(C.c_uint64),
                                     C.POINTER(C.c_uint32)]
        self.L = L

    @classmethod
    def available(cls) -> bool:
        return REF_SO.exists()

    @classmethod
    def get(cls) -> "RefLib":
        if cls._inst is None:
            cls._inst = RefLib()
        return cls._inst

    def terrain(self, w, h, seed):
        out = np.empty((h, w), np.float64)
        self.L.lr_generate_terrain(w, h, seed, out.ctypes.data)
        return out

    def step(self, elev: np.ndarray, conn=8, params=None):
        h, w = elev.shape
        n = w * h
        p = params or make_params()
        out = {"rec": np.empty(n, np.uint32), "donor": np.empty(n * conn, np.uint32), "dnum": np.empty(n, np.uint8),
               "order": np.empty(n, np.uint32), "levels": np.empty(n + 2, np.uint32), "A": np.empty(n, np.float64)}
        nl, nt, pits, ec = C.c_uint32(0), C.c_uint64(0), C.c_uint32(0), C.c_uint32(NOFLOW)
        rc = self.L.lr_simulate_step(w, h, conn, C.byref(p), elev.ctypes.data, _p(out["rec"]), _p(out["donor"]),
                                     _p(out["dnum"]), _p(out["order"]), _p(out["levels"]), C.byref(nl), _p(out["A"]),
                                     C.byref(nt), C.byref(pits), C.byref(ec))
        out.update(status=rc, nlevels=nl.value, newton_iters=nt.value, interior_noflow=pits.value, err_cell=ec.value)
        out["levels"] = out["levels"][: nl.value + 1].copy()
        return out

    def step_mfd(self, elev: np.ndarray, exponent=1.0, conn=8, params=None):
        """lem::simulate_step with routing = kMfd: h, MFD A and the MFD plan."""
        h, w = elev.shape
        n = w * h
        p = params or make_params()
        out = {"A": np.empty(n, np.float64), "mfd_order": np.empty(n, np.uint32), "mfd_levels": np.empty(n + 2, np.uint32)}
        nl, nt, ec = C.c_uint32(0), C.c_uint64(0), C.c_uint32(NOFLOW)
        rc = self.L.lr_simulate_step_mfd(w, h, conn, C.byref(p), exponent, elev.ctypes.data, _p(out["A"]),
                                         _p(out["mfd_order"]), _p(out["mfd_levels"]), C.byref(nl), C.byref(nt),
                                         C.byref(ec))
        out.update(status=rc, mfd_nlevels=nl.value, newton_iters=nt.value, err_cell=ec.value)
        out["mfd_levels"] = out["mfd_levels"][: nl.value + 1].copy()
        return out

    def run(self, elev: np.ndarray, steps: int, strategy="rb_serial", workers=1, conn=8, params=None, routing=0,
            mfd_exponent=1.0):
        h, w = elev.shape
        p = params or make_params()
        nt, ec = C.c_uint64(0), C.c_uint32(NOFLOW)
        if routing:
            rc = self.L.lr_run_routing(w, h, conn, C.byref(p), strategy.encode(), workers, steps, int(routing),
                                       float(mfd_exponent), elev.ctypes.data, C.byref(nt), C.byref(ec))
        else:
            rc = self.L.lr_run(w, h, conn, C.byref(p), strategy.encode(), workers, steps, elev.ctypes.data,
                               C.byref(nt), C.byref(ec))
        if rc not in (0, 3):
            raise RuntimeError(self.L.lr_last_error().decode())
        return rc, nt.value, ec.value

    def bench(self, w, h, steps, warmup=0, strategy="rb_private_queues", workers=None, seed=42, conn=8, params=None,
              fill=0, fill_eps=1e-8, routing=0, mfd_exponent=1.0):
        """Per-step wall seconds of lem::strategy_step on a persistent workspace
        (fill: 0 off, 1 exact, 2 epsilon -- lem::priority_flood_fill first)."""
        p = params or make_params()
        secs = np.zeros(max(1, steps), np.float64)
        nt = C.c_uint64(0)
        rc = self.L.lr_bench_routing(w, h, conn, C.byref(p), strategy.encode(), workers or self.max_threads(), seed,
                                     warmup, steps, secs.ctypes.data, C.byref(nt), int(fill), float(fill_eps),
                                     int(routing), float(mfd_exponent))
        if rc != 0:
            raise RuntimeError(self.L.lr_last_error().decode())
        return secs[:steps], nt.value

    def fill(self, elev: np.ndarray, mode: int, eps: float = 1e-8) -> np.ndarray:
        """lem::priority_flood_fill itself."""
        h, w = elev.shape
        e = np.ascontiguousarray(elev, np.float64)
        out = np.empty_like(e)
        if self.L.lr_fill(w, h, e.ctypes.data, mode, eps, out.ctypes.data) != 0:
            raise RuntimeError(self.L.lr_last_error().decode())
        return out

    def max_threads(self) -> int:
        return int(self.L.lr_max_threads())
