"""Host-side mirror of the reference's step API for the ``rb_gpu`` strategy.

Same names, argument meaning and error behaviour as the reference's C++
entry points, so code written against ``lem`` reads the same here:

=====================================  ==================================================
this module                            reference (proj/)
=====================================  ==================================================
``SimParams``                          include/lem/erosion.hpp:15-25
``Neighborhood.d8/d4/make``            include/lem/neighborhood.hpp:31-45, src/neighborhood.cpp
``GridGraph``                          include/lem/grid_graph.hpp:15-66
``StrategyKind`` / ``Strategy``        include/lem/strategy.hpp:12-56 (+ ``rb_gpu``)
``StepSetup`` / ``OrderKind``          include/lem/simulation.hpp:54-60
``SimWorkspace``                       include/lem/simulation.hpp:43-52
``StepDiagnostics``                    include/lem/simulation.hpp:34-40
``strategy_step``                      include/lem/scheduler.hpp:38-41, src/scheduler.cpp:408-464
``RunConfig`` / ``run_simulation``     include/lem/config.hpp:55-76, scheduler.hpp:61-65
``generate_terrain``                   include/lem/terrain.hpp:18 (runs on the device)
``Error`` & subclasses                 include/lem/error.hpp:10-43
=====================================  ==================================================

Every compute call goes through the C-ABI (``_abi``) into the sm_100a
kernels; the CPU strategies of the reference are not re-implemented here.
Elevations are ``numpy.float64`` arrays of shape ``(height, width)``
(row-major, index ``y*width + x`` like ``Raster<double>``).
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import Callable, List, Optional

import numpy as np

from . import _abi

NoFlow = _abi.NOFLOW  # kNoFlow, include/lem/raster.hpp:16
PHASE_NAMES = ("receivers", "donors", "order", "accum", "uplift", "erosion")


# ---------------------------------------------------------------- errors
class Error(RuntimeError):
    """lem::Error (error.hpp:10-13)."""


class ConfigError(Error):
    """lem::ConfigError (error.hpp:16-19)."""


class StructureError(Error):
    """lem::StructureError (error.hpp:28-31)."""


class ConvergenceError(Error):
    """lem::ConvergenceError (error.hpp:35-43): carries the failing cell."""

    def __init__(self, cell: int, what: str):
        super().__init__(what)
        self._cell = int(cell)

    def cell(self) -> int:
        return self._cell


def _raise(status: int, msg: str, cell: int = NoFlow):
    # ErrorCollector::rethrow mapping (scheduler.cpp:45-49)
    if status == _abi.ECONFIG:
        raise ConfigError(msg)
    if status == _abi.ESTRUCTURE:
        raise StructureError(msg)
    if status == _abi.ECONVERGENCE:
        raise ConvergenceError(cell, msg)
    raise Error(msg)


# ---------------------------------------------------------------- params
@dataclass
class SimParams:
    """lem::SimParams with the reference defaults (erosion.hpp:16-24)."""

    K: float = 2e-6
    m_exp: float = 0.5
    n_exp: float = 1.0
    uplift_rate: float = 2e-3
    dt: float = 1000.0
    epsilon: float = 1e-6
    dx: float = 1.0
    dy: float = 1.0
    max_newton_iters: int = 100

    def cell_area(self) -> float:
        return self.dx * self.dy

    def validate(self) -> None:
        """SimParams::validate (erosion.cpp:10-17)."""
        if not self.dt > 0:
            raise ConfigError("dt must be > 0")
        if not self.epsilon > 0:
            raise ConfigError("epsilon must be > 0")
        if not self.K >= 0:
            raise ConfigError("K must be >= 0")
        if not self.n_exp > 0:
            raise ConfigError("n_exp must be > 0")
        if not (self.dx > 0) or not (self.dy > 0):
            raise ConfigError("cell spacing must be > 0")
        if self.max_newton_iters < 1:
            raise ConfigError("max_newton_iters must be >= 1")

    def to_abi(self, connectivity: int) -> _abi.lemgpu_params:
        return _abi.lemgpu_params(
            self.K, self.m_exp, self.n_exp, self.uplift_rate, self.dt, self.epsilon,
            self.dx, self.dy, int(self.max_newton_iters), int(connectivity),
        )


@dataclass
class Neighborhood:
    """lem::Neighborhood (neighborhood.hpp:31-45); only the shape matters here."""

    connectivity: int = 8
    dx: float = 1.0
    dy: float = 1.0

    @staticmethod
    def d8(dx: float = 1.0, dy: float = 1.0) -> "Neighborhood":
        return Neighborhood(8, dx, dy)

    @staticmethod
    def d4(dx: float = 1.0, dy: float = 1.0) -> "Neighborhood":
        return Neighborhood(4, dx, dy)

    @staticmethod
    def make(connectivity: int, dx: float = 1.0, dy: float = 1.0) -> "Neighborhood":
        """Neighborhood::make (neighborhood.cpp:32-43)."""
        if connectivity == 6:
            raise ConfigError("hexagonal (6-connected) grids are not implemented")
        if connectivity not in (4, 8):
            raise ConfigError(f"connectivity must be 4 or 8, got {connectivity}")
        return Neighborhood(connectivity, dx, dy)

    def max_degree(self) -> int:
        return self.connectivity


@dataclass
class GridGraph:
    """lem::GridGraph (grid_graph.hpp:15-66)."""

    width: int
    height: int
    nbh: Neighborhood = field(default_factory=Neighborhood.d8)

    def size(self) -> int:
        return self.width * self.height

    def max_degree(self) -> int:
        return self.nbh.connectivity

    def neighborhood(self) -> Neighborhood:
        return self.nbh


class StrategyKind(enum.Enum):
    """lem::StrategyKind (strategy.hpp:12-19) plus the B200 strategy."""

    kBwSerial = "bw_serial"
    kRbSerial = "rb_serial"
    kBwParErosion = "bw_par_erosion"
    kRbParErosion = "rb_par_erosion"
    kRbParAll = "rb_par_all"
    kRbPrivateQueues = "rb_private_queues"
    kRbGpu = "rb_gpu"


kAllStrategies = tuple(StrategyKind)


def to_string(k: StrategyKind) -> str:
    return k.value


def strategy_from_string(s: str) -> Optional[StrategyKind]:
    """strategy_from_string (strategy.hpp:52-56)."""
    for k in StrategyKind:
        if k.value == s:
            return k
    return None


@dataclass
class Strategy:
    kind: StrategyKind = StrategyKind.kRbGpu
    workers: int = 1  # ignored by rb_gpu (one device)
    device: int = 0


class OrderKind(enum.Enum):
    kQueue = 0
    kStack = 1


class Routing(enum.Enum):
    kD8 = 0
    kMfd = 1


@dataclass
class StepSetup:
    order: OrderKind = OrderKind.kQueue
    routing: Routing = Routing.kD8
    mfd_exponent: float = 1.0


@dataclass
class StepDiagnostics:
    """lem::StepDiagnostics (simulation.hpp:34-40) + device facts."""

    seconds: List[float] = field(default_factory=lambda: [0.0] * 6)
    newton_iters: int = 0
    interior_noflow: int = 0
    nlevels: int = 0
    lut_misses: int = 0
    escaped_trees: int = 0  # trees finished by the escape path (tile path), else source chunks
    kernel_seconds: List[float] = field(default_factory=lambda: [0.0] * 4)  # receiver, tile, escape-levels, escape-physics spans
    escaped_cells: int = 0
    mfd_passes: int = 0  # routing = kMfd: tile passes of the MFD accumulation (k_mfd_tiles)

    @staticmethod
    def from_abi(d: _abi.lemgpu_diag) -> "StepDiagnostics":
        return StepDiagnostics(list(d.seconds), int(d.newton_iters), int(d.interior_noflow),
                               int(d.nlevels), int(d.lut_misses), int(d.escaped_trees), list(d.kernel_s),
                               int(d.escaped_cells), int(d.mfd_passes))

    @property
    def timings(self):
        return dict(zip(PHASE_NAMES, self.seconds))


# ------------------------------------------------------------- device ctx
# lemgpu_options knobs under the names DESIGN.md's knob table uses
_KNOB_NAMES = {
    "LEMGPU_PATH": ("global_path", lambda v: 1 if str(v) == "global" else 0),
    "LEMGPU_FORCE_ESCAPE": ("force_escape", int), "LEMGPU_FORCE_DEEP": ("force_deep", int),
    "LEMGPU_EAGER": ("eager", int), "LEMGPU_NO_TMA": ("no_tma", int), "LEMGPU_NO_NARROW": ("no_narrow", int),
    "LEMGPU_ESC_SMALL": ("no_esc_small", lambda v: 0 if int(v) else 1),
    "LEMGPU_PIPE": ("pipe", lambda v: int(v) if int(v) > 0 else -1),
    "LEMGPU_PIPE_CHAIN": ("pipe_unchained", lambda v: 0 if int(v) else 1),
    "LEMGPU_TILE_GRID": ("tile_grid", int), "LEMGPU_ESC_GRID": ("esc_grid", int),
    "LEMGPU_ESC_SMALL_GRID": ("esc_small_grid", int), "LEMGPU_PIPE_TILE_GRID": ("pipe_tile_grid", int),
    "LEMGPU_LUT_ENTRIES": ("lut_entries", int), "LEMGPU_HOST_BANDS": ("host_bands", int),
    "LEMGPU_PATCH_CAP": ("patch_cap", int), "LEMGPU_HOST_PROFILE": ("host_profile", int),
    "LEMGPU_ESC_FOREST": ("esc_forest", int), "LEMGPU_MFD_LEVELS": ("mfd_levels", int),
    "LEMGPU_PHASE_CLOCKS": ("phase_clocks", int),
}


def make_options(options) -> Optional[_abi.lemgpu_options]:
    """lemgpu_options from a dict of field names (or DESIGN.md knob names)."""
    if not options:
        return None
    o = _abi.lemgpu_options()
    for k, v in options.items():
        if k in _KNOB_NAMES:
            k, conv = _KNOB_NAMES[k]
            v = conv(v)
        setattr(o, k, int(v))
    return o


class DeviceContext:
    """Owner of one ``lemgpu_ctx`` (device buffers + stream).  ``options``:
    schedule / test knobs (lemgpu_options fields or DESIGN.md knob names)."""

    def __init__(self, width: int, height: int, params: SimParams, connectivity: int = 8,
                 device: int = 0, members: int = 1, per_member=None, options=None):
        L = _abi.lib()
        self.width, self.height, self.members = int(width), int(height), int(members)
        self.connectivity = connectivity
        p = params.to_abi(connectivity)
        h = C.c_void_p()
        opts = make_options(options)
        if members == 1 and per_member is None and opts is None:
            rc = L.lemgpu_create(device, self.width, self.height, C.byref(p), C.byref(h))
        else:
            arr = None
            if per_member is not None:
                arr = (_abi.lemgpu_member * members)(*[_abi.lemgpu_member(float(k), float(m)) for k, m in per_member])
            rc = L.lemgpu_create_ex(device, self.width, self.height, self.members, C.byref(p), arr,
                                    C.byref(opts) if opts is not None else None, C.byref(h))
        if rc != _abi.OK:
            _raise(rc, L.lemgpu_error_message(None).decode())
        self._h = h
        self._L = L
        self.n = self.width * self.height * self.members

    def close(self):
        if getattr(self, "_h", None):
            self._L.lemgpu_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc: int):
        if rc != _abi.OK:
            L = self._L
            _raise(rc, L.lemgpu_error_message(self._h).decode(), L.lemgpu_error_cell(self._h))

    @property
    def handle(self):
        return self._h

    def upload(self, elev: np.ndarray):
        a = np.ascontiguousarray(elev, dtype=np.float64)
        if a.size != self.n:
            raise ConfigError(f"elevation has {a.size} cells, context holds {self.n}")
        self._check(self._L.lemgpu_upload_elev(self._h, a.ctypes.data))

    def download(self, out: Optional[np.ndarray] = None) -> np.ndarray:
        if out is None:
            shape = (self.height, self.width) if self.members == 1 else (self.members, self.height, self.width)
            out = np.empty(shape, dtype=np.float64)
        assert out.flags.c_contiguous and out.dtype == np.float64 and out.size == self.n
        self._check(self._L.lemgpu_download_elev(self._h, out.ctypes.data))
        return out

    def generate_terrain(self, seeds=None):
        arr = None
        if seeds is not None:
            seeds = list(seeds)
            arr = (C.c_uint64 * len(seeds))(*seeds)
        self._check(self._L.lemgpu_generate_terrain(self._h, arr))

    def fill(self, opts: Optional["FillOptions"] = None, mode: Optional[int] = None, epsilon: float = 1e-8):
        """Priority-Flood fill of the device elevation in place (lemgpu_fill)."""
        if opts is not None:
            mode, epsilon = int(opts.mode), opts.epsilon_increment
        self._check(self._L.lemgpu_fill(self._h, int(mode or 0), float(epsilon)))

    def step(self, nsteps: int = 1) -> List[StepDiagnostics]:
        diags = (_abi.lemgpu_diag * max(1, nsteps))()
        self._check(self._L.lemgpu_step(self._h, nsteps, diags))
        return [StepDiagnostics.from_abi(diags[i]) for i in range(nsteps)]

    def step_async(self, nsteps: int = 1):
        self._check(self._L.lemgpu_step_async(self._h, nsteps))

    def sync(self) -> List[StepDiagnostics]:
        cap = 4096
        diags = (_abi.lemgpu_diag * cap)()
        cnt = C.c_uint32(0)
        self._check(self._L.lemgpu_sync(self._h, diags, cap, C.byref(cnt)))
        return [StepDiagnostics.from_abi(diags[i]) for i in range(min(cap, cnt.value))]

    def step_host(self, elev: np.ndarray) -> StepDiagnostics:
        assert elev.flags.c_contiguous and elev.dtype == np.float64 and elev.size == self.n
        d = _abi.lemgpu_diag()
        self._check(self._L.lemgpu_step_host(self._h, elev.ctypes.data, C.byref(d)))
        return StepDiagnostics.from_abi(d)

    def download_graph(self, rec=True, dnum=True, donor=False, order=True, levels=True, A=True):
        n = self.n
        out = {}
        ptr = lambda a: a.ctypes.data if a is not None else None  # noqa: E731
        r = np.empty(n, np.uint32) if rec else None
        d = np.empty(n, np.uint8) if dnum else None
        dn = np.empty(n * self.connectivity, np.uint32) if donor else None
        o = np.empty(n, np.uint32) if order else None
        lv = np.empty(n + 2, np.uint32) if levels else None
        a = np.empty(n, np.float64) if A else None
        nl = C.c_uint32(0)
        self._check(self._L.lemgpu_download_graph(self._h, ptr(r), ptr(d), ptr(dn), ptr(o), ptr(lv), C.byref(nl), ptr(a)))
        if rec:
            out["rec"] = r
        if dnum:
            out["dnum"] = d
        if donor:
            out["donor"] = dn
        if order:
            out["order"] = o
        if levels:
            out["levels"] = lv[: nl.value + 1].copy()
        if A:
            out["A"] = a
        out["nlevels"] = nl.value
        return out

    def set_routing(self, routing, mfd_exponent: float = 1.0):
        """StepSetup::routing / mfd_exponent (simulation.hpp:55-60): Routing.kMfd
        feeds the erosion the multiple-flow drainage area (mfd.cpp:33-132)."""
        self._check(self._L.lemgpu_set_routing(self._h, int(Routing(routing) == Routing.kMfd), float(mfd_exponent)))

    def download_mfd(self, A=True, plan=True):
        """The last step's MFD drainage area (ws.accum) and MFD plan (ws.mfd_plan)."""
        n = self.n
        a = np.empty(n, np.float64) if A else None
        o = np.empty(n, np.uint32) if plan else None
        lv = np.empty(n + 2, np.uint32) if plan else None
        nl = C.c_uint32(0)
        ptr = lambda x: x.ctypes.data if x is not None else None  # noqa: E731
        self._check(self._L.lemgpu_download_mfd(self._h, ptr(a), ptr(o), ptr(lv), C.byref(nl)))
        out = {"nlevels": nl.value}
        if A:
            out["A"] = a
        if plan:
            out["order"] = o
            out["levels"] = lv[: nl.value + 1].copy()
        return out

    def stream_ptr(self) -> int:
        return int(self._L.lemgpu_stream(self._h) or 0)

    def kernel_timing(self, enable: bool):
        self._check(self._L.lemgpu_kernel_timing(self._h, 1 if enable else 0))

    def kernel_times(self):
        ms = (C.c_double * 5)()
        n = C.c_uint32(0)
        self._check(self._L.lemgpu_kernel_times(self._h, ms, C.byref(n)))
        return {"step": ms[0], "recv_donor": ms[1], "order": ms[2], "physics": ms[3], "tiles": ms[4],
                "launches": n.value}

    # ---- ensemble statistics
    def stats_enable(self, member_offset: int = 0, members_total: Optional[int] = None, interval: int = 1):
        """{mean, max, min, sum} of every member's elevation after every
        `interval`-th step, inside the step graph; rows member_offset.. of a
        [members_total, 4] table."""
        total = self.members if members_total is None else int(members_total)
        self._check(self._L.lemgpu_stats_enable(self._h, int(member_offset), total, int(interval)))
        self.stats_total = total

    def stats_comm_init(self, nccl_id: bytes, nranks: int, rank: int):
        buf = C.create_string_buffer(bytes(nccl_id), len(nccl_id))
        self._check(self._L.lemgpu_stats_comm_init(self._h, buf, len(nccl_id), int(nranks), int(rank)))

    def stats_table(self) -> np.ndarray:
        out = np.empty((self.stats_total, 4), np.float64)
        self._check(self._L.lemgpu_stats_table(self._h, out.ctypes.data))
        return out

    def tile_capture(self, enable: bool = True):
        """Debug: make every step's tile pass record each finished cell's level and
        drainage area (lemgpu_debug_tile_capture); read them with tile_levels()."""
        self._check(self._L.lemgpu_debug_tile_capture(self._h, 1 if enable else 0))

    def tile_levels(self):
        """(level u8 [N], A f64 [N]) written by the last step's tile pass; level 0xFF
        marks a cell of a tree that escaped its tile (finished by the escape path)."""
        n = self.n
        lv = np.empty(n, np.uint8)
        A = np.empty(n, np.float64)
        self._check(self._L.lemgpu_debug_copy(self._h, 3, lv.ctypes.data, lv.nbytes))
        self._check(self._L.lemgpu_debug_copy(self._h, 4, A.ctypes.data, A.nbytes))
        return lv, A

    def debug_timeline(self):
        """k_flow barrier timestamps of the last step, as ms offsets from its start."""
        buf = (C.c_uint64 * 96)()
        n = C.c_uint32(0)
        self._check(self._L.lemgpu_debug_timeline(self._h, buf, 96, C.byref(n)))
        t = [buf[i] for i in range(n.value)]
        return [(x - t[0]) * 1e-6 for x in t]

    def kernels_per_step(self) -> int:
        return int(self._L.lemgpu_kernels_per_step(self._h))

    def pipeline_bands(self) -> int:
        """Bands of the receiver / tile pipeline (0: the step graph is not pipelined)."""
        return int(self._L.lemgpu_pipeline_bands(self._h))

    def pow_variant(self) -> int:
        """The host glibc pow the device reproduces: 1 __pow_fma, 0 __pow_sse2, -1 none."""
        return int(self._L.lemgpu_pow_variant(self._h))

    def device_bytes(self) -> int:
        b = C.c_uint64(0)
        self._check(self._L.lemgpu_device_bytes(self._h, C.byref(b)))
        return b.value

    def member_stats_device(self, device_ptr: int):
        self._check(self._L.lemgpu_member_stats_device(self._h, C.c_void_p(device_ptr)))


class SimWorkspace:
    """lem::SimWorkspace (simulation.hpp:43-52): scratch reused across steps.

    For rb_gpu it owns the device context; graph arrays of the last step are
    fetched lazily (``fg``/``plan``/``accum``) for parity checks."""

    def __init__(self):
        self.gpu: Optional[DeviceContext] = None
        self._key = None

    def ensure(self, grid: GridGraph, params: SimParams, device: int = 0, setup=None) -> DeviceContext:
        key = (grid.width, grid.height, grid.nbh.connectivity, device, tuple(vars(params).items()))
        if self.gpu is None or self._key != key:
            if self.gpu is not None:
                self.gpu.close()
            self.gpu = DeviceContext(grid.width, grid.height, params, grid.nbh.connectivity, device,
                                     options={"phase_clocks": 1})  # StepDiagnostics::timings
            self._key = key
            self._routing = (Routing.kD8, 1.0)
        want = (setup.routing, setup.mfd_exponent) if setup is not None else (Routing.kD8, 1.0)
        if want != self._routing:
            self.gpu.set_routing(want[0], want[1])
            self._routing = want
        return self.gpu

    def graph(self, **kw):
        if self.gpu is None:
            raise ConfigError("no step has run in this workspace")
        return self.gpu.download_graph(**kw)


def _check_strategy(setup: StepSetup, strategy: Strategy):
    if strategy.kind != StrategyKind.kRbGpu:
        raise ConfigError(
            f"strategy {strategy.kind.value!r} is a CPU strategy of the reference library; "
            "this package provides only 'rb_gpu'")
    if setup.routing == Routing.kMfd and not setup.mfd_exponent > 0.0:
        raise ConfigError("mfd_exponent must be > 0")
    if setup.order == OrderKind.kStack:
        raise ConfigError("rb_gpu uses the breadth-first queue order")


def strategy_step(elev: np.ndarray, grid: GridGraph, params: SimParams, setup: StepSetup,
                  strategy: Strategy, ws: SimWorkspace, instr=None) -> StepDiagnostics:
    """lem::strategy_step for StrategyKind::kRbGpu: one timestep of ``elev`` in place."""
    _check_strategy(setup, strategy)
    params.validate()
    if instr is not None:
        raise ConfigError("StepInstrumentation is not supported by rb_gpu")
    if elev.shape != (grid.height, grid.width) or elev.dtype != np.float64 or not elev.flags.c_contiguous:
        raise ConfigError("elev must be a C-contiguous float64 array of shape (height, width)")
    ctx = ws.ensure(grid, params, strategy.device, setup)
    return ctx.step_host(elev)


class FillMode(enum.IntEnum):
    """lem::FillMode (depressions.hpp:8-12)."""

    kOff = 0
    kExact = 1
    kEpsilonAscending = 2


@dataclass
class FillOptions:
    """lem::FillOptions (depressions.hpp:14-19)."""

    mode: FillMode = FillMode.kOff
    epsilon_increment: float = 1e-8


def priority_flood_fill(elev: np.ndarray, opts: Optional[FillOptions] = None) -> np.ndarray:
    """lem::priority_flood_fill (depressions.cpp:26-68), computed on the device
    (lemgpu_fill: tile relaxation to the flood's fixed point, bit-identical)."""
    opts = opts or FillOptions()
    a = np.ascontiguousarray(elev, dtype=np.float64)
    if opts.mode == FillMode.kOff:
        return a.copy()
    ctx = DeviceContext(a.shape[-1], a.shape[-2], SimParams())
    try:
        ctx.upload(a)
        ctx.fill(opts)
        return ctx.download()
    finally:
        ctx.close()


@dataclass
class RunConfig:
    """lem::RunConfig subset that the step consumes (config.hpp:55-76)."""

    width: int = 500
    height: int = 500
    seed: int = 42
    timesteps: int = 120
    strategy: Strategy = field(default_factory=Strategy)
    params: SimParams = field(default_factory=SimParams)
    connectivity: int = 8
    routing: Routing = Routing.kD8
    mfd_exponent: float = 1.0
    fill: FillOptions = field(default_factory=FillOptions)

    def validate(self):
        """RunConfig::validate (config.cpp:155-173), step-relevant part."""
        if self.width < 3 or self.height < 3:
            raise ConfigError("width and height must be >= 3")
        if self.width * self.height > 0xFFFFFFFF:
            raise ConfigError("grid exceeds 2^32-1 cells")
        self.params.validate()
        Neighborhood.make(self.connectivity)
        if not self.mfd_exponent > 0.0:
            raise ConfigError("mfd_exponent must be > 0")
        if self.fill.mode == FillMode.kEpsilonAscending and not self.fill.epsilon_increment > 0.0:
            raise ConfigError("fill_epsilon must be > 0 for epsilon_ascending fill")


@dataclass
class RunResult:
    """lem::RunResult (scheduler.hpp:43-52)."""

    elevation: np.ndarray
    per_step: List[StepDiagnostics]
    phase_totals: List[float]
    newton_iters: int
    interior_noflow_last: int


def generate_terrain(width: int, height: int, seed: int = 42) -> np.ndarray:
    """lem::generate_terrain (terrain.cpp:19-31), computed on the device."""
    ctx = DeviceContext(width, height, SimParams())
    try:
        ctx.generate_terrain([seed])
        return ctx.download()
    finally:
        ctx.close()


def run_simulation(initial, cfg: Optional[RunConfig] = None,
                   on_step: Optional[Callable[[int, np.ndarray, StepDiagnostics], None]] = None) -> RunResult:
    """lem::run_simulation (scheduler.cpp:466-507).

    ``run_simulation(initial, cfg)`` or ``run_simulation(cfg)`` (terrain made on
    the device).  The elevation stays device-resident across steps; it is
    downloaded per step only when ``on_step`` is given (as the reference's
    callback needs the raster)."""
    if cfg is None:
        cfg, initial = initial, None
    cfg.validate()
    _check_strategy(StepSetup(routing=cfg.routing, mfd_exponent=cfg.mfd_exponent), cfg.strategy)
    ctx = DeviceContext(cfg.width, cfg.height, cfg.params, cfg.connectivity, cfg.strategy.device,
                        options={"phase_clocks": 1})  # RunResult::phase_totals
    try:
        if cfg.routing == Routing.kMfd:
            ctx.set_routing(cfg.routing, cfg.mfd_exponent)
        if initial is None:  # generate_terrain + optional depression fill (scheduler.cpp:503-506)
            ctx.generate_terrain([cfg.seed])
            ctx.fill(cfg.fill)
        else:
            a = np.asarray(initial, dtype=np.float64)
            if a.shape != (cfg.height, cfg.width):
                raise ConfigError(
                    f"initial raster is {a.shape[1]}x{a.shape[0]} but config says {cfg.width}x{cfg.height}")
            ctx.upload(a)
        per_step: List[StepDiagnostics] = []
        if on_step is None:
            per_step = ctx.step(cfg.timesteps) if cfg.timesteps else []
        else:
            buf = np.empty((cfg.height, cfg.width), np.float64)
            for s in range(1, cfg.timesteps + 1):
                d = ctx.step(1)[0]
                ctx.download(buf)
                on_step(s, buf, d)
                per_step.append(d)
        elev = ctx.download()
    finally:
        ctx.close()
    totals = [sum(d.seconds[i] for d in per_step) for i in range(6)]
    return RunResult(elev, per_step, totals, sum(d.newton_iters for d in per_step),
                     per_step[-1].interior_noflow if per_step else 0)
