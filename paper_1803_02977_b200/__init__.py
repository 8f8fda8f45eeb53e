"""B200-native (sm_100a) D8 landscape-evolution timestep (Barnes 2018).

The product is ``liblemgpu.so`` (CUDA kernels + the C-ABI of
``include/lemgpu.h``).  This package is the host-side mirror of the
reference's step API (``lem.py``) over that C-ABI (``_abi.py``).
"""
from . import _abi
from .lem import (  # noqa: F401
    ConfigError,
    ConvergenceError,
    DeviceContext,
    Error,
    FillMode,
    FillOptions,
    GridGraph,
    Neighborhood,
    NoFlow,
    OrderKind,
    Routing,
    RunConfig,
    RunResult,
    SimParams,
    SimWorkspace,
    StepDiagnostics,
    StepSetup,
    Strategy,
    StrategyKind,
    StructureError,
    generate_terrain,
    priority_flood_fill,
    run_simulation,
    strategy_step,
)

__all__ = [n for n in dir() if not n.startswith("_")]
