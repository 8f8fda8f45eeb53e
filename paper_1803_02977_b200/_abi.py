"""ctypes binding of the C-ABI in include/lemgpu.h.

This is the Python-side equivalent of the binding a maintainer would add to
the reference.  It loads the in-tree sm_100a library
``liblemgpu.so`` and fails loudly when it is missing: there is no CPU
fallback anywhere in this package.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
LIB_PATH = PKG_DIR / "liblemgpu.so"

ABI_VERSION = 3
NOFLOW = 0xFFFFFFFF

OK, ECONFIG, ESTRUCTURE, ECONVERGENCE, ECUDA, EOTHER = range(6)


class lemgpu_params(C.Structure):
    """POD mirror of lem::SimParams (proj/include/lem/erosion.hpp:15-25)."""

    _fields_ = [
        ("K", C.c_double),
        ("m_exp", C.c_double),
        ("n_exp", C.c_double),
        ("uplift_rate", C.c_double),
        ("dt", C.c_double),
        ("epsilon", C.c_double),
        ("dx", C.c_double),
        ("dy", C.c_double),
        ("max_newton_iters", C.c_int32),
        ("connectivity", C.c_int32),
    ]


class lemgpu_member(C.Structure):
    _fields_ = [("K", C.c_double), ("m_exp", C.c_double)]


class lemgpu_diag(C.Structure):
    """Mirror of lem::StepDiagnostics (proj/include/lem/simulation.hpp:34-40)."""

    _fields_ = [
        ("seconds", C.c_double * 6),
        ("newton_iters", C.c_uint64),
        ("interior_noflow", C.c_uint32),
        ("nlevels", C.c_uint32),
        ("lut_misses", C.c_uint32),
        ("status", C.c_uint32),
        ("err_cell", C.c_uint32),
        ("escaped_trees", C.c_uint32),
        ("kernel_s", C.c_double * 4),
        ("escaped_cells", C.c_uint32),
        ("mfd_passes", C.c_uint32),
    ]


class lemgpu_options(C.Structure):
    """Schedule / tuning / test knobs (include/lemgpu.h); zero = defaults."""

    _fields_ = [(n, C.c_int32) for n in ("global_path", "force_escape", "force_deep", "eager", "no_tma", "no_narrow",
                                         "no_esc_small", "pipe", "pipe_unchained")] + \
               [(n, C.c_uint32) for n in ("tile_grid", "esc_grid", "esc_small_grid", "pipe_tile_grid", "lut_entries",
                                          "host_bands", "patch_cap")] + \
               [("host_profile", C.c_int32), ("esc_forest", C.c_int32), ("mfd_levels", C.c_int32), ("phase_clocks", C.c_int32)]


# Every symbol include/lemgpu.h declares, with its ctypes signature.
_P = C.c_void_p
_SIGS = {
    "lemgpu_abi_version": (C.c_uint32, []),
    "lemgpu_create": (C.c_int, [C.c_int, C.c_uint32, C.c_uint32, C.POINTER(lemgpu_params), C.POINTER(_P)]),
    "lemgpu_create_ensemble": (
        C.c_int,
        [C.c_int, C.c_uint32, C.c_uint32, C.c_uint32, C.POINTER(lemgpu_params), C.POINTER(lemgpu_member), C.POINTER(_P)],
    ),
    "lemgpu_create_ex": (
        C.c_int,
        [C.c_int, C.c_uint32, C.c_uint32, C.c_uint32, C.POINTER(lemgpu_params), C.POINTER(lemgpu_member),
         C.POINTER(lemgpu_options), C.POINTER(_P)],
    ),
    "lemgpu_destroy": (None, [_P]),
    "lemgpu_upload_elev": (C.c_int, [_P, _P]),
    "lemgpu_download_elev": (C.c_int, [_P, _P]),
    "lemgpu_generate_terrain": (C.c_int, [_P, _P]),
    "lemgpu_fill": (C.c_int, [_P, C.c_int, C.c_double]),
    "lemgpu_step": (C.c_int, [_P, C.c_uint32, C.POINTER(lemgpu_diag)]),
    "lemgpu_step_async": (C.c_int, [_P, C.c_uint32]),
    "lemgpu_sync": (C.c_int, [_P, C.POINTER(lemgpu_diag), C.c_uint32, C.POINTER(C.c_uint32)]),
    "lemgpu_step_host": (C.c_int, [_P, _P, C.POINTER(lemgpu_diag)]),
    "lemgpu_snapshot_async": (C.c_int, [_P, _P, C.POINTER(lemgpu_diag)]),
    "lemgpu_snapshot_wait": (C.c_int, [_P]),
    "lemgpu_download_graph": (C.c_int, [_P, _P, _P, _P, _P, _P, C.POINTER(C.c_uint32), _P]),
    "lemgpu_set_routing": (C.c_int, [_P, C.c_int, C.c_double]),
    "lemgpu_download_mfd": (C.c_int, [_P, _P, _P, _P, C.POINTER(C.c_uint32)]),
    "lemgpu_member_stats_device": (C.c_int, [_P, _P]),
    "lemgpu_shard_members": (C.c_int, [C.c_uint32, C.c_int, C.c_int, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]),
    "lemgpu_create_ensemble_shard": (
        C.c_int,
        [C.c_int, C.c_uint32, C.c_uint32, C.c_uint32, C.c_int, C.c_int, C.POINTER(lemgpu_params),
         C.POINTER(lemgpu_member), C.c_uint32, C.POINTER(lemgpu_options), C.POINTER(_P)],
    ),
    "lemgpu_stats_enable": (C.c_int, [_P, C.c_uint32, C.c_uint32, C.c_uint32]),
    "lemgpu_nccl_unique_id": (C.c_int, [_P, C.c_uint32]),
    "lemgpu_stats_comm_init": (C.c_int, [_P, _P, C.c_uint32, C.c_int, C.c_int]),
    "lemgpu_stats_table": (C.c_int, [_P, _P]),
    "lemgpu_stats_table_device": (_P, [_P]),
    "lemgpu_error_message": (C.c_char_p, [_P]),
    "lemgpu_error_cell": (C.c_uint32, [_P]),
    "lemgpu_num_cells": (C.c_uint64, [_P]),
    "lemgpu_stream": (_P, [_P]),
    "lemgpu_device_bytes": (C.c_int, [_P, C.POINTER(C.c_uint64)]),
    "lemgpu_kernels_per_step": (C.c_uint32, [_P]),
    "lemgpu_pipeline_bands": (C.c_uint32, [_P]),
    "lemgpu_kernel_timing": (C.c_int, [_P, C.c_int]),
    "lemgpu_kernel_times": (C.c_int, [_P, C.POINTER(C.c_double), C.POINTER(C.c_uint32)]),
    "lemgpu_debug_timeline": (C.c_int, [_P, C.POINTER(C.c_uint64), C.c_uint32, C.POINTER(C.c_uint32)]),
    "lemgpu_debug_copy": (C.c_int, [_P, C.c_int, C.c_void_p, C.c_uint64]),
    "lemgpu_debug_tile_capture": (C.c_int, [_P, C.c_int]),
    "lemgpu_pow_variant": (C.c_int, [_P]),
    "lemgpu_debug_pow": (C.c_int, [C.c_int, C.c_int, _P, _P, _P, C.c_uint64]),
    "lemgpu_host_register": (C.c_int, [_P, C.c_size_t]),
    "lemgpu_host_unregister": (C.c_int, [_P]),
}

_lib = None


class ExtensionMissing(ImportError):
    pass


def lib():
    """The loaded sm_100a library (raises ExtensionMissing if it was not built)."""
    global _lib
    if _lib is None:
        path = Path(os.environ.get("LEMGPU_LIB", LIB_PATH))
        if not path.exists():
            raise ExtensionMissing(
                f"{path} is missing: build the CUDA extension first "
                "(`make lib` or `python -c 'import __graft_entry__ as g; g.build()'`). "
                "There is no CPU fallback."
            )
        L = C.CDLL(str(path))
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        if L.lemgpu_abi_version() != ABI_VERSION:
            raise ExtensionMissing(f"{path}: ABI version {L.lemgpu_abi_version()} != {ABI_VERSION}")
        _lib = L
    return _lib


def exported_symbols():
    return list(_SIGS)
