"""C-ABI boundary checks that need no GPU: the in-tree sm_100a library loads,
exports exactly what include/lemgpu.h declares, validates parameters like
SimParams::validate, and fails loudly (no CPU fallback) without a device."""
import ctypes as C
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "lemgpu.h"


def _declared():
    txt = HEADER.read_text()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(lemgpu_[a-z_0-9]+)\s*\(", txt)))


def test_library_loads_and_exports_every_declared_symbol():
    from paper_1803_02977_b200 import _abi

    L = _abi.lib()
    declared = _declared()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(L, name), name
    assert sorted(_abi.exported_symbols()) == declared
    out = subprocess.run(["nm", "-D", "--defined-only", str(_abi.LIB_PATH)], capture_output=True, text=True).stdout
    exported = sorted(set(re.findall(r"\bT (lemgpu_\w+)", out)))
    assert exported == declared
    assert L.lemgpu_abi_version() == _abi.ABI_VERSION


def test_library_is_sm100a():
    from paper_1803_02977_b200 import _abi

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(_abi.LIB_PATH)],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_struct_layouts_match_header():
    from paper_1803_02977_b200 import _abi

    src = r"""
    #include <stdio.h>
    #include <stddef.h>
    #include "lemgpu.h"
    int main(void){ printf("%zu %zu %zu %zu %zu %zu %zu %zu\n", sizeof(lemgpu_params), sizeof(lemgpu_diag),
        sizeof(lemgpu_member), offsetof(lemgpu_diag, newton_iters), offsetof(lemgpu_params, connectivity),
        sizeof(lemgpu_options), offsetof(lemgpu_diag, kernel_s), offsetof(lemgpu_options, host_profile)); return 0; }
    """
    exe = Path("/tmp/lemgpu_layout")
    subprocess.run(["gcc", "-x", "c", "-I", str(ROOT / "include"), "-o", str(exe), "-"], input=src, text=True,
                   check=True)
    got = list(map(int, subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()))
    assert got == [C.sizeof(_abi.lemgpu_params), C.sizeof(_abi.lemgpu_diag), C.sizeof(_abi.lemgpu_member),
                   _abi.lemgpu_diag.newton_iters.offset, _abi.lemgpu_params.connectivity.offset,
                   C.sizeof(_abi.lemgpu_options), _abi.lemgpu_diag.kernel_s.offset,
                   _abi.lemgpu_options.host_profile.offset]


@pytest.mark.parametrize("field,value,msg", [
    ("dt", 0.0, "dt must be > 0"),
    ("epsilon", -1.0, "epsilon must be > 0"),
    ("K", -1.0, "K must be >= 0"),
    ("n_exp", 0.0, "n_exp must be > 0"),
    ("dx", 0.0, "cell spacing must be > 0"),
    ("max_newton_iters", 0, "max_newton_iters must be >= 1"),
    ("connectivity", 6, "hexagonal"),
    ("connectivity", 5, "connectivity must be 4 or 8"),
])
def test_create_validates_like_simparams(field, value, msg):
    from paper_1803_02977_b200 import _abi

    L = _abi.lib()
    p = _abi.lemgpu_params(2e-6, 0.5, 1.0, 2e-3, 1000.0, 1e-6, 1.0, 1.0, 100, 8)
    setattr(p, field, value)
    h = C.c_void_p()
    assert L.lemgpu_create(0, 10, 10, C.byref(p), C.byref(h)) == _abi.ECONFIG
    assert msg in L.lemgpu_error_message(None).decode()
    assert not h.value


def test_create_rejects_bad_geometry():
    from paper_1803_02977_b200 import _abi

    L = _abi.lib()
    p = _abi.lemgpu_params(2e-6, 0.5, 1.0, 2e-3, 1000.0, 1e-6, 1.0, 1.0, 100, 8)
    h = C.c_void_p()
    assert L.lemgpu_create(0, 2, 10, C.byref(p), C.byref(h)) == _abi.ECONFIG
    assert L.lemgpu_create(0, 70000, 70000, C.byref(p), C.byref(h)) == _abi.ECONFIG
    assert "2^32-1" in L.lemgpu_error_message(None).decode()


def test_no_silent_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_1803_02977_b200 import _abi

    L = _abi.lib()
    p = _abi.lemgpu_params(2e-6, 0.5, 1.0, 2e-3, 1000.0, 1e-6, 1.0, 1.0, 100, 8)
    h = C.c_void_p()
    assert L.lemgpu_create(0, 10, 10, C.byref(p), C.byref(h)) == _abi.ECUDA
    import paper_1803_02977_b200 as lem

    with pytest.raises(lem.Error):
        lem.run_simulation(lem.RunConfig(width=10, height=10, timesteps=1))
