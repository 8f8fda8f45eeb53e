"""Host-compiled checks of device logic that must be exact (no GPU needed)."""
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_receiver_division_skipping_is_exact(tmp_path):
    """receiver_code<8> == the reference's steepest_receiver loop on 2M random +
    adversarial drop vectors (ties, one-ulp neighbours, subnormals)."""
    exe = tmp_path / "test_receiver_code"
    subprocess.run(["/usr/local/cuda/bin/nvcc", "-std=c++17", "-O2", "-I", str(ROOT / "include"),
                    "-gencode", "arch=compute_100a,code=sm_100a", "-Xcompiler", "-ffp-contract=off",
                    "--fmad=false", "-o", str(exe), str(ROOT / "tests/native/test_receiver_code.cu")], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout
    assert "0 mismatches" in out.stdout


def test_division_from_table_reciprocal_is_exact(tmp_path):
    """div_rn_recip (Markstein correction from the host-rounded reciprocal of
    the Newton slope) == IEEE a / b on 1.6e8 random, table-shaped and
    near-midpoint operands."""
    exe = tmp_path / "test_div_recip"
    subprocess.run(["/usr/local/cuda/bin/nvcc", "-std=c++17", "-O2", "-I", str(ROOT / "include"),
                    "-gencode", "arch=compute_100a,code=sm_100a", "-Xcompiler", "-ffp-contract=off",
                    "--fmad=false", "-o", str(exe), str(ROOT / "tests/native/test_div_recip.cu")], check=True)
    out = subprocess.run([str(exe), "160000000"], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout
    assert " 0 mismatches" in out.stdout


def _build_glibc_pow_test(tmp_path):
    exe = tmp_path / "test_glibc_pow"
    subprocess.run(["/usr/bin/g++", "-std=c++17", "-O2", "-ffp-contract=off",
                    "-I", str(ROOT / "paper_1803_02977_b200" / "csrc"), "-o", str(exe),
                    str(ROOT / "tests/native/test_glibc_pow.cpp"), "-lm"], check=True)
    return exe


def _cpu_has_fma_avx2():
    flags = Path("/proc/cpuinfo").read_text().split()
    return "fma" in flags and "avx2" in flags


def test_glibc_pow_restatement_matches_host_libm(tmp_path):
    """glibc_pow.cuh (the device pow) == the host libm's pow, bit for bit, on
    2e7 inputs of every regime (drainage areas^m, Newton differences^n,
    random bit patterns, specials), for the variant this CPU's ifunc selects;
    plus the identities pow(x,1) == x and pow(x,0) == 1 on 5e6 inputs."""
    exe = _build_glibc_pow_test(tmp_path)
    variant = "fma" if _cpu_has_fma_avx2() else "sse2"
    out = subprocess.run([str(exe), variant, "20000000"], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout
    assert " 0 mismatches" in out.stdout and " 0 failures" in out.stdout


def test_glibc_pow_sse2_restatement_matches_masked_libm(tmp_path):
    """With FMA/AVX2 masked (GLIBC_TUNABLES), glibc's ifunc selects __pow_sse2;
    glibc_pow<false> must equal it bit for bit too -- and lemgpu_pow_variant
    must detect the switch (the context then runs the sse2 restatement)."""
    import os
    exe = _build_glibc_pow_test(tmp_path)
    env = dict(os.environ, GLIBC_TUNABLES="glibc.cpu.hwcaps=-AVX2,-FMA")
    out = subprocess.run([str(exe), "sse2", "4000000"], capture_output=True, text=True, env=env)
    assert out.returncode == 0, out.stdout
    assert " 0 mismatches" in out.stdout
    if _cpu_has_fma_avx2():  # the two variants really differ: the fma restatement fails here
        out = subprocess.run([str(exe), "fma", "400000"], capture_output=True, text=True, env=env)
        assert out.returncode == 1
    probe = ("import sys; sys.path.insert(0, %r); from paper_1803_02977_b200 import _abi; "
             "print(_abi.lib().lemgpu_pow_variant(None))" % str(ROOT))
    v = subprocess.run([sys.executable, "-c", probe], capture_output=True, text=True, env=env)
    assert v.stdout.strip() == "0", v.stdout + v.stderr
    v = subprocess.run([sys.executable, "-c", probe], capture_output=True, text=True)
    assert v.stdout.strip() == ("1" if _cpu_has_fma_avx2() else "0"), v.stdout + v.stderr
