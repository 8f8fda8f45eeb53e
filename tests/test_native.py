"""Host-compiled checks of device logic that must be exact (no GPU needed)."""
import subprocess
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
