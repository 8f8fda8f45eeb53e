"""the reference's own CLI (`lem run|compare|bench`,
proj/tools/lem.cpp:143-250) with the rb_gpu strategy wired in by the
INTEGRATION.md patch (paper_1803_02977_b200/host/rb_gpu.patch, built out of
tree by oracle/Makefile `lem`).  `lem compare` is the reference's correctness
harness (byte-identical rasters across strategies, exit 3 on a mismatch);
`lem run` writes LEM1 snapshots (raster_io.cpp:30-39) through the StepCallback,
which the shim feeds from asynchronous device-to-host copies."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
LEM = ROOT / "oracle" / "_ref" / "lem"

pytestmark = pytest.mark.gpu


def lem(*args, timeout=900):
    if not LEM.exists():
        pytest.skip("oracle/_ref/lem not built (needs /root/reference at build time)")
    return subprocess.run([str(LEM), *args], capture_output=True, text=True, timeout=timeout)


@pytest.mark.parametrize("extra", [
    ["width=300", "height=200", "timesteps=20", "seed=5"],
    ["width=257", "height=131", "timesteps=15", "seed=6", "n_exp=2"],
    ["width=160", "height=120", "timesteps=10", "seed=7", "fill=epsilon_ascending"],
    ["width=150", "height=100", "timesteps=10", "seed=8", "connectivity=4", "dx=0.5", "dy=2"],
    ["width=1000", "height=1000", "timesteps=5", "seed=42", "workers=8"],
], ids=["d8", "n2", "filled", "d4-aniso", "1000sq"])
def test_lem_compare_rb_gpu_against_cpu_strategies(extra):
    out = lem("compare", "strategies=rb_serial,rb_private_queues,rb_gpu", *extra)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "3 strategies produced byte-identical rasters" in out.stdout


def test_lem_compare_detects_a_mismatch():
    # perturbing the first strategy's terrain must make rb_gpu differ: exit 3
    out = lem("compare", "strategies=rb_serial,rb_gpu", "width=64", "height=48", "timesteps=3",
              "debug_perturb_cell=1000", "debug_perturb_amount=0.5")
    assert out.returncode == 3, out.stdout + out.stderr
    assert "mismatch: rb_serial and rb_gpu" in out.stderr


def test_lem_compare_all_strategies_default():
    # no strategies= : all seven, rb_gpu included (kAllStrategies)
    out = lem("compare", "width=120", "height=90", "timesteps=6", "workers=4")
    assert out.returncode == 0, out.stdout + out.stderr
    assert "7 strategies produced byte-identical rasters" in out.stdout


def test_lem_run_snapshots_byte_identical(tmp_path):
    outs = {}
    for strat in ("rb_serial", "rb_gpu"):
        d = tmp_path / strat
        d.mkdir()
        r = lem("run", f"strategy={strat}", "width=200", "height=170", "timesteps=30", "seed=9",
                "snapshot_interval=10", f"output={d / 'final.lem'}")
        assert r.returncode == 0, r.stdout + r.stderr
        assert f"ran 30 steps ({strat}" in r.stdout
        outs[strat] = {p.name: p.read_bytes() for p in sorted(d.glob("*.lem"))}
    assert sorted(outs["rb_gpu"]) == ["final.000010.lem", "final.000020.lem", "final.000030.lem", "final.lem"]
    for name, data in outs["rb_serial"].items():
        assert data[:4] == b"LEM1"
        assert outs["rb_gpu"][name] == data, name


def test_lem_bench_prints_rb_gpu_phases():
    r = lem("bench", "strategies=rb_gpu", "sizes=300,500", "timesteps=5")
    assert r.returncode == 0, r.stdout + r.stderr
    rows = [l.split("\t") for l in r.stdout.strip().splitlines()[1:]]
    assert len(rows) == 2 * 6 and all(x[0] == "rb_gpu" for x in rows)
    for size in ("300", "500"):
        secs = [float(x[3]) for x in rows if x[1] == size]
        assert sum(secs) > 0 and all(s >= 0 for s in secs)  # lem::Phase split of the device time


@pytest.mark.parametrize("extra", [
    ["width=200", "height=150", "timesteps=8", "seed=3"],
    ["width=131", "height=97", "timesteps=5", "seed=4", "mfd_exponent=1.3", "connectivity=4"],
    ["width=120", "height=90", "timesteps=5", "seed=6", "fill=epsilon_ascending", "n_exp=2"],
], ids=["d8", "d4-e13", "filled-n2"])
def test_lem_compare_rb_gpu_mfd_routing(extra):
    # routing=mfd: rb_gpu against the reference's serial and level-parallel strategies
    out = lem("compare", "strategies=rb_serial,rb_par_all,rb_gpu", "routing=mfd", "workers=4", *extra)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "3 strategies produced byte-identical rasters" in out.stdout


def test_lem_rb_gpu_rejects_bad_mfd_exponent():
    r = lem("run", "strategy=rb_gpu", "routing=mfd", "mfd_exponent=0", "width=50", "height=40", "timesteps=2",
            "output=/tmp/lem_mfd_reject.lem")
    assert r.returncode != 0 and "mfd_exponent" in (r.stdout + r.stderr)
