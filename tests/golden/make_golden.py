"""Generate the golden fixtures under tests/golden/ from the REAL reference.

Runs the unmodified reference library (oracle/_ref/liblemref.so, compiled
from /root/reference/proj/src by oracle/Makefile) in this container and
writes:

  anchors.json        FNV-1a-64 fingerprints of full-size runs
                      (1000^2 / 10000^2, seed 42, defaults, fill=off)
  small_*.npz         complete step-1 outputs of small rasters (every array)
  fill_*.npz          lem::priority_flood_fill of small rasters (exact and
                      epsilon-ascending modes)
  mfd_*.npz           lem::simulate_step with StepSetup::routing = kMfd:
                      h after the step, the MFD drainage area and MFD plan

Usage:  python tests/golden/make_golden.py [--big] [--big120] [--fill-only]
  --big     add the 10000^2 step-1 anchors (~1 min, 6 GB RAM)
  --big120  add the 10000^2 120-step anchor (rb_private_queues, ~10 min)
  --mfd-only  only the mfd_*.npz fixtures
"""
from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
from _oracle import RefLib, fnv1a64, make_params  # noqa: E402

SMALL = [
    # name, w, h, seed, conn, params
    ("d8_17x13_s3", 17, 13, 3, 8, {}),
    ("d8_64x48_s42", 64, 48, 42, 8, {}),
    ("d8_3x3_s1", 3, 3, 1, 8, {}),
    ("d8_5x40_s9", 5, 40, 9, 8, {}),
    ("d4_30x22_s5", 30, 22, 5, 4, {}),
    ("d8_aniso_33x21_s7", 33, 21, 7, 8, {"dx": 0.5, "dy": 2.0}),
    ("d8_m035_K9_40x40_s11", 40, 40, 11, 8, {"m_exp": 0.35, "K": 9e-6}),
    ("d8_n2_48x36_s13", 48, 36, 13, 8, {"n_exp": 2.0}),
]


def anchors_for(ref: RefLib, n: int, steps: int, strategy: str, workers: int):
    e = ref.terrain(n, n, 42)
    out = {"terrain": fnv1a64(e)}
    e1 = e.copy()
    s1 = ref.step(e1)
    assert s1["status"] == 0
    out["step1"] = {
        "rec": fnv1a64(s1["rec"]), "dnum": fnv1a64(s1["dnum"]), "order": fnv1a64(s1["order"]),
        "A": fnv1a64(s1["A"]), "h": fnv1a64(e1), "levels": [int(x) for x in s1["levels"]],
        "interior_noflow": int(s1["interior_noflow"]), "newton_iters": int(s1["newton_iters"]),
        "maxA": float(s1["A"].max()),
    }
    if steps:
        t0 = time.time()
        rc, newton, _ = ref.run(e, steps, strategy=strategy, workers=workers)
        assert rc == 0
        out[f"step{steps}"] = {
            "h": fnv1a64(e), "newton_total": int(newton), "min": float(e.min()), "max": float(e.max()),
            "mean": float(e.mean()), "strategy": strategy, "workers": workers, "seconds": time.time() - t0,
        }
    return out


FILL = [
    # w, h, seed, mode (1 exact, 2 epsilon ascending), epsilon
    (100, 100, 1, 1, 1e-8), (100, 100, 1, 2, 1e-8), (100, 100, 2, 2, 1e-8), (100, 100, 3, 1, 1e-8),
    (257, 131, 7, 2, 1e-8), (257, 131, 7, 1, 1e-8), (70, 45, 9, 2, 1e-3), (3, 3, 1, 2, 1e-8),
]


def fill_goldens(ref: RefLib):
    for w, h, seed, mode, eps in FILL:
        e0 = ref.terrain(w, h, seed)
        f = ref.fill(e0, mode, eps)
        name = f"fill_{'exact' if mode == 1 else 'eps'}_{w}x{h}_s{seed}" + ("" if eps == 1e-8 else "_e3")
        np.savez_compressed(HERE / f"{name}.npz", w=w, h=h, seed=seed, mode=mode, eps=eps, h0=e0, f=f)


MFD = [
    # name, w, h, seed, conn, exponent, params
    ("d8_e1_40x30_s3", 40, 30, 3, 8, 1.0, {}),
    ("d8_e1_64x48_s42", 64, 48, 42, 8, 1.0, {}),
    ("d8_e11_33x29_s5", 33, 29, 5, 8, 1.1, {}),
    ("d8_e2_25x25_s2", 25, 25, 2, 8, 2.0, {}),
    ("d4_e1_30x22_s5", 30, 22, 5, 4, 1.0, {}),
    ("d8_aniso_e1_33x21_s7", 33, 21, 7, 8, 1.0, {"dx": 0.5, "dy": 2.0}),
    ("d8_n2_e1_48x36_s13", 48, 36, 13, 8, 1.0, {"n_exp": 2.0}),
]


def mfd_goldens(ref: RefLib):
    for name, w, h, seed, conn, ex, kw in MFD:
        p = make_params(**kw)
        e0 = ref.terrain(w, h, seed)
        e = e0.copy()
        s = ref.step_mfd(e, exponent=ex, conn=conn, params=p)
        assert s["status"] == 0, name
        np.savez_compressed(
            HERE / f"mfd_{name}.npz", w=w, h=h, seed=seed, conn=conn, exponent=ex, params=json.dumps(kw), h0=e0,
            h1=e, A=s["A"], mfd_order=s["mfd_order"], mfd_levels=s["mfd_levels"], newton_iters=s["newton_iters"])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true")
    ap.add_argument("--big120", action="store_true")
    ap.add_argument("--fill-only", action="store_true")
    ap.add_argument("--mfd-only", action="store_true")
    args = ap.parse_args()
    ref = RefLib.get()
    mfd_goldens(ref)
    if args.mfd_only:
        return
    fill_goldens(ref)
    if args.fill_only:
        return
    path = HERE / "anchors.json"
    anchors = json.loads(path.read_text()) if path.exists() else {}
    anchors["_about"] = ("FNV-1a-64 of raw little-endian arrays from the unmodified reference "
                         "(oracle/_ref/liblemref.so) in the build container; seed 42, default SimParams, D8, fill=off")
    anchors["1000"] = anchors_for(ref, 1000, 120, "rb_private_queues", ref.max_threads())
    if args.big or args.big120:
        anchors["10000"] = anchors_for(ref, 10000, 120 if args.big120 else 0, "rb_private_queues", ref.max_threads())
    path.write_text(json.dumps(anchors, indent=1, sort_keys=True) + "\n")

    for name, w, h, seed, conn, kw in SMALL:
        p = make_params(**kw)
        e0 = ref.terrain(w, h, seed)
        e = e0.copy()
        s = ref.step(e, conn=conn, params=p)
        assert s["status"] == 0, name
        np.savez_compressed(
            HERE / f"small_{name}.npz", w=w, h=h, seed=seed, conn=conn, params=json.dumps(kw), h0=e0, h1=e,
            rec=s["rec"], dnum=s["dnum"], donor=s["donor"], order=s["order"], levels=s["levels"], A=s["A"],
            newton_iters=s["newton_iters"], interior_noflow=s["interior_noflow"])
    print(json.dumps(anchors, indent=1))


if __name__ == "__main__":
    main()
