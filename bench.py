#!/usr/bin/env python
"""Benchmark of the B200 D8 landscape-evolution step (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl mine|reference]
                    [--workload dem10000|dem1000|dem4000n2|dem1000fill|dem4000fill|dem1000mfd|dem10000mfd|ens64]

A "step" is one timestep (receivers, donors, level order, accumulation,
uplift + erosion) over the whole workload.  Default workload at N=1: the
10000x10000 random-noise DEM of BASELINE.json configs[1].  Default at N>1:
configs[4], the ensemble of 64 x 2000^2 members sharded over the ranks
(strong scaling: the same 64 members whatever N; its N=1 counterpart is
``--workload ens64``), each rank's members batched in one context, the
per-member statistics fused into the step and all-reduced by ONE
ncclAllReduce captured in the step's CUDA graph.  ``--workload dem10000`` at
N>1 runs one independent 10000^2 replica per rank ("replicas only": one DEM
does not shard) -- weak scaling.

Rank 0 prints one JSON line.  ``value`` is device-resident throughput
(inputs in HBM), ``e2e`` is the same metric through the C-ABI's
strategy_step entry (lemgpu_step_host) with pinned host buffers copied in and
out every step.  ``--impl reference`` times the unmodified reference CPU
implementation (oracle/_ref/liblemref.so) on the host cores instead.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "cell-steps/s, 10000² DEM, 1 GPU; ensemble cell-steps/s at 1/2/4/8 B200"
UNIT = "cell-steps/s"
PAPER_P100 = 1e8 * 120 / 70.0  # RB+GPU 10000^2 x 120 steps in 70 s on one P100
# Algorithmic bytes per cell-step: receivers 12 + donors 5 + order 9 + accumulation 21 +
# uplift/erosion 40 = 87.  k_recv does receivers + donors (17 B/cell); k_tiles does order,
# accumulation, uplift and erosion (70 B/cell) for the cells it finishes, moving only ~18 B/cell
# (h in 8, h out 8, receiver code 1, code bit planes 0.5) -- the 'traffic' key, from ncu.
B_STEP = 87
B_RECV = 17
B_TILES = 70
B_TILES_MIN = 18
# MFD routing (not in SURVEY 8(d); same counting rule, the reference's MFD work): graph 17 (read h 8,
# write lower mask 1 + weight sum 8) + plan 9 (read mask 1, write order 4 + level 4) + accumulation 37
# (read order 4, h 8, mask 1, donors' weight sums 8 and A 8, write A 8) = 63 B/cell on top of the D8
# step's 87 (the device builds no plan in the step: k_mfd_tiles finishes cells in dependency order)
B_MFD = 63
WORKLOADS = {
    "dem10000": dict(w=10000, h=10000, members=1, n_exp=1.0,
                     desc="10000x10000 random-noise DEM, D8, m=0.5 n=1, fixed-perimeter base level, seed 42 (configs[1])"),
    "dem1000": dict(w=1000, h=1000, members=1, n_exp=1.0, desc="1000x1000 random-noise DEM, D8, n=1 (configs[0]; L2-resident)"),
    "dem4000n2": dict(w=4000, h=4000, members=1, n_exp=2.0, desc="4000x4000 random-noise DEM, D8, n=2 Newton (configs[2])"),
    "dem1000fill": dict(w=1000, h=1000, members=1, n_exp=1.0, fill=2,
                        desc="1000x1000 random-noise DEM, Priority-Flood epsilon-filled (1e-8), D8, n=1: "
                             "the deep-level regime (SURVEY 8(f) rank 1)"),
    "dem4000fill": dict(w=4000, h=4000, members=1, n_exp=1.0, fill=2,
                        desc="4000x4000 random-noise DEM, Priority-Flood epsilon-filled (1e-8), D8, n=1: "
                             "the deep-level regime (SURVEY 8(f) rank 1)"),
    "dem1000mfd": dict(w=1000, h=1000, members=1, n_exp=1.0, routing=1,
                       desc="1000x1000 random-noise DEM, D8 erosion fed by the MFD drainage area (routing=mfd, "
                            "mfd_exponent 1), n=1 (SURVEY 8(f) rank 3)"),
    "dem10000mfd": dict(w=10000, h=10000, members=1, n_exp=1.0, routing=1,
                        desc="10000x10000 random-noise DEM, D8 erosion fed by the MFD drainage area (routing=mfd, "
                             "mfd_exponent 1), n=1 (SURVEY 8(f) rank 3)"),
    "ens64": dict(w=2000, h=2000, members=64, n_exp=1.0,
                  desc="ensemble of 64 x 2000^2 DEMs, seeds 1000+i, K_i=1e-6(1+i%8), m_i=0.35+0.05*floor(i/8) (configs[4])"),
}


def arm_config(workload, world):
    """The `config` both arms print (identical keys and values for the same
    workload and world size, so the driver can match the two lines)."""
    wl = WORKLOADS[workload]
    return {"workload": wl["desc"] + (" -- one independent replica per GPU" if (world > 1 and wl["members"] == 1) else ""),
            "grid": [wl["w"], wl["h"]], "members": wl["members"] * (world if wl["members"] == 1 else 1),
            "params": "K=2e-6 m=0.5 n=%g u=2e-3 dt=1000 eps=1e-6 D8" % wl["n_exp"]
                      + (" routing=mfd mfd_exponent=1" if wl.get("routing") else "")
                      + (" (per-member K, m)" if wl["members"] > 1 else ""),
            "fill": "epsilon_ascending 1e-8" if wl.get("fill") else "off"}


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def host_threads():
    """All host cores this process may use (torchrun sets OMP_NUM_THREADS=1, so
    the OpenMP default is not used: the reference's strategies take an explicit
    worker count, scheduler.cpp:365)."""
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            j = json.loads(p.read_text())
            return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
        except Exception:
            pass
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """NVML sampling of SM clock + throttle reasons during the timed region."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks_setting", 0x10: "sync_boost"}

    def __init__(self, device_index: int, period=0.005):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self.period = period
        self._stop = threading.Event()
        try:
            import pynvml as N

            N.nvmlInit()
            self.N = N
            self.h = N.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM)
        except Exception as e:  # pragma: no cover - no NVML
            self.N = None
            self.err = str(e)
        self.t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.N.nvmlDeviceGetClockInfo(self.h, self.N.NVML_CLOCK_SM))
                r = self.N.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.N is not None:
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.N is not None:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def member_table(workload, rank, world):
    """Member ids / seeds / (K, m) owned by this rank (paper_1803_02977_b200.ensemble)."""
    from paper_1803_02977_b200 import ensemble

    wl = WORKLOADS[workload]
    if wl["members"] == 1:
        # replicas only: one independent 10000^2 realisation per rank
        return [rank], [42 + rank], [(2e-6, 0.5)], world
    M = wl["members"]
    ids = ensemble.member_ids(M, world, rank)
    ps = [ensemble.member_params(i) for i in ids]
    return ids, [p[0] for p in ps], [(p[1], p[2]) for p in ps], M


def traffic_from_profiles(workload):
    """dram bytes per launch of the dominant kernel from the committed ncu summary."""
    for p in sorted((ROOT / "profiles").glob("ncu_summary_r*.json"), reverse=True):
        try:
            j = json.loads(p.read_text())
        except Exception:
            continue
        if j.get("workload") == workload:
            return j.get("kernels", {}), p.name
    return {}, None


def ref_strategy(wl):
    """The reference's fastest strategy for the workload: rb_private_queues, or
    rb_par_all under MFD routing (private queues reject it, scheduler.cpp:413-416)."""
    return "rb_par_all" if wl.get("routing") else "rb_private_queues"


def _ens_member_worker(args):
    """One ensemble member on one host core: the reference's rb_serial steps
    (test-infrastructure checker, CPU baseline only)."""
    w, h, i, steps = args
    sys.path.insert(0, str(ROOT / "tests"))
    from _oracle import RefLib, make_params  # test-infrastructure checker
    from paper_1803_02977_b200 import ensemble

    seed, K, m = ensemble.member_params(i)
    secs, _ = RefLib.get().bench(w, h, steps, warmup=1, strategy="rb_serial", workers=1, seed=seed,
                                 params=make_params(K=K, m_exp=m))
    return float(np.median(secs))


def cpu_ensemble_reference(w, h, members, steps, threads):
    """The ensemble on the host as SURVEY 8(d) config 5 prescribes: one
    single-thread rb_serial run per core over distinct members (their own
    seed, K, m), all concurrent; returns (ensemble seconds per step, sample)."""
    import multiprocessing as mpr

    n = min(threads, members)
    with mpr.get_context("spawn").Pool(n) as pool:
        per = pool.map(_ens_member_worker, [(w, h, i, steps) for i in range(n)])
    rate = sum(w * h / t for t in per)  # cell-steps/s of n concurrent members
    return w * h * members / rate, (f"{n} concurrent single-thread lem::strategy_step(rb_serial) runs, members "
                                    f"0..{n - 1} (own seed, K, m), {steps} timed steps each after 1 warm-up, "
                                    f"{w}x{h}; the {members}-member step extrapolated from their aggregate rate")


def cpu_baseline_reference(workload, budget_s=30.0):
    """The unmodified reference on this host's cores: lem::strategy_step with
    rb_private_queues (its fastest strategy), all OpenMP threads, a bounded
    number of steps of the same workload."""
    sys.path.insert(0, str(ROOT / "tests"))
    from _oracle import RefLib, make_params  # test-infrastructure checker

    wl = WORKLOADS[workload]
    w, h = wl["w"], wl["h"]
    if not RefLib.available():
        return None
    ref = RefLib.get()
    threads = host_threads()
    if wl["members"] > 1:
        per_step, sample = cpu_ensemble_reference(w, h, wl["members"], 3, threads)
        return {"value": w * h * wl["members"] / per_step, "unit": UNIT, "cores": min(threads, wl["members"]),
                "kind": "reference", "sample": sample + f": {per_step:.3f} s per ensemble step (oracle/_ref, -O2 "
                                                        "-ffp-contract=off)"}
    p = make_params(n_exp=wl["n_exp"])
    # bounded sample: ~budget_s of CPU work, at least 2 timed steps after 1 warm-up
    est = 3e-8 * w * h * 16 / max(threads, 1)  # ~3 s per 10000^2 step on 16 cores
    n = int(max(2, min(10, budget_s // max(est, 1e-3))))
    strat = ref_strategy(wl)
    samples, _ = ref.bench(w, h, n, warmup=1, strategy=strat, workers=threads, params=p,
                           fill=wl.get("fill", 0), routing=wl.get("routing", 0))
    per_step = float(np.median(samples))
    cells = w * h
    return {"value": cells / per_step, "unit": UNIT, "cores": threads, "kind": "reference",
            "sample": f"{len(samples)} lem::strategy_step({strat}, {threads} threads) timesteps of the "
                      f"{w}x{h} seed-42 DEM{' (priority_flood_fill first)' if wl.get('fill') else ''}, median wall time {per_step:.3f} s/step (oracle/_ref, -O2 -ffp-contract=off)"}


def run_reference_arm(args):
    rank = env_int("RANK", 0)
    if rank != 0:
        return 0
    sys.path.insert(0, str(ROOT / "tests"))
    from _oracle import RefLib, make_params

    wl = WORKLOADS[args.workload]
    w, h = wl["w"], wl["h"]
    cfg = arm_config(args.workload, env_int("WORLD_SIZE", 1))
    if not RefLib.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/liblemref.so not built"}))
        return 0
    ref = RefLib.get()
    threads = host_threads()
    p = make_params(n_exp=wl["n_exp"])
    members = wl["members"]
    if members > 1:
        # the ensemble: one single-thread rb_serial run per core over distinct
        # members, concurrently
        per_step, sample = cpu_ensemble_reference(w, h, members, 3, threads)
        value = w * h * members / per_step
        out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": 3, "warmup": 1,
               "ms_per_step": per_step * 1e3, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
               "dtype": "f64", "data": "synthetic (splitmix64 random-noise DEMs, lem::generate_terrain)", "config": cfg,
               "details": {"impl": "reference CPU: lem::strategy_step(rb_serial), one member per core, of the "
                                   "unmodified reference (oracle/_ref/liblemref.so)"},
               "impl": "reference",
               "cpu_baseline": {"value": value, "unit": UNIT, "cores": min(threads, members), "kind": "reference",
                                "sample": sample},
               "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(out))
        return 0
    # one "step" = one timestep of the whole workload
    t0 = time.time()
    fill = wl.get("fill", 0)
    strat, routing = ref_strategy(wl), wl.get("routing", 0)
    wsecs, _ = ref.bench(w, h, 1, warmup=0, strategy=strat, workers=threads, params=p, fill=fill, routing=routing)
    est = float(wsecs[0]) * members
    budget = 180.0
    k = args.steps
    warm = max(0, min(args.warmup - 1, int((budget / 4) // max(est, 1e-3))))
    k_run = int(max(1, min(k, (budget - (time.time() - t0)) // max(est, 1e-3) - warm)))
    secs, _ = ref.bench(w, h, k_run, warmup=warm, strategy=strat, workers=threads, params=p, fill=fill,
                        routing=routing)
    per_step = float(np.mean(secs)) * members
    value = w * h * members / per_step
    sample = (f"{k_run} timed + {warm + 1} warm-up lem::strategy_step({strat}, {threads} threads) on "
              f"{w}x{h}" + (f" (one member, scaled x{members})" if members > 1 else "") +
              (f"; steps capped from {k} to fit the time budget" if k_run < k else ""))
    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": k_run, "warmup": warm + 1,
           "ms_per_step": per_step * 1e3, "higher_is_better": True,
           "scaling": "weak" if wl["members"] == 1 else "strong", "vs_baseline": None,
           "dtype": "f64", "data": "synthetic (splitmix64 random-noise DEM, lem::generate_terrain)", "config": cfg,
           "details": {"impl": f"reference CPU: lem::strategy_step({strat}) of the unmodified reference "
                               "(oracle/_ref/liblemref.so)"},
           "impl": "reference",
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference", "sample": sample},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="mine", choices=["mine", "reference"])
    ap.add_argument("--workload", default=None, choices=sorted(WORKLOADS),
                    help="default: dem10000 (configs[1]) on 1 GPU, ens64 (configs[4], strong scaling) on N > 1")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--options", default=None,
                    help="JSON dict of lemgpu_options knobs (profiling / tuning), e.g. '{\"eager\": 1}'")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3  # timing rule: >= 3 warm-up steps
    if args.workload is None:
        args.workload = "dem10000" if max(args.gpus, env_int("WORLD_SIZE", 1)) == 1 else "ens64"
    if args.impl == "reference":
        return run_reference_arm(args)

    import torch
    import torch.distributed as dist

    import paper_1803_02977_b200 as lem

    rank, world, local = env_int("RANK", 0), env_int("WORLD_SIZE", 1), env_int("LOCAL_RANK", 0)
    # one process per GPU; LEMGPU_BENCH_BACKEND=gloo lets several ranks share
    # one device to exercise the multi-rank path on a single-GPU box
    backend = os.environ.get("LEMGPU_BENCH_BACKEND", "nccl")
    local = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    wl = WORKLOADS[args.workload]
    w, h = wl["w"], wl["h"]
    ids, seeds, km, members_total = member_table(args.workload, rank, world)
    M = len(ids)
    params = lem.SimParams(n_exp=wl["n_exp"])
    opts = json.loads(args.options) if args.options else {}
    if os.environ.get("LEMGPU_EAGER") == "1":  # profiling (tools/profile_round.sh): ncu cannot see graph kernel nodes
        opts["eager"] = 1
    ens = world > 1 or wl["members"] > 1
    from paper_1803_02977_b200 import ensemble

    if ens:
        # the product ensemble path: this rank's member range in one context,
        # per-member statistics fused into every step, ONE ncclAllReduce of the
        # table captured in the step graph; replicas of a single
        # DEM (--workload dem10000 at N > 1) are an ensemble of one member per rank
        if wl["members"] > 1:
            mfn, mtot = ensemble.member_params, wl["members"]
        else:
            mfn, mtot = (lambda i: (42 + i, 2e-6, 0.5)), world
        dens = ensemble.DeviceEnsemble(w, h, mtot, params, member_fn=mfn, device=local, rank=rank, world=world,
                                       options=opts or None, use_nccl=(backend == "nccl"))
        ctx = dens.ctx
        M = len(dens.ids)
        dens.generate_terrain()
    else:
        ctx = lem.DeviceContext(w, h, params, 8, device=local, members=M, options=opts or None)
        ctx.generate_terrain(seeds)
        if wl.get("routing"):
            ctx.set_routing(lem.Routing.kMfd, 1.0)
    fill_ms = None
    if wl.get("fill"):  # lem::priority_flood_fill on the device, once, before the timed steps
        torch.cuda.synchronize(local)
        tf = time.perf_counter()
        ctx.fill(mode=wl["fill"], epsilon=1e-8)
        fill_ms = (time.perf_counter() - tf) * 1e3
    cells = w * h * M
    ext = torch.cuda.ExternalStream(ctx.stream_ptr(), device=torch.device("cuda", local))

    def one_step():
        ctx.step_async(1)  # one graph launch: the step, the member statistics, their all-reduce

    # ---- warm-up
    for _ in range(args.warmup):
        one_step()
    ctx.sync()
    # no per-step timing events inside the timed region (an event pair around
    # every graph launch costs ~15 us a step, tools/probe_events.py): the step
    # time is the timed region's own events / K, the kernel spans come from the
    # steps' diagnostics (device %globaltimer stamps, lemgpu_diag::kernel_s)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    try:
        nvml_index = torch.cuda._get_nvml_device_index(local)
    except Exception:
        nvml_index = local
    with ClockSampler(nvml_index) as clk:
        start = torch.cuda.Event(enable_timing=True)
        end = torch.cuda.Event(enable_timing=True)
        start.record(ext)
        for _ in range(args.steps):
            one_step()
        end.record(ext)
        diags = ctx.sync()  # raises on any failing step
        torch.cuda.synchronize()
    ms = start.elapsed_time(end)
    timed = diags[-args.steps:]
    kt = {"launches": len(timed), "step": ms / args.steps * len(timed),
          "recv_donor": sum(d.kernel_seconds[0] for d in timed) * 1e3,
          "tiles": sum(d.kernel_seconds[1] for d in timed) * 1e3,
          "order": sum(d.kernel_seconds[2] for d in timed) * 1e3,
          "physics": sum(d.kernel_seconds[3] for d in timed) * 1e3}
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    total_cells = cells * world if wl["members"] == 1 else w * h * wl["members"]
    value = total_cells * args.steps / (ms / 1e3)

    # ---- end to end through the C-ABI strategy_step entry, pinned host buffers
    e2e = None
    if args.e2e_steps > 0:
        # page-locked host raster from cudaHostAlloc (torch pin_memory): its DMA
        # runs ~9 % faster than cudaHostRegister on a numpy array (tools/e2e_probe.py)
        host_t = torch.empty(cells, dtype=torch.float64).pin_memory()
        host = host_t.numpy()
        reg = False
        lem._abi.lib().lemgpu_download_elev(ctx.handle, host.ctypes.data)
        ctx.step_host(host)  # warm
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            ctx.step_host(host)
        dt = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([dt], dtype=torch.float64, device=f"cuda:{local}")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        if reg:
            lem._abi.lib().lemgpu_host_unregister(host.ctypes.data)
        # the PCIe floor of that contract: the raster up and a raster down,
        # concurrently on two streams, nothing else (pinned, same sizes)
        floor_ms = None
        try:
            dev_in = torch.empty(cells, dtype=torch.float64, device=f"cuda:{local}")
            dev_out = torch.empty(cells, dtype=torch.float64, device=f"cuda:{local}")
            host_out = torch.empty(cells, dtype=torch.float64).pin_memory()
            s_up, s_dn = torch.cuda.Stream(), torch.cuda.Stream()
            best = None
            for _ in range(3):
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                s_up.wait_event(e0)
                s_dn.wait_event(e0)
                with torch.cuda.stream(s_up):
                    dev_in.copy_(host_t, non_blocking=True)
                with torch.cuda.stream(s_dn):
                    host_out.copy_(dev_out, non_blocking=True)
                torch.cuda.current_stream().wait_stream(s_up)
                torch.cuda.current_stream().wait_stream(s_dn)
                e1.record()
                e1.synchronize()
                t = e0.elapsed_time(e1)
                best = t if best is None else min(best, t)
            floor_ms = best
            del dev_in, dev_out, host_out
        except RuntimeError:
            pass
        del host, host_t
        e2e = {"value": total_cells * args.e2e_steps / dt, "unit": UNIT, "h2d_bytes_per_step": cells * 8,
               "d2h_bytes_per_step": cells * 8, "steps": args.e2e_steps,
               "ms_per_step": dt / args.e2e_steps * 1e3,
               "pcie_copy_floor_ms": floor_ms,
               "frac_of_copy_floor": (floor_ms / (dt / args.e2e_steps * 1e3)) if floor_ms else None,
               "path": "lemgpu_step_host (strategy_step on a host raster: the whole raster H2D and D2H per call, "
                       "in bands overlapped with the step; escaped trees patched in)",
               "pinned": True, "host_alloc": "cudaHostAlloc (torch pin_memory)"}

    peak, peak_src = load_peaks()
    n_l = max(kt["launches"], 1)
    step_ms_ev = kt["step"] / n_l
    # kernel spans per step (device %globaltimer; lemgpu_diag::kernel_s)
    k1_ms, tiles_ms = kt["recv_donor"] / n_l, kt["tiles"] / n_l
    esc_ord_ms, esc_phys_ms = kt["order"] / n_l, kt["physics"] / n_l
    esc_cells = float(np.mean([d.escaped_cells for d in diags])) if diags else 0.0
    tile_cells = max(cells - esc_cells, 0.0)
    traffic_tbl, traffic_src = traffic_from_profiles(args.workload)
    pipelined = ctx.pipeline_bands() > 0
    # candidate kernels with their algorithmic bytes per step:
    # k_recv 17 B/cell (receivers 12 + donors 5) for every cell; k_tiles and the
    # escape path 70 B/cell (order 9 + accumulation 21 + uplift/erosion 40) for
    # the cells each finishes.  The dominant one is the longest.
    cands = []
    if wl.get("routing"):
        # MFD routing: the MFD area (k_mfd_tiles pass 0 + pass 1, k_mfd_tail rounds)
        # runs first, then the D8 tile path reads it; the MFD kernels' span is the
        # step minus the D8 kernels' spans
        mfd_ms = max(step_ms_ev - k1_ms - tiles_ms - esc_ord_ms - esc_phys_ms, 1e-9)
        cands.append(("k_mfd_tiles + k_mfd_tail (MFD area)", mfd_ms, B_MFD * cells, ("k_mfd_tiles", "k_mfd_tail")))
        cands.append(("k_tiles", tiles_ms, B_TILES * tile_cells, ("k_tiles",)))
        cands.append(("k_recv", k1_ms, B_RECV * cells, ("k_recv",)))
    elif pipelined:
        # tall rasters: k_recv and k_tiles run in interleaved bands (receiver band
        # b+1 beside tile band b): one unit, the step minus the escape kernels
        cands.append(("k_recv+k_tiles (pipelined bands)", max(step_ms_ev - esc_ord_ms - esc_phys_ms, 1e-9),
                      B_RECV * cells + B_TILES * tile_cells, ("k_recv", "k_tiles")))
    else:
        cands.append(("k_tiles", tiles_ms, B_TILES * tile_cells, ("k_tiles",)))
        cands.append(("k_recv", k1_ms, B_RECV * cells, ("k_recv",)))
    cands.append(("escape path (k_esc_small | k_esc_forest | k_esc_bfs + k_chunks/k_deep_coop)",
                  esc_ord_ms + esc_phys_ms, B_TILES * esc_cells,
                  ("k_esc_small", "k_esc_forest", "k_esc_bfs", "k_chunks", "k_deep_coop")))
    dom, dom_ms, dom_bytes, dom_kernels = max(cands, key=lambda c: c[1])
    achieved = dom_bytes / (dom_ms / 1e3) / 1e9 if dom_ms > 0 else None
    traffic = None
    if traffic_tbl and dom_kernels and all(k in traffic_tbl for k in dom_kernels[:1]):
        traffic = sum(traffic_tbl[k].get("dram_bytes_per_step", traffic_tbl[k]["dram_bytes_per_launch"])
                      for k in dom_kernels if k in traffic_tbl)
    per_gpu = value / world
    roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": (achieved / peak) if achieved else None, "traffic": traffic, "peak_source": peak_src,
                "alg_bytes_per_launch": dom_bytes,
                "alg_bytes_note": "SURVEY 8(d): k_recv 17 B/cell (receivers 12 + donors 5) over all cells; k_tiles / "
                                  "escape path 70 B/cell (order 9 + accumulation 21 + uplift/erosion 40) over the "
                                  "cells each finishes" +
                                  ("; pipelined: k_recv + k_tiles bands as one unit over their joint span "
                                   "(step events minus the escape kernels)" if pipelined else ""),
                "dominant_by": "longest measured kernel span per step (device %globaltimer)",
                "dram_frac": (traffic / (dom_ms / 1e3) / 1e9 / peak) if (traffic and dom_ms > 0) else None,
                "dram_frac_note": "ncu DRAM bytes of the same kernel(s) per launch / their span / peak: the bandwidth "
                                  "actually moved (the kernels are issue/latency-bound, see DESIGN.md)",
                "candidates_ms": {c[0]: round(c[1], 5) for c in cands},
                "escaped_cells_per_step": esc_cells,
                "kernel_ms": {"step(events)": step_ms_ev, "k_recv": k1_ms, "k_tiles": tiles_ms,
                              "escape:levels": esc_ord_ms, "escape:physics": esc_phys_ms},
                "timing_source": "step: CUDA events around the K timed graph launches on the context stream / K "
                                 "(no per-step events inside the timed region); kernel spans: device %globaltimer "
                                 "stamps taken by the kernels in those steps (lemgpu_diag::kernel_s)",
                "step": {"alg_bytes_per_cell": B_STEP, "achieved": per_gpu * B_STEP / 1e9,
                         "frac": per_gpu * B_STEP / 1e9 / peak},
                "traffic_source": traffic_src}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline_reference(args.workload)
        except Exception as e:  # report, never fail the bench
            cpu = {"value": None, "error": str(e)}
    # per step (one CUDA graph): k_recv and k_tiles (in bands for tall rasters),
    # k_esc_small, k_esc_bfs (cooperative, every escape level inside),
    # k_chunks, k_deep_coop (cooperative), [k_stats_reduce], k_finalize --
    # the kernel nodes of the step graph (the NCCL all-reduce is a library kernel)
    # the step graph's unconditional kernel nodes, plus the MFD tail rounds
    # (a WHILE node: mfd_passes - 2 per step); the escape kernels behind the IF
    # node after k_esc_small run only when it could not finish the escaped trees
    launches = args.steps * ctx.kernels_per_step() + sum(max(d.mfd_passes - 2, 0) for d in diags[-args.steps:])
    last = diags[-1] if diags else None
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "weak" if wl["members"] == 1 else "strong",
        "vs_baseline": value / PAPER_P100 if (args.workload == "dem10000" and world == 1) else None,
        "dtype": "f64", "data": "synthetic (splitmix64 random-noise DEM generated on device, bit-exact lem::generate_terrain)",
        "config": arm_config(args.workload, world),
        "details": {"members_per_gpu": M,
                   "parallelism": f"replicas{world}" if wl["members"] == 1 else f"members/{world}",
                   "collective": ("one ncclAllReduce per step of the [members, 4] statistics table, captured in the "
                                  "step's CUDA graph (lemgpu_stats_comm_init)" if (world > 1 and backend == "nccl")
                                  else None),
                   "member_stats": "fused into the receiver pass (lemgpu_stats_enable)" if ens else None,
                   "pow_variant": {1: "glibc __pow_fma", 0: "glibc __pow_sse2", -1: "NONE MATCHES"}[ctx.pow_variant()],
                   "l2": f"inputs larger than L2: {ctx.device_bytes() / 1e9:.1f} GB device state per GPU vs 126 MB L2, no flush",
                   "vs_baseline_ref": "paper RB+GPU on 1x P100: 10000^2 x 120 steps in 70 s (PAPER.md:14) = 1.71e8 cell-steps/s",
                   "nlevels_last_step": last.nlevels if last else None,
                   "phase_ms_last_step": ({k: round(v * 1e3, 4) for k, v in zip(
                       ("receivers", "donors", "order", "accumulation", "uplift", "erosion"), last.seconds)}
                       if last else None),
                   "lut_misses_last_step": last.lut_misses if last else None,
                   "escaped_trees_last_step": last.escaped_trees if last else None,
                   "newton_iters_last_step": last.newton_iters if last else None,
                   **({"mfd_passes_last_step": last.mfd_passes if last else None,
                       "mfd_path": "k_mfd_tiles pass 0 + pass 1 (shifted grid) + k_mfd_tail rounds, then the D8 "
                                   "tile path reading the MFD area"} if wl.get("routing") else {}),
                   **({"fill": "lem::priority_flood_fill epsilon_ascending 1e-8 on the device (lemgpu_fill), once, "
                               "untimed", "fill_ms": fill_ms} if fill_ms is not None else {})},
        "clocks": clk.summary(),
        "e2e": e2e,
        "gpu_launches": launches,
        "gpu_launches_note": "graph kernel nodes executed every step + MFD tail rounds; the escape kernels inside "
                             "the IF node (k_esc_forest, k_esc_bfs, k_chunks, k_deep_coop) are not counted",
        "roofline": roofline,
        "cpu_baseline": cpu,
    }
    if rank == 0:
        print(json.dumps(out))
    ctx.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
