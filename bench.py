#!/usr/bin/env python
"""Benchmark of the TT-FV SWE hot path (one SSP-RK3 step = one unit).

Metric (BASELINE.json): TT-FV SWE steps/sec & equivalent cell-updates/sec at N=4096, with
the dominant kernel class's roofline fraction. Default workload: configs[3] (C4: nonlinear,
f=10, N=4096, WENO5 via TT-cross, tol 1e-10), the configuration the metric is quoted at —
see DESIGN.md §Measurement.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl ours|reference]

CPU legs: the oracle (restated reference, single thread) from the oracle's own step-5 state of
the metric's configuration (tests/golden/long/, the state at which the timed region starts
under --warmup 5). --impl reference times whole steps, measured end to end (minutes per
step at C4); our arm's cpu_baseline is a bounded 30 s sample of the same step, extrapolated by
the completed share of that step's rounding work when the step does not finish.

Under torchrun (N>1) every rank advances its own replica (the path does not shard,
DESIGN.md: "replicas only"); value = all ranks' steps / max-over-ranks device time.
"""
import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")  # before torch/CUDA init (see capi.py)

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "TT-FV SWE steps/sec & equiv. cell-updates/sec at N=4096; % HBM/FP64 roofline"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=None)
    p.add_argument("--warmup", type=int, default=None)
    p.add_argument("--config", default="C4")
    p.add_argument("--cpu-budget", type=float, default=30.0, help="seconds of oracle work per CPU sample")
    p.add_argument("--ref-budget", type=float, default=1.0,
                   help="reference arm: keep timing whole oracle steps until this many seconds have passed")
    p.add_argument("--n", type=int, default=0, help="override grid size (testing only)")
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--rep", default="tt", choices=["tt", "dense"],
                   help="tt: the TT path (the metric); dense: the device full-tensor DenseRep path on the same config")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--members", type=int, default=64, help="C5 ensemble size (all ranks)")
    p.add_argument("--member-threads", type=int, default=8, help="C5 members in flight per GPU")
    return p.parse_args()


DEFAULT_STEPS = {"C1": (100, 5), "C2": (100, 5), "C3": (20, 5), "C4": (20, 5), "C5": (2, 3)}


def make_spec(args):
    from paper_2408_03483_b200 import ics

    kw = {"n": args.n} if args.n else {}
    if args.config == "C5":
        spec = ics.config5_member(0, **kw)
        spec.name = "C5"
    else:
        spec = ics.CONFIGS[args.config](**kw)
    k, w = DEFAULT_STEPS.get(args.config, (5, 3))
    if args.steps is None:
        args.steps = k
    if args.warmup is None:
        args.warmup = w
    return spec


def round_work(trace):
    """SURVEY App. B rounding flops per trace row (columns m, n, r_in, k_out at 1..4)."""
    m, n, R, k = (trace[:, i].astype(float) for i in (1, 2, 3, 4))
    return 2 * n * R * R + 3 * m * R * R + 2 * (m + n) * R * k + 11 * R ** 3


def trace_path(spec):
    return os.path.join(ROOT, "profiles", f"step0_trace_{spec.name}_N{spec.n}.json")


def measured_traffic(spec):
    """DRAM bytes (read + write) per rounding of the rounding-class kernels, from the
    committed ncu pass over one step of this configuration (scripts/traffic.py), or None."""
    p = os.path.join(ROOT, "profiles", f"traffic_{spec.name}_N{spec.n}.json")
    if not os.path.exists(p):
        return None
    d = json.load(open(p))
    return {"bytes_per_rounding": d["round_class_dram_bytes"] / max(d["roundings"], 1), "source": d["source"]}


def workload(spec):
    models = ["linear", "nonlinear"]
    schemes = ["upwind3", "upwind5", "weno5"]
    return {"workload": f"{spec.name}: {models[spec.model]} SWE N={spec.n} {schemes[spec.scheme]} "
                        f"f={spec.f} tol={spec.tol:g} dt={spec.dt:.6g}, seeded IC ({spec.notes or 'separable'})",
            "N": spec.n, "tol": spec.tol, "dt": spec.dt, "model": models[spec.model],
            "scheme": schemes[spec.scheme]}


def dist_init():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist

        backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
        dist.init_process_group(backend=backend)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def allreduce_max(world, v, local):
    if world == 1:
        return v
    import torch
    import torch.distributed as dist

    dev = f"cuda:{local}" if torch.cuda.is_available() else "cpu"
    t = torch.tensor([v], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={index}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.f,
                                      stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        rows = [r.split(",") for r in open(self.f.name).read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm = [float(r[1]) for r in rows if len(r) >= 9 and r[1].strip().replace(".", "").isdigit()]
        if not sm:
            return None
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for k, name in enumerate(names):
                if len(r) > 5 + k and "Active" in r[5 + k] and "Not" not in r[5 + k]:
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": float(rows[0][2]), "samples": len(sm),
                "reasons": sorted(reasons)}


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        return {}


def fp64_peak_tflops(torch, dev):
    """cuBLAS DGEMM 8192^3 best-of-3 on this GPU (MEASURED_PEAKS.json has no fp64 entry)."""
    a = torch.randn(8192, 8192, dtype=torch.float64, device=dev)
    b = torch.randn(8192, 8192, dtype=torch.float64, device=dev)
    torch.matmul(a, b)
    torch.cuda.synchronize()
    best = 0.0
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b)
        e1.record()
        e1.synchronize()
        best = max(best, 2 * 8192 ** 3 / (e0.elapsed_time(e1) * 1e-3) / 1e12)
    del a, b
    torch.cuda.empty_cache()
    return best


SNAPSHOT_STEP = 5


def snapshot_path(spec):
    return os.path.join(ROOT, "tests", "golden", "long", f"{spec.name.lower()}_n{spec.n}.npz")


def oracle_snapshot(spec):
    """The oracle's own state after SNAPSHOT_STEP steps from the IC (tests/golden/make_long.py,
    committed for the metric's configuration), or None: the state both arms time from."""
    p = snapshot_path(spec)
    if not os.path.exists(p):
        return None
    d = np.load(p)
    if SNAPSHOT_STEP not in set(d["checkpoints"].tolist()):
        return None
    return [(d[f"ck_{SNAPSHOT_STEP}_{c}_x"], d[f"ck_{SNAPSHOT_STEP}_{c}_y"]) for c in range(3)]


def oracle_solver(spec):
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle

    pyoracle.build()
    cfg = pyoracle.CrossCfg.make(seed=1, max_rank=spec.cross_max_rank)
    s = pyoracle.Solver(spec.model, spec.scheme, spec.n, spec.g, spec.f, spec.H, spec.dt, spec.tol, cfg)
    snap = oracle_snapshot(spec)
    if snap is not None:
        s.set_state([pyoracle.TT.from_cores(cx, cy) for cx, cy in snap])
        start = f"from the oracle's own step-{SNAPSHOT_STEP} state ({os.path.relpath(snapshot_path(spec), ROOT)})"
    else:
        s.set_state([pyoracle.round_(pyoracle.TT.from_cores(cx, cy), spec.tol) for cx, cy in spec.ic])
        start = "from the IC"
    return s, start


def oracle_whole_steps(spec, budget):
    """Reference arm: whole oracle SSP-RK3 steps (at least one, more while the budget lasts),
    timed end to end with no extrapolation. Returns (steps/s, steps, seconds, description)."""
    s, start = oracle_solver(spec)
    done = 0
    t0 = time.perf_counter()
    while True:
        s.step(1)
        done += 1
        secs = time.perf_counter() - t0
        if secs >= budget:
            break
    desc = (f"{done} whole SSP-RK3 step(s) of {spec.name} N={spec.n} {start} in {secs:.1f} s, measured "
            "(no extrapolation), one host core, oracle (restated reference)")
    return done / secs, done, secs, desc


def oracle_sample(spec, budget, step_work=None):
    """cpu_baseline of our arm: a bounded sample (the default bench run must end within minutes).

    From the same start state as the reference arm, whole steps are timed when they finish
    inside the budget; otherwise the step is cut at the first rounding that starts after
    the deadline and the rate is the completed share of that step's rounding work
    (step_work = App. B flops of every rounding of the step, from the GPU's trace of the same
    step) over the elapsed time — labelled as such. Returns (steps/s, description)."""
    s, start = oracle_solver(spec)
    t0 = time.perf_counter()
    done, t_done = 0, 0.0
    while True:
        left = budget - (time.perf_counter() - t0)
        if done and left <= 0:
            break
        finished = s.step_sample(max(left, 1e-3))
        tr = s.trace()[0]
        if not finished:
            break
        done += 1
        t_done = time.perf_counter() - t0
    secs = t_done if done else time.perf_counter() - t0
    if done:
        return done / secs, (f"{done} whole SSP-RK3 step(s) of {spec.name} N={spec.n} {start} in {secs:.1f} s, "
                             "one host core, oracle (restated reference)")
    if step_work is None or len(tr) == 0:
        return None, "oracle did not finish a step within the budget and no step trace is available"
    w = round_work(tr).sum()
    frac = float(w / step_work.sum())
    return frac / secs, (f"bounded sample, extrapolated: first {len(tr)} of {len(step_work)} roundings of one "
                         f"SSP-RK3 step of {spec.name} N={spec.n} {start} ({100 * frac:.2f}% of that step's "
                         f"App.-B rounding work) in {secs:.1f} s, one host core, oracle (restated reference); "
                         "steps/s = work share / time (the reference arm times whole steps)")


def run_reference(args, world, rank):
    """--impl reference: the restated reference (the reference itself cannot be built here,
    DESIGN.md §3) on this host, whole steps from the oracle's own step-5 state of the
    metric's configuration — the state at which our arm's timed region starts under the
    driver's --warmup 5 — timed end to end. Under torchrun only rank 0 runs."""
    spec = make_spec(args)
    if rank != 0:
        return
    rate, done, secs, desc = oracle_whole_steps(spec, args.ref_budget)
    cfg = workload(spec)
    line = {"impl": "reference", "metric": METRIC, "value": rate, "unit": "steps/s", "n_gpus": args.gpus,
            "steps": done, "warmup": 0, "ms_per_step": 1e3 / rate, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": cfg,
            "cell_updates_per_s": rate * spec.n * spec.n,
            "cpu_baseline": {"value": rate, "unit": "steps/s", "cores": 1, "kind": "port",
                             "sample": desc + " (the reference itself is unbuildable here: no Eigen; its path "
                                              "is single-threaded)"},
            "e2e": {"value": rate, "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    if done < args.steps:
        line["steps_note"] = (f"{done} whole step(s) instead of --steps {args.steps}: one oracle step of this "
                              f"configuration takes {secs / done:.0f} s on one core")
    print(json.dumps(line), flush=True)


def run_ours(args, world, rank, local):
    import torch

    from paper_2408_03483_b200 import capi

    spec = make_spec(args)
    dev = torch.device(f"cuda:{local}")
    torch.cuda.set_device(dev)
    ctx = capi.Context(local)
    stream = torch.cuda.ExternalStream(ctx.stream, device=dev)
    cfg = capi.CrossCfg.make(seed=1, max_rank=spec.cross_max_rank)
    solver = capi.Solver(ctx, spec.model, spec.scheme, spec.n, spec.g, spec.f, spec.H, spec.dt, spec.tol, cfg)
    init = [ctx.round(ctx.tt(cx, cy), spec.tol) for cx, cy in spec.ic]
    solver.set_state(init)
    solver.set_tracing(False)
    for _ in range(args.warmup):
        solver.step(1)
    ctx.sync()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device=dev)  # 512 MiB > 126 MB L2

    snapshot = [t.cores() for t in solver.state()]  # the e2e leg replays the timed steps from here
    # the headline steps run exactly as a user's would: no per-rounding event timing
    # (its event syncs would add host round trips); the roofline pass below replays them
    ctx.time_rounds(False)
    launches0 = ctx.launches
    barrier(world)
    clocks = Clocks(local)
    total_ms = 0.0
    for _ in range(args.steps):
        flush.fill_(1.0)  # L2 flush between timed steps (not timed)
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        solver.step(1)
        e1.record(stream)
        e1.synchronize()
        total_ms += e0.elapsed_time(e1)
    clk = clocks.stop()
    launches = ctx.launches - launches0
    barrier(world)
    max_ms = allreduce_max(world, total_ms, local)
    value = world * args.steps / (max_ms * 1e-3)

    # End to end through the public C ABI with host buffers: every step uploads the
    # state cores from host memory, advances one step and reads the result back; the
    # same steps as the timed region (replayed from its starting state).
    ranks_timed = [t.rank for t in solver.state()]
    host = snapshot
    e2e_steps = max(1, min(args.steps, 50))
    h2d = d2h = 0
    e2e_ms = 0.0
    for _ in range(e2e_steps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(stream)
        tts = [ctx.tt(cx, cy) for cx, cy in host]
        h2d = sum(cx.nbytes + cy.nbytes for cx, cy in host)
        solver.set_state(tts)
        solver.step(1)
        host = [t.cores() for t in solver.state()]
        d2h = sum(cx.nbytes + cy.nbytes for cx, cy in host)
        e1.record(stream)
        e1.synchronize()
        e2e_ms += max(e0.elapsed_time(e1), (time.perf_counter() - t0) * 1e3)
    e2e_max = allreduce_max(world, e2e_ms, local)
    e2e_value = world * e2e_steps / (e2e_max * 1e-3)

    # Roofline pass: the same steps replayed from the snapshot with every rounding (group)
    # bracketed by CUDA events on the library's stream (achieved = App.-B work / event time)
    solver.set_state([ctx.tt(cx, cy) for cx, cy in snapshot])
    ctx.sync()
    ctx.time_rounds(True)
    ctx.round_stats(reset=True)
    roof_ms = 0.0
    for _ in range(args.steps):
        flush.fill_(1.0)
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        solver.step(1)
        e1.record(stream)
        e1.synchronize()
        roof_ms += e0.elapsed_time(e1)
    rs = ctx.round_stats(reset=True)
    ctx.time_rounds(False)

    # rounding trace of the step the CPU legs time (from the oracle's step-5 state when the
    # snapshot exists, else from the IC): the bounded cpu_baseline sample's work denominator
    ranks_final = ranks_timed
    snap = oracle_snapshot(spec)
    if snap is not None:
        solver.set_state([ctx.tt(cx, cy) for cx, cy in snap])
    else:
        solver.set_state([ctx.round(ctx.tt(cx, cy), spec.tol) for cx, cy in spec.ic])
    solver.set_tracing(True)
    solver.trace(clear=True)
    solver.step(1)
    tr0 = solver.trace()[0]
    step_work = round_work(tr0)
    if rank != 0:
        return
    if not args.n:
        os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
        json.dump({"config": spec.name, "N": spec.n, "columns": "step, m, n, r_in, k_out, crosses_before",
                   "start": f"oracle step-{SNAPSHOT_STEP} state" if snap is not None else "IC",
                   "trace": tr0.tolist()}, open(trace_path(spec), "w"))
    traffic = measured_traffic(spec)
    peaks = measured_peaks()
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    fp64 = fp64_peak_tflops(torch, dev)
    intensity = rs["flops"] / rs["bytes"] if rs["bytes"] else 0.0
    ridge = fp64 * 1e12 / (hbm * 1e9)
    if rs["ms"] > 0 and intensity < ridge:
        achieved = rs["bytes"] / (rs["ms"] * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                "traffic": traffic["bytes_per_rounding"] if traffic else None}
    else:
        achieved = rs["flops"] / (rs["ms"] * 1e-3) / 1e12 if rs["ms"] else 0.0
        # "tensor": the FP64 tensor-core (DMMA) roofline, i.e. the cuBLAS DGEMM rate measured in this run
        roof = {"bound": "tensor", "bound_detail": "fp64 tensor cores (DMMA; cuBLAS DGEMM rate)", "achieved": achieved,
                "peak": fp64, "unit": "TFLOP/s", "frac": achieved / fp64,
                "traffic": traffic["bytes_per_rounding"] if traffic else None}
    sk = ctx.sketch_stats()
    roof.update({"kernel": "round (sketched pre-compression on FP64 tensor-core GEMMs where R >> k, else CAQR of both "
                           "cores; cluster-QRCP-truncated Jacobi SVD; Q apply; tt.hpp:120-138)",
                 "sketched_roundings": sk["used"], "sketch_retries": sk["fallback"],
                 "launches_timed": rs["count"], "avg_launch_us": 1e3 * rs["ms"] / max(rs["count"], 1),
                 "share_of_step": rs["ms"] / roof_ms if roof_ms else None,
                 "timing": "separate replay of the timed steps with per-rounding CUDA events "
                           "(the headline steps run without them)",
                 "algorithmic": "SURVEY.md App. B per rounding: flops 2nR^2+3mR^2+2(m+n)Rk+11R^3, "
                                "bytes 8(m+n)(R+k), summed over the timed roundings (the work of the "
                                "reference's algorithm at the run's ranks; the sketched roundings execute fewer flops)",
                 "intensity_flop_per_byte": intensity, "fp64_peak_tflops_measured": fp64,
                 "algorithmic_bytes_per_rounding": rs["bytes"] / max(rs["count"], 1),
                 "traffic_source": traffic["source"] if traffic else None,
                 "peak_source": "MEASURED_PEAKS.json hbm_gbs" if roof["bound"] == "hbm"
                 else "cuBLAS DGEMM 8192^3 measured in this run"})
    cfgd = workload(spec)
    cfgd.update({"l2": "flushed (512 MiB write) between timed steps", "parallelism": f"replicas x{world}"})
    line = {"metric": METRIC, "value": value, "unit": "steps/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": max_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": cfgd,
            "cell_updates_per_s": value * spec.n * spec.n, "roofline": roof,
            "e2e": {"value": e2e_value, "unit": "steps/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "gpu_launches": launches, "clocks": clk,
            "ranks_final": ranks_final}
    if world == 1 and not args.no_cpu_baseline:
        rate, desc = oracle_sample(spec, args.cpu_budget, step_work)
        line["cpu_baseline"] = {"value": rate, "unit": "steps/s", "cores": 1, "kind": "port", "sample": desc}
    print(json.dumps(line), flush=True)


def run_dense(args, world, rank, local):
    """--rep dense: the same configuration on the device full-tensor path (DenseRep,
    ttsw_dense_*), the paper's TT-vs-full comparison on B200. The IC is the
    TT IC expanded to N x N. Roofline: HBM bound; algorithmic bytes per SSP-RK3 stage = the
    ghost copies, both axis passes over the ghosted fields (two for the nonlinear model: the
    dissipation speed pass and the flux pass), the F-hat writes and the combine pass."""
    import torch

    from paper_2408_03483_b200 import capi

    spec = make_spec(args)
    dev = torch.device(f"cuda:{local}")
    torch.cuda.set_device(dev)
    ctx = capi.Context(local)
    stream = torch.cuda.ExternalStream(ctx.stream, device=dev)
    s = capi.DenseSolver(ctx, spec.model, spec.scheme, spec.n, spec.g, spec.f, spec.H, spec.dt)
    s.set_state([cx @ cy for cx, cy in spec.ic])
    for _ in range(args.warmup):
        s.step(1)
    launches0 = ctx.launches
    barrier(world)
    clocks = Clocks(local)
    total_ms = 0.0
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device=dev)
    for _ in range(args.steps):
        flush.fill_(1.0)
        torch.cuda.synchronize(dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        s.step(1)
        e1.record(stream)
        e1.synchronize()
        total_ms += e0.elapsed_time(e1)
    clk = clocks.stop()
    launches = ctx.launches - launches0
    max_ms = allreduce_max(world, total_ms, local)
    value = world * args.steps / (max_ms * 1e-3)
    if rank != 0:
        return
    n, ng = spec.n, spec.n + 6
    passes = 2 if spec.model == 1 else 1
    stage = 3 * (n * n + ng * ng) + 2 * passes * 3 * ng * ng + 2 * 3 * n * (n + 1) + (3 * 2 * n * n + 3 * 2 * n * (n + 1) + 3 * n * n)
    step_bytes = 8.0 * 3 * stage
    hbm = float(measured_peaks().get("hbm_gbs", 6650.0))
    achieved = step_bytes / (max_ms / args.steps * 1e-3) / 1e9
    cfgd = workload(spec)
    cfgd.update({"representation": "dense (device DenseRep, ttsw_dense_*)", "l2": "flushed (512 MiB write) between timed steps",
                 "parallelism": f"replicas x{world}"})
    print(json.dumps({"metric": METRIC, "value": value, "unit": "steps/s", "n_gpus": world, "steps": args.steps,
                      "warmup": args.warmup, "ms_per_step": max_ms / args.steps, "higher_is_better": True,
                      "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": cfgd,
                      "cell_updates_per_s": value * n * n,
                      "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                                   "traffic": None, "kernel": "whole dense step (k_dense_ghost, k_dense_axis, k_dense_combine)",
                                   "algorithmic_bytes_per_step": step_bytes},
                      "gpu_launches": launches, "clocks": clk}), flush=True)


def run_ensemble(args, world, rank, local):
    """C5: `--members` independent C3 trajectories (per-member seeds) sharded in contiguous
    blocks over the ranks (no data-path collective); on each GPU the library's native
    ensemble runtime (ttsw_ensemble_*) keeps `--member-threads` members in flight
    concurrently (one worker thread and stream each). value = all member-steps / max-over-ranks
    device time of the timed steps; one all-gather of the per-member records at the end."""
    import torch

    from paper_2408_03483_b200 import capi, ensemble

    spec = make_spec(args)
    dev = torch.device(f"cuda:{local}")
    torch.cuda.set_device(dev)
    mine = list(ensemble.shard(args.members, world, rank))
    ev = {}
    clocks = []

    def timer(which):
        torch.cuda.synchronize(dev)
        barrier(world)
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        ev[which] = e
        if which == "start":
            clocks.append(Clocks(local))
        else:
            e.synchronize()

    t0 = time.perf_counter()
    recs = ensemble.run_native(local, mine, spec.n, args.warmup, args.steps, args.member_threads, timer)
    wall = time.perf_counter() - t0
    ms = ev["start"].elapsed_time(ev["stop"])
    clk = clocks[0].stop() if clocks else None
    max_ms = allreduce_max(world, ms, local)
    wall_max = allreduce_max(world, wall, local)
    value = args.members * args.steps / (max_ms * 1e-3)
    e2e_value = args.members * (args.steps + args.warmup) / wall_max
    allrec = ensemble.gather_records(recs, world, device=dev if world > 1 else None)
    if rank != 0:
        return
    cfgd = workload(spec)
    cfgd.update({"workload": f"C5: {args.members}-member ensemble of C3 (nonlinear SWE N={spec.n}, upwind5, "
                             f"tol 1e-10), member m seeded S5+m; {len(mine)} members on this rank x {world} ranks",
                 "members": args.members, "member_threads_per_gpu": args.member_threads,
                 "parallelism": f"members sharded x{world} (contiguous blocks, no data-path collective)",
                 "l2": "members' working sets (> 126 MB L2 in aggregate) cycle through L2"})
    # CPU leg: oracle sample of member 0 step 0 with the GPU trace of that step
    step_work = None
    if world == 1 and not args.no_cpu_baseline:
        ctx = capi.Context(local)
        s = capi.Solver(ctx, spec.model, spec.scheme, spec.n, spec.g, spec.f, spec.H, spec.dt, spec.tol,
                        capi.CrossCfg.make(seed=1, max_rank=spec.cross_max_rank))
        s.set_state([ctx.round(ctx.tt(cx, cy), spec.tol) for cx, cy in spec.ic])
        s.set_tracing(True)
        s.step(1)
        tr0 = s.trace()[0]
        step_work = round_work(tr0)
        if not args.n:
            json.dump({"config": "C5 member 0", "N": spec.n, "columns": "step, m, n, r_in, k_out, crosses_before",
                       "trace": tr0.tolist()}, open(trace_path(spec), "w"))
    line = {"metric": METRIC, "value": value, "unit": "member-steps/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": max_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": cfgd,
            "cell_updates_per_s": value * spec.n * spec.n, "roofline": None,
            "e2e": {"value": e2e_value, "unit": "member-steps/s", "h2d_bytes_per_step": None,
                    "d2h_bytes_per_step": None,
                    "note": "whole run through the public API (contexts, host ICs uploaded, warm-up + timed "
                            "steps, records read back) over wall time"},
            "gpu_launches": None, "clocks": clk,
            "members": {"count": int(allrec.shape[0]), "final_ranks_max": allrec[:, 3:6].max(axis=0).tolist(),
                        "mass_min": float(allrec[:, 2].min()), "mass_max": float(allrec[:, 2].max())}}
    if step_work is not None:
        rate, desc = oracle_sample(spec, args.cpu_budget, step_work)
        line["cpu_baseline"] = {"value": rate, "unit": "member-steps/s", "cores": 1, "kind": "port",
                                "sample": desc}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    world, rank, local = dist_init()
    if args.impl == "reference":
        run_reference(args, world, rank)
    elif args.config == "C5":
        run_ensemble(args, world, rank, local)
    elif args.rep == "dense":
        run_dense(args, world, rank, local)
    else:
        run_ours(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
