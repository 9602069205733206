"""Ensemble of independent trajectories (BASELINE config 5), sharded across ranks.

Members are fully independent: each rank advances a contiguous block
of members on its own GPU with no data-path collective; the only collective is one
all-gather of a fixed-size diagnostics record per member at the end (NCCL on GPUs,
gloo on CPU for tests).
"""
from __future__ import annotations

import time

import numpy as np

# record layout: member, steps, mass (sum h), final ranks[3], max ranks[3], device ms
RECORD = 10


def shard(members: int, world: int, rank: int) -> range:
    """Contiguous block of member ids for `rank` (sizes differ by at most one)."""
    base, rem = divmod(members, world)
    start = rank * base + min(rank, rem)
    return range(start, start + base + (1 if rank < rem else 0))


def run_member(ctx, member: int, steps: int, n: int = 2048):
    """Advance one C5 member on this rank's GPU through the C ABI; returns its record."""
    from . import capi, ics

    spec = ics.config5_member(member, n=n, steps=steps)
    s = capi.Solver(ctx, spec.model, spec.scheme, spec.n, spec.g, spec.f, spec.H, spec.dt, spec.tol,
                    capi.CrossCfg.make(seed=1, max_rank=spec.cross_max_rank))
    s.set_state([ctx.round(ctx.tt(cx, cy), spec.tol) for cx, cy in spec.ic])
    s.set_tracing(False)
    max_ranks = [0, 0, 0]
    t0 = time.perf_counter()
    for _ in range(steps):
        s.step(1)
        ranks = [t.rank for t in s.state()]
        max_ranks = [max(a, b) for a, b in zip(max_ranks, ranks)]
    ctx.sync()
    ms = (time.perf_counter() - t0) * 1e3
    st = s.state()
    mass = ctx.sum_entries(st[0]) / (spec.n * spec.n)
    return [member, steps, mass, *[t.rank for t in st], *max_ranks, ms]


def run_concurrent(device: int, members, n: int, warmup: int, steps: int, threads: int = 16, timer=None):
    """Advance several members at once on one GPU: `threads` host threads, each with its own
    context (stream), own its share of the members and step them in turn; ctypes releases
    the GIL inside every library call, so the members' kernels overlap on the device.
    All threads finish `warmup` steps, then `timer("start")` runs (after a device sync),
    the `steps` timed steps follow, and `timer("stop")` runs after the last thread.
    Returns one record per member (same layout as run_member)."""
    import threading

    from . import capi, ics

    members = list(members)
    nt = max(1, min(threads, len(members)))
    parts = [members[i::nt] for i in range(nt)]
    records = {}
    errors = []
    barrier = threading.Barrier(nt + 1)

    def worker(mine):
        try:
            ctx = capi.Context(device)
            solvers = []
            for m in mine:
                spec = ics.config5_member(m, n=n, steps=warmup + steps)
                s = capi.Solver(ctx, spec.model, spec.scheme, spec.n, spec.g, spec.f, spec.H, spec.dt, spec.tol,
                                capi.CrossCfg.make(seed=1, max_rank=spec.cross_max_rank))
                s.set_state([ctx.round(ctx.tt(cx, cy), spec.tol) for cx, cy in spec.ic])
                s.set_tracing(False)
                solvers.append((m, spec, s, [0, 0, 0]))
            for _ in range(warmup):
                for m, spec, s, mx in solvers:
                    s.step(1)
            ctx.sync()
        except Exception as e:  # noqa: BLE001 - reported after the barrier
            errors.append(e)
            solvers = []
        barrier.wait()
        barrier.wait()  # timed region starts
        try:
            t0 = time.perf_counter()
            for _ in range(steps):
                for m, spec, s, mx in solvers:
                    s.step(1)
                    mx[:] = [max(a, t.rank) for a, t in zip(mx, s.state())]
            ctx.sync()
            ms = (time.perf_counter() - t0) * 1e3
            for m, spec, s, mx in solvers:
                st = s.state()
                mass = ctx.sum_entries(st[0]) / (spec.n * spec.n)
                records[m] = [m, warmup + steps, mass, *[t.rank for t in st], *mx, ms]
        except Exception as e:  # noqa: BLE001
            errors.append(e)
        barrier.wait()

    ts = [threading.Thread(target=worker, args=(p,)) for p in parts]
    for t in ts:
        t.start()
    barrier.wait()  # warm-up done everywhere
    if timer:
        timer("start")
    barrier.wait()
    barrier.wait()  # timed steps done everywhere
    if timer:
        timer("stop")
    for t in ts:
        t.join()
    if errors:
        raise errors[0]
    return [records[m] for m in members]


def run_native(device: int, members, n: int, warmup: int, steps: int, threads: int = 16, timer=None):
    """The same as run_concurrent on the library's native ensemble runtime
    (ttsw_ensemble_*: C++ worker threads, one context each, no Python in the step loop).
    Returns one record per member (run_member layout; member ids are the global ones)."""
    from . import capi, ics

    members = list(members)
    specs = [ics.config5_member(m, n=n, steps=warmup + steps) for m in members]
    descs = [capi.SolverDesc(s.model, s.scheme, s.n, s.g, s.f, s.H, s.dt, s.tol, 1e-6,
                             capi.CrossCfg.make(seed=1, max_rank=s.cross_max_rank)) for s in specs]
    e = capi.Ensemble(device, descs, threads)
    for i, s in enumerate(specs):
        for c, (cx, cy) in enumerate(s.ic):
            e.set_state(i, c, cx, cy, round_eps=s.tol)
    if warmup:
        e.step(warmup)
    if timer:
        timer("start")
    e.step(steps)
    if timer:
        timer("stop")
    rec = e.records()
    rec[:, 0] = members
    return [list(r) for r in rec]


def gather_records(records, world: int, device=None):
    """All-gather fixed-size per-member records (one collective for the whole run)."""
    import torch
    import torch.distributed as dist

    local = torch.tensor(np.asarray(records, dtype=np.float64).reshape(-1, RECORD), device=device)
    if world == 1:
        return local.cpu().numpy()
    counts = [torch.zeros(1, dtype=torch.int64, device=device) for _ in range(world)]
    dist.all_gather(counts, torch.tensor([local.shape[0]], dtype=torch.int64, device=device))
    cap = int(max(c.item() for c in counts))
    padded = torch.full((cap, RECORD), float("nan"), dtype=torch.float64, device=device)
    padded[: local.shape[0]] = local
    out = [torch.empty_like(padded) for _ in range(world)]
    dist.all_gather(out, padded)
    rows = [o[: int(c.item())] for o, c in zip(out, counts)]
    return torch.cat(rows).cpu().numpy()
