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
