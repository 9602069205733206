"""Diagnose a C5 member against the oracle step by step (cross traces, field errors)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2408_03483_b200 import capi, ics
from oracle import pyoracle as O
m, n, steps = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
spec = ics.config5_member(m, n=n, steps=steps)
ctx = capi.Context(0)
g = capi.Solver(ctx, spec.model, spec.scheme, spec.n, spec.g, spec.f, spec.H, spec.dt, spec.tol, capi.CrossCfg.make(seed=1, max_rank=spec.cross_max_rank))
o = O.Solver(spec.model, spec.scheme, spec.n, spec.g, spec.f, spec.H, spec.dt, spec.tol, O.CrossCfg.make(seed=1, max_rank=spec.cross_max_rank))
g.set_state([ctx.round(ctx.tt(cx, cy), spec.tol) for cx, cy in spec.ic])
o.set_state([O.round_(O.TT.from_cores(cx, cy), spec.tol) for cx, cy in spec.ic])
rel = lambda a, b: np.linalg.norm(a - b) / np.linalg.norm(b)
for k in range(steps):
    g.step(1); o.step(1)
    gt = g.trace()[0]; ot = o.trace()[0]
    gc = g.cross_trace()[0]; oc = o.cross_trace()[0]
    rk = [(i, gt[i, 3], gt[i, 4], ot[i, 4]) for i in range(min(len(gt), len(ot))) if gt[i, 4] != ot[i, 4]]
    cs = [(i, tuple(gc[i]), tuple(oc[i])) for i in range(min(len(gc), len(oc))) if tuple(gc[i]) != tuple(oc[i])]
    errs = [rel(a.full(), b.full()) for a, b in zip(g.state(), o.state())]
    print(f"step {k}: field rel errs {['%.2e' % e for e in errs]} rank diffs {rk[:3]} cross diffs {cs[:3]} ncross {len(gc)}/{len(oc)}")
