"""Margins of the large roundings of a solver step with and without the sketch (diagnostic)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2408_03483_b200 import capi, ics
name, n, steps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
spec = ics.CONFIGS[name](n=n)
runs = []
for on in (True, False):
    ctx = capi.Context(0)
    ctx.set_sketch(on, 160, 64)
    s = capi.Solver(ctx, spec.model, spec.scheme, spec.n, spec.g, spec.f, spec.H, spec.dt, spec.tol,
                    capi.CrossCfg.make(seed=1, max_rank=spec.cross_max_rank))
    s.set_state([ctx.round(ctx.tt(cx, cy), spec.tol) for cx, cy in spec.ic])
    s.step(steps)
    runs.append(s.trace())
(t1, m1, k1), (t0, m0, k0) = runs
for i in range(min(len(t1), len(t0))):
    if t1[i, 3] >= 160 or (len(sys.argv) > 4 and i >= int(sys.argv[4])):
        flag = "" if t1[i, 4] == t0[i, 4] else "  <-- rank differs"
        print(i, "R", t1[i, 3], "k", t1[i, 4], t0[i, 4], "margin %.6f %.6f" % (m1[i], m0[i]), "kappa %.3g" % k0[i], flag)
    if t1[i, 3] != t0[i, 3]:
        print("input ranks diverge at", i)
        break
