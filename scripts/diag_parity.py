"""Diagnostic: step GPU and oracle solvers side by side and report where rounding
margins / cross pivots first diverge (used to investigate parity failures)."""
import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np
import pyoracle as O
from paper_2408_03483_b200 import capi, ics

name, n, steps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
spec = ics.CONFIGS[name](n=n)
ctx = capi.Context(0)
gs = capi.Solver(ctx, spec.model, spec.scheme, spec.n, spec.g, spec.f, spec.H, spec.dt, spec.tol,
                 capi.CrossCfg.make(seed=1, max_rank=spec.cross_max_rank))
os_ = O.Solver(spec.model, spec.scheme, spec.n, spec.g, spec.f, spec.H, spec.dt, spec.tol,
               O.CrossCfg.make(seed=1, max_rank=spec.cross_max_rank))
gs.set_state([ctx.round(ctx.tt(cx, cy), spec.tol) for cx, cy in spec.ic])
os_.set_state([O.round_(O.TT.from_cores(cx, cy), spec.tol) for cx, cy in spec.ic])
for k in range(steps):
    gs.step(1); os_.step(1)
    gt, gm, gk = gs.trace(); ot, om, ok = os_.trace()
    gc, gr = gs.cross_trace(); oc, orr = os_.cross_trace()
    print(f"step {k}: roundings {len(gt)}/{len(ot)} crosses {len(gc)}/{len(oc)}")
    for i in range(min(len(gc), len(oc))):
        print(f"  cross {i}: gpu rank {gc[i,0]} sweeps {gc[i,1]} res {gr[i]:.3e} hash {gc[i,2]} | "
              f"cpu rank {oc[i,0]} sweeps {oc[i,1]} res {orr[i]:.3e} hash {oc[i,2]}")
    dm = np.abs(gm - om) / np.maximum(1e-30, np.minimum(np.abs(gm), np.abs(om))) if len(gt) == len(ot) else None
    shown = 0
    for i in range(min(len(gt), len(ot))):
        bad = gt[i, 4] != ot[i, 4] or (dm is not None and np.isfinite(dm[i]) and dm[i] > 1e-2)
        if bad and shown < 12:
            print(f"  round {i}: R {gt[i,3]}/{ot[i,3]} k {gt[i,4]}/{ot[i,4]} margin {gm[i]:.3e}/{om[i]:.3e} kappa {gk[i]:.2e}/{ok[i]:.2e}")
            shown += 1
    for c, (a, b) in enumerate(zip(gs.state(), os_.state())):
        fa, fb = a.full(), b.full()
        print(f"  comp {c}: ranks {a.rank}/{b.rank} rel {np.linalg.norm(fa-fb)/max(np.linalg.norm(fb),1e-300):.3e}")
