"""vel = hu * (1/h) on the faces of a C3 state after one step, rounded with and without the
sketch (diagnostic): ranks, margins, numpy tails, difference of the two results."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2408_03483_b200 import capi, ics
n = int(sys.argv[1])
L = int(sys.argv[2]) if len(sys.argv) > 2 else 64
spec = ics.CONFIGS["C3"](n=n)
ctx = capi.Context(0)
tol = spec.tol
ctx.set_sketch(False)
s = capi.Solver(ctx, spec.model, spec.scheme, spec.n, spec.g, spec.f, spec.H, spec.dt, spec.tol,
                capi.CrossCfg.make(seed=1, max_rank=spec.cross_max_rank))
s.set_state([ctx.round(ctx.tt(cx, cy), tol) for cx, cy in spec.ic])
s.step(1)
st = s.state()
for axis in (0, 1):
    faces = [ctx.reconstruct_faces(ctx.periodic_ghost(q), axis, spec.scheme, tol, None, 1.0 / n, 1.0 / n) for q in st]
    for side in (0, 1):
        hf, huf, hvf = (f[side] for f in faces)
        inv = ctx.recip(hf, tol)[0]
        for nm, a in (("hu*inv", huf), ("hv*inv", hvf)):
            prod = ctx.hadamard(a, inv)
            ctx.set_sketch(False)
            d0, i0 = ctx.round(prod, tol, with_info=True)
            ctx.set_sketch(True, 160, L)
            d1, i1 = ctx.round(prod, tol, with_info=True)
            cx, cy = prod.cores()
            rx = np.linalg.qr(cx, mode="r"); ry = np.linalg.qr(cy.T, mode="r")
            sv = np.linalg.svd(rx @ ry.T, compute_uv=False)
            tot = (sv ** 2).sum(); bud = (0.9 * tol) ** 2 * tot
            k = d0.rank
            tails = {kk: round(float((sv[kk:] ** 2).sum() / bud), 4) for kk in (k - 1, k, k + 1)}
            print(f"axis {axis} side {side} {nm}: R={prod.rank} k off/on {d0.rank}/{d1.rank} margins {i0.margin:.5f}/{i1.margin:.5f} "
                  f"kappa {i0.kappa:.3g} numpy tails/budget {tails} beyond 56: {float((sv[56:]**2).sum()/bud):.2e} "
                  f"sv[k..k+6]/s0 {np.array2string(sv[k-1:k+6]/sv[0], precision=2)} diff {np.linalg.norm(d0.full()-d1.full())/np.sqrt(tot):.2e}")
