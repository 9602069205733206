"""The Taylor-reciprocal products dy * xt of a C3 face field, rounded with and without the sketch
(diagnostic): ranks, margins, and the difference of the two results."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2408_03483_b200 import capi, ics
n = int(sys.argv[1])
spec = ics.CONFIGS["C3"](n=n)
ctx = capi.Context(0)
tol = spec.tol
h = ctx.round(ctx.tt(*spec.ic[0]), tol)
fm, fp = ctx.reconstruct_faces(ctx.periodic_ghost(h), 0, spec.scheme, tol, None, 1.0 / n, 1.0 / n)
x = fm
m, nn = x.shape[0], x.shape[1]
avg = ctx.sum_entries(x) / (m * nn)
one = ctx.constant(m, nn, 1.0)
ctx.set_sketch(False)
xt = ctx.round(ctx.add(one, ctx.scale(x, -1.0 / avg)), tol)
dy = one
for it in range(1, 9):
    prod = ctx.hadamard(dy, xt)
    ctx.set_sketch(False)
    d0, i0 = ctx.round(prod, tol, with_info=True)
    ctx.set_sketch(True, 160, 64)
    d1, i1 = ctx.round(prod, tol, with_info=True)
    cx, cy = prod.cores()
    rx = np.linalg.qr(cx, mode="r"); ry = np.linalg.qr(cy.T, mode="r")
    sv = np.linalg.svd(rx @ ry.T, compute_uv=False)
    tot = (sv ** 2).sum(); bud = (0.9 * tol) ** 2 * tot
    k = d0.rank
    tails = {kk: float((sv[kk:] ** 2).sum() / bud) for kk in (k - 1, k, k + 1)}
    print(f"it {it}: R={prod.rank} k off/on {d0.rank}/{d1.rank} margins {i0.margin:.5f}/{i1.margin:.5f} kappa {i0.kappa:.3g} "
          f"numpy tails/budget {tails} tail beyond 56: {float((sv[56:]**2).sum()/bud):.3e} "
          f"diff of results {np.linalg.norm(d0.full()-d1.full())/np.sqrt(tot):.3e} {ctx.sketch_stats()}")
    dy = d0
