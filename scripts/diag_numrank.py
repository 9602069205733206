"""Numerical ranks of the cores of typical large rounding inputs (diagnostic): C4 at N, after `steps`
steps; the X-axis faces, the Taylor reciprocal, and the unrounded flux products' cores."""
import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
from paper_2408_03483_b200 import capi, ics

n, steps = int(sys.argv[1]), int(sys.argv[2])
spec = ics.CONFIGS["C4"](n=n)
ctx = capi.Context(0)
cfg = capi.CrossCfg.make(seed=1, max_rank=spec.cross_max_rank)
s = capi.Solver(ctx, spec.model, spec.scheme, spec.n, spec.g, spec.f, spec.H, spec.dt, spec.tol, cfg)
s.set_state([ctx.round(ctx.tt(cx, cy), spec.tol) for cx, cy in spec.ic])
s.step(steps)
st = s.state()
print("state ranks", [t.rank for t in st])


def numrank(a, name):
    sv = np.linalg.svd(a, compute_uv=False)
    sv = sv / sv[0]
    out = {lvl: int((sv > lvl).sum()) for lvl in (1e-8, 1e-10, 1e-12, 1e-14, 1e-15, 1e-16)}
    print(f"  {name}: shape {a.shape} numerical rank at", out)


def report(x, name):
    cx, cy = x.cores()
    print(f"{name}: m={cx.shape[0]} n={cy.shape[1]} R={cx.shape[1]}")
    numrank(cx, "core_x")
    numrank(cy.T, "core_y^T")
    # the product's singular values through the two R factors
    rx = np.linalg.qr(cx, mode="r")
    ry = np.linalg.qr(cy.T, mode="r")
    numrank(rx @ ry.T, "product")
    y = ctx.round(x, spec.tol)
    print(f"  rounded at {spec.tol}: k={y.rank}")
    return y


for axis in (0, 1):
    g = [ctx.periodic_ghost(x) for x in st]
    faces = [ctx.reconstruct_faces(q, axis, spec.scheme, spec.tol, cfg, 1.0 / n, 1.0 / n) for q in g]
    h, hu, hv = (f[0] for f in faces)
    print(f"axis {axis} face ranks", h.rank, hu.rank, hv.rank)
    inv = ctx.recip(h, spec.tol)[0]
    print("recip rank", inv.rank)
    vx = report(ctx.hadamard(hu, inv), "vel_x = hu * inv_h")
    report(ctx.hadamard(h, h), "h * h")
    f1 = report(ctx.hadamard(hu, vx), "hu * vel_x")
    report(ctx.add(f1, ctx.scale(ctx.round(ctx.hadamard(h, h), spec.tol), 0.5)), "hu*vel_x + p")
    report(ctx.add(ctx.scale(faces[1][0], 0.5), ctx.scale(faces[1][1], 0.5)), "central-like sum of the two sides of hu")
