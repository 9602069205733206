"""Sketched vs two-core rounding of one TT with a prescribed spectrum (diagnostic)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2408_03483_b200 import capi
m, n, r, k10 = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
rng = np.random.default_rng(1)
dec = np.maximum(10.0 ** (-10.0 / k10 * np.arange(r)), 1e-17)
U, _ = np.linalg.qr(rng.standard_normal((m, r)))
V, _ = np.linalg.qr(rng.standard_normal((n, r)))
A = rng.standard_normal((r, r)) / np.sqrt(r) + np.eye(r)
cx = (U * dec) @ A
cy = np.linalg.solve(A, V.T)
ctx = capi.Context(0)
x = ctx.tt(cx, cy)
sv = np.linalg.svd((U * dec) @ V.T, compute_uv=False)
tot = (sv ** 2).sum(); bud = (0.9e-10) ** 2 * tot
print("true tails/budget:", {k: float((sv[k:] ** 2).sum() / bud) for k in range(k10 - 3, k10 + 4)})
for on in (False, True):
    ctx.set_sketch(on, 160, 64)
    y, info = ctx.round(x, 1e-10, with_info=True)
    print("sketch", on, "k", y.rank, "margin", info.margin, "kappa", info.kappa, ctx.sketch_stats())
    full = y.full()
    print("   err vs M", np.linalg.norm(full - (U * dec) @ V.T) / np.sqrt(tot))
