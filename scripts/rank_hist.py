"""Histogram of pre-rounding ranks R and output ranks k over one SSP-RK3 step (diagnostic)."""
import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
from paper_2408_03483_b200 import capi, ics
name, n, steps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
spec = ics.CONFIGS[name](n=n)
ctx = capi.Context(0)
s = capi.Solver(ctx, spec.model, spec.scheme, spec.n, spec.g, spec.f, spec.H, spec.dt, spec.tol,
                capi.CrossCfg.make(seed=1, max_rank=spec.cross_max_rank))
s.set_state([ctx.round(ctx.tt(cx, cy), spec.tol) for cx, cy in spec.ic])
for k in range(steps):
    s.step(1)
tr, mg, ka = s.trace()
R, K, m, nn = tr[:, 3], tr[:, 4], tr[:, 1], tr[:, 2]
print("roundings", len(tr), "shapes", sorted(set(zip(m.tolist(), nn.tolist()))))
edges = [0, 8, 16, 32, 64, 96, 128, 168, 256, 512, 10**6]
h, _ = np.histogram(R, edges)
work = [(2 * (m[(R >= a) & (R < b)] + nn[(R >= a) & (R < b)]) * R[(R >= a) & (R < b)] ** 2).sum() for a, b in zip(edges[:-1], edges[1:])]
for (a, b), c, w in zip(zip(edges[:-1], edges[1:]), h, work):
    print(f"R in [{a},{b}): {c:5d} roundings, QR work {w/1e9:8.2f} GFLOP")
print("k max", K.max(), "k mean", K.mean())
