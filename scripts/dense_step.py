"""Steps of a BASELINE config on the device full-tensor path (diagnostic / ncu target).

  python scripts/dense_step.py C4 4096 3
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2408_03483_b200 import capi, ics  # noqa: E402

name, n, steps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
spec = ics.CONFIGS[name](n=n)
ctx = capi.Context(0)
s = capi.DenseSolver(ctx, spec.model, spec.scheme, spec.n, spec.g, spec.f, spec.H, spec.dt)
s.set_state([cx @ cy for cx, cy in spec.ic])
for k in range(steps):
    t0 = time.perf_counter()
    s.step(1)
    print(f"step {k}: {1e3 * (time.perf_counter() - t0):.2f} ms", flush=True)
