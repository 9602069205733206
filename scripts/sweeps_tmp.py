import sys, os, ctypes as C
sys.path.insert(0, '/root/repo')
import numpy as np
from paper_2408_03483_b200 import capi, ics
spec = ics.config2(n=1024)
ctx = capi.Context(0)
s = capi.Solver(ctx, spec.model, spec.scheme, spec.n, spec.g, spec.f, spec.H, spec.dt, spec.tol)
s.set_state([ctx.round(ctx.tt(cx, cy), spec.tol) for cx, cy in spec.ic])
import time
for k in range(3):
    t0 = time.perf_counter(); s.step(1); ctx.sync(); print("step ms", (time.perf_counter()-t0)*1e3)
