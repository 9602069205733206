"""Time SSP-RK3 steps of a BASELINE config on the GPU (diagnostic)."""
import sys, os, time
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
ctx.time_rounds(True)
for k in range(steps):
    l0 = ctx.launches
    t0 = time.perf_counter()
    s.step(1)
    ctx.sync()
    dt = time.perf_counter() - t0
    tr, mg, ka = s.trace()
    ct, cres = s.cross_trace()
    rs = ctx.round_stats(reset=True)
    print(f"step {k}: {dt*1e3:.1f} ms, launches {ctx.launches-l0}, ranks {[t.rank for t in s.state()]}, "
          f"roundings {len(tr)} R_in max {tr[:,3].max()} mean {tr[:,3].mean():.1f}, k max {tr[:,4].max()}, "
          f"round time {rs['ms']:.1f} ms ({rs['flops']/max(rs['ms'],1e-9)/1e9:.2f} TFLOP/s), "
          f"crosses {len(ct)} ranks {list(ct[:,0])} sweeps {list(ct[:,1])}", flush=True)
