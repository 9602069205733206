"""ms/step and state-rank curve of a whole BASELINE run on the GPU (evidence for DESIGN §10).

  python scripts/long_curve.py C4 4096 500 out.json

Steps run exactly as in bench.py's timed region (no per-rounding events, tracing off),
one CUDA-event pair per step on the library's stream, no L2 flush."""
import json
import os
import sys
import time

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2408_03483_b200 import capi, ics  # noqa: E402

name, n, steps, out = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
spec = ics.CONFIGS[name](n=n)
ctx = capi.Context(0)
stream = torch.cuda.ExternalStream(ctx.stream, device="cuda:0")
s = capi.Solver(ctx, spec.model, spec.scheme, spec.n, spec.g, spec.f, spec.H, spec.dt, spec.tol,
                capi.CrossCfg.make(seed=1, max_rank=spec.cross_max_rank))
s.set_state([ctx.round(ctx.tt(cx, cy), spec.tol) for cx, cy in spec.ic])
s.set_tracing(False)
rows = []
t_start = time.time()
for k in range(steps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = ctx.launches
    e0.record(stream)
    s.step(1)
    e1.record(stream)
    e1.synchronize()
    ms = e0.elapsed_time(e1)
    rows.append({"step": k, "ms": ms, "ranks": [t.rank for t in s.state()], "launches": ctx.launches - l0})
    if k % 10 == 0 or k == steps - 1:
        print(f"step {k}: {ms:.1f} ms ranks {rows[-1]['ranks']} launches {rows[-1]['launches']}", flush=True)
        json.dump({"config": name, "N": n, "steps_done": k + 1, "wall_s": time.time() - t_start, "rows": rows},
                  open(out, "w"))
tot = sum(r["ms"] for r in rows)
print(f"{name} N={n}: {steps} steps in {tot / 1e3:.1f} s device time, mean {steps / (tot / 1e3):.3f} steps/s")
