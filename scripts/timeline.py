"""GPU timeline of SSP-RK3 steps (diagnostic): torch.profiler (CUPTI) records every kernel
of the library with device timestamps; reports the busy fraction of the GPU (union of
kernel intervals over the step's wall time), the idle gaps, and in-situ per-kernel totals
(concurrent, not serialised as under ncu). Usage: timeline.py C4 4096 [warm] [steps]"""
import collections
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402  (CUPTI via the profiler; the library itself does not use torch)
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2408_03483_b200 import capi, ics  # noqa: E402

name, n = sys.argv[1], int(sys.argv[2])
warm = int(sys.argv[3]) if len(sys.argv) > 3 else 3
steps = int(sys.argv[4]) if len(sys.argv) > 4 else 1
spec = ics.CONFIGS[name](n=n)
torch.cuda.init()
ctx = capi.Context(0)
s = capi.Solver(ctx, spec.model, spec.scheme, spec.n, spec.g, spec.f, spec.H, spec.dt, spec.tol,
                capi.CrossCfg.make(seed=1, max_rank=spec.cross_max_rank))
s.set_state([ctx.round(ctx.tt(cx, cy), spec.tol) for cx, cy in spec.ic])
for _ in range(warm):
    s.step(1)
ctx.sync()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    t0 = time.perf_counter()
    s.step(steps)
    ctx.sync()
    wall = time.perf_counter() - t0
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
iv = sorted((e.time_range.start, e.time_range.end, e.name) for e in ev if e.time_range.end > e.time_range.start)
if not iv:
    print("no CUDA events captured")
    sys.exit(0)
busy, cur_s, cur_e = 0.0, iv[0][0], iv[0][1]
gaps = []
for a, b, _ in iv[1:]:
    if a > cur_e:
        busy += cur_e - cur_s
        gaps.append(a - cur_e)
        cur_s, cur_e = a, b
    else:
        cur_e = max(cur_e, b)
busy += cur_e - cur_s
span = iv[-1][1] - iv[0][0]
tot = collections.Counter()
cnt = collections.Counter()
for a, b, nm in iv:
    k = nm.split("(")[0].replace("void ", "").split("::")[-1]
    tot[k] += b - a
    cnt[k] += 1
print(f"{name} N={n} steps={steps}: wall {wall * 1e3:.1f} ms, kernel span {span / 1e3:.1f} ms, "
      f"GPU busy (union) {busy / 1e3:.1f} ms = {100 * busy / span:.1f}% of the span, "
      f"{len(iv)} kernels, {len(gaps)} idle gaps (sum {sum(gaps) / 1e3:.1f} ms, "
      f"> 50 us: {sum(1 for g in gaps if g > 50)} totalling {sum(g for g in gaps if g > 50) / 1e3:.1f} ms)")
print(f"{'kernel':34s} {'count':>6s} {'sum ms':>9s} {'avg us':>8s}")
for k, v in tot.most_common(20):
    print(f"{k[:34]:34s} {cnt[k]:6d} {v / 1e3:9.2f} {v / cnt[k]:8.1f}")
