"""Time ctx.round on one random decaying-spectrum TT (diagnostic): m n r [reps] [eps]."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2408_03483_b200 import capi
m, n, r = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 5
eps = float(sys.argv[5]) if len(sys.argv) > 5 else 1e-10
true_rank = int(sys.argv[6]) if len(sys.argv) > 6 else 0
rng = np.random.default_rng(0)
ctx = capi.Context(0)
if true_rank:  # R columns spanning a rank-true_rank space with a decaying spectrum
    decay = np.logspace(0, -12, true_rank)
    cx = (rng.standard_normal((m, true_rank)) * decay) @ rng.standard_normal((true_rank, r))
else:
    decay = np.logspace(0, -14, r)[rng.permutation(r)]
    cx = rng.standard_normal((m, r)) * decay
x = ctx.tt(cx, rng.standard_normal((r, n)))
ctx.time_rounds(True)
for i in range(reps):
    l0 = ctx.launches
    t0 = time.perf_counter()
    y = ctx.round(x, eps)
    ctx.sync()
    print(f"round m={m} n={n} r={r} -> k={y.rank}: {1e3*(time.perf_counter()-t0):.3f} ms, launches {ctx.launches-l0}")
