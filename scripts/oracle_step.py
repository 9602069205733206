"""Step a BASELINE config in the oracle (CPU) and report the outcome (diagnostic)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import pyoracle as O
from paper_2408_03483_b200 import ics
name, n, steps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
kw = dict(arg.split("=") for arg in sys.argv[4:])
spec = ics.CONFIGS[name](n=n)
cfg = O.CrossCfg.make(seed=1, max_rank=int(kw.get("max_rank", spec.cross_max_rank)))
s = O.Solver(spec.model, spec.scheme, spec.n, spec.g, spec.f, spec.H, spec.dt, spec.tol, cfg)
s.set_state([O.round_(O.TT.from_cores(cx, cy), spec.tol) for cx, cy in spec.ic])
print("IC ranks", [t.rank for t in s.state()])
for k in range(steps):
    t0 = time.perf_counter()
    try:
        s.step(1)
    except Exception as e:
        print("step", k, "raised", type(e).__name__, e); break
    ct = s.cross_trace()[0]
    print(f"step {k}: {time.perf_counter()-t0:.2f}s ranks {[t.rank for t in s.state()]} crosses {len(ct)} max cross rank {ct[:,0].max() if len(ct) else 0}", flush=True)
