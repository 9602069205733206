"""Oracle self-sensitivity: clean run vs runs with elementwise ±1ulp noise on the state cores every step."""
import sys, numpy as np
sys.path.insert(0, '/root/repo')
from oracle import pyoracle as O
from paper_2408_03483_b200 import ics
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
spec = ics.CONFIGS[name]()
cfg = O.CrossCfg.make(seed=1, max_rank=spec.cross_max_rank)
rel = lambda x, y: np.linalg.norm(x - y) / np.linalg.norm(y)
def mk():
    s = O.Solver(spec.model, spec.scheme, spec.n, spec.g, spec.f, spec.H, spec.dt, spec.tol, cfg)
    s.set_state([O.round_(O.TT.from_cores(cx, cy), spec.tol) for cx, cy in spec.ic]); return s
a = mk(); ref = []
for k in range(spec.steps):
    a.step(1); ref.append([t.full() for t in a.state()]) if k % 50 == 49 or k == spec.steps - 1 else None
for seed in range(3):
    rng = np.random.default_rng(seed); b = mk(); worst = 0; j = 0
    for k in range(spec.steps):
        b.step(1)
        st = []
        for t in b.state():
            cx, cy = t.cores()
            st.append(O.TT.from_cores(cx * (1 + 2.2e-16 * rng.uniform(-1, 1, cx.shape)), cy))
        b.set_state(st)
        if k % 50 == 49 or k == spec.steps - 1:
            e = max(rel(p.full(), q) for p, q in zip(b.state(), ref[j])); j += 1
            worst = max(worst, e)
    print(name, "seed", seed, "worst self-gap", f"{worst:.2e}", "final", f"{e:.2e}")
