"""Generates the committed golden fixtures from the CPU oracle (restated reference).

  python tests/golden/make_golden.py

Each fixture stores the per-rounding trace (m, n, r_in, k_out, margin, kappa) and the
final dense fields of a short seeded run; tests/test_golden.py pins the oracle to them
and tests/test_gpu_golden.py checks the CUDA path against them on the B200."""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import numpy as np  # noqa: E402

import pyoracle  # noqa: E402
from paper_2408_03483_b200 import ics  # noqa: E402

# c4_n16 keeps the rough rank-4 noise (frozen before the C4 default became smooth4);
# c4s_n16 is the default (smooth4) C4 setup
CASES = {"c1_n32": ("C1", 32, 10, {}), "c2_n64": ("C2", 64, 10, {}), "c3_n16": ("C3", 16, 2, {}),
         "c4_n16": ("C4", 16, 1, {"noise": "rank4"}), "c4s_n16": ("C4", 16, 1, {})}


def run(name, n, steps, kw=None):
    spec = ics.CONFIGS[name](n=n, **(kw or {}))
    s = pyoracle.Solver(spec.model, spec.scheme, spec.n, spec.g, spec.f, spec.H, spec.dt, spec.tol,
                        pyoracle.CrossCfg.make(seed=1, max_rank=spec.cross_max_rank))
    s.set_state([pyoracle.round_(pyoracle.TT.from_cores(cx, cy), spec.tol) for cx, cy in spec.ic])
    traces, margins, kappas, crosses = [], [], [], []
    for k in range(steps):
        s.step(1)
        tr, mg, ka = s.trace()
        tr[:, 0] = k  # column 0 := step index (rounding index is the row order within a step)
        traces.append(tr)
        margins.append(mg)
        kappas.append(ka)
        crosses.append(s.cross_trace()[0])
    fields = np.stack([t.full() for t in s.state()])
    cross = np.concatenate(crosses) if crosses else np.zeros((0, 3), dtype=np.int64)
    return np.concatenate(traces), np.concatenate(margins), np.concatenate(kappas), fields, cross


if __name__ == "__main__":
    pyoracle.build()
    for key, (name, n, steps, kw) in CASES.items():
        if len(sys.argv) > 1 and key not in sys.argv[1:]:
            continue
        tr, mg, ka, f, cr = run(name, n, steps, kw)
        np.savez_compressed(os.path.join(HERE, key + ".npz"), trace=tr, margin=mg, kappa=ka, fields=f, cross=cr,
                            config=np.array([name]), n=n, steps=steps)
        print(key, tr.shape, f.shape)
