"""CUDA path vs the committed golden fixtures (same seeded runs as the oracle produced)."""
import os

import numpy as np
import pytest

from paper_2408_03483_b200 import capi, ics
from parity import rank_mismatch_is_ill_posed, rel

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
CASES = {"c1_n32": ("C1", 32, 10), "c2_n64": ("C2", 64, 10), "c3_n16": ("C3", 16, 2), "c4_n16": ("C4", 16, 1)}


@pytest.mark.parametrize("key", list(CASES))
def test_gpu_matches_golden(ctx, key):
    ref = np.load(os.path.join(HERE, "golden", key + ".npz"))
    name, n, steps = CASES[key]
    spec = ics.CONFIGS[name](n=n)
    s = capi.Solver(ctx, spec.model, spec.scheme, spec.n, spec.g, spec.f, spec.H, spec.dt, spec.tol,
                    capi.CrossCfg.make(seed=1, max_rank=spec.cross_max_rank))
    s.set_state([ctx.round(ctx.tt(cx, cy), spec.tol) for cx, cy in spec.ic])
    traces, margins, kappas = [], [], []
    for k in range(steps):
        s.step(1)
        tr, mg, ka = s.trace()
        tr[:, 0] = k
        traces.append(tr); margins.append(mg); kappas.append(ka)
    tr, mg, ka = np.concatenate(traces), np.concatenate(margins), np.concatenate(kappas)
    rt, rm, rk = ref["trace"], ref["margin"], ref["kappa"]
    if tr.shape == rt.shape and np.array_equal(tr[:, 4], rt[:, 4]):
        pass  # identical rank after every rounding
    else:
        n_cmp = min(len(tr), len(rt))
        i = int(np.nonzero(tr[:n_cmp, 4] != rt[:n_cmp, 4])[0][0])
        assert rank_mismatch_is_ill_posed(tr[i, 3], mg[i], rm[i], ka[i], rk[i], spec.tol), (i, tr[i], rt[i])
    for c, t in enumerate(s.state()):
        assert rel(t.full(), ref["fields"][c]) <= 1e-10 * steps, (c, rel(t.full(), ref["fields"][c]))
