"""The committed full-length oracle trajectories (tests/golden/long/, made by
tests/golden/make_long.py) are reproducible: one oracle step from a fixture's checkpoint
gives the next checkpoint bit for bit, with the recorded rank trace. (CPU; the N=4096
fixture is skipped here — one oracle step at that size takes minutes.)"""
import glob
import os

import numpy as np
import pytest

from paper_2408_03483_b200 import ics

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FIXTURES = [p for p in sorted(glob.glob(os.path.join(ROOT, "tests", "golden", "long", "*.npz")))
            if "n4096" not in p]


@pytest.mark.parametrize("path", FIXTURES, ids=[os.path.basename(p)[:-4] for p in FIXTURES])
def test_fixture_step_is_reproducible(oracle, path):
    d = np.load(path)
    meta = eval(str(d["meta"]))
    spec = ics.config5_member(meta["member"], n=meta["n"]) if meta["config"] == "C5" else \
        ics.CONFIGS[meta["config"]](n=meta["n"])
    cks = [int(c) for c in d["checkpoints"]]
    s0 = next(c for c in cks if c + 1 in cks and f"step_trace_{c}" in d)
    cfg = oracle.CrossCfg.make(seed=1, max_rank=spec.cross_max_rank)
    o = oracle.Solver(spec.model, spec.scheme, spec.n, spec.g, spec.f, spec.H, spec.dt, spec.tol, cfg)
    if s0 == 0:  # the IC rounds to the recorded state
        r0 = [oracle.round_(oracle.TT.from_cores(cx, cy), spec.tol) for cx, cy in spec.ic]
        for c, t in enumerate(r0):
            cx, cy = t.cores()
            assert np.array_equal(cx, d[f"ck_0_{c}_x"]) and np.array_equal(cy, d[f"ck_0_{c}_y"])
    o.set_state([oracle.TT.from_cores(d[f"ck_{s0}_{c}_x"], d[f"ck_{s0}_{c}_y"]) for c in range(3)])
    o.step(1)
    tr = o.trace()[0]
    want = d[f"step_trace_{s0}"]
    assert np.array_equal(tr[:, 3], want[:, 0].astype(int)) and np.array_equal(tr[:, 4], want[:, 1].astype(int))
    for c, t in enumerate(o.state()):
        cx, cy = t.cores()
        assert np.array_equal(cx, d[f"ck_{s0 + 1}_{c}_x"]) and np.array_equal(cy, d[f"ck_{s0 + 1}_{c}_y"])
