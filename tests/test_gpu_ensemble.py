"""Native ensemble runtime (ttsw_ensemble_*, C5): members stepped by the library's worker
threads give the same per-member records as the same members stepped one by one through
the single-solver API (independent, deterministic trajectories), and a member failure is
reported with its index."""
import numpy as np
import pytest

from paper_2408_03483_b200 import capi, ensemble, ics

pytestmark = pytest.mark.gpu


def test_native_ensemble_matches_sequential_members():
    members, n = [0, 1, 2, 3, 4], 40
    native = ensemble.run_native(0, members, n, warmup=1, steps=2, threads=3)
    ctx = capi.Context(0)
    seq = [ensemble.run_member(ctx, m, steps=3, n=n) for m in members]
    for a, b in zip(native, seq):
        assert a[0] == b[0] and a[1] == b[1]
        assert a[3:6] == b[3:6]  # final ranks
        assert a[6:9] == b[6:9]  # max ranks
        assert abs(a[2] - b[2]) <= 1e-12 * abs(b[2])


def test_native_ensemble_reports_the_failing_member():
    spec = ics.config5_member(0, n=24)
    descs = [capi.SolverDesc(spec.model, spec.scheme, spec.n, spec.g, spec.f, spec.H, spec.dt, spec.tol, 1e-6,
                             capi.CrossCfg.make(seed=1)) for _ in range(2)]
    e = capi.Ensemble(0, descs, threads=2)
    for c, (cx, cy) in enumerate(spec.ic):
        e.set_state(0, c, cx, cy, round_eps=spec.tol)
        # member 1: a negative layer thickness -> StateError from its lambda cross
        e.set_state(1, c, -cx if c == 0 else cx, cy, round_eps=spec.tol)
    with pytest.raises(capi.StateError) as err:
        e.step(1)
    assert "member 1" in str(err.value)
