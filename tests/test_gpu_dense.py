"""GPU parity of the full-tensor DenseRep path (ttsw_dense_*, csrc/dense.cu) against the numpy
restatement oracle/dense_oracle.py (rhs<DenseRep> / ssprk3<DenseRep>, swe.hpp:45-80, 362-454,
dense reconstruction reconstruction.hpp:253-423). Floating point, not bitwise: the device
contracts to FMA and sums the Gauss points in another order -> 1e-12 relative per rhs,
1e-11 after 10 steps."""
import numpy as np
import pytest

import dense_oracle as D
from paper_2408_03483_b200 import capi
from parity import rel

pytestmark = pytest.mark.gpu


def smooth(n, mean, amp, kx, ky, phase=0.0):
    x = (np.arange(n) + 0.5) / n
    return mean + amp * np.outer(np.sin(2 * np.pi * kx * x + phase), np.cos(2 * np.pi * ky * x + 0.2))


def states(n, model):
    if model == 0:
        return [smooth(n, 0.0, 0.01, 1, 2), smooth(n, 0.0, 0.02, 2, 1, 0.3), smooth(n, 0.0, 0.015, 1, 1, 0.7)]
    return [smooth(n, 1.0, 0.05, 1, 2), smooth(n, 0.0, 0.02, 2, 1, 0.3), smooth(n, 0.0, 0.015, 3, 1, 0.7)]


@pytest.mark.parametrize("scheme", [capi.UPWIND3, capi.UPWIND5, capi.WENO5])
@pytest.mark.parametrize("model", [capi.LINEAR, capi.NONLINEAR])
@pytest.mark.parametrize("n", [16, 45, 100])
def test_dense_rhs_matches_oracle(ctx, oracle, scheme, model, n):
    g, f, H = 1.0, 5.0, 1.0
    q = states(n, model)
    s = capi.DenseSolver(ctx, model, scheme, n, g, f, H, 1e-3)
    s.set_state(q)
    got = s.rhs()
    want = D.rhs(q, oracle.tables(scheme), scheme, model, g, f, H)
    for c in range(3):
        scale = max(np.linalg.norm(want[c]), 1e-300)
        assert np.linalg.norm(got[c] - want[c]) / scale < 1e-12, (c, np.linalg.norm(got[c] - want[c]) / scale)


@pytest.mark.parametrize("scheme", [capi.UPWIND5, capi.WENO5])
def test_dense_dirichlet_mms_rhs_matches_oracle(ctx, oracle, scheme):
    rng = np.random.default_rng(9)
    n, g, f, H = 24, 1.0, 2.0, 1.0
    q = states(n, 1)
    strips = {c: (1.0 + 0.01 * rng.standard_normal((6, n + 6)) if c == 0 else 0.01 * rng.standard_normal((6, n + 6)),
                  1.0 + 0.01 * rng.standard_normal((n + 6, 6)) if c == 0 else 0.01 * rng.standard_normal((n + 6, 6)))
              for c in range(3)}
    extra = [0.1 * rng.standard_normal((n, n)) for _ in range(3)]
    for bx, by in [(1, 0), (0, 1), (1, 1)]:
        s = capi.DenseSolver(ctx, 1, scheme, n, g, f, H, 1e-3)
        s.set_state(q)
        s.set_hooks(bx, by, lambda t, c: strips[c], lambda t: extra)
        got = s.rhs()
        want = D.rhs(q, oracle.tables(scheme), scheme, 1, g, f, H,
                     ghost=lambda c: (bx, by, strips[c][0], strips[c][1]), extra=extra)
        for c in range(3):
            assert rel(got[c], want[c]) < 1e-12, (bx, by, c, rel(got[c], want[c]))


@pytest.mark.parametrize("scheme,model", [(capi.UPWIND3, capi.LINEAR), (capi.UPWIND5, capi.NONLINEAR),
                                          (capi.WENO5, capi.NONLINEAR)])
def test_dense_ssprk3_steps_match_oracle(ctx, oracle, scheme, model):
    n, g, f, H, dt = 32, 1.0, 10.0, 1.0, 2e-3
    q = states(n, model)
    s = capi.DenseSolver(ctx, model, scheme, n, g, f, H, dt)
    s.set_state(q)
    w = q
    t = oracle.tables(scheme)
    for k in range(10):
        s.step(1)
        w = D.ssprk3(w, dt, k * dt, t, scheme, model, g, f, H)
    got = s.state()
    for c in range(3):
        assert rel(got[c], w[c]) < 1e-11, (c, rel(got[c], w[c]))
    assert s.time == pytest.approx(10 * dt)


def test_dense_nonpositive_h_is_a_state_error(ctx):
    n = 16
    q = [np.full((n, n), 1.0), np.zeros((n, n)), np.zeros((n, n))]
    q[0][5, 7] = -1.0
    s = capi.DenseSolver(ctx, 1, capi.UPWIND5, n, 1.0, 0.0, 1.0, 1e-3)
    s.set_state(q)
    with pytest.raises(capi.StateError):
        s.step(1)


def test_dense_constant_state_is_a_fixed_point(ctx):
    n = 40
    q = [np.full((n, n), 1.7), np.zeros((n, n)), np.zeros((n, n))]
    s = capi.DenseSolver(ctx, 1, capi.WENO5, n, 1.0, 10.0, 1.0, 1e-3)
    s.set_state(q)
    s.step(5)
    got = s.state()
    assert np.abs(got[0] - 1.7).max() < 1e-13 and np.abs(got[1]).max() < 1e-13 and np.abs(got[2]).max() < 1e-13
