"""CPU checks of the dense (DenseRep) oracle restatement (oracle/dense_oracle.py) against the
TT oracle and the reference's dense-path known answers (test_swe.cpp, test_reconstruction.cpp)."""
import numpy as np
import pytest

import dense_oracle as D
from ghost_ref import dense_ghosted
from parity import rel


def smooth(n, mean, amp, kx, ky, phase=0.0):
    x = (np.arange(n) + 0.5) / n
    return mean + amp * np.outer(np.sin(2 * np.pi * kx * x + phase), np.cos(2 * np.pi * ky * x))


@pytest.mark.parametrize("scheme", [D.U3, D.U5])
def test_dense_linear_rhs_matches_tt_oracle(oracle, scheme):
    # rhs<DenseRep> vs rhs<TTRep> (linear: no rounding in the flux, exact maps): test_swe.cpp:271-309
    n, g, f, H = 24, 1.0, 3.0, 1.0
    q = [smooth(n, 0.0, 0.01, 1, 2), smooth(n, 0.0, 0.02, 2, 1, 0.3), smooth(n, 0.0, 0.015, 1, 1, 0.7)]
    want = D.rhs(q, oracle.tables(scheme), scheme, 0, g, f, H)
    s = oracle.Solver(0, scheme, n, g, f, H, 1e-3, 1e-13)
    s.set_state([oracle.from_full(a, 1e-15) for a in q])
    got = [t.full() for t in s.rhs()]
    for c in range(3):
        assert rel(got[c], want[c]) < 1e-9, (c, rel(got[c], want[c]))


@pytest.mark.parametrize("scheme", [D.U3, D.U5, D.W5])
@pytest.mark.parametrize("model", [0, 1])
def test_dense_constant_state_zero_tendency(oracle, scheme, model):
    # test_swe.cpp:193-227 (dense half): a constant state at rest has zero tendency
    n = 16
    q = [np.full((n, n), 1.3), np.zeros((n, n)), np.zeros((n, n))]
    k = D.rhs(q, oracle.tables(scheme), scheme, model, 1.0, 0.0, 1.0)
    for c in range(3):
        assert np.abs(k[c]).max() < 1e-12


def test_dense_ghosts_match_ghost_ref():
    rng = np.random.default_rng(3)
    n = 10
    a = rng.standard_normal((n, n))
    sx, sy = rng.standard_normal((6, n + 6)), rng.standard_normal((n + 6, 6))
    for bx, by in [(0, 0), (1, 0), (0, 1), (1, 1)]:
        got = D.ghosted(a, bx, by, sx, sy)
        # ghost_ref adds the strips to a zero-padded Dirichlet axis: the same values
        want = dense_ghosted(a, bx, by, sx, sy)
        assert np.array_equal(got, want), (bx, by)


def test_dense_nonpositive_h_is_a_state_error(oracle):
    n = 12
    q = [np.full((n, n), 1.0), np.zeros((n, n)), np.zeros((n, n))]
    q[0][3, 4] = -0.5
    with pytest.raises(D.StateError):
        D.rhs(q, oracle.tables(D.U5), D.U5, 1, 1.0, 0.0, 1.0)


def test_dense_ssprk3_temporal_order(oracle):
    # ssprk3 is third order (test_swe.cpp: temporal order ~3): errors vs a fine-dt run
    n = 16
    q = [smooth(n, 1.0, 0.05, 1, 1), smooth(n, 0.0, 0.01, 1, 2), smooth(n, 0.0, 0.01, 2, 1)]
    t = oracle.tables(D.U5)

    def run(dt, steps):
        w = q
        for k in range(steps):
            w = D.ssprk3(w, dt, k * dt, t, D.U5, 1, 1.0, 0.0, 1.0)
        return w

    T = 0.02
    ref = run(T / 64, 64)
    e = [np.linalg.norm(run(T / s, s)[0] - ref[0]) for s in (4, 8)]
    assert 2.5 < np.log2(e[0] / e[1]) < 3.5, e
