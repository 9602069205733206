"""Oracle pin: maxvol / cross known-answer tests (/root/reference/proj/tests/test_cross.cpp:13-176)."""
import itertools

import numpy as np
import pytest

from parity import rel


def test_maxvol_dominant_2x2():  # test_cross.cpp:13-30
    import pyoracle as O

    m = np.array([[1, 0], [0, 1], [0.5, 0.5]])
    best, best_det = None, 0
    for a, b in itertools.combinations(range(3), 2):
        d = abs(np.linalg.det(m[[a, b]]))
        if d > best_det:
            best, best_det = [a, b], d
    assert best == [0, 1] and O.maxvol(m) == best


def test_maxvol_square_keeps_all(oracle):  # :32-36
    g = oracle.Rng(31)
    assert oracle.maxvol(g.random_matrix(5, 5)) == [0, 1, 2, 3, 4]


def test_maxvol_beats_random_subsets(oracle):  # :38-57
    g = oracle.Rng(32)
    m = g.random_matrix(64, 4)
    rows = oracle.maxvol(m)
    chosen = abs(np.linalg.det(m[rows]))
    picks = g.uniform_int(0, 63, 4 * 20000)
    k = 0
    for _ in range(2000):  # (10^4 in the reference; 2000 keeps the CPU suite fast)
        pick = []
        while len(pick) < 4:
            i = int(picks[k]); k += 1
            if i not in pick:
                pick.append(i)
        assert chosen >= abs(np.linalg.det(m[pick])) * (1 - 1e-12)


def test_maxvol_degenerate(oracle):  # :59-65
    g = oracle.Rng(33)
    m = np.zeros((6, 3))
    m[:, :2] = g.random_matrix(6, 2)
    m[:, 2] = m[:, 0] + m[:, 1]
    with pytest.raises(oracle.DegeneracyError):
        oracle.maxvol(m)
    with pytest.raises(oracle.ShapeError):
        oracle.maxvol(np.ones((2, 3)))


def cfg(oracle, eps, **kw):
    return oracle.CrossCfg.make(eps=eps, seed=99, **kw)


def test_cross_identity(oracle):  # :78-85
    g = oracle.Rng(34)
    x = g.random_tt(40, 30, 3)
    z, _ = oracle.cross(oracle.FN_IDENTITY, [x], x, cfg(oracle, 1e-10))
    assert rel(z.full(), x.full()) < 1e-10


def test_cross_product(oracle):  # :87-97
    g = oracle.Rng(35)
    x, y = g.random_tt(48, 40, 2), g.random_tt(48, 40, 3)
    z, st = oracle.cross(oracle.FN_PRODUCT, [x, y], x, cfg(oracle, 1e-10))
    assert rel(z.full(), x.full() * y.full()) < 1e-9
    assert z.rank <= 6 + 2


def test_cross_sqrt_constant(oracle):  # :99-106
    four = oracle.TT.constant(16, 12, 4.0)
    z, _ = oracle.cross(oracle.FN_SQRT, [four], four, cfg(oracle, 1e-12))
    assert z.rank == 1 and rel(z.full(), np.full((16, 12), 2.0)) < 1e-12


def test_cross_exact_rank_within_10eps(oracle):  # :108-120
    g = oracle.Rng(36)
    eps = 1e-8
    for n in (64, 256):
        x = g.random_tt(n, n - 5, 5)
        guess = oracle.TT.constant(n, n - 5, 1.0)
        z, _ = oracle.cross(oracle.FN_AFFINE, [x], guess, cfg(oracle, eps))
        ref = 2.0 * x.full() + 1.0
        assert np.linalg.norm(z.full() - ref) <= 10 * eps * np.linalg.norm(ref)


def test_cross_evaluation_budget(oracle):  # :122-134
    g = oracle.Rng(37)
    n = 256
    x = g.random_tt(n, n, 4)
    c = cfg(oracle, 1e-9)
    z, st = oracle.cross(oracle.FN_SQUARE, [x], x, c)
    assert st.evaluations < n * n
    assert st.evaluations <= 2 * ((2 * n) * z.rank * st.sweeps + c.validation_sample * st.sweeps)


def test_cross_deterministic(oracle):  # :136-144
    g = oracle.Rng(38)
    x = g.random_tt(32, 32, 3)
    a, _ = oracle.cross(oracle.FN_SQUARE, [x], x, cfg(oracle, 1e-9))
    b, _ = oracle.cross(oracle.FN_SQUARE, [x], x, cfg(oracle, 1e-9))
    assert np.array_equal(a.full(), b.full())


def test_cross_throwing_function(oracle):  # :146-157
    a = np.ones((8, 8))
    a[5, 2] = -4.0
    x = oracle.from_full(a, 0.0)
    with pytest.raises(oracle.EvaluationError) as e:
        oracle.cross(oracle.FN_SQRT, [x], x, cfg(oracle, 1e-10))
    assert (e.value.row, e.value.col) == (5, 2)


def test_cross_rank_cap_failure(oracle):  # :159-176
    g = oracle.Rng(39)
    noise = g.random_matrix(40, 40)
    x = oracle.from_full(noise, 0.0)
    guess = oracle.TT.constant(40, 40, 1.0)
    with pytest.raises(oracle.ConvergenceError) as e:
        oracle.cross(oracle.FN_IDENTITY, [x], guess, cfg(oracle, 1e-12, max_rank=4, max_sweeps=5))
    assert e.value.residual > 1e-12 and e.value.iterations == 5


def test_cross_llf_domain_error(oracle):  # swe.hpp:343-344: h <= 0 -> EvaluationError
    h = oracle.TT.constant(6, 5, 1.0)
    bad = oracle.TT.constant(6, 5, -1.0)
    m = oracle.TT.constant(6, 5, 0.5)
    with pytest.raises(oracle.EvaluationError):
        oracle.cross(oracle.FN_LLF_LAMBDA, [h, m, bad, m], h, cfg(oracle, 1e-6), param=1.0)
