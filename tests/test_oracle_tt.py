"""Oracle pin: the reference's TT-algebra known-answer tests
(/root/reference/proj/tests/test_tt.cpp:13-249) ported against the CPU oracle, with the
same seeded std::mt19937_64 + std::normal_distribution streams (tests/support.hpp:10-40)."""
import numpy as np
import pytest

from parity import rel


def dense_rank(A, tol):
    s = np.linalg.svd(A, compute_uv=False)
    return int(np.sum(s > tol * s[0]))


def test_rank1_round_trip(oracle):  # test_tt.cpp:13-21
    g = oracle.Rng(11)
    a, b = g.random_matrix(8, 1), g.random_matrix(8, 1)
    A = a @ b.T
    t = oracle.from_full(A, 1e-12)
    assert t.rank == 1 and rel(t.full(), A) < 1e-14


def test_zero_is_canonical_rank1(oracle):  # :23-29
    t = oracle.from_full(np.zeros((16, 16)), 1e-12)
    cx, cy = t.cores()
    assert t.rank == 1 and np.linalg.norm(cx) == 0 and np.linalg.norm(cy) == 0


def test_three_outer_products_rank3(oracle):  # :31-47
    g = oracle.Rng(12)
    A = np.zeros((32, 32))
    for _ in range(3):
        A += g.random_matrix(32, 1) @ g.random_matrix(32, 1).T
    assert dense_rank(A, 1e-12) == 3
    t = oracle.from_full(A, 1e-12)
    assert t.rank == 3 and np.linalg.norm(t.full() - A) <= 1e-12 * np.linalg.norm(A)


def test_non_finite_rejected(oracle):  # :49-53
    A = np.ones((4, 4))
    A[1, 2] = np.nan
    with pytest.raises(oracle.InputError):
        oracle.from_full(A, 1e-10)
    with pytest.raises(oracle.InputError):
        oracle.TT.from_cores(np.array([[np.inf]]), np.ones((1, 3)))


def test_to_full_hand_values(oracle):  # :55-67
    t = oracle.TT.from_cores(np.array([[1.0], [2.0]]), np.array([[3.0, 4.0]]))
    assert np.array_equal(t.full(), np.array([[3.0, 4.0], [6.0, 8.0]]))
    assert np.allclose(oracle.TT.constant(4, 4, 1.0).full(), np.ones((4, 4)))


def test_round_trip_lossless(oracle):  # :69-75
    g = oracle.Rng(13)
    for n in (1, 3, 17, 64, 128):
        A = g.random_matrix(n, n)
        assert rel(oracle.from_full(A, 0.0).full(), A) < 1e-12


def test_duplicated_cores_compress_to_rank1(oracle):  # :77-86
    g = oracle.Rng(14)
    a, b = g.random_matrix(12, 1), g.random_matrix(1, 9)
    r = oracle.round_(oracle.TT.from_cores(np.hstack([a, a]), np.vstack([0.5 * b, 0.5 * b])), 1e-12)
    assert r.rank == 1 and rel(r.full(), a @ b) < 1e-12


def test_eps0_keeps_value(oracle):  # :88-94
    g = oracle.Rng(15)
    x = g.random_tt(20, 14, 7)
    r = oracle.round_(x, 0.0)
    assert r.rank <= 7 and rel(r.full(), x.full()) < 1e-13


def test_truncation_rule(oracle):  # :96-110
    g = oracle.Rng(16)
    s = np.array([1.0, 1e-4, 1e-9])
    U, V = g.random_orthonormal(24, 3), g.random_orthonormal(18, 3)
    A = U @ np.diag(s) @ V.T
    x = oracle.TT.from_cores(U * s, V.T)
    r = oracle.round_(x, 1e-6)
    assert r.rank == 2 and np.linalg.norm(r.full() - A) <= 1e-6 * np.linalg.norm(A)


def test_round_contract_fuzz(oracle):  # :112-125
    g = oracle.Rng(17)
    for _ in range(200):
        n, m = g.uniform_int(1, 128, 2)
        r = min(int(g.uniform_int(1, 16, 1)[0]), n, m)
        x = g.random_tt(int(n), int(m), r)
        eps = 10.0 ** g.uniform_real(-12.0, -2.0, 1)[0]
        rr = oracle.round_(x, eps)
        assert rr.rank <= x.rank
        assert np.linalg.norm(rr.full() - x.full()) <= eps * np.linalg.norm(x.full())


def test_truncation_rank_rule_direct(oracle):  # tt.hpp:61-77 semantics
    assert oracle.truncation_rank([1.0, 1e-4, 1e-9], 1e-6)[0] == 2
    assert oracle.truncation_rank([0.0, 0.0], 1e-6)[0] == 1          # total == 0 -> 1
    assert oracle.truncation_rank([1.0, 0.0, 0.0], 0.0)[0] == 1      # exact zeros always dropped
    assert oracle.truncation_rank([1.0, 1e-20], 0.0)[0] == 2         # eps = 0 keeps nonzero sigma
    # (0.9 eps)^2 budget: a tail exactly at eps is not dropped
    assert oracle.truncation_rank([1.0, 1e-6], 1e-6)[0] == 2


def test_add_scale_exact(oracle):  # :127-142
    g = oracle.Rng(18)
    x = g.random_tt(10, 12, 3)
    cancel = oracle.add(x, oracle.scale(x, -1.0))
    assert cancel.rank == 6 and np.linalg.norm(cancel.full()) < 1e-12 * np.linalg.norm(x.full())
    threes = oracle.scale(oracle.TT.constant(4, 4, 1.0), 3.0)
    assert np.allclose(threes.full(), 3.0)
    y = g.random_tt(10, 12, 2)
    s = oracle.add(oracle.scale(x, 0.3), y)
    assert s.rank == 5 and rel(s.full(), 0.3 * x.full() + y.full()) < 1e-13


def test_add_shape_mismatch(oracle):  # :144-147
    g = oracle.Rng(19)
    with pytest.raises(oracle.ShapeError):
        oracle.add(g.random_tt(4, 4, 1), g.random_tt(4, 5, 1))


def test_hadamard(oracle):  # :149-163
    g = oracle.Rng(20)
    x = g.random_tt(9, 11, 2)
    ones = oracle.TT.constant(9, 11, 1.0)
    assert rel(oracle.hadamard(x, ones).full(), x.full()) < 1e-13
    a, b = g.random_tt(9, 11, 1), g.random_tt(9, 11, 1)
    assert oracle.hadamard(a, b).rank == 1
    y = g.random_tt(9, 11, 3)
    p = oracle.hadamard(x, y)
    assert p.rank <= 6 and rel(p.full(), x.full() * y.full()) < 1e-13


def test_norm_and_sum(oracle):  # :165-179
    ones = oracle.TT.constant(4, 4, 1.0)
    assert abs(oracle.norm_fro(ones) - 4.0) <= 4e-14 and abs(oracle.sum_entries(ones) - 16.0) <= 16e-14
    z = oracle.TT.zero(6, 5)
    assert oracle.norm_fro(z) == 0.0 and oracle.sum_entries(z) == 0.0
    g = oracle.Rng(21)
    x = g.random_tt(32, 32, 3)
    d = x.full()
    assert abs(oracle.norm_fro(x) - np.linalg.norm(d)) <= 1e-12 * np.linalg.norm(d)
    assert abs(oracle.sum_entries(x) - d.sum()) <= 1e-12 * np.linalg.norm(d)


def test_apply_core_map(oracle):  # :181-202
    g = oracle.Rng(22)
    x = g.random_tt(8, 6, 3)
    assert rel(oracle.core_map_dense(x, 0, np.eye(8)).full(), x.full()) == 0.0
    shift = np.zeros((8, 8))
    for i in range(8):
        shift[i, (i + 1) % 8] = 1.0
    sh = oracle.core_map_dense(x, 0, shift).full()
    d = x.full()
    for i in range(8):
        assert np.linalg.norm(sh[i] - d[(i + 1) % 8]) == 0.0
    my = g.random_matrix(4, 6)
    mp = oracle.core_map_dense(x, 1, my)
    assert mp.rank == 3 and rel(mp.full(), d @ my.T) < 1e-13
    with pytest.raises(oracle.ShapeError):
        oracle.core_map_dense(x, 0, np.eye(5))


def test_reciprocal_constant_one_iteration(oracle):  # :204-210
    inv, it = oracle.recip(oracle.TT.constant(6, 6, 2.0), 1e-12)
    assert it == 1 and rel(inv.full(), np.full((6, 6), 0.5)) < 1e-13


def test_reciprocal_cos_pattern(oracle):  # :212-226
    n = 24
    i, j = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    A = 1.0 + 0.1 * np.cos(2 * np.pi * (i + 0.3 * j) / n)
    x = oracle.from_full(A, 1e-14)
    inv, it = oracle.recip(x, 1e-10)
    assert 8 <= it <= 12
    res = oracle.hadamard(x, inv).full() - 1.0
    assert np.linalg.norm(res) / n <= 1e-9
    assert rel(inv.full(), 1.0 / A) < 1e-9


def test_reciprocal_zero_entry_fails(oracle):  # :228-233
    A = np.ones((8, 8))
    A[3, 4] = 0.0
    with pytest.raises(oracle.ConvergenceError):
        oracle.recip(oracle.from_full(A, 0.0), 1e-10, 50)


def test_reciprocal_identity_mean_dominated(oracle):  # :235-249
    g = oracle.Rng(23)
    eps = 1e-9
    for _ in range(5):
        bump = g.random_tt(20, 20, 2).full()
        bump *= 0.5 / np.abs(bump).max()
        A = 1.0 + bump
        x = oracle.from_full(A, 1e-14)
        inv, _ = oracle.recip(x, eps)
        rms = np.linalg.norm(oracle.hadamard(x, inv).full() - 1.0) / 20
        assert rms <= 10 * eps
