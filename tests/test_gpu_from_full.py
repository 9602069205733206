"""GPU parity of the device tt_from_full (tt.hpp:82-97; TTRep::compress, swe.hpp:93-95)
against the oracle's restatement (oracle/src/tt.hpp tt_from_full) and the reference's own
KATs (proj/tests/test_tt.cpp:13-75). Bars: identical truncation rank unless the decision
is ill-posed at roundoff (parity.rank_mismatch_is_ill_posed), dense results within
10 eps + 1e-13 relative of the oracle's, and the reference's error bound
||A - full(result)||_F <= eps ||A||_F."""
import numpy as np
import pytest

from paper_2408_03483_b200 import capi
from parity import rank_mismatch_is_ill_posed, rel

pytestmark = pytest.mark.gpu


def test_from_full_kats(ctx, oracle):
    # rank-1 outer product round-trips exactly (test_tt.cpp:13-21)
    rng = oracle.Rng(11)
    a = rng.random_matrix(8, 1)
    b = rng.random_matrix(8, 1)
    A = a @ b.T
    t = ctx.from_full(A, 1e-12)
    assert t.rank == 1
    assert rel(t.full(), A) < 1e-14
    # zero matrix is the canonical rank-1 zero (test_tt.cpp:23-29)
    z = ctx.from_full(np.zeros((16, 16)), 1e-12)
    assert z.rank == 1
    cx, cy = z.cores()
    assert np.linalg.norm(cx) == 0.0 and np.linalg.norm(cy) == 0.0
    # sum of three outer products has rank 3 (test_tt.cpp:31-47)
    rng = oracle.Rng(12)
    A = np.zeros((32, 32))
    for _ in range(3):
        u = rng.random_matrix(32, 1)
        v = rng.random_matrix(32, 1)
        A += u @ v.T
    t = ctx.from_full(A, 1e-12)
    assert t.rank == 3
    assert np.linalg.norm(t.full() - A) <= 1e-12 * np.linalg.norm(A)
    # non-finite input and negative eps are InputErrors (test_tt.cpp:49-53)
    A = np.ones((4, 4))
    A[1, 2] = np.nan
    with pytest.raises(capi.InputError):
        ctx.from_full(A, 1e-10)
    with pytest.raises(capi.InputError):
        ctx.from_full(np.ones((4, 4)), -1.0)
    # tt_from_full(A, 0) is lossless (test_tt.cpp:69-75)
    rng = oracle.Rng(13)
    for n in (1, 3, 17, 64, 128):
        A = rng.random_matrix(n, n)
        assert rel(ctx.from_full(A, 0.0).full(), A) < 1e-12


@pytest.mark.parametrize("m,n", [(1, 1), (1, 37), (37, 1), (7, 5), (5, 7), (64, 64), (200, 130), (130, 200),
                                 (300, 300), (515, 260)])
def test_from_full_matches_oracle(ctx, oracle, m, n):
    rng = np.random.default_rng(m * 1000 + n)
    for trial in range(3):
        k = min(m, n)
        u, _ = np.linalg.qr(rng.standard_normal((m, k)))
        v, _ = np.linalg.qr(rng.standard_normal((n, k)))
        s = np.logspace(0, -14, k) * rng.uniform(0.5, 2.0, k)
        A = (u * s) @ v.T
        eps = 10.0 ** rng.uniform(-12, -2)
        g, info = ctx.from_full(A, eps, with_info=True)
        o = oracle.from_full(A, eps)
        assert (info.m, info.n, info.r_in) == (m, n, k)
        if g.rank != o.rank:
            sv = oracle.svd_values(A)
            ko = oracle.truncation_rank(sv, eps)
            assert ko == o.rank
            assert rank_mismatch_is_ill_posed(k, info.margin, info.margin, info.kappa, info.kappa, eps), \
                (m, n, trial, g.rank, o.rank, info.margin)
            continue
        assert rel(g.full(), o.full()) <= 10 * eps + 1e-13
        assert np.linalg.norm(g.full() - A) <= eps * np.linalg.norm(A) * (1 + 1e-9)


def test_from_full_initial_condition(ctx, oracle):
    """A smooth non-separable field (the shape a dense IC takes, cf. test_tt.cpp:212-218)."""
    n = 256
    i = np.arange(n)[:, None]
    j = np.arange(n)[None, :]
    A = 1.0 + 0.1 * np.cos(2.0 * np.pi * (i + 0.3 * j) / n) + 0.05 * np.exp(-((i - 100.0) ** 2 + (j - 80.0) ** 2) / 400.0)
    for eps in (1e-14, 1e-10, 1e-6):
        g = ctx.from_full(A, eps)
        o = oracle.from_full(A, eps)
        assert g.rank == o.rank
        assert rel(g.full(), o.full()) <= 10 * eps + 1e-13
        assert np.linalg.norm(g.full() - A) <= eps * np.linalg.norm(A) * (1 + 1e-9)
