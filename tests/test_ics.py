"""BASELINE initial conditions and run constants."""
import math

import numpy as np

from paper_2408_03483_b200 import ics


def test_mt19937_64_matches_libstdcxx(oracle):
    g = oracle.Rng(240803483)
    m = ics.MT19937_64(240803483)
    import ctypes as C

    lib = oracle.lib()
    assert [lib.ttor_rng_raw(g.h) for _ in range(1000)] == [m.next_u64() for _ in range(1000)]


def test_uniform_is_53bit():
    m = ics.MT19937_64(5)
    x = m.next_u64()
    assert ics.MT19937_64(5).uniform() == (x >> 11) * 2.0 ** -53


def test_c1_constants_and_rank(oracle):
    s = ics.config1()
    assert s.n == 256 and s.scheme == 0 and s.model == 0 and s.tol == 1e-8 and s.steps == 100
    assert abs(s.dt - 1.5625e-3) < 1e-18
    ranks = [oracle.round_(oracle.TT.from_cores(cx, cy), s.tol).rank for cx, cy in s.ic]
    assert ranks == [1, 1, 1]
    eta = s.ic[0][0] @ s.ic[0][1]
    assert abs(eta.max() - 0.01) < 1e-4 and eta.min() > 0


def test_c2_geostrophic_balance():
    s = ics.config2(n=128)
    assert s.f == 10.0 and s.scheme == 1 and s.tol == 1e-10 and abs(s.dt - 0.4 / 128) < 1e-18
    eta, u, v = [cx @ cy for cx, cy in s.ic]
    # discrete geostrophic check: u ~ -(g/f) d(eta)/dy, v ~ (g/f) d(eta)/dx (centred differences)
    h = 1.0 / 128
    dedy = (np.roll(eta, -1, 1) - np.roll(eta, 1, 1)) / (2 * h)
    dedx = (np.roll(eta, -1, 0) - np.roll(eta, 1, 0)) / (2 * h)
    assert np.linalg.norm(u + 0.1 * dedy) < 5e-2 * np.linalg.norm(u)
    assert np.linalg.norm(v - 0.1 * dedx) < 5e-2 * np.linalg.norm(v)


def test_c3_bumps_and_rank(oracle):
    s = ics.config3(n=256)
    rng = ics.MT19937_64(ics.SEEDS[3])
    for _ in range(4):
        A, w = rng.uniform_range(0.02, 0.1), rng.uniform_range(0.03, 0.1)
        assert 0.02 <= A <= 0.1 and 0.03 <= w <= 0.1
        rng.uniform(); rng.uniform()
    h = s.ic[0][0] @ s.ic[0][1]
    assert h.min() >= 1.0 and s.ic[0][0].shape[1] == 5
    assert oracle.round_(oracle.TT.from_cores(*s.ic[0]), 1e-10).rank <= 5
    assert abs(s.dt - 0.4 / 256 / math.sqrt(h.max())) < 1e-15


def test_c4_noise_is_low_rank_and_scaled():
    s = ics.config4(n=64)
    assert s.cross_max_rank == 64 and s.scheme == 2 and s.f == 10.0
    assert s.ic[0][0].shape[1] == 1 + 2 + 4  # constant + two vortices + rank-4 noise


def test_c5_members_differ():
    a, b = ics.config5_member(0, n=32), ics.config5_member(1, n=32)
    assert not np.allclose(a.ic[0][0], b.ic[0][0])
