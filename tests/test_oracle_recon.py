"""Oracle pin: reconstruction known-answer tests
(/root/reference/proj/tests/test_reconstruction.cpp:29-495). The dense reference path
(step1_dense / step2_dense, reconstruction.hpp:253-377) is re-implemented here in numpy
as an independent checker of the TT path."""
import math

import numpy as np
import pytest

from parity import rel

U3, U5, W5 = 0, 1, 2
MAP_PAD, MAP_STEP1, MAP_QPOINT, MAP_QSUM, MAP_DIFF = 0, 1, 2, 3, 4


def sine_avg(c, h):
    return (np.cos(2 * np.pi * (c - 0.5 * h)) - np.cos(2 * np.pi * (c + 0.5 * h))) / (2 * np.pi * h)


def mono_avg(deg, c, h):
    a, b = c - 0.5 * h, c + 0.5 * h
    return (b ** (deg + 1) - a ** (deg + 1)) / ((deg + 1) * h)


def line_tt(oracle, v):
    v = np.asarray(v, dtype=float).reshape(-1, 1)
    return oracle.TT.from_cores(v, np.ones((1, 1)))


# --- independent dense restatement of step1_blocks / step2_blocks --------------------
def beta(v):
    c = 13.0 / 12.0
    return [c * (v[2] - 2 * v[3] + v[4]) ** 2 + 0.25 * (3 * v[2] - 4 * v[3] + v[4]) ** 2,
            c * (v[1] - 2 * v[2] + v[3]) ** 2 + 0.25 * (v[1] - v[3]) ** 2,
            c * (v[0] - 2 * v[1] + v[2]) ** 2 + 0.25 * (v[0] - 4 * v[1] + 3 * v[2]) ** 2]


def step1_blocks(t, v, scheme, eps):
    k = t["radius"]
    if scheme != W5:
        out = 0
        for r in range(k + 1):
            for l in range(k + 1):
                out = out + t["step1_ideal"][r] * t["step1_c"][r, l] * v[k - r + l]
        return out
    b = beta(v)
    a = [t["weno_d"][r] / (b[r] + eps) ** 2 for r in range(3)]
    cand = [sum(t["step1_c"][r, l] * v[2 - r + l] for l in range(3)) for r in range(3)]
    return (a[0] * cand[0] + a[1] * cand[1] + a[2] * cand[2]) / (a[0] + a[1] + a[2])


def step2_blocks(t, v, scheme, m, eps):
    k = t["radius"]
    cand = [sum(t["c"][m][r, l] * v[k - r + l] for l in range(k + 1)) for r in range(k + 1)]
    if scheme == U3:
        return 0.5 * cand[0] + 0.5 * cand[1]
    if scheme == U5:
        if m == 1:
            up = sum(t["gamma_plus"][r] * cand[r] for r in range(3))
            um = sum(t["gamma_minus"][r] * cand[r] for r in range(3))
            return t["sigma_plus"] * up - t["sigma_minus"] * um
        return sum(t["gamma"][m][r] * cand[r] for r in range(3))
    b = beta(v)

    def comb(g):
        a = [g[r] / (b[r] + eps) ** 2 for r in range(3)]
        return (a[0] * cand[0] + a[1] * cand[1] + a[2] * cand[2]) / (a[0] + a[1] + a[2])

    if m == 1:
        return t["sigma_plus"] * comb(t["gamma_plus"]) - t["sigma_minus"] * comb(t["gamma_minus"])
    return comb(t["gamma"][m])


def step1_dense(t, g, axis, scheme, side, eps):
    k = t["radius"]
    n = (g.shape[0] if axis == 0 else g.shape[1]) - 6
    base = 3 - k - 1 if side == 0 else 3 - k
    blocks = [g[base + s: base + s + n + 1, :] if axis == 0 else g[:, base + s: base + s + n + 1]
              for s in range(2 * k + 1)]
    if side == 1:
        blocks = blocks[::-1]
    return step1_blocks(t, blocks, scheme, eps)


def step2_dense(t, lines, axis, scheme, eps):
    k, nq = t["radius"], t["nq"]
    n = (lines.shape[0] if axis == 0 else lines.shape[1]) - 6
    blocks = [lines[3 - k + s: 3 - k + s + n, :] if axis == 0 else lines[:, 3 - k + s: 3 - k + s + n]
              for s in range(2 * k + 1)]
    out = np.zeros((n * nq, lines.shape[1]) if axis == 0 else (lines.shape[0], n * nq))
    for m in range(nq):
        vals = step2_blocks(t, blocks, scheme, m, eps)
        if axis == 0:
            out[m::nq, :] = vals
        else:
            out[:, m::nq] = vals
    return out


def dense_faces(oracle, g, axis, scheme, dx, dy):
    t = oracle.tables(scheme)
    e1, e2 = (dx * dx, dy * dy) if axis == 0 else (dy * dy, dx * dx)
    trans = 1 - axis
    return (step2_dense(t, step1_dense(t, g, axis, scheme, 0, e1), trans, scheme, e2),
            step2_dense(t, step1_dense(t, g, axis, scheme, 1, e1), trans, scheme, e2))


# --- KATs ---------------------------------------------------------------------------
def test_gauss_rule(oracle):  # test_reconstruction.cpp:29-48
    t2, t3 = oracle.tables(U3), oracle.tables(U5)
    assert abs(t2["offset"][0] + 0.28867513459481287) <= 1e-15 and t2["weight"][0] == 0.5
    assert abs(t3["offset"][2] - 0.3872983346207417) <= 1e-15 and t3["offset"][1] == 0.0
    assert abs(t3["weight"][0] - 5 / 18) <= 1e-15 and abs(t3["weight"][1] - 8 / 18) <= 1e-15
    for t in (t2, t3):
        assert abs(sum(t["weight"]) - 1.0) <= 1e-15


def test_step1_tables(oracle):  # :50-73
    u3 = oracle.tables(U3)
    assert np.allclose(u3["step1_c"], [[0.5, 0.5], [-0.5, 1.5]], atol=1e-14)
    assert np.allclose(u3["step1_ideal"], [2 / 3, 1 / 3], atol=1e-14)
    u5 = oracle.tables(U5)
    assert np.abs(u5["step1_c"] - np.array([[2, 5, -1], [-1, 5, 2], [2, -7, 11]]) / 6).max() < 1e-14
    assert np.allclose(u5["step1_ideal"], [0.3, 0.6, 0.1], atol=1e-14)
    assert np.abs(u5["step1_row"] - np.array([2, -13, 47, 27, -3]) / 60).max() < 1e-14


def test_tables_preserve_constants(oracle):  # :75-87
    for s in (U3, U5, W5):
        t = oracle.tables(s)
        for m in range(t["nq"]):
            assert np.all(np.abs(t["c"][m].sum(axis=1) - 1) < 1e-12)
            assert abs(t["point_row"][m].sum() - 1) < 1e-12 and abs(t["gamma"][m].sum() - 1) < 1e-12
        assert abs(t["step1_row"].sum() - 1) < 1e-12 and abs(t["step1_ideal"].sum() - 1) < 1e-12


def test_printed_rationals(oracle):  # :89-134
    u3 = oracle.tables(U3)
    p1 = np.array([[808 / 627, -390 / 1351], [390 / 1351, 961 / 1351]])
    p2 = np.array([[961 / 1351, 390 / 1351], [-390 / 1351, 808 / 627]])
    assert np.abs(u3["c"][0] - p1).max() < 2e-6 and np.abs(u3["c"][1] - p2).max() < 2e-6
    u5 = oracle.tables(U5)
    q1 = np.array([[4725 / 2927, -2051 / 2438, 249 / 1097], [249 / 1097, 14 / 15, -467 / 2913],
                   [-467 / 2913, 366 / 517, 2209 / 4883]])
    q2 = np.array([[23 / 24, 1 / 12, -1 / 24], [-1 / 24, 13 / 12, -1 / 24], [-1 / 24, 1 / 12, 23 / 24]])
    assert np.abs(u5["c"][0] - q1).max() < 2e-6 and np.abs(u5["c"][1] - q2).max() < 1e-14
    assert np.abs(u5["c"][2] - q1[::-1, ::-1]).max() < 2e-6
    assert np.abs(u5["gamma"][0] - [882 / 6305, 403 / 655, 463 / 1891]).max() < 1e-6
    assert np.abs(u5["gamma"][1] - [-9 / 80, 49 / 40, -9 / 80]).max() < 1e-12
    rec = u5["sigma_plus"] * u5["gamma_plus"] - u5["sigma_minus"] * u5["gamma_minus"]
    assert np.abs(rec - [-9 / 80, 49 / 40, -9 / 80]).max() < 1e-14
    assert abs(u5["sigma_plus"] - u5["sigma_minus"] - 1) < 1e-15


def test_step1_constant_and_linear(oracle):  # :136-154
    n = 12
    for s in (U3, U5):
        for side in (0, 1):
            out = oracle.core_map(line_tt(oracle, np.full(n + 6, 4.25)), 0, MAP_STEP1, s, side, n).full()
            assert np.abs(out - 4.25).max() < 1e-13
    lin = np.arange(-3, n + 3, dtype=float)
    out = oracle.core_map(line_tt(oracle, lin), 0, MAP_STEP1, U3, 0, n).full()[:, 0]
    assert np.allclose(out, np.arange(n + 1) - 0.5, rtol=1e-14, atol=1e-14)


def test_step1_upwind5_quartic_exact(oracle):  # :156-169
    n, h = 16, 1.0 / 16
    for deg in range(5):
        line = [mono_avg(deg, (i + 0.5) * h, h) for i in range(-3, n + 3)]
        for side in (0, 1):
            out = oracle.core_map(line_tt(oracle, line), 0, MAP_STEP1, U5, side, n).full()[:, 0]
            exact = (np.arange(n + 1) * h) ** deg
            assert np.allclose(out, exact, rtol=1e-12, atol=1e-12)


def test_smoothness_and_weights(oracle):  # :171-203
    assert np.all(oracle.smoothness([2, 2, 2, 2, 2]) == 0)
    assert np.allclose(oracle.smoothness([0, 1, 2, 3, 4]), 1.0, rtol=1e-14)
    b = oracle.smoothness([0, 0, 0, 1, 1])
    assert b[2] == 0 and b[0] > 1
    ideal = [0.3, 0.6, 0.1]
    assert np.allclose(oracle.weno_weights([0, 0, 0], ideal, 1e-4), ideal, rtol=1e-14)
    assert np.allclose(oracle.weno_weights([7.5, 7.5, 7.5], ideal, 1e-4), ideal, rtol=1e-14)
    assert oracle.weno_weights([0, 0, 1e6], ideal, 1e-4)[2] <= 1e-19


def test_step2_constant_and_linear(oracle):  # :205-223
    n = 10
    for s in (U3, U5, W5):
        out = oracle.core_map(line_tt(oracle, np.full(n + 6, -1.75)), 0, MAP_QPOINT, s, 0, n).full()
        assert np.abs(out + 1.75).max() < 1e-13
    off = oracle.tables(U3)["offset"]
    lin = np.arange(-3, n + 3, dtype=float)
    out = oracle.core_map(line_tt(oracle, lin), 0, MAP_QPOINT, U3, 0, n).full()[:, 0]
    for m in range(2):
        assert np.allclose(out[m::2], np.arange(n) + off[m], rtol=1e-13, atol=1e-13)
    with pytest.raises(oracle.InputError):
        oracle.weno_step2([0, 1, 2, 3, 4], 3, 0.0)


def test_step2_split_formula_equals_signed(oracle):  # :225-247 (table identity)
    t = oracle.tables(U5)
    g = np.random.default_rng(41)
    for _ in range(20):
        v = g.standard_normal(5)
        split = step2_blocks(t, list(v), U5, 1, 0.0)
        direct = sum(t["gamma"][1][r] * sum(t["c"][1][r, l] * v[2 - r + l] for l in range(3)) for r in range(3))
        assert abs(split - direct) < 1e-12 * (1 + abs(direct))


def test_faces_constant(oracle):  # :249-258 (TT path)
    for s in (U3, U5, W5):
        g = oracle.TT.constant(14, 12, 0.7)
        for axis in (0, 1):
            mi, pl = oracle.reconstruct_faces(g, axis, s, 1e-11, dx=0.1, dy=0.1)
            assert np.abs(mi.full() - 0.7).max() < 1e-12 and np.abs(pl.full() - 0.7).max() < 1e-12


def test_tt_linear_equals_dense(oracle):  # :357-377
    g = oracle.Rng(42)
    n = 20
    interior = g.random_tt(n, n, 3)
    ghosted = oracle.periodic_ghost(interior)
    gd = ghosted.full()
    for s in (U3, U5):
        for axis in (0, 1):
            mi, pl = oracle.reconstruct_faces(ghosted, axis, s)
            dm, dp = dense_faces(oracle, gd, axis, s, 1.0 / n, 1.0 / n)
            assert mi.rank == pl.rank == 3
            assert rel(mi.full(), dm) < 1e-12 and rel(pl.full(), dp) < 1e-12


def test_tt_linear_rank1_stays_rank1(oracle):  # :379-394
    g = oracle.Rng(43)
    ghosted = oracle.periodic_ghost(g.random_tt(16, 16, 1))
    mi, pl = oracle.reconstruct_faces(ghosted, 0, U5)
    assert mi.rank == 1 and pl.rank == 1
    c = oracle.reconstruct_faces(oracle.TT.constant(22, 22, 3.5), 1, U5)[0]
    assert c.rank == 1 and np.abs(c.full() - 3.5).max() < 1e-13


def test_tt_weno_matches_dense_smooth(oracle):  # :396-421
    n, h = 24, 1.0 / 24
    x = sine_avg((np.arange(n) + 0.5) * h, h)
    interior = np.outer(x, 2.0 + x)
    tt = oracle.from_full(interior, 1e-13)
    ghosted = oracle.periodic_ghost(tt)
    gd = ghosted.full()
    for axis in (0, 1):
        mi, pl = oracle.reconstruct_faces(ghosted, axis, W5, 1e-10, dx=h, dy=h)
        dm, dp = dense_faces(oracle, gd, axis, W5, h, h)
        denom = math.sqrt(dm.size)
        assert np.linalg.norm(mi.full() - dm) / denom <= 1e-8
        assert np.linalg.norm(pl.full() - dp) / denom <= 1e-8


def test_tt_weno_constant_rank1(oracle):  # :423-432
    mi, _ = oracle.reconstruct_faces(oracle.TT.constant(26, 26, -2.25), 0, W5, 1e-11)
    assert mi.rank == 1 and np.abs(mi.full() + 2.25).max() < 1e-12


def test_operator_difference_and_pad(oracle):  # :478-495
    d = oracle.core_map(line_tt(oracle, [1, 3, 6, 10, 15]), 0, MAP_DIFF, 0, 0, 4).full()[:, 0]
    assert d[0] == 2.0 and d[3] == 5.0
    p = oracle.core_map(line_tt(oracle, [0, 1, 2, 3, 4]), 0, MAP_PAD, 0, 0, 5).full()[:, 0]
    assert p[0] == 2.0 and p[3] == 0.0 and p[3 + 5] == 0.0 and p[3 + 7] == 2.0


def test_quadrature_sum_of_points_is_identity_for_linear_schemes(oracle):
    # sum_q w_q point_row[q] == e_k: the transverse map round trip preserves averages
    for s in (U3, U5):
        t = oracle.tables(s)
        comb = sum(t["weight"][q] * t["point_row"][q] for q in range(t["nq"]))
        e = np.zeros(2 * t["radius"] + 1)
        e[t["radius"]] = 1.0
        assert np.abs(comb - e).max() < 1e-14
