"""GPU parity of tt_ghosted with Dirichlet strips (cases.cpp:298-344) through the C ABI
(ttsw_ghosted) against the oracle (oracle/src/swe.hpp ghosted) and the dense restatement
in ghost_ref.py. Bars: unrounded results exact to 1e-13 (pads and strips are copies and
one addition each); rounded results with the oracle's rank and within 10 eps_tt + 1e-13."""
import numpy as np
import pytest

from ghost_ref import case, dense_ghosted
from paper_2408_03483_b200 import capi
from parity import rel

pytestmark = pytest.mark.gpu

BCS = [(0, 0), (1, 0), (0, 1), (1, 1)]


@pytest.mark.parametrize("bc", BCS)
def test_ghosted_matches_oracle(ctx, oracle, bc):
    rng = np.random.default_rng(70 + 2 * bc[0] + bc[1])
    for nx, ny, r in ((9, 7, 2), (64, 40, 5), (256, 256, 12), (1030, 700, 9)):
        cx, cy, sx, sy = case(rng, nx, ny, r)
        want = dense_ghosted(cx @ cy, *bc, sx, sy)
        g = ctx.ghosted(ctx.tt(cx, cy), *bc, sx, sy, eps_tt=-1.0)
        assert g.shape[:2] == (nx + 6, ny + 6)
        assert np.abs(g.full() - want).max() <= 1e-13 * max(1.0, np.abs(want).max())
        o = oracle.ghosted(oracle.TT.from_cores(cx, cy), *bc, sx, sy, eps_tt=1e-10)
        gr = ctx.ghosted(ctx.tt(cx, cy), *bc, sx, sy, eps_tt=1e-10)
        assert gr.rank == o.rank, (nx, ny, gr.rank, o.rank)
        assert rel(gr.full(), o.full()) <= 10 * 1e-10 + 1e-13
        assert np.linalg.norm(gr.full() - want) <= 1e-10 * np.linalg.norm(want) * (1 + 1e-9)


def test_ghosted_smooth_exact_strips_keep_low_rank(ctx, oracle):
    """A separable field with strips taken from the same field (the exact-solution case):
    the rounded ghosted TT stays at the field's rank, as in the reference."""
    nx, ny = 128, 96
    xs = (np.arange(-3, nx + 3) + 0.5) / nx
    ys = (np.arange(-3, ny + 3) + 0.5) / ny
    full = np.outer(np.sin(2 * np.pi * xs), np.cos(2 * np.pi * ys)) + 1.0
    a = full[3:-3, 3:-3]
    sx = full[[0, 1, 2, nx + 3, nx + 4, nx + 5], :]
    sy = full[:, [0, 1, 2, ny + 3, ny + 4, ny + 5]]
    u, s, vt = np.linalg.svd(a)
    cx, cy = u[:, :2] * s[:2], vt[:2]
    g = ctx.ghosted(ctx.tt(cx, cy), 1, 1, sx, sy, eps_tt=1e-12)
    o = oracle.ghosted(oracle.TT.from_cores(cx, cy), 1, 1, sx, sy, eps_tt=1e-12)
    assert g.rank == o.rank == 2
    assert rel(g.full(), full) < 1e-11


def test_ghosted_errors(ctx):
    x = ctx.tt(np.ones((8, 1)), np.ones((1, 6)))
    with pytest.raises(capi.ShapeError):
        ctx.ghosted(x, 1, 0, np.ones((6, 6)))
    with pytest.raises(capi.InputError):
        ctx.ghosted(x, 2, 0)
    bad = np.ones((6, 12))
    bad[2, 3] = np.inf
    with pytest.raises(capi.InputError):
        ctx.ghosted(x, 1, 0, bad)
