"""GPU parity of the solver's RhsHooks (swe.hpp:276-282, used by the reference's Dirichlet
and MMS verification cases, cases.cpp:198-220 / :298-344): a fill_ghost hook that pads with
Dirichlet strips through ttsw_ghosted and an extra_source hook, installed on the device
solver and on the oracle solver, run side by side with the same per-step bars as the
periodic runs (test_gpu_parity._run_both)."""
import math

import numpy as np
import pytest

from paper_2408_03483_b200 import ics
from test_gpu_parity import _run_both

pytestmark = pytest.mark.gpu


def _dirichlet_mms_hooks(ctx, oracle, spec, bc):
    """Strips: the IC's periodic ghost values scaled by (1 + t) (time-dependent boundary data);
    source: 1e-3 cos(2 pi t) sin(2 pi x) cos(2 pi y) on every component (rank 1)."""
    n = spec.n
    full = [cx @ cy for cx, cy in spec.ic]
    idx = (np.arange(-3, n + 3)) % n
    ghosted = [f[np.ix_(idx, idx)] for f in full]
    xs = (np.arange(n) + 0.5) / n
    sx_rows = [0, 1, 2, n + 3, n + 4, n + 5]

    def strips(c, t):
        g = ghosted[c] * (1.0 + t)
        return g[sx_rows, :], g[:, sx_rows]

    src_x = np.sin(2 * math.pi * xs)[:, None]
    src_y = np.cos(2 * math.pi * xs)[None, :]

    def install(gs, os_):
        def g_ghost(q, t):
            return [ctx.ghosted(q[c], *bc, *strips(c, t), eps_tt=spec.tol) for c in range(3)]

        def o_ghost(q, t):
            return [oracle.ghosted(q[c], *bc, *strips(c, t), eps_tt=spec.tol) for c in range(3)]

        def g_src(t):
            a = 1e-3 * math.cos(2 * math.pi * t)
            return [ctx.tt(a * src_x, src_y) for _ in range(3)]

        def o_src(t):
            a = 1e-3 * math.cos(2 * math.pi * t)
            return [oracle.TT.from_cores(a * src_x, src_y) for _ in range(3)]

        gs.set_hooks(g_ghost, g_src)
        os_.set_hooks(o_ghost, o_src)
        return gs, os_

    return install


@pytest.mark.parametrize("bc", [(1, 0), (0, 1), (1, 1)])
def test_dirichlet_mms_hooks_linear_match_oracle(ctx, oracle, bc):
    spec = ics.config1(n=48)
    worst, diverged = _run_both(ctx, oracle, spec, 6, hooks=_dirichlet_mms_hooks(ctx, oracle, spec, bc))
    assert diverged is None and worst < 1e-9


def test_dirichlet_mms_hooks_nonlinear_weno_match_oracle(ctx, oracle):
    spec = ics.config3(n=24)
    worst, diverged = _run_both(ctx, oracle, spec, 3, hooks=_dirichlet_mms_hooks(ctx, oracle, spec, (1, 1)))
    assert worst < 1e-6, (worst, diverged)


def test_periodic_hook_is_the_default(ctx, oracle):
    """fill_ghost = ttsw_periodic_ghost and no source reproduces the hook-free solver bitwise."""
    from paper_2408_03483_b200 import capi

    spec = ics.config1(n=32)
    cfg = capi.CrossCfg.make(seed=1, max_rank=spec.cross_max_rank)
    a = capi.Solver(ctx, spec.model, spec.scheme, spec.n, spec.g, spec.f, spec.H, spec.dt, spec.tol, cfg)
    b = capi.Solver(ctx, spec.model, spec.scheme, spec.n, spec.g, spec.f, spec.H, spec.dt, spec.tol, cfg)
    b.set_hooks(lambda q, t: [ctx.periodic_ghost(x) for x in q])
    for s in (a, b):
        s.set_state([ctx.round(ctx.tt(cx, cy), spec.tol) for cx, cy in spec.ic])
        s.step(3)
    assert b.time == pytest.approx(3 * spec.dt) and a.time == b.time
    for x, y in zip(a.state(), b.state()):
        assert np.array_equal(x.full(), y.full())
    b.set_hooks()  # back to periodic, still identical
    a.step(1)
    b.step(1)
    for x, y in zip(a.state(), b.state()):
        assert np.array_equal(x.full(), y.full())


def test_mms_dirichlet_nonlinear_weno_matches_oracle(ctx, oracle):
    """The reference's MMS wiring (cases.hpp:143-171): Dirichlet exact strips on both axes and
    the cell-averaged manufactured source compressed by tt_from_full (Rep::compress) at every
    stage time; device solver vs oracle solver, nonlinear WENO5 at n = 24. The states are
    full-rank (24), so the WENO/LLF crosses split on pivot ties between the two (their
    results agree to the cross tolerance): the bar is absolute, 1e-9 against fields of
    size 0.1-1 (the v = 0 momentum is pure discretisation error, ~1e-7, so a relative bar
    on it would be meaningless), and both runs must sit at the same distance from the exact
    cell averages."""
    import mms_ref

    from paper_2408_03483_b200 import capi

    n, tol, dt = 24, 1e-10, 0.2 / 24
    ic = mms_ref.cell_averages(mms_ref.exact_conserved, n, 0.0)
    gs = capi.Solver(ctx, 1, 2, n, mms_ref.G, mms_ref.F, mms_ref.H, dt, tol, capi.CrossCfg.make(seed=1))
    os_ = oracle.Solver(1, 2, n, mms_ref.G, mms_ref.F, mms_ref.H, dt, tol, oracle.CrossCfg.make(seed=1))
    gs.set_state([ctx.round(ctx.from_full(a, tol), tol) for a in ic])
    os_.set_state([oracle.round_(oracle.from_full(a, tol), tol) for a in ic])

    def fill(lib_ghosted):
        def f(q, t):
            st = mms_ref.ghost_strips(n, t)
            return [lib_ghosted(q[c], 1, 1, st[c][0], st[c][1], eps_tt=tol) for c in range(3)]
        return f

    gs.set_hooks(fill(ctx.ghosted), lambda t: [ctx.from_full(a, tol) for a in mms_ref.cell_averages(mms_ref.mms_source, n, t)])
    os_.set_hooks(fill(oracle.ghosted),
                  lambda t: [oracle.from_full(a, tol) for a in mms_ref.cell_averages(mms_ref.mms_source, n, t)])
    for k in range(3):
        gs.step(1)
        os_.step(1)
        assert gs.time == os_.time
        ex = mms_ref.cell_averages(mms_ref.exact_conserved, n, os_.time)
        for c in range(3):
            a, b = gs.state()[c].full(), os_.state()[c].full()
            assert np.abs(a - b).max() <= 1e-9 * (k + 1), (k, c, np.abs(a - b).max())
            ea, eb = np.abs(a - ex[c]).max(), np.abs(b - ex[c]).max()
            assert eb < 1e-5 and abs(ea - eb) <= 1e-9 * (k + 1), (k, c, ea, eb)


def test_failing_hook_is_a_state_error(ctx):
    """A hook that fails surfaces as StateError at the step (the reference's run_impl wraps
    step failures the same way, harness.cpp); the solver stays usable after clearing it."""
    from paper_2408_03483_b200 import capi

    spec = ics.config1(n=16)
    s = capi.Solver(ctx, spec.model, spec.scheme, spec.n, spec.g, spec.f, spec.H, spec.dt, spec.tol,
                    capi.CrossCfg.make(seed=1))
    s.set_state([ctx.round(ctx.tt(cx, cy), spec.tol) for cx, cy in spec.ic])
    s.set_hooks(None, lambda t: 1 / 0)
    with pytest.raises(capi.StateError):
        s.step(1)
    s.set_hooks()
    s.time = 0.0
    s.step(1)
    assert s.time == pytest.approx(spec.dt)


def test_raising_fill_ghost_and_shared_source_handles(ctx):
    """fill_ghost raising after it received the library's borrowed stage handles is a
    StateError (the borrowed handles are never freed from Python); an extra_source that
    returns the same TT in all three slots is taken over once; a later standalone call on
    the context does not touch the failed solver's traces."""
    import gc

    from paper_2408_03483_b200 import capi

    spec = ics.config1(n=16)
    s = capi.Solver(ctx, spec.model, spec.scheme, spec.n, spec.g, spec.f, spec.H, spec.dt, spec.tol,
                    capi.CrossCfg.make(seed=1))
    s.set_state([ctx.round(ctx.tt(cx, cy), spec.tol) for cx, cy in spec.ic])
    kept = []

    def bad_ghost(q, t):
        kept.extend(q)  # the user keeps the borrowed views: they must not free anything
        raise RuntimeError("boom")

    s.set_hooks(bad_ghost, None)
    with pytest.raises(capi.StateError):
        s.step(1)
    kept.clear()
    gc.collect()
    n = spec.n
    s.set_hooks(None, lambda t: [ctx.zero(n, n)] * 3)  # one handle in three slots
    s.time = 0.0
    s.step(1)
    gc.collect()
    s.set_hooks()
    s.step(1)
    # standalone crosses after a failed/finished step leave the solver's cross trace alone
    s.cross_trace(clear=True)
    four = ctx.constant(16, 12, 4.0)
    ctx.cross(capi.FN_SQRT, [four], four, capi.CrossCfg.make(eps=1e-12, seed=99))
    assert len(s.cross_trace()[0]) == 0
    del s
    gc.collect()
    ctx.cross(capi.FN_SQRT, [four], four, capi.CrossCfg.make(eps=1e-12, seed=99))
