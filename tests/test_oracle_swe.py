"""Oracle pin: SWE-level known-answer tests (/root/reference/proj/tests/test_swe.cpp:31-465)
restricted to the TT path, plus an independent dense numpy finite-volume rhs used as the
checker of the oracle's TT rhs on the linear model (test_swe.cpp:271-309 analogue)."""
import numpy as np
import pytest

from parity import rel
from test_oracle_recon import dense_faces

LIN, NONLIN = 0, 1
U3, U5, W5 = 0, 1, 2


def scalar(oracle, v):
    return oracle.TT.from_cores(np.array([[float(v)]]), np.array([[1.0]]))


def test_physical_flux_linear_point_values(oracle):  # test_swe.cpp:31-43
    u = [scalar(oracle, 1.0), scalar(oracle, 2.0), scalar(oracle, 3.0)]
    f = [t.full()[0, 0] for t in oracle.physical_flux(u, 0, LIN, 10.0, 1e-4, 1000.0, -1.0)]
    assert abs(f[0] - 2000.0) <= 2000e-14 and abs(f[1] - 10.0) <= 1e-13 and f[2] == 0.0
    g = [t.full()[0, 0] for t in oracle.physical_flux(u, 1, LIN, 10.0, 1e-4, 1000.0, -1.0)]
    assert abs(g[0] - 3000.0) <= 3000e-14 and g[1] == 0.0 and abs(g[2] - 10.0) <= 1e-13


def test_physical_flux_nonlinear_rest_state(oracle):  # :45-53
    u = [scalar(oracle, 1000.0), scalar(oracle, 0.0), scalar(oracle, 0.0)]
    f = [t.full()[0, 0] for t in oracle.physical_flux(u, 0, NONLIN, 10.0, 0.0, 1000.0, 1e-12)]
    assert f[0] == 0.0 and abs(f[1] - 0.5 * 10 * 1e6) <= 5e6 * 1e-14 and f[2] == 0.0


def smooth(n, mean, amp, kx, ky):
    i = (np.arange(n) + 0.5) / n
    return mean + amp * np.outer(np.sin(2 * np.pi * kx * i), np.cos(2 * np.pi * ky * i))


def test_physical_flux_nonlinear_tt_tracks_dense(oracle):  # :55-74
    n, eps, g = 24, 1e-9, 2.0
    h, hu, hv = smooth(n, 1.0, 0.2, 1, 2), smooth(n, 0.1, 0.05, 2, 1), smooth(n, -0.05, 0.04, 1, 1)
    ut = [oracle.from_full(a, 1e-14) for a in (h, hu, hv)]
    for axis in (0, 1):
        ft = oracle.physical_flux(ut, axis, NONLIN, g, 0.0, 1.0, eps)
        if axis == 0:
            fd = [hu, hu * hu / h + 0.5 * g * h * h, hu * hv / h]
        else:
            fd = [hv, hv * hu / h, hv * hv / h + 0.5 * g * h * h]
        for c in range(3):
            assert np.linalg.norm(ft[c].full() - fd[c]) / n <= 10 * eps


def dense_linear_rhs(oracle, q, scheme, g, f, H):
    """Independent dense FV rhs (swe.hpp:362-423 with DenseRep semantics, periodic)."""
    n = q[0].shape[0]
    dx = dy = 1.0 / n
    t = oracle.tables(scheme)
    pad = lambda a: np.pad(a, 3, mode="wrap")
    gh = [pad(a) for a in q]
    div = [np.zeros((n, n)) for _ in range(3)]
    lam = np.sqrt(g * H)
    for axis in (0, 1):
        faces = [dense_faces(oracle, x, axis, scheme, dx, dy) for x in gh]
        um = [fc[0] for fc in faces]
        up = [fc[1] for fc in faces]
        def flux(u):
            z = np.zeros_like(u[0])
            return [H * u[1], g * u[0], z] if axis == 0 else [H * u[2], z, g * u[0]]
        fm, fp = flux(um), flux(up)
        nq = t["nq"]
        for c in range(3):
            fh = 0.5 * fm[c] + 0.5 * fp[c] - 0.5 * lam * (up[c] - um[c])
            if axis == 0:  # faces (n+1) x (n nq): sum quadrature over columns, difference over rows
                integ = sum(t["weight"][m] * fh[:, m::nq] for m in range(nq))
                div[c] += (integ[1:, :] - integ[:-1, :]) / dx
            else:
                integ = sum(t["weight"][m] * fh[m::nq, :] for m in range(nq))
                div[c] += (integ[:, 1:] - integ[:, :-1]) / dy
    src = [np.zeros((n, n)), f * q[2], -f * q[1]]
    return [-div[c] + src[c] for c in range(3)]


@pytest.mark.parametrize("scheme", [U3, U5])
def test_tt_rhs_matches_dense_linear(oracle, scheme):  # :271-309 analogue
    n, g, f, H, tol = 32, 1.0, 10.0, 1.0, 1e-12
    q = [smooth(n, 0.0, 0.01, 1, 1), smooth(n, 0.0, 0.02, 1, 2), smooth(n, 0.0, 0.015, 2, 1)]
    s = oracle.Solver(LIN, scheme, n, g, f, H, 1e-3, tol)
    s.set_state([oracle.from_full(a, 1e-14) for a in q])
    rt = s.rhs()
    rd = dense_linear_rhs(oracle, q, scheme, g, f, H)
    for c in range(3):
        assert np.linalg.norm(rt[c].full() - rd[c]) <= 50 * tol * np.linalg.norm(rd[c]) + 1e-12


def test_constant_state_zero_tendency(oracle):  # :193-227 (TT half)
    n, g, H, eps = 20, 10.0, 1.0, 1e-10
    s = oracle.Solver(NONLIN, U5, n, g, 0.0, H, 1e-3, eps)
    s.set_state([oracle.TT.constant(n, n, H), oracle.TT.zero(n, n), oracle.TT.zero(n, n)])
    r = s.rhs()
    flux_scale = 0.5 * g * H * H * n
    for c in range(3):
        assert oracle.norm_fro(r[c]) / n <= eps * flux_scale


def test_rest_state_fixed_point(oracle):  # :422-445 (TT path, WENO5)
    n, g, H = 16, 10.0, 1.0
    s = oracle.Solver(NONLIN, W5, n, g, 0.0, H, 1e-9, 1e-10)
    s.set_state([oracle.TT.constant(n, n, H), oracle.TT.zero(n, n), oracle.TT.zero(n, n)])
    s.step(1)
    st = s.state()
    assert np.abs(st[0].full() - H).max() < 1e-10 and np.abs(st[1].full()).max() < 1e-10


def test_dt_must_be_positive(oracle):  # :311-345 (dt validation)
    s = oracle.Solver(LIN, U3, 16, 1.0, 0.0, 1.0, 0.0, 1e-8)
    s.set_state([oracle.TT.constant(16, 16, 1.0), oracle.TT.zero(16, 16), oracle.TT.zero(16, 16)])
    with pytest.raises(oracle.StateError):
        s.step(1)


def test_nonlinear_mass_conserved_to_rounding(oracle):  # :386-420 analogue (TT, periodic)
    from paper_2408_03483_b200 import ics

    spec = ics.config3(n=16)
    s = oracle.Solver(spec.model, spec.scheme, spec.n, spec.g, spec.f, spec.H, spec.dt, spec.tol,
                      oracle.CrossCfg.make(seed=1))
    s.set_state([oracle.round_(oracle.TT.from_cores(cx, cy), spec.tol) for cx, cy in spec.ic])
    m0 = oracle.sum_entries(s.state()[0])
    s.step(2)
    m1 = oracle.sum_entries(s.state()[0])
    # periodic flux form conserves mass exactly; TT rounding perturbs it at tol * ||h||
    assert abs(m1 - m0) <= 20 * spec.tol * oracle.norm_fro(s.state()[0]) * spec.n


def test_linear_ssprk3_run_is_deterministic_and_traced(oracle):
    from paper_2408_03483_b200 import ics

    spec = ics.config1(n=32)
    runs = []
    for _ in range(2):
        s = oracle.Solver(spec.model, spec.scheme, spec.n, spec.g, spec.f, spec.H, spec.dt, spec.tol)
        s.set_state([oracle.round_(oracle.TT.from_cores(cx, cy), spec.tol) for cx, cy in spec.ic])
        s.step(3)
        tr, mg, ka = s.trace()
        assert len(tr) == 3 * 24  # 24 roundings per linear step (swe.hpp:420-452)
        runs.append((tr, [t.full() for t in s.state()]))
    assert np.array_equal(runs[0][0], runs[1][0])
    for a, b in zip(runs[0][1], runs[1][1]):
        assert np.array_equal(a, b)


def test_eps_policy_schedule_follows_the_formula(oracle):
    """Policy mode (swe.hpp:134-183, harness.cpp:108-116): before each step the schedule is
    eps_var[c] = min(clip, C_eps V^(1/2) dx^(p-1/2) / ||q_c||_F) (clip for a vanishing
    component) and eps_global = C_eps V^(1/2) dx^(p-1/2) / max_c ||q_c||_F."""
    import math

    from paper_2408_03483_b200 import ics

    spec = ics.config1(n=32)
    s = oracle.Solver(spec.model, spec.scheme, spec.n, spec.g, spec.f, spec.H, spec.dt, spec.tol,
                      oracle.CrossCfg.make(seed=1, max_rank=spec.cross_max_rank))
    s.set_state([oracle.round_(oracle.TT.from_cores(cx, cy), spec.tol) for cx, cy in spec.ic])
    c_eps, order, clip = 2e-3, 3, 1e-3
    s.set_eps_policy(c_eps, order=order, volume=1.0, clip=clip)
    for _ in range(2):
        norms = [float(np.linalg.norm(t.full())) for t in s.state()]
        s.step(1)
        scale = c_eps * math.pow(1.0 / spec.n, order - 0.5)
        want = [clip if q <= 0 else min(clip, scale / q) for q in norms] + [scale / max(norms)]
        got = s.eps()
        assert np.allclose(got, want, rtol=1e-12, atol=0), (got, want)


@pytest.mark.parametrize("bc", [(0, 0), (1, 0), (0, 1), (1, 1)])
def test_oracle_ghosted_matches_dense(oracle, bc):
    """tt_ghosted (cases.cpp:298-344): pads + Dirichlet strips, unrounded and rounded."""
    from ghost_ref import case, dense_ghosted

    rng = np.random.default_rng(40 + 2 * bc[0] + bc[1])
    for nx, ny, r in ((9, 7, 2), (20, 33, 4)):
        cx, cy, sx, sy = case(rng, nx, ny, r)
        a = cx @ cy
        want = dense_ghosted(a, *bc, sx, sy)
        x = oracle.TT.from_cores(cx, cy)
        got = oracle.ghosted(x, *bc, sx, sy, eps_tt=-1.0)
        assert got.shape[:2] == (nx + 6, ny + 6)
        assert np.abs(got.full() - want).max() <= 1e-13 * max(1.0, np.abs(want).max())
        rounded = oracle.ghosted(x, *bc, sx, sy, eps_tt=1e-10)
        assert np.linalg.norm(rounded.full() - want) <= 1e-10 * np.linalg.norm(want) * (1 + 1e-9)
        if bc == (0, 0):
            assert rounded.rank == r * 1  # all-periodic: no strip, no rounding


def test_oracle_solver_hooks(oracle):
    """RhsHooks (swe.hpp:276-282): a periodic fill_ghost hook is the default bitwise; the
    hooks see the stage times t, t+dt, t+dt/2 (swe.hpp:441-448); a failing hook is a StateError."""
    from paper_2408_03483_b200 import ics

    spec = ics.config1(n=16)

    def make():
        s = oracle.Solver(spec.model, spec.scheme, spec.n, spec.g, spec.f, spec.H, spec.dt, spec.tol)
        s.set_state([oracle.round_(oracle.TT.from_cores(cx, cy), spec.tol) for cx, cy in spec.ic])
        return s

    a, b = make(), make()
    times = []

    def ghost(q, t):
        times.append(t)
        return [oracle.periodic_ghost(x) for x in q]

    b.set_hooks(ghost)
    a.step(2)
    b.step(2)
    for x, y in zip(a.state(), b.state()):
        assert np.array_equal(x.full(), y.full())
    dt = spec.dt
    assert np.allclose(times, [0, dt, dt / 2, dt, 2 * dt, 1.5 * dt], rtol=1e-12, atol=0)
    assert b.time == pytest.approx(2 * dt)
    c = make()
    c.set_hooks(None, lambda t: 1 / 0)
    with pytest.raises(oracle.StateError):
        c.step(1)


def test_oracle_mms_dirichlet_tracks_exact_solution(oracle):
    """MMS wiring through the hooks (cases.hpp:143-171): with the manufactured source and
    exact Dirichlet strips the oracle stays on the exact cell averages to discretisation
    error; without the source it drifts by O(omega A t)."""
    import mms_ref

    n, tol, dt = 24, 1e-10, 0.2 / 24
    ic = mms_ref.cell_averages(mms_ref.exact_conserved, n, 0.0)

    def run(with_source):
        s = oracle.Solver(1, 2, n, mms_ref.G, mms_ref.F, mms_ref.H, dt, tol)
        s.set_state([oracle.round_(oracle.from_full(a, tol), tol) for a in ic])

        def fill(q, t):
            st = mms_ref.ghost_strips(n, t)
            return [oracle.ghosted(q[c], 1, 1, st[c][0], st[c][1], eps_tt=tol) for c in range(3)]

        src = (lambda t: [oracle.from_full(a, tol) for a in mms_ref.cell_averages(mms_ref.mms_source, n, t)])
        s.set_hooks(fill, src if with_source else None)
        s.step(2)
        ex = mms_ref.cell_averages(mms_ref.exact_conserved, n, s.time)
        return max(np.abs(s.state()[c].full() - ex[c]).max() for c in range(3))

    e_src, e_none = run(True), run(False)
    assert e_src < 1e-5
    assert e_none > 20 * e_src
