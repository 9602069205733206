"""TEST INFRASTRUCTURE ONLY — numpy restatement of the reference's full-tensor path (the
`DenseRep` plugin, /root/reference/proj/include/ttsw/swe.hpp:45-80, driven through
rhs<Rep> swe.hpp:362-423 and ssprk3<Rep> swe.hpp:428-454) for the parity tests of the
device DenseRep path (ttsw_dense_*). Only tests/ may import it.

Followed op for op:
* ghosts: dense_ghosted (proj/src/cases.cpp:271-296) — periodic wrap, or the exact ghost
  averages on DirichletExact axes (passed in as the ttsw_ghosted strips);
* faces: reconstruct_faces (reconstruction.hpp:412-423) = step2_dense(step1_dense(...))
  with step1_blocks / step2_blocks (reconstruction.hpp:253-323), WENO eps dx^2 / dy^2;
* physical_flux (swe.hpp:190-213) with DenseRep ops (cwiseProduct, cwiseInverse);
* face_wave_speed DenseRep branch (swe.hpp:329-339): a scalar, max over both sides,
  StateError on h <= 0; the linear speed sqrt(gH) (swe.hpp:217);
* llf_flux with a scalar speed (swe.hpp:235-248);
* quadrature_sum_matrix / interface_difference_matrix (reconstruction.hpp:454-470)
  applied along the transverse / normal axis; the rhs assembly (swe.hpp:397-421).
The reconstruction tables are the oracle's (pyoracle.tables, reconstruction.hpp:113-171).
"""
import numpy as np

G = 3
U3, U5, W5 = 0, 1, 2


class StateError(Exception):
    pass


def _beta(v):
    c = 13.0 / 12.0
    return [c * (v[2] - 2 * v[3] + v[4]) ** 2 + 0.25 * (3 * v[2] - 4 * v[3] + v[4]) ** 2,
            c * (v[1] - 2 * v[2] + v[3]) ** 2 + 0.25 * (v[1] - v[3]) ** 2,
            c * (v[0] - 2 * v[1] + v[2]) ** 2 + 0.25 * (v[0] - 4 * v[1] + 3 * v[2]) ** 2]


def step1_blocks(t, v, scheme, eps):
    """reconstruction.hpp:253-286"""
    k = t["radius"]
    if scheme != W5:
        out = 0
        for r in range(k + 1):
            for l in range(k + 1):
                out = out + t["step1_ideal"][r] * t["step1_c"][r, l] * v[k - r + l]
        return out
    b = _beta(v)
    a = [t["weno_d"][r] / (b[r] + eps) ** 2 for r in range(3)]
    cand = [t["step1_c"][r, 0] * v[2 - r] + t["step1_c"][r, 1] * v[3 - r] + t["step1_c"][r, 2] * v[4 - r]
            for r in range(3)]
    return (a[0] * cand[0] + a[1] * cand[1] + a[2] * cand[2]) / (a[0] + a[1] + a[2])


def step2_blocks(t, v, scheme, m, eps):
    """reconstruction.hpp:289-323"""
    k = t["radius"]
    cand = []
    for r in range(k + 1):
        s = 0
        for l in range(k + 1):
            s = s + t["c"][m][r, l] * v[k - r + l]
        cand.append(s)
    if scheme == U3:
        return 0.5 * cand[0] + 0.5 * cand[1]
    if scheme == U5:
        if m == 1:
            up = t["gamma_plus"][0] * cand[0] + t["gamma_plus"][1] * cand[1] + t["gamma_plus"][2] * cand[2]
            um = t["gamma_minus"][0] * cand[0] + t["gamma_minus"][1] * cand[1] + t["gamma_minus"][2] * cand[2]
            return t["sigma_plus"] * up - t["sigma_minus"] * um
        return t["gamma"][m][0] * cand[0] + t["gamma"][m][1] * cand[1] + t["gamma"][m][2] * cand[2]
    b = _beta(v)

    def comb(g):
        a = [g[r] / (b[r] + eps) ** 2 for r in range(3)]
        return (a[0] * cand[0] + a[1] * cand[1] + a[2] * cand[2]) / (a[0] + a[1] + a[2])

    if m == 1:
        return t["sigma_plus"] * comb(t["gamma_plus"]) - t["sigma_minus"] * comb(t["gamma_minus"])
    return comb(t["gamma"][m])


def step1_dense(t, g, axis, scheme, side, eps):
    """reconstruction.hpp:329-349"""
    k = t["radius"]
    n = (g.shape[0] if axis == 0 else g.shape[1]) - 2 * G
    base = G - k - 1 if side == 0 else G - k
    blocks = [g[base + s: base + s + n + 1, :] if axis == 0 else g[:, base + s: base + s + n + 1]
              for s in range(2 * k + 1)]
    if side == 1:
        blocks = blocks[::-1]
    return step1_blocks(t, blocks, scheme, eps)


def step2_dense(t, lines, axis, scheme, eps):
    """reconstruction.hpp:353-377"""
    k, nq = t["radius"], t["nq"]
    n = (lines.shape[0] if axis == 0 else lines.shape[1]) - 2 * G
    blocks = [lines[G - k + s: G - k + s + n, :] if axis == 0 else lines[:, G - k + s: G - k + s + n]
              for s in range(2 * k + 1)]
    out = np.zeros((n * nq, lines.shape[1]) if axis == 0 else (lines.shape[0], n * nq))
    for m in range(nq):
        vals = step2_blocks(t, blocks, scheme, m, eps)
        if axis == 0:
            out[m::nq, :] = vals
        else:
            out[:, m::nq] = vals
    return out


def faces(t, g, axis, scheme, dx, dy):
    """reconstruct_faces, dense (reconstruction.hpp:412-423): (minus, plus)."""
    e1, e2 = (dx * dx, dy * dy) if axis == 0 else (dy * dy, dx * dx)
    trans = 1 - axis
    return (step2_dense(t, step1_dense(t, g, axis, scheme, 0, e1), trans, scheme, e2),
            step2_dense(t, step1_dense(t, g, axis, scheme, 1, e1), trans, scheme, e2))


def ghosted(q, bc_x=0, bc_y=0, strip_x=None, strip_y=None):
    """dense_ghosted (cases.cpp:271-296) with caller-evaluated exact ghost averages."""
    n = q.shape[0]
    ng = n + 2 * G
    out = np.empty((ng, ng))
    for i in range(ng):
        for j in range(ng):
            ii, jj = i - G, j - G
            gx, gy = ii < 0 or ii >= n, jj < 0 or jj >= n
            if gx and bc_x:
                s = i if i < G else i - n
                out[i, j] = strip_x[s, j]
            elif gy and bc_y:
                s = j if j < G else j - n
                out[i, j] = strip_y[i, s]
            else:
                out[i, j] = q[ii % n, jj % n]
    return out


def physical_flux(u, axis, model, g, H):
    """swe.hpp:190-213 with DenseRep ops."""
    if model == 0:
        z = np.zeros_like(u[0])
        return [H * u[1], g * u[0], z] if axis == 0 else [H * u[2], z, g * u[0]]
    if np.any(u[0] == 0.0):
        raise StateError("recip: field has zero entries")
    inv_h = 1.0 / u[0]
    vx, vy = u[1] * inv_h, u[2] * inv_h
    p = (0.5 * g) * (u[0] * u[0])
    if axis == 0:
        return [u[1], 1.0 * (u[1] * vx) + 1.0 * p, u[1] * vy]
    return [u[2], u[2] * vx, 1.0 * (u[2] * vy) + 1.0 * p]


def wave_speed(um, up, axis, model, g, H):
    """face_wave_speed (swe.hpp:325-339): sqrt(gH) linear, scalar max over both sides."""
    if model == 0:
        return np.sqrt(g * H)
    mom = 1 if axis == 0 else 2

    def side_max(u):
        if np.any(u[0] <= 0.0):
            raise StateError("face_wave_speed: nonpositive layer thickness")
        return (np.abs(u[mom] / u[0]) + np.sqrt(g * u[0])).max()

    return max(side_max(um), side_max(up))


def rhs(q, t_tab, scheme, model, g, f, H, ghost=None, extra=None):
    """rhs<DenseRep> (swe.hpp:362-423). ghost(c) -> (bc_x, bc_y, strip_x, strip_y) or None
    for periodic; extra -> three n x n cell-average sources or None."""
    n = q[0].shape[0]
    dx = dy = 1.0 / n
    nq = t_tab["nq"]
    gh = []
    for c in range(3):
        if ghost is None:
            gh.append(ghosted(q[c]))
        else:
            gh.append(ghosted(q[c], *ghost(c)))
    div = [None] * 3
    for axis in (0, 1):
        fm = [faces(t_tab, gh[c], axis, scheme, dx, dy) for c in range(3)]
        um = [p[0] for p in fm]
        up = [p[1] for p in fm]
        fmin = physical_flux(um, axis, model, g, H)
        fpl = physical_flux(up, axis, model, g, H)
        lam = wave_speed(um, up, axis, model, g, H)
        fhat = [1.0 * (0.5 * fmin[c] + 0.5 * fpl[c]) + (-0.5 * lam) * (1.0 * up[c] + (-1.0) * um[c]) for c in range(3)]
        w = np.asarray(t_tab["weight"][:nq])
        for c in range(3):
            if axis == 0:  # (n+1) x (n nq): sum the points of each transverse cell, then difference
                integ = sum(w[m] * fhat[c][:, m::nq] for m in range(nq))
                d = integ[1:, :] - integ[:-1, :]
                div[c] = (1.0 / dx) * d
            else:
                integ = sum(w[m] * fhat[c][m::nq, :] for m in range(nq))
                d = integ[:, 1:] - integ[:, :-1]
                div[c] = 1.0 * div[c] + (1.0 / dy) * d
    src = [np.zeros_like(q[0]), f * q[2], -f * q[1]]
    if extra is not None:
        src = [1.0 * src[c] + 1.0 * extra[c] for c in range(3)]
    return [-1.0 * div[c] + 1.0 * src[c] for c in range(3)]


def ssprk3(q, dt, t, t_tab, scheme, model, g, f, H, ghost_at=None, extra_at=None):
    """ssprk3<DenseRep> (swe.hpp:428-454); ghost_at(t) / extra_at(t) give the hooks at the
    stage times t, t + dt, t + dt/2."""
    def euler(w, tw):
        k = rhs(w, t_tab, scheme, model, g, f, H, ghost_at(tw) if ghost_at else None,
                extra_at(tw) if extra_at else None)
        return [1.0 * w[c] + dt * k[c] for c in range(3)]

    u1 = euler(q, t)
    f1 = euler(u1, t + dt)
    u2 = [0.75 * q[c] + 0.25 * f1[c] for c in range(3)]
    f2 = euler(u2, t + 0.5 * dt)
    return [(1.0 / 3.0) * q[c] + (2.0 / 3.0) * f2[c] for c in range(3)]
