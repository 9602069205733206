"""Manufactured-solution helpers for the hook tests: a numpy restatement of the
reference's nonlinear MMS (cases.cpp:190-220: exact_conserved, mms_source on
h = H + A sin(phase), u = B cos(phase), v = 0, phase = kx x + ky y - omega t) and cell
averages by tensor Gauss-Legendre quadrature (cell_average_field, cases.cpp:222-240).
Parameters are this test's own, not a reference case's."""
import math

import numpy as np

H, G, F = 1.0, 1.0, 0.5
AMP, U_AMP = 0.05, 0.1
KX, KY, OMEGA = 2 * math.pi, 2 * math.pi, math.pi


def exact_conserved(x, y, t):
    ph = KX * x + KY * y - OMEGA * t
    h = H + AMP * np.sin(ph)
    u = U_AMP * np.cos(ph)
    return [h, h * u, 0.0 * h]


def mms_source(x, y, t):
    ph = KX * x + KY * y - OMEGA * t
    cp, sp = np.cos(ph), np.sin(ph)
    h = H + AMP * sp
    A, B = AMP, U_AMP
    s1 = -OMEGA * A * cp + KX * B * (A * cp * cp - h * sp)
    s2 = B * OMEGA * (-A * cp * cp + h * sp) + KX * B * B * (A * cp ** 3 - 2.0 * h * cp * sp) + G * h * A * KX * cp
    s3 = G * h * A * KY * cp + F * h * B * cp
    return [s1, s2, s3]


def cell_averages(fn, n, t, nq=3, lo=0, hi=None):
    """(hi-lo) x (hi-lo) cell averages of fn over cells lo..hi-1 (ghost cells when lo < 0)."""
    hi = n if hi is None else hi
    xg, wg = np.polynomial.legendre.leggauss(nq)
    c = (np.arange(lo, hi) + 0.5) / n
    pts = (c[:, None] + 0.5 * xg[None, :] / n).ravel()
    w = np.tile(0.5 * wg, hi - lo)
    X, Y = np.meshgrid(pts, pts, indexing="ij")
    vals = fn(X, Y, t)
    m = hi - lo
    out = []
    for v in vals:
        v = np.broadcast_to(v, X.shape) * np.outer(w, w)
        out.append(v.reshape(m, nq, m, nq).sum(axis=(1, 3)))
    return out


def ghost_strips(n, t, nq=3):
    """Exact ghost strips (strip_x 6 x (n+6), strip_y (n+6) x 6) per component."""
    full = cell_averages(exact_conserved, n, t, nq, lo=-3, hi=n + 3)
    rows = [0, 1, 2, n + 3, n + 4, n + 5]
    return [(f[rows, :], f[:, rows]) for f in full]
