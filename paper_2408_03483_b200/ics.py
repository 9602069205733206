"""Seeded initial conditions and run constants for the five BASELINE configs.

The reference ships only the paper's four verification cases (proj/src/cases.cpp:11-81),
so the BASELINE ICs are built here:

* cell averages use the n_q-point tensor Gauss rule of ``cell_average_field``
  (proj/src/cases.cpp:222-239 / 413-430), applied to separable terms as products of
  1-D averages (identical in exact arithmetic);
* every field is returned as an *unrounded* sum of rank-1 terms (core_x m×R,
  core_y R×n, column-major) — the solver compresses it at the run tolerance like
  ``run_impl`` does (proj/src/harness.cpp:93-95);
* random draws use std::mt19937_64 with u = (x >> 11) * 2^-53.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

MASK64 = (1 << 64) - 1


class MT19937_64:
    """std::mt19937_64 (the standard's 64-bit Mersenne Twister parameters)."""

    NN, MM = 312, 156
    MATRIX_A = 0xB5026F5AA96619E9
    UM, LM = 0xFFFFFFFF80000000, 0x7FFFFFFF

    def __init__(self, seed: int):
        self.mt = [0] * self.NN
        self.mt[0] = seed & MASK64
        for i in range(1, self.NN):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) & MASK64
        self.mti = self.NN

    def _twist(self):
        mt = self.mt
        for i in range(self.NN):
            x = (mt[i] & self.UM) | (mt[(i + 1) % self.NN] & self.LM)
            xa = x >> 1
            if x & 1:
                xa ^= self.MATRIX_A
            mt[i] = mt[(i + self.MM) % self.NN] ^ xa
        self.mti = 0

    def next_u64(self) -> int:
        if self.mti >= self.NN:
            self._twist()
        x = self.mt[self.mti]
        self.mti += 1
        x ^= (x >> 29) & 0x5555555555555555
        x ^= (x << 17) & 0x71D67FFFEDA60000
        x ^= (x << 37) & 0xFFF7EEE000000000
        x ^= x >> 43
        return x & MASK64

    def uniform(self) -> float:
        return (self.next_u64() >> 11) * (1.0 / 9007199254740992.0)

    def uniform_range(self, lo: float, hi: float) -> float:
        return lo + (hi - lo) * self.uniform()


SEEDS = {2: 240803482, 3: 240803483, 4: 240803484, 5: 240803485}


def gauss_rule(n_q: int):
    """gauss_rule (reconstruction.hpp:33-49) on [-1/2, 1/2]."""
    if n_q == 2:
        a = 1.0 / (2.0 * math.sqrt(3.0))
        return np.array([-a, a]), np.array([0.5, 0.5])
    if n_q == 3:
        b = math.sqrt(3.0 / 5.0) / 2.0
        return np.array([-b, 0.0, b]), np.array([5.0 / 18.0, 8.0 / 18.0, 5.0 / 18.0])
    raise ValueError("only 2- and 3-point rules")


def cell_avg_1d(f, n: int, n_q: int, length: float = 1.0) -> np.ndarray:
    """1-D n_q-point Gauss cell averages of f on n uniform cells of [0, length)."""
    off, w = gauss_rule(n_q)
    dx = length / n
    xc = (np.arange(n) + 0.5) * dx
    acc = np.zeros(n)
    for a in range(n_q):
        acc += w[a] * f(xc + off[a] * dx)
    return acc


def min_image(x, c):
    """Minimum-image signed distance on the unit circle."""
    d = x - c
    return d - np.floor(d + 0.5)


def gaussian(c, w):
    return lambda x: np.exp(-(min_image(x, c) ** 2) / (w * w))


def dgaussian(c, w):
    return lambda x: -2.0 * min_image(x, c) / (w * w) * np.exp(-(min_image(x, c) ** 2) / (w * w))


@dataclasses.dataclass
class RunSpec:
    """One BASELINE configuration, resolved to solver parameters and IC cores."""

    name: str
    model: int  # 0 linear, 1 nonlinear
    scheme: int  # 0 upwind3, 1 upwind5, 2 weno5
    n: int
    g: float
    f: float
    H: float
    tol: float
    dt: float
    steps: int
    ic: list  # [(core_x, core_y)] x 3, unrounded
    cross_max_rank: int = 128
    notes: str = ""


def _sum_rank1(terms, n):
    """Stack rank-1 terms [(coef, ax, by)] into cores (n x R, R x n)."""
    if not terms:
        return np.zeros((n, 1), order="F"), np.zeros((1, n), order="F")
    cx = np.asfortranarray(np.stack([c * ax for c, ax, _ in terms], axis=1))
    cy = np.asfortranarray(np.stack([by for _, _, by in terms], axis=0))
    return cx, cy


def config1(n: int = 256, steps: int = 100) -> RunSpec:
    """C1: linear, N=256, upwind3, tol 1e-8; eta = 0.01 exp(-r^2/0.01), u = v = 0."""
    nq = 2
    gx = cell_avg_1d(lambda x: np.exp(-((x - 0.5) ** 2) / 0.01), n, nq)
    eta = _sum_rank1([(0.01, gx, gx)], n)
    zero = _sum_rank1([], n)
    dt = 0.4 * (1.0 / n) / math.sqrt(1.0 * 1.0)
    return RunSpec("C1", 0, 0, n, 1.0, 0.0, 1.0, 1e-8, dt, steps, [eta, zero, zero])


def config2(n: int = 1024, steps: int = 500, seed: int = SEEDS[2]) -> RunSpec:
    """C2: linear f=10, N=1024, upwind5, tol 1e-10; geostrophic Gaussian (amp 0.01, width 0.05)."""
    nq, g, f, w, amp = 3, 1.0, 10.0, 0.05, 0.01
    rng = MT19937_64(seed)
    cx0, cy0 = rng.uniform(), rng.uniform()
    Gx = cell_avg_1d(gaussian(cx0, w), n, nq)
    Gy = cell_avg_1d(gaussian(cy0, w), n, nq)
    dGx = cell_avg_1d(dgaussian(cx0, w), n, nq)
    dGy = cell_avg_1d(dgaussian(cy0, w), n, nq)
    eta = _sum_rank1([(amp, Gx, Gy)], n)
    u = _sum_rank1([(-(g / f) * amp, Gx, dGy)], n)   # u = -(g/f) d(eta)/dy
    v = _sum_rank1([((g / f) * amp, dGx, Gy)], n)    # v = (g/f) d(eta)/dx
    dt = 0.4 * (1.0 / n) / math.sqrt(g * 1.0)
    return RunSpec("C2", 0, 1, n, g, f, 1.0, 1e-10, dt, steps, [eta, u, v],
                   notes=f"centre=({cx0:.6f},{cy0:.6f}) seed={seed}")


def _bumps(rng: MT19937_64, count: int = 4):
    out = []
    for _ in range(count):
        A = rng.uniform_range(0.02, 0.1)
        w = rng.uniform_range(0.03, 0.1)
        cx, cy = rng.uniform(), rng.uniform()
        out.append((A, w, cx, cy))
    return out


def config3(n: int = 2048, steps: int = 1000, seed: int = SEEDS[3]) -> RunSpec:
    """C3: nonlinear, N=2048, upwind5, tol 1e-10; h = 1 + 4 seeded Gaussian bumps, hu = hv = 0."""
    nq, g = 3, 1.0
    rng = MT19937_64(seed)
    bumps = _bumps(rng)
    ones = np.ones(n)
    terms = [(1.0, ones, ones)]
    for A, w, cx, cy in bumps:
        terms.append((A, cell_avg_1d(gaussian(cx, w), n, nq), cell_avg_1d(gaussian(cy, w), n, nq)))
    h = _sum_rank1(terms, n)
    zero = _sum_rank1([], n)
    hmax = float(np.max(h[0] @ h[1]))
    dt = 0.4 * (1.0 / n) / math.sqrt(g * hmax)
    return RunSpec("C3", 1, 1, n, g, 0.0, 1.0, 1e-10, dt, steps, [h, zero, zero],
                   notes=f"bumps={bumps} seed={seed}")


def config4(n: int = 4096, steps: int = 500, seed: int = SEEDS[4], noise: str = "smooth4") -> RunSpec:
    """C4: nonlinear f=10, N=4096, WENO5, tol 1e-10; two balanced vortices + low-rank noise.

    SURVEY App. A D5: iid 1e-4 noise makes h full-rank at 1e-10 and the reference's WENO
    cross throws ConvergenceError at step 0. A rough rank-4 noise (outer products of
    per-cell U[-1,1] vectors, noise="rank4") still makes the WENO faces non-smooth: the
    oracle's cross stalls at relative RMS 1.2e-9 > 1e-10 after 30 sweeps at N=512 and
    throws too (both sides agree; scripts/oracle_step.py). The default noise="smooth4" is
    a seeded sum of four rank-1 products of periodic trigonometric polynomials
    (wavenumbers 1..8, U[-1,1] coefficients), scaled to max |noise| = 1e-4 (flagged).
    """
    nq, g, f, a, w = 3, 1.0, 10.0, 0.05, 0.04
    centres = [(0.4, 0.5), (0.6, 0.5)]
    Gx = [cell_avg_1d(gaussian(c[0], w), n, nq) for c in centres]
    Gy = [cell_avg_1d(gaussian(c[1], w), n, nq) for c in centres]
    dGx = [cell_avg_1d(dgaussian(c[0], w), n, nq) for c in centres]
    dGy = [cell_avg_1d(dgaussian(c[1], w), n, nq) for c in centres]
    off, wq = gauss_rule(nq)
    ones = np.ones(n)
    rng = MT19937_64(seed)
    nx = [np.array([rng.uniform_range(-1, 1) for _ in range(n)]) for _ in range(4)]
    ny = [np.array([rng.uniform_range(-1, 1) for _ in range(n)]) for _ in range(4)]
    noise_full = sum(np.outer(nx[k], ny[k]) for k in range(4))
    nscale = 1e-4 / np.max(np.abs(noise_full))
    h_terms = [(1.0, ones, ones)] + [(a, Gx[i], Gy[i]) for i in range(2)]
    if noise == "rank4":
        h_terms += [(nscale, nx[k], ny[k]) for k in range(4)]
    elif noise == "smooth4":
        # four rank-1 terms whose 1-D factors are periodic trigonometric polynomials
        # (wavenumbers 1..8, U[-1,1] coefficients from the seeded stream), cell-averaged
        srng = MT19937_64(seed + 1)
        def trig(coef):
            return lambda x: sum(coef[2 * k] * np.cos(2 * np.pi * (k + 1) * x) +
                                 coef[2 * k + 1] * np.sin(2 * np.pi * (k + 1) * x) for k in range(8))
        fx = [cell_avg_1d(trig([srng.uniform_range(-1, 1) for _ in range(16)]), n, nq) for _ in range(4)]
        fy = [cell_avg_1d(trig([srng.uniform_range(-1, 1) for _ in range(16)]), n, nq) for _ in range(4)]
        sfull = sum(np.outer(fx[k], fy[k]) for k in range(4))
        sscale = 1e-4 / np.max(np.abs(sfull))
        h_terms += [(sscale, fx[k], fy[k]) for k in range(4)]
    elif noise != "none":
        raise ValueError(f"unknown C4 noise kind {noise!r}")
    # hu = h * u with u = -(g/f) dh/dy: pointwise products of separable functions, each
    # averaged per axis from its 1-D Gauss-point values (separable terms).
    dx = 1.0 / n
    xc = (np.arange(n) + 0.5) * dx
    def pts(fun, c):
        return [fun(c, w)(xc + o * dx) for o in off]
    gxp = [pts(gaussian, c[0]) for c in centres]
    gyp = [pts(gaussian, c[1]) for c in centres]
    dgxp = [pts(dgaussian, c[0]) for c in centres]
    dgyp = [pts(dgaussian, c[1]) for c in centres]
    def avg(vals):
        return sum(wq[q] * vals[q] for q in range(nq))
    hu_terms, hv_terms = [], []
    cu, cv = -(g / f) * a, (g / f) * a
    for j in range(2):
        hu_terms.append((cu, avg(gxp[j]), avg(dgyp[j])))
        hv_terms.append((cv, avg(dgxp[j]), avg(gyp[j])))
        for i in range(2):
            hu_terms.append((a * cu, avg([gxp[i][q] * gxp[j][q] for q in range(nq)]),
                             avg([gyp[i][q] * dgyp[j][q] for q in range(nq)])))
            hv_terms.append((a * cv, avg([gxp[i][q] * dgxp[j][q] for q in range(nq)]),
                             avg([gyp[i][q] * gyp[j][q] for q in range(nq)])))
    h = _sum_rank1(h_terms, n)
    hu = _sum_rank1(hu_terms, n)
    hv = _sum_rank1(hv_terms, n)
    hd = h[0] @ h[1]
    ud = (hu[0] @ hu[1]) / hd
    vd = (hv[0] @ hv[1]) / hd
    lam = float(np.max(np.maximum(np.abs(ud), np.abs(vd)) + np.sqrt(g * hd)))
    dt = 0.4 * (1.0 / n) / lam
    return RunSpec("C4", 1, 2, n, g, f, 1.0, 1e-10, dt, steps, [h, hu, hv], cross_max_rank=64,
                   notes=f"{noise} seeded low-rank noise instead of iid noise: SURVEY App. A D5")


def config5_member(member: int, n: int = 2048, steps: int = 500) -> RunSpec:
    """C5 member m: the C3 setup with per-member seed S5 + m."""
    spec = config3(n=n, steps=steps, seed=SEEDS[5] + member)
    spec.name = f"C5[{member}]"
    return spec


CONFIGS = {"C1": config1, "C2": config2, "C3": config3, "C4": config4}
