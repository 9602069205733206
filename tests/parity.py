"""Shared parity helpers (rank-decision contract and field comparisons)."""
import numpy as np

U = np.finfo(float).eps


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / nb if nb > 0 else np.linalg.norm(a)


def decision_tolerance(r_in, kappa, eps):
    """Largest truncation-margin change a backward-stable rounding can cause.

    The singular values of the pre-rounding TT carry absolute errors
    ~ r_in * u * ||core_x|| ||core_y|| (forming the core product and the SVD), i.e.
    r_in * u * kappa * ||X|| with kappa the cancellation ratio. Relative to the
    (0.9 eps)^2 ||X||^2 budget of truncation_rank (tt.hpp:61-77) that moves the margin
    by about 2 r_in u kappa / (0.9 eps); the factor 2 more covers the tail sum.
    A rank decision whose margin is below this is implementation-defined (the
    reference's BDCSVD would be just as arbitrary there)."""
    if not np.isfinite(kappa):
        return np.inf
    return max(1e-6, 4.0 * r_in * U * kappa / (0.9 * eps))


def rank_mismatch_is_ill_posed(r_in, margin_a, margin_b, kappa_a, kappa_b, eps):
    tol = decision_tolerance(r_in, max(kappa_a, kappa_b), eps)
    return min(abs(margin_a), abs(margin_b)) <= tol


def first_cross_split(ct_a, ct_b):
    """Index of the first cross call whose pivots differ (tie split), or None."""
    for i in range(min(len(ct_a), len(ct_b))):
        if tuple(ct_a[i]) != tuple(ct_b[i]):
            return i
    return None


def check_rank_traces(tr_a, mg_a, ka_a, tr_b, mg_b, ka_b, eps, cross_split=None):
    """Rank-parity contract over two per-rounding traces (columns: op, m, n, r_in, k_out,
    crosses-before). Ranks must be identical until the first rounding whose decision is
    ill-posed, or which follows a cross call whose pivots split on a tie (then the two
    runs legitimately continue from inputs that differ at the cross tolerance).
    Returns the index of that first divergence or None."""
    n = min(len(tr_a), len(tr_b))
    for i in range(n):
        if tr_a[i, 4] == tr_b[i, 4] and tr_a[i, 3] == tr_b[i, 3]:
            continue
        if cross_split is not None and tr_a[i, 5] > cross_split:
            return i
        assert rank_mismatch_is_ill_posed(tr_a[i, 3], mg_a[i], mg_b[i], ka_a[i], ka_b[i], eps), \
            (i, tr_a[i].tolist(), tr_b[i].tolist(), mg_a[i], mg_b[i], ka_a[i], ka_b[i], cross_split)
        return i
    assert len(tr_a) == len(tr_b) or cross_split is not None
    return None


def oracle_noise_floor(oracle, spec, steps, seed=0, cross_seed=1):
    """How far the oracle drifts from itself when its state cores get elementwise ±1 ulp
    noise after every step. On roundoff-dominated configurations (C2: geostrophic balance,
    the rhs is at the noise level and the rank-1 state only absorbs truncated noise) this
    floor exceeds any fixed end-of-run bar; a non-bitwise-identical implementation can
    only be held to a small multiple of it."""
    cfg = oracle.CrossCfg.make(seed=cross_seed, max_rank=spec.cross_max_rank)

    def make():
        s = oracle.Solver(spec.model, spec.scheme, spec.n, spec.g, spec.f, spec.H, spec.dt, spec.tol, cfg)
        s.set_state([oracle.round_(oracle.TT.from_cores(cx, cy), spec.tol) for cx, cy in spec.ic])
        return s

    a, b = make(), make()
    rng = np.random.default_rng(seed)
    for _ in range(steps):
        a.step(1)
        b.step(1)
        noisy = []
        for t in b.state():
            cx, cy = t.cores()
            noisy.append(oracle.TT.from_cores(cx * (1 + 2.2e-16 * rng.uniform(-1, 1, cx.shape)), cy))
        b.set_state(noisy)
    return max(rel(p.full(), q.full()) for p, q in zip(b.state(), a.state()))
