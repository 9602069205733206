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
