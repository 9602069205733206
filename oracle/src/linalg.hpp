// TEST INFRASTRUCTURE ONLY — CPU oracle for parity tests. Never linked into the
// product library (paper_2408_03483_b200/csrc). Only tests/, __graft_entry__.smoke()
// and bench.py's cpu_baseline / --impl reference legs may load it.
//
// Dense linear algebra used by the restated reference path. The reference calls
// Eigen 3.4 (absent from /root/reference and from this image; pinned only as
// `find_package(Eigen3 3.4 REQUIRED)`, proj/CMakeLists.txt:12). This file restates
// the published algorithms of the Eigen entry points the hot path uses:
//   * HouseholderQR              (tt.hpp:128, cross.hpp:151)  -> householder_qr / thin_q
//   * BDCSVD thin                (tt.hpp:92, :133)             -> svd_thin (one-sided Jacobi,
//                                                                SPEC.md:113 allows Jacobi)
//   * FullPivLU permutation/rank (cross.hpp:37-45)             -> full_piv_lu
//   * PartialPivLU solve         (cross.hpp:51, :205)          -> lu_solve_right
//   * maxCoeff first-index ties  (cross.hpp:53)                -> column-major scan, strict '>'
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

namespace ttor {

using Index = long;  // Eigen::Index (std::ptrdiff_t) on LP64

struct InputError : std::invalid_argument { using std::invalid_argument::invalid_argument; };
struct ShapeError : std::invalid_argument { using std::invalid_argument::invalid_argument; };
struct StateError : std::runtime_error { using std::runtime_error::runtime_error; };
/// Bench-only: a bounded CPU sample ran out of its wall-clock budget (not a reference error).
struct DeadlineReached : std::runtime_error { using std::runtime_error::runtime_error; };
struct DegeneracyError : std::runtime_error { using std::runtime_error::runtime_error; };
struct ConvergenceError : std::runtime_error {
  ConvergenceError(const std::string& w, double r, int it)
      : std::runtime_error(w), residual(r), iterations(it) {}
  double residual;
  int iterations;
};
struct EvaluationError : std::runtime_error {
  EvaluationError(const std::string& w, Index i, Index j)
      : std::runtime_error(w), row(i), col(j) {}
  Index row, col;
};

/// Column-major dense matrix (Eigen's default storage order).
struct Mat {
  Index r = 0, c = 0;
  std::vector<double> a;
  Mat() = default;
  Mat(Index rows, Index cols, double v = 0.0) : r(rows), c(cols), a(size_t(rows * cols), v) {}
  double& operator()(Index i, Index j) { return a[size_t(i + j * r)]; }
  double operator()(Index i, Index j) const { return a[size_t(i + j * r)]; }
  double* col(Index j) { return a.data() + j * r; }
  const double* col(Index j) const { return a.data() + j * r; }
  static Mat identity(Index rows, Index cols) {
    Mat m(rows, cols);
    for (Index k = 0; k < std::min(rows, cols); ++k) m(k, k) = 1.0;
    return m;
  }
  Mat transpose() const {
    Mat t(c, r);
    for (Index j = 0; j < c; ++j)
      for (Index i = 0; i < r; ++i) t(j, i) = (*this)(i, j);
    return t;
  }
  bool all_finite() const {
    for (double v : a)
      if (!std::isfinite(v)) return false;
    return true;
  }
  double norm() const {
    double s = 0;
    for (double v : a) s += v * v;
    return std::sqrt(s);
  }
};

inline Mat matmul(const Mat& A, const Mat& B) {
  if (A.c != B.r) throw ShapeError("matmul: inner dimensions");
  Mat C(A.r, B.c);
  for (Index j = 0; j < B.c; ++j)
    for (Index k = 0; k < A.c; ++k) {
      const double b = B(k, j);
      if (b == 0.0) continue;
      const double* a = A.col(k);
      double* cc = C.col(j);
      for (Index i = 0; i < A.r; ++i) cc[i] += a[i] * b;
    }
  return C;
}

// A^T * B
inline Mat matmul_tn(const Mat& A, const Mat& B) {
  if (A.r != B.r) throw ShapeError("matmul_tn: inner dimensions");
  Mat C(A.c, B.c);
  for (Index j = 0; j < B.c; ++j)
    for (Index i = 0; i < A.c; ++i) {
      const double* a = A.col(i);
      const double* b = B.col(j);
      double s = 0;
      for (Index k = 0; k < A.r; ++k) s += a[k] * b[k];
      C(i, j) = s;
    }
  return C;
}

/// Householder vector in Eigen's makeHouseholder convention:
/// beta = -sign(c0)*||x||, tau = (beta-c0)/beta, v = [1; x_tail/(c0-beta)].
/// A zero tail gives tau = 0 (identity reflector) and beta = c0.
inline void make_householder(double* x, Index len, double& tau, double& beta) {
  const double c0 = x[0];
  double tail2 = 0;
  for (Index i = 1; i < len; ++i) tail2 += x[i] * x[i];
  if (tail2 <= std::numeric_limits<double>::min()) {
    tau = 0.0;
    beta = c0;
    for (Index i = 1; i < len; ++i) x[i] = 0.0;
  } else {
    beta = std::sqrt(c0 * c0 + tail2);
    if (c0 >= 0) beta = -beta;
    const double d = c0 - beta;
    for (Index i = 1; i < len; ++i) x[i] /= d;
    tau = (beta - c0) / beta;
  }
  x[0] = beta;
}

/// In-place Householder QR (unblocked dgeqr2 order). Reflector k is stored
/// below the diagonal of column k with an implicit unit head.
struct HouseholderQR {
  Mat qr;
  std::vector<double> tau;
  explicit HouseholderQR(Mat a) : qr(std::move(a)) {
    const Index m = qr.r, n = qr.c, q = std::min(m, n);
    tau.assign(size_t(q), 0.0);
    for (Index k = 0; k < q; ++k) {
      double beta;
      make_householder(qr.col(k) + k, m - k, tau[k], beta);
      const double t = tau[k];
      if (t == 0.0) continue;
      const double* v = qr.col(k) + k;  // v[0] := 1 implicitly
      for (Index j = k + 1; j < n; ++j) {
        double* a = qr.col(j) + k;
        double w = a[0];
        for (Index i = 1; i < m - k; ++i) w += v[i] * a[i];
        w *= t;
        a[0] -= w;
        for (Index i = 1; i < m - k; ++i) a[i] -= w * v[i];
      }
    }
  }
  /// Apply Q = H_0 H_1 ... H_{q-1} to B from the left (B has qr.r rows).
  void apply_q(Mat& B) const {
    const Index m = qr.r, q = Index(tau.size());
    for (Index k = q - 1; k >= 0; --k) {
      const double t = tau[size_t(k)];
      if (t == 0.0) continue;
      const double* v = qr.col(k) + k;
      for (Index j = 0; j < B.c; ++j) {
        double* b = B.col(j) + k;
        double w = b[0];
        for (Index i = 1; i < m - k; ++i) w += v[i] * b[i];
        w *= t;
        b[0] -= w;
        for (Index i = 1; i < m - k; ++i) b[i] -= w * v[i];
      }
    }
  }
  Mat thin_q() const {
    const Index q = std::min(qr.r, qr.c);
    Mat Q = Mat::identity(qr.r, q);
    apply_q(Q);
    return Q;
  }
  /// Top q rows of the triangular factor (q = min(m,n)), shape q x n.
  Mat r_factor() const {
    const Index q = std::min(qr.r, qr.c);
    Mat R(q, qr.c);
    for (Index j = 0; j < qr.c; ++j)
      for (Index i = 0; i <= std::min(j, q - 1); ++i) R(i, j) = qr(i, j);
    return R;
  }
};

/// detail::thin_q (cross.hpp:148-153).
inline Mat thin_q(const Mat& m) { return HouseholderQR(m).thin_q(); }

struct SVD {
  Mat U;                   // m x p
  std::vector<double> s;   // p, descending
  Mat V;                   // n x p
};

/// One-sided (Hestenes) Jacobi on a square or tall matrix A (m >= n): returns
/// A = U diag(s) V^T with s unsorted.
inline void jacobi_one_sided(Mat& A, Mat& V) {
  const Index m = A.r, n = A.c;
  V = Mat::identity(n, n);
  const double tol = std::numeric_limits<double>::epsilon();
  for (int sweep = 0; sweep < 80; ++sweep) {
    bool rotated = false;
    for (Index p = 0; p < n - 1; ++p)
      for (Index q = p + 1; q < n; ++q) {
        double* ap = A.col(p);
        double* aq = A.col(q);
        double alpha = 0, beta = 0, gamma = 0;
        for (Index i = 0; i < m; ++i) {
          alpha += ap[i] * ap[i];
          beta += aq[i] * aq[i];
          gamma += ap[i] * aq[i];
        }
        if (gamma == 0.0 || std::abs(gamma) <= tol * std::sqrt(alpha * beta)) continue;
        rotated = true;
        const double zeta = (beta - alpha) / (2.0 * gamma);
        const double t = (zeta >= 0 ? 1.0 : -1.0) / (std::abs(zeta) + std::sqrt(1.0 + zeta * zeta));
        const double cs = 1.0 / std::sqrt(1.0 + t * t);
        const double sn = cs * t;
        for (Index i = 0; i < m; ++i) {
          const double x = ap[i], y = aq[i];
          ap[i] = cs * x - sn * y;
          aq[i] = sn * x + cs * y;
        }
        double* vp = V.col(p);
        double* vq = V.col(q);
        for (Index i = 0; i < n; ++i) {
          const double x = vp[i], y = vq[i];
          vp[i] = cs * x - sn * y;
          vq[i] = sn * x + cs * y;
        }
      }
    if (!rotated) return;
  }
}

/// Thin SVD, singular values descending (stands in for Eigen::BDCSVD with
/// ComputeThinU | ComputeThinV). Tall inputs are QR-preconditioned.
inline SVD svd_thin(const Mat& A_in) {
  const bool trans = A_in.r < A_in.c;
  Mat A = trans ? A_in.transpose() : A_in;  // m >= n
  const Index m = A.r, n = A.c;
  SVD out;
  Mat W, V;
  HouseholderQR* qrp = nullptr;
  HouseholderQR qr(m > n ? A : Mat(0, 0));
  if (m > n) {
    qrp = &qr;
    W = qr.r_factor();  // n x n
  } else {
    W = A;
  }
  jacobi_one_sided(W, V);
  std::vector<double> s(static_cast<size_t>(n));
  for (Index j = 0; j < n; ++j) {
    double t = 0;
    for (Index i = 0; i < W.r; ++i) t += W(i, j) * W(i, j);
    s[size_t(j)] = std::sqrt(t);
  }
  std::vector<Index> order(static_cast<size_t>(n));
  for (Index j = 0; j < n; ++j) order[size_t(j)] = j;
  std::stable_sort(order.begin(), order.end(),
                   [&](Index a, Index b) { return s[size_t(a)] > s[size_t(b)]; });
  Mat Us(W.r, n), Vs(n, n);
  out.s.resize(size_t(n));
  for (Index k = 0; k < n; ++k) {
    const Index j = order[size_t(k)];
    const double sj = s[size_t(j)];
    out.s[size_t(k)] = sj;
    for (Index i = 0; i < W.r; ++i) Us(i, k) = sj > 0 ? W(i, j) / sj : (i == k ? 1.0 : 0.0);
    for (Index i = 0; i < n; ++i) Vs(i, k) = V(i, j);
  }
  if (qrp) {
    Mat Ufull(m, n);
    for (Index j = 0; j < n; ++j)
      for (Index i = 0; i < n; ++i) Ufull(i, j) = Us(i, j);
    qrp->apply_q(Ufull);
    Us = std::move(Ufull);
  }
  if (trans) {
    out.U = std::move(Vs);
    out.V = std::move(Us);
  } else {
    out.U = std::move(Us);
    out.V = std::move(Vs);
  }
  return out;
}

/// Solve X * P = B for X (X = B * P^{-1}) with partial-pivot LU of P^T, i.e.
/// the reference's `pivot.transpose().partialPivLu().solve(B.transpose()).transpose()`
/// (cross.hpp:51, :205). P is r x r, B is n x r.
inline Mat solve_right(const Mat& P, const Mat& B) {
  const Index r = P.r;
  Mat lu = P.transpose();
  std::vector<Index> perm(static_cast<size_t>(r));
  for (Index i = 0; i < r; ++i) perm[size_t(i)] = i;
  for (Index k = 0; k < r; ++k) {
    Index piv = k;
    double best = std::abs(lu(k, k));
    for (Index i = k + 1; i < r; ++i)
      if (std::abs(lu(i, k)) > best) { best = std::abs(lu(i, k)); piv = i; }
    if (piv != k) {
      for (Index j = 0; j < r; ++j) std::swap(lu(k, j), lu(piv, j));
      std::swap(perm[size_t(k)], perm[size_t(piv)]);
    }
    const double d = lu(k, k);
    if (d != 0.0)
      for (Index i = k + 1; i < r; ++i) lu(i, k) /= d;
    for (Index j = k + 1; j < r; ++j) {
      const double u = lu(k, j);
      for (Index i = k + 1; i < r; ++i) lu(i, j) -= lu(i, k) * u;
    }
  }
  // Solve (P^T) Y = B^T, Y is r x n; X = Y^T.
  const Index n = B.r;
  Mat X(n, r);
  std::vector<double> y(static_cast<size_t>(r));
  for (Index c = 0; c < n; ++c) {
    for (Index i = 0; i < r; ++i) y[size_t(i)] = B(c, perm[size_t(i)]);
    for (Index i = 0; i < r; ++i)
      for (Index k = 0; k < i; ++k) y[size_t(i)] -= lu(i, k) * y[size_t(k)];
    for (Index i = r - 1; i >= 0; --i) {
      for (Index k = i + 1; k < r; ++k) y[size_t(i)] -= lu(i, k) * y[size_t(k)];
      y[size_t(i)] /= lu(i, i);
    }
    for (Index i = 0; i < r; ++i) X(c, i) = y[size_t(i)];
  }
  return X;
}

/// Full-pivot LU as in Eigen::FullPivLU: returns the original row index of
/// each pivot (in pivot order) and the numerical rank with the default
/// threshold (max|pivot| * min(rows,cols) * machine eps).
struct FullPivResult {
  std::vector<Index> row_order;  // row_order[k] = original row at pivot k
  Index rank = 0;
};

inline FullPivResult full_piv_lu(Mat lu) {
  const Index rows = lu.r, cols = lu.c, size = std::min(rows, cols);
  std::vector<Index> orig(static_cast<size_t>(rows));
  for (Index i = 0; i < rows; ++i) orig[size_t(i)] = i;
  Index nonzero = size;
  double maxpivot = 0;
  for (Index k = 0; k < size; ++k) {
    Index bi = k, bj = k;
    double best = -1;
    for (Index j = k; j < cols; ++j)
      for (Index i = k; i < rows; ++i) {
        const double v = std::abs(lu(i, j));
        if (v > best) { best = v; bi = i; bj = j; }
      }
    if (best == 0.0) { nonzero = k; break; }
    if (best > maxpivot) maxpivot = best;
    if (bi != k) {
      for (Index j = 0; j < cols; ++j) std::swap(lu(k, j), lu(bi, j));
      std::swap(orig[size_t(k)], orig[size_t(bi)]);
    }
    if (bj != k)
      for (Index i = 0; i < rows; ++i) std::swap(lu(i, k), lu(i, bj));
    const double d = lu(k, k);
    for (Index i = k + 1; i < rows; ++i) lu(i, k) /= d;
    for (Index j = k + 1; j < cols; ++j) {
      const double u = lu(k, j);
      for (Index i = k + 1; i < rows; ++i) lu(i, j) -= lu(i, k) * u;
    }
  }
  FullPivResult res;
  res.row_order = orig;
  const double thr = maxpivot * double(size) * std::numeric_limits<double>::epsilon();
  for (Index i = 0; i < nonzero; ++i) res.rank += (std::abs(lu(i, i)) > thr);
  return res;
}

/// Least-squares solve of a consistent full-column-rank system via Householder
/// QR (stands in for colPivHouseholderQr().solve, reconstruction.hpp:82).
inline std::vector<double> lstsq(const Mat& A, const std::vector<double>& b) {
  HouseholderQR qr(A);
  Mat B(A.r, 1);
  for (Index i = 0; i < A.r; ++i) B(i, 0) = b[size_t(i)];
  // Q^T b: apply reflectors in forward order.
  const Index m = A.r, q = Index(qr.tau.size());
  for (Index k = 0; k < q; ++k) {
    const double t = qr.tau[size_t(k)];
    if (t == 0.0) continue;
    const double* v = qr.qr.col(k) + k;
    double* bb = B.col(0) + k;
    double w = bb[0];
    for (Index i = 1; i < m - k; ++i) w += v[i] * bb[i];
    w *= t;
    bb[0] -= w;
    for (Index i = 1; i < m - k; ++i) bb[i] -= w * v[i];
  }
  const Index n = A.c;
  std::vector<double> x(static_cast<size_t>(n));
  for (Index i = n - 1; i >= 0; --i) {
    double s = B(i, 0);
    for (Index k = i + 1; k < n; ++k) s -= qr.qr(i, k) * x[size_t(k)];
    x[size_t(i)] = s / qr.qr(i, i);
  }
  return x;
}

/// Square solve with partial pivoting (stands in for fullPivLu().solve on the
/// k x k moment systems, reconstruction.hpp:69).
inline std::vector<double> solve_square(Mat A, std::vector<double> b) {
  const Index n = A.r;
  for (Index k = 0; k < n; ++k) {
    Index piv = k;
    for (Index i = k + 1; i < n; ++i)
      if (std::abs(A(i, k)) > std::abs(A(piv, k))) piv = i;
    if (piv != k) {
      for (Index j = 0; j < n; ++j) std::swap(A(k, j), A(piv, j));
      std::swap(b[size_t(k)], b[size_t(piv)]);
    }
    for (Index i = k + 1; i < n; ++i) {
      const double f = A(i, k) / A(k, k);
      for (Index j = k; j < n; ++j) A(i, j) -= f * A(k, j);
      b[size_t(i)] -= f * b[size_t(k)];
    }
  }
  std::vector<double> x(static_cast<size_t>(n));
  for (Index i = n - 1; i >= 0; --i) {
    double s = b[size_t(i)];
    for (Index k = i + 1; k < n; ++k) s -= A(i, k) * x[size_t(k)];
    x[size_t(i)] = s / A(i, i);
  }
  return x;
}

}  // namespace ttor
