// TEST INFRASTRUCTURE ONLY — CPU oracle (see linalg.hpp header).
//
// Restatement of /root/reference/proj/include/ttsw/tt.hpp (two-core TT algebra).
// Every function cites the reference lines it follows.
#pragma once

#include <chrono>
#include <functional>
#include <sstream>

#include "linalg.hpp"

namespace ttor {

enum class Axis { X = 0, Y = 1 };
inline constexpr Index kGhost = 3;  // types.hpp:24

/// TTMatrix<double> (tt.hpp:19-53): X(i,j) = sum_a cx(i,a) cy(a,j).
struct TT {
  Mat cx;  // rows x rank
  Mat cy;  // rank x cols
  TT() : cx(1, 1), cy(1, 1) {}
  TT(Mat x, Mat y) : cx(std::move(x)), cy(std::move(y)) {
    if (cx.c != cy.r) throw ShapeError("TTMatrix: core inner dimensions do not match");
    if (cx.c < 1) throw ShapeError("TTMatrix: rank must be positive");
    if (!cx.all_finite() || !cy.all_finite())
      throw InputError("TTMatrix: cores contain non-finite entries");
  }
  static TT zero(Index rows, Index cols) { return TT(Mat(rows, 1), Mat(1, cols)); }
  static TT constant(Index rows, Index cols, double v) { return TT(Mat(rows, 1, v), Mat(1, cols, 1.0)); }
  Index rows() const { return cx.r; }
  Index cols() const { return cy.c; }
  Index rank() const { return cx.c; }
};

/// One record per rounding: the decision and its margin (SURVEY §7 hard part (i)).
struct RoundRecord {
  int op = 0;
  Index m = 0, n = 0, r_in = 0, k_out = 0;
  double margin = 0;  // relative distance of the closest truncation comparison to the budget
  double kappa = 1;   // ||core_x||_F ||core_y||_F / ||X||_F: cancellation ratio of the input
  long crosses = 0;   // cross calls completed before this rounding (trace alignment)
};

/// Number of successful cross calls (for trace alignment).
inline long& cross_calls() {
  static thread_local long n = 0;
  return n;
}

/// Wall-clock deadline for bounded CPU samples (bench.py cpu_baseline); checked when a
/// rounding starts, so the trace holds exactly the completed roundings. 0 = none.
inline double& sample_deadline() {
  static thread_local double t = 0;
  return t;
}
inline double wall_seconds() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

/// Global trace sink (set by the solver driver; nullptr disables).
inline std::vector<RoundRecord>*& round_trace() {
  static thread_local std::vector<RoundRecord>* p = nullptr;
  return p;
}

/// detail::truncation_rank (tt.hpp:61-77), long-double accumulation, plus the
/// decision margin min over the accepted drop and the rejecting comparison.
inline Index truncation_rank(const std::vector<double>& sv, double eps, double* margin = nullptr) {
  const Index n = Index(sv.size());
  long double total2 = 0;
  for (Index k = 0; k < n; ++k) total2 += static_cast<long double>(sv[size_t(k)]) * sv[size_t(k)];
  if (margin) *margin = std::numeric_limits<double>::infinity();
  if (total2 == 0) return 1;
  const long double budget = static_cast<long double>(0.9 * eps) * (0.9 * eps) * total2;
  Index keep = n;
  long double tail2 = 0;
  long double mg = std::numeric_limits<long double>::infinity();
  while (keep > 1) {
    const long double s = sv[size_t(keep - 1)];
    if (s != 0 && tail2 + s * s > budget) {
      if (budget > 0) mg = std::min(mg, (tail2 + s * s - budget) / budget);
      break;
    }
    tail2 += s * s;
    if (s != 0 && budget > 0) mg = std::min(mg, (budget - tail2) / budget);
    --keep;
  }
  if (margin) *margin = double(mg);
  return keep;
}

/// tt_from_full (tt.hpp:82-97).
inline TT tt_from_full(const Mat& A, double eps) {
  if (!A.all_finite()) throw InputError("tt_from_full: non-finite entries");
  if (eps < 0) throw InputError("tt_from_full: eps must be non-negative");
  if (A.norm() == 0.0) return TT::zero(A.r, A.c);
  SVD svd = svd_thin(A);
  const Index r = truncation_rank(svd.s, eps);
  Mat cx(A.r, r), cy(r, A.c);
  for (Index k = 0; k < r; ++k) {
    for (Index i = 0; i < A.r; ++i) cx(i, k) = svd.U(i, k) * svd.s[size_t(k)];
    for (Index j = 0; j < A.c; ++j) cy(k, j) = svd.V(j, k);
  }
  return TT(std::move(cx), std::move(cy));
}

/// to_full (tt.hpp:99-102).
inline Mat to_full(const TT& x) { return matmul(x.cx, x.cy); }

/// norm_fro (tt.hpp:105-111): Gram-based, clamped at zero.
inline double norm_fro(const TT& x) {
  Mat gx = matmul_tn(x.cx, x.cx);
  Mat cyt = x.cy.transpose();
  Mat gy = matmul_tn(cyt, cyt);
  double v = 0;
  for (size_t i = 0; i < gx.a.size(); ++i) v += gx.a[i] * gy.a[i];
  return std::sqrt(std::max(v, 0.0));
}

/// sum_entries (tt.hpp:113-116).
inline double sum_entries(const TT& x) {
  double s = 0;
  for (Index a = 0; a < x.rank(); ++a) {
    double cs = 0, rs = 0;
    for (Index i = 0; i < x.rows(); ++i) cs += x.cx(i, a);
    for (Index j = 0; j < x.cols(); ++j) rs += x.cy(a, j);
    s += cs * rs;
  }
  return s;
}

/// round (tt.hpp:120-138): QR of core_y^T, W = core_x R^T, thin SVD of W,
/// truncation, core_x' = U_k S_k, core_y' = (Q V_k)^T.
inline TT round(const TT& x, double eps) {
  if (eps < 0) throw InputError("round: eps must be non-negative");
  if (sample_deadline() > 0 && wall_seconds() > sample_deadline()) throw DeadlineReached("sample deadline");
  if (norm_fro(x) == 0.0) {
    if (auto* t = round_trace())
      t->push_back({int(t->size()), x.rows(), x.cols(), x.rank(), 1, std::numeric_limits<double>::infinity(),
                    std::numeric_limits<double>::infinity(), cross_calls()});
    return TT::zero(x.rows(), x.cols());
  }
  HouseholderQR qr(x.cy.transpose());
  Mat Q = qr.thin_q();     // cols x q
  Mat R = qr.r_factor();   // q x rank
  Mat W = matmul(x.cx, R.transpose());
  SVD svd = svd_thin(W);
  double margin = 0;
  const Index keep = truncation_rank(svd.s, eps, &margin);
  if (auto* t = round_trace()) {
    double s2 = 0;
    for (double s : svd.s) s2 += s * s;
    const double kappa = s2 > 0 ? x.cx.norm() * x.cy.norm() / std::sqrt(s2) : std::numeric_limits<double>::infinity();
    t->push_back({int(t->size()), x.rows(), x.cols(), x.rank(), keep, margin, kappa, cross_calls()});
  }
  Mat cx(x.rows(), keep);
  for (Index k = 0; k < keep; ++k)
    for (Index i = 0; i < x.rows(); ++i) cx(i, k) = svd.U(i, k) * svd.s[size_t(k)];
  Mat Vk(svd.V.r, keep);
  for (Index k = 0; k < keep; ++k)
    for (Index i = 0; i < svd.V.r; ++i) Vk(i, k) = svd.V(i, k);
  Mat QV = matmul(Q, Vk);
  return TT(std::move(cx), QV.transpose());
}

inline void check_same_shape(const TT& x, const TT& y, const char* where) {
  if (x.rows() != y.rows() || x.cols() != y.cols())
    throw ShapeError(std::string(where) + ": operand shapes do not match");
}

/// add (tt.hpp:152-161): block concatenation, x first.
inline TT add(const TT& x, const TT& y) {
  check_same_shape(x, y, "add");
  Mat cx(x.rows(), x.rank() + y.rank()), cy(x.rank() + y.rank(), x.cols());
  std::copy(x.cx.a.begin(), x.cx.a.end(), cx.a.begin());
  std::copy(y.cx.a.begin(), y.cx.a.end(), cx.a.begin() + long(x.cx.a.size()));
  for (Index j = 0; j < x.cols(); ++j) {
    for (Index a = 0; a < x.rank(); ++a) cy(a, j) = x.cy(a, j);
    for (Index b = 0; b < y.rank(); ++b) cy(x.rank() + b, j) = y.cy(b, j);
  }
  return TT(std::move(cx), std::move(cy));
}

/// scale (tt.hpp:163-166): scales core_x only.
inline TT scale(const TT& x, double a) {
  Mat cx = x.cx;
  for (double& v : cx.a) v *= a;
  return TT(std::move(cx), x.cy);
}

/// hadamard (tt.hpp:169-181): column a*ry+b = x.cx(:,a) .* y.cx(:,b).
inline TT hadamard(const TT& x, const TT& y) {
  check_same_shape(x, y, "hadamard");
  const Index rx = x.rank(), ry = y.rank();
  Mat cx(x.rows(), rx * ry), cy(rx * ry, x.cols());
  for (Index a = 0; a < rx; ++a)
    for (Index b = 0; b < ry; ++b) {
      for (Index i = 0; i < x.rows(); ++i) cx(i, a * ry + b) = y.cx(i, b) * x.cx(i, a);
      for (Index j = 0; j < x.cols(); ++j) cy(a * ry + b, j) = y.cy(b, j) * x.cy(a, j);
    }
  return TT(std::move(cx), std::move(cy));
}

/// A banded one-mode operator: out[i] = sum_t coef[i][t] * in[col[i][t]].
/// Replaces the dense operator matrices of reconstruction.hpp:428-501 and
/// cases.cpp:302-308 (identical in exact arithmetic; only the nonzero taps are
/// summed, in increasing column order).
struct BandOp {
  Index n_out = 0, n_in = 0;
  std::vector<std::vector<std::pair<Index, double>>> rows;
  Mat dense() const {
    Mat m(n_out, n_in);
    for (Index i = 0; i < n_out; ++i)
      for (auto& [c, v] : rows[size_t(i)]) m(i, c) = v;
    return m;
  }
  static BandOp from_dense(const Mat& m) {
    BandOp op;
    op.n_out = m.r;
    op.n_in = m.c;
    op.rows.resize(size_t(m.r));
    for (Index i = 0; i < m.r; ++i)
      for (Index j = 0; j < m.c; ++j)
        if (m(i, j) != 0.0) op.rows[size_t(i)].push_back({j, m(i, j)});
    return op;
  }
};

/// apply_core_map (tt.hpp:185-194): Axis::X -> M core_x, Axis::Y -> core_y M^T.
inline TT apply_core_map(const TT& x, Axis axis, const BandOp& m) {
  if (axis == Axis::X) {
    if (m.n_in != x.rows()) throw ShapeError("apply_core_map: operator/mode size mismatch");
    Mat cx(m.n_out, x.rank());
    for (Index a = 0; a < x.rank(); ++a)
      for (Index i = 0; i < m.n_out; ++i) {
        double s = 0;
        for (auto& [c, v] : m.rows[size_t(i)]) s += v * x.cx(c, a);
        cx(i, a) = s;
      }
    return TT(std::move(cx), x.cy);
  }
  if (m.n_in != x.cols()) throw ShapeError("apply_core_map: operator/mode size mismatch");
  Mat cy(x.rank(), m.n_out);
  for (Index i = 0; i < m.n_out; ++i)
    for (Index a = 0; a < x.rank(); ++a) {
      double s = 0;
      for (auto& [c, v] : m.rows[size_t(i)]) s += v * x.cy(a, c);
      cy(a, i) = s;
    }
  return TT(x.cx, std::move(cy));
}

struct ReciprocalStats { int iterations = 0; };

/// reciprocal_taylor (tt.hpp:204-241).
inline TT reciprocal_taylor(const TT& x, double eps, int max_iterations = 200,
                            ReciprocalStats* stats = nullptr) {
  if (eps <= 0) throw InputError("reciprocal_taylor: eps must be positive");
  const double n_entries = double(x.rows()) * double(x.cols());
  const double x_avg = sum_entries(x) / n_entries;
  if (x_avg == 0.0) throw ConvergenceError("reciprocal_taylor: field has zero mean", 1.0, 0);
  const TT ones = TT::constant(x.rows(), x.cols(), 1.0);
  const TT xt = round(add(ones, scale(x, -1.0 / x_avg)), eps);
  auto fail = [&](const char* reason, double err, int it) {
    Mat d = to_full(xt);
    double mx = 0;
    for (double v : d.a) mx = std::max(mx, std::abs(v));
    std::ostringstream os;
    os << "reciprocal_taylor: " << reason << " after " << it
       << " iterations (max|1 - x/x_avg| = " << mx << ", residual = " << err << ")";
    return ConvergenceError(os.str(), err, it);
  };
  TT y = ones, dy = ones;
  double prev_err = std::numeric_limits<double>::infinity();
  int growth = 0;
  for (int it = 1; it <= max_iterations; ++it) {
    dy = round(hadamard(dy, xt), eps);
    y = round(add(y, dy), eps);
    const double err = norm_fro(dy) / std::sqrt(n_entries);
    if (stats) stats->iterations = it;
    if (err <= eps) return scale(y, 1.0 / x_avg);
    growth = (err > prev_err) ? growth + 1 : 0;
    if (growth >= 5) throw fail("diverging increments", err, it);
    prev_err = err;
  }
  throw fail("iteration cap exceeded", prev_err, max_iterations);
}

}  // namespace ttor
