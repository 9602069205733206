// TEST INFRASTRUCTURE ONLY — CPU oracle (see linalg.hpp header).
//
// Restatement of the TT half of /root/reference/proj/include/ttsw/reconstruction.hpp:
// tables (:33-171), pointwise WENO functors (:174-247), banded operator builders
// (:428-501), tt_recon_linear (:515-529), tt_recon_weno (:531-604).
#pragma once

#include <array>

#include "cross.hpp"

namespace ttor {

enum class Scheme { Upwind3 = 0, Upwind5 = 1, Weno5 = 2 };
enum class Side { Minus = 0, Plus = 1 };

constexpr int order(Scheme s) { return s == Scheme::Upwind3 ? 3 : 5; }
constexpr int stencil_radius(Scheme s) { return s == Scheme::Upwind3 ? 1 : 2; }
constexpr int quadrature_points(Scheme s) { return s == Scheme::Upwind3 ? 2 : 3; }
constexpr bool is_weno(Scheme s) { return s == Scheme::Weno5; }

struct Quad {
  int n = 0;
  std::array<double, 3> offset{}, weight{};
};

/// gauss_rule (reconstruction.hpp:33-49).
inline Quad gauss_rule(int n_q) {
  Quad q;
  q.n = n_q;
  if (n_q == 2) {
    const double a = 1.0 / (2.0 * std::sqrt(3.0));
    q.offset = {-a, a, 0.0};
    q.weight = {0.5, 0.5, 0.0};
  } else if (n_q == 3) {
    const double b = std::sqrt(3.0 / 5.0) / 2.0;
    q.offset = {-b, 0.0, b};
    q.weight = {5.0 / 18.0, 8.0 / 18.0, 5.0 / 18.0};
  } else {
    throw InputError("gauss_rule: only 2- and 3-point rules are supported");
  }
  return q;
}

/// point_reconstruction_coefficients (reconstruction.hpp:55-70).
inline std::vector<double> point_coeffs(const std::vector<int>& cells, double delta) {
  const Index k = Index(cells.size());
  Mat a(k, k);
  std::vector<double> rhs(static_cast<size_t>(k));
  for (Index q = 0; q < k; ++q) {
    for (Index l = 0; l < k; ++l) {
      const double lo = double(cells[size_t(l)]) - 0.5, hi = double(cells[size_t(l)]) + 0.5;
      a(q, l) = (std::pow(hi, double(q + 1)) - std::pow(lo, double(q + 1))) / double(q + 1);
    }
    rhs[size_t(q)] = std::pow(delta, double(q));
  }
  return solve_square(a, rhs);
}

/// ideal_weights (reconstruction.hpp:74-83).
inline std::vector<double> ideal_weights(const Mat& cand, const std::vector<double>& wide, int radius) {
  const Index n_cand = radius + 1;
  Mat a(Index(wide.size()), n_cand);
  for (Index r = 0; r < n_cand; ++r)
    for (Index l = 0; l < radius + 1; ++l) a(radius - r + l, r) = cand(r, l);
  return lstsq(a, wide);
}

/// ReconTables (reconstruction.hpp:89-111).
struct Tables {
  Scheme scheme{};
  int radius = 0;
  Quad quad;
  Mat step1_c;
  std::vector<double> step1_ideal, step1_row;
  std::array<Mat, 3> c;
  std::array<std::vector<double>, 3> gamma, point_row;
  std::vector<double> gamma_plus, gamma_minus;
  double sigma_plus = 107.0 / 40.0, sigma_minus = 67.0 / 40.0;
  std::vector<double> weno_d;
};

/// make_recon_tables (reconstruction.hpp:113-160).
inline Tables make_tables(Scheme scheme) {
  Tables t;
  t.scheme = scheme;
  t.radius = stencil_radius(scheme);
  t.quad = gauss_rule(quadrature_points(scheme));
  const int k = t.radius;
  auto cells = [](int first, int count) -> std::vector<int> {
    std::vector<int> v(static_cast<size_t>(count));
    for (int i = 0; i < count; ++i) v[size_t(i)] = first + i;
    return v;
  };
  const std::vector<int> wide = cells(-k, 2 * k + 1);
  t.step1_c = Mat(k + 1, k + 1);
  for (int r = 0; r <= k; ++r) {
    auto c = point_coeffs(cells(-r, k + 1), 0.5);
    for (int l = 0; l <= k; ++l) t.step1_c(r, l) = c[size_t(l)];
  }
  t.step1_row = point_coeffs(wide, 0.5);
  t.step1_ideal = ideal_weights(t.step1_c, t.step1_row, k);
  for (int m = 0; m < t.quad.n; ++m) {
    const double delta = t.quad.offset[size_t(m)];
    t.c[size_t(m)] = Mat(k + 1, k + 1);
    for (int r = 0; r <= k; ++r) {
      auto c = point_coeffs(cells(-r, k + 1), delta);
      for (int l = 0; l <= k; ++l) t.c[size_t(m)](r, l) = c[size_t(l)];
    }
    t.point_row[size_t(m)] = point_coeffs(wide, delta);
    t.gamma[size_t(m)] = ideal_weights(t.c[size_t(m)], t.point_row[size_t(m)], k);
  }
  if (k == 2) {
    t.gamma_plus = {9.0 / 214, 98.0 / 107, 9.0 / 214};
    t.gamma_minus = {9.0 / 67, 49.0 / 67, 9.0 / 67};
    t.weno_d = {3.0 / 10, 3.0 / 5, 1.0 / 10};
  }
  return t;
}

/// recon_tables (reconstruction.hpp:162-171).
inline const Tables& recon_tables(Scheme s) {
  static const Tables u3 = make_tables(Scheme::Upwind3);
  static const Tables u5 = make_tables(Scheme::Upwind5);
  static const Tables w5 = make_tables(Scheme::Weno5);
  return s == Scheme::Upwind3 ? u3 : (s == Scheme::Upwind5 ? u5 : w5);
}

/// smoothness_indicators (reconstruction.hpp:174-185).
inline std::array<double, 3> smoothness(const double* v) {
  const double c = 13.0 / 12.0;
  std::array<double, 3> b;
  b[0] = c * std::pow(v[2] - 2 * v[3] + v[4], 2) + 0.25 * std::pow(3 * v[2] - 4 * v[3] + v[4], 2);
  b[1] = c * std::pow(v[1] - 2 * v[2] + v[3], 2) + 0.25 * std::pow(v[1] - v[3], 2);
  b[2] = c * std::pow(v[0] - 2 * v[1] + v[2], 2) + 0.25 * std::pow(v[0] - 4 * v[1] + 3 * v[2], 2);
  return b;
}

/// weno_weights (reconstruction.hpp:188-200).
inline std::array<double, 3> weno_weights(const std::array<double, 3>& beta,
                                          const std::array<double, 3>& ideal, double eps) {
  std::array<double, 3> alpha;
  double total = 0;
  for (int r = 0; r < 3; ++r) {
    const double d = beta[size_t(r)] + eps;
    alpha[size_t(r)] = ideal[size_t(r)] / (d * d);
    total += alpha[size_t(r)];
  }
  for (auto& a : alpha) a /= total;
  return alpha;
}

/// weno5_step1_value (reconstruction.hpp:205-218).
inline double weno5_step1(const double* v, const Tables& t, double eps) {
  const auto beta = smoothness(v);
  const auto w = weno_weights(beta, {t.weno_d[0], t.weno_d[1], t.weno_d[2]}, eps);
  double out = 0;
  for (int r = 0; r < 3; ++r) {
    double cand = 0;
    for (int l = 0; l < 3; ++l) cand += t.step1_c(r, l) * v[2 - r + l];
    out += w[size_t(r)] * cand;
  }
  return out;
}

/// weno5_step2_value (reconstruction.hpp:221-247).
inline double weno5_step2(const double* v, int m, const Tables& t, double eps) {
  const auto beta = smoothness(v);
  std::array<double, 3> cand;
  for (int r = 0; r < 3; ++r) {
    cand[size_t(r)] = 0;
    for (int l = 0; l < 3; ++l) cand[size_t(r)] += t.c[size_t(m)](r, l) * v[2 - r + l];
  }
  if (m == 1) {
    const auto wp = weno_weights(beta, {t.gamma_plus[0], t.gamma_plus[1], t.gamma_plus[2]}, eps);
    const auto wm = weno_weights(beta, {t.gamma_minus[0], t.gamma_minus[1], t.gamma_minus[2]}, eps);
    double up = 0, um = 0;
    for (int r = 0; r < 3; ++r) {
      up += wp[size_t(r)] * cand[size_t(r)];
      um += wm[size_t(r)] * cand[size_t(r)];
    }
    return t.sigma_plus * up - t.sigma_minus * um;
  }
  const auto& g = t.gamma[size_t(m)];
  const auto w = weno_weights(beta, {g[0], g[1], g[2]}, eps);
  double out = 0;
  for (int r = 0; r < 3; ++r) out += w[size_t(r)] * cand[size_t(r)];
  return out;
}

// --- banded operators (reconstruction.hpp:428-501, cases.cpp:302-308) --------

/// step1_matrix (reconstruction.hpp:428-438): (n+1) x (n+6).
inline BandOp step1_op(Scheme scheme, Side side, Index n) {
  const auto& t = recon_tables(scheme);
  const int k = t.radius;
  std::vector<double> row = t.step1_row;
  if (side == Side::Plus) std::reverse(row.begin(), row.end());
  const Index base = (side == Side::Minus) ? kGhost - k - 1 : kGhost - k;
  BandOp op;
  op.n_out = n + 1;
  op.n_in = n + 2 * kGhost;
  op.rows.resize(size_t(n + 1));
  for (Index i = 0; i <= n; ++i)
    for (int l = 0; l < 2 * k + 1; ++l) op.rows[size_t(i)].push_back({i + base + l, row[size_t(l)]});
  return op;
}

/// quadrature_point_matrix (reconstruction.hpp:441-451): (n*n_q) x (n+6).
inline BandOp quadrature_point_op(Scheme scheme, Index n) {
  const auto& t = recon_tables(scheme);
  const int k = t.radius, n_q = t.quad.n;
  BandOp op;
  op.n_out = n * n_q;
  op.n_in = n + 2 * kGhost;
  op.rows.resize(size_t(n * n_q));
  for (Index j = 0; j < n; ++j)
    for (int q = 0; q < n_q; ++q)
      for (int l = 0; l < 2 * k + 1; ++l)
        op.rows[size_t(j * n_q + q)].push_back({j + kGhost - k + l, t.point_row[size_t(q)][size_t(l)]});
  return op;
}

/// quadrature_sum_matrix (reconstruction.hpp:454-460): n x (n*n_q).
inline BandOp quadrature_sum_op(Scheme scheme, Index n) {
  const auto& t = recon_tables(scheme);
  BandOp op;
  op.n_out = n;
  op.n_in = n * t.quad.n;
  op.rows.resize(size_t(n));
  for (Index j = 0; j < n; ++j)
    for (int q = 0; q < t.quad.n; ++q) op.rows[size_t(j)].push_back({j * t.quad.n + q, t.quad.weight[size_t(q)]});
  return op;
}

/// interface_difference_matrix (reconstruction.hpp:463-470): n x (n+1).
inline BandOp difference_op(Index n) {
  BandOp op;
  op.n_out = n;
  op.n_in = n + 1;
  op.rows.resize(size_t(n));
  for (Index i = 0; i < n; ++i) op.rows[size_t(i)] = {{i, -1.0}, {i + 1, 1.0}};
  return op;
}

/// periodic_pad_matrix (reconstruction.hpp:473-478): (n+6) x n.
inline BandOp periodic_pad_op(Index n) {
  BandOp op;
  op.n_out = n + 2 * kGhost;
  op.n_in = n;
  op.rows.resize(size_t(n + 2 * kGhost));
  for (Index i = 0; i < n + 2 * kGhost; ++i) op.rows[size_t(i)] = {{((i - kGhost) % n + n) % n, 1.0}};
  return op;
}

/// interior_pad_matrix (reconstruction.hpp:481-485): (n+6) x n, ghost rows zero.
inline BandOp interior_pad_op(Index n) {
  BandOp op;
  op.n_out = n + 2 * kGhost;
  op.n_in = n;
  op.rows.resize(size_t(n + 2 * kGhost));
  for (Index i = 0; i < n; ++i) op.rows[size_t(i + kGhost)] = {{i, 1.0}};
  return op;
}

/// row_slice_matrix (reconstruction.hpp:488-492).
inline BandOp row_slice_op(Index offset, Index rows, Index in_rows) {
  BandOp op;
  op.n_out = rows;
  op.n_in = in_rows;
  op.rows.resize(size_t(rows));
  for (Index i = 0; i < rows; ++i) op.rows[size_t(i)] = {{offset + i, 1.0}};
  return op;
}

/// quadrature_slice_matrix (reconstruction.hpp:496-501).
inline BandOp quadrature_slice_op(Index s, Index n, int n_q, int radius) {
  BandOp op;
  op.n_out = n * n_q;
  op.n_in = n + 2 * kGhost;
  op.rows.resize(size_t(n * n_q));
  for (Index j = 0; j < n; ++j)
    for (int q = 0; q < n_q; ++q) op.rows[size_t(j * n_q + q)] = {{j + kGhost - radius + s, 1.0}};
  return op;
}

struct FacePair {
  TT minus, plus;
};

/// TTReconContext (reconstruction.hpp:505-511).
struct ReconContext {
  Scheme scheme{};
  double eps_tt = 1e-12;
  CrossConfig cross;
  double dx = 1.0, dy = 1.0;
};

/// tt_recon_linear (reconstruction.hpp:515-529).
inline FacePair tt_recon_linear(const TT& g, Axis axis, Scheme scheme) {
  const Index nx = g.rows() - 2 * kGhost, ny = g.cols() - 2 * kGhost;
  const Index n_axis = axis == Axis::X ? nx : ny, n_trans = axis == Axis::X ? ny : nx;
  const Axis trans = axis == Axis::X ? Axis::Y : Axis::X;
  BandOp q = quadrature_point_op(scheme, n_trans);
  return {apply_core_map(apply_core_map(g, axis, step1_op(scheme, Side::Minus, n_axis)), trans, q),
          apply_core_map(apply_core_map(g, axis, step1_op(scheme, Side::Plus, n_axis)), trans, q)};
}

/// tt_recon_weno (reconstruction.hpp:531-604).
inline FacePair tt_recon_weno(const TT& g, Axis axis, const ReconContext& ctx) {
  const auto& t = recon_tables(Scheme::Weno5);
  const Index nx = g.rows() - 2 * kGhost, ny = g.cols() - 2 * kGhost;
  const Index n_axis = axis == Axis::X ? nx : ny, n_trans = axis == Axis::X ? ny : nx;
  const Axis trans = axis == Axis::X ? Axis::Y : Axis::X;
  const int n_q = t.quad.n;
  const double eps1 = axis == Axis::X ? ctx.dx * ctx.dx : ctx.dy * ctx.dy;
  const double eps2 = axis == Axis::X ? ctx.dy * ctx.dy : ctx.dx * ctx.dx;
  CrossConfig cfg = ctx.cross;
  cfg.eps = ctx.eps_tt;

  EntryFn fun_minus = [&t, eps1](std::span<const double> v) { return weno5_step1(v.data(), t, eps1); };
  EntryFn fun_plus = [&t, eps1](std::span<const double> v) {
    const double rev[5] = {v[4], v[3], v[2], v[1], v[0]};
    return weno5_step1(rev, t, eps1);
  };
  EntryFn fun_quad = [&t, eps2](std::span<const double> v) {
    const int m = int(v[5] + 0.5);
    return weno5_step2(v.data(), m, t, eps2);
  };

  auto step1 = [&](Side side) {
    std::vector<TT> ops;
    const Index base = side == Side::Minus ? 0 : 1;
    for (Index s = 0; s < 5; ++s)
      ops.push_back(apply_core_map(g, axis, row_slice_op(base + s, n_axis + 1, n_axis + 2 * kGhost)));
    const auto& fun = side == Side::Minus ? fun_minus : fun_plus;
    try {
      return cross_elementwise(fun, ops, ops[2], cfg);
    } catch (const ConvergenceError& e) {
      throw ConvergenceError(std::string("tt WENO step 1 (") + (side == Side::Minus ? "minus" : "plus") +
                                 " side): " + e.what(),
                             e.residual, e.iterations);
    }
  };
  auto step2 = [&](const TT& lines, Side side) {
    std::vector<TT> ops;
    for (Index s = 0; s < 5; ++s)
      ops.push_back(apply_core_map(lines, trans, quadrature_slice_op(s, n_trans, n_q, t.radius)));
    Mat pattern(1, n_trans * n_q);
    for (Index j = 0; j < n_trans; ++j)
      for (int q = 0; q < n_q; ++q) pattern(0, j * n_q + q) = q;
    if (trans == Axis::Y)
      ops.emplace_back(Mat(n_axis + 1, 1, 1.0), pattern);
    else
      ops.emplace_back(pattern.transpose(), Mat(1, n_axis + 1, 1.0));
    try {
      return cross_elementwise(fun_quad, ops, ops[2], cfg);
    } catch (const ConvergenceError& e) {
      throw ConvergenceError(std::string("tt WENO step 2 (") + (side == Side::Minus ? "minus" : "plus") +
                                 " side): " + e.what(),
                             e.residual, e.iterations);
    }
  };
  TT m1 = step1(Side::Minus);
  TT minus = step2(m1, Side::Minus);
  TT p1 = step1(Side::Plus);
  TT plus = step2(p1, Side::Plus);
  return {std::move(minus), std::move(plus)};
}

/// reconstruct_faces (reconstruction.hpp:611-616).
inline FacePair reconstruct_faces(const TT& g, Axis axis, const ReconContext& ctx) {
  if (is_weno(ctx.scheme)) return tt_recon_weno(g, axis, ctx);
  return tt_recon_linear(g, axis, ctx.scheme);
}

}  // namespace ttor
