// TEST INFRASTRUCTURE ONLY — CPU oracle (see linalg.hpp header).
//
// Restatement of the TTRep path of /root/reference/proj/include/ttsw/swe.hpp
// (:84-119, :190-273, :299-454) and the periodic branch of tt_ghosted
// (/root/reference/proj/src/cases.cpp:298-309).
#pragma once

#include <functional>
#include <variant>

#include "recon.hpp"

namespace ttor {

enum class Model { Linear = 0, Nonlinear = 1 };

struct PhysParams {  // swe.hpp:19-26
  double g = 10.0, f = 1e-4, H = 1000.0;
};
struct Grid {  // swe.hpp:28-38
  Index nx = 0, ny = 0;
  double lx = 1.0, ly = 1.0;
  double dx() const { return lx / double(nx); }
  double dy() const { return ly / double(ny); }
};

inline constexpr double kNoRound = -1.0;  // swe.hpp:41

/// TTRep (swe.hpp:84-119).
struct Rep {
  static TT round_to(const TT& x, double eps) { return eps < 0 ? x : round(x, eps); }
  static TT zero_like(const TT& x) { return TT::zero(x.rows(), x.cols()); }
  static TT scaled(const TT& x, double a) { return scale(x, a); }
  static TT axpy(double a, const TT& x, double b, const TT& y, double eps) {
    return round_to(add(scale(x, a), scale(y, b)), eps);
  }
  static TT mul(const TT& x, const TT& y, double eps) { return round_to(hadamard(x, y), eps); }
  static TT lin(Axis axis, const BandOp& m, const TT& x) { return apply_core_map(x, axis, m); }
  static TT recip(const TT& x, double eps) { return reciprocal_taylor(x, eps); }
  static TT elementwise(const EntryFn& f, std::span<const TT> ops, const TT& guess, double eps,
                        const CrossConfig& base) {
    CrossConfig cfg = base;
    cfg.eps = eps;
    return cross_elementwise(f, ops, guess, cfg);
  }
};

using Triple = std::array<TT, 3>;

struct EpsSchedule {  // swe.hpp:156-159
  std::array<double, 3> var{kNoRound, kNoRound, kNoRound};
  double global = kNoRound;
};

/// Policy-mode rounding tolerance (swe.hpp:134-138): C_eps V^(1/2) dx^(p-1/2) / ||q||_F.
struct EpsPolicy {
  double c_eps = 1.0;
  int order = 3;
  double volume = 1.0;
  double clip = 1e-3;
};

/// eps_global (swe.hpp:143-146): clip when every component vanishes, otherwise unclipped.
inline double eps_global(const EpsPolicy& p, double dx, double max_norm) {
  if (max_norm <= 0.0) return p.clip;
  return p.c_eps * std::sqrt(p.volume) * std::pow(dx, p.order - 0.5) / max_norm;
}

/// eps_for_variable (swe.hpp:150-154): clipped at p.clip.
inline double eps_for_variable(double q_norm, const EpsPolicy& p, double dx) {
  if (q_norm <= 0.0) return p.clip;
  const double value = p.c_eps * std::sqrt(p.volume) * std::pow(dx, p.order - 0.5) / q_norm;
  return std::min(p.clip, value);
}

/// physical_flux (swe.hpp:190-213).
inline Triple physical_flux(const Triple& u, Axis dir, Model model, const PhysParams& p, double eps) {
  if (model == Model::Linear) {
    const TT zero = Rep::zero_like(u[0]);
    if (dir == Axis::X) return {Rep::scaled(u[1], p.H), Rep::scaled(u[0], p.g), zero};
    return {Rep::scaled(u[2], p.H), zero, Rep::scaled(u[0], p.g)};
  }
  const TT inv_h = Rep::recip(u[0], eps);
  const TT vel_x = Rep::mul(u[1], inv_h, eps);
  const TT vel_y = Rep::mul(u[2], inv_h, eps);
  const TT pressure = Rep::scaled(Rep::mul(u[0], u[0], eps), 0.5 * p.g);
  if (dir == Axis::X) {
    // Brace-init evaluates left to right (same rounding order as the reference).
    TT f1 = Rep::axpy(1.0, Rep::mul(u[1], vel_x, eps), 1.0, pressure, eps);
    TT f2 = Rep::mul(u[1], vel_y, eps);
    return {u[1], std::move(f1), std::move(f2)};
  }
  TT f1 = Rep::mul(u[2], vel_x, eps);
  TT f2 = Rep::axpy(1.0, Rep::mul(u[2], vel_y, eps), 1.0, pressure, eps);
  return {u[2], std::move(f1), std::move(f2)};
}

/// LLF wave-speed functor (swe.hpp:342-347).
inline EntryFn llf_lambda_fn(double g) {
  return [g](std::span<const double> v) {
    if (v[0] <= 0.0 || v[2] <= 0.0) throw std::domain_error("nonpositive layer thickness");
    return std::max(std::abs(v[1] / v[0]) + std::sqrt(g * v[0]), std::abs(v[3] / v[2]) + std::sqrt(g * v[2]));
  };
}

/// wave_speed field functor (swe.hpp:225-228).
inline EntryFn wave_speed_fn(double g) {
  return [g](std::span<const double> v) {
    if (v[0] <= 0.0) throw std::domain_error("nonpositive layer thickness");
    return std::abs(v[1] / v[0]) + std::sqrt(g * v[0]);
  };
}

/// llf_flux scalar (swe.hpp:235-248).
inline Triple llf_flux(const Triple& um, const Triple& up, const Triple& fm, const Triple& fp, double lambda,
                       double eps) {
  Triple out;
  for (int c = 0; c < 3; ++c) {
    auto central = Rep::axpy(0.5, fm[c], 0.5, fp[c], eps);
    auto jump = Rep::axpy(1.0, up[c], -1.0, um[c], eps);
    out[c] = Rep::axpy(1.0, central, -0.5 * lambda, jump, eps);
  }
  return out;
}

/// llf_flux field (swe.hpp:251-265).
inline Triple llf_flux(const Triple& um, const Triple& up, const Triple& fm, const Triple& fp, const TT& lambda,
                       double eps) {
  Triple out;
  for (int c = 0; c < 3; ++c) {
    auto central = Rep::axpy(0.5, fm[c], 0.5, fp[c], eps);
    auto jump = Rep::axpy(1.0, up[c], -1.0, um[c], eps);
    out[c] = Rep::axpy(1.0, central, -0.5, Rep::mul(lambda, jump, eps), eps);
  }
  return out;
}

/// coriolis_source (swe.hpp:269-273).
inline Triple coriolis_source(const Triple& u, const PhysParams& p) {
  return {Rep::zero_like(u[0]), Rep::scaled(u[2], p.f), Rep::scaled(u[1], -p.f)};
}

/// SolverOptions (swe.hpp:285-295).
struct SolverOptions {
  Scheme scheme = Scheme::Upwind3;
  Model model = Model::Linear;
  PhysParams params;
  CrossConfig cross;
  double lambda_eps_floor = 1e-6;
};

/// tt_ghosted, both axes periodic (cases.cpp:298-309; no rounding, :343).
inline TT periodic_ghost(const TT& x) {
  TT padded = apply_core_map(x, Axis::Y, periodic_pad_op(x.cols()));
  return apply_core_map(padded, Axis::X, periodic_pad_op(x.rows()));
}

/// tt_ghosted (cases.cpp:298-344) with the DirichletExact strips supplied by the caller:
/// strip_x (6 x (ny+6), rows = ghost rows 0-2 and nx+3..nx+5) holds the exact cell averages
/// the reference evaluates at :319-320, strip_y ((nx+6) x 6, columns = ghost columns) those
/// of :332-333 (its corner rows are zeroed here when both axes are Dirichlet, :336-339).
/// Pad Y then X (periodic or interior), add the rank-6 strips, round when corrected.
inline TT ghosted(const TT& x, bool dir_x, bool dir_y, const Mat* strip_x, const Mat* strip_y, double eps_tt) {
  const Index nx = x.rows(), ny = x.cols();
  TT padded = apply_core_map(x, Axis::Y, dir_y ? interior_pad_op(ny) : periodic_pad_op(ny));
  padded = apply_core_map(padded, Axis::X, dir_x ? interior_pad_op(nx) : periodic_pad_op(nx));
  if (dir_x) {
    if (!strip_x || strip_x->r != 2 * kGhost || strip_x->c != ny + 2 * kGhost)
      throw ShapeError("tt_ghosted: x strip must be 6 x (ny+6)");
    Mat sel(nx + 2 * kGhost, 2 * kGhost);
    for (Index s = 0; s < 2 * kGhost; ++s) sel(s < kGhost ? s : nx + s, s) = 1.0;
    padded = add(padded, TT(sel, *strip_x));
  }
  if (dir_y) {
    if (!strip_y || strip_y->r != nx + 2 * kGhost || strip_y->c != 2 * kGhost)
      throw ShapeError("tt_ghosted: y strip must be (nx+6) x 6");
    Mat sel(2 * kGhost, ny + 2 * kGhost);
    for (Index s = 0; s < 2 * kGhost; ++s) sel(s, s < kGhost ? s : ny + s) = 1.0;
    Mat strip = *strip_y;
    if (dir_x)
      for (Index s = 0; s < 2 * kGhost; ++s)
        for (Index i = 0; i < kGhost; ++i) {
          strip(i, s) = 0.0;
          strip(nx + kGhost + i, s) = 0.0;
        }
    padded = add(padded, TT(strip, sel));
  }
  if ((dir_x || dir_y) && eps_tt >= 0.0) padded = round(padded, eps_tt);
  return padded;
}

/// reconstruct_components (swe.hpp:299-320), both sides at once. The reference
/// calls it once per side and keeps one face each time; the cross RNG is
/// re-seeded per call (cross.hpp:179), so computing both sides once is
/// bit-identical.
inline std::pair<Triple, Triple> reconstruct_components(const Triple& ghosted, Axis axis, const SolverOptions& opt,
                                                        const Grid& grid, double eps_tt) {
  std::pair<Triple, Triple> out;
  for (int c = 0; c < 3; ++c) {
    ReconContext ctx;
    ctx.scheme = opt.scheme;
    ctx.eps_tt = eps_tt < 0 ? 1e-14 : eps_tt;
    ctx.cross = opt.cross;
    ctx.dx = grid.dx();
    ctx.dy = grid.dy();
    auto faces = reconstruct_faces(ghosted[size_t(c)], axis, ctx);
    out.first[size_t(c)] = std::move(faces.minus);
    out.second[size_t(c)] = std::move(faces.plus);
  }
  return out;
}

/// face_wave_speed (swe.hpp:325-354).
inline std::variant<double, TT> face_wave_speed(const Triple& um, const Triple& up, Axis axis,
                                                const SolverOptions& opt, double eps) {
  if (opt.model == Model::Linear) return std::sqrt(opt.params.g * opt.params.H);
  const int mom = axis == Axis::X ? 1 : 2;
  std::array<TT, 4> ops{um[0], um[size_t(mom)], up[0], up[size_t(mom)]};
  const double lambda_eps = std::max(eps, opt.lambda_eps_floor);
  return Rep::elementwise(llf_lambda_fn(opt.params.g), ops, um[0], lambda_eps, opt.cross);
}

/// rhs<TTRep> (swe.hpp:362-423) with periodic fill_ghost.
/// RhsHooks (swe.hpp:276-282): ghost fill of the state at time t (default: both axes
/// periodic, cases.cpp:298-309) and an optional manufactured source at time t.
struct RhsHooks {
  std::function<Triple(const Triple&, double)> fill_ghost;
  std::function<Triple(double)> extra_source;
};

inline Triple rhs(const Triple& u, const Grid& grid, const SolverOptions& opt, const EpsSchedule& eps,
                  double t = 0.0, const RhsHooks* hooks = nullptr) {
  const double flux_eps = opt.model == Model::Nonlinear ? eps.global : kNoRound;
  Triple ghosted;
  if (hooks && hooks->fill_ghost)
    ghosted = hooks->fill_ghost(u, t);
  else
    for (int c = 0; c < 3; ++c) ghosted[size_t(c)] = periodic_ghost(u[size_t(c)]);
  Triple flux_div;
  for (Axis axis : {Axis::X, Axis::Y}) {
    auto [u_minus, u_plus] = reconstruct_components(ghosted, axis, opt, grid, eps.global);
    auto f_minus = physical_flux(u_minus, axis, opt.model, opt.params, flux_eps);
    auto f_plus = physical_flux(u_plus, axis, opt.model, opt.params, flux_eps);
    auto lambda = face_wave_speed(u_minus, u_plus, axis, opt, eps.global);
    Triple fhat = std::holds_alternative<double>(lambda)
                      ? llf_flux(u_minus, u_plus, f_minus, f_plus, std::get<double>(lambda), flux_eps)
                      : llf_flux(u_minus, u_plus, f_minus, f_plus, std::get<TT>(lambda), flux_eps);
    const Index n_axis = axis == Axis::X ? grid.nx : grid.ny;
    const Index n_trans = axis == Axis::X ? grid.ny : grid.nx;
    const Axis trans = axis == Axis::X ? Axis::Y : Axis::X;
    const BandOp w = quadrature_sum_op(opt.scheme, n_trans);
    const BandOp d = difference_op(n_axis);
    const double inv = axis == Axis::X ? 1.0 / grid.dx() : 1.0 / grid.dy();
    for (int c = 0; c < 3; ++c) {
      TT integrated = Rep::lin(trans, w, fhat[size_t(c)]);
      TT difference = Rep::lin(axis, d, integrated);
      if (axis == Axis::X)
        flux_div[size_t(c)] = Rep::scaled(difference, inv);
      else
        flux_div[size_t(c)] = Rep::axpy(1.0, flux_div[size_t(c)], inv, difference, flux_eps);
    }
  }
  auto source = coriolis_source(u, opt.params);
  if (hooks && hooks->extra_source) {  // swe.hpp:412-416
    Triple extra = hooks->extra_source(t);
    for (int c = 0; c < 3; ++c)
      source[size_t(c)] = Rep::axpy(1.0, source[size_t(c)], 1.0, extra[size_t(c)], flux_eps);
  }
  Triple out;
  for (int c = 0; c < 3; ++c) out[size_t(c)] = Rep::axpy(-1.0, flux_div[size_t(c)], 1.0, source[size_t(c)], eps.var[size_t(c)]);
  return out;
}

/// ssprk3 (swe.hpp:428-454).
/// compute_eps_schedule<TTRep> (swe.hpp:167-183): recomputed once per step from the state.
inline EpsSchedule compute_eps_schedule(const Triple& u, const EpsPolicy& policy, double dx) {
  EpsSchedule eps;
  double max_norm = 0.0;
  for (int c = 0; c < 3; ++c) {
    const double n = norm_fro(u[size_t(c)]);
    eps.var[size_t(c)] = eps_for_variable(n, policy, dx);
    max_norm = std::max(max_norm, n);
  }
  eps.global = eps_global(policy, dx, max_norm);
  return eps;
}

inline Triple ssprk3(const Triple& u, double dt, const Grid& grid, const SolverOptions& opt, const EpsSchedule& eps,
                     double t = 0.0, const RhsHooks* hooks = nullptr) {
  if (!(dt > 0)) throw InputError("ssprk3: dt must be positive");
  // stage times t, t + dt, t + dt/2 (swe.hpp:436-449)
  auto euler = [&](const Triple& w, double ts) {
    Triple k = rhs(w, grid, opt, eps, ts, hooks);
    Triple out;
    for (int c = 0; c < 3; ++c) out[size_t(c)] = Rep::axpy(1.0, w[size_t(c)], dt, k[size_t(c)], eps.var[size_t(c)]);
    return out;
  };
  Triple u1 = euler(u, t);
  Triple f1 = euler(u1, t + dt);
  Triple u2;
  for (int c = 0; c < 3; ++c) u2[size_t(c)] = Rep::axpy(0.75, u[size_t(c)], 0.25, f1[size_t(c)], eps.var[size_t(c)]);
  Triple f2 = euler(u2, t + 0.5 * dt);
  Triple out;
  for (int c = 0; c < 3; ++c) out[size_t(c)] = Rep::axpy(1.0 / 3.0, u[size_t(c)], 2.0 / 3.0, f2[size_t(c)], eps.var[size_t(c)]);
  return out;
}

}  // namespace ttor
