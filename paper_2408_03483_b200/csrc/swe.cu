// SWE right-hand side and SSP-RK3 on device TTs: the TTRep path of
// /root/reference/proj/include/ttsw/swe.hpp (:84-119, :190-273, :299-454), the TT
// reconstruction of reconstruction.hpp (:515-616) and the periodic ghosting of
// proj/src/cases.cpp:298-309. Every rounding point and tolerance follows the reference.
#include <cmath>
#include <variant>

#include "kernels.cuh"

namespace ttsw {

/// TTRep static methods (swe.hpp:84-119) over device TTs.
struct CudaTTRep {
  static TT round_to(const TT& x, double eps) { return eps < 0 ? x : round(x, eps); }
  static TT zero_like(const TT& x) { return tt_zero(x->ctx, x->m, x->n); }
  static TT scaled(const TT& x, double a) { return scale(x, a); }
  static TT axpy(double a, const TT& x, double b, const TT& y, double eps) {
    return round_to(add(scale(x, a), scale(y, b)), eps);
  }
  static TT mul(const TT& x, const TT& y, double eps) { return round_to(hadamard(x, y), eps); }
  static TT recip(const TT& x, double eps) { return reciprocal_taylor(x, eps); }
  static TT elementwise(int fn, double param, const std::vector<TT>& ops, const TT& guess, double eps,
                        const CrossConfig& base) {
    CrossConfig cfg = base;
    cfg.eps = eps;
    return cross_elementwise(fn, param, ops, guess, cfg);
  }
};
using Rep = CudaTTRep;

/// Rep::axpy on the three components at once: the three roundings are independent, so
/// they run as one batch (one fused kernel launch); trace order stays c = 0, 1, 2.
static Triple axpy3(double a, const Triple& x, double b, const Triple& y, const std::array<double, 3>& eps) {
  Triple out;
  std::vector<TT> in;
  std::vector<double> e;
  std::vector<int> idx;
  for (int c = 0; c < 3; ++c) {
    TT s = add(scale(x[size_t(c)], a), scale(y[size_t(c)], b));
    if (eps[size_t(c)] < 0) {
      out[size_t(c)] = s;
    } else {
      in.push_back(s);
      e.push_back(eps[size_t(c)]);
      idx.push_back(c);
    }
  }
  auto r = round_batch(in, e);
  for (size_t i = 0; i < idx.size(); ++i) out[size_t(idx[i])] = r[i];
  return out;
}

/// tt_ghosted, both axes periodic: pad Y then X, no rounding (cases.cpp:298-309, :343).
TT periodic_ghost(const TT& x) {
  const TT padded = apply_core_map(x, Axis::Y, make_band_map(0, Scheme::Upwind3, Side::Minus, x->n, 0, 0));
  return apply_core_map(padded, Axis::X, make_band_map(0, Scheme::Upwind3, Side::Minus, x->m, 0, 0));
}

namespace {

/// tt_recon_linear (reconstruction.hpp:515-529).
FacePair tt_recon_linear(const TT& g, Axis axis, Scheme scheme) {
  const Index nx = g->m - 2 * kGhost, ny = g->n - 2 * kGhost;
  const Index n_axis = axis == Axis::X ? nx : ny, n_trans = axis == Axis::X ? ny : nx;
  const Axis trans = axis == Axis::X ? Axis::Y : Axis::X;
  const BandMap q = make_band_map(2, scheme, Side::Minus, n_trans, 0, 0);
  return {apply_core_map(apply_core_map(g, axis, make_band_map(1, scheme, Side::Minus, n_axis, 0, 0)), trans, q),
          apply_core_map(apply_core_map(g, axis, make_band_map(1, scheme, Side::Plus, n_axis, 0, 0)), trans, q)};
}

/// tt_recon_weno (reconstruction.hpp:531-604).
FacePair tt_recon_weno(const TT& g, Axis axis, const ReconContext& ctx) {
  Context* c = g->ctx;
  const Tables& t = recon_tables(Scheme::Weno5);
  const Index nx = g->m - 2 * kGhost, ny = g->n - 2 * kGhost;
  const Index n_axis = axis == Axis::X ? nx : ny, n_trans = axis == Axis::X ? ny : nx;
  const Axis trans = axis == Axis::X ? Axis::Y : Axis::X;
  const int nq = t.nq;
  const double eps1 = axis == Axis::X ? ctx.dx * ctx.dx : ctx.dy * ctx.dy;
  const double eps2 = axis == Axis::X ? ctx.dy * ctx.dy : ctx.dx * ctx.dx;
  CrossConfig cfg = ctx.cross;
  cfg.eps = ctx.eps_tt;

  auto step1 = [&](Side side) {
    std::vector<TT> ops;
    const Index base = side == Side::Minus ? 0 : 1;
    for (Index s = 0; s < 5; ++s)
      ops.push_back(apply_core_map(g, axis, make_band_map(5, Scheme::Weno5, side, n_axis, base + s, n_axis + 1)));
    try {
      return cross_elementwise(side == Side::Minus ? FN_WENO5_S1_MINUS : FN_WENO5_S1_PLUS, eps1, ops, ops[2], cfg);
    } catch (const ConvergenceError& e) {
      throw ConvergenceError(std::string("tt WENO step 1 (") + (side == Side::Minus ? "minus" : "plus") +
                                 " side): " + e.what(),
                             e.residual, e.iterations);
    }
  };
  auto step2 = [&](const TT& lines, Side side) {
    std::vector<TT> ops;
    for (Index s = 0; s < 5; ++s)
      ops.push_back(apply_core_map(lines, trans, make_band_map(6, Scheme::Weno5, side, n_trans, s, 0)));
    // Rank-1 quadrature-index pattern operand (reconstruction.hpp:584-590).
    std::vector<double> pattern(static_cast<size_t>(n_trans * nq)), ones(size_t(n_axis + 1), 1.0);
    for (Index j = 0; j < n_trans; ++j)
      for (int q = 0; q < nq; ++q) pattern[size_t(j * nq + q)] = q;
    if (trans == Axis::Y)
      ops.push_back(tt_from_host(c, n_axis + 1, n_trans * nq, 1, ones.data(), pattern.data()));
    else
      ops.push_back(tt_from_host(c, n_trans * nq, n_axis + 1, 1, pattern.data(), ones.data()));
    try {
      return cross_elementwise(FN_WENO5_S2_QUAD, eps2, ops, ops[2], cfg);
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
  return {minus, plus};
}

}  // namespace

/// reconstruct_faces(TT) (reconstruction.hpp:611-616).
FacePair reconstruct_faces(const TT& g, Axis axis, const ReconContext& ctx) {
  if (ctx.scheme == Scheme::Weno5) return tt_recon_weno(g, axis, ctx);
  return tt_recon_linear(g, axis, ctx.scheme);
}

namespace {

/// physical_flux (swe.hpp:190-213).
Triple physical_flux(const Triple& u, Axis dir, Model model, const PhysParams& p, double eps) {
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
    TT f1 = Rep::axpy(1.0, Rep::mul(u[1], vel_x, eps), 1.0, pressure, eps);
    TT f2 = Rep::mul(u[1], vel_y, eps);
    return {u[1], f1, f2};
  }
  TT f1 = Rep::mul(u[2], vel_x, eps);
  TT f2 = Rep::axpy(1.0, Rep::mul(u[2], vel_y, eps), 1.0, pressure, eps);
  return {u[2], f1, f2};
}

/// Appends region records to the trace in the reference's sequential order.
void emit(Context* ctx, const std::vector<RoundRecord>& recs) {
  if (ctx->trace) ctx->trace->insert(ctx->trace->end(), recs.begin(), recs.end());
}

/// physical_flux (swe.hpp:190-213) of both face sides (minus, plus). Nonlinear: the two
/// sides' roundings run as joint batches (Taylor reciprocals in lock step, then the
/// velocity/pressure products, then the flux products and sums); the records are emitted
/// in the reference order — all of the minus side, then the plus side.
std::array<Triple, 2> physical_flux_pair(const Triple& um, const Triple& up, Axis dir, Model model,
                                         const PhysParams& p, double eps) {
  if (model == Model::Linear || eps <= 0)
    return {physical_flux(um, dir, model, p, eps), physical_flux(up, dir, model, p, eps)};
  Context* ctx = um[0]->ctx;
  const Triple* u[2] = {&um, &up};
  std::vector<RoundRecord> rrec[2];
  auto inv = reciprocal_taylor_batch({um[0], up[0]}, eps, {&rrec[0], &rrec[1]});
  RoundRecord ops[2][6];
  const std::vector<double> e6(6, eps), e4(4, eps), e2(2, eps);
  // vel_x, vel_y, pressure (reference slots 0, 1, 2)
  auto b1 = round_batch_into({hadamard((*u[0])[1], inv[0]), hadamard((*u[0])[2], inv[0]), hadamard((*u[0])[0], (*u[0])[0]),
                              hadamard((*u[1])[1], inv[1]), hadamard((*u[1])[2], inv[1]), hadamard((*u[1])[0], (*u[1])[0])},
                             e6, {&ops[0][0], &ops[0][1], &ops[0][2], &ops[1][0], &ops[1][1], &ops[1][2]});
  std::array<Triple, 2> out;
  if (dir == Axis::X) {
    // u1 * vel_x (slot 3, summed with the pressure at slot 4), f2 = u1 * vel_y (slot 5)
    auto b2 = round_batch_into({hadamard((*u[0])[1], b1[0]), hadamard((*u[0])[1], b1[1]),
                                hadamard((*u[1])[1], b1[3]), hadamard((*u[1])[1], b1[4])},
                               e4, {&ops[0][3], &ops[0][5], &ops[1][3], &ops[1][5]});
    auto b3 = round_batch_into({add(b2[0], scale(b1[2], 0.5 * p.g)), add(b2[2], scale(b1[5], 0.5 * p.g))}, e2,
                               {&ops[0][4], &ops[1][4]});
    out[0] = {(*u[0])[1], b3[0], b2[1]};
    out[1] = {(*u[1])[1], b3[1], b2[3]};
  } else {
    // f1 = u2 * vel_x (slot 3), u2 * vel_y (slot 4, summed with the pressure at slot 5)
    auto b2 = round_batch_into({hadamard((*u[0])[2], b1[0]), hadamard((*u[0])[2], b1[1]),
                                hadamard((*u[1])[2], b1[3]), hadamard((*u[1])[2], b1[4])},
                               e4, {&ops[0][3], &ops[0][4], &ops[1][3], &ops[1][4]});
    auto b3 = round_batch_into({add(b2[1], scale(b1[2], 0.5 * p.g)), add(b2[3], scale(b1[5], 0.5 * p.g))}, e2,
                               {&ops[0][5], &ops[1][5]});
    out[0] = {(*u[0])[2], b2[0], b3[0]};
    out[1] = {(*u[1])[2], b2[2], b3[1]};
  }
  for (int side = 0; side < 2; ++side) {
    emit(ctx, rrec[side]);
    emit(ctx, std::vector<RoundRecord>(ops[side], ops[side] + 6));
  }
  return out;
}

/// llf_flux (swe.hpp:235-265) with the three components' roundings batched: per component
/// the reference order is central, jump, [lambda * jump,] out; the batches are {central,
/// jump} x 3, [{lambda * jump} x 3,] {out} x 3 and the records are emitted in that order.
Triple llf_flux_batched(const Triple& um, const Triple& up, const Triple& fm, const Triple& fp,
                        const std::variant<double, TT>& lambda, double eps) {
  Context* ctx = um[0]->ctx;
  const bool field = std::holds_alternative<TT>(lambda);
  const int per = field ? 4 : 3;
  std::vector<RoundRecord> recs(size_t(3 * per));
  std::vector<TT> in;
  std::vector<RoundRecord*> dst;
  for (int c = 0; c < 3; ++c) {
    in.push_back(add(scale(fm[size_t(c)], 0.5), scale(fp[size_t(c)], 0.5)));
    in.push_back(add(scale(up[size_t(c)], 1.0), scale(um[size_t(c)], -1.0)));
    dst.push_back(&recs[size_t(per * c)]);
    dst.push_back(&recs[size_t(per * c + 1)]);
  }
  auto b1 = round_batch_into(in, std::vector<double>(6, eps), dst);
  std::vector<TT> dis(3);
  if (field) {
    const TT& lam = std::get<TT>(lambda);
    in.clear();
    dst.clear();
    for (int c = 0; c < 3; ++c) {
      in.push_back(hadamard(lam, b1[size_t(2 * c + 1)]));
      dst.push_back(&recs[size_t(per * c + 2)]);
    }
    auto b2 = round_batch_into(in, std::vector<double>(3, eps), dst);
    for (int c = 0; c < 3; ++c) dis[size_t(c)] = scale(b2[size_t(c)], -0.5);
  } else {
    for (int c = 0; c < 3; ++c) dis[size_t(c)] = scale(b1[size_t(2 * c + 1)], -0.5 * std::get<double>(lambda));
  }
  in.clear();
  dst.clear();
  for (int c = 0; c < 3; ++c) {
    in.push_back(add(scale(b1[size_t(2 * c)], 1.0), dis[size_t(c)]));
    dst.push_back(&recs[size_t(per * c + per - 1)]);
  }
  auto b3 = round_batch_into(in, std::vector<double>(3, eps), dst);
  emit(ctx, recs);
  return {b3[0], b3[1], b3[2]};
}

/// llf_flux, scalar dissipation (swe.hpp:235-248).
Triple llf_flux(const Triple& um, const Triple& up, const Triple& fm, const Triple& fp, double lambda, double eps) {
  Triple out;
  for (int c = 0; c < 3; ++c) {
    auto central = Rep::axpy(0.5, fm[c], 0.5, fp[c], eps);
    auto jump = Rep::axpy(1.0, up[c], -1.0, um[c], eps);
    out[c] = Rep::axpy(1.0, central, -0.5 * lambda, jump, eps);
  }
  return out;
}

/// llf_flux, field dissipation (swe.hpp:251-265).
Triple llf_flux(const Triple& um, const Triple& up, const Triple& fm, const Triple& fp, const TT& lambda, double eps) {
  Triple out;
  for (int c = 0; c < 3; ++c) {
    auto central = Rep::axpy(0.5, fm[c], 0.5, fp[c], eps);
    auto jump = Rep::axpy(1.0, up[c], -1.0, um[c], eps);
    out[c] = Rep::axpy(1.0, central, -0.5, Rep::mul(lambda, jump, eps), eps);
  }
  return out;
}

/// coriolis_source (swe.hpp:269-273).
Triple coriolis_source(const Triple& u, const PhysParams& p) {
  return {Rep::zero_like(u[0]), Rep::scaled(u[2], p.f), Rep::scaled(u[1], -p.f)};
}

/// face_wave_speed (swe.hpp:325-354).
std::variant<double, TT> face_wave_speed(const Triple& um, const Triple& up, Axis axis, const SolverOptions& opt,
                                         double eps) {
  if (opt.model == Model::Linear) return std::sqrt(opt.params.g * opt.params.H);
  const int mom = axis == Axis::X ? 1 : 2;
  std::vector<TT> ops{um[0], um[size_t(mom)], up[0], up[size_t(mom)]};
  const double lambda_eps = std::max(eps, opt.lambda_eps_floor);
  return Rep::elementwise(FN_LLF_LAMBDA, opt.params.g, ops, um[0], lambda_eps, opt.cross);
}

}  // namespace

/// rhs<TTRep> (swe.hpp:362-423) with periodic fill_ghost. Faces of both sides are
/// reconstructed once per axis (the reference builds them twice, :378-381; the
/// cross RNG is re-seeded per call so reuse is bit-identical).
Triple Solver::rhs(const Triple& u) {
  const double flux_eps = opt.model == Model::Nonlinear ? eps.global : kNoRound;
  const double dx = 1.0 / double(n), dy = 1.0 / double(n);
  Triple ghosted;
  for (int c = 0; c < 3; ++c) ghosted[size_t(c)] = periodic_ghost(u[size_t(c)]);
  Triple flux_div;
  for (Axis axis : {Axis::X, Axis::Y}) {
    Triple um, up;
    for (int c = 0; c < 3; ++c) {
      ReconContext rc;
      rc.scheme = opt.scheme;
      rc.eps_tt = eps.global < 0 ? 1e-14 : eps.global;
      rc.cross = opt.cross;
      rc.dx = dx;
      rc.dy = dy;
      FacePair f = reconstruct_faces(ghosted[size_t(c)], axis, rc);
      um[size_t(c)] = f.minus;
      up[size_t(c)] = f.plus;
    }
    auto fpair = physical_flux_pair(um, up, axis, opt.model, opt.params, flux_eps);
    const Triple& fm = fpair[0];
    const Triple& fp = fpair[1];
    auto lambda = face_wave_speed(um, up, axis, opt, eps.global);
    Triple fhat;
    if (flux_eps >= 0)
      fhat = llf_flux_batched(um, up, fm, fp, lambda, flux_eps);
    else
      fhat = std::holds_alternative<double>(lambda) ? llf_flux(um, up, fm, fp, std::get<double>(lambda), flux_eps)
                                                     : llf_flux(um, up, fm, fp, std::get<TT>(lambda), flux_eps);
    const Index n_axis = n, n_trans = n;
    const Axis trans = axis == Axis::X ? Axis::Y : Axis::X;
    const BandMap w = make_band_map(3, opt.scheme, Side::Minus, n_trans, 0, 0);
    const BandMap d = make_band_map(4, opt.scheme, Side::Minus, n_axis, 0, 0);
    const double inv = axis == Axis::X ? 1.0 / dx : 1.0 / dy;
    Triple difference;
    for (int c = 0; c < 3; ++c) {
      TT integrated = apply_core_map(fhat[size_t(c)], trans, w);
      difference[size_t(c)] = apply_core_map(integrated, axis, d);
    }
    if (axis == Axis::X) {
      for (int c = 0; c < 3; ++c) flux_div[size_t(c)] = Rep::scaled(difference[size_t(c)], inv);
    } else {
      // the three component sums are independent roundings: one batch, records in order c
      flux_div = axpy3(1.0, flux_div, inv, difference, {flux_eps, flux_eps, flux_eps});
    }
  }
  auto source = coriolis_source(u, opt.params);
  return axpy3(-1.0, flux_div, 1.0, source, eps.var);
}

/// ssprk3 (swe.hpp:428-454); tolerances frozen for the step.
void Solver::step() {
  if (!(dt > 0)) throw InputError("ssprk3: dt must be positive");
  ctx->trace = tracing ? &trace : nullptr;
  ctx->ctrace = tracing ? &ctrace : nullptr;
  auto euler = [&](const Triple& w) {
    Triple k = rhs(w);
    return axpy3(1.0, w, dt, k, eps.var);
  };
  const Triple& u = state;
  Triple u1 = euler(u);
  Triple f1 = euler(u1);
  Triple u2 = axpy3(0.75, u, 0.25, f1, eps.var);
  Triple f2 = euler(u2);
  state = axpy3(1.0 / 3.0, u, 2.0 / 3.0, f2, eps.var);
  ctx->trace = nullptr;
  ctx->ctrace = nullptr;
}

}  // namespace ttsw
