// SWE right-hand side and SSP-RK3 on device TTs: the TTRep path of
// /root/reference/proj/include/ttsw/swe.hpp (:84-119, :190-273, :299-454), the TT
// reconstruction of reconstruction.hpp (:515-616) and the periodic ghosting of
// proj/src/cases.cpp:298-309. Every rounding point and tolerance follows the reference.
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <chrono>
#include <variant>
#include <memory>
#include <thread>
#include <functional>
#include <exception>

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

/// interior_pad_matrix (reconstruction.hpp:481-485) applied to one core: the (n+6) x r
/// padded core is the input in rows 3..n+2 and zero ghost rows (a memset and one strided
/// device-to-device copy; the other core is shared).
static TT interior_pad(const TT& xin, Axis axis) {
  const TT x = materialize(xin);
  Context* ctx = x->ctx;
  const Index n = axis == Axis::X ? x->m : x->n, r = x->r, np = n + 2 * kGhost;
  auto buf = std::make_shared<DBuf>(ctx, size_t(np * r));
  TTSW_CUDA(cudaMemsetAsync(buf->p, 0, sizeof(double) * size_t(np * r), ctx->stream));
  TTSW_CUDA(cudaMemcpy2DAsync(buf->p + kGhost, sizeof(double) * size_t(np), axis == Axis::X ? x->X : x->Yt,
                              sizeof(double) * size_t(n), sizeof(double) * size_t(n), size_t(r),
                              cudaMemcpyDeviceToDevice, ctx->stream));
  if (axis == Axis::X) return std::make_shared<DevTT>(ctx, np, x->n, r, buf, x->yb);
  return std::make_shared<DevTT>(ctx, x->m, np, r, x->xb, buf);
}

/// tt_ghosted (cases.cpp:298-344) with the DirichletExact strips supplied by the caller
/// (the exact cell averages of :319-320 / :332-333 are the verification case's, not the
/// solver's): pad Y then X (periodic_pad_matrix or interior_pad_matrix), add the rank-6
/// strips TT(selector, strip_x) and TT(strip_y, selector^T) (strip_y's corner rows zeroed
/// when both axes are Dirichlet, :336-339), round at eps_tt when a strip was added.
TT ghosted(const TT& x, bool dir_x, bool dir_y, const double* strip_x, const double* strip_y, double eps_tt,
           RoundRecord* rec) {
  Context* ctx = x->ctx;
  const Index nx = x->m, ny = x->n, gx = nx + 2 * kGhost, gy = ny + 2 * kGhost, w = 2 * kGhost;
  TT padded = dir_y ? interior_pad(x, Axis::Y)
                    : apply_core_map(x, Axis::Y, make_band_map(0, Scheme::Upwind3, Side::Minus, ny, 0, 0));
  padded = dir_x ? interior_pad(padded, Axis::X)
                 : apply_core_map(padded, Axis::X, make_band_map(0, Scheme::Upwind3, Side::Minus, nx, 0, 0));
  if (dir_x) {
    if (!strip_x) throw ShapeError("tt_ghosted: x strip required for a Dirichlet x boundary");
    std::vector<double> sel(size_t(gx * w), 0.0);
    for (Index s = 0; s < w; ++s) sel[size_t((s < kGhost ? s : nx + s) + s * gx)] = 1.0;
    padded = add(padded, tt_from_host(ctx, gx, gy, w, sel.data(), strip_x));
  }
  if (dir_y) {
    if (!strip_y) throw ShapeError("tt_ghosted: y strip required for a Dirichlet y boundary");
    std::vector<double> sel(size_t(w * gy), 0.0), strip(strip_y, strip_y + gx * w);
    for (Index s = 0; s < w; ++s) sel[size_t(s + (s < kGhost ? s : ny + s) * w)] = 1.0;
    if (dir_x)
      for (Index s = 0; s < w; ++s)
        for (Index i = 0; i < kGhost; ++i) strip[size_t(i + s * gx)] = strip[size_t(nx + kGhost + i + s * gx)] = 0.0;
    padded = add(padded, tt_from_host(ctx, gx, gy, w, strip.data(), sel.data()));
  }
  if ((dir_x || dir_y) && eps_tt >= 0.0) return round(padded, eps_tt, rec);
  return padded;
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
/// WENO5 step-1 operands (reconstruction.hpp:558-565): five shifted row slices of the
/// ghosted field along `axis`, base 0 for the minus side and 1 for the plus side.
std::vector<TT> weno_step1_ops(const TT& g, Axis axis, Side side) {
  const Index nx = g->m - 2 * kGhost, ny = g->n - 2 * kGhost;
  const Index n_axis = axis == Axis::X ? nx : ny;
  std::vector<TT> ops;
  const Index base = side == Side::Minus ? 0 : 1;
  for (Index s = 0; s < 5; ++s)
    ops.push_back(apply_core_map(g, axis, make_band_map(5, Scheme::Weno5, side, n_axis, base + s, n_axis + 1)));
  return ops;
}

/// One side of tt_recon_weno (reconstruction.hpp:531-604) on context `k`: the step-1
/// cross over `ops1` (weno_step1_ops) and the step-2 cross over its quadrature slices.
TT weno_side(Context* k, const std::vector<TT>& ops1, Index nx, Index ny, Axis axis, Side side,
             const ReconContext& ctx) {
  const Tables& t = recon_tables(Scheme::Weno5);
  const Index n_axis = axis == Axis::X ? nx : ny, n_trans = axis == Axis::X ? ny : nx;
  const Axis trans = axis == Axis::X ? Axis::Y : Axis::X;
  const int nq = t.nq;
  const double eps1 = axis == Axis::X ? ctx.dx * ctx.dx : ctx.dy * ctx.dy;
  const double eps2 = axis == Axis::X ? ctx.dy * ctx.dy : ctx.dx * ctx.dx;
  CrossConfig cfg = ctx.cross;
  cfg.eps = ctx.eps_tt;
  TT lines;
  try {
    lines = cross_elementwise_on(k, side == Side::Minus ? FN_WENO5_S1_MINUS : FN_WENO5_S1_PLUS, eps1, ops1, ops1[2],
                                 cfg);
  } catch (const ConvergenceError& e) {
    throw ConvergenceError(std::string("tt WENO step 1 (") + (side == Side::Minus ? "minus" : "plus") +
                               " side): " + e.what(),
                           e.residual, e.iterations);
  }
  std::vector<TT> ops;
  for (Index s = 0; s < 5; ++s)
    ops.push_back(apply_core_map(lines, trans, make_band_map(6, Scheme::Weno5, side, n_trans, s, 0)));
  // Rank-1 quadrature-index pattern operand (reconstruction.hpp:584-590).
  std::vector<double> pattern(static_cast<size_t>(n_trans * nq)), ones(size_t(n_axis + 1), 1.0);
  for (Index j = 0; j < n_trans; ++j)
    for (int q = 0; q < nq; ++q) pattern[size_t(j * nq + q)] = q;
  if (trans == Axis::Y)
    ops.push_back(tt_from_host(k, n_axis + 1, n_trans * nq, 1, ones.data(), pattern.data()));
  else
    ops.push_back(tt_from_host(k, n_trans * nq, n_axis + 1, 1, pattern.data(), ones.data()));
  try {
    return cross_elementwise_on(k, FN_WENO5_S2_QUAD, eps2, ops, ops[2], cfg);
  } catch (const ConvergenceError& e) {
    throw ConvergenceError(std::string("tt WENO step 2 (") + (side == Side::Minus ? "minus" : "plus") +
                               " side): " + e.what(),
                           e.residual, e.iterations);
  }
}

FacePair tt_recon_weno(const TT& g, Axis axis, const ReconContext& ctx) {
  const Index nx = g->m - 2 * kGhost, ny = g->n - 2 * kGhost;
  TT minus = weno_side(g->ctx, weno_step1_ops(g, axis, Side::Minus), nx, ny, axis, Side::Minus, ctx);
  TT plus = weno_side(g->ctx, weno_step1_ops(g, axis, Side::Plus), nx, ny, axis, Side::Plus, ctx);
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

/// physical_flux (swe.hpp:190-213), nonlinear, of several face sides at once (side s:
/// state u[s], direction dir[s]). The sides' roundings run as joint batches — the Taylor
/// reciprocals in lock step, then {vel_x, vel_y, pressure} of every side, then the flux
/// products, then the sums with the pressure — and recs[s] receives side s's rounding
/// records in the reference's order (reciprocal, then slots 0..5 below).
std::vector<Triple> physical_flux_multi(const std::vector<const Triple*>& u, const std::vector<Axis>& dir,
                                        const PhysParams& p, double eps,
                                        std::vector<std::vector<RoundRecord>>& recs) {
  const size_t ns = u.size();
  recs.assign(ns, {});
  std::vector<TT> h(ns);
  std::vector<std::vector<RoundRecord>*> sinks(ns);
  for (size_t s = 0; s < ns; ++s) {
    h[s] = (*u[s])[0];
    sinks[s] = &recs[s];
  }
  static const bool prof_on = std::getenv("TTSW_PROFILE_RHS") != nullptr;
  Context* pc = h[0]->ctx;
  auto t0 = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (!prof_on) return;
    pc->sync();
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "phys %-8s %8.2f ms\n", what, std::chrono::duration<double, std::milli>(now - t0).count());
    t0 = now;
  };
  auto inv = reciprocal_taylor_batch(h, eps, sinks);
  lap("recip");
  std::vector<std::array<RoundRecord, 6>> ops(ns);
  std::vector<TT> in;
  std::vector<RoundRecord*> dst;
  // vel_x, vel_y, pressure (slots 0, 1, 2)
  for (size_t s = 0; s < ns; ++s) {
    const Triple& us = *u[s];
    in.insert(in.end(), {hadamard(us[1], inv[s]), hadamard(us[2], inv[s]), hadamard(us[0], us[0])});
    dst.insert(dst.end(), {&ops[s][0], &ops[s][1], &ops[s][2]});
  }
  auto b1 = round_batch_into(in, std::vector<double>(in.size(), eps), dst);
  lap("b1");
  // X: u1*vel_x (slot 3; + pressure at slot 4), f2 = u1*vel_y (slot 5)
  // Y: f1 = u2*vel_x (slot 3), u2*vel_y (slot 4; + pressure at slot 5)
  in.clear();
  dst.clear();
  for (size_t s = 0; s < ns; ++s) {
    const TT& mom = dir[s] == Axis::X ? (*u[s])[1] : (*u[s])[2];
    in.insert(in.end(), {hadamard(mom, b1[3 * s]), hadamard(mom, b1[3 * s + 1])});
    if (dir[s] == Axis::X)
      dst.insert(dst.end(), {&ops[s][3], &ops[s][5]});
    else
      dst.insert(dst.end(), {&ops[s][3], &ops[s][4]});
  }
  auto b2 = round_batch_into(in, std::vector<double>(in.size(), eps), dst);
  lap("b2");
  in.clear();
  dst.clear();
  for (size_t s = 0; s < ns; ++s) {
    const TT pressure = scale(b1[3 * s + 2], 0.5 * p.g);
    if (dir[s] == Axis::X) {
      in.push_back(add(b2[2 * s], pressure));
      dst.push_back(&ops[s][4]);
    } else {
      in.push_back(add(b2[2 * s + 1], pressure));
      dst.push_back(&ops[s][5]);
    }
  }
  auto b3 = round_batch_into(in, std::vector<double>(in.size(), eps), dst);
  lap("b3");
  std::vector<Triple> out(ns);
  for (size_t s = 0; s < ns; ++s) {
    if (dir[s] == Axis::X)
      out[s] = {(*u[s])[1], b3[s], b2[2 * s + 1]};
    else
      out[s] = {(*u[s])[2], b2[2 * s], b3[s]};
    recs[s].insert(recs[s].end(), ops[s].begin(), ops[s].end());
  }
  return out;
}

/// One axis' operands of the LLF flux.
struct LlfIn {
  const Triple* um;
  const Triple* up;
  const Triple* fm;
  const Triple* fp;
  const std::variant<double, TT>* lambda;
};

/// llf_flux (swe.hpp:235-265) of several axes at once, rounded (eps >= 0): per component
/// the reference order is central, jump, [lambda * jump,] out; the batches are
/// {central, jump} x 3 x axes, [{lambda * jump} x 3 x axes,] {out} x 3 x axes, and recs[a]
/// receives axis a's records in the reference's order.
/// lambda_pending: the lambda fields (TTs) are still being computed; before_lambda() is
/// called once the first batch (central averages and jumps, which do not need them) has
/// been issued, and must leave every *ax[a].lambda set.
std::vector<Triple> llf_flux_multi(const std::vector<LlfIn>& ax, double eps,
                                   std::vector<std::vector<RoundRecord>>& recs, bool lambda_pending = false,
                                   const std::function<void()>& before_lambda = {}) {
  const size_t na = ax.size();
  recs.assign(na, {});
  std::vector<int> per(na);
  for (size_t a = 0; a < na; ++a) {
    per[a] = (lambda_pending || std::holds_alternative<TT>(*ax[a].lambda)) ? 4 : 3;
    recs[a].resize(size_t(3 * per[a]));
  }
  std::vector<TT> in;
  std::vector<RoundRecord*> dst;
  for (size_t a = 0; a < na; ++a)
    for (int c = 0; c < 3; ++c) {
      in.push_back(add(scale((*ax[a].fm)[size_t(c)], 0.5), scale((*ax[a].fp)[size_t(c)], 0.5)));
      in.push_back(add(scale((*ax[a].up)[size_t(c)], 1.0), scale((*ax[a].um)[size_t(c)], -1.0)));
      dst.push_back(&recs[a][size_t(per[a] * c)]);
      dst.push_back(&recs[a][size_t(per[a] * c + 1)]);
    }
  auto b1 = round_batch_into(in, std::vector<double>(in.size(), eps), dst);
  if (before_lambda) before_lambda();
  std::vector<TT> dis(3 * na);
  in.clear();
  dst.clear();
  std::vector<size_t> field_idx;
  for (size_t a = 0; a < na; ++a)
    for (int c = 0; c < 3; ++c) {
      const TT& jump = b1[6 * a + size_t(2 * c + 1)];
      if (per[a] == 4) {
        in.push_back(hadamard(std::get<TT>(*ax[a].lambda), jump));
        dst.push_back(&recs[a][size_t(per[a] * c + 2)]);
        field_idx.push_back(3 * a + size_t(c));
      } else {
        dis[3 * a + size_t(c)] = scale(jump, -0.5 * std::get<double>(*ax[a].lambda));
      }
    }
  if (!in.empty()) {
    auto b2 = round_batch_into(in, std::vector<double>(in.size(), eps), dst);
    for (size_t q = 0; q < field_idx.size(); ++q) dis[field_idx[q]] = scale(b2[q], -0.5);
  }
  in.clear();
  dst.clear();
  for (size_t a = 0; a < na; ++a)
    for (int c = 0; c < 3; ++c) {
      in.push_back(add(scale(b1[6 * a + size_t(2 * c)], 1.0), dis[3 * a + size_t(c)]));
      dst.push_back(&recs[a][size_t(per[a] * c + per[a] - 1)]);
    }
  auto b3 = round_batch_into(in, std::vector<double>(in.size(), eps), dst);
  std::vector<Triple> out(na);
  for (size_t a = 0; a < na; ++a) out[a] = {b3[3 * a], b3[3 * a + 1], b3[3 * a + 2]};
  return out;
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

namespace {

/// Runs job(i, k_i) for i < njobs concurrently, each on its own child context k_i (same
/// device and pool, own stream) from its own host thread, all ordered after the parent
/// stream's queued work; the parent stream then waits for every child. Exceptions are
/// returned per job; launch and cross counters are folded into the parent.
/// Independent jobs on child contexts (own streams, ordered after everything already on
/// the parent stream), one short-lived host thread each. fork_start returns at once;
/// fork_finish joins the threads, orders the parent stream after every child's work and
/// adds the children's counters. fork_join = both.
struct ForkHandle {
  Context* parent = nullptr;
  cudaEvent_t start = nullptr;
  std::vector<Context*> kids;
  std::vector<std::thread> threads;
  std::function<void(size_t, Context*)> job;
};

std::unique_ptr<ForkHandle> fork_start(Context* parent, size_t njobs, std::function<void(size_t, Context*)> job,
                                       std::vector<std::exception_ptr>& errs) {
  auto h = std::make_unique<ForkHandle>();
  h->parent = parent;
  h->job = std::move(job);
  errs.assign(njobs, nullptr);
  if (njobs == 0) return h;
  TTSW_CUDA(cudaEventCreateWithFlags(&h->start, cudaEventDisableTiming));
  TTSW_CUDA(cudaEventRecord(h->start, parent->stream));
  h->kids.resize(njobs);
  for (size_t i = 0; i < njobs; ++i) {
    h->kids[i] = parent->child(i);
    h->kids[i]->launches = 0;
    h->kids[i]->cross_calls = 0;
    h->kids[i]->trace = nullptr;
    h->kids[i]->ctrace = nullptr;
  }
  h->threads.reserve(njobs);
  ForkHandle* hp = h.get();
  std::vector<std::exception_ptr>* ep = &errs;
  for (size_t i = 0; i < njobs; ++i)
    h->threads.emplace_back([hp, ep, i] {
      try {
        TTSW_CUDA(cudaSetDevice(hp->parent->device));
        TTSW_CUDA(cudaStreamWaitEvent(hp->kids[i]->stream, hp->start, 0));
        hp->job(i, hp->kids[i]);
      } catch (...) {
        (*ep)[i] = std::current_exception();
      }
    });
  return h;
}

void fork_finish(ForkHandle& h) {
  for (auto& t : h.threads) t.join();
  h.threads.clear();
  for (Context* k : h.kids) {
    cudaEvent_t done;
    TTSW_CUDA(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
    TTSW_CUDA(cudaEventRecord(done, k->stream));
    TTSW_CUDA(cudaStreamWaitEvent(h.parent->stream, done, 0));
    TTSW_CUDA(cudaEventDestroy(done));
    h.parent->launches += k->launches;
    h.parent->cross_calls += k->cross_calls;
    k->ctrace = nullptr;
  }
  h.kids.clear();
  if (h.start) TTSW_CUDA(cudaEventDestroy(h.start));
  h.start = nullptr;
}

void fork_join(Context* parent, size_t njobs, const std::function<void(size_t, Context*)>& job,
               std::vector<std::exception_ptr>& errs) {
  auto h = fork_start(parent, njobs, job, errs);
  fork_finish(*h);
}

void rethrow_first(const std::vector<std::exception_ptr>& errs) {
  for (const auto& e : errs)
    if (e) std::rethrow_exception(e);
}

}  // namespace

/// rhs<TTRep> (swe.hpp:362-423) with periodic fill_ghost. Faces of both sides are
/// reconstructed once per axis (the reference builds them twice, :378-381; the cross RNG
/// is re-seeded per call so reuse is bit-identical).
///
/// Execution order differs from the reference's, results and records do not: all crosses
/// (WENO faces and the LLF lambda of both axes) run first, then the physical fluxes of
/// all four face sides as one lock-step batch, then the LLF fluxes of both axes, then the
/// maps. Every operation's inputs are the reference's, crosses re-seed per call, and the
/// rounding and cross records are re-emitted in the reference order (per axis: face
/// crosses, physical-flux roundings, lambda cross, LLF roundings; then the Y-axis sums)
/// with each rounding's crosses-before count taken in that order.
Triple Solver::rhs(const Triple& u, double t_stage) {
  HostRegion hr_rhs(ctx, "rhs");
  const double flux_eps = opt.model == Model::Nonlinear ? eps.global : kNoRound;
  const double dx = 1.0 / double(n), dy = 1.0 / double(n);
  Context* cx = ctx;
  std::vector<RoundRecord>* trace_out = cx->trace;
  std::vector<CrossRecord>* ctrace_out = cx->ctrace;
  const long cross_base = cx->cross_calls;
  std::vector<CrossRecord> cr_faces[2], cr_lambda[2];
  std::vector<RoundRecord> rr_tail;
  std::vector<std::vector<RoundRecord>> rr_phys, rr_llf;
  auto restore = [&] {
    cx->trace = trace_out;
    cx->ctrace = ctrace_out;
  };
  Triple ghosted;
  if (fill_ghost)
    ghosted = fill_ghost(u, t_stage);
  else
    for (int c = 0; c < 3; ++c) ghosted[size_t(c)] = periodic_ghost(u[size_t(c)]);
  const Axis axes[2] = {Axis::X, Axis::Y};
  Triple um[2], up[2];
  std::variant<double, TT> lambda[2];
  Triple fhat[2];
  Triple flux_div;
  static const bool prof_on = std::getenv("TTSW_PROFILE_RHS") != nullptr;
  auto tprev = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (!prof_on) return;
    cx->sync();
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "rhs %-10s %8.2f ms\n", what, std::chrono::duration<double, std::milli>(now - tprev).count());
    tprev = now;
  };
  std::unique_ptr<ForkHandle> lam_fork;  // lambda crosses in flight during the physical fluxes
  std::vector<std::exception_ptr> lam_errs;
  TT lam[2];
  try {
    lap("ghost");
    // crosses: faces (WENO) and lambda of both axes, independent chains run concurrently
    ReconContext rc;
    rc.scheme = opt.scheme;
    rc.eps_tt = eps.global < 0 ? 1e-14 : eps.global;
    rc.cross = opt.cross;
    rc.dx = dx;
    rc.dy = dy;
    if (opt.scheme == Scheme::Weno5) {
      // 12 chains (axis, component, side), each step 1 then step 2 (reconstruction.hpp:
      // 531-604); reference order: axis, component, minus then plus
      struct Chain {
        int a, c;
        Side side;
        std::vector<TT> ops1;
        TT out;
        std::vector<CrossRecord> cr;
      };
      std::vector<Chain> chains;
      for (int a = 0; a < 2; ++a)
        for (int c = 0; c < 3; ++c)
          for (Side side : {Side::Minus, Side::Plus}) {
            Chain ch{a, c, side, {}, nullptr, {}};
            for (const TT& o : weno_step1_ops(ghosted[size_t(c)], axes[a], side)) ch.ops1.push_back(materialize(o));
            chains.push_back(std::move(ch));
          }
      const Index nx = ghosted[0]->m - 2 * kGhost, ny = ghosted[0]->n - 2 * kGhost;
      std::vector<std::exception_ptr> errs;
      fork_join(cx, chains.size(), [&](size_t i, Context* k) {
        Chain& ch = chains[i];
        k->ctrace = ctrace_out ? &ch.cr : nullptr;
        ch.out = weno_side(k, ch.ops1, nx, ny, axes[ch.a], ch.side, rc);
      }, errs);
      rethrow_first(errs);
      for (auto& ch : chains) {
        const TT f = adopt(cx, ch.out);
        (ch.side == Side::Minus ? um : up)[ch.a][size_t(ch.c)] = f;
        cr_faces[ch.a].insert(cr_faces[ch.a].end(), ch.cr.begin(), ch.cr.end());
        ch.ops1.clear();
      }
    } else {
      cx->trace = nullptr;
      for (int a = 0; a < 2; ++a)
        for (int c = 0; c < 3; ++c) {
          FacePair f = reconstruct_faces(ghosted[size_t(c)], axes[a], rc);
          um[a][size_t(c)] = f.minus;
          up[a][size_t(c)] = f.plus;
        }
      cx->trace = trace_out;
    }
    if (opt.model == Model::Nonlinear) {
      for (int a = 0; a < 2; ++a)
        for (int c = 0; c < 3; ++c) {
          um[a][size_t(c)] = materialize(um[a][size_t(c)]);
          up[a][size_t(c)] = materialize(up[a][size_t(c)]);
        }
      // the two lambda crosses need only the faces: they run on child contexts while the
      // physical fluxes of the four face sides are computed on this one (joined below,
      // before the LLF fluxes that use them)
      lam_fork = fork_start(cx, 2, [&](size_t a, Context* k) {
        k->ctrace = ctrace_out ? &cr_lambda[a] : nullptr;
        const int mom = axes[a] == Axis::X ? 1 : 2;
        std::vector<TT> ops{um[a][0], um[a][size_t(mom)], up[a][0], up[a][size_t(mom)]};
        CrossConfig cfg = opt.cross;
        cfg.eps = std::max(eps.global, opt.lambda_eps_floor);
        lam[a] = cross_elementwise_on(k, FN_LLF_LAMBDA, opt.params.g, ops, um[a][0], cfg);
      }, lam_errs);
    } else {
      for (int a = 0; a < 2; ++a) lambda[a] = face_wave_speed(um[a], up[a], axes[a], opt, eps.global);
    }
    cx->ctrace = ctrace_out;
    lap("crosses");
    // physical fluxes of the four face sides
    Triple fm[2], fp[2];
    if (opt.model == Model::Nonlinear && flux_eps > 0) {
      auto fl = physical_flux_multi({&um[0], &up[0], &um[1], &up[1]}, {Axis::X, Axis::X, Axis::Y, Axis::Y},
                                    opt.params, flux_eps, rr_phys);
      fm[0] = fl[0];
      fp[0] = fl[1];
      fm[1] = fl[2];
      fp[1] = fl[3];
    } else {
      cx->trace = nullptr;  // no roundings (linear) / unbatched fallback records discarded below
      for (int a = 0; a < 2; ++a) {
        fm[a] = physical_flux(um[a], axes[a], opt.model, opt.params, flux_eps);
        fp[a] = physical_flux(up[a], axes[a], opt.model, opt.params, flux_eps);
      }
      cx->trace = trace_out;
      rr_phys.assign(4, {});
    }
    // joined once the LLF's first batch (central averages and jumps) has been issued
    auto join_lambda = [&] {
      if (!lam_fork) return;
      fork_finish(*lam_fork);
      lam_fork.reset();
      rethrow_first(lam_errs);
      for (int a = 0; a < 2; ++a) lambda[a] = adopt(cx, lam[a]);
      cx->ctrace = ctrace_out;
    };
    lap("physflux");
    // LLF fluxes of both axes
    if (flux_eps >= 0) {
      fhat[0] = Triple{};
      std::vector<LlfIn> in{{&um[0], &up[0], &fm[0], &fp[0], &lambda[0]}, {&um[1], &up[1], &fm[1], &fp[1], &lambda[1]}};
      auto fl = llf_flux_multi(in, flux_eps, rr_llf, bool(lam_fork), join_lambda);
      fhat[0] = fl[0];
      fhat[1] = fl[1];
    } else {
      join_lambda();
      for (int a = 0; a < 2; ++a)
        fhat[a] = std::holds_alternative<double>(lambda[a])
                      ? llf_flux(um[a], up[a], fm[a], fp[a], std::get<double>(lambda[a]), flux_eps)
                      : llf_flux(um[a], up[a], fm[a], fp[a], std::get<TT>(lambda[a]), flux_eps);
      rr_llf.assign(2, {});
    }
    lap("llf");
    // quadrature sum across the transverse axis, difference along the axis
    for (int a = 0; a < 2; ++a) {
      const Axis axis = axes[a];
      const Index n_axis = n, n_trans = n;
      const Axis trans = axis == Axis::X ? Axis::Y : Axis::X;
      const BandMap w = make_band_map(3, opt.scheme, Side::Minus, n_trans, 0, 0);
      const BandMap d = make_band_map(4, opt.scheme, Side::Minus, n_axis, 0, 0);
      const double inv = axis == Axis::X ? 1.0 / dx : 1.0 / dy;
      Triple difference;
      for (int c = 0; c < 3; ++c) {
        TT integrated = apply_core_map(fhat[a][size_t(c)], trans, w);
        difference[size_t(c)] = apply_core_map(integrated, axis, d);
      }
      if (axis == Axis::X) {
        for (int c = 0; c < 3; ++c) flux_div[size_t(c)] = Rep::scaled(difference[size_t(c)], inv);
      } else {
        // the three component sums are independent roundings: one batch, records in order c
        cx->trace = trace_out ? &rr_tail : nullptr;
        flux_div = axpy3(1.0, flux_div, inv, difference, {flux_eps, flux_eps, flux_eps});
        cx->trace = trace_out;
      }
    }
    lap("maps+sums");
  } catch (...) {
    if (lam_fork) fork_finish(*lam_fork);  // the lambda crosses never outlive this frame
    restore();
    throw;
  }
  restore();
  // records in the reference's order, crosses-before counted in that order
  long crosses = cross_base;
  auto emit_r = [&](const std::vector<RoundRecord>& rs) {
    if (!trace_out) return;
    for (RoundRecord r : rs) {
      r.crosses = crosses;
      trace_out->push_back(r);
    }
  };
  auto emit_c = [&](const std::vector<CrossRecord>& cs) {
    if (ctrace_out) ctrace_out->insert(ctrace_out->end(), cs.begin(), cs.end());
    crosses += long(cs.size());
  };
  for (int a = 0; a < 2; ++a) {
    emit_c(cr_faces[a]);
    emit_r(rr_phys[size_t(2 * a)]);
    emit_r(rr_phys[size_t(2 * a + 1)]);
    emit_c(cr_lambda[a]);
    emit_r(rr_llf[size_t(a)]);
  }
  emit_r(rr_tail);
  auto source = coriolis_source(u, opt.params);
  if (extra_source) {  // swe.hpp:412-416
    const Triple extra = extra_source(t_stage);
    source = axpy3(1.0, source, 1.0, extra, {flux_eps, flux_eps, flux_eps});
  }
  Triple out = axpy3(-1.0, flux_div, 1.0, source, eps.var);
  lap("final axpy");
  return out;
}

/// ssprk3 (swe.hpp:428-454); tolerances frozen for the step.
/// eps_global / eps_for_variable (swe.hpp:143-154).
EpsSchedule compute_eps_schedule(const Triple& u, const EpsPolicy& p, double dx) {
  const std::vector<double> norms = norm_fro_batch({u[0], u[1], u[2]});
  const double scale = p.c_eps * std::sqrt(p.volume) * std::pow(dx, p.order - 0.5);
  EpsSchedule eps;
  double max_norm = 0.0;
  for (int c = 0; c < 3; ++c) {
    const double q = norms[size_t(c)];
    eps.var[size_t(c)] = q <= 0.0 ? p.clip : std::min(p.clip, scale / q);
    max_norm = std::max(max_norm, q);
  }
  eps.global = max_norm <= 0.0 ? p.clip : scale / max_norm;
  return eps;
}

void Solver::step() {
  if (!(dt > 0)) throw InputError("ssprk3: dt must be positive");
  HostRegion hr_step(ctx, "ssprk3_step");
  const auto t_step = std::chrono::steady_clock::now();
  const double sync0 = ctx->sync_ms;
  const long nsync0 = ctx->sync_count, launch0 = ctx->launches;
  if (use_policy) eps = compute_eps_schedule(state, policy, 1.0 / double(n));
  // the context points at this solver's trace vectors only while the step runs (also
  // when it throws): later standalone calls on the context must not append to them
  struct TraceScope {
    Context* c;
    ~TraceScope() {
      c->trace = nullptr;
      c->ctrace = nullptr;
      c->hint_active = false;
    }
  } trace_scope{ctx};
  // the step's large roundings are issued in the same order every step: their last output
  // ranks size the sketches of this step (runtime.cu: round_caqr_group)
  ctx->hint_pos = 0;
  ctx->hint_active = true;
  ctx->trace = tracing ? &trace : nullptr;
  ctx->ctrace = tracing ? &ctrace : nullptr;
  auto euler = [&](const Triple& w, double ts) {
    Triple k = rhs(w, ts);
    return axpy3(1.0, w, dt, k, eps.var);
  };
  const Triple& u = state;
  // stage times t, t + dt, t + dt/2 (swe.hpp:441-448)
  Triple u1 = euler(u, t);
  Triple f1 = euler(u1, t + dt);
  Triple u2 = axpy3(0.75, u, 0.25, f1, eps.var);
  Triple f2 = euler(u2, t + 0.5 * dt);
  state = axpy3(1.0 / 3.0, u, 2.0 / 3.0, f2, eps.var);
  t += dt;
  if (ctx->prof_host) {
    for (auto& r : ctx->host_regions)
      std::fprintf(stderr, "host %-18s calls %6.0f  wall %8.2f ms  of which sync %8.2f ms\n", r.first.c_str(),
                   r.second[2], r.second[0], r.second[1]);
    ctx->host_regions.clear();
  }
  if (ctx->count_sync) {
    ctx->sync();
    const double wall = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_step).count();
    std::fprintf(stderr, "step wall %.1f ms, host blocked in %ld syncs %.1f ms, host busy %.1f ms, launches %ld\n",
                 wall, ctx->sync_count - nsync0, ctx->sync_ms - sync0, wall - (ctx->sync_ms - sync0),
                 ctx->launches - launch0);
  }
}

}  // namespace ttsw
