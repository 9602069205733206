// TEST INFRASTRUCTURE ONLY — C ABI wrapper of the CPU oracle (see ttsw_oracle.h).
#include <cstring>
#include <memory>

#include "swe.hpp"
#include "ttsw_oracle.h"

using namespace ttor;

struct ttor_tt { TT v; };
struct ttor_rng { std::mt19937_64 gen; };
struct ttor_solver {
  Grid grid;
  SolverOptions opt;
  EpsSchedule eps;
  bool use_policy = false;  // harness.cpp:108-116: schedule recomputed per step
  EpsPolicy policy;
  double dt = 0;
  double t = 0;  // advanced by dt per step; stage times reach the hooks
  RhsHooks hooks;
  Triple state;
  std::vector<RoundRecord> trace;
  std::vector<CrossRecord> ctrace;
};

namespace {

thread_local std::string g_err;
thread_local double g_res = 0;
thread_local int g_it = 0;
thread_local long g_row = -1, g_col = -1;

template <class F>
int guard(F&& f) {
  try {
    f();
    return TTOR_OK;
  } catch (const DeadlineReached& e) {
    g_err = e.what(); return TTOR_DEADLINE;
  } catch (const ConvergenceError& e) {
    g_err = e.what(); g_res = e.residual; g_it = e.iterations; return TTOR_CONVERGENCE;
  } catch (const EvaluationError& e) {
    g_err = e.what(); g_row = e.row; g_col = e.col; return TTOR_EVALUATION;
  } catch (const DegeneracyError& e) {
    g_err = e.what(); return TTOR_DEGENERACY;
  } catch (const StateError& e) {
    g_err = e.what(); return TTOR_STATE;
  } catch (const ShapeError& e) {
    g_err = e.what(); return TTOR_SHAPE;
  } catch (const InputError& e) {
    g_err = e.what(); return TTOR_INPUT;
  } catch (const std::exception& e) {
    g_err = e.what(); return TTOR_INTERNAL;
  }
}

ttor_tt* wrap(TT v) { return new ttor_tt{std::move(v)}; }

CrossConfig to_cfg(const ttor_cross_cfg* c) {
  CrossConfig cfg;
  if (c) {
    cfg.eps = c->eps;
    cfg.max_rank = c->max_rank;
    cfg.max_sweeps = c->max_sweeps;
    cfg.rank_increment = c->rank_increment;
    cfg.validation_sample = c->validation_sample;
    cfg.seed = c->seed;
  }
  return cfg;
}

EntryFn make_fn(int fn, const double* p) {
  const double a = p ? p[0] : 0.0;
  switch (fn) {
    case 0: return [](std::span<const double> v) { return v[0]; };
    case 1: return [](std::span<const double> v) { return v[0] * v[1]; };
    case 2: return [](std::span<const double> v) {
        if (v[0] < 0) throw std::domain_error("sqrt of negative value");
        return std::sqrt(v[0]);
      };
    case 3: return [](std::span<const double> v) { return 2.0 * v[0] + 1.0; };
    case 4: return [](std::span<const double> v) { return v[0] * v[0]; };
    case 10: {
      const Tables* t = &recon_tables(Scheme::Weno5);
      return [t, a](std::span<const double> v) { return weno5_step1(v.data(), *t, a); };
    }
    case 11: {
      const Tables* t = &recon_tables(Scheme::Weno5);
      return [t, a](std::span<const double> v) {
        const double rev[5] = {v[4], v[3], v[2], v[1], v[0]};
        return weno5_step1(rev, *t, a);
      };
    }
    case 12: {
      const Tables* t = &recon_tables(Scheme::Weno5);
      return [t, a](std::span<const double> v) { return weno5_step2(v.data(), int(v[5] + 0.5), *t, a); };
    }
    case 20: return llf_lambda_fn(a);
    case 21: return wave_speed_fn(a);
    default: throw InputError("unknown functor kind");
  }
}

BandOp make_op(int op, int scheme, int side, Index n, Index a0, Index a1) {
  const Scheme s = Scheme(scheme);
  switch (op) {
    case 0: return periodic_pad_op(n);
    case 1: return step1_op(s, Side(side), n);
    case 2: return quadrature_point_op(s, n);
    case 3: return quadrature_sum_op(s, n);
    case 4: return difference_op(n);
    case 5: return row_slice_op(a0, a1, n + 2 * kGhost);
    case 6: return quadrature_slice_op(a0, n, quadrature_points(s), stencil_radius(s));
    default: throw InputError("unknown core map");
  }
}

}  // namespace

extern "C" {

int ttor_last_error(char* buf, long len, double* residual, int* iterations, long* row, long* col) {
  if (buf && len > 0) {
    std::strncpy(buf, g_err.c_str(), size_t(len - 1));
    buf[len - 1] = 0;
  }
  if (residual) *residual = g_res;
  if (iterations) *iterations = g_it;
  if (row) *row = g_row;
  if (col) *col = g_col;
  return 0;
}

ttor_tt* ttor_tt_new(long m, long n, long r, const double* cx, const double* cy) {
  ttor_tt* out = nullptr;
  int st = guard([&] {
    Mat x(m, r), y(r, n);
    std::memcpy(x.a.data(), cx, sizeof(double) * size_t(m * r));
    std::memcpy(y.a.data(), cy, sizeof(double) * size_t(r * n));
    out = wrap(TT(std::move(x), std::move(y)));
  });
  return st == TTOR_OK ? out : nullptr;
}
void ttor_tt_free(ttor_tt* x) { delete x; }
void ttor_tt_dims(const ttor_tt* x, long* m, long* n, long* r) {
  *m = x->v.rows(); *n = x->v.cols(); *r = x->v.rank();
}
void ttor_tt_get(const ttor_tt* x, double* cx, double* cy) {
  std::memcpy(cx, x->v.cx.a.data(), sizeof(double) * x->v.cx.a.size());
  std::memcpy(cy, x->v.cy.a.data(), sizeof(double) * x->v.cy.a.size());
}

int ttor_from_full(long m, long n, const double* a, double eps, ttor_tt** out) {
  return guard([&] {
    Mat A(m, n);
    std::memcpy(A.a.data(), a, sizeof(double) * size_t(m * n));
    *out = wrap(tt_from_full(A, eps));
  });
}
int ttor_to_full(const ttor_tt* x, double* out) {
  return guard([&] {
    Mat d = to_full(x->v);
    std::memcpy(out, d.a.data(), sizeof(double) * d.a.size());
  });
}
int ttor_round(const ttor_tt* x, double eps, ttor_tt** out, long* k_out, double* margin, double* kappa) {
  return guard([&] {
    std::vector<RoundRecord> tr;
    auto* prev = round_trace();
    round_trace() = &tr;
    try {
      *out = wrap(round(x->v, eps));
    } catch (...) {
      round_trace() = prev;
      throw;
    }
    round_trace() = prev;
    if (k_out) *k_out = tr.empty() ? -1 : tr.back().k_out;
    if (margin) *margin = tr.empty() ? 0 : tr.back().margin;
    if (kappa) *kappa = tr.empty() ? 0 : tr.back().kappa;
  });
}
int ttor_add(const ttor_tt* x, const ttor_tt* y, ttor_tt** out) {
  return guard([&] { *out = wrap(add(x->v, y->v)); });
}
int ttor_scale(const ttor_tt* x, double a, ttor_tt** out) {
  return guard([&] { *out = wrap(scale(x->v, a)); });
}
int ttor_axpy(double a, const ttor_tt* x, double b, const ttor_tt* y, double eps, ttor_tt** out) {
  return guard([&] { *out = wrap(Rep::axpy(a, x->v, b, y->v, eps)); });
}
int ttor_hadamard(const ttor_tt* x, const ttor_tt* y, ttor_tt** out) {
  return guard([&] { *out = wrap(hadamard(x->v, y->v)); });
}
int ttor_norm_fro(const ttor_tt* x, double* out) {
  return guard([&] { *out = norm_fro(x->v); });
}
int ttor_sum_entries(const ttor_tt* x, double* out) {
  return guard([&] { *out = sum_entries(x->v); });
}
int ttor_core_map(const ttor_tt* x, int axis, int op, int scheme, int side, long n, long a0, long a1,
                  ttor_tt** out) {
  return guard([&] { *out = wrap(apply_core_map(x->v, Axis(axis), make_op(op, scheme, side, n, a0, a1))); });
}
int ttor_core_map_dense(const ttor_tt* x, int axis, long rows, long cols, const double* m, ttor_tt** out) {
  return guard([&] {
    Mat M(rows, cols);
    std::memcpy(M.a.data(), m, sizeof(double) * size_t(rows * cols));
    *out = wrap(apply_core_map(x->v, Axis(axis), BandOp::from_dense(M)));
  });
}
int ttor_recip(const ttor_tt* x, double eps, int max_iterations, int* iterations, ttor_tt** out) {
  return guard([&] {
    ReciprocalStats st;
    try {
      *out = wrap(reciprocal_taylor(x->v, eps, max_iterations, &st));
    } catch (...) {
      if (iterations) *iterations = st.iterations;
      throw;
    }
    if (iterations) *iterations = st.iterations;
  });
}
int ttor_cross(int fn, const double* params, const ttor_tt* const* ops, int nops, const ttor_tt* guess,
               const ttor_cross_cfg* cfg, ttor_tt** out, ttor_cross_stats* stats) {
  return guard([&] {
    std::vector<TT> v;
    for (int k = 0; k < nops; ++k) v.push_back(ops[k]->v);
    EntryFn f = make_fn(fn, params);
    CrossResult r = cross_elementwise_stats(f, v, guess->v, to_cfg(cfg));
    if (stats) *stats = {r.evaluations, r.sweeps, r.residual};
    *out = wrap(std::move(r.tt));
  });
}
int ttor_maxvol(long n, long r, const double* m, long* rows_out) {
  return guard([&] {
    Mat M(n, r);
    std::memcpy(M.a.data(), m, sizeof(double) * size_t(n * r));
    auto rows = maxvol(M);
    for (size_t k = 0; k < rows.size(); ++k) rows_out[k] = rows[k];
  });
}
int ttor_svd_values(long m, long n, const double* a, double* s_out) {
  return guard([&] {
    Mat A(m, n);
    std::memcpy(A.a.data(), a, sizeof(double) * size_t(m * n));
    SVD s = svd_thin(A);
    for (size_t k = 0; k < s.s.size(); ++k) s_out[k] = s.s[k];
  });
}
int ttor_truncation_rank(const double* sv, long n, double eps, long* keep, double* margin) {
  return guard([&] {
    std::vector<double> s(sv, sv + n);
    *keep = truncation_rank(s, eps, margin);
  });
}
int ttor_tables(int scheme, double* o) {
  return guard([&] {
    const Tables& t = recon_tables(Scheme(scheme));
    std::memset(o, 0, sizeof(double) * 96);
    const int k = t.radius;
    for (int r = 0; r <= k; ++r)
      for (int l = 0; l <= k; ++l) o[r * 3 + l] = t.step1_c(r, l);
    for (size_t i = 0; i < t.step1_ideal.size(); ++i) o[9 + i] = t.step1_ideal[i];
    for (size_t i = 0; i < t.step1_row.size(); ++i) o[12 + i] = t.step1_row[i];
    for (int m = 0; m < t.quad.n; ++m) {
      for (int r = 0; r <= k; ++r)
        for (int l = 0; l <= k; ++l) o[17 + m * 9 + r * 3 + l] = t.c[size_t(m)](r, l);
      for (size_t i = 0; i < t.gamma[size_t(m)].size(); ++i) o[44 + m * 3 + i] = t.gamma[size_t(m)][i];
      for (size_t i = 0; i < t.point_row[size_t(m)].size(); ++i) o[53 + m * 5 + i] = t.point_row[size_t(m)][i];
    }
    for (size_t i = 0; i < t.gamma_plus.size(); ++i) o[68 + i] = t.gamma_plus[i];
    for (size_t i = 0; i < t.gamma_minus.size(); ++i) o[71 + i] = t.gamma_minus[i];
    for (size_t i = 0; i < t.weno_d.size(); ++i) o[74 + i] = t.weno_d[i];
    for (int i = 0; i < 3; ++i) { o[77 + i] = t.quad.offset[size_t(i)]; o[80 + i] = t.quad.weight[size_t(i)]; }
    o[83] = t.radius;
    o[84] = t.quad.n;
    o[85] = t.sigma_plus;
    o[86] = t.sigma_minus;
  });
}
int ttor_weno_step1(const double* v5, double eps, double* out) {
  return guard([&] { *out = weno5_step1(v5, recon_tables(Scheme::Weno5), eps); });
}
int ttor_weno_step2(const double* v5, int m, double eps, double* out) {
  return guard([&] {
    if (m < 0 || m > 2) throw InputError("step2: invalid quadrature index");
    *out = weno5_step2(v5, m, recon_tables(Scheme::Weno5), eps);
  });
}
int ttor_smoothness(const double* v5, double* b) {
  return guard([&] {
    auto r = smoothness(v5);
    for (int i = 0; i < 3; ++i) b[i] = r[size_t(i)];
  });
}
int ttor_weno_weights(const double* beta, const double* ideal, double eps, double* out) {
  return guard([&] {
    auto w = weno_weights({beta[0], beta[1], beta[2]}, {ideal[0], ideal[1], ideal[2]}, eps);
    for (int i = 0; i < 3; ++i) out[i] = w[size_t(i)];
  });
}
int ttor_periodic_ghost(const ttor_tt* x, ttor_tt** out) {
  return guard([&] { *out = wrap(periodic_ghost(x->v)); });
}
int ttor_ghosted(const ttor_tt* x, int bc_x, int bc_y, const double* strip_x, const double* strip_y, double eps_tt,
                 ttor_tt** out) {
  return guard([&] {
    const Index nx = x->v.rows(), ny = x->v.cols();
    Mat sx, sy;
    if (bc_x) {
      sx = Mat(2 * kGhost, ny + 2 * kGhost);
      std::copy(strip_x, strip_x + sx.a.size(), sx.a.begin());
    }
    if (bc_y) {
      sy = Mat(nx + 2 * kGhost, 2 * kGhost);
      std::copy(strip_y, strip_y + sy.a.size(), sy.a.begin());
    }
    *out = wrap(ghosted(x->v, bc_x != 0, bc_y != 0, bc_x ? &sx : nullptr, bc_y ? &sy : nullptr, eps_tt));
  });
}
int ttor_reconstruct_faces(const ttor_tt* g, int axis, int scheme, double eps_tt, const ttor_cross_cfg* cfg,
                           double dx, double dy, ttor_tt** minus, ttor_tt** plus) {
  return guard([&] {
    ReconContext ctx;
    ctx.scheme = Scheme(scheme);
    ctx.eps_tt = eps_tt;
    ctx.cross = to_cfg(cfg);
    ctx.dx = dx;
    ctx.dy = dy;
    FacePair f = reconstruct_faces(g->v, Axis(axis), ctx);
    *minus = wrap(std::move(f.minus));
    *plus = wrap(std::move(f.plus));
  });
}
int ttor_physical_flux(ttor_tt* const* u3, int axis, int model, double g, double f, double H, double eps,
                       ttor_tt** out3) {
  return guard([&] {
    Triple u{u3[0]->v, u3[1]->v, u3[2]->v};
    PhysParams p{g, f, H};
    Triple r = physical_flux(u, Axis(axis), Model(model), p, eps);
    for (int c = 0; c < 3; ++c) out3[c] = wrap(std::move(r[size_t(c)]));
  });
}

ttor_solver* ttor_solver_new(const ttor_solver_desc* d) {
  auto* s = new ttor_solver;
  s->grid.nx = s->grid.ny = d->n;
  s->opt.scheme = Scheme(d->scheme);
  s->opt.model = Model(d->model);
  s->opt.params = {d->g, d->f, d->H};
  s->opt.cross = to_cfg(&d->cross);
  s->opt.lambda_eps_floor = d->lambda_eps_floor;
  s->eps.var = {d->tol, d->tol, d->tol};
  s->eps.global = d->tol;
  s->dt = d->dt;
  cross_calls() = 0;
  for (int c = 0; c < 3; ++c) s->state[size_t(c)] = TT::zero(d->n, d->n);
  return s;
}
void ttor_solver_free(ttor_solver* s) { delete s; }
int ttor_solver_set_state(ttor_solver* s, int c, const ttor_tt* x) {
  return guard([&] { s->state[size_t(c)] = x->v; });
}
ttor_tt* ttor_solver_get_state(ttor_solver* s, int c) { return wrap(s->state[size_t(c)]); }
int ttor_solver_set_time(ttor_solver* s, double t) {
  return guard([&] { s->t = t; });
}
double ttor_solver_time(const ttor_solver* s) { return s->t; }
int ttor_solver_set_hooks(ttor_solver* s, ttor_fill_ghost_fn ghost, ttor_extra_source_fn source, void* user) {
  return guard([&] {
    s->hooks = RhsHooks{};
    auto take = [](ttor_tt** h, const char* what) {
      Triple out;
      for (int c = 0; c < 3; ++c) {
        if (!h[c]) throw StateError(std::string(what) + ": hook returned no field");
        out[size_t(c)] = h[c]->v;
        delete h[c];
      }
      return out;
    };
    if (ghost)
      s->hooks.fill_ghost = [ghost, user, take](const Triple& u, double t) {
        ttor_tt in[3] = {{u[0]}, {u[1]}, {u[2]}};
        const ttor_tt* q3[3] = {&in[0], &in[1], &in[2]};
        ttor_tt* out[3] = {nullptr, nullptr, nullptr};
        if (ghost(user, q3, t, out) != 0) throw StateError("fill_ghost hook failed");
        return take(out, "fill_ghost");
      };
    if (source)
      s->hooks.extra_source = [source, user, take](double t) {
        ttor_tt* out[3] = {nullptr, nullptr, nullptr};
        if (source(user, t, out) != 0) throw StateError("extra_source hook failed");
        return take(out, "extra_source");
      };
  });
}
int ttor_solver_rhs(ttor_solver* s, ttor_tt** out3) {
  return guard([&] {
    auto* prev = round_trace();
    round_trace() = &s->trace;
    try {
      Triple r = rhs(s->state, s->grid, s->opt, s->eps, s->t, &s->hooks);
      for (int c = 0; c < 3; ++c) out3[c] = wrap(std::move(r[size_t(c)]));
    } catch (...) {
      round_trace() = prev;
      throw;
    }
    round_trace() = prev;
  });
}
int ttor_solver_step(ttor_solver* s, long nsteps) {
  return guard([&] {
    auto* prev = round_trace();
    round_trace() = &s->trace;
    cross_trace() = &s->ctrace;
    long k = 0;
    try {
      for (; k < nsteps; ++k) {
        if (s->use_policy) s->eps = compute_eps_schedule(s->state, s->policy, s->grid.dx());
        s->state = ssprk3(s->state, s->dt, s->grid, s->opt, s->eps, s->t, &s->hooks);
        s->t += s->dt;
      }
    } catch (const DeadlineReached&) {
      round_trace() = prev;
      cross_trace() = nullptr;
      throw;
    } catch (const std::exception& e) {
      round_trace() = prev;
      cross_trace() = nullptr;
      std::ostringstream os;
      os << "run: failed at step " << k << ": " << e.what();
      throw StateError(os.str());
    }
    round_trace() = prev;
    cross_trace() = nullptr;
  });
}
void ttor_set_sample_deadline(double seconds) { sample_deadline() = seconds > 0 ? wall_seconds() + seconds : 0.0; }
int ttor_solver_set_eps_policy(ttor_solver* s, double c_eps, int order, double volume, double clip) {
  return guard([&] {
    if (!(clip > 0) || order < 1 || !(volume > 0)) throw InputError("eps policy: invalid parameters");
    s->use_policy = true;
    s->policy = EpsPolicy{c_eps, order, volume, clip};
  });
}
int ttor_solver_eps(const ttor_solver* s, double* out4) {
  for (int c = 0; c < 3; ++c) out4[c] = s->eps.var[size_t(c)];
  out4[3] = s->eps.global;
  return TTOR_OK;
}
long ttor_solver_cross_trace_len(const ttor_solver* s) { return long(s->ctrace.size()); }
void ttor_solver_cross_trace(ttor_solver* s, long* ints, double* residuals, int clear) {
  for (size_t i = 0; i < s->ctrace.size(); ++i) {
    ints[3 * i] = s->ctrace[i].rank;
    ints[3 * i + 1] = s->ctrace[i].sweeps;
    ints[3 * i + 2] = s->ctrace[i].pivot_hash;
    residuals[i] = s->ctrace[i].residual;
  }
  if (clear) s->ctrace.clear();
}
long ttor_solver_trace_len(const ttor_solver* s) { return long(s->trace.size()); }
void ttor_solver_trace(const ttor_solver* s, long* ints, double* margins, double* kappas) {
  for (size_t i = 0; i < s->trace.size(); ++i) {
    const auto& r = s->trace[i];
    ints[6 * i + 0] = long(i);
    ints[6 * i + 1] = r.m;
    ints[6 * i + 2] = r.n;
    ints[6 * i + 3] = r.r_in;
    ints[6 * i + 4] = r.k_out;
    ints[6 * i + 5] = r.crosses;
    margins[i] = r.margin;
    if (kappas) kappas[i] = r.kappa;
  }
}
void ttor_solver_trace_clear(ttor_solver* s) { s->trace.clear(); }

ttor_rng* ttor_rng_new(unsigned long long seed) { return new ttor_rng{std::mt19937_64(seed)}; }
void ttor_rng_free(ttor_rng* g) { delete g; }
void ttor_rng_normal(ttor_rng* g, long count, double* out) {
  // One fresh distribution per call, like tests/support.hpp:10-16 random_matrix.
  std::normal_distribution<double> dist(0.0, 1.0);
  for (long i = 0; i < count; ++i) out[i] = dist(g->gen);
}
void ttor_rng_uniform_int(ttor_rng* g, long lo, long hi, long count, long* out) {
  std::uniform_int_distribution<long> d(lo, hi);
  for (long i = 0; i < count; ++i) out[i] = d(g->gen);
}
void ttor_rng_uniform_real(ttor_rng* g, double lo, double hi, long count, double* out) {
  std::uniform_real_distribution<double> d(lo, hi);
  for (long i = 0; i < count; ++i) out[i] = d(g->gen);
}
unsigned long long ttor_rng_raw(ttor_rng* g) { return g->gen(); }

}  // extern "C"
