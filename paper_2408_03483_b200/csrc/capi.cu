// C ABI (include/ttsw_capi.h) over the device runtime. Exceptions of the reference's
// types (types.hpp:28-56) become status codes; the message and payload are kept per
// context for ttsw_last_error.
#include <cmath>
#include <cstring>
#include <chrono>
#include <functional>
#include <thread>
#include <sstream>

#include "../../include/ttsw_capi.h"
#include "kernels.cuh"

using namespace ttsw;

struct ttsw_ctx {
  std::shared_ptr<Context> owner;  // device buffers hold further references
  Context* c = nullptr;
  std::string err;
  ttsw_err_info info{0, 0, -1, -1};
};
struct ttsw_tt {
  TT v;
};
struct ttsw_solver {
  ttsw_ctx* ctx;
  Solver s;
  std::shared_ptr<Context> owner;
};
// C5 ensembles: independent members, each a Solver on the context of the host worker
// thread that owns it (one stream per worker, so the members' kernels overlap).
struct EnsembleMember {
  Solver s;
  long steps = 0;
  std::array<long, 3> max_rank{0, 0, 0};
  double ms = 0;
};
struct ttsw_ensemble {
  int device = 0;
  std::vector<std::shared_ptr<Context>> workers;
  std::vector<std::unique_ptr<EnsembleMember>> members;
  std::string err;
  int status = TTSW_OK;
  Context* ctx_of(size_t m) const { return workers[m % workers.size()].get(); }
};
struct ttsw_dense {
  ttsw_ctx* ctx;
  std::shared_ptr<Context> owner;
  std::unique_ptr<DenseSolver> s;
};

namespace {

template <class F>
int guard(ttsw_ctx* ctx, F&& f) {
  auto set = [&](const std::string& m) {
    if (ctx) ctx->err = m;
  };
  try {
    if (ctx && ctx->c) TTSW_CUDA(cudaSetDevice(ctx->c->device));  // a context may not own the current device
    f();
    return TTSW_OK;
  } catch (const ConvergenceError& e) {
    set(e.what());
    if (ctx) {
      ctx->info.residual = e.residual;
      ctx->info.iterations = e.iterations;
    }
    return TTSW_CONVERGENCE;
  } catch (const EvaluationError& e) {
    set(e.what());
    if (ctx) {
      ctx->info.row = e.row;
      ctx->info.col = e.col;
    }
    return TTSW_EVALUATION;
  } catch (const DegeneracyError& e) {
    set(e.what());
    return TTSW_DEGENERACY;
  } catch (const StateError& e) {
    set(e.what());
    return TTSW_STATE;
  } catch (const ShapeError& e) {
    set(e.what());
    return TTSW_SHAPE;
  } catch (const InputError& e) {
    set(e.what());
    return TTSW_INPUT;
  } catch (const CudaError& e) {
    set(e.what());
    return TTSW_CUDA;
  } catch (const std::exception& e) {
    set(e.what());
    return TTSW_INTERNAL;
  }
}

ttsw_tt* wrap(TT v) { return new ttsw_tt{std::move(v)}; }

CrossConfig to_cfg(const ttsw_cross_cfg* c) {
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

}  // namespace

extern "C" {

int ttsw_ctx_create(int device, ttsw_ctx** out) {
  auto* c = new ttsw_ctx;
  int st = guard(c, [&] {
    c->owner = std::make_shared<Context>(device);
    c->c = c->owner.get();
  });
  if (st != TTSW_OK) {
    *out = c;  // caller may read the error, then destroy
    return st;
  }
  *out = c;
  return TTSW_OK;
}

void ttsw_ctx_destroy(ttsw_ctx* ctx) {
  if (!ctx) return;
  delete ctx;  // the Context itself lives until its last device buffer is freed
}

int ttsw_last_error(ttsw_ctx* ctx, char* buf, long len, ttsw_err_info* info) {
  if (!ctx) return TTSW_INPUT;
  if (buf && len > 0) {
    std::strncpy(buf, ctx->err.c_str(), size_t(len - 1));
    buf[len - 1] = 0;
  }
  if (info) *info = ctx->info;
  return TTSW_OK;
}

int ttsw_ctx_sync(ttsw_ctx* ctx) {
  return guard(ctx, [&] { ctx->c->sync(); });
}

void* ttsw_ctx_stream(ttsw_ctx* ctx) { return ctx && ctx->c ? ctx->c->stream : nullptr; }
long ttsw_ctx_launches(ttsw_ctx* ctx) { return ctx && ctx->c ? ctx->c->launches : 0; }

void ttsw_ctx_time_rounds(ttsw_ctx* ctx, int enabled) {
  if (ctx && ctx->c) ctx->c->time_rounds = enabled != 0;
}

void ttsw_ctx_set_sketch(ttsw_ctx* ctx, int enabled, int min_rank, int default_columns) {
  if (!ctx || !ctx->c) return;
  Context* c = ctx->c;
  c->sketch_on = enabled != 0;
  if (min_rank > 0) c->sketch_min_r = min_rank;
  if (default_columns > 0) c->sketch_default_l = (default_columns + 31) / 32 * 32;
  c->sketch_hint.clear();
}

void ttsw_ctx_sketch_stats(ttsw_ctx* ctx, long* used, long* fallback) {
  if (!ctx || !ctx->c) return;
  if (used) *used = ctx->c->sketch_used;
  if (fallback) *fallback = ctx->c->sketch_fallback;
}

void ttsw_ctx_round_stats(ttsw_ctx* ctx, double* s, int reset) {
  if (!ctx || !ctx->c) return;
  Context* c = ctx->c;
  if (s) {
    s[0] = c->round_ms;
    s[1] = c->round_flops;
    s[2] = c->round_bytes;
    s[3] = double(c->round_count);
  }
  if (reset) {
    c->round_ms = c->round_flops = c->round_bytes = 0;
    c->round_count = 0;
  }
}

int ttsw_tt_from_host(ttsw_ctx* ctx, long m, long n, long r, const double* cx, const double* cy, ttsw_tt** out) {
  return guard(ctx, [&] { *out = wrap(tt_from_host(ctx->c, m, n, r, cx, cy)); });
}

int ttsw_tt_from_full(ttsw_ctx* ctx, long m, long n, const double* a, double eps, ttsw_tt** out,
                      ttsw_round_info* info) {
  return guard(ctx, [&] {
    RoundRecord rec{};
    *out = wrap(tt_from_full(ctx->c, m, n, a, eps, &rec));
    if (info) *info = {rec.m, rec.n, rec.r_in, rec.k_out, rec.margin, rec.kappa};
  });
}

int ttsw_tt_to_host(ttsw_ctx* ctx, const ttsw_tt* x, double* cx, double* cy) {
  return guard(ctx, [&] { tt_to_host(x->v, cx, cy); });
}

void ttsw_tt_dims(const ttsw_tt* x, long* m, long* n, long* r) {
  *m = x->v->m;
  *n = x->v->n;
  *r = x->v->r;
}

void ttsw_tt_free(ttsw_tt* x) { delete x; }

int ttsw_tt_constant(ttsw_ctx* ctx, long m, long n, double value, ttsw_tt** out) {
  return guard(ctx, [&] { *out = wrap(tt_constant(ctx->c, m, n, value)); });
}

int ttsw_round(ttsw_ctx* ctx, const ttsw_tt* x, double eps, ttsw_tt** out, ttsw_round_info* info) {
  return guard(ctx, [&] {
    RoundRecord rec{};
    *out = wrap(round(x->v, eps, &rec));
    if (info) *info = {rec.m, rec.n, rec.r_in, rec.k_out, rec.margin, rec.kappa};
  });
}

int ttsw_add(ttsw_ctx* ctx, const ttsw_tt* x, const ttsw_tt* y, ttsw_tt** out) {
  return guard(ctx, [&] { *out = wrap(add(x->v, y->v)); });
}

int ttsw_scale(ttsw_ctx* ctx, const ttsw_tt* x, double a, ttsw_tt** out) {
  return guard(ctx, [&] { *out = wrap(scale(x->v, a)); });
}

int ttsw_axpy(ttsw_ctx* ctx, double a, const ttsw_tt* x, double b, const ttsw_tt* y, double eps, ttsw_tt** out) {
  return guard(ctx, [&] {
    TT s = add(scale(x->v, a), scale(y->v, b));
    *out = wrap(eps < 0 ? s : round(s, eps));
  });
}

int ttsw_hadamard(ttsw_ctx* ctx, const ttsw_tt* x, const ttsw_tt* y, ttsw_tt** out) {
  return guard(ctx, [&] { *out = wrap(hadamard(x->v, y->v)); });
}

int ttsw_mul(ttsw_ctx* ctx, const ttsw_tt* x, const ttsw_tt* y, double eps, ttsw_tt** out) {
  return guard(ctx, [&] {
    TT h = hadamard(x->v, y->v);
    *out = wrap(eps < 0 ? h : round(h, eps));
  });
}

int ttsw_core_map(ttsw_ctx* ctx, const ttsw_tt* x, int axis, int op, int scheme, int side, long n, long a0, long a1,
                  ttsw_tt** out) {
  return guard(ctx, [&] {
    *out = wrap(apply_core_map(x->v, Axis(axis), make_band_map(op, Scheme(scheme), Side(side), n, a0, a1)));
  });
}

int ttsw_core_map_csr(ttsw_ctx* ctx, const ttsw_tt* x, int axis, long rows, long cols, const long* rowptr,
                      const long* colidx, const double* vals, ttsw_tt** out) {
  return guard(ctx, [&] {
    const TT v = materialize(x->v);
    Context* c = ctx->c;
    const Index mode = axis == 0 ? v->m : v->n;
    if (cols != mode) throw ShapeError("apply_core_map: operator/mode size mismatch");
    const long nnz = rowptr[rows];
    for (long p = 0; p < nnz; ++p)
      if (colidx[p] < 0 || colidx[p] >= cols) throw InputError("core_map_csr: column index out of range");
    double* d = c->alloc(size_t(rows + 1 + 2 * nnz + 1));
    long* drp = reinterpret_cast<long*>(d);
    long* dci = drp + rows + 1;
    double* dv = d + rows + 1 + nnz;
    TTSW_CUDA(cudaMemcpyAsync(drp, rowptr, sizeof(long) * size_t(rows + 1), cudaMemcpyHostToDevice, c->stream));
    if (nnz) {
      TTSW_CUDA(cudaMemcpyAsync(dci, colidx, sizeof(long) * size_t(nnz), cudaMemcpyHostToDevice, c->stream));
      TTSW_CUDA(cudaMemcpyAsync(dv, vals, sizeof(double) * size_t(nnz), cudaMemcpyHostToDevice, c->stream));
    }
    auto buf = std::make_shared<DBuf>(c, size_t(rows * v->r));
    launch_csr_map(c, axis == 0 ? v->X : v->Yt, mode, buf->p, rows, v->r, drp, dci, dv);
    c->sync();  // host index arrays are the caller's
    c->free(d);
    if (axis == 0)
      *out = wrap(std::make_shared<DevTT>(c, rows, v->n, v->r, buf, v->yb));
    else
      *out = wrap(std::make_shared<DevTT>(c, v->m, rows, v->r, v->xb, buf));
  });
}

int ttsw_norm_fro(ttsw_ctx* ctx, const ttsw_tt* x, double* out) {
  return guard(ctx, [&] { *out = norm_fro(x->v); });
}

int ttsw_sum_entries(ttsw_ctx* ctx, const ttsw_tt* x, double* out) {
  return guard(ctx, [&] { *out = sum_entries(x->v); });
}

int ttsw_recip_taylor(ttsw_ctx* ctx, const ttsw_tt* x, double eps, int max_iterations, int* iterations,
                      ttsw_tt** out) {
  return guard(ctx, [&] { *out = wrap(reciprocal_taylor(x->v, eps, max_iterations, iterations)); });
}

int ttsw_cross(ttsw_ctx* ctx, int fn, const double* params, const ttsw_tt* const* ops, int nops, const ttsw_tt* guess,
               const ttsw_cross_cfg* cfg, ttsw_tt** out, ttsw_cross_stats* stats) {
  return guard(ctx, [&] {
    std::vector<TT> v;
    for (int k = 0; k < nops; ++k) v.push_back(ops[k]->v);
    CrossStats st;
    *out = wrap(cross_elementwise(fn, params ? params[0] : 0.0, v, guess->v, to_cfg(cfg), &st));
    if (stats) *stats = {st.evaluations, st.sweeps, st.residual};
  });
}

int ttsw_maxvol(ttsw_ctx* ctx, long n, long r, const double* m, long* rows_out) {
  return guard(ctx, [&] {
    auto rows = maxvol_host(ctx->c, n, r, m);
    for (size_t k = 0; k < rows.size(); ++k) rows_out[k] = rows[k];
  });
}

int ttsw_periodic_ghost(ttsw_ctx* ctx, const ttsw_tt* x, ttsw_tt** out) {
  return guard(ctx, [&] { *out = wrap(periodic_ghost(x->v)); });
}

int ttsw_ghosted(ttsw_ctx* ctx, const ttsw_tt* x, int bc_x, int bc_y, const double* strip_x, const double* strip_y,
                 double eps_tt, ttsw_tt** out) {
  return guard(ctx, [&] {
    if ((bc_x != 0 && bc_x != 1) || (bc_y != 0 && bc_y != 1)) throw InputError("tt_ghosted: unknown boundary kind");
    *out = wrap(ghosted(x->v, bc_x == 1, bc_y == 1, strip_x, strip_y, eps_tt));
  });
}

int ttsw_reconstruct_faces(ttsw_ctx* ctx, const ttsw_tt* g, int axis, int scheme, double eps_tt,
                           const ttsw_cross_cfg* cfg, double dx, double dy, ttsw_tt** minus, ttsw_tt** plus) {
  return guard(ctx, [&] {
    ReconContext rc;
    rc.scheme = Scheme(scheme);
    rc.eps_tt = eps_tt;
    rc.cross = to_cfg(cfg);
    rc.dx = dx;
    rc.dy = dy;
    FacePair f = reconstruct_faces(g->v, Axis(axis), rc);
    *minus = wrap(f.minus);
    *plus = wrap(f.plus);
  });
}

int ttsw_solver_create(ttsw_ctx* ctx, const ttsw_solver_desc* d, ttsw_solver** out) {
  return guard(ctx, [&] {
    if (d->n < 1) throw InputError("solver: grid must be non-empty");
    auto* s = new ttsw_solver{ctx, Solver{}, ctx->owner};
    s->s.ctx = ctx->c;
    ctx->c->cross_calls = 0;  // trace alignment counts crosses from solver creation
    s->s.n = d->n;
    s->s.opt.scheme = Scheme(d->scheme);
    s->s.opt.model = Model(d->model);
    s->s.opt.params = {d->g, d->f, d->H};
    s->s.opt.cross = to_cfg(&d->cross);
    s->s.opt.lambda_eps_floor = d->lambda_eps_floor;
    s->s.eps.var = {d->tol, d->tol, d->tol};
    s->s.eps.global = d->tol;
    s->s.dt = d->dt;
    for (int c = 0; c < 3; ++c) s->s.state[size_t(c)] = tt_zero(ctx->c, d->n, d->n);
    *out = s;
  });
}

void ttsw_solver_destroy(ttsw_solver* s) { delete s; }

int ttsw_solver_set_state(ttsw_solver* s, int c, const ttsw_tt* x) {
  return guard(s->ctx, [&] {
    if (c < 0 || c > 2) throw InputError("solver: component out of range");
    if (x->v->m != s->s.n || x->v->n != s->s.n) throw ShapeError("solver: state shape mismatch");
    s->s.state[size_t(c)] = x->v;
  });
}

int ttsw_solver_get_state(ttsw_solver* s, int c, ttsw_tt** out) {
  return guard(s->ctx, [&] {
    if (c < 0 || c > 2) throw InputError("solver: component out of range");
    *out = wrap(s->s.state[size_t(c)]);
  });
}

int ttsw_solver_rhs(ttsw_solver* s, ttsw_tt** out3) {
  return guard(s->ctx, [&] {
    struct TraceScope {
      Context* c;
      ~TraceScope() {
        c->trace = nullptr;
        c->ctrace = nullptr;
      }
    } trace_scope{s->s.ctx};
    s->s.ctx->trace = s->s.tracing ? &s->s.trace : nullptr;
    s->s.ctx->ctrace = s->s.tracing ? &s->s.ctrace : nullptr;
    Triple r = s->s.rhs(s->s.state, s->s.t);
    for (int c = 0; c < 3; ++c) out3[c] = wrap(r[size_t(c)]);
  });
}

int ttsw_solver_step(ttsw_solver* s, long nsteps) {
  return guard(s->ctx, [&] {
    long k = 0;
    try {
      for (; k < nsteps; ++k) s->s.step();  // Solver::step resets the context's trace pointers
    } catch (const CudaError&) {
      throw;
    } catch (const std::exception& e) {
      std::ostringstream os;
      os << "run: failed at step " << k << ": " << e.what();
      throw StateError(os.str());
    }
  });
}

int ttsw_solver_set_dt(ttsw_solver* s, double dt) {
  return guard(s->ctx, [&] {
    if (!(dt > 0)) throw InputError("ssprk3: dt must be positive");
    s->s.dt = dt;
  });
}

int ttsw_solver_set_time(ttsw_solver* s, double t) {
  return guard(s->ctx, [&] { s->s.t = t; });
}
double ttsw_solver_time(const ttsw_solver* s) { return s->s.t; }

int ttsw_solver_set_hooks(ttsw_solver* s, ttsw_fill_ghost_fn ghost, ttsw_extra_source_fn source, void* user) {
  return guard(s->ctx, [&] {
    // The library owns the handles a hook writes to out[0..2], also when the hook fails
    // or leaves a slot empty. The same handle may fill several slots (freed once).
    auto release = [](ttsw_tt** h) {
      for (int c = 0; c < 3; ++c) {
        if (!h[c]) continue;
        for (int d = c + 1; d < 3; ++d)
          if (h[d] == h[c]) h[d] = nullptr;
        delete h[c];
        h[c] = nullptr;
      }
    };
    auto take = [release](ttsw_tt** h, int status, const char* what) {
      if (status != 0) {
        release(h);
        throw StateError(std::string(what) + " hook failed");
      }
      for (int c = 0; c < 3; ++c)
        if (!h[c]) {
          release(h);
          throw StateError(std::string(what) + ": hook returned no field");
        }
      Triple out;
      for (int c = 0; c < 3; ++c) out[size_t(c)] = h[c]->v;
      release(h);
      return out;
    };
    s->s.fill_ghost = nullptr;
    s->s.extra_source = nullptr;
    if (ghost)
      s->s.fill_ghost = [ghost, user, take](const Triple& u, double t) {
        ttsw_tt in[3] = {{u[0]}, {u[1]}, {u[2]}};
        const ttsw_tt* q3[3] = {&in[0], &in[1], &in[2]};
        ttsw_tt* out[3] = {nullptr, nullptr, nullptr};
        const int status = ghost(user, q3, t, out);
        return take(out, status, "fill_ghost");
      };
    if (source)
      s->s.extra_source = [source, user, take](double t) {
        ttsw_tt* out[3] = {nullptr, nullptr, nullptr};
        const int status = source(user, t, out);
        return take(out, status, "extra_source");
      };
  });
}

long ttsw_solver_trace_len(const ttsw_solver* s) { return long(s->s.trace.size()); }

void ttsw_solver_trace(const ttsw_solver* s, long* ints, double* margins, double* kappas) {
  for (size_t i = 0; i < s->s.trace.size(); ++i) {
    const auto& r = s->s.trace[i];
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

void ttsw_solver_trace_clear(ttsw_solver* s) { s->s.trace.clear(); }

long ttsw_solver_cross_trace_len(const ttsw_solver* s) { return long(s->s.ctrace.size()); }

void ttsw_solver_cross_trace(ttsw_solver* s, long* ints, double* residuals, int clear) {
  for (size_t i = 0; i < s->s.ctrace.size(); ++i) {
    ints[3 * i] = s->s.ctrace[i].rank;
    ints[3 * i + 1] = s->s.ctrace[i].sweeps;
    ints[3 * i + 2] = s->s.ctrace[i].pivot_hash;
    residuals[i] = s->s.ctrace[i].residual;
  }
  if (clear) s->s.ctrace.clear();
}
void ttsw_solver_set_tracing(ttsw_solver* s, int enabled) { s->s.tracing = enabled != 0; }
int ttsw_solver_set_eps_policy(ttsw_solver* s, double c_eps, int order, double volume, double clip) {
  return guard(s->ctx, [&] {
    if (!(clip > 0) || order < 1 || !(volume > 0)) throw InputError("eps policy: invalid parameters");
    s->s.use_policy = true;
    s->s.policy = EpsPolicy{c_eps, order, volume, clip};
  });
}
void ttsw_solver_eps(const ttsw_solver* s, double* out4) {
  for (int c = 0; c < 3; ++c) out4[c] = s->s.eps.var[size_t(c)];
  out4[3] = s->s.eps.global;
}

/* --- full-tensor DenseRep path (swe.hpp:45-80) ---------------------------------- */
int ttsw_dense_create(ttsw_ctx* ctx, const ttsw_solver_desc* d, ttsw_dense** out) {
  return guard(ctx, [&] {
    if (d->n < 1) throw InputError("dense solver: grid must be non-empty");
    SolverOptions o;
    o.scheme = Scheme(d->scheme);
    o.model = Model(d->model);
    o.params = {d->g, d->f, d->H};
    auto* s = new ttsw_dense{ctx, ctx->owner, nullptr};
    try {
      s->s = std::make_unique<DenseSolver>(ctx->c, o, d->n, d->dt);
    } catch (...) {
      delete s;
      throw;
    }
    *out = s;
  });
}
void ttsw_dense_destroy(ttsw_dense* s) { delete s; }
int ttsw_dense_set_state(ttsw_dense* s, int c, const double* host_colmajor) {
  return guard(s->ctx, [&] {
    if (c < 0 || c > 2) throw InputError("dense solver: component out of range");
    const size_t nn = size_t(s->s->n * s->s->n);
    for (size_t e = 0; e < nn; ++e)
      if (!std::isfinite(host_colmajor[e])) throw InputError("dense solver: state has non-finite entries");
    TTSW_CUDA(cudaMemcpyAsync(s->s->q[c], host_colmajor, nn * sizeof(double), cudaMemcpyHostToDevice,
                              s->s->ctx->stream));
    s->s->ctx->sync();
  });
}
int ttsw_dense_get_state(ttsw_dense* s, int c, double* host_colmajor) {
  return guard(s->ctx, [&] {
    if (c < 0 || c > 2) throw InputError("dense solver: component out of range");
    const size_t nn = size_t(s->s->n * s->s->n);
    TTSW_CUDA(cudaMemcpyAsync(host_colmajor, s->s->q[c], nn * sizeof(double), cudaMemcpyDeviceToHost,
                              s->s->ctx->stream));
    s->s->ctx->sync();
  });
}
double* ttsw_dense_device_state(ttsw_dense* s, int c) { return (c < 0 || c > 2) ? nullptr : s->s->q[c]; }
int ttsw_dense_set_dt(ttsw_dense* s, double dt) {
  return guard(s->ctx, [&] {
    if (!(dt > 0)) throw InputError("ssprk3: dt must be positive");
    s->s->dt = dt;
  });
}
int ttsw_dense_set_time(ttsw_dense* s, double t) {
  return guard(s->ctx, [&] { s->s->t = t; });
}
double ttsw_dense_time(const ttsw_dense* s) { return s->s->t; }
int ttsw_dense_set_hooks(ttsw_dense* s, int bc_x, int bc_y, ttsw_dense_strip_fn strips, ttsw_dense_source_fn source,
                         void* user) {
  return guard(s->ctx, [&] {
    if ((bc_x || bc_y) && !strips) throw InputError("dense solver: Dirichlet axes need a strip callback");
    s->s->bc_x = bc_x ? 1 : 0;
    s->s->bc_y = bc_y ? 1 : 0;
    s->s->strip_fn = nullptr;
    s->s->source_fn = nullptr;
    if (strips)
      s->s->strip_fn = [strips, user](double t, int c, double* sx, double* sy) { return strips(user, t, c, sx, sy); };
    if (source)
      s->s->source_fn = [source, user](double t, double* out) { return source(user, t, out); };
  });
}
int ttsw_dense_step(ttsw_dense* s, long nsteps) {
  return guard(s->ctx, [&] {
    long k = 0;
    try {
      for (; k < nsteps; ++k) s->s->step();
      s->s->ctx->sync();
    } catch (const CudaError&) {
      throw;
    } catch (const std::exception& e) {
      std::ostringstream os;
      os << "run: failed at step " << k << ": " << e.what();
      throw StateError(os.str());
    }
  });
}
int ttsw_dense_rhs(ttsw_dense* s, double* out3_host) {
  return guard(s->ctx, [&] {
    const size_t nn = size_t(s->s->n * s->s->n);
    double* d = s->s->ctx->alloc(3 * nn);
    double* outs[3] = {d, d + nn, d + 2 * nn};
    try {
      s->s->rhs(outs);
    } catch (...) {
      s->s->ctx->free(d);
      throw;
    }
    TTSW_CUDA(cudaMemcpyAsync(out3_host, d, 3 * nn * sizeof(double), cudaMemcpyDeviceToHost, s->s->ctx->stream));
    s->s->ctx->sync();
    s->s->ctx->free(d);
  });
}

/* --- C5 ensembles (native runtime) ------------------------------------ */
namespace {
int ensemble_status(ttsw_ensemble* e, const std::function<void()>& f) {
  // same exception -> status mapping as guard(), kept per ensemble
  ttsw_ctx tmp{};
  const int st = guard(&tmp, f);
  if (st != TTSW_OK) {
    e->err = tmp.err;
    e->status = st;
  }
  return st;
}
}  // namespace

int ttsw_ensemble_create(int device, int members, const ttsw_solver_desc* descs, int threads, ttsw_ensemble** out) {
  auto* e = new ttsw_ensemble{};
  const int st = ensemble_status(e, [&] {
    if (members < 1) throw InputError("ensemble: at least one member");
    TTSW_CUDA(cudaSetDevice(device));
    e->device = device;
    // at most 32 workers: beyond the device's 32 hardware work queues
    // (CUDA_DEVICE_MAX_CONNECTIONS) more concurrent member streams add no throughput
    // (11.1 member-steps/s at 16 and 32 workers, C5 N=2048), and 64 concurrent workers
    // (each with its children's streams) faulted once on the B200 (profiles/r02_bench_C5_*)
    const int nt = std::max(1, std::min({threads, members, 32}));
    for (int w = 0; w < nt; ++w) e->workers.push_back(std::make_shared<Context>(device));
    for (int m = 0; m < members; ++m) {
      const ttsw_solver_desc& d = descs[m];
      if (d.n < 1) throw InputError("ensemble: grid must be non-empty");
      auto mem = std::make_unique<EnsembleMember>();
      Solver& s = mem->s;
      s.ctx = e->ctx_of(size_t(m));
      s.n = d.n;
      s.opt.scheme = Scheme(d.scheme);
      s.opt.model = Model(d.model);
      s.opt.params = {d.g, d.f, d.H};
      s.opt.cross = to_cfg(&d.cross);
      s.opt.lambda_eps_floor = d.lambda_eps_floor;
      s.eps.var = {d.tol, d.tol, d.tol};
      s.eps.global = d.tol;
      s.dt = d.dt;
      s.tracing = false;
      for (int c = 0; c < 3; ++c) s.state[size_t(c)] = tt_zero(s.ctx, d.n, d.n);
      e->members.push_back(std::move(mem));
    }
  });
  if (st != TTSW_OK) {
    delete e;
    *out = nullptr;
    return st;
  }
  *out = e;
  return TTSW_OK;
}

void ttsw_ensemble_destroy(ttsw_ensemble* e) {
  if (!e) return;
  for (auto& w : e->workers) w->sync();
  e->members.clear();
  delete e;
}

int ttsw_ensemble_set_state_host(ttsw_ensemble* e, int member, int c, long m, long n, long r, const double* cx,
                                 const double* cy, double round_eps) {
  return ensemble_status(e, [&] {
    if (member < 0 || member >= int(e->members.size()) || c < 0 || c > 2) throw InputError("ensemble: index out of range");
    Solver& s = e->members[size_t(member)]->s;
    TTSW_CUDA(cudaSetDevice(e->device));
    if (m != s.n || n != s.n) throw ShapeError("ensemble: state shape mismatch");
    TT x = tt_from_host(s.ctx, m, n, r, cx, cy);
    s.state[size_t(c)] = round_eps >= 0 ? round(x, round_eps) : x;
  });
}

int ttsw_ensemble_step(ttsw_ensemble* e, long nsteps) {
  return ensemble_status(e, [&] {
    const size_t nw = e->workers.size();
    std::vector<std::exception_ptr> errs(nw);
    std::vector<std::thread> ts;
    for (size_t w = 0; w < nw; ++w)
      ts.emplace_back([e, w, nw, nsteps, &errs] {
        try {
          TTSW_CUDA(cudaSetDevice(e->device));
          const auto t0 = std::chrono::steady_clock::now();
          for (long k = 0; k < nsteps; ++k)
            for (size_t m = w; m < e->members.size(); m += nw) {
              EnsembleMember& mem = *e->members[m];
              try {
                mem.s.step();
              } catch (const CudaError&) {
                throw;
              } catch (const std::exception& ex) {
                std::ostringstream os;
                os << "ensemble member " << m << ": run: failed at step " << mem.steps << ": " << ex.what();
                throw StateError(os.str());
              }
              ++mem.steps;
              for (int c = 0; c < 3; ++c)
                mem.max_rank[size_t(c)] = std::max<long>(mem.max_rank[size_t(c)], mem.s.state[size_t(c)]->r);
            }
          e->workers[w]->sync();
          const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
          for (size_t m = w; m < e->members.size(); m += nw) e->members[m]->ms += ms;
        } catch (...) {
          errs[w] = std::current_exception();
        }
      });
    for (auto& t : ts) t.join();
    for (auto& ep : errs)
      if (ep) std::rethrow_exception(ep);
  });
}

int ttsw_ensemble_records(ttsw_ensemble* e, double* out) {
  return ensemble_status(e, [&] {
    TTSW_CUDA(cudaSetDevice(e->device));
    for (size_t m = 0; m < e->members.size(); ++m) {
      const EnsembleMember& mem = *e->members[m];
      const double n = double(mem.s.n);
      double* r = out + 10 * m;
      r[0] = double(m);
      r[1] = double(mem.steps);
      r[2] = sum_entries(mem.s.state[0]) / (n * n);
      for (int c = 0; c < 3; ++c) {
        r[3 + c] = double(mem.s.state[size_t(c)]->r);
        r[6 + c] = double(mem.max_rank[size_t(c)]);
      }
      r[9] = mem.ms;
    }
  });
}

int ttsw_ensemble_last_error(ttsw_ensemble* e, char* buf, long len) {
  if (buf && len > 0) {
    std::strncpy(buf, e->err.c_str(), size_t(len - 1));
    buf[len - 1] = 0;
  }
  return e->status;
}

}  // extern "C"
