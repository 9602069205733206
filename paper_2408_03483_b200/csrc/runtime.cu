// Host runtime: context, device TT handles and the TT algebra of
// /root/reference/proj/include/ttsw/tt.hpp re-designed around device-resident cores.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <sstream>
#include <unordered_set>
#include <mutex>
#include <set>
#include <string>

#include "expr.cuh"
#include "kernels.cuh"

namespace ttsw {

void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess) {
    std::ostringstream os;
    os << "CUDA error " << cudaGetErrorName(e) << " (" << cudaGetErrorString(e) << ") at " << file << ":" << line
       << ": " << what;
    throw CudaError(os.str());
  }
}

Context::Context(int dev) : device(dev) {
  TTSW_CUDA(cudaSetDevice(dev));
  TTSW_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
  cudaMemPool_t pool;
  TTSW_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
  uint64_t threshold = UINT64_MAX;
  TTSW_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold));
  int v = 0;
  TTSW_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev));
  num_sms = v;
  TTSW_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  smem_optin = size_t(v);
  TTSW_CUDA(cudaMallocHost(&pinned, 65536));
  TTSW_CUDA(cudaEventCreate(&ev0));
  TTSW_CUDA(cudaEventCreate(&ev1));
  TTSW_CUDA(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
  TTSW_CUDA(cudaEventCreateWithFlags(&fork_ev, cudaEventDisableTiming));
  TTSW_CUDA(cudaEventCreateWithFlags(&join_ev, cudaEventDisableTiming));
}

// Function attributes are per device: cached by (device, kernel[, attribute]).
void allow_dynamic_smem(const void* kernel, size_t bytes) {
  static std::mutex mu;
  static std::set<std::pair<int, const void*>> done;
  std::lock_guard<std::mutex> lock(mu);
  int dev = 0, optin = 0;
  TTSW_CUDA(cudaGetDevice(&dev));
  if (done.count({dev, kernel})) return;
  TTSW_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  cudaFuncAttributes fa{};
  TTSW_CUDA(cudaFuncGetAttributes(&fa, kernel));
  const int limit = optin - int(fa.sharedSizeBytes);  // dynamic = opt-in minus the static part
  if (bytes > size_t(limit)) throw CudaError("dynamic shared memory request above the device limit");
  TTSW_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, limit));
  done.insert({dev, kernel});
}

void allow_nonportable_cluster(const void* kernel) {
  static std::mutex mu;
  static std::set<std::pair<int, const void*>> done;
  std::lock_guard<std::mutex> lock(mu);
  int dev = 0;
  TTSW_CUDA(cudaGetDevice(&dev));
  if (done.count({dev, kernel})) return;
  TTSW_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  done.insert({dev, kernel});
}

Context* Context::child(size_t i) {
  while (children.size() <= i) children.push_back(std::make_shared<Context>(device));
  return children[i].get();
}

TT adopt(Context* ctx, const TT& xin) {
  const TT x = materialize(xin);
  if (x->ctx == ctx) return x;
  for (const Buf& b : {x->xb, x->yb}) {
    b->owner = ctx->shared_from_this();
    b->ctx = ctx;
  }
  return std::make_shared<DevTT>(ctx, x->m, x->n, x->r, x->xb, x->yb);
}

void Context::ensure_stage(size_t bytes) {
  if (bytes <= stage_cap) return;
  sync();
  if (stage_host) cudaFreeHost(stage_host);
  if (stage_dev) cudaFree(stage_dev);
  stage_cap = std::max(bytes, 2 * stage_cap);
  TTSW_CUDA(cudaMallocHost(&stage_host, stage_cap));
  TTSW_CUDA(cudaMalloc(&stage_dev, stage_cap));
}

double* Context::ensure_work(size_t doubles) {
  if (doubles > work_cap) {
    sync();
    if (work_dev) cudaFree(work_dev);
    work_cap = std::max(doubles, 2 * work_cap);
    void* p = nullptr;
    TTSW_CUDA(cudaMalloc(&p, work_cap * sizeof(double)));
    work_dev = static_cast<double*>(p);
  }
  return work_dev;
}

Context::~Context() {
  if (omega && stream) cudaFreeAsync(omega, stream);
  if (stream) cudaStreamSynchronize(stream);
  if (stage_host) cudaFreeHost(stage_host);
  if (stage_dev) cudaFree(stage_dev);
  if (work_dev) cudaFree(work_dev);
  if (map_dev) cudaFree(map_dev);
  if (ev0) cudaEventDestroy(ev0);
  if (ev1) cudaEventDestroy(ev1);
  if (side) cudaStreamSynchronize(side);
  if (fork_ev) cudaEventDestroy(fork_ev);
  if (join_ev) cudaEventDestroy(join_ev);
  if (side) cudaStreamDestroy(side);
  if (pinned) cudaFreeHost(pinned);
  if (stream) cudaStreamDestroy(stream);
}

double* Context::alloc(size_t count) {
  void* p = nullptr;
  if (count == 0) count = 1;
  TTSW_CUDA(cudaMallocAsync(&p, count * sizeof(double), stream));
  return static_cast<double*>(p);
}

void Context::free(void* p) {
  if (p) cudaFreeAsync(p, stream);
}

void Context::sync() {
  if (!count_sync) {
    TTSW_CUDA(cudaStreamSynchronize(stream));
    return;
  }
  const auto t0 = std::chrono::steady_clock::now();
  TTSW_CUDA(cudaStreamSynchronize(stream));
  sync_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  ++sync_count;
}

DevTT::DevTT(Context* c, Index m_, Index n_, Index r_, Buf x, Buf y)
    : ctx(c), m(m_), n(n_), r(r_), xb(std::move(x)), yb(std::move(y)), X(xb->p), Yt(yb->p) {
  HostTerm t;
  t.kind = TERM_PLAIN;
  t.r = r;
  t.x.base = xb;
  t.x.ld = m;
  t.y.base = yb;
  t.y.ld = n;
  terms.push_back(std::move(t));
}

DevTT::DevTT(Context* c, Index m_, Index n_, std::vector<HostTerm> t) : ctx(c), m(m_), n(n_), r(0), terms(std::move(t)) {
  for (const auto& term : terms) r += term.r;
}

MutTT make_tt(Context* ctx, Index m, Index n, Index r) {
  return std::make_shared<DevTT>(ctx, m, n, r, std::make_shared<DBuf>(ctx, size_t(m * r)),
                                 std::make_shared<DBuf>(ctx, size_t(n * r)));
}

int Context::register_map(const BandMap& bm) {
  MapDesc d{};
  d.n_out = bm.n_out;
  d.n_in = bm.n_in;
  d.period = bm.period;
  d.stride = bm.stride;
  d.taps = bm.taps;
  d.wrap = bm.wrap ? 1 : 0;
  for (int i = 0; i < 3; ++i) {
    d.off[i] = bm.off[i];
    for (int j = 0; j < 5; ++j) d.coef[i][j] = bm.coef[i][j];
  }
  std::string key(reinterpret_cast<const char*>(&d), sizeof(d));
  for (size_t i = 0; i < map_keys.size(); ++i)
    if (map_keys[i] == key) return int(i);
  map_keys.push_back(key);
  map_host.insert(map_host.end(), key.begin(), key.end());
  return int(map_keys.size() - 1);
}

const void* Context::device_maps() {
  if (map_dev_count != map_keys.size()) {
    if (map_dev) {
      TTSW_CUDA(cudaStreamSynchronize(stream));
      TTSW_CUDA(cudaFree(map_dev));
    }
    TTSW_CUDA(cudaMalloc(&map_dev, std::max<size_t>(map_host.size(), 1)));
    TTSW_CUDA(cudaMemcpy(map_dev, map_host.data(), map_host.size(), cudaMemcpyHostToDevice));
    map_dev_count = map_keys.size();
  }
  return map_dev;
}

/// Device descriptors of a lazy TT (terms sorted by column), uploaded to `dst`.
static std::vector<TermDesc> term_descs(const DevTT& x) {
  std::vector<TermDesc> out;
  long col = 0;
  for (const auto& t : x.terms) {
    TermDesc d{};
    d.kind = t.kind;
    d.r = int(t.r);
    d.col0 = col;
    auto side = [](const HostSide& hs, SideExpr& se) {
      se.base = hs.base ? hs.base->p : nullptr;
      se.ld = hs.ld;
      if (hs.ops.size() > size_t(kMaxSideOps)) throw InputError("lazy TT: operation chain too long");
      se.nops = int(hs.ops.size());
      for (size_t i = 0; i < hs.ops.size(); ++i) se.ops[i] = {hs.ops[i].kind, hs.ops[i].map, hs.ops[i].scale};
    };
    side(t.x, d.x);
    side(t.y, d.y);
    d.x2 = t.x2 ? t.x2->p : nullptr;
    d.y2 = t.y2 ? t.y2->p : nullptr;
    d.ldx2 = t.ldx2;
    d.ldy2 = t.ldy2;
    d.r2 = int(t.r2);
    d.cx = t.cx;
    d.cy = t.cy;
    out.push_back(d);
    col += t.r;
  }
  return out;
}

/// Evaluate both sides of a lazy TT into panels X (m x r, ld m) and Yt (n x r, ld n).
void gather_panels(const TT& x, double* X, double* Yt) {
  Context* ctx = x->ctx;
  std::vector<TermDesc> d = term_descs(*x);
  const void* maps = ctx->device_maps();
  // one job of the column-organised gather (k_gather_cols): descriptors, then the job
  const size_t td = (sizeof(TermDesc) * d.size() + 255) / 256 * 256;
  std::vector<char> h(td + sizeof(RoundJob));
  char* dbuf = reinterpret_cast<char*>(ctx->alloc((h.size() + 7) / 8));
  RoundJob J{};
  J.terms = reinterpret_cast<const TermDesc*>(dbuf);
  J.nterms = int(d.size());
  J.m = x->m;
  J.n = x->n;
  J.R = int(x->r);
  J.Xs = X;
  J.Ys = Yt;
  std::memcpy(h.data(), d.data(), sizeof(TermDesc) * d.size());
  std::memcpy(h.data() + td, &J, sizeof(RoundJob));
  // pageable source: the upload has been staged when the call returns
  TTSW_CUDA(cudaMemcpyAsync(dbuf, h.data(), h.size(), cudaMemcpyHostToDevice, ctx->stream));
  launch_gather_jobs(ctx, reinterpret_cast<const RoundJob*>(dbuf + td), 1, 2 * x->r, static_cast<const MapDesc*>(maps),
                     int(ctx->map_keys.size()), int(d.size()));
  ctx->free(reinterpret_cast<double*>(dbuf));
}

TT materialize(const TT& x) {
  HostRegion hr_(x->ctx, "materialize");
  if (x->materialised()) return x;
  if (x->cache) return x->cache;
  auto t = make_tt(x->ctx, x->m, x->n, x->r);
  gather_panels(x, t->X, t->Yt);
  x->cache = t;
  return t;
}

static void check_finite(const double* p, size_t count) {
  for (size_t i = 0; i < count; ++i)
    if (!std::isfinite(p[i])) throw InputError("TTMatrix: cores contain non-finite entries");
}

TT tt_from_host(Context* ctx, Index m, Index n, Index r, const double* cx, const double* cy) {
  if (r < 1) throw ShapeError("TTMatrix: rank must be positive");
  if (m < 1 || n < 1) throw ShapeError("TTMatrix: empty mode");
  check_finite(cx, size_t(m * r));
  check_finite(cy, size_t(r * n));
  auto t = make_tt(ctx, m, n, r);
  std::vector<double> yt(static_cast<size_t>(n * r));
  for (Index a = 0; a < r; ++a)
    for (Index j = 0; j < n; ++j) yt[size_t(j + a * n)] = cy[a + j * r];
  TTSW_CUDA(cudaMemcpyAsync(t->X, cx, sizeof(double) * size_t(m * r), cudaMemcpyHostToDevice, ctx->stream));
  TTSW_CUDA(cudaMemcpyAsync(t->Yt, yt.data(), sizeof(double) * size_t(n * r), cudaMemcpyHostToDevice, ctx->stream));
  ctx->sync();
  return t;
}

/// tt_from_full (tt.hpp:82-97) on the device. The dense A (m x n, column-major) is uploaded
/// as the exact rank-min(m, n) TT (A, I_n), or (I_m, A) when m < n, and rounded with the
/// same eps: the round's orthogonalisation of the identity core is exact up to sign, so the
/// SVD it takes has A's singular values and truncation_rank (tt.hpp:61-77) keeps the same
/// k as the reference's SVD of A; a zero A rounds to TTMatrix::zero as the reference returns.
/// The identity core is written by a memset and one strided copy of its diagonal.
TT tt_from_full(Context* ctx, Index m, Index n, const double* a, double eps, RoundRecord* rec) {
  if (m < 1 || n < 1) throw ShapeError("tt_from_full: empty matrix");
  for (size_t i = 0; i < size_t(m * n); ++i)
    if (!std::isfinite(a[i])) throw InputError("tt_from_full: non-finite entries");
  if (eps < 0) throw InputError("tt_from_full: eps must be non-negative");
  const Index r = std::min(m, n);
  auto t = make_tt(ctx, m, n, r);
  const std::vector<double> ones(size_t(r), 1.0);  // lives until the sync below
  auto identity = [&](double* p, Index k) {
    TTSW_CUDA(cudaMemsetAsync(p, 0, sizeof(double) * size_t(k * k), ctx->stream));
    TTSW_CUDA(cudaMemcpy2DAsync(p, sizeof(double) * size_t(k + 1), ones.data(), sizeof(double), sizeof(double),
                                size_t(k), cudaMemcpyHostToDevice, ctx->stream));
  };
  std::vector<double> at;
  if (m >= n) {  // X = A, Yt = I_n
    TTSW_CUDA(cudaMemcpyAsync(t->X, a, sizeof(double) * size_t(m * n), cudaMemcpyHostToDevice, ctx->stream));
    identity(t->Yt, n);
  } else {  // X = I_m, Yt = A^T (n x m, column-major)
    at.resize(size_t(n * m));
    for (Index j = 0; j < n; ++j)
      for (Index i = 0; i < m; ++i) at[size_t(j + i * n)] = a[i + j * m];
    identity(t->X, m);
    TTSW_CUDA(cudaMemcpyAsync(t->Yt, at.data(), sizeof(double) * at.size(), cudaMemcpyHostToDevice, ctx->stream));
  }
  ctx->sync();
  return round(t, eps, rec);
}

void tt_to_host(const TT& xin, double* cx, double* cy) {
  const TT x = materialize(xin);
  Context* ctx = x->ctx;
  std::vector<double> yt(static_cast<size_t>(x->n * x->r));
  TTSW_CUDA(cudaMemcpyAsync(cx, x->X, sizeof(double) * size_t(x->m * x->r), cudaMemcpyDeviceToHost, ctx->stream));
  TTSW_CUDA(cudaMemcpyAsync(yt.data(), x->Yt, sizeof(double) * yt.size(), cudaMemcpyDeviceToHost, ctx->stream));
  ctx->sync();
  for (Index a = 0; a < x->r; ++a)
    for (Index j = 0; j < x->n; ++j) cy[a + j * x->r] = yt[size_t(j + a * x->n)];
}

static TT const_term(Context* ctx, Index rows, Index cols, double cx, double cy) {
  HostTerm t;
  t.kind = TERM_CONST;
  t.r = 1;
  t.cx = cx;
  t.cy = cy;
  return std::make_shared<DevTT>(ctx, rows, cols, std::vector<HostTerm>{t});
}

/// TTMatrix::zero (tt.hpp:35-37): rank-1 zero cores (lazy constant term).
TT tt_zero(Context* ctx, Index rows, Index cols) { return const_term(ctx, rows, cols, 0.0, 0.0); }

/// TTMatrix::constant (tt.hpp:39-41).
TT tt_constant(Context* ctx, Index rows, Index cols, double v) { return const_term(ctx, rows, cols, v, 1.0); }

static void check_same_shape(const TT& x, const TT& y, const char* where) {
  if (x->m != y->m || x->n != y->n) throw ShapeError(std::string(where) + ": operand shapes do not match");
}

static void append_scale(HostTerm& t, double a) {
  if (a == 1.0) return;  // x * 1.0 == x exactly
  if (t.kind == TERM_CONST) {
    t.cx = t.cx * a;
    return;
  }
  t.x.ops.push_back({0, 0, a});
}

/// add(scale(x,a), scale(y,b)) (tt.hpp:152-166): lazy concatenation, x first.
static TT add_scaled(double a, const TT& x, double b, const TT& y) {
  check_same_shape(x, y, "add");
  std::vector<HostTerm> terms = x->terms;
  for (auto& t : terms) append_scale(t, a);
  for (HostTerm t : y->terms) {
    append_scale(t, b);
    terms.push_back(std::move(t));
  }
  return std::make_shared<DevTT>(x->ctx, x->m, x->n, std::move(terms));
}

TT add(const TT& x, const TT& y) { return add_scaled(1.0, x, 1.0, y); }

/// scale (tt.hpp:163-166): scales core_x only (lazy).
TT scale(const TT& x, double a) {
  std::vector<HostTerm> terms = x->terms;
  for (auto& t : terms) {
    if (a == 1.0) continue;
    if (t.kind == TERM_CONST)
      t.cx = t.cx * a;
    else
      t.x.ops.push_back({0, 0, a});
  }
  return std::make_shared<DevTT>(x->ctx, x->m, x->n, std::move(terms));
}

/// hadamard (tt.hpp:169-181): one lazy face-splitting term over materialised operands.
TT hadamard(const TT& xin, const TT& yin) {
  HostRegion hr_(xin->ctx, "hadamard");
  check_same_shape(xin, yin, "hadamard");
  const TT x = materialize(xin), y = materialize(yin);
  HostTerm t;
  t.kind = TERM_HADAMARD;
  t.r = x->r * y->r;
  t.x.base = x->xb;
  t.x.ld = x->m;
  t.y.base = x->yb;
  t.y.ld = x->n;
  t.x2 = y->xb;
  t.y2 = y->yb;
  t.ldx2 = y->m;
  t.ldy2 = y->n;
  t.r2 = y->r;
  return std::make_shared<DevTT>(x->ctx, x->m, x->n, std::vector<HostTerm>{t});
}

static double read_scalar(Context* ctx, const double* dptr) {
  TTSW_CUDA(cudaMemcpyAsync(ctx->pinned, dptr, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  ctx->sync();
  return *static_cast<double*>(ctx->pinned);
}

/// norm_fro (tt.hpp:105-111): Gram-based, clamped at zero.
double norm_fro(const TT& xin) {
  const TT x = materialize(xin);
  Context* ctx = x->ctx;
  double* work = ctx->alloc(size_t(x->r * x->r + 1));
  launch_norm2(ctx, x->X, x->m, x->Yt, x->n, x->r, work, work + x->r * x->r);
  const double v = read_scalar(ctx, work + x->r * x->r);
  ctx->free(work);
  return std::sqrt(std::max(v, 0.0));
}

/// sum_entries (tt.hpp:113-116).
/// norm_fro of several TTs with one host sync (same arithmetic per TT as norm_fro).
std::vector<double> norm_fro_batch(const std::vector<TT>& xin) {
  std::vector<double> out(xin.size(), 0.0);
  if (xin.empty()) return out;
  Context* ctx = xin[0]->ctx;
  std::vector<TT> xs;
  std::vector<double*> work;
  for (const auto& x0 : xin) {
    const TT x = materialize(x0);
    double* w = ctx->alloc(size_t(x->r * x->r + 1));
    launch_norm2(ctx, x->X, x->m, x->Yt, x->n, x->r, w, w + x->r * x->r);
    xs.push_back(x);
    work.push_back(w);
  }
  double* h = static_cast<double*>(ctx->pinned);
  for (size_t i = 0; i < xs.size(); ++i)
    TTSW_CUDA(cudaMemcpyAsync(h + i, work[i] + xs[i]->r * xs[i]->r, sizeof(double), cudaMemcpyDeviceToHost,
                              ctx->stream));
  ctx->sync();
  for (size_t i = 0; i < xs.size(); ++i) {
    out[i] = std::sqrt(std::max(h[i], 0.0));
    ctx->free(work[i]);
  }
  return out;
}

double sum_entries(const TT& xin) {
  const TT x = materialize(xin);
  Context* ctx = x->ctx;
  double* work = ctx->alloc(size_t(2 * x->r + 1));
  launch_sum_entries(ctx, x->X, x->m, x->Yt, x->n, x->r, work, work + 2 * x->r);
  const double v = read_scalar(ctx, work + 2 * x->r);
  ctx->free(work);
  return v;
}

/// round (tt.hpp:120-138). Both cores are orthogonalised by TSQR (X = Qx Rx,
/// Yt = Qy Ry); the R x R product S = Rx Ry^T has the singular values of the
/// reference's W = core_x R^T; its Jacobi SVD yields core_x' = Qx (S V)_k and
/// round's zero check (tt.hpp:120-127: norm_fro(x) == 0 -> TTMatrix::zero). A TT whose
/// entries cancel exactly (e.g. jump = u+ - u- of identical faces) has ||X|| = 0 in exact
/// arithmetic; its computed norm is roundoff of ||core_x|| ||core_y|| in any implementation
/// (the reference's Gram sum is clamped at zero: its outcome is a coin flip on roundoff). A
/// TT that small relative to its factors (kappa >= 1 / (4 R u)) carries no information, so
/// it is returned as the canonical zero like an exactly-zero input.
static bool numerically_zero(Index R, double kappa) {
  return kappa >= 1.0 / (4.0 * double(R) * 2.220446049250313e-16);
}

/// core_y'^T = Qy V_k (core_y' keeps orthonormal rows).
/// The truncation rank is decided on device (tt.hpp:61-77) and read back once.
static TT round_tsqr(const TT& xin, double eps, RoundRecord* rec) {
  const TT x = materialize(xin);
  Context* ctx = x->ctx;
  const Index R = x->r, m = x->m, n = x->n;
  QRPlan px = plan_tsqr(ctx, m, R);
  QRPlan py = plan_tsqr(ctx, n, R);
  tsqr_factor(ctx, px, x->X, m);
  tsqr_factor(ctx, py, x->Yt, n);
  double* A = ctx->alloc(size_t(R * R));
  double* B = ctx->alloc(size_t(R * R));
  double* sig = ctx->alloc(size_t(R + 4));
  double* info = sig + R;
  launch_svd_small(ctx, px.levels.back().Rst, py.levels.back().Rst, R, eps, A, B, sig, info);
  TTSW_CUDA(cudaMemcpyAsync(ctx->pinned, info, 4 * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  ctx->sync();
  const double* hinfo = static_cast<double*>(ctx->pinned);
  const double margin = hinfo[1];
  const double kappa = hinfo[3];
  const Index k = numerically_zero(R, kappa) ? 0 : Index(hinfo[0]);
  TT out;
  if (k == 0) {
    out = tt_zero(ctx, m, n);
  } else {
    auto t = make_tt(ctx, m, n, k);
    tsqr_apply(ctx, px, A, R, int(k), t->X, m);
    tsqr_apply(ctx, py, B, R, int(k), t->Yt, n);
    out = t;
  }
  ctx->free(A);
  ctx->free(B);
  ctx->free(sig);
  free_tsqr(ctx, px);
  free_tsqr(ctx, py);
  RoundRecord r{m, n, R, out->r, k == 0 ? INFINITY : margin, k == 0 ? INFINITY : kappa, ctx->cross_calls};
  if (rec) *rec = r;
  return out;
}

static bool caqr_eligible(const DevTT& x) {
  return x.r >= kCaqrMinR && caqr_fits(x.m, x.r) && caqr_fits(x.n, x.r);
}

/// Large roundings on the CAQR path, several at once: the X and Y cores of every input
/// are factored panel by panel in the same launches, the SVDs run as one batch, one host
/// sync reads all truncation ranks, and the Q applies share launches again.
static void round_caqr_group(const std::vector<TT>& xin, const std::vector<double>& eps, std::vector<TT>& out,
                             std::vector<RoundRecord>& rec) {
  HostRegion hr_(xin[0]->ctx, "round_caqr_group");
  const size_t nb = xin.size();
  // dims only: lazy inputs are gathered straight into the CAQR working panels below
  const std::vector<TT>& xs = xin;
  Context* ctx = xs[0]->ctx;
  static const bool prof_on = std::getenv("TTSW_PROFILE_TSQR") != nullptr;
  cudaEvent_t pev[4];
  auto mark = [&](int i) {
    if (prof_on) TTSW_CUDA(cudaEventRecord(pev[i], ctx->stream));
  };
  if (prof_on)
    for (auto& e : pev) TTSW_CUDA(cudaEventCreate(&e));
  mark(0);
  std::vector<CaqrFactor> f(2 * nb);
  std::vector<CaqrFactor*> fp;
  std::vector<size_t> lazy;  // inputs gathered in one batched launch
  for (size_t i = 0; i < nb; ++i) {
    const DevTT& x = *xs[i];
    CaqrFactor& fx = f[2 * i];
    CaqrFactor& fy = f[2 * i + 1];
    fx.rows = fx.lda = x.m;
    fy.rows = fy.lda = x.n;
    fx.R = fy.R = int(x.r);
    fx.A = ctx->alloc(size_t(x.m * x.r));
    fy.A = ctx->alloc(size_t(x.n * x.r));
    const TT src = x.materialised() ? xs[i] : x.cache;
    if (src) {  // factored in place: work on a copy
      TTSW_CUDA(cudaMemcpyAsync(fx.A, src->X, sizeof(double) * size_t(x.m * x.r), cudaMemcpyDeviceToDevice,
                                ctx->stream));
      TTSW_CUDA(cudaMemcpyAsync(fy.A, src->Yt, sizeof(double) * size_t(x.n * x.r), cudaMemcpyDeviceToDevice,
                                ctx->stream));
    } else {  // lazy term list evaluated directly into the working panels (no extra copy)
      lazy.push_back(i);
    }
    fp.push_back(&fx);
    fp.push_back(&fy);
  }
  if (!lazy.empty()) {
    // all lazy inputs of the group in one gather launch (descriptors in one upload)
    std::vector<TermDesc> all;
    std::vector<size_t> off;
    int max_terms = 0;
    Index max_elems = 0;
    for (size_t i : lazy) {
      off.push_back(all.size());
      auto d = term_descs(*xs[i]);
      max_terms = std::max(max_terms, int(d.size()));
      all.insert(all.end(), d.begin(), d.end());
      max_elems = std::max(max_elems, 2 * xs[i]->r);  // panel columns (X and Yt)
    }
    const size_t td = (sizeof(TermDesc) * all.size() + 255) / 256 * 256;
    std::vector<char> hbuf(td + sizeof(RoundJob) * lazy.size());
    char* dbuf = reinterpret_cast<char*>(ctx->alloc((hbuf.size() + 7) / 8));
    std::vector<RoundJob> jobs(lazy.size());
    for (size_t q = 0; q < lazy.size(); ++q) {
      const DevTT& x = *xs[lazy[q]];
      RoundJob J{};
      J.terms = reinterpret_cast<const TermDesc*>(dbuf) + off[q];
      J.nterms = int((q + 1 < lazy.size() ? off[q + 1] : all.size()) - off[q]);
      J.m = x.m;
      J.n = x.n;
      J.R = int(x.r);
      J.Xs = f[2 * lazy[q]].A;
      J.Ys = f[2 * lazy[q] + 1].A;
      jobs[q] = J;
    }
    std::memcpy(hbuf.data(), all.data(), sizeof(TermDesc) * all.size());
    std::memcpy(hbuf.data() + td, jobs.data(), sizeof(RoundJob) * jobs.size());
    // pageable source: the upload is complete when the call returns
    TTSW_CUDA(cudaMemcpyAsync(dbuf, hbuf.data(), hbuf.size(), cudaMemcpyHostToDevice, ctx->stream));
    const MapDesc* maps = static_cast<const MapDesc*>(ctx->device_maps());
    launch_gather_jobs(ctx, reinterpret_cast<const RoundJob*>(dbuf + td), int(lazy.size()), max_elems, maps,
                       int(ctx->map_keys.size()), max_terms);
    ctx->free(reinterpret_cast<double*>(dbuf));
  }
  // ---- sketched pre-compression (sketch.cu) of the members whose rank dwarfs the expected
  // output rank: the range of M = X Yt^T from a Gaussian sketch, the rounding continues on
  // the rank-l TT (Qz, Bt) with the uncaptured energy as hidden tail energy. A member whose
  // probes show too much uncaptured energy retries with a wider sketch while that is still
  // cheaper than factoring both cores (2 L <= R), then falls back to the two-core path -----
  constexpr int q = kSketchProbes;
  constexpr int kInfo = 6;  // k, margin, sweeps, kappa, ambiguous, ||S||^2 (the last two: sketched members)
  const int nchunk = 64;
  static const bool verbose = std::getenv("TTSW_SKETCH_VERBOSE") != nullptr;
  auto round32 = [](double v) { return (int(v) + 31) / 32 * 32; };
  struct Sketch {
    int l = 0, L = 0;
    double *G = nullptr, *Z = nullptr, *Qz = nullptr, *Id = nullptr, *Ct = nullptr, *Bt = nullptr, *probe = nullptr;
    CaqrFactor fz, fb;
  };
  struct Member {
    int L = 0;          // sketch columns of the current attempt (0: both cores are factored)
    bool done = false, accepted = false, factored = false;
    int attempts = 0;
    Sketch s;
    double *Aw = nullptr, *Bw = nullptr, *sig = nullptr;
    int Rs = 0;         // rank the SVD works at
    double kappa = 0, ratio = 0;
    size_t key = SIZE_MAX;
  };
  std::vector<Member> mem(nb);
  for (size_t i = 0; i < nb; ++i) {
    Member& M = mem[i];
    const int R = int(xs[i]->r);
    if (ctx->hint_active) {
      M.key = ctx->hint_pos++;
      if (ctx->sketch_hint.size() <= M.key) ctx->sketch_hint.resize(M.key + 1);
    }
    if (!ctx->sketch_on || R < ctx->sketch_min_r || eps[i] <= 0.0) continue;
    int L = ctx->sketch_default_l;
    if (M.key != SIZE_MAX && ctx->sketch_hint[M.key].k >= 0) {
      const SketchHint& h = ctx->sketch_hint[M.key];
      const int floor_l = round32(1.25 * h.k + 16 + q);
      if (h.L > 0)  // the width that captured this call site last time, narrowed when it had margin to spare
        L = std::max(floor_l, h.spare && h.L - 32 > h.fail ? h.L - 32 : h.L);
      else
        L = floor_l;
      if (L <= h.fail) L = h.fail + 32;
    }
    L = std::max(L, 64);
    if (2 * L > R) continue;  // too little to gain over factoring both cores
    M.L = L;
  }
  auto free_sketch = [&](Sketch& s) {
    for (double* pbuf : {s.G, s.Z, s.Qz, s.Id, s.Ct, s.Bt, s.probe})
      if (pbuf) ctx->free(pbuf);
    caqr_free(ctx, s.fz);
    caqr_free(ctx, s.fb);
    s = Sketch{};
  };
  double* hinfo = static_cast<double*>(ctx->pinned);
  bool first_attempt = true;
  for (;;) {
    std::vector<size_t> pend, skm;
    for (size_t i = 0; i < nb; ++i)
      if (!mem[i].done) {
        pend.push_back(i);
        if (mem[i].L > 0) skm.push_back(i);
      }
    if (pend.empty()) break;
    double* sumsq_part = nullptr;
    if (!skm.empty()) {
      HostRegion hs_(ctx, "round_sketch");
      Index maxn = 0;
      int maxL = 0;
      for (size_t i : skm) {
        maxn = std::max(maxn, xs[i]->n);
        maxL = std::max(maxL, mem[i].L);
      }
      const double* Om = sketch_omega(ctx, maxn, maxL);
      std::vector<SumsqJob> sq;
      std::vector<GemmJob> g1, g2, g3, g4;
      std::vector<CaqrFactor*> fzs;
      std::vector<ProbeJob> pj;
      std::vector<const double*> Wi;
      std::vector<Index> ldwi, ldoi;
      std::vector<int> ki;
      std::vector<double*> qo;
      for (size_t i : skm) {
        const DevTT& x = *xs[i];
        Sketch& sk = mem[i].s;
        const int R = int(x.r);
        sk.L = mem[i].L;
        sk.l = sk.L - q;
        sk.G = ctx->alloc(size_t(R) * sk.L);
        sk.Z = ctx->alloc(size_t(x.m) * sk.L);
        sk.Qz = ctx->alloc(size_t(x.m) * sk.l);
        sk.Id = ctx->alloc(size_t(sk.l) * sk.l);
        sk.Ct = ctx->alloc(size_t(R) * sk.l);
        sk.Bt = ctx->alloc(size_t(x.n) * sk.l);
        sk.probe = ctx->alloc(2);
        sq.push_back({f[2 * i].A, x.m * x.r});
        sq.push_back({f[2 * i + 1].A, x.n * x.r});
        // G = Yt^T Omega (R x L), Z = X G (m x L), Ct = X^T Qz (R x l), Bt = Yt Ct (n x l)
        g1.push_back(GemmJob{f[2 * i + 1].A, x.n, Om, kSketchOmegaLd, sk.G, Index(R), R, sk.L, int(x.n)});
        g2.push_back(GemmJob{f[2 * i].A, x.m, sk.G, Index(R), sk.Z, x.m, int(x.m), sk.L, R});
        g3.push_back(GemmJob{f[2 * i].A, x.m, sk.Qz, x.m, sk.Ct, Index(R), R, sk.l, int(x.m)});
        g4.push_back(GemmJob{f[2 * i + 1].A, x.n, sk.Ct, Index(R), sk.Bt, x.n, int(x.n), sk.l, R});
        sk.fz.A = sk.Z;
        sk.fz.rows = sk.fz.lda = x.m;
        sk.fz.R = sk.l;
        sk.fz.extra = q;
        sk.fb.A = sk.Bt;
        sk.fb.rows = sk.fb.lda = x.n;
        sk.fb.R = sk.l;
        fzs.push_back(&sk.fz);
        pj.push_back(ProbeJob{sk.Z + Index(sk.l) * x.m, x.m, x.m, sk.l, q, sk.probe});
        launch_fill_identity(ctx, sk.Id, sk.l);
        Wi.push_back(sk.Id);
        ldwi.push_back(sk.l);
        ki.push_back(sk.l);
        qo.push_back(sk.Qz);
        ldoi.push_back(x.m);
      }
      sumsq_part = ctx->alloc(sq.size() * size_t(nchunk));
      launch_sumsq_batch(ctx, sq, nchunk, sumsq_part);
      launch_gemm_batch(ctx, g1, true);
      launch_gemm_batch(ctx, g2, false);
      caqr_factor(ctx, fzs);
      launch_probe_energy(ctx, pj);
      caqr_apply(ctx, fzs, Wi, ldwi, ki, qo, ldoi);
      launch_gemm_batch(ctx, g3, true);
      launch_gemm_batch(ctx, g4, false);
    }
    // factorisations: Bt of the sketched members, both cores of the others
    std::vector<CaqrFactor*> fall;
    for (size_t i : pend)
      if (mem[i].L > 0) {
        fall.push_back(&mem[i].s.fb);
      } else {
        fall.push_back(&f[2 * i]);
        fall.push_back(&f[2 * i + 1]);
        mem[i].factored = true;
      }
    caqr_factor(ctx, fall);
    if (first_attempt) mark(1);
    std::vector<SvdRequest> reqs;
    for (size_t i : pend) {
      Member& M = mem[i];
      const Index R = M.L > 0 ? Index(M.s.l) : xs[i]->r;
      M.Rs = int(R);
      for (double* pbuf : {M.Aw, M.Bw, M.sig})
        if (pbuf) ctx->free(pbuf);
      M.Aw = ctx->alloc(size_t(R * R));
      M.Bw = ctx->alloc(size_t(R * R));
      M.sig = ctx->alloc(size_t(R + 8));
      SvdRequest rq{M.L > 0 ? M.s.Id : f[2 * i].Rout, M.L > 0 ? M.s.fb.Rout : f[2 * i + 1].Rout, R, eps[i], M.Aw, M.Bw,
                    M.sig, M.sig + R};
      rq.hidden_rel = M.L > 0 ? M.s.probe : nullptr;
      reqs.push_back(rq);
    }
    launch_svd_batch(ctx, reqs);
    for (size_t i : pend)
      TTSW_CUDA(cudaMemcpyAsync(hinfo + kInfo * i, mem[i].sig + mem[i].Rs, kInfo * sizeof(double),
                                cudaMemcpyDeviceToHost, ctx->stream));
    double* hprobe = hinfo + kInfo * nb;          // 2 per sketched member
    double* hsumsq = hprobe + 2 * skm.size();     // nchunk per panel, 2 panels per sketched member
    for (size_t qi = 0; qi < skm.size(); ++qi)
      TTSW_CUDA(cudaMemcpyAsync(hprobe + 2 * qi, mem[skm[qi]].s.probe, 2 * sizeof(double), cudaMemcpyDeviceToHost,
                                ctx->stream));
    if (!skm.empty())
      TTSW_CUDA(cudaMemcpyAsync(hsumsq, sumsq_part, sizeof(double) * 2 * skm.size() * nchunk, cudaMemcpyDeviceToHost,
                                ctx->stream));
    if (first_attempt) mark(2);
    first_attempt = false;
    ctx->sync();
    if (sumsq_part) ctx->free(sumsq_part);
    // A sketch is accepted when 4 x the probes' uncaptured fraction is below 1e-3 of the
    // truncation budget (the first stop level of the pivoted-QR pre-truncation) and the rank
    // decision does not depend on it.
    for (size_t qi = 0; qi < skm.size(); ++qi) {
      const size_t i = skm[qi];
      Member& M = mem[i];
      const int R = int(xs[i]->r);
      const double e9 = 0.9 * eps[i];
      const double thr = std::min(1e-3 * e9 * e9, 9e-24);
      M.ratio = hprobe[2 * qi];
      const bool ambiguous = hinfo[kInfo * i + 4] != 0.0;
      double nx2 = 0.0, ny2 = 0.0;
      for (int c = 0; c < nchunk; ++c) {
        nx2 += hsumsq[(2 * qi) * nchunk + c];
        ny2 += hsumsq[(2 * qi + 1) * nchunk + c];
      }
      const double total2 = hinfo[kInfo * i + 5];
      M.kappa = total2 > 0 ? std::sqrt(nx2) * std::sqrt(ny2) / std::sqrt(total2) : INFINITY;
      const int kobs = int(hinfo[kInfo * i]);
      M.attempts++;
      const bool ok = std::isfinite(M.ratio) && 4.0 * M.ratio <= thr && !ambiguous;
      if (verbose)
        std::fprintf(stderr, "sketch R=%d l=%d ratio=%.3e thr=%.3e ambiguous=%d k=%d kappa=%.3e attempt=%d %s\n", R,
                     M.s.l, M.ratio, thr, int(ambiguous), kobs, M.kappa, M.attempts, ok ? "ok" : "retry");
      if (ok) {
        M.accepted = true;
        M.done = true;
        ctx->sketch_used++;
        continue;
      }
      ctx->sketch_fallback++;
      // wider sketch while it still pays (a noise-level input has no low-rank range: kappa says so)
      // captured well enough but the rank decision is a near tie on the hidden energy: a
      // wider sketch shrinks it by orders of magnitude, and the two-core path would only hit
      // the same tie in its pivoted-QR pre-truncation (slow second pass at this size)
      const bool tie = ambiguous && std::isfinite(M.ratio) && 4.0 * M.ratio <= thr;
      const bool near = 4.0 * M.ratio <= 1e3 * thr && !ambiguous;
      const int Lnext = round32(std::max(tie ? M.L + 64.0 : (near ? M.L + 32.0 : 1.5 * M.L + 32.0), 1.25 * kobs + 16.0 + q));
      if (M.key != SIZE_MAX && !tie) ctx->sketch_hint[M.key].fail = std::max(ctx->sketch_hint[M.key].fail, M.L);
      free_sketch(M.s);
      const bool feasible = tie ? 4 * Lnext <= 3 * R : 2 * Lnext <= R;
      if (M.attempts < (tie ? 5 : 3) && feasible && !numerically_zero(R, M.kappa))
        M.L = Lnext;
      else
        M.L = 0;
    }
    for (size_t i : pend)
      if (mem[i].L == 0 && mem[i].factored) mem[i].done = true;
  }
  std::vector<CaqrFactor*> fap;
  std::vector<const double*> W;
  std::vector<Index> ldw, ldo;
  std::vector<int> ks;
  std::vector<double*> dst;
  for (size_t i = 0; i < nb; ++i) {
    const DevTT& x = *xs[i];
    Member& M = mem[i];
    const double margin = hinfo[kInfo * i + 1];
    const double kappa = M.accepted ? M.kappa : hinfo[kInfo * i + 3];
    const Index k = numerically_zero(x.r, kappa) ? 0 : Index(hinfo[kInfo * i]);
    double* ox = nullptr;
    double* oy = nullptr;
    if (k == 0) {
      out[i] = tt_zero(ctx, x.m, x.n);
    } else {
      auto t = make_tt(ctx, x.m, x.n, k);
      ox = t->X;
      oy = t->Yt;
      out[i] = t;
    }
    if (M.accepted)
      fap.insert(fap.end(), {&M.s.fz, &M.s.fb});
    else
      fap.insert(fap.end(), {&f[2 * i], &f[2 * i + 1]});
    W.insert(W.end(), {M.Aw, M.Bw});
    ldw.insert(ldw.end(), {Index(M.Rs), Index(M.Rs)});
    ks.insert(ks.end(), {int(k), int(k)});
    dst.insert(dst.end(), {ox, oy});
    ldo.insert(ldo.end(), {x.m, x.n});
    rec[i] = RoundRecord{x.m, x.n, x.r, out[i]->r, k == 0 ? INFINITY : margin, k == 0 ? INFINITY : kappa,
                         ctx->cross_calls};
    if (M.key != SIZE_MAX) {
      SketchHint& h = ctx->sketch_hint[M.key];
      h.k = int(out[i]->r);
      h.L = M.accepted ? M.s.L : 0;
      const double e9 = 0.9 * eps[i];
      const double thr_h = std::min(1e-3 * e9 * e9, 9e-24);
      h.spare = M.accepted && 4.0 * M.ratio <= 1e-4 * thr_h;
      // close to the limit: the ranks of a run grow, so the next sketch here is a panel wider
      if (M.accepted && 4.0 * M.ratio > 0.1 * thr_h && 2 * (h.L + 32) <= int(x.r)) h.L += 32;
    }
  }
  caqr_apply(ctx, fap, W, ldw, ks, dst, ldo);
  mark(3);
  if (prof_on) {
    TTSW_CUDA(cudaStreamSynchronize(ctx->stream));
    float t[3] = {0, 0, 0};
    for (int i = 0; i < 3; ++i) TTSW_CUDA(cudaEventElapsedTime(&t[i], pev[i], pev[i + 1]));
    for (size_t i = 0; i < nb; ++i)
      std::fprintf(stderr, "caqr group %zu/%zu m=%ld n=%ld R=%ld k=%ld sketch=%d ms: qr %.3f svd %.3f apply %.3f\n", i,
                   nb, long(xs[i]->m), long(xs[i]->n), long(xs[i]->r), long(out[i]->r),
                   mem[i].accepted ? mem[i].Rs : -mem[i].attempts, t[0] / nb, t[1] / nb, t[2] / nb);
    for (auto& e : pev) TTSW_CUDA(cudaEventDestroy(e));
  }
  for (auto& M : mem) {
    for (double* pbuf : {M.Aw, M.Bw, M.sig})
      if (pbuf) ctx->free(pbuf);
    free_sketch(M.s);
  }
  for (auto& g : f) {
    ctx->free(g.A);
    caqr_free(ctx, g);
  }
}

static void account_round(Context* ctx, Index m_, Index n_, Index R, Index k) {
  // round flops 2nR^2 + 3mR^2 + 2(m+n)Rk + 11R^3 (fixed convention),
  // bytes 8(m+n)(R+k).
  const double m = double(m_), n = double(n_), Rd = double(R), kd = double(k);
  ctx->round_flops += 2 * n * Rd * Rd + 3 * m * Rd * Rd + 2 * (m + n) * Rd * kd + 11 * Rd * Rd * Rd;
  ctx->round_bytes += 8 * (m + n) * (Rd + kd);
  ctx->round_count++;
}

static bool fused_fits(const Context* ctx, Index m, Index n, Index R) {
  return m >= R && n >= R && fused_round_smem(m, n, R) + 4096 <= ctx->smem_optin;
}

/// Batched rounding (independent inputs): every input that fits runs in one fused
/// single-CTA kernel launch (one CTA per rounding); the rest take the TSQR path.
/// Records are emitted in input order.
std::vector<TT> round_batch(const std::vector<TT>& xs, const std::vector<double>& eps,
                            std::vector<RoundRecord>* recs) {
  HostRegion hr_(xs.empty() ? nullptr : xs[0]->ctx, "round_batch");
  std::vector<TT> out(xs.size());
  if (xs.empty()) return out;
  Context* ctx = xs[0]->ctx;
  std::vector<RoundRecord> rr(xs.size());
  std::vector<size_t> fused;
  size_t smem = 0;
  std::vector<size_t> large;
  for (size_t i = 0; i < xs.size(); ++i) {
    if (eps[i] < 0) throw InputError("round: eps must be non-negative");
    const DevTT& x = *xs[i];
    if (small_round_fits(ctx, x.m, x.n, x.r) || fused_fits(ctx, x.m, x.n, x.r)) {
      fused.push_back(i);
    } else if (caqr_eligible(x)) {
      large.push_back(i);
    } else {
      if (ctx->time_rounds) TTSW_CUDA(cudaEventRecord(ctx->ev0, ctx->stream));
      out[i] = round_tsqr(xs[i], eps[i], &rr[i]);
      if (ctx->time_rounds) {
        TTSW_CUDA(cudaEventRecord(ctx->ev1, ctx->stream));
        TTSW_CUDA(cudaEventSynchronize(ctx->ev1));
        float ms = 0;
        TTSW_CUDA(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
        ctx->round_ms += ms;
        account_round(ctx, x.m, x.n, x.r, out[i]->r);
      }
    }
  }
  // CAQR roundings in groups of up to kCaqrMaxProbs / 2 (two cores each)
  for (size_t g0 = 0; g0 < large.size(); g0 += kCaqrMaxProbs / 2) {
    const size_t g1 = std::min(large.size(), g0 + kCaqrMaxProbs / 2);
    std::vector<TT> gx;
    std::vector<double> ge;
    for (size_t q = g0; q < g1; ++q) {
      gx.push_back(xs[large[q]]);
      ge.push_back(eps[large[q]]);
    }
    std::vector<TT> go(gx.size());
    std::vector<RoundRecord> gr(gx.size());
    if (ctx->time_rounds) TTSW_CUDA(cudaEventRecord(ctx->ev0, ctx->stream));
    round_caqr_group(gx, ge, go, gr);
    if (ctx->time_rounds) {
      TTSW_CUDA(cudaEventRecord(ctx->ev1, ctx->stream));
      TTSW_CUDA(cudaEventSynchronize(ctx->ev1));
      float ms = 0;
      TTSW_CUDA(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
      ctx->round_ms += ms;
    }
    for (size_t q = g0; q < g1; ++q) {
      out[large[q]] = go[q - g0];
      rr[large[q]] = gr[q - g0];
      if (ctx->time_rounds) account_round(ctx, xs[large[q]]->m, xs[large[q]]->n, xs[large[q]]->r, go[q - g0]->r);
    }
  }
  if (!fused.empty()) {
    std::vector<TermDesc> all;
    std::vector<size_t> off;
    for (size_t i : fused) {
      off.push_back(all.size());
      auto d = term_descs(*xs[i]);
      all.insert(all.end(), d.begin(), d.end());
    }
    const MapDesc* maps = static_cast<const MapDesc*>(ctx->device_maps());
    // one kernel variant per batch: the row-parallel small kernel when every job fits it
    bool small = true;
    Index rmax = 0, nmax = 0, elems = 0;
    for (size_t i : fused) {
      const DevTT& x = *xs[i];
      small = small && small_round_fits(ctx, x.m, x.n, x.r);
      rmax = std::max(rmax, x.r);
      nmax = std::max({nmax, x.m, x.n});
      elems = std::max(elems, (x.m + x.n) * x.r);
    }
    const int rm = rmax <= 8 ? 8 : 16, rows = nmax <= 512 ? 1 : 2;
    if (small)
      for (size_t i : fused) smem = std::max(smem, small_round_smem(xs[i]->m, xs[i]->n, xs[i]->r, rm));
    else
      for (size_t i : fused) {
        if (!fused_fits(ctx, xs[i]->m, xs[i]->n, xs[i]->r)) small = true;  // never: fits checked above
        smem = std::max(smem, fused_round_smem(xs[i]->m, xs[i]->n, xs[i]->r));
      }
    size_t ws = 0;
    for (size_t i : fused) ws += size_t(2 * xs[i]->r * xs[i]->r + xs[i]->r + (small ? (xs[i]->m + xs[i]->n) * xs[i]->r : 0));
    const size_t nj = fused.size();
    double* dws = ctx->ensure_work(ws + 4 * nj);
    double* dinfo = dws + ws;
    const size_t td_bytes = (sizeof(TermDesc) * all.size() + 255) / 256 * 256;
    const size_t stage_bytes = td_bytes + sizeof(RoundJob) * nj + sizeof(double) * 4 * nj + 256;
    ctx->ensure_stage(stage_bytes);
    char* hst = static_cast<char*>(ctx->stage_host);
    char* dst = static_cast<char*>(ctx->stage_dev);
    TermDesc* dd = reinterpret_cast<TermDesc*>(dst);
    RoundJob* dj = reinterpret_cast<RoundJob*>(dst + td_bytes);
    double* hinfo = reinterpret_cast<double*>(hst + td_bytes + (sizeof(RoundJob) * nj + 255) / 256 * 256);
    std::vector<RoundJob> jobs;
    std::vector<Buf> xb, yb;
    double* w = dws;
    for (size_t j = 0; j < nj; ++j) {
      const DevTT& x = *xs[fused[j]];
      xb.push_back(std::make_shared<DBuf>(ctx, size_t(x.m * x.r)));
      yb.push_back(std::make_shared<DBuf>(ctx, size_t(x.n * x.r)));
      RoundJob J{};
      J.terms = dd + off[j];
      J.nterms = int(x.terms.size());
      J.m = x.m;
      J.n = x.n;
      J.R = int(x.r);
      J.eps = eps[fused[j]];
      J.Xout = xb.back()->p;
      J.Ytout = yb.back()->p;
      J.A = w;
      J.B = w + x.r * x.r;
      J.sigma = w + 2 * x.r * x.r;
      J.info = dinfo + 4 * j;
      w += 2 * x.r * x.r + x.r;
      if (small) {
        J.Xs = w;
        J.Ys = w + x.m * x.r;
        w += (x.m + x.n) * x.r;
      }
      jobs.push_back(J);
    }
    std::memcpy(hst, all.data(), sizeof(TermDesc) * all.size());
    std::memcpy(hst + td_bytes, jobs.data(), sizeof(RoundJob) * nj);
    TTSW_CUDA(cudaMemcpyAsync(dst, hst, td_bytes + sizeof(RoundJob) * nj, cudaMemcpyHostToDevice, ctx->stream));
    if (ctx->time_rounds) TTSW_CUDA(cudaEventRecord(ctx->ev0, ctx->stream));
    int max_terms = 0;
    for (size_t i : fused) max_terms = std::max(max_terms, int(xs[i]->terms.size()));
    static const bool prof_on = std::getenv("TTSW_PROFILE_ROUND") != nullptr;
    long long* dprof = nullptr;
    if (prof_on && small) {
      dprof = reinterpret_cast<long long*>(ctx->alloc(8 * nj));
      TTSW_CUDA(cudaMemsetAsync(dprof, 0, 64 * nj, ctx->stream));
      for (size_t j = 0; j < nj; ++j) jobs[j].prof = dprof + 8 * j;
      std::memcpy(hst + td_bytes, jobs.data(), sizeof(RoundJob) * nj);
      TTSW_CUDA(cudaMemcpyAsync(dst, hst, td_bytes + sizeof(RoundJob) * nj, cudaMemcpyHostToDevice, ctx->stream));
    }
    if (small)
      launch_round_small(ctx, dj, int(nj), elems, maps, int(ctx->map_keys.size()), max_terms, rm, rows, smem);
    else
      launch_round_fused(ctx, dj, int(nj), maps, smem);
    if (ctx->time_rounds) TTSW_CUDA(cudaEventRecord(ctx->ev1, ctx->stream));
    TTSW_CUDA(cudaMemcpyAsync(hinfo, dinfo, sizeof(double) * 4 * nj, cudaMemcpyDeviceToHost, ctx->stream));
    ctx->sync();
    const double* info = hinfo;
    if (dprof) {
      std::vector<long long> pr(8 * nj);
      TTSW_CUDA(cudaMemcpy(pr.data(), dprof, 64 * nj, cudaMemcpyDeviceToHost));
      for (size_t j = 0; j < nj; ++j)
        std::fprintf(stderr, "round_small R=%lld k=%lld sweeps=%lld cycles: copy %lld qr %lld svd %lld apply %lld\n",
                     pr[8 * j + 6], pr[8 * j + 5], pr[8 * j + 7], pr[8 * j + 1] - pr[8 * j], pr[8 * j + 2] - pr[8 * j + 1],
                     pr[8 * j + 3] - pr[8 * j + 2], pr[8 * j + 4] - pr[8 * j + 3]);
      ctx->free(dprof);
    }
    if (ctx->time_rounds) {
      float ms = 0;
      TTSW_CUDA(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
      ctx->round_ms += ms;
    }
    for (size_t j = 0; j < nj; ++j) {
      const size_t i = fused[j];
      const DevTT& x = *xs[i];
      const Index k = numerically_zero(x.r, info[4 * j + 3]) ? 0 : Index(info[4 * j]);
      out[i] = k == 0 ? tt_zero(ctx, x.m, x.n) : std::make_shared<DevTT>(ctx, x.m, x.n, k, xb[j], yb[j]);
      rr[i] = RoundRecord{x.m, x.n, x.r, out[i]->r, k == 0 ? INFINITY : info[4 * j + 1],
                          k == 0 ? INFINITY : info[4 * j + 3], ctx->cross_calls};
      if (ctx->time_rounds) account_round(ctx, x.m, x.n, x.r, out[i]->r);
    }
  }
  for (size_t i = 0; i < xs.size(); ++i) {
    if (ctx->trace) ctx->trace->push_back(rr[i]);
    if (recs) recs->push_back(rr[i]);
  }
  return out;
}

/// round (tt.hpp:120-138).
TT round(const TT& x, double eps, RoundRecord* rec) {
  std::vector<RoundRecord> recs;
  TT out = round_batch({x}, {eps}, &recs)[0];
  if (rec) *rec = recs[0];
  return out;
}

/// apply_core_map (tt.hpp:185-194) with a banded operator: appended lazily to the
/// mapped side of every term (the other core is shared untouched).
TT apply_core_map(const TT& x, Axis axis, const BandMap& m, double scale_x) {
  HostRegion hr_(x->ctx, "apply_core_map");
  Context* ctx = x->ctx;
  if ((axis == Axis::X ? x->m : x->n) != m.n_in) throw ShapeError("apply_core_map: operator/mode size mismatch");
  const int id = ctx->register_map(m);
  std::vector<HostTerm> terms = x->terms;
  for (auto& t : terms) {
    // an exactly-zero constant side stays zero under any linear map (sum of c * 0)
    if (t.kind == TERM_CONST && (axis == Axis::X ? t.cx : t.cy) == 0.0) continue;
    if (t.kind == TERM_CONST) {  // materialise the constant side before mapping it
      HostTerm p;
      p.kind = TERM_PLAIN;
      p.r = 1;
      auto xb = std::make_shared<DBuf>(ctx, size_t(x->m));
      auto yb = std::make_shared<DBuf>(ctx, size_t(x->n));
      launch_fill(ctx, xb->p, x->m, t.cx);
      launch_fill(ctx, yb->p, x->n, t.cy);
      p.x.base = xb;
      p.x.ld = x->m;
      p.y.base = yb;
      p.y.ld = x->n;
      t = std::move(p);
    }
    (axis == Axis::X ? t.x : t.y).ops.push_back({1, id, 0.0});
    if (scale_x != 1.0) t.x.ops.push_back({0, 0, scale_x});
  }
  return std::make_shared<DevTT>(ctx, axis == Axis::X ? m.n_out : x->m, axis == Axis::X ? x->n : m.n_out,
                                 std::move(terms));
}

/// reciprocal_taylor (tt.hpp:204-241).
std::vector<TT> round_batch_into(const std::vector<TT>& xs, const std::vector<double>& eps,
                                 const std::vector<RoundRecord*>& dst) {
  if (xs.empty()) return {};
  Context* ctx = xs[0]->ctx;
  std::vector<RoundRecord>* saved = ctx->trace;
  ctx->trace = nullptr;
  std::vector<RoundRecord> recs;
  std::vector<TT> out;
  try {
    out = round_batch(xs, eps, &recs);
  } catch (...) {
    ctx->trace = saved;
    throw;
  }
  ctx->trace = saved;
  for (size_t i = 0; i < xs.size() && i < dst.size(); ++i)
    if (dst[i]) *dst[i] = recs[i];
  return out;
}

std::vector<TT> reciprocal_taylor_batch(const std::vector<TT>& xs, double eps,
                                        const std::vector<std::vector<RoundRecord>*>& sinks, int max_iterations) {
  if (eps <= 0) throw InputError("reciprocal_taylor: eps must be positive");
  const size_t ns = xs.size();
  std::vector<TT> result(ns);
  if (ns == 0) return result;
  Context* ctx = xs[0]->ctx;
  std::vector<double> n_entries(ns), x_avg(ns), prev_err(ns, INFINITY);
  std::vector<int> growth(ns, 0);
  std::vector<std::string> fail_msg(ns);
  std::vector<double> fail_err(ns, 0.0);
  std::vector<int> fail_it(ns, -1);
  std::vector<TT> ones(ns), xt(ns), y(ns), dy(ns);
  std::vector<size_t> active;
  auto fail = [&](size_t s, const char* reason, double err, int it) {
    std::ostringstream os;
    os << "reciprocal_taylor: " << reason << " after " << it << " iterations (residual = " << err << ")";
    fail_msg[s] = os.str();
    fail_err[s] = err;
    fail_it[s] = it;
  };
  // one record slot per rounding of side s, appended in that side's own order
  auto round_active = [&](const std::vector<TT>& in) {
    std::vector<RoundRecord> recs(in.size());
    std::vector<RoundRecord*> dst(in.size());
    for (size_t q = 0; q < in.size(); ++q) dst[q] = &recs[q];
    auto out = round_batch_into(in, std::vector<double>(in.size(), eps), dst);
    for (size_t q = 0; q < in.size(); ++q)
      if (sinks.size() > active[q] && sinks[active[q]] && ctx->trace) sinks[active[q]]->push_back(recs[q]);
    return out;
  };
  for (size_t s = 0; s < ns; ++s) {
    n_entries[s] = double(xs[s]->m) * double(xs[s]->n);
    x_avg[s] = sum_entries(xs[s]) / n_entries[s];
    if (x_avg[s] == 0.0) {
      fail_msg[s] = "reciprocal_taylor: field has zero mean";
      fail_err[s] = 1.0;
      fail_it[s] = 0;
      continue;
    }
    ones[s] = tt_constant(ctx, xs[s]->m, xs[s]->n, 1.0);
    active.push_back(s);
  }
  {
    std::vector<TT> in;
    for (size_t s : active) in.push_back(add_scaled(1.0, ones[s], -1.0 / x_avg[s], xs[s]));
    auto out = round_active(in);
    for (size_t q = 0; q < active.size(); ++q) {
      xt[active[q]] = out[q];
      y[active[q]] = dy[active[q]] = ones[active[q]];
    }
  }
  // Iteration it: dy_it = round(dy_{it-1} * xt), y_it = round(y_{it-1} + dy_it), stop on
  // RMS(dy_it) <= eps (tt.hpp:222-236). The stop test needs dy_it only and dy_{it+1} does
  // not need y_it, so y_it and dy_{it+1} of a continuing side share one batch (records in
  // the reference order: y_it, then dy_{it+1}); nothing is computed that the sequential
  // reference would not compute.
  if (!active.empty()) {
    std::vector<TT> in;
    for (size_t s : active) in.push_back(hadamard(dy[s], xt[s]));
    auto o = round_active(in);
    for (size_t q = 0; q < active.size(); ++q) dy[active[q]] = o[q];
  }
  for (int it = 1; it <= max_iterations && !active.empty(); ++it) {
    // stop rule of iteration it (one sync for all sides)
    std::vector<char> done(ns, 0), cont(ns, 0);
    std::vector<TT> dys;
    for (size_t s : active) dys.push_back(dy[s]);
    const std::vector<double> norms = norm_fro_batch(dys);
    size_t qn = 0;
    for (size_t s : active) {
      const double err = norms[qn++] / std::sqrt(n_entries[s]);
      if (err <= eps) {
        done[s] = 1;
        continue;
      }
      growth[s] = (err > prev_err[s]) ? growth[s] + 1 : 0;
      if (growth[s] >= 5) {
        fail(s, "diverging increments", err, it);
        done[s] = 2;
        continue;
      }
      prev_err[s] = err;
      if (it < max_iterations) cont[s] = 1;
      else done[s] = 3;
    }
    // batch: y_it for every active side (the reference computes it before the test), then
    // dy_{it+1} for the sides that continue; per side records y_it, dy_{it+1}
    std::vector<TT> in;
    std::vector<size_t> owner;
    for (size_t s : active) {
      in.push_back(add(y[s], dy[s]));
      owner.push_back(s);
      if (cont[s]) {
        in.push_back(hadamard(dy[s], xt[s]));
        owner.push_back(s);
      }
    }
    std::vector<RoundRecord> recs(in.size());
    std::vector<RoundRecord*> dst(in.size());
    for (size_t q = 0; q < in.size(); ++q) dst[q] = &recs[q];
    auto out = round_batch_into(in, std::vector<double>(in.size(), eps), dst);
    std::vector<size_t> next;
    for (size_t q = 0; q < in.size(); ++q) {
      const size_t s = owner[q];
      if (sinks.size() > s && sinks[s] && ctx->trace) sinks[s]->push_back(recs[q]);
      const bool is_y = (q == 0 || owner[q - 1] != s);
      if (is_y) {
        y[s] = out[q];
        if (done[s] == 1) result[s] = scale(y[s], 1.0 / x_avg[s]);
        if (cont[s]) next.push_back(s);
      } else {
        dy[s] = out[q];
      }
    }
    for (size_t s : active)
      if (done[s] == 3) fail(s, "iteration cap exceeded", prev_err[s], max_iterations);
    active.swap(next);
  }
  for (size_t s = 0; s < ns; ++s)  // the reference stops at the first failing side in order
    if (fail_it[s] >= 0) throw ConvergenceError(fail_msg[s], fail_err[s], fail_it[s]);
  return result;
}

TT reciprocal_taylor(const TT& x, double eps, int max_iterations, int* iterations) {
  if (eps <= 0) throw InputError("reciprocal_taylor: eps must be positive");
  Context* ctx = x->ctx;
  const double n_entries = double(x->m) * double(x->n);
  const double x_avg = sum_entries(x) / n_entries;
  if (x_avg == 0.0) throw ConvergenceError("reciprocal_taylor: field has zero mean", 1.0, 0);
  const TT ones = tt_constant(ctx, x->m, x->n, 1.0);
  const TT xt = round(add_scaled(1.0, ones, -1.0 / x_avg, x), eps);
  auto fail = [&](const char* reason, double err, int it) {
    std::ostringstream os;
    os << "reciprocal_taylor: " << reason << " after " << it << " iterations (residual = " << err << ")";
    return ConvergenceError(os.str(), err, it);
  };
  TT y = ones, dy = ones;
  double prev_err = INFINITY;
  int growth = 0;
  for (int it = 1; it <= max_iterations; ++it) {
    dy = round(hadamard(dy, xt), eps);
    y = round(add(y, dy), eps);
    const double err = norm_fro(dy) / std::sqrt(n_entries);
    if (iterations) *iterations = it;
    if (err <= eps) return scale(y, 1.0 / x_avg);
    growth = (err > prev_err) ? growth + 1 : 0;
    if (growth >= 5) throw fail("diverging increments", err, it);
    prev_err = err;
  }
  throw fail("iteration cap exceeded", prev_err, max_iterations);
}

// ---- reconstruction tables (reconstruction.hpp:33-171) -------------------------------

namespace {

std::vector<double> solve_dense(std::vector<double> a, std::vector<double> b, int n) {
  for (int k = 0; k < n; ++k) {
    int p = k;
    for (int i = k + 1; i < n; ++i)
      if (std::fabs(a[size_t(i + k * n)]) > std::fabs(a[size_t(p + k * n)])) p = i;
    if (p != k) {
      for (int j = 0; j < n; ++j) std::swap(a[size_t(k + j * n)], a[size_t(p + j * n)]);
      std::swap(b[size_t(k)], b[size_t(p)]);
    }
    for (int i = k + 1; i < n; ++i) {
      const double f = a[size_t(i + k * n)] / a[size_t(k + k * n)];
      for (int j = k; j < n; ++j) a[size_t(i + j * n)] -= f * a[size_t(k + j * n)];
      b[size_t(i)] -= f * b[size_t(k)];
    }
  }
  std::vector<double> x(size_t(n), 0.0);
  for (int i = n - 1; i >= 0; --i) {
    double s = b[size_t(i)];
    for (int k = i + 1; k < n; ++k) s -= a[size_t(i + k * n)] * x[size_t(k)];
    x[size_t(i)] = s / a[size_t(i + i * n)];
  }
  return x;
}

// point_reconstruction_coefficients (reconstruction.hpp:55-70)
std::vector<double> point_coeffs(int first, int count, double delta) {
  std::vector<double> a(static_cast<size_t>(count * count)), rhs(static_cast<size_t>(count));
  for (int q = 0; q < count; ++q) {
    for (int l = 0; l < count; ++l) {
      const double lo = double(first + l) - 0.5, hi = double(first + l) + 0.5;
      a[size_t(q + l * count)] = (std::pow(hi, double(q + 1)) - std::pow(lo, double(q + 1))) / double(q + 1);
    }
    rhs[size_t(q)] = std::pow(delta, double(q));
  }
  return solve_dense(a, rhs, count);
}

// ideal_weights (reconstruction.hpp:74-83): consistent overdetermined system solved
// by normal equations of the (2k+1) x (k+1) candidate matrix.
std::vector<double> ideal_weights(const double cand[3][3], const double* wide, int k) {
  const int rows = 2 * k + 1, cols = k + 1;
  std::vector<double> a(size_t(rows * cols), 0.0);
  for (int r = 0; r <= k; ++r)
    for (int l = 0; l <= k; ++l) a[size_t((k - r + l) + r * rows)] = cand[r][l];
  // Householder least squares
  std::vector<double> b(wide, wide + rows);
  for (int j = 0; j < cols; ++j) {
    double nrm = 0;
    for (int i = j; i < rows; ++i) nrm += a[size_t(i + j * rows)] * a[size_t(i + j * rows)];
    nrm = std::sqrt(nrm);
    const double c0 = a[size_t(j + j * rows)];
    const double beta = c0 >= 0 ? -nrm : nrm;
    std::vector<double> v(size_t(rows), 0.0);
    v[size_t(j)] = c0 - beta;
    for (int i = j + 1; i < rows; ++i) v[size_t(i)] = a[size_t(i + j * rows)];
    double vv = 0;
    for (int i = j; i < rows; ++i) vv += v[size_t(i)] * v[size_t(i)];
    if (vv == 0) continue;
    for (int c = j; c < cols; ++c) {
      double w = 0;
      for (int i = j; i < rows; ++i) w += v[size_t(i)] * a[size_t(i + c * rows)];
      w = 2 * w / vv;
      for (int i = j; i < rows; ++i) a[size_t(i + c * rows)] -= w * v[size_t(i)];
    }
    double w = 0;
    for (int i = j; i < rows; ++i) w += v[size_t(i)] * b[size_t(i)];
    w = 2 * w / vv;
    for (int i = j; i < rows; ++i) b[size_t(i)] -= w * v[size_t(i)];
  }
  std::vector<double> x(static_cast<size_t>(cols));
  for (int i = cols - 1; i >= 0; --i) {
    double s = b[size_t(i)];
    for (int c = i + 1; c < cols; ++c) s -= a[size_t(i + c * rows)] * x[size_t(c)];
    x[size_t(i)] = s / a[size_t(i + i * rows)];
  }
  return x;
}

Tables make_tables(Scheme scheme) {
  Tables t;
  t.radius = stencil_radius(scheme);
  t.nq = quadrature_points(scheme);
  const int k = t.radius;
  if (t.nq == 2) {
    const double a = 1.0 / (2.0 * std::sqrt(3.0));
    t.offset[0] = -a;
    t.offset[1] = a;
    t.weight[0] = t.weight[1] = 0.5;
  } else {
    const double b = std::sqrt(3.0 / 5.0) / 2.0;
    t.offset[0] = -b;
    t.offset[1] = 0.0;
    t.offset[2] = b;
    t.weight[0] = 5.0 / 18.0;
    t.weight[1] = 8.0 / 18.0;
    t.weight[2] = 5.0 / 18.0;
  }
  for (int r = 0; r <= k; ++r) {
    auto c = point_coeffs(-r, k + 1, 0.5);
    for (int l = 0; l <= k; ++l) t.step1_c[r][l] = c[size_t(l)];
  }
  auto row = point_coeffs(-k, 2 * k + 1, 0.5);
  for (int l = 0; l < 2 * k + 1; ++l) t.step1_row[l] = row[size_t(l)];
  auto ideal = ideal_weights(t.step1_c, t.step1_row, k);
  for (int r = 0; r <= k; ++r) t.step1_ideal[r] = ideal[size_t(r)];
  for (int m = 0; m < t.nq; ++m) {
    for (int r = 0; r <= k; ++r) {
      auto c = point_coeffs(-r, k + 1, t.offset[m]);
      for (int l = 0; l <= k; ++l) t.c[m][r][l] = c[size_t(l)];
    }
    auto pr = point_coeffs(-k, 2 * k + 1, t.offset[m]);
    for (int l = 0; l < 2 * k + 1; ++l) t.point_row[m][l] = pr[size_t(l)];
    auto g = ideal_weights(t.c[m], t.point_row[m], k);
    for (int r = 0; r <= k; ++r) t.gamma[m][r] = g[size_t(r)];
  }
  if (k == 2) {
    const double gp[3] = {9.0 / 214, 98.0 / 107, 9.0 / 214}, gm[3] = {9.0 / 67, 49.0 / 67, 9.0 / 67},
                 wd[3] = {3.0 / 10, 3.0 / 5, 1.0 / 10};
    for (int i = 0; i < 3; ++i) {
      t.gamma_plus[i] = gp[i];
      t.gamma_minus[i] = gm[i];
      t.weno_d[i] = wd[i];
    }
  }
  return t;
}

}  // namespace

const Tables& recon_tables(Scheme s) {
  static const Tables u3 = make_tables(Scheme::Upwind3);
  static const Tables u5 = make_tables(Scheme::Upwind5);
  static const Tables w5 = make_tables(Scheme::Weno5);
  return s == Scheme::Upwind3 ? u3 : (s == Scheme::Upwind5 ? u5 : w5);
}

/// Banded forms of the operator matrices of reconstruction.hpp:428-501 and
/// periodic_pad_matrix (:473-478); never materialised as dense N x N matrices.
BandMap make_band_map(int op, Scheme scheme, Side side, Index n, Index a0, Index a1) {
  const Tables& t = recon_tables(scheme);
  const int k = t.radius, nq = t.nq;
  BandMap m;
  switch (op) {
    case 0:  // periodic pad, (n+6) x n
      m.n_out = n + 2 * kGhost;
      m.n_in = n;
      m.off[0] = -int(kGhost);
      m.coef[0][0] = 1.0;
      m.wrap = true;
      break;
    case 1: {  // step1, (n+1) x (n+6)
      m.n_out = n + 1;
      m.n_in = n + 2 * kGhost;
      m.taps = 2 * k + 1;
      m.off[0] = side == Side::Minus ? int(kGhost) - k - 1 : int(kGhost) - k;
      for (int l = 0; l < m.taps; ++l)
        m.coef[0][l] = side == Side::Minus ? t.step1_row[l] : t.step1_row[m.taps - 1 - l];
      break;
    }
    case 2:  // quadrature point, (n nq) x (n+6), rows cell-major / point-minor
      m.n_out = n * nq;
      m.n_in = n + 2 * kGhost;
      m.period = nq;
      m.taps = 2 * k + 1;
      for (int q = 0; q < nq; ++q) {
        m.off[q] = int(kGhost) - k;
        for (int l = 0; l < m.taps; ++l) m.coef[q][l] = t.point_row[q][l];
      }
      break;
    case 3:  // quadrature sum, n x (n nq)
      m.n_out = n;
      m.n_in = n * nq;
      m.stride = nq;
      m.taps = nq;
      for (int q = 0; q < nq; ++q) m.coef[0][q] = t.weight[q];
      break;
    case 4:  // interface difference, n x (n+1): out_i = -in_i + in_{i+1}
      m.n_out = n;
      m.n_in = n + 1;
      m.taps = 2;
      m.coef[0][0] = -1.0;
      m.coef[0][1] = 1.0;
      break;
    case 5:  // row slice, a1 x (n+6) starting at a0
      m.n_out = a1;
      m.n_in = n + 2 * kGhost;
      m.off[0] = int(a0);
      m.coef[0][0] = 1.0;
      if (a0 < 0 || a0 + a1 > m.n_in) throw ShapeError("row_slice: out of range");
      break;
    case 6:  // quadrature slice s = a0, (n nq) x (n+6)
      m.n_out = n * nq;
      m.n_in = n + 2 * kGhost;
      m.period = nq;
      for (int q = 0; q < nq; ++q) {
        m.off[q] = int(kGhost) - k + int(a0);
        m.coef[q][0] = 1.0;
      }
      break;
    default:
      throw InputError("unknown core map");
  }
  return m;
}

}  // namespace ttsw
