// Host runtime: context, device TT handles and the TT algebra of
// /root/reference/proj/include/ttsw/tt.hpp re-designed around device-resident cores.
#include <cmath>
#include <cstring>
#include <sstream>

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
  TTSW_CUDA(cudaMallocHost(&pinned, 4096));
  TTSW_CUDA(cudaEventCreate(&ev0));
  TTSW_CUDA(cudaEventCreate(&ev1));
}

Context::~Context() {
  if (stream) cudaStreamSynchronize(stream);
  if (ev0) cudaEventDestroy(ev0);
  if (ev1) cudaEventDestroy(ev1);
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

void Context::sync() { TTSW_CUDA(cudaStreamSynchronize(stream)); }

MutTT make_tt(Context* ctx, Index m, Index n, Index r) {
  return std::make_shared<DevTT>(ctx, m, n, r, std::make_shared<DBuf>(ctx, size_t(m * r)),
                                 std::make_shared<DBuf>(ctx, size_t(n * r)));
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

void tt_to_host(const TT& x, double* cx, double* cy) {
  Context* ctx = x->ctx;
  std::vector<double> yt(static_cast<size_t>(x->n * x->r));
  TTSW_CUDA(cudaMemcpyAsync(cx, x->X, sizeof(double) * size_t(x->m * x->r), cudaMemcpyDeviceToHost, ctx->stream));
  TTSW_CUDA(cudaMemcpyAsync(yt.data(), x->Yt, sizeof(double) * yt.size(), cudaMemcpyDeviceToHost, ctx->stream));
  ctx->sync();
  for (Index a = 0; a < x->r; ++a)
    for (Index j = 0; j < x->n; ++j) cy[a + j * x->r] = yt[size_t(j + a * x->n)];
}

/// TTMatrix::zero (tt.hpp:35-37): rank-1 zero cores.
TT tt_zero(Context* ctx, Index rows, Index cols) {
  auto t = make_tt(ctx, rows, cols, 1);
  launch_fill(ctx, t->X, rows, 0.0);
  launch_fill(ctx, t->Yt, cols, 0.0);
  return t;
}

/// TTMatrix::constant (tt.hpp:39-41).
TT tt_constant(Context* ctx, Index rows, Index cols, double v) {
  auto t = make_tt(ctx, rows, cols, 1);
  launch_fill(ctx, t->X, rows, v);
  launch_fill(ctx, t->Yt, cols, 1.0);
  return t;
}

static void check_same_shape(const TT& x, const TT& y, const char* where) {
  if (x->m != y->m || x->n != y->n) throw ShapeError(std::string(where) + ": operand shapes do not match");
}

/// Concatenation with per-operand core_x scaling: add(scale(x,a), scale(y,b))
/// (tt.hpp:152-166) in one pass; identical values to scaling then concatenating.
static TT add_scaled(double a, const TT& x, double b, const TT& y) {
  check_same_shape(x, y, "add");
  Context* ctx = x->ctx;
  auto t = make_tt(ctx, x->m, x->n, x->r + y->r);
  if (a == 1.0)
    TTSW_CUDA(cudaMemcpyAsync(t->X, x->X, sizeof(double) * size_t(x->m * x->r), cudaMemcpyDeviceToDevice, ctx->stream));
  else
    launch_scale_copy(ctx, t->X, x->X, x->m * x->r, a);
  if (b == 1.0)
    TTSW_CUDA(cudaMemcpyAsync(t->X + x->m * x->r, y->X, sizeof(double) * size_t(y->m * y->r), cudaMemcpyDeviceToDevice,
                              ctx->stream));
  else
    launch_scale_copy(ctx, t->X + x->m * x->r, y->X, y->m * y->r, b);
  TTSW_CUDA(cudaMemcpyAsync(t->Yt, x->Yt, sizeof(double) * size_t(x->n * x->r), cudaMemcpyDeviceToDevice, ctx->stream));
  TTSW_CUDA(cudaMemcpyAsync(t->Yt + x->n * x->r, y->Yt, sizeof(double) * size_t(y->n * y->r), cudaMemcpyDeviceToDevice,
                            ctx->stream));
  return t;
}

TT add(const TT& x, const TT& y) { return add_scaled(1.0, x, 1.0, y); }

/// scale (tt.hpp:163-166): scales core_x only; core_y is shared.
TT scale(const TT& x, double a) {
  Context* ctx = x->ctx;
  auto xb = std::make_shared<DBuf>(ctx, size_t(x->m * x->r));
  launch_scale_copy(ctx, xb->p, x->X, x->m * x->r, a);
  return std::make_shared<DevTT>(ctx, x->m, x->n, x->r, xb, x->yb);
}

/// hadamard (tt.hpp:169-181).
TT hadamard(const TT& x, const TT& y) {
  check_same_shape(x, y, "hadamard");
  Context* ctx = x->ctx;
  auto t = make_tt(ctx, x->m, x->n, x->r * y->r);
  launch_hadamard(ctx, x->X, x->r, y->X, y->r, x->m, t->X);
  launch_hadamard(ctx, x->Yt, x->r, y->Yt, y->r, x->n, t->Yt);
  return t;
}

static double read_scalar(Context* ctx, const double* dptr) {
  TTSW_CUDA(cudaMemcpyAsync(ctx->pinned, dptr, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  ctx->sync();
  return *static_cast<double*>(ctx->pinned);
}

/// norm_fro (tt.hpp:105-111): Gram-based, clamped at zero.
double norm_fro(const TT& x) {
  Context* ctx = x->ctx;
  double* work = ctx->alloc(size_t(x->r * x->r + 1));
  launch_norm2(ctx, x->X, x->m, x->Yt, x->n, x->r, work, work + x->r * x->r);
  const double v = read_scalar(ctx, work + x->r * x->r);
  ctx->free(work);
  return std::sqrt(std::max(v, 0.0));
}

/// sum_entries (tt.hpp:113-116).
double sum_entries(const TT& x) {
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
/// core_y'^T = Qy V_k (core_y' keeps orthonormal rows).
/// The truncation rank is decided on device (tt.hpp:61-77) and read back once.
TT round(const TT& x, double eps, RoundRecord* rec) {
  if (eps < 0) throw InputError("round: eps must be non-negative");
  Context* ctx = x->ctx;
  const Index R = x->r;
  if (ctx->time_rounds) TTSW_CUDA(cudaEventRecord(ctx->ev0, ctx->stream));
  QRPlan px = plan_tsqr(ctx, x->m, R);
  QRPlan py = plan_tsqr(ctx, x->n, R);
  tsqr_factor(ctx, px, x->X, x->m);
  tsqr_factor(ctx, py, x->Yt, x->n);
  double* A = ctx->alloc(size_t(R * R));
  double* B = ctx->alloc(size_t(R * R));
  double* sig = ctx->alloc(size_t(R + 4));
  double* info = sig + R;
  launch_svd_small(ctx, px.levels.back().Rst, py.levels.back().Rst, R, eps, A, B, sig, info);
  TTSW_CUDA(cudaMemcpyAsync(ctx->pinned, info, 4 * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
  ctx->sync();
  const double* hinfo = static_cast<double*>(ctx->pinned);
  const Index k = Index(hinfo[0]);
  const double margin = hinfo[1];
  const double kappa = hinfo[3];
  TT out;
  if (k == 0) {
    out = tt_zero(ctx, x->m, x->n);
  } else {
    auto t = make_tt(ctx, x->m, x->n, k);
    tsqr_apply(ctx, px, A, R, int(k), t->X, x->m);
    tsqr_apply(ctx, py, B, R, int(k), t->Yt, x->n);
    out = t;
  }
  ctx->free(A);
  ctx->free(B);
  ctx->free(sig);
  free_tsqr(ctx, px);
  free_tsqr(ctx, py);
  if (ctx->time_rounds) {
    TTSW_CUDA(cudaEventRecord(ctx->ev1, ctx->stream));
    TTSW_CUDA(cudaEventSynchronize(ctx->ev1));
    float ms = 0;
    TTSW_CUDA(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
    // round flops 2nR^2 + 3mR^2 + 2(m+n)Rk + 11R^3 (fixed convention),
    // bytes 8(m+n)(R+k).
    const double m = double(x->m), n = double(x->n), Rd = double(R), kd = double(out->r);
    ctx->round_ms += ms;
    ctx->round_flops += 2 * n * Rd * Rd + 3 * m * Rd * Rd + 2 * (m + n) * Rd * kd + 11 * Rd * Rd * Rd;
    ctx->round_bytes += 8 * (m + n) * (Rd + kd);
    ctx->round_count++;
  }
  RoundRecord r{x->m, x->n, R, out->r, k == 0 ? INFINITY : margin, k == 0 ? INFINITY : kappa};
  if (rec) *rec = r;
  if (ctx->trace) ctx->trace->push_back(r);
  return out;
}

/// apply_core_map (tt.hpp:185-194) with a banded operator; the untouched core is shared.
TT apply_core_map(const TT& x, Axis axis, const BandMap& m, double scale_x) {
  Context* ctx = x->ctx;
  if (axis == Axis::X) {
    if (m.n_in != x->m) throw ShapeError("apply_core_map: operator/mode size mismatch");
    auto xb = std::make_shared<DBuf>(ctx, size_t(m.n_out * x->r));
    launch_band_map(ctx, x->X, x->m, xb->p, m.n_out, x->r, m);
    if (scale_x != 1.0) launch_scale_copy(ctx, xb->p, xb->p, m.n_out * x->r, scale_x);
    return std::make_shared<DevTT>(ctx, m.n_out, x->n, x->r, xb, x->yb);
  }
  if (m.n_in != x->n) throw ShapeError("apply_core_map: operator/mode size mismatch");
  auto yb = std::make_shared<DBuf>(ctx, size_t(m.n_out * x->r));
  launch_band_map(ctx, x->Yt, x->n, yb->p, m.n_out, x->r, m);
  Buf xb = x->xb;
  if (scale_x != 1.0) {
    xb = std::make_shared<DBuf>(ctx, size_t(x->m * x->r));
    launch_scale_copy(ctx, xb->p, x->X, x->m * x->r, scale_x);
  }
  return std::make_shared<DevTT>(ctx, x->m, m.n_out, x->r, xb, yb);
}

/// reciprocal_taylor (tt.hpp:204-241).
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
