// Full-tensor (DenseRep) path on the device: the reference's `DenseRep` plugin
// (/root/reference/proj/include/ttsw/swe.hpp:45-80) driven through the same rhs<Rep> /
// ssprk3<Rep> (swe.hpp:362-454) with the dense reconstruction of
// reconstruction.hpp:253-423 (step1_blocks / step2_blocks on stencil blocks). Fields are
// N x N column-major cell averages resident in HBM; every operation of the reference's
// dense rhs is pointwise or a short stencil, so one rhs is a handful of fused kernels:
//
//   k_dense_ghost   (N+6)^2 ghosted copy per component: periodic wrap, or the exact
//                   Dirichlet ghost averages the host evaluated (cases.cpp:271-296)
//   k_dense_axis    per axis and CTA tile: the ghosted tile in shared memory, step 1 of
//                   both sides along the axis (interface lines), step 2 across it at the
//                   n_q Gauss points, physical flux, LLF with the scalar dissipation speed,
//                   Gauss-weighted sum over the points -> Fhat at (interface, cell);
//                   MODE_LAMBDA only reduces max(|m/h| + sqrt(g h)) over both sides
//                   (face_wave_speed, swe.hpp:329-339) into a device scalar
//   k_dense_combine difference of Fhat along each axis / spacing, Coriolis (+ manufactured)
//                   source, the Euler stage and the SSP-RK3 combination in one pass
//
// Arithmetic follows the reference's operation order (step1/step2 candidate sums,
// flux products, llf axpys, the rhs sum -(fx + fy/dy..) + source); it is not bitwise
// (FMA contraction, summation order of the Gauss sum), parity is to 1e-12 relative.
#include <algorithm>
#include <cmath>
#include <cstring>

#include "kernels.cuh"

namespace ttsw {

namespace {

constexpr int G = 3;        // kGhost
constexpr int TI = 32;      // interfaces per tile (along the axis)
constexpr int TJ = 32;      // transverse cells per tile
constexpr int DT = 256;     // threads of k_dense_axis
constexpr int MODE_LAMBDA = 0, MODE_FLUX = 1;

struct DenseTables {
  int k, nq, scheme;
  double s1[3][3];      // step1_ideal[r] * step1_c(r, l) (Upwind) / step1_c (WENO)
  double c[3][3][3];    // c[m](r, l)
  double gamma[3][3], gamma_plus[3], gamma_minus[3], weno_d[3];
  double sigma_plus, sigma_minus;
  double weight[3];
  double step1_c[3][3];
  double ideal[3];
};

struct DenseArgs {
  const double* gh[3];  // ghosted (N+6) x (N+6), column-major
  double* fhat[3];      // axis X: (N+1) x N, axis Y: N x (N+1)
  double* lam;          // [0] max speed (as ordered bits), [1] nonpositive-h flag
  long n;
  int model;
  double g, H;
  double eps1, eps2;    // WENO epsilon of step 1 (along the axis) and step 2
  double lam_linear;    // sqrt(gH) for the linear model
};

__device__ __forceinline__ double step1_value(const double* v, const DenseTables& t, double eps) {
  // step1_blocks (reconstruction.hpp:253-286) for one interface; v in minus orientation
  if (t.scheme == 0) {
    double out = 0.0;
    for (int r = 0; r <= 1; ++r)
      for (int l = 0; l <= 1; ++l) out += t.s1[r][l] * v[1 - r + l];
    return out;
  }
  if (t.scheme == 1) {
    double out = 0.0;
    for (int r = 0; r <= 2; ++r)
      for (int l = 0; l <= 2; ++l) out += t.s1[r][l] * v[2 - r + l];
    return out;
  }
  const double c1312 = 13.0 / 12.0;
  double a = v[2] - 2 * v[3] + v[4], b = 3 * v[2] - 4 * v[3] + v[4];
  const double b0 = c1312 * (a * a) + 0.25 * (b * b);
  a = v[1] - 2 * v[2] + v[3];
  b = v[1] - v[3];
  const double b1 = c1312 * (a * a) + 0.25 * (b * b);
  a = v[0] - 2 * v[1] + v[2];
  b = v[0] - 4 * v[1] + 3 * v[2];
  const double b2 = c1312 * (a * a) + 0.25 * (b * b);
  const double d0 = b0 + eps, d1 = b1 + eps, d2 = b2 + eps;
  const double a0 = t.weno_d[0] / (d0 * d0), a1 = t.weno_d[1] / (d1 * d1), a2 = t.weno_d[2] / (d2 * d2);
  const double total = a0 + a1 + a2;
  const double c0 = t.step1_c[0][0] * v[2] + t.step1_c[0][1] * v[3] + t.step1_c[0][2] * v[4];
  const double c1 = t.step1_c[1][0] * v[1] + t.step1_c[1][1] * v[2] + t.step1_c[1][2] * v[3];
  const double c2 = t.step1_c[2][0] * v[0] + t.step1_c[2][1] * v[1] + t.step1_c[2][2] * v[2];
  return (a0 * c0 + a1 * c1 + a2 * c2) / total;
}

__device__ __forceinline__ double weno_combine(const double* g, const double* b, const double* cand, double eps) {
  const double d0 = b[0] + eps, d1 = b[1] + eps, d2 = b[2] + eps;
  const double a0 = g[0] / (d0 * d0), a1 = g[1] / (d1 * d1), a2 = g[2] / (d2 * d2);
  return (a0 * cand[0] + a1 * cand[1] + a2 * cand[2]) / (a0 + a1 + a2);
}

__device__ __forceinline__ double step2_value(const double* v, int m, const DenseTables& t, double eps) {
  // step2_blocks (reconstruction.hpp:289-323) at quadrature point m on a centred block
  const int k = t.k;
  double cand[3];
  for (int r = 0; r <= k; ++r) {
    double s = 0.0;
    for (int l = 0; l <= k; ++l) s += t.c[m][r][l] * v[k - r + l];
    cand[r] = s;
  }
  if (t.scheme == 0) return 0.5 * cand[0] + 0.5 * cand[1];
  if (t.scheme == 1) {
    if (m == 1) {
      const double up = t.gamma_plus[0] * cand[0] + t.gamma_plus[1] * cand[1] + t.gamma_plus[2] * cand[2];
      const double um = t.gamma_minus[0] * cand[0] + t.gamma_minus[1] * cand[1] + t.gamma_minus[2] * cand[2];
      return t.sigma_plus * up - t.sigma_minus * um;
    }
    return t.gamma[m][0] * cand[0] + t.gamma[m][1] * cand[1] + t.gamma[m][2] * cand[2];
  }
  const double c1312 = 13.0 / 12.0;
  double b[3];
  double a = v[2] - 2 * v[3] + v[4], bb = 3 * v[2] - 4 * v[3] + v[4];
  b[0] = c1312 * (a * a) + 0.25 * (bb * bb);
  a = v[1] - 2 * v[2] + v[3];
  bb = v[1] - v[3];
  b[1] = c1312 * (a * a) + 0.25 * (bb * bb);
  a = v[0] - 2 * v[1] + v[2];
  bb = v[0] - 4 * v[1] + 3 * v[2];
  b[2] = c1312 * (a * a) + 0.25 * (bb * bb);
  if (m == 1)
    return t.sigma_plus * weno_combine(t.gamma_plus, b, cand, eps) -
           t.sigma_minus * weno_combine(t.gamma_minus, b, cand, eps);
  return weno_combine(t.gamma[m], b, cand, eps);
}

// Ghosted copy (dense_ghosted, cases.cpp:271-296): interior, periodic wrap per periodic
// axis, the host's exact strip values on Dirichlet ghost cells (strip_x: 6 x (N+6) ghost
// rows, strip_y: (N+6) x 6 ghost columns, as ttsw_ghosted).
__global__ void k_dense_ghost(const double* __restrict__ q, double* __restrict__ gh, long n, int bcx, int bcy,
                              const double* __restrict__ sx, const double* __restrict__ sy) {
  const long ng = n + 2 * G;
  for (long e = blockIdx.x * long(blockDim.x) + threadIdx.x; e < ng * ng; e += long(gridDim.x) * blockDim.x) {
    const long i = e % ng, j = e / ng;
    long ii = i - G, jj = j - G;
    const bool gx = ii < 0 || ii >= n, gy = jj < 0 || jj >= n;
    double v;
    if (gx && bcx) {
      const long s = i < G ? i : i - n;  // ghost row index 0..5
      v = sx[s + 6 * j];
    } else if (gy && bcy) {
      const long s = j < G ? j : j - n;
      v = sy[i + ng * s];
    } else {
      if (gx) ii = ((ii % n) + n) % n;
      if (gy) jj = ((jj % n) + n) % n;
      v = q[ii + n * jj];
    }
    gh[e] = v;
  }
}

__device__ __forceinline__ void atomic_max_pos(double* addr, double v) {
  // non-negative doubles order like their bit patterns
  atomicMax(reinterpret_cast<unsigned long long*>(addr), __double_as_longlong(v));
}

// One axis of the dense rhs on a tile of TI interfaces x TJ transverse cells.
// AXIS 0 (X): interfaces along rows i in [0, N], cells along columns j; the ghosted
// element (row r, col s) is gh[r + ng s]. AXIS 1 (Y) is the transpose.
template <int AXIS, int MODE>
__global__ void __launch_bounds__(DT) k_dense_axis(const __grid_constant__ DenseArgs A,
                                                   const __grid_constant__ DenseTables t) {
  extern __shared__ double sm[];
  const int k = t.k, nq = t.nq;
  const long n = A.n, ng = n + 2 * G;
  const long i0 = long(blockIdx.x) * TI, j0 = long(blockIdx.y) * TJ;
  const int RI = TI + 2 * k + 1;  // ghosted lines along the axis: [i0 + 2 - k, i0 + TI + 2 + k]
  const int RJ = TJ + 2 * k;      // transverse ghosted positions: [j0 + 3 - k, j0 + TJ + 2 + k]
  double* tile = sm;                          // [3][RI][RJ]
  double* lines = tile + 3 * RI * RJ;         // [2 sides][3][TI][RJ]
  const long abase = i0 + 2 - k, tbase = j0 + 3 - k;
  for (int e = threadIdx.x; e < 3 * RI * RJ; e += DT) {
    const int c = e / (RI * RJ), rem = e % (RI * RJ), a = rem % RI, b = rem / RI;
    const long ga = abase + a, gt = tbase + b;
    double v = 0.0;
    if (ga < ng && gt < ng) v = AXIS == 0 ? A.gh[c][ga + ng * gt] : A.gh[c][gt + ng * ga];
    tile[(c * RJ + b) * RI + a] = v;
  }
  __syncthreads();
  // step 1 along the axis: line value of interface i (local ii) at transverse position b
  for (int e = threadIdx.x; e < 2 * 3 * TI * RJ; e += DT) {
    const int side = e / (3 * TI * RJ), rem = e % (3 * TI * RJ);
    const int c = rem / (TI * RJ), r2 = rem % (TI * RJ), ii = r2 % TI, b = r2 / TI;
    double v[5];
    // minus: rows i + (G - k - 1) + s; plus: rows i + (G - k) + s, reversed (minus orientation)
    const int off = ii + (side == 0 ? 0 : 1);  // relative to abase = i0 + 2 - k
    const double* col = tile + (c * RJ + b) * RI;
    for (int s = 0; s <= 2 * k; ++s) v[side == 0 ? s : 2 * k - s] = col[off + s];
    lines[((side * 3 + c) * RJ + b) * TI + ii] = step1_value(v, t, A.eps1);
  }
  __syncthreads();
  double lmax = 0.0;
  bool bad = false;
  for (int e = threadIdx.x; e < TI * TJ; e += DT) {  // TI * TJ is a multiple of DT: no divergent trip count
    const int ii = e % TI, jj = e / TI;
    const long i = i0 + ii, j = j0 + jj;
    if (i > n || j >= n) continue;
    double acc[3] = {0.0, 0.0, 0.0};
    for (int m = 0; m < nq; ++m) {
      double u[2][3];
      for (int side = 0; side < 2; ++side)
        for (int c = 0; c < 3; ++c) {
          double v[5];
          const double* ln = lines + (side * 3 + c) * RJ * TI;
          for (int s = 0; s <= 2 * k; ++s) v[s] = ln[(jj + s) * TI + ii];
          u[side][c] = step2_value(v, m, t, A.eps2);
        }
      if (MODE == MODE_LAMBDA) {  // face_wave_speed, DenseRep branch (swe.hpp:329-339)
        const int mom = AXIS == 0 ? 1 : 2;
        for (int side = 0; side < 2; ++side) {
          const double h = u[side][0];
          if (!(h > 0.0)) bad = true;
          lmax = fmax(lmax, fabs(u[side][mom] / h) + sqrt(A.g * h));
        }
        continue;
      }
      double f[2][3];
      for (int side = 0; side < 2; ++side) {
        const double* w = u[side];
        if (A.model == 0) {  // F = (H u, g eta, 0), G = (H v, 0, g eta) (swe.hpp:195-201)
          if (AXIS == 0) {
            f[side][0] = A.H * w[1];
            f[side][1] = A.g * w[0];
            f[side][2] = 0.0;
          } else {
            f[side][0] = A.H * w[2];
            f[side][1] = 0.0;
            f[side][2] = A.g * w[0];
          }
        } else {  // physical_flux, nonlinear (swe.hpp:203-212) with DenseRep ops
          const double inv_h = 1.0 / w[0];
          const double vx = w[1] * inv_h, vy = w[2] * inv_h;
          const double p = (0.5 * A.g) * (w[0] * w[0]);
          if (AXIS == 0) {
            f[side][0] = w[1];
            f[side][1] = w[1] * vx + p;
            f[side][2] = w[1] * vy;
          } else {
            f[side][0] = w[2];
            f[side][1] = w[2] * vx;
            f[side][2] = w[2] * vy + p;
          }
        }
      }
      const double lam = A.model == 0 ? A.lam_linear : A.lam[0];
      for (int c = 0; c < 3; ++c) {  // llf_flux with a scalar speed (swe.hpp:235-248)
        const double central = 0.5 * f[0][c] + 0.5 * f[1][c];
        const double jump = u[1][c] - u[0][c];
        acc[c] += t.weight[m] * (central + (-0.5 * lam) * jump);
      }
    }
    if (MODE == MODE_FLUX) {
      const long idx = AXIS == 0 ? i + (n + 1) * j : j + n * i;
      for (int c = 0; c < 3; ++c) A.fhat[c][idx] = acc[c];
    }
  }
  if (MODE == MODE_LAMBDA) {
    if (bad) A.lam[1] = 1.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) lmax = fmax(lmax, __shfl_xor_sync(0xffffffffu, lmax, o));
    if ((threadIdx.x & 31) == 0 && lmax > 0.0) atomic_max_pos(A.lam, lmax);
  }
}

struct CombineArgs {
  const double* w[3];     // stage input (the rhs is evaluated at w)
  const double* u[3];     // step start state (RK combination), may equal w
  double* out[3];
  const double* fx[3];    // (N+1) x N
  const double* fy[3];    // N x (N+1)
  const double* extra[3]; // manufactured source or nullptr
  long n;
  double inv_dx, inv_dy, f, dt, a, b;  // mode 1: out = a u + b (w + dt k)
  int mode;                            // 0: out = w + dt k, 1: the combination, 2: out = k
};

// k = -(D_x Fx / dx + D_y Fy / dy) + S, S = (0, f q3, -f q2) [+ extra] (swe.hpp:397-421);
// Euler stage w + dt k (swe.hpp:432-437) and the SSP-RK3 combination (swe.hpp:440-452).
__global__ void k_dense_combine(const __grid_constant__ CombineArgs C) {
  const long n = C.n;
  for (long e = blockIdx.x * long(blockDim.x) + threadIdx.x; e < n * n; e += long(gridDim.x) * blockDim.x) {
    const long i = e % n, j = e / n;
    double src[3] = {0.0, C.f * C.w[2][e], -C.f * C.w[1][e]};
    for (int c = 0; c < 3; ++c) {
      const double dxv = C.fx[c][(i + 1) + (n + 1) * j] - C.fx[c][i + (n + 1) * j];
      const double dyv = C.fy[c][i + n * (j + 1)] - C.fy[c][i + n * j];
      const double div = C.inv_dx * dxv + C.inv_dy * dyv;
      double s = src[c];
      if (C.extra[c]) s = s + C.extra[c][e];
      const double kc = -div + s;
      if (C.mode == 2) {
        C.out[c][e] = kc;
        continue;
      }
      const double stage = C.w[c][e] + C.dt * kc;
      C.out[c][e] = C.mode == 0 ? stage : C.a * C.u[c][e] + C.b * stage;
    }
  }
}

DenseTables make_tables(Scheme s) {
  const Tables& t = recon_tables(s);
  DenseTables d{};
  d.k = t.radius;
  d.nq = t.nq;
  d.scheme = int(s);
  for (int r = 0; r < 3; ++r) {
    for (int l = 0; l < 3; ++l) {
      d.s1[r][l] = t.step1_ideal[r] * t.step1_c[r][l];
      d.step1_c[r][l] = t.step1_c[r][l];
      d.gamma[r][l] = t.gamma[r][l];
      for (int q = 0; q < 3; ++q) d.c[r][l][q] = t.c[r][l][q];
    }
    d.gamma_plus[r] = t.gamma_plus[r];
    d.gamma_minus[r] = t.gamma_minus[r];
    d.weno_d[r] = t.weno_d[r];
    d.weight[r] = t.weight[r];
    d.ideal[r] = t.step1_ideal[r];
  }
  d.sigma_plus = t.sigma_plus;
  d.sigma_minus = t.sigma_minus;
  return d;
}

size_t axis_smem(int k) {
  const int RI = TI + 2 * k + 1, RJ = TJ + 2 * k;
  return sizeof(double) * size_t(3 * RI * RJ + 2 * 3 * TI * RJ);
}

}  // namespace

DenseSolver::DenseSolver(Context* c, const SolverOptions& o, Index n_, double dt_)
    : ctx(c), n(n_), opt(o), dt(dt_) {
  if (n < 1) throw InputError("dense solver: grid must have at least one cell");
  const size_t nn = size_t(n * n), ng = size_t((n + 2 * G) * (n + 2 * G));
  const size_t faces = size_t((n + 1) * n);
  for (int c = 0; c < 3; ++c) {
    q[c] = ctx->alloc(nn);
    s1[c] = ctx->alloc(nn);
    s2[c] = ctx->alloc(nn);
    gh[c] = ctx->alloc(ng);
    fx[c] = ctx->alloc(faces);
    fy[c] = ctx->alloc(faces);
    TTSW_CUDA(cudaMemsetAsync(q[c], 0, nn * sizeof(double), ctx->stream));
  }
  lam = ctx->alloc(4);
  strips = ctx->alloc(3 * 2 * 6 * size_t(n + 2 * G));
  src = ctx->alloc(3 * nn);
}

DenseSolver::~DenseSolver() {
  for (int c = 0; c < 3; ++c)
    for (double* p : {q[c], s1[c], s2[c], gh[c], fx[c], fy[c]}) ctx->free(p);
  ctx->free(lam);
  ctx->free(strips);
  ctx->free(src);
}

void DenseSolver::rhs_stage(double* const w[3], double* const u[3], double* const out[3], double ts, int mode,
                            double a, double b) {
  const long ng = n + 2 * G;
  const int gblocks = int(std::min<long>(4L * ctx->num_sms, (ng * ng + 255) / 256));
  const bool dirichlet = bc_x || bc_y;
  const size_t sz = size_t(2 * 6 * ng);  // strip_x + strip_y of one component
  if (dirichlet) {
    if (!strip_fn) throw StateError("dense solver: Dirichlet axes need a strip callback");
    std::vector<double> hs(3 * sz, 0.0);
    for (int c = 0; c < 3; ++c)
      if (strip_fn(ts, c, hs.data() + c * sz, hs.data() + c * sz + 6 * ng) != 0)
        throw StateError("fill_ghost hook failed");
    // the previous stage's ghost kernels may still read the strips: wait before overwriting
    TTSW_CUDA(cudaStreamSynchronize(ctx->stream));
    TTSW_CUDA(cudaMemcpyAsync(strips, hs.data(), sizeof(double) * hs.size(), cudaMemcpyHostToDevice, ctx->stream));
  }
  for (int c = 0; c < 3; ++c) {
    const double* sx = dirichlet ? strips + c * sz : nullptr;
    const double* sy = dirichlet ? strips + c * sz + 6 * ng : nullptr;
    k_dense_ghost<<<gblocks, 256, 0, ctx->stream>>>(w[c], gh[c], n, bc_x, bc_y, sx, sy);
    ctx->launches++;
  }
  TTSW_CUDA(cudaGetLastError());
  const DenseTables t = make_tables(opt.scheme);
  const size_t smem = axis_smem(t.k);
  const double dx = 1.0 / double(n), dy = 1.0 / double(n);
  for (int axis = 0; axis < 2; ++axis) {
    DenseArgs A{};
    for (int c = 0; c < 3; ++c) {
      A.gh[c] = gh[c];
      A.fhat[c] = axis == 0 ? fx[c] : fy[c];
    }
    A.lam = lam + 2 * axis;
    A.n = n;
    A.model = int(opt.model);
    A.g = opt.params.g;
    A.H = opt.params.H;
    A.eps1 = axis == 0 ? dx * dx : dy * dy;
    A.eps2 = axis == 0 ? dy * dy : dx * dx;
    A.lam_linear = std::sqrt(opt.params.g * opt.params.H);
    const dim3 grid(unsigned((n + 1 + TI - 1) / TI), unsigned((n + TJ - 1) / TJ));
    if (opt.model == Model::Nonlinear) {
      TTSW_CUDA(cudaMemsetAsync(A.lam, 0, 2 * sizeof(double), ctx->stream));
      if (axis == 0) {
        allow_dynamic_smem(reinterpret_cast<const void*>(k_dense_axis<0, MODE_LAMBDA>), smem);
        k_dense_axis<0, MODE_LAMBDA><<<grid, DT, smem, ctx->stream>>>(A, t);
      } else {
        allow_dynamic_smem(reinterpret_cast<const void*>(k_dense_axis<1, MODE_LAMBDA>), smem);
        k_dense_axis<1, MODE_LAMBDA><<<grid, DT, smem, ctx->stream>>>(A, t);
      }
      ctx->launches++;
    }
    if (axis == 0) {
      allow_dynamic_smem(reinterpret_cast<const void*>(k_dense_axis<0, MODE_FLUX>), smem);
      k_dense_axis<0, MODE_FLUX><<<grid, DT, smem, ctx->stream>>>(A, t);
    } else {
      allow_dynamic_smem(reinterpret_cast<const void*>(k_dense_axis<1, MODE_FLUX>), smem);
      k_dense_axis<1, MODE_FLUX><<<grid, DT, smem, ctx->stream>>>(A, t);
    }
    ctx->launches++;
    TTSW_CUDA(cudaGetLastError());
  }
  CombineArgs C{};
  const size_t nn = size_t(n * n);
  if (source_fn) {
    std::vector<double> hsrc(3 * nn);
    if (source_fn(ts, hsrc.data()) != 0) throw StateError("extra_source hook failed");
    TTSW_CUDA(cudaStreamSynchronize(ctx->stream));
    TTSW_CUDA(cudaMemcpyAsync(src, hsrc.data(), sizeof(double) * hsrc.size(), cudaMemcpyHostToDevice, ctx->stream));
  }
  for (int c = 0; c < 3; ++c) {
    C.w[c] = w[c];
    C.u[c] = u[c];
    C.out[c] = out[c];
    C.fx[c] = fx[c];
    C.fy[c] = fy[c];
    C.extra[c] = source_fn ? src + c * nn : nullptr;
  }
  C.n = n;
  C.inv_dx = 1.0 / dx;
  C.inv_dy = 1.0 / dy;
  C.f = opt.params.f;
  C.dt = dt;
  C.a = a;
  C.b = b;
  C.mode = mode;
  k_dense_combine<<<int(std::min<long>(4L * ctx->num_sms, (long(nn) + 255) / 256)), 256, 0, ctx->stream>>>(C);
  ctx->launches++;
  TTSW_CUDA(cudaGetLastError());
}

void DenseSolver::check_positive() {
  if (opt.model != Model::Nonlinear) return;
  double h[4];
  TTSW_CUDA(cudaMemcpyAsync(h, lam, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
  ctx->sync();
  if (h[1] != 0.0 || h[3] != 0.0) throw StateError("face_wave_speed: nonpositive layer thickness");
}

void DenseSolver::step() {
  if (!(dt > 0)) throw InputError("ssprk3: dt must be positive");
  // the positivity flag is per stage (the speed buffers are reset by every axis pass):
  // check after each stage, as the reference throws inside the stage
  rhs_stage(q, q, s1, t, 0, 0.0, 1.0);            // u1 = u + dt L(u)
  check_positive();
  rhs_stage(s1, q, s2, t + dt, 1, 0.75, 0.25);    // u2 = 3/4 u + 1/4 (u1 + dt L(u1))
  check_positive();
  rhs_stage(s2, q, s1, t + 0.5 * dt, 1, 1.0 / 3.0, 2.0 / 3.0);  // u^{n+1} = 1/3 u + 2/3 (u2 + dt L(u2))
  check_positive();
  std::swap(q, s1);
  t += dt;
}

void DenseSolver::rhs(double* const out[3]) {
  rhs_stage(q, q, out, t, 2, 0.0, 0.0);  // k = L(u) at the solver time (rhs<DenseRep>)
  check_positive();
}

}  // namespace ttsw
