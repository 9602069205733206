// fp64 kernels for the TT-FV hot path on sm_100a.
//
//  * k_band_map      — banded one-mode core maps (apply_core_map with the banded
//                      operators of reconstruction.hpp:428-501 / cases.cpp:302-308);
//                      HBM-bound, one thread per output element, coalesced along rows.
//  * k_scale_copy / k_hadamard — concatenation/scale (tt.hpp:152-166) and the
//                      face-splitting product (tt.hpp:169-181).
//  * k_qr_blocks / k_apply_blocks — tall-skinny Householder QR (TSQR) of the core
//                      panels for round (tt.hpp:120-138): one CTA per row block, the
//                      block resident in shared memory when it fits.
//  * k_svd_small    — one-sided Jacobi SVD of the R x R core product with the
//                      truncation decision taken on device in double-double.
#include <cfloat>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include <cooperative_groups.h>
#include <climits>

#include "expr.cuh"
#include "kernels.cuh"

namespace ttsw {

namespace cg = cooperative_groups;

namespace {

constexpr int kThreads = 256;
constexpr Index kQrcpThreshold = 7;  // R above which the SVD pre-truncates by QRCP (cluster path)

__host__ __device__ inline void block_range(Index rows, int L, int i, Index& start, Index& size) {
  const Index base = rows / L, rem = rows % L;
  start = Index(i) * base + (Index(i) < rem ? Index(i) : rem);
  size = base + (Index(i) < rem ? 1 : 0);
}

__device__ inline double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Deterministic block reduction; result broadcast to all threads.
__device__ inline double block_sum(double v, double* scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  double t = 0;
  if (warp == 0) {
    t = lane < nw ? scratch[lane] : 0.0;
    t = warp_sum(t);
    if (lane == 0) scratch[32] = t;
  }
  __syncthreads();
  return scratch[32];
}

__global__ void k_band_map(const double* __restrict__ in, Index ld_in, double* __restrict__ out, Index ld_out,
                           Index r, BandMap m) {
  const Index total = m.n_out * r;
  for (Index idx = Index(blockIdx.x) * blockDim.x + threadIdx.x; idx < total; idx += Index(gridDim.x) * blockDim.x) {
    const Index i = idx % m.n_out, a = idx / m.n_out;
    const int ph = int(i % m.period);
    const Index base = (i / m.period) * m.stride + m.off[ph];
    const double* col = in + a * ld_in;
    double acc = 0.0;
    for (int t = 0; t < m.taps; ++t) {
      Index row = base + t;
      if (m.wrap) row = ((row % m.n_in) + m.n_in) % m.n_in;
      acc += m.coef[ph][t] * col[row];
    }
    out[i + a * ld_out] = acc;
  }
}

// out[i, a] = sum_{p in row i} vals[p] * in[colidx[p], a]  (CSR operator on a core panel)
__global__ void k_csr_map(const double* __restrict__ in, Index ld_in, double* __restrict__ out, Index rows, Index r,
                          const long* __restrict__ rowptr, const long* __restrict__ colidx,
                          const double* __restrict__ vals) {
  const Index total = rows * r;
  for (Index idx = Index(blockIdx.x) * blockDim.x + threadIdx.x; idx < total; idx += Index(gridDim.x) * blockDim.x) {
    const Index i = idx % rows, a = idx / rows;
    double acc = 0.0;
    for (long p = rowptr[i]; p < rowptr[i + 1]; ++p) acc += vals[p] * in[colidx[p] + a * ld_in];
    out[idx] = acc;
  }
}

__global__ void k_scale_copy(double* __restrict__ dst, const double* __restrict__ src, Index count, double a) {
  for (Index i = Index(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += Index(gridDim.x) * blockDim.x)
    dst[i] = src[i] * a;
}

__global__ void k_fill(double* __restrict__ dst, Index count, double v) {
  for (Index i = Index(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += Index(gridDim.x) * blockDim.x)
    dst[i] = v;
}

// out[:, a*ry + b] = y[:, b] .* x[:, a]   (hadamard column order, tt.hpp:177-180)
__global__ void k_hadamard(const double* __restrict__ x, Index rx, const double* __restrict__ y, Index ry,
                           Index rows, double* __restrict__ out) {
  const Index total = rows * rx * ry;
  for (Index idx = Index(blockIdx.x) * blockDim.x + threadIdx.x; idx < total; idx += Index(gridDim.x) * blockDim.x) {
    const Index i = idx % rows, c = idx / rows;
    const Index a = c / ry, b = c % ry;
    out[idx] = y[i + b * rows] * x[i + a * rows];
  }
}

__global__ void k_transpose(const double* __restrict__ in, Index rows, Index cols, double* __restrict__ out) {
  __shared__ double tile[32][33];
  const Index bx = Index(blockIdx.x) * 32, by = Index(blockIdx.y) * 32;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const Index i = bx + threadIdx.x, j = by + k;
    if (i < rows && j < cols) tile[k][threadIdx.x] = in[i + j * rows];
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const Index j = by + threadIdx.x, i = bx + k;
    if (i < rows && j < cols) out[j + i * cols] = tile[threadIdx.x][k];
  }
}

// work[a*r+b] = (X^T X)_{ab} * (Yt^T Yt)_{ab}
__global__ void k_gram_prod(const double* __restrict__ X, Index m, const double* __restrict__ Yt, Index n, Index r,
                            double* __restrict__ work) {
  __shared__ double scratch[33];
  const Index a = blockIdx.x, b = blockIdx.y;
  double gx = 0, gy = 0;
  for (Index i = threadIdx.x; i < m; i += blockDim.x) gx += X[i + a * m] * X[i + b * m];
  for (Index j = threadIdx.x; j < n; j += blockDim.x) gy += Yt[j + a * n] * Yt[j + b * n];
  gx = block_sum(gx, scratch);
  gy = block_sum(gy, scratch);
  if (threadIdx.x == 0) work[a * r + b] = gx * gy;
}

// work[a] = colsum(X)_a, work[r+a] = colsum(Yt)_a
__global__ void k_colsums(const double* __restrict__ X, Index m, const double* __restrict__ Yt, Index n,
                          double* __restrict__ work, Index r) {
  __shared__ double scratch[33];
  const Index a = blockIdx.x;
  double sx = 0, sy = 0;
  for (Index i = threadIdx.x; i < m; i += blockDim.x) sx += X[i + a * m];
  for (Index j = threadIdx.x; j < n; j += blockDim.x) sy += Yt[j + a * n];
  sx = block_sum(sx, scratch);
  sy = block_sum(sy, scratch);
  if (threadIdx.x == 0) {
    work[a] = sx;
    work[r + a] = sy;
  }
}

// out = sum_i w[i] (mode 0) or sum_a w[a] * w[r+a] (mode 1); fixed order, one CTA.
__global__ void k_reduce_final(const double* __restrict__ w, Index count, int mode, Index r, double* out) {
  __shared__ double scratch[33];
  double s = 0;
  if (mode == 0)
    for (Index i = threadIdx.x; i < count; i += blockDim.x) s += w[i];
  else
    for (Index a = threadIdx.x; a < r; a += blockDim.x) s += w[a] * w[r + a];
  s = block_sum(s, scratch);
  if (threadIdx.x == 0) *out = s;
}

// ---------------------------------------------------------------------------------------
// Householder QR of one nr x R block (column-major, leading dimension ld) by a CTA.
// Reflector convention of Eigen's makeHouseholder: beta = -sign(c0)||x||,
// tau = (beta - c0)/beta, v = [1; x_tail / (c0 - beta)]; zero tail -> tau = 0.
__device__ void cta_householder_qr(double* a, Index ld, Index nr, int R, double* tau, double* scratch) {
  // Two barriers per column: the warp that updates column k+1 also computes its new
  // tail norm (look-ahead), so the next reflector needs no separate block reduction.
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int q = int(nr < R ? nr : R);
  __shared__ double tail_sh;
  {
    double part = 0;
    for (Index i = 1 + threadIdx.x; i < nr; i += blockDim.x) part += a[i] * a[i];
    const double t0 = block_sum(part, scratch);
    if (threadIdx.x == 0) tail_sh = t0;
  }
  __syncthreads();
  for (int k = 0; k < q; ++k) {
    double* ak = a + Index(k) * ld;
    const double tail2 = tail_sh;
    const double c0 = ak[k];
    double t, beta, d;
    if (tail2 <= DBL_MIN) {
      t = 0.0;
      beta = c0;
      d = 1.0;
    } else {
      beta = sqrt(c0 * c0 + tail2);
      if (c0 >= 0) beta = -beta;
      d = c0 - beta;
      t = (beta - c0) / beta;
    }
    for (Index i = k + 1 + threadIdx.x; i < nr; i += blockDim.x) ak[i] = (t == 0.0) ? 0.0 : ak[i] / d;
    __syncthreads();
    if (threadIdx.x == 0) {
      ak[k] = beta;
      tau[k] = t;
    }
    for (int j = k + 1 + warp; j < R; j += nw) {
      double* aj = a + Index(j) * ld;
      if (t != 0.0) {
        double w = 0;
        for (Index i = k + 1 + lane; i < nr; i += 32) w += ak[i] * aj[i];
        w = warp_sum(w);
        w = (aj[k] + w) * t;
        __syncwarp();
        if (lane == 0) aj[k] -= w;
        for (Index i = k + 1 + lane; i < nr; i += 32) aj[i] -= w * ak[i];
        __syncwarp();
      }
      if (j == k + 1) {  // look-ahead: tail norm of the next column (rows > k+1)
        double p = 0;
        for (Index i = k + 2 + lane; i < nr; i += 32) p += aj[i] * aj[i];
        p = warp_sum(p);
        if (lane == 0) tail_sh = p;
      }
    }
    __syncthreads();
  }
  for (int k = q + threadIdx.x; k < R; k += blockDim.x) tau[k] = 0.0;
  __syncthreads();
}

template <bool SMEM>
__global__ void __launch_bounds__(1024) k_qr_blocks(const double* __restrict__ A, Index lda, Index rows, int R,
                                                        int L, double* V, double* tau, double* Rst) {
  extern __shared__ double smem[];
  __shared__ double scratch[33];
  Index start, nr;
  block_range(rows, L, blockIdx.x, start, nr);
  double* a;
  Index ld;
  if (SMEM) {
    a = smem;
    ld = nr;
  } else {
    a = V + start;
    ld = rows;
  }
  for (Index idx = threadIdx.x; idx < nr * R; idx += blockDim.x) {
    const Index i = idx % nr, j = idx / nr;
    a[i + j * ld] = A[start + i + j * lda];
  }
  __syncthreads();
  cta_householder_qr(a, ld, nr, R, tau + Index(blockIdx.x) * R, scratch);
  const Index ldr = Index(L) * R;
  for (Index idx = threadIdx.x; idx < Index(R) * R; idx += blockDim.x) {
    const Index i = idx % R, j = idx / R;
    Rst[Index(blockIdx.x) * R + i + j * ldr] = (i <= j && i < nr) ? a[i + j * ld] : 0.0;
  }
  if (SMEM)
    for (Index idx = threadIdx.x; idx < nr * R; idx += blockDim.x) {
      const Index i = idx % nr, j = idx / nr;
      V[start + i + j * rows] = a[i + j * ld];
    }
}

// Cout[block rows] = Q_block * [Cin(block's R rows); 0]
template <bool SMEM>
__global__ void __launch_bounds__(1024) k_apply_blocks(const double* __restrict__ V, const double* __restrict__ tau,
                                                           Index rows, int R, int L, const double* __restrict__ Cin,
                                                           Index ldcin, int kc, double* Cout, Index ldcout) {
  extern __shared__ double smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  Index start, nr;
  block_range(rows, L, blockIdx.x, start, nr);
  double* c;
  Index ld;
  if (SMEM) {
    c = smem;
    ld = nr;
  } else {
    c = Cout + start;
    ld = ldcout;
  }
  const Index top = nr < R ? nr : R;
  for (Index idx = threadIdx.x; idx < nr * kc; idx += blockDim.x) {
    const Index i = idx % nr, j = idx / nr;
    c[i + j * ld] = i < top ? Cin[Index(blockIdx.x) * R + i + j * ldcin] : 0.0;
  }
  __syncthreads();
  const double* tb = tau + Index(blockIdx.x) * R;
  const int q = int(top);
  // output columns are independent: each warp carries its columns through every
  // reflector (H_{q-1} first), so no block barrier is needed between reflectors
  for (int j = warp; j < kc; j += nw) {
    double* cj = c + Index(j) * ld;
    for (int k = q - 1; k >= 0; --k) {
      const double t = tb[k];
      if (t == 0.0) continue;
      const double* v = V + start + Index(k) * rows;
      double w = 0;
      for (Index i = k + 1 + lane; i < nr; i += 32) w += v[i] * cj[i];
      w = warp_sum(w);
      w = (cj[k] + w) * t;
      __syncwarp();
      if (lane == 0) cj[k] -= w;
      for (Index i = k + 1 + lane; i < nr; i += 32) cj[i] -= w * v[i];
      __syncwarp();
    }
  }
  __syncthreads();
  if (SMEM)
    for (Index idx = threadIdx.x; idx < nr * kc; idx += blockDim.x) {
      const Index i = idx % nr, j = idx / nr;
      Cout[start + i + j * ldcout] = c[i + j * ld];
    }
}

// ---- double-double helpers for the truncation decision --------------------------------
struct dd {
  double hi, lo;
};
__device__ inline dd two_sum(double a, double b) {
  const double s = a + b, bb = s - a;
  return {s, (a - (s - bb)) + (b - bb)};
}
__device__ inline dd dd_add(dd a, dd b) {
  dd s = two_sum(a.hi, b.hi);
  s.lo += a.lo + b.lo;
  return two_sum(s.hi, s.lo);
}
__device__ inline dd two_prod(double a, double b) {
  const double p = a * b;
  return {p, fma(a, b, -p)};
}
__device__ inline dd dd_mul(dd a, dd b) {
  dd p = two_prod(a.hi, b.hi);
  p.lo += a.hi * b.lo + a.lo * b.hi;
  return two_sum(p.hi, p.lo);
}
__device__ inline bool dd_gt(dd a, dd b) { return a.hi > b.hi || (a.hi == b.hi && a.lo > b.lo); }
__device__ inline double dd_to_d(dd a) { return a.hi + a.lo; }

// Round-robin (circle method) pairing for n players (n even).
__device__ inline void rr_pair(int round, int i, int n, int& p, int& q) {
  const int m = n - 1;
  int a, b;
  if (i == 0) {
    a = m;
    b = round;
  } else {  // round, i < m: one conditional subtraction instead of an integer modulo
    a = round + i;
    if (a >= m) a -= m;
    b = round - i + m;
    if (b >= m) b -= m;
  }
  p = a < b ? a : b;
  q = a < b ? b : a;
}

/// Rotation (cs, sn) that orthogonalises two columns with Gram entries al = |x|^2,
/// be = |y|^2, ga = x.y (Rutishauser's t = sign(zeta) / (|zeta| + sqrt(1 + zeta^2)),
/// zeta = (be - al) / (2 ga), written with one sqrt, one division and one rsqrt: the
/// rotation parameters are the latency chain of every Jacobi round). False when the pair
/// is already orthogonal to tol (|ga| <= tol sqrt(al be)).
__device__ inline bool jacobi_rotation(double al, double be, double ga, double tol, double& cs, double& sn) {
  if (ga == 0.0 || ga * ga <= (tol * tol) * (al * be)) return false;
  const double d = be - al, g2 = 2.0 * ga;
  const double sgn = (d == 0.0 || (d > 0.0) == (g2 > 0.0)) ? 1.0 : -1.0;
  const double t = sgn * fabs(g2) / (fabs(d) + sqrt(d * d + g2 * g2));
  cs = rsqrt(1.0 + t * t);
  sn = cs * t;
  return true;
}

/// One-sided Jacobi SVD of S = Rx Ry^T (both R x R upper triangular, leading dims
/// ldx/ldy) by one CTA, descending order, truncation rank on device in double-double
/// (truncation_rank, tt.hpp:61-77). work: 2 Rp^2 + 2 Rp doubles (Rp = R rounded to even).
/// Writes A = S V (columns U_j sigma_j), B = V (R x R, ld R), sigma (R) and
/// info = {k, margin, sweeps, kappa}; k = 0 flags an all-zero input.
__device__ void cta_svd(const double* __restrict__ Rx, Index ldx, const double* __restrict__ Ry, Index ldy, int R,
                        double eps, double* work, double* A, double* B, double* sigma, double* info,
                        double hidden_tail = 0.0, int warp_variant_max = 64, double* vext = nullptr,
                        double hidden_rel = -1.0, int sweeps_done = -1) {
  // sweeps_done >= 0: S (rotated to orthogonal columns) and V are already in `work`
  // (k_jacobi_cluster ran the sweeps): only the norms, the ordering, the outputs and the
  // truncation decision are computed here
  // hidden_rel >= 0: further hidden energy as a fraction of sum sigma^2 (sketched inputs);
  // info[4] (decision differs without the hidden energy) is then always written
  __shared__ int rotated;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int Rp = R + (R & 1);
  // work: S (Rp^2), [V (Rp^2) unless vext holds it elsewhere], sigma (Rp), positions
  double* S = work;
  double* Vm = vext ? vext : S + Index(Rp) * Rp;
  double* sg = vext ? S + Index(Rp) * Rp : Vm + Index(Rp) * Rp;
  int* pos = reinterpret_cast<int*>(sg + Rp);
  __shared__ double red[2][32];
  {
    // ||Rx||_F^2 and ||Ry||_F^2 (= ||core_x||^2, ||core_y||^2) for the cancellation ratio
    double px = 0, py = 0;
    for (Index idx = threadIdx.x; idx < Index(R) * R; idx += blockDim.x) {
      const int i = int(idx % R), j = int(idx / R);
      if (i <= j) {
        const double a = Rx[i + Index(j) * ldx], b = Ry[i + Index(j) * ldy];
        px += a * a;
        py += b * b;
      }
    }
    px = warp_sum(px);
    py = warp_sum(py);
    if (lane == 0) {
      red[0][warp] = px;
      red[1][warp] = py;
    }
  }
  // S = Rx Ry^T, both upper triangular (ld R)
  if (sweeps_done < 0)
  for (Index idx = threadIdx.x; idx < Index(Rp) * Rp; idx += blockDim.x) {
    const int i = int(idx % Rp), j = int(idx / Rp);
    double s = 0;
    if (i < R && j < R) {
      const int l0 = i > j ? i : j;
      for (int l = l0; l < R; ++l) s += Rx[i + Index(l) * ldx] * Ry[j + Index(l) * ldy];
    }
    S[idx] = s;
    Vm[idx] = (i == j) ? 1.0 : 0.0;
  }
  __syncthreads();
  const double tol = DBL_EPSILON * double(Rp);  // LAPACK dgesvj-style relative stop
  int sweep = 0;
  if (sweeps_done >= 0) {
    sweep = sweeps_done;
  } else if (Rp <= warp_variant_max) {
    // One warp; lane i owns pair i of the round-robin round (<= 32 disjoint pairs), so
    // the whole round runs without block barriers or shuffle reductions.
    if (warp == 0) {
      for (; sweep < 60; ++sweep) {
        bool any_rot = false;
        for (int rd = 0; rd < Rp - 1; ++rd) {
          if (lane < Rp / 2) {
            int p, q;
            rr_pair(rd, lane, Rp, p, q);
            double* sp = S + Index(p) * Rp;
            double* sq = S + Index(q) * Rp;
            double al = 0, be = 0, ga = 0;
            for (int i = 0; i < Rp; ++i) {
              const double x = sp[i], y = sq[i];
              al += x * x;
              be += y * y;
              ga += x * y;
            }
            double cs, sn;
            if (jacobi_rotation(al, be, ga, tol, cs, sn)) {
              for (int i = 0; i < Rp; ++i) {
                const double x = sp[i], y = sq[i];
                sp[i] = cs * x - sn * y;
                sq[i] = sn * x + cs * y;
              }
              double* vp = Vm + Index(p) * Rp;
              double* vq = Vm + Index(q) * Rp;
              for (int i = 0; i < Rp; ++i) {
                const double x = vp[i], y = vq[i];
                vp[i] = cs * x - sn * y;
                vq[i] = sn * x + cs * y;
              }
              any_rot = true;
            }
          }
          __syncwarp();
        }
        if (!__any_sync(0xffffffffu, any_rot)) break;
      }
      if (lane == 0) rotated = sweep;
    }
    __syncthreads();
    sweep = rotated;
  } else if (Rp / 2 > nw) {
    // More pairs than warps (Rp > 64 at 1024 threads): one half-warp per pair, so a round
    // is one pass instead of two. Loops are warp-uniform (full-mask shuffles); a half-warp
    // without a pair computes nothing it keeps.
    const int hl = lane & 15, half = lane >> 4;
    for (; sweep < 60; ++sweep) {
      if (threadIdx.x == 0) rotated = 0;
      __syncthreads();
      for (int rd = 0; rd < Rp - 1; ++rd) {
        for (int base = warp; 2 * base < Rp / 2; base += nw) {
          const int pi = 2 * base + half;
          const bool valid = pi < Rp / 2;
          int p = 0, q = 1;
          if (valid) rr_pair(rd, pi, Rp, p, q);
          double* sp = S + Index(p) * Rp;
          double* sq = S + Index(q) * Rp;
          double al = 0, be = 0, ga = 0;
          if (valid)
            for (int i = hl; i < Rp; i += 16) {
              const double x = sp[i], y = sq[i];
              al += x * x;
              be += y * y;
              ga += x * y;
            }
#pragma unroll
          for (int o = 8; o > 0; o >>= 1) {
            al += __shfl_xor_sync(0xffffffffu, al, o);
            be += __shfl_xor_sync(0xffffffffu, be, o);
            ga += __shfl_xor_sync(0xffffffffu, ga, o);
          }
          double cs, sn;
          if (valid && jacobi_rotation(al, be, ga, tol, cs, sn)) {
            for (int i = hl; i < Rp; i += 16) {
              const double x = sp[i], y = sq[i];
              sp[i] = cs * x - sn * y;
              sq[i] = sn * x + cs * y;
            }
            double* vp = Vm + Index(p) * Rp;
            double* vq = Vm + Index(q) * Rp;
            for (int i = hl; i < Rp; i += 16) {
              const double x = vp[i], y = vq[i];
              vp[i] = cs * x - sn * y;
              vq[i] = sn * x + cs * y;
            }
            if (hl == 0) rotated = 1;
          }
        }
        __syncthreads();
      }
      if (!rotated) break;
      __syncthreads();
    }
  } else
  for (; sweep < 60; ++sweep) {
    if (threadIdx.x == 0) rotated = 0;
    __syncthreads();
    for (int rd = 0; rd < Rp - 1; ++rd) {
      for (int pi = warp; pi < Rp / 2; pi += nw) {
        int p, q;
        rr_pair(rd, pi, Rp, p, q);
        double* sp = S + Index(p) * Rp;
        double* sq = S + Index(q) * Rp;
        double al = 0, be = 0, ga = 0;
        for (int i = lane; i < Rp; i += 32) {
          const double x = sp[i], y = sq[i];
          al += x * x;
          be += y * y;
          ga += x * y;
        }
        al = warp_sum(al);
        be = warp_sum(be);
        ga = warp_sum(ga);
        double cs, sn;
        if (jacobi_rotation(al, be, ga, tol, cs, sn)) {
          for (int i = lane; i < Rp; i += 32) {
            const double x = sp[i], y = sq[i];
            sp[i] = cs * x - sn * y;
            sq[i] = sn * x + cs * y;
          }
          double* vp = Vm + Index(p) * Rp;
          double* vq = Vm + Index(q) * Rp;
          for (int i = lane; i < Rp; i += 32) {
            const double x = vp[i], y = vq[i];
            vp[i] = cs * x - sn * y;
            vq[i] = sn * x + cs * y;
          }
          if (lane == 0) rotated = 1;
        }
      }
      __syncthreads();
    }
    if (!rotated) break;
    __syncthreads();
  }
  for (int j = warp; j < Rp; j += nw) {
    const double* sj = S + Index(j) * Rp;
    double s = 0;
    for (int i = lane; i < Rp; i += 32) s += sj[i] * sj[i];
    s = warp_sum(s);
    if (lane == 0) sg[j] = sqrt(s);
  }
  __syncthreads();
  for (int j = threadIdx.x; j < Rp; j += blockDim.x) {
    int p = 0;
    const double v = sg[j];
    for (int i = 0; i < Rp; ++i) p += (sg[i] > v) || (sg[i] == v && i < j);
    pos[j] = p;
  }
  __syncthreads();
  for (Index idx = threadIdx.x; idx < Index(Rp) * R; idx += blockDim.x) {
    const int i = int(idx % Rp), j = int(idx / Rp);
    const int pj = pos[j];
    if (pj < R && i < R) {
      A[i + Index(pj) * R] = S[i + Index(j) * Rp];
      B[i + Index(pj) * R] = Vm[i + Index(j) * Rp];
    }
  }
  for (int j = threadIdx.x; j < Rp; j += blockDim.x)
    if (pos[j] < R) sigma[pos[j]] = sg[j];
  __syncthreads();
  if (threadIdx.x == 0) {
    // sorted singular values: sigma[0..R-1] written by this CTA (global), re-read after fence
    __threadfence_block();
    dd ssum{0, 0};
    for (int k = 0; k < R; ++k) ssum = dd_add(ssum, two_prod(sigma[k], sigma[k]));
    if (hidden_rel > 0.0) hidden_tail += hidden_rel * ssum.hi;
    const dd total = dd_add(dd{hidden_tail, 0}, ssum);
    if (hidden_rel >= 0.0) {
      info[4] = 0.0;
      info[5] = dd_to_d(total);
    }
    double keep_d, margin = INFINITY;
    if (total.hi == 0.0) {
      keep_d = 0;  // all-zero input -> canonical zero TT
    } else {
      const double e = 0.9 * eps;
      const dd budget = dd_mul(two_prod(e, e), total);
      int keep = R;
      dd tail{hidden_tail, 0};  // energy of the QRCP-truncated block (all below the budget)
      while (keep > 1) {
        const double s = sigma[keep - 1];
        const dd s2 = two_prod(s, s);
        const dd cand = dd_add(tail, s2);
        if (s != 0 && dd_gt(cand, budget)) {
          if (budget.hi > 0) margin = fmin(margin, (dd_to_d(cand) - dd_to_d(budget)) / dd_to_d(budget));
          break;
        }
        tail = cand;
        if (s != 0 && budget.hi > 0) {
          const dd diff = dd_add(budget, dd{-tail.hi, -tail.lo});
          margin = fmin(margin, dd_to_d(diff) / dd_to_d(budget));
        }
        --keep;
      }
      keep_d = keep;
      if (hidden_tail > 0) {  // the same decision without the hidden energy: equal -> exact
        int keep_lo = R;
        dd tl{0, 0};
        while (keep_lo > 1) {
          const double s = sigma[keep_lo - 1];
          const dd cand = dd_add(tl, two_prod(s, s));
          if (s != 0 && dd_gt(cand, budget)) break;
          tl = cand;
          --keep_lo;
        }
        info[4] = (keep_lo != keep) ? 1.0 : 0.0;
      }
    }
    double nx2 = 0, ny2 = 0;
    for (int w = 0; w < nw; ++w) {
      nx2 += red[0][w];
      ny2 += red[1][w];
    }
    info[0] = keep_d;
    info[1] = margin;
    info[2] = sweep;
    info[3] = total.hi > 0 ? sqrt(nx2) * sqrt(ny2) / sqrt(dd_to_d(total)) : INFINITY;
  }
}

template <bool SMEM>
__global__ void __launch_bounds__(kThreads) k_svd_small(const double* __restrict__ Rx, const double* __restrict__ Ry,
                                                        int R, double eps, double* gwork, double* A, double* B,
                                                        double* sigma, double* info) {
  extern __shared__ double smem[];
  cta_svd(Rx, R, Ry, R, R, eps, SMEM ? smem : gwork, A, B, sigma, info);
}

/// out (nr x kc, ld ldo; global) = Q [C; 0] with Q = H_0 ... H_{q-1} stored as reflectors
/// below the diagonal of `a` (ld lda) and tau; C is R x kc (ld ldc).
__device__ void cta_apply_q(const double* a, Index lda, const double* tau, Index nr, int R, const double* C, Index ldc,
                            int kc, double* out, Index ldo) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const Index top = nr < R ? nr : R;
  for (Index idx = threadIdx.x; idx < nr * kc; idx += blockDim.x) {
    const Index i = idx % nr, j = idx / nr;
    out[i + j * ldo] = i < top ? C[i + j * ldc] : 0.0;
  }
  __syncthreads();
  for (int j = warp; j < kc; j += nw) {  // independent output columns: no block barriers
    double* cj = out + Index(j) * ldo;
    for (int k = int(top) - 1; k >= 0; --k) {
      const double t = tau[k];
      if (t == 0.0) continue;
      const double* v = a + Index(k) * lda;
      double w = 0;
      for (Index i = k + 1 + lane; i < nr; i += 32) w += v[i] * cj[i];
      w = warp_sum(w);
      w = (cj[k] + w) * t;
      __syncwarp();
      if (lane == 0) cj[k] -= w;
      for (Index i = k + 1 + lane; i < nr; i += 32) cj[i] -= w * v[i];
      __syncwarp();
    }
  }
  __syncthreads();
}

/// Fused rounding of one lazy TT per CTA (SURVEY §7 K2+K3+K4): the input panels are
/// evaluated from the term list straight into shared memory, Householder-QR'd in place,
/// S = R_x R_y^T is SVD'd with on-device truncation, and Q_x (SV)_k / Q_y V_k are written
/// to the output cores. Requires m, n >= R and both panels resident in shared memory.
__global__ void __launch_bounds__(1024) k_round_fused(const RoundJob* __restrict__ jobs,
                                                      const MapDesc* __restrict__ maps) {
  extern __shared__ double smem[];
  __shared__ double scratch[33];
  const RoundJob J = jobs[blockIdx.x];
  const Index m = J.m, n = J.n;
  const int R = J.R;
  const int Rp = R + (R & 1);
  double* ax = smem;
  double* ay = ax + m * R;
  double* tx = ay + n * R;
  double* ty = tx + R;
  double* work = ty + R;
  for (Index idx = threadIdx.x; idx < m * R; idx += blockDim.x)
    ax[idx] = expr_value(J.terms, J.nterms, maps, 0, idx % m, idx / m);
  for (Index idx = threadIdx.x; idx < n * R; idx += blockDim.x)
    ay[idx] = expr_value(J.terms, J.nterms, maps, 1, idx % n, idx / n);
  __syncthreads();
  cta_householder_qr(ax, m, m, R, tx, scratch);
  cta_householder_qr(ay, n, n, R, ty, scratch);
  cta_svd(ax, m, ay, n, R, J.eps, work, J.A, J.B, J.sigma, J.info);
  __syncthreads();
  const int k = int(J.info[0]);
  if (k == 0) {  // all-zero input: canonical rank-1 zero cores
    for (Index i = threadIdx.x; i < m; i += blockDim.x) J.Xout[i] = 0.0;
    for (Index i = threadIdx.x; i < n; i += blockDim.x) J.Ytout[i] = 0.0;
    return;
  }
  (void)Rp;
  cta_apply_q(ax, m, tx, m, R, J.A, R, k, J.Xout, m);
  cta_apply_q(ay, n, ty, n, R, J.B, R, k, J.Ytout, n);
}

/// S = Rx Ry^T (R x R, both factors upper triangular with explicit zeros, ld R) by 32 x 32
/// output tiles, plus per-tile partial sums of ||Rx||^2, ||Ry||^2 (first tile row/column)
/// and ||S||^2 in part[3 * tile] (summed in fixed order by k_svd_qrcp).
__device__ void form_s_tile(const double* __restrict__ Rx, Index ldx, const double* __restrict__ Ry, Index ldy,
                            int R, double* __restrict__ S, double* __restrict__ part, int bx, int by, int tiles) {
  __shared__ double As[32][33], Bs[32][33];
  __shared__ double red[3][8];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int i0 = bx * 32, j0 = by * 32;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  const int lstart = (max(i0, j0) / 32) * 32;
  for (int l0 = lstart; l0 < R; l0 += 32) {
    for (int e = threadIdx.x; e < 32 * 32; e += 256) {
      const int r = e & 31, l = e >> 5;
      As[l][r] = (i0 + r < R && l0 + l < R) ? Rx[(i0 + r) + Index(l0 + l) * ldx] : 0.0;
      Bs[l][r] = (j0 + r < R && l0 + l < R) ? Ry[(j0 + r) + Index(l0 + l) * ldy] : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int l = 0; l < 32; ++l) {
      const double a = As[l][tx];
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[q] += a * Bs[l][ty + 8 * q];
    }
    __syncthreads();
  }
  double ps = 0.0, px = 0.0, py = 0.0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int i = i0 + tx, j = j0 + ty + 8 * q;
    if (i < R && j < R) {
      S[i + Index(j) * R] = acc[q];
      ps += acc[q] * acc[q];
    }
  }
  // ||Rx||^2 over this tile row (blockIdx.y == 0), ||Ry||^2 over this tile column (blockIdx.x == 0)
  if (by == 0)
    for (int l = ty; l < R; l += 8)
      if (i0 + tx < R && i0 + tx <= l) {
        const double a = Rx[(i0 + tx) + Index(l) * ldx];
        px += a * a;
      }
  if (bx == 0)
    for (int l = ty; l < R; l += 8)
      if (j0 + tx < R && j0 + tx <= l) {
        const double b = Ry[(j0 + tx) + Index(l) * ldy];
        py += b * b;
      }
  ps = warp_sum(ps);
  px = warp_sum(px);
  py = warp_sum(py);
  if (tx == 0) {
    red[0][ty] = px;
    red[1][ty] = py;
    red[2][ty] = ps;
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += red[threadIdx.x][w];
    part[3 * (bx + Index(by) * tiles) + threadIdx.x] = t;
  }
}

/// One large-R SVD request of a batch (k_form_s_batch / k_svd_qrcp_batch: one job per
/// grid z-slice / CTA).
struct SvdJob {
  const double* Rx;
  const double* Ry;
  int R;
  double eps;
  double* A;
  double* B;
  double* sigma;
  double* info;
  double* ws;
  int* perm;
  double* S;
  double* part;
  int tiles;
  long long* prof;
  double* qinfo;  // cluster QRCP result {p1, p2, hidden1, hidden2} (null: the CTA pivots itself)
  double* ainfo;  // {p, k} for k_qrcp_apply_batch (null: the SVD CTA applies Q itself)
  const double* hidden_rel;  // SvdRequest::hidden_rel
  double* cinfo;  // cluster Jacobi hand-over {state (1: sweeps pending / done), sweeps, p} (null: never split)
};

__global__ void __launch_bounds__(256) k_form_s_batch(const SvdJob* __restrict__ jobs) {
  const SvdJob& J = jobs[blockIdx.z];
  if (int(blockIdx.x) >= J.tiles || int(blockIdx.y) >= J.tiles) return;
  form_s_tile(J.Rx, J.R, J.Ry, J.R, J.R, J.S, J.part, blockIdx.x, blockIdx.y, J.tiles);
}

constexpr double kQrcpFirstStop = 1e-3;  // first-pass QRCP stop (fraction of the budget)

/// Stop levels of the pivoted-QR pre-truncation, as fractions of the truncation budget
/// (0.9 eps)^2 ||S||^2. The hidden trailing energy E moves the kept singular vectors by
/// about sqrt(E) = sqrt(stop) 0.9 eps ||S||, so the levels are capped to keep that below
/// 3e-12 ||S|| whatever eps is (at eps = 1e-10 the cap is 1.1e-3, i.e. the default first
/// stop; at policy-mode tolerances ~1e-6 the pivoted QR runs much further).
__device__ inline void qrcp_stops(double eps, double first, double& s1, double& s2) {
  const double e9 = 0.9 * eps;
  const double cap = e9 > 0.0 ? (3e-12 / e9) * (3e-12 / e9) : first;
  s1 = fmin(first, cap);
  s2 = fmin(1e-6, 1e-3 * s1);
}
constexpr int kQrcpRegRows = 16;  // rows per lane kept in registers by the QRCP column pass (R <= 512)
constexpr int kJcC = 8;        // CTAs of the cluster Jacobi (k_jacobi_cluster)
constexpr int kJcMinP = 96;    // first-pass factors below this stay in the single SVD CTA
constexpr int kJcMaxRp = 320;  // and above this (kJcC x 225 KB holds S and V up to Rp = 320)

/// SVD of S = Rx Ry^T (formed by k_form_s) for large R, pre-truncated by column-pivoted
/// Householder QR: the pivoted QR stops at the first p whose trailing column energy E_p is
/// <= 1e-6 of the truncation budget (0.9 eps)^2 ||S||^2; the p x R leading block is
/// reduced by an LQ step to the p x p factor L, whose one-sided Jacobi SVD (in shared
/// memory when it fits) takes the truncation decision of cta_svd with E_p carried as
/// hidden tail energy (identical decisions except inside the ill-posed band of the parity
/// contract). Each QRCP step is one pass over the trailing columns that applies the
/// reflector and recomputes the exact tail norms from the same registers. Outputs
/// A = Q1 [(L V)_k; 0] and B = Q_l V_k (R x k, ld R) like cta_svd.
__device__ void svd_qrcp_body(double* S, const double* __restrict__ part, int nparts, int R, double eps,
                              double* ws, int* perm, double* A, double* B, double* sigma, double* info,
                              long long* prof, size_t smem_bytes, const double* qinfo, double* ainfo,
                              const double* hidden_rel, double* vremote = nullptr, int mode = 0,
                              double* cinfo = nullptr) {
  // mode 0: the whole SVD. mode 1: as mode 0 unless the first-pass factor is large enough for
  // the cluster Jacobi (k_jacobi_cluster): then S = L and V = I are written to the global work
  // area, cinfo = {1, -, p} and the CTA returns. mode 2: nothing unless cinfo[0] == 1: then the
  // first pass continues after the sweeps (cinfo[1]) that k_jacobi_cluster ran.
  if (mode == 2 && !(cinfo && cinfo[0] == 1.0)) return;
  if (mode == 1 && cinfo && threadIdx.x == 0) cinfo[0] = 0.0;  // until the first pass decides to split
  extern __shared__ double dsm[];
  __shared__ double scratch[33];
  __shared__ double sh_bv;
  __shared__ int sh_bj, sh_stop;
  if (prof && threadIdx.x == 0) prof[0] = clock64();
  if (ainfo && threadIdx.x == 0) ainfo[1] = 0;  // nothing to apply unless set at the end
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const Index RR = Index(R) * R;
  double* Tt = ws;          // R x p (ld R)
  double* cn = Tt + RR;     // R
  double* tau1 = cn + R;    // R
  double* taul = tau1 + R;  // R
  double* Id = taul + R;    // R x R identity (p x p used)
  double* As = Id + RR;     // p x p
  double* Bs = As + RR;     // p x p
  double* gwork = Bs + RR;  // 2 Rp^2 + 2 Rp  (Rp <= R + 1)
  double* info2 = gwork + 2 * Index(R + 1) * (R + 1) + 2 * (R + 1) + 8;
  double* vk = dsm;         // reflector of the current step (R), shared
  // the pivoted QR works on S in shared memory when it fits (written back for the apply)
  double* const Sg = S;
  // qinfo: the pivoted QR already ran on a thread-block cluster (k_qrcp_cluster), S holds
  // its result; both stop levels {p1, p2} and hidden energies are given
  const bool s_shared = !qinfo && (size_t(R) * R + size_t(R)) * sizeof(double) <= smem_bytes;
  if (s_shared) {
    S = dsm + R;
    for (Index idx = threadIdx.x; idx < RR; idx += blockDim.x) S[idx] = Sg[idx];
    __syncthreads();
  }
  double nx2 = 0, ny2 = 0, total2 = 0;
  for (int i = 0; i < nparts; ++i) {
    nx2 += part[3 * i];
    ny2 += part[3 * i + 1];
    total2 += part[3 * i + 2];
  }
  const double e9 = 0.9 * eps;
  const double budget = e9 * e9 * total2;
  // energy the sketch did not capture (4 x the probe estimate), carried with the pivoted QR's own
  const double hidden_ext = hidden_rel ? 4.0 * (*hidden_rel) * total2 : 0.0;
  // first pass stops at trailing energy <= 1e-3 of the budget (smaller Jacobi; the outputs
  // move by <= sqrt(1e-3) ~ 3 % of the truncation error); only when that hidden energy
  // could change the rank does the pivoted QR resume to 1e-6 and the SVD repeat
  double stop1, stop2;
  qrcp_stops(eps, kQrcpFirstStop, stop1, stop2);
  double stop_energy = stop1 * budget;
  if (!qinfo) {
    for (int j = threadIdx.x; j < R; j += blockDim.x) perm[j] = j;
    for (int j = warp; j < R; j += nw) {
      const double* c = S + Index(j) * R;
      double t = 0;
      for (int i = lane; i < R; i += 32) t += c[i] * c[i];
      t = warp_sum(t);
      if (lane == 0) cn[j] = t;
    }
  }
  __syncthreads();
  int p = R;
  int kdone = 0;
  for (int pass = 0; pass < 2; ++pass) {
  double hidden = 0.0;
  if (qinfo) {
    p = int(qinfo[pass]);
    hidden = qinfo[2 + pass];
  } else {
  if (pass == 1 && s_shared) {  // resume on the shared copy
    S = dsm + R;
    for (Index idx = threadIdx.x; idx < RR; idx += blockDim.x) S[idx] = Sg[idx];
    __syncthreads();
  }
  p = R;
  for (int k = kdone; k < R; ++k) {
    // pivot: largest trailing column energy (first index on ties), stop on the total
    if (warp == 0) {
      double bv = -1.0, e = 0.0;
      int bj = R;
      for (int j = k + lane; j < R; j += 32) {
        const double v = cn[j];
        e += v;
        if (v > bv) {
          bv = v;
          bj = j;
        }
      }
      e = warp_sum(e);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
        if (ov > bv || (ov == bv && oj < bj)) {
          bv = ov;
          bj = oj;
        }
      }
      if (lane == 0) {
        sh_stop = (e <= stop_energy) ? 1 : 0;
        sh_bv = e;
        sh_bj = bj;
      }
    }
    __syncthreads();
    if (prof && threadIdx.x == 0) {  // first k whose trailing energy is below 1e-2 / 1e-4 of the budget
      if (prof[8] == 0 && sh_bv <= 1e-2 * budget) prof[8] = k;
      if (prof[9] == 0 && sh_bv <= 1e-4 * budget) prof[9] = k;
    }
    if (sh_stop) {
      p = k;
      break;
    }
    const int bj = sh_bj;
    if (bj != k) {
      for (int i = threadIdx.x; i < R; i += blockDim.x) {
        const double t = S[i + Index(k) * R];
        S[i + Index(k) * R] = S[i + Index(bj) * R];
        S[i + Index(bj) * R] = t;
      }
      if (threadIdx.x == 0) {
        const int t = perm[k];
        perm[k] = perm[bj];
        perm[bj] = t;
        const double c = cn[k];
        cn[k] = cn[bj];
        cn[bj] = c;
      }
    }
    __syncthreads();
    // Householder on column k (rows k..R-1), same convention as cta_householder_qr
    double* ak = S + Index(k) * R;
    double part2 = 0;
    for (int i = k + 1 + threadIdx.x; i < R; i += blockDim.x) part2 += ak[i] * ak[i];
    const double tail2 = block_sum(part2, scratch);
    const double c0 = ak[k];
    double t, beta, d;
    if (tail2 <= DBL_MIN) {
      t = 0.0;
      beta = c0;
      d = 1.0;
    } else {
      beta = sqrt(c0 * c0 + tail2);
      if (c0 >= 0) beta = -beta;
      d = c0 - beta;
      t = (beta - c0) / beta;
    }
    for (int i = k + 1 + threadIdx.x; i < R; i += blockDim.x) {
      const double v = (t == 0.0) ? 0.0 : ak[i] / d;
      ak[i] = v;
      vk[i] = v;
    }
    if (threadIdx.x == 0) {
      vk[k] = 1.0;
      tau1[k] = t;
    }
    __syncthreads();
    if (threadIdx.x == 0) ak[k] = beta;
    // trailing columns: apply H_k and recompute the exact tail energy (rows > k) from the
    // same registers (one pass per column, loads issued before the reductions)
    const int nrow = R - k;
    for (int j = k + 1 + warp; j < R; j += nw) {
      double* aj = S + Index(j) * R + k;
      if (nrow <= 32 * kQrcpRegRows) {
        double x[kQrcpRegRows];
#pragma unroll
        for (int q = 0; q < kQrcpRegRows; ++q) {
          const int i = lane + 32 * q;
          x[q] = i < nrow ? aj[i] : 0.0;
        }
        if (t != 0.0) {
          double w = 0.0;
#pragma unroll
          for (int q = 0; q < kQrcpRegRows; ++q) {
            const int i = lane + 32 * q;
            if (i < nrow) w += vk[k + i] * x[q];
          }
          w = warp_sum(w) * t;
#pragma unroll
          for (int q = 0; q < kQrcpRegRows; ++q) {
            const int i = lane + 32 * q;
            if (i < nrow) {
              x[q] -= w * vk[k + i];
              aj[i] = x[q];
            }
          }
        }
        double e = 0.0;
#pragma unroll
        for (int q = 0; q < kQrcpRegRows; ++q) {
          const int i = lane + 32 * q;
          if (i >= 1 && i < nrow) e += x[q] * x[q];
        }
        e = warp_sum(e);
        if (lane == 0) cn[j] = e;
      } else {
        if (t != 0.0) {
          double w = 0.0;
          for (int i = lane; i < nrow; i += 32) w += vk[k + i] * aj[i];
          w = warp_sum(w) * t;
          for (int i = lane; i < nrow; i += 32) aj[i] -= w * vk[k + i];
        }
        double e = 0.0;
        for (int i = 1 + lane; i < nrow; i += 32) e += aj[i] * aj[i];
        e = warp_sum(e);
        if (lane == 0) cn[j] = e;
      }
    }
    __syncthreads();
  }
  __syncthreads();
  hidden = (p < R) ? sh_bv : 0.0;
  }
  if (s_shared) {  // reflectors and R1 back to global memory (cta_apply_q reads them last)
    __syncthreads();
    for (Index idx = threadIdx.x; idx < RR; idx += blockDim.x) Sg[idx] = S[idx];
    __syncthreads();
    S = Sg;
  }
  if (prof && threadIdx.x == 0) {
    prof[1] = clock64();
    prof[6] = p;
  }
  if (p == 0) {  // all energy below the stop level: only possible for S == 0 (budget 0) or tiny eps
    if (threadIdx.x == 0) {
      info[0] = total2 == 0.0 ? 0 : 1;
      info[1] = INFINITY;
      info[2] = 0;
      info[3] = INFINITY;
      if (hidden_rel) {
        info[4] = 0;
        info[5] = total2;
      }
    }
    // rank-1 fallback: leading column of S (rarely reached; exact zero handled by k = 0)
    for (int i = threadIdx.x; i < R; i += blockDim.x) {
      A[i] = 0.0;
      B[i] = (i == 0) ? 1.0 : 0.0;
    }
    return;
  }
  for (Index idx = threadIdx.x; idx < Index(p) * p; idx += blockDim.x) {
    const int i = int(idx % p), j = int(idx / p);
    Id[idx] = (i == j) ? 1.0 : 0.0;
  }
  const bool lq_done = qinfo && pass == 0 && qinfo[8] == 1.0;  // k_lq_cluster factored Tt
  if (!lq_done) {
  // Tt (R x p): Tt[perm[j] + i R] = R1[i, j] for j >= i, i < p
  for (Index idx = threadIdx.x; idx < Index(R) * p; idx += blockDim.x) {
    const int j = int(idx % R), i = int(idx / R);
    Tt[perm[j] + Index(i) * R] = (j >= i) ? S[i + Index(j) * R] : 0.0;
  }
  }
  __syncthreads();
  if (lq_done) {
  } else if (size_t(R) * p * sizeof(double) <= smem_bytes) {  // Tt = Q_l R_l in shared memory
    double* Ts = dsm;
    for (Index idx = threadIdx.x; idx < Index(R) * p; idx += blockDim.x) Ts[idx] = Tt[idx];
    __syncthreads();
    cta_householder_qr(Ts, R, R, p, taul, scratch);
    for (Index idx = threadIdx.x; idx < Index(R) * p; idx += blockDim.x) Tt[idx] = Ts[idx];
    __syncthreads();
  } else {
    cta_householder_qr(Tt, R, R, p, taul, scratch);  // Tt = Q_l R_l (R_l p x p upper in the top rows)
  }
  if (prof && threadIdx.x == 0) prof[2] = clock64();
  // L = R_l^T = Id * R_l^T: cta_svd(Rx = Id, Ry = R_l) forms Id R_l^T; Jacobi work in shared
  // memory when it fits, warp-per-pair rounds (block variant) at every size
  const int Rp = p + (p & 1);
  const size_t jac_bytes = (2 * size_t(Rp) * Rp + 2 * size_t(Rp)) * sizeof(double);
  const size_t half_bytes = (size_t(Rp) * Rp + 2 * size_t(Rp)) * sizeof(double);
  const double hid = hidden + hidden_ext;
  const bool split_ok = cinfo && pass == 0 && lq_done && p >= kJcMinP && Rp <= kJcMaxRp;
  if (mode == 1 && threadIdx.x == 0 && cinfo) cinfo[0] = split_ok ? 1.0 : 0.0;
  if (mode == 1 && split_ok) {
    // S = Id R_l^T = L (lower triangular) and V = I for k_jacobi_cluster, column-major ld Rp
    double* Sg = gwork;
    double* Vg = gwork + Index(Rp) * Rp;
    for (Index idx = threadIdx.x; idx < Index(Rp) * Rp; idx += blockDim.x) {
      const int i = int(idx % Rp), j = int(idx / Rp);
      Sg[idx] = (i < p && j <= i) ? Tt[j + Index(i) * R] : 0.0;
      Vg[idx] = (i == j) ? 1.0 : 0.0;
    }
    if (threadIdx.x == 0) cinfo[2] = p;
    return;
  }
  if (mode == 2 && pass == 0)
    cta_svd(Id, p, Tt, R, p, eps, gwork, As, Bs, sigma, info2, hid, 0, nullptr, 0.0, int(cinfo[1]));
  else if (jac_bytes <= smem_bytes)  // S and V shared
    cta_svd(Id, p, Tt, R, p, eps, dsm, As, Bs, sigma, info2, hid, 0, nullptr, 0.0);
  else if (half_bytes <= smem_bytes)  // S shared, V in global memory
    cta_svd(Id, p, Tt, R, p, eps, dsm, As, Bs, sigma, info2, hid, 0, vremote ? vremote : gwork, 0.0);
  else
    cta_svd(Id, p, Tt, R, p, eps, gwork, As, Bs, sigma, info2, hid, 0, nullptr, 0.0);
  __syncthreads();
  if (pass == 0 && p < R && info2[4] != 0.0 && !(qinfo && qinfo[1] == qinfo[0])) {  // ambiguous: tighten, repeat
    kdone = p;
    stop_energy = stop2 * budget;
    continue;
  }
  break;
  }
  __syncthreads();
  if (prof && threadIdx.x == 0) {
    prof[3] = clock64();
    prof[7] = (long long)info2[2];
  }
  const int kk = int(info2[0]);
  if (threadIdx.x == 0) {
    info[0] = kk;
    info[1] = info2[1];
    info[2] = info2[2];
    info[3] = total2 > 0 ? sqrt(nx2) * sqrt(ny2) / sqrt(total2) : INFINITY;
    if (hidden_rel) {
      info[4] = info2[4];
      info[5] = total2;
    }
  }
  if (kk == 0) return;
  if (ainfo) {  // the Q applications run on many CTAs (k_qrcp_apply_batch)
    if (threadIdx.x == 0) {
      ainfo[0] = p;
      ainfo[1] = kk;
    }
    return;
  }
  // A = Q1 [As_k; 0], B = Q_l [Bs_k; 0]   (R x kk, ld R)
  cta_apply_q(S, R, tau1, R, p, As, p, kk, A, R);
  __syncthreads();
  cta_apply_q(Tt, R, taul, R, p, Bs, p, kk, B, R);
  __syncthreads();
  if (prof && threadIdx.x == 0) prof[4] = clock64();
}

/// Launched as clusters of two CTAs per job: rank 0 runs the SVD; when the Jacobi's S and V do
/// not both fit one SM's shared memory (p > ~106), V lives in rank 1's shared memory and is
/// rotated through distributed shared memory instead of global memory (rank 1 only lends it).
__global__ void __launch_bounds__(1024) k_svd_qrcp_batch(const SvdJob* __restrict__ jobs, size_t smem_bytes,
                                                         int mode) {
  extern __shared__ double dsm_k[];
  cg::cluster_group cl = cg::this_cluster();
  const bool paired = cl.num_blocks() == 2;
  const SvdJob& J = jobs[paired ? blockIdx.x / 2 : blockIdx.x];
  if (paired) cl.sync();  // both CTAs run before either touches the other's shared memory
  if (!paired || cl.block_rank() == 0)
    svd_qrcp_body(J.S, J.part, J.tiles * J.tiles, J.R, J.eps, J.ws, J.perm, J.A, J.B, J.sigma, J.info, J.prof,
                  smem_bytes, J.qinfo, J.ainfo, J.hidden_rel, paired ? cl.map_shared_rank(dsm_k, 1) : nullptr, mode,
                  J.cinfo);
  if (paired) cl.sync();  // rank 1 keeps its shared memory alive until rank 0 is done
}

/// The one-sided Jacobi sweeps of a large first-pass factor (kJcMinP <= p, Rp <= kJcMaxRp) on a
/// thread-block cluster of kJcC CTAs: columns j of S and V live in CTA j % kJcC's shared
/// memory; every round of the round-robin ordering gives each CTA Rp / 2 / kJcC disjoint column
/// pairs (one warp per pair, both columns in registers between the Gram entries and the
/// rotation), read and written through distributed shared memory, and ends in one cluster
/// barrier. A single CTA is bound by its shared-memory bandwidth and FP64 issue (p = 160: 9 ms,
/// p = 210: 25 ms, profiles/r02i); here the same rotations run on kJcC SMs. The sweep count is
/// handed to the second k_svd_qrcp_batch launch through cinfo[1].
constexpr int kJcThreads = 512;
constexpr int kJcRegs = kJcMaxRp / 32;
__global__ void __launch_bounds__(kJcThreads, 1) k_jacobi_cluster(const SvdJob* __restrict__ jobs) {
  extern __shared__ double jsm[];
  __shared__ int rot;
  cg::cluster_group cl = cg::this_cluster();
  const int rank = int(cl.block_rank());
  const SvdJob& J = jobs[blockIdx.x / kJcC];
  if (!J.cinfo || J.cinfo[0] != 1.0) return;  // uniform over the cluster: no barrier was entered
  const int p = int(J.cinfo[2]);
  const int Rp = p + (p & 1);
  const int ncl = (Rp + kJcC - 1) / kJcC;
  const Index RR = Index(J.R) * J.R;
  double* Sg = J.ws + 4 * RR + 3 * J.R;  // gwork of svd_qrcp_body
  double* Vg = Sg + Index(Rp) * Rp;
  double* Sl = jsm;
  double* Vl = jsm + Index(ncl) * Rp;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int sl = warp; sl < ncl; sl += nw) {
    const int j = sl * kJcC + rank;
    for (int i = lane; i < Rp; i += 32) {
      Sl[Index(sl) * Rp + i] = j < Rp ? Sg[Index(j) * Rp + i] : 0.0;
      Vl[Index(sl) * Rp + i] = j < Rp ? Vg[Index(j) * Rp + i] : 0.0;
    }
  }
  if (threadIdx.x == 0) rot = 0;
  cl.sync();
  const double tol = DBL_EPSILON * double(Rp);
  int sweep = 0;
  for (; sweep < 60; ++sweep) {
    for (int rd = 0; rd < Rp - 1; ++rd) {
      for (int pi = rank + kJcC * warp; pi < Rp / 2; pi += kJcC * nw) {
        int cp, cq;
        rr_pair(rd, pi, Rp, cp, cq);
        double* sp = cl.map_shared_rank(Sl, cp % kJcC) + Index(cp / kJcC) * Rp;
        double* sq = cl.map_shared_rank(Sl, cq % kJcC) + Index(cq / kJcC) * Rp;
        double x[kJcRegs], y[kJcRegs];
        double al = 0, be = 0, ga = 0;
#pragma unroll
        for (int t = 0; t < kJcRegs; ++t) {
          const int i = lane + 32 * t;
          x[t] = i < Rp ? sp[i] : 0.0;
          y[t] = i < Rp ? sq[i] : 0.0;
          al += x[t] * x[t];
          be += y[t] * y[t];
          ga += x[t] * y[t];
        }
        al = warp_sum(al);
        be = warp_sum(be);
        ga = warp_sum(ga);
        double cs, sn;
        if (jacobi_rotation(al, be, ga, tol, cs, sn)) {
#pragma unroll
          for (int t = 0; t < kJcRegs; ++t) {
            const int i = lane + 32 * t;
            if (i < Rp) {
              sp[i] = cs * x[t] - sn * y[t];
              sq[i] = sn * x[t] + cs * y[t];
            }
          }
          double* vp = cl.map_shared_rank(Vl, cp % kJcC) + Index(cp / kJcC) * Rp;
          double* vq = cl.map_shared_rank(Vl, cq % kJcC) + Index(cq / kJcC) * Rp;
#pragma unroll
          for (int t = 0; t < kJcRegs; ++t) {
            const int i = lane + 32 * t;
            if (i < Rp) {
              const double a = vp[i], b = vq[i];
              vp[i] = cs * a - sn * b;
              vq[i] = sn * a + cs * b;
            }
          }
          if (lane == 0) rot = 1;
        }
      }
      cl.sync();
    }
    int any = 0;
    for (int r = 0; r < kJcC; ++r) any |= *cl.map_shared_rank(&rot, r);
    cl.sync();  // every CTA has read the flags of this sweep
    if (threadIdx.x == 0) rot = 0;
    __syncthreads();
    if (!any) break;
  }
  for (int sl = warp; sl < ncl; sl += nw) {
    const int j = sl * kJcC + rank;
    if (j < Rp)
      for (int i = lane; i < Rp; i += 32) {
        Sg[Index(j) * Rp + i] = Sl[Index(sl) * Rp + i];
        Vg[Index(j) * Rp + i] = Vl[Index(sl) * Rp + i];
      }
  }
  if (rank == 0 && threadIdx.x == 0) J.cinfo[1] = sweep;
  cl.sync();  // no CTA leaves while another may still access its shared memory
}

/// Column-pivoted Householder QR of S (R x R) on a thread-block cluster of C CTAs (one per
/// SM), S distributed over their shared memories by interleaved columns (column j lives in
/// CTA j % C). The single-CTA pivoted QR of svd_qrcp_body is bound by one SM's issue rate
/// and, above R ~ 165, by S living in global memory; here every step costs one cluster
/// barrier: each CTA publishes its best trailing column (energy, index) and its partial
/// trailing energy; every warp then reads the C candidates over DSMEM and takes the same
/// decision (largest energy, lowest index on ties; the energy sum in fixed rank order), every
/// CTA copies the pivot column from its owner and forms the reflector redundantly (identical
/// arithmetic everywhere), and updates its own trailing columns and their exact tail norms.
/// The pivot column itself is left untouched until the end, so no second barrier is
/// needed. The QR runs to the tighter stop level (stop2 * budget) and records the first
/// step at which the trailing energy is below stop1 * budget as well: the first p1 steps are
/// exactly the ones a run stopped at stop1 would take. Output in the layout the rest of
/// svd_qrcp_body expects: column s < p2 of S = pivot of step s (R above the diagonal, beta on
/// it, the reflector below), then the unpivoted columns in increasing original index, perm,
/// tau1 and qinfo = {p1, p2, hidden1, hidden2}.
constexpr int kQcThreads = 512;

__host__ __device__ inline size_t qrcp_cluster_smem(int R, int C) {
  const size_t nc = size_t((R + C - 1) / C);
  return (nc * size_t(R) + size_t(R) + 3 * nc + 8) * sizeof(double) + (size_t(R) + 2 * nc) * sizeof(int) +
         size_t(R) + 16;
}

__global__ void __launch_bounds__(kQcThreads, 1) k_qrcp_cluster(const SvdJob* __restrict__ jobs, double stop1,
                                                                double stop2) {
  cg::cluster_group cl = cg::this_cluster();
  const int C = int(cl.num_blocks());
  const int rank = int(cl.block_rank());
  const SvdJob& J = jobs[blockIdx.x / C];
  const int R = J.R;
  const int nc = (R + C - 1) / C;
  const int nl = (R - rank + C - 1) / C;  // own columns j = rank + l C, l < nl
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  extern __shared__ double sm[];
  double* A = sm;                       // own column l at A + l R
  double* vb = A + size_t(nc) * R;      // pivot column of the current step (rows k..R-1)
  double* cn = vb + R;                  // trailing energy (rows >= k) of own columns
  double* betl = cn + nc;               // beta and 1/(c0 - beta) of own pivoted columns
  double* invl = betl + nc;
  double* cand = invl + nc;             // 2 x {best energy, partial trailing energy, index, -}
  int* piv = reinterpret_cast<int*>(cand + 8);  // pivot (original column) of step s
  int* stepl = piv + R;                 // step at which own column l was pivoted (-1: not yet)
  int* posl = stepl + nc;               // output position of own column l
  unsigned char* done = reinterpret_cast<unsigned char*>(posl + nc);  // column j pivoted
  double* tau1 = J.ws + Index(R) * R + R;  // svd_qrcp_body's tau1
  const double* Sg = J.S;
  for (Index idx = threadIdx.x; idx < Index(nl) * R; idx += blockDim.x) {
    const int l = int(idx / R), i = int(idx % R);
    A[idx] = Sg[i + Index(rank + l * C) * R];
  }
  for (int j = threadIdx.x; j < R; j += blockDim.x) done[j] = 0;
  for (int l = threadIdx.x; l < nc; l += blockDim.x) stepl[l] = -1;
  __syncthreads();
  for (int l = warp; l < nl; l += nw) {
    const double* a = A + size_t(l) * R;
    double t = 0.0;
    for (int i = lane; i < R; i += 32) t += a[i] * a[i];
    t = warp_sum(t);
    if (lane == 0) cn[l] = t;
  }
  double total2 = 0.0;
  const int nparts = J.tiles * J.tiles;
  for (int i = 0; i < nparts; ++i) total2 += J.part[3 * i + 2];
  const double e9 = 0.9 * J.eps;
  const double budget = e9 * e9 * total2;
  double f1, f2;
  qrcp_stops(J.eps, stop1, f1, f2);
  (void)stop2;
  const double s1 = f1 * budget, s2 = f2 * budget;
  int p1 = -1, k = 0;
  double h1 = 0.0, h2 = 0.0;
  __syncthreads();
  for (; k < R; ++k) {
    double* cb = cand + 4 * (k & 1);
    if (warp == 0) {
      double bv = -1.0, es = 0.0;
      int bj = INT_MAX;
      for (int l = lane; l < nl; l += 32)
        if (stepl[l] < 0) {
          const double v = cn[l];
          const int j = rank + l * C;
          es += v;
          if (v > bv || (v == bv && j < bj)) {
            bv = v;
            bj = j;
          }
        }
      es = warp_sum(es);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
        if (ov > bv || (ov == bv && oj < bj)) {
          bv = ov;
          bj = oj;
        }
      }
      if (lane == 0) {
        cb[0] = bv;
        cb[1] = es;
        cb[2] = double(bj);
      }
    }
    cl.sync();
    // the global decision, taken identically by every warp of every CTA
    double bv = -1.0, e = 0.0;
    int bj = INT_MAX;
    if (lane < C) {
      const double* rc = cl.map_shared_rank(cb, lane);
      bv = rc[0];
      e = rc[1];
      bj = int(rc[2]);
    }
    e = warp_sum(e);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
      if (ov > bv || (ov == bv && oj < bj)) {
        bv = ov;
        bj = oj;
      }
    }
    if (p1 < 0 && e <= s1) {
      p1 = k;
      h1 = e;
    }
    if (e <= s2) {
      h2 = e;
      break;
    }
    const int owner = bj % C, lo = bj / C;
    if (threadIdx.x == 0) {
      piv[k] = bj;
      done[bj] = 1;
      if (rank == owner) stepl[lo] = k;
    }
    const double* src = cl.map_shared_rank(A + size_t(lo) * R, owner);
    for (int i = k + threadIdx.x; i < R; i += blockDim.x) vb[i] = src[i];
    __syncthreads();
    // reflector of the pivot column (Eigen's makeHouseholder convention, as cta_householder_qr)
    double t2 = 0.0;
    for (int i = k + 1 + lane; i < R; i += 32) t2 += vb[i] * vb[i];
    t2 = warp_sum(t2);
    const double c0 = vb[k];
    double tau, beta, d;
    if (t2 <= DBL_MIN) {
      tau = 0.0;
      beta = c0;
      d = 1.0;
    } else {
      beta = sqrt(c0 * c0 + t2);
      if (c0 >= 0) beta = -beta;
      d = c0 - beta;
      tau = (beta - c0) / beta;
    }
    const double invd = (tau == 0.0) ? 0.0 : 1.0 / d;
    if (threadIdx.x == 0) {
      if (rank == owner) {
        betl[lo] = beta;
        invl[lo] = invd;
      }
      if (rank == 0) tau1[k] = tau;
    }
    // own trailing columns: apply H_k, recompute the exact tail energy (rows > k)
    for (int l = warp; l < nl; l += nw) {
      if (stepl[l] >= 0) continue;
      double* a = A + size_t(l) * R;
      double en = 0.0;
      if (tau != 0.0) {
        double w = 0.0;
        for (int i = k + 1 + lane; i < R; i += 32) w += vb[i] * a[i];
        w = (a[k] + invd * warp_sum(w)) * tau;
        __syncwarp();
        if (lane == 0) a[k] -= w;
        const double wi = w * invd;
        for (int i = k + 1 + lane; i < R; i += 32) {
          const double x = a[i] - wi * vb[i];
          a[i] = x;
          en += x * x;
        }
      } else {
        for (int i = k + 1 + lane; i < R; i += 32) en += a[i] * a[i];
      }
      en = warp_sum(en);
      if (lane == 0) cn[l] = en;
    }
    __syncthreads();
  }
  const int p2 = k;
  if (p1 < 0) {
    p1 = p2;
    h1 = h2;
  }
  // output positions: pivots at their step, the rest after p2 in original order
  for (int l = threadIdx.x; l < nl; l += blockDim.x) {
    const int j = rank + l * C;
    if (stepl[l] >= 0) {
      posl[l] = stepl[l];
    } else {
      int c = 0;
      for (int q = 0; q < j; ++q) c += done[q] ? 0 : 1;
      posl[l] = p2 + c;
    }
  }
  __syncthreads();
  double* Sw = J.S;
  for (Index idx = threadIdx.x; idx < Index(nl) * R; idx += blockDim.x) {
    const int l = int(idx / R), i = int(idx % R);
    const int st = stepl[l];
    const double a = A[idx];
    double v = a;
    if (st >= 0 && i == st) v = betl[l];
    else if (st >= 0 && i > st) v = a * invl[l];
    Sw[i + Index(posl[l]) * R] = v;
  }
  if (rank == 0 && threadIdx.x == 0) {
    for (int s = 0; s < p2; ++s) J.perm[s] = piv[s];
    int c = p2;
    for (int j = 0; j < R; ++j)
      if (!done[j]) J.perm[c++] = j;
    J.qinfo[0] = p1;
    J.qinfo[1] = p2;
    J.qinfo[2] = h1;
    J.qinfo[3] = h2;
    J.qinfo[8] = 0.0;  // set by k_lq_cluster when it factors Tt
  }
  cl.sync();  // no CTA leaves while another may still read its candidates
}

/// The LQ step of svd_qrcp_body (Householder QR of Tt = R1^T, R x p, p = qinfo[0]) on the
/// same thread-block cluster layout as k_qrcp_cluster: row r of Tt (original column r of S)
/// lives in CTA r % C, so every CTA holds <= ceil(R / C) rows of p entries in shared memory.
/// Per column: one cluster barrier for the tail norm (CTA partials summed in rank order),
/// one for the trailing dot products w_j (CTA partial vectors summed in rank order); the
/// reflector and w are then identical in every CTA, which updates its own rows. Writes Tt
/// (R_l in the top rows, reflectors below, ld R) and taul as the single-CTA QR does and
/// sets qinfo[8] = 1 so svd_qrcp_body skips its own LQ in the first pass.
__host__ __device__ inline size_t lq_cluster_smem(int R, int C) {
  const size_t nc = size_t((R + C - 1) / C);
  return (nc * size_t(R + 1) + nc + size_t(R) + 8) * sizeof(double) + nc * sizeof(int) + 16;
}

__global__ void __launch_bounds__(kQcThreads, 1) k_lq_cluster(const SvdJob* __restrict__ jobs) {
  cg::cluster_group cl = cg::this_cluster();
  const int C = int(cl.num_blocks());
  const int rank = int(cl.block_rank());
  const SvdJob& J = jobs[blockIdx.x / C];
  if (!J.qinfo) return;  // uniform per cluster
  const int R = J.R;
  const int p = int(J.qinfo[0]);
  const int nc = (R + C - 1) / C;
  const int nl = (R - rank + C - 1) / C;  // own rows r = rank + l C
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (p <= 0) return;
  const int ld = R + 1;  // row stride of the local block (p <= R)
  extern __shared__ double sm[];
  double* T = sm;                        // own rows: T[l ld + i], i < p
  double* vl = T + size_t(nc) * ld;      // reflector entries of own rows (current column)
  double* dpart = vl + nc;               // this CTA's partial dot products (p)
  double* npart = dpart + R;             // {partial tail norm, c0 (owner of the diagonal)}
  int* posl = reinterpret_cast<int*>(npart + 8);  // position of own row r in the pivoted order
  const Index RR = Index(R) * R;
  double* Tt = J.ws;                     // svd_qrcp_body's layout
  double* taul = Tt + RR + 2 * R;
  const double* S = J.S;
  // own rows: Tt[r, i] = R1[i, pos(r)] for pos(r) >= i (perm[pos] = r)
  for (int q = threadIdx.x; q < R; q += blockDim.x) {
    const int r = J.perm[q];
    if (r % C == rank) posl[r / C] = q;
  }
  __syncthreads();
  for (Index idx = threadIdx.x; idx < Index(nl) * p; idx += blockDim.x) {
    const int l = int(idx / p), i = int(idx % p);
    const int pos = posl[l];
    T[l * ld + i] = (pos >= i) ? S[i + Index(pos) * R] : 0.0;
  }
  __syncthreads();
  for (int i = 0; i < p; ++i) {
    const int own_i = i % C, li = i / C;
    if (warp == 0) {
      double t = 0.0;
      for (int l = lane; l < nl; l += 32)
        if (rank + l * C > i) {
          const double x = T[l * ld + i];
          t += x * x;
        }
      t = warp_sum(t);
      if (lane == 0) {
        npart[0] = t;
        if (rank == own_i) npart[1] = T[li * ld + i];
      }
    }
    cl.sync();
    double tail2 = 0.0;
    if (lane < C) tail2 = cl.map_shared_rank(npart, lane)[0];
    tail2 = warp_sum(tail2);
    const double c0 = cl.map_shared_rank(npart, own_i)[1];
    double tau, beta, d;
    if (tail2 <= DBL_MIN) {
      tau = 0.0;
      beta = c0;
      d = 1.0;
    } else {
      beta = sqrt(c0 * c0 + tail2);
      if (c0 >= 0) beta = -beta;
      d = c0 - beta;
      tau = (beta - c0) / beta;
    }
    for (int l = threadIdx.x; l < nl; l += blockDim.x) {
      const int r = rank + l * C;
      vl[l] = r > i ? (tau == 0.0 ? 0.0 : T[l * ld + i] / d) : (r == i ? 1.0 : 0.0);
    }
    __syncthreads();
    // partial w_j = sum over own rows r >= i of v_r T[r, j], trailing columns j > i
    for (int j = i + 1 + threadIdx.x; j < p; j += blockDim.x) {
      double w = 0.0;
      for (int l = 0; l < nl; ++l) w += vl[l] * T[l * ld + j];
      dpart[j] = w;
    }
    cl.sync();
    for (int j = i + 1 + threadIdx.x; j < p; j += blockDim.x) {
      double w = 0.0;
      for (int c = 0; c < C; ++c) w += cl.map_shared_rank(dpart, c)[j];
      const double tw = tau * w;
      if (tau != 0.0)
        for (int l = 0; l < nl; ++l) T[l * ld + j] -= tw * vl[l];
    }
    for (int l = threadIdx.x; l < nl; l += blockDim.x) {
      const int r = rank + l * C;
      if (r > i) T[l * ld + i] = vl[l];
      else if (r == i) T[l * ld + i] = beta;
    }
    if (rank == 0 && threadIdx.x == 0) taul[i] = tau;
    __syncthreads();
  }
  for (Index idx = threadIdx.x; idx < Index(nl) * p; idx += blockDim.x) {
    const int l = int(idx / p), i = int(idx % p);
    Tt[(rank + l * C) + Index(i) * R] = T[l * ld + i];
  }
  if (rank == 0 && threadIdx.x == 0) J.qinfo[8] = 1.0;
  cl.sync();  // no CTA leaves while another may still read its partials
}

/// The two Q applications that end svd_qrcp_body, A = Q1 [As_k; 0] and B = Q_l [Bs_k; 0]
/// (R x k each, Q1 and Q_l products of p reflectors), spread over many CTAs: output columns
/// are independent, so every warp owns one column in registers (lane = rows lane + 32 q)
/// and runs the p reflectors (last to first) with one warp reduction each, no block
/// barriers. grid = (column groups of 8, {A, B}, jobs).
template <int NQ>
__global__ void __launch_bounds__(256) k_qrcp_apply_batch(const SvdJob* __restrict__ jobs) {
  const SvdJob& J = jobs[blockIdx.z];
  if (!J.ainfo) return;
  const int p = int(J.ainfo[0]), kk = int(J.ainfo[1]);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int j = int(blockIdx.x) * 8 + warp;
  if (j >= kk) return;
  const int R = J.R;
  const Index RR = Index(R) * R;
  double* Tt = J.ws;
  double* tau1 = Tt + RR + R;
  double* taul = tau1 + R;
  const double* As = taul + R + RR;
  const double* Bs = As + RR;
  const bool second = blockIdx.y == 1;
  const double* V = second ? Tt : J.S;  // reflectors below the diagonal, ld R
  const double* tau = second ? taul : tau1;
  const double* W = second ? Bs : As;   // p x p, ld p
  double* out = second ? J.B : J.A;
  double c[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const int i = lane + 32 * q;
    c[q] = (i < p) ? W[i + Index(j) * p] : 0.0;
  }
  for (int k = p - 1; k >= 0; --k) {
    const double t = tau[k];
    if (t == 0.0) continue;
    const double* v = V + Index(k) * R;
    double vr[NQ];
    double w = 0.0;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int i = lane + 32 * q;
      vr[q] = (i > k && i < R) ? v[i] : (i == k ? 1.0 : 0.0);
      w += vr[q] * c[q];
    }
    w = warp_sum(w) * t;
#pragma unroll
    for (int q = 0; q < NQ; ++q) c[q] -= w * vr[q];
  }
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const int i = lane + 32 * q;
    if (i < R) out[i + Index(j) * R] = c[q];
  }
}

/// Small-R (R <= kQrcpThreshold) batch: one cta_svd per CTA, work arrays in shared memory.
constexpr int kSvdSmallThreads = 512;
__global__ void __launch_bounds__(kSvdSmallThreads) k_svd_small_batch(const SvdJob* __restrict__ jobs) {
  extern __shared__ double smem[];
  const SvdJob& J = jobs[blockIdx.x];
  // lane-per-pair rounds in one warp up to Rp = 24, warp-per-pair rounds above
  cta_svd(J.Rx, J.R, J.Ry, J.R, J.R, J.eps, smem, J.A, J.B, J.sigma, J.info, 0.0, 24, nullptr,
          J.hidden_rel ? 4.0 * (*J.hidden_rel) : -1.0);
}

// Gather both sides of a lazy TT into column-major panels (one thread per element).
__global__ void k_gather(const TermDesc* __restrict__ terms, int nterms, const MapDesc* __restrict__ maps, Index m,
                         Index n, Index r, double* __restrict__ X, double* __restrict__ Yt) {
  const Index tx = m * r, total = tx + n * r;
  for (Index idx = Index(blockIdx.x) * blockDim.x + threadIdx.x; idx < total; idx += Index(gridDim.x) * blockDim.x) {
    if (idx < tx) {
      const Index i = idx % m, c = idx / m;
      X[idx] = expr_value(terms, nterms, maps, 0, i, c);
    } else {
      const Index k = idx - tx, j = k % n, c = k / n;
      Yt[k] = expr_value(terms, nterms, maps, 1, j, c);
    }
  }
}

inline int grid_for(Index total, int threads = kThreads) {
  Index b = (total + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > 148 * 16) b = 148 * 16;
  return int(b);
}

template <class K>
void set_smem(K kernel, size_t bytes) {
  allow_dynamic_smem(reinterpret_cast<const void*>(kernel), bytes);
}

}  // namespace

void launch_band_map(Context* ctx, const double* in, Index ld_in, double* out, Index ld_out, Index r,
                     const BandMap& m) {
  const Index total = m.n_out * r;
  if (total == 0) return;
  k_band_map<<<grid_for(total), kThreads, 0, ctx->stream>>>(in, ld_in, out, ld_out, r, m);
  ctx->launches++;
  TTSW_CUDA(cudaGetLastError());
}

void launch_gather(Context* ctx, const TermDesc* terms, int nterms, const MapDesc* maps, Index m, Index n, Index r,
                   double* X, double* Yt) {
  const Index total = (m + n) * r;
  if (total == 0) return;
  k_gather<<<grid_for(total), kThreads, 0, ctx->stream>>>(terms, nterms, maps, m, n, r, X, Yt);
  ctx->launches++;
  TTSW_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------------------------------
// Small-rank fused rounding, v2: grid-wide gather into L2 scratch, then one CTA per
// rounding split into two 512-thread groups (X panel / Y panel, named barriers 1 and 2)
// doing a row-parallel Householder QR (each thread owns rows; the column dots are
// multi-value group reductions), a CTA-wide Jacobi SVD, and a row-parallel Q
// application with the output rows held in registers.

// Batched gather of every job's lazy input into its scratch panels.
__global__ void k_gather_jobs(const RoundJob* __restrict__ jobs, const MapDesc* __restrict__ maps, int nmaps) {
  // term and map descriptors are staged in shared memory (the recursive evaluator
  // re-reads them for every tap)
  extern __shared__ double gsm[];
  const RoundJob J = jobs[blockIdx.y];
  TermDesc* st = reinterpret_cast<TermDesc*>(gsm);
  MapDesc* sm = reinterpret_cast<MapDesc*>(st + J.nterms);
  {
    const int* src = reinterpret_cast<const int*>(J.terms);
    int* dst = reinterpret_cast<int*>(st);
    for (int i = threadIdx.x; i < int(J.nterms * sizeof(TermDesc) / sizeof(int)); i += blockDim.x) dst[i] = src[i];
    src = reinterpret_cast<const int*>(maps);
    dst = reinterpret_cast<int*>(sm);
    for (int i = threadIdx.x; i < int(nmaps * sizeof(MapDesc) / sizeof(int)); i += blockDim.x) dst[i] = src[i];
  }
  __syncthreads();
  const Index tx = J.m * J.R, total = tx + J.n * J.R;
  for (Index idx = Index(blockIdx.x) * blockDim.x + threadIdx.x; idx < total; idx += Index(gridDim.x) * blockDim.x) {
    if (idx < tx)
      const_cast<double*>(J.Xs)[idx] = expr_value(st, J.nterms, sm, 0, idx % J.m, idx / J.m);
    else {
      const Index k = idx - tx;
      const_cast<double*>(J.Ys)[k] = expr_value(st, J.nterms, sm, 1, k % J.n, k / J.n);
    }
  }
}

// Column-organised batched gather: CTA (x, job) evaluates whole columns of the job's X
// panel (x < R) and Yt panel (R <= x < 2R), so the owning term, the Hadamard factor
// columns (a, b) and the source pointers are resolved once per column instead of per
// element (no 64-bit division, no per-element term search); rows are coalesced. Terms
// with map chains use the same evaluator as k_gather_jobs (identical arithmetic).
__global__ void __launch_bounds__(256, 4) k_gather_cols(const RoundJob* __restrict__ jobs,
                                                     const MapDesc* __restrict__ maps, int nmaps) {
  extern __shared__ double gsm[];
  const RoundJob J = jobs[blockIdx.y];
  TermDesc* st = reinterpret_cast<TermDesc*>(gsm);
  MapDesc* sm = reinterpret_cast<MapDesc*>(st + J.nterms);
  {
    const int* src = reinterpret_cast<const int*>(J.terms);
    int* dst = reinterpret_cast<int*>(st);
    for (int i = threadIdx.x; i < int(J.nterms * sizeof(TermDesc) / sizeof(int)); i += blockDim.x) dst[i] = src[i];
    src = reinterpret_cast<const int*>(maps);
    dst = reinterpret_cast<int*>(sm);
    for (int i = threadIdx.x; i < int(nmaps * sizeof(MapDesc) / sizeof(int)); i += blockDim.x) dst[i] = src[i];
  }
  __syncthreads();
  const int R = J.R;
  for (int col = blockIdx.x; col < 2 * R; col += gridDim.x) {
    const int side = col >= R ? 1 : 0;
    const int c = col - side * R;
    const Index rows = side ? J.n : J.m;
    double* out = const_cast<double*>(side ? J.Ys : J.Xs) + Index(c) * rows;
    // small launches split every column over gridDim.z row slices (rows [rb, re))
    const Index rb = rows * blockIdx.z / gridDim.z, re = rows * (blockIdx.z + 1) / gridDim.z;
    const TermDesc& t = st[find_term(st, J.nterms, c)];
    const SideExpr& e = side == 0 ? t.x : t.y;
    const int cc = c - int(t.col0);
    if (e.nops == 0 && t.kind != TERM_CONST) {
      const double* p1;
      const double* p2 = nullptr;
      if (t.kind == TERM_HADAMARD) {
        const int a = cc / t.r2, b = cc % t.r2;
        p1 = e.base + Index(a) * e.ld;
        p2 = side == 0 ? t.x2 + Index(b) * t.ldx2 : t.y2 + Index(b) * t.ldy2;
      } else {
        p1 = e.base + Index(cc) * e.ld;
      }
      if (p2) {
        // four independent rows per thread in flight (the column is a pure HBM stream)
        Index r = rb + threadIdx.x;
        const Index st = blockDim.x;
        for (; r + 3 * st < re; r += 4 * st) {
          const double a0 = p1[r], a1 = p1[r + st], a2 = p1[r + 2 * st], a3 = p1[r + 3 * st];
          const double b0 = p2[r], b1 = p2[r + st], b2 = p2[r + 2 * st], b3 = p2[r + 3 * st];
          out[r] = b0 * a0;  // y.cx(i,b) * x.cx(i,a)
          out[r + st] = b1 * a1;
          out[r + 2 * st] = b2 * a2;
          out[r + 3 * st] = b3 * a3;
        }
        for (; r < re; r += st) out[r] = p2[r] * p1[r];
      } else {
        for (Index r = rb + threadIdx.x; r < re; r += blockDim.x) out[r] = p1[r];
      }
    } else {
      bool only_scale = true;
      for (int k = 0; k < e.nops; ++k) only_scale = only_scale && e.ops[k].kind == 0;
      if (only_scale) {
        // scalings only (the sums of the LLF flux and the RK stages): the base value times the
        // factors in op order, exactly eval_side's arithmetic without its recursion
        const double* p1 = nullptr;
        const double* p2 = nullptr;
        if (t.kind == TERM_HADAMARD) {
          const int a = cc / t.r2, b = cc % t.r2;
          p1 = e.base + Index(a) * e.ld;
          p2 = side == 0 ? t.x2 + Index(b) * t.ldx2 : t.y2 + Index(b) * t.ldy2;
        } else if (t.kind == TERM_PLAIN) {
          p1 = e.base + Index(cc) * e.ld;
        }
        const double cv = side == 0 ? t.cx : t.cy;
        const int nops = e.nops;
        for (Index r = rb + threadIdx.x; r < re; r += blockDim.x) {
          double v = p1 ? (p2 ? p2[r] * p1[r] : p1[r]) : cv;
          for (int k = 0; k < nops; ++k) v = v * e.ops[k].scale;
          out[r] = v;
        }
      } else {
        for (Index r = rb + threadIdx.x; r < re; r += blockDim.x) out[r] = eval_side(t, side, sm, e.nops, r, cc);
      }
    }
  }
}

constexpr int kGroup = 512;
constexpr int kGroupWarps = kGroup / 32;

__device__ __forceinline__ void group_sync(int id) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(kGroup) : "memory");
}

/// Row-parallel Householder QR of a (nr x R, ld lda; shared memory) by one 512-thread
/// group; thread gt owns rows gt + r*512. Same reflector convention as cta_householder_qr.
/// sh: 16 + 16*RMAX + RMAX doubles of group scratch.
template <int RMAX, int ROWS>
__device__ void group_qr_rows(double* a, Index lda, Index nr, int R, double* tau, double* sh, int bar, int gt) {
  const int lane = gt & 31, w = gt >> 5;
  double* redT = sh;                        // 16
  double* redP = sh + kGroupWarps;          // 16 x RMAX
  double* wsh = redP + kGroupWarps * RMAX;  // RMAX
  const int q = int(nr < R ? nr : R);
  for (int k = 0; k < q; ++k) {
    double xi[ROWS];
    double part = 0;
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {
      const Index i = gt + Index(r) * kGroup;
      xi[r] = (i > k && i < nr) ? a[i + Index(k) * lda] : 0.0;
      part += xi[r] * xi[r];
    }
    part = warp_sum(part);
    if (lane == 0) redT[w] = part;
    group_sync(bar);
    double tail2 = 0;
#pragma unroll
    for (int ww = 0; ww < kGroupWarps; ++ww) tail2 += redT[ww];
    const double c0 = a[k + Index(k) * lda];
    double t, beta, d;
    if (tail2 <= DBL_MIN) {
      t = 0.0;
      beta = c0;
      d = 1.0;
    } else {
      beta = sqrt(c0 * c0 + tail2);
      if (c0 >= 0) beta = -beta;
      d = c0 - beta;
      t = (beta - c0) / beta;
    }
    double v[ROWS];
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {
      const Index i = gt + Index(r) * kGroup;
      v[r] = 0.0;
      if (i > k && i < nr) {
        v[r] = (t == 0.0) ? 0.0 : xi[r] / d;
        a[i + Index(k) * lda] = v[r];
      }
    }
    for (int j = k + 1; j < R; ++j) {
      double pj = 0.0;
#pragma unroll
      for (int r = 0; r < ROWS; ++r) {
        const Index i = gt + Index(r) * kGroup;
        if (i > k && i < nr) pj += v[r] * a[i + Index(j) * lda];
      }
      pj = warp_sum(pj);
      if (lane == 0) redP[w * RMAX + j] = pj;
    }
    group_sync(bar);
    if (gt < R && gt > k && t != 0.0) {
      double s = 0;
#pragma unroll
      for (int ww = 0; ww < kGroupWarps; ++ww) s += redP[ww * RMAX + gt];
      const double wj = (a[k + Index(gt) * lda] + s) * t;
      wsh[gt] = wj;
      a[k + Index(gt) * lda] -= wj;
    }
    if (gt == 0) {
      tau[k] = t;
      a[k + Index(k) * lda] = beta;
    }
    group_sync(bar);
    if (t != 0.0) {
#pragma unroll
      for (int r = 0; r < ROWS; ++r) {
        const Index i = gt + Index(r) * kGroup;
        if (i > k && i < nr) {
#pragma unroll
          for (int j = 0; j < RMAX; ++j)
            if (j > k && j < R) a[i + Index(j) * lda] -= wsh[j] * v[r];
        }
      }
    }
  }
  for (int k = q + gt; k < R; k += kGroup) tau[k] = 0.0;
  group_sync(bar);
}

/// out (nr x kc, ld ldo; global) = Q [C; 0] by one group, output rows in registers.
/// sh: 2 x (16*KMAX + 2*KMAX) doubles (double-buffered by reflector parity).
template <int KMAX, int ROWS>
__device__ void group_apply_rows(const double* a, Index lda, const double* tau, Index nr, int R, const double* C,
                                 Index ldc, int kc, double* out, Index ldo, double* sh, int bar, int gt) {
  const int lane = gt & 31, w = gt >> 5;
  const Index top = nr < R ? nr : R;
  double o[ROWS][KMAX];
#pragma unroll
  for (int r = 0; r < ROWS; ++r) {
    const Index i = gt + Index(r) * kGroup;
#pragma unroll
    for (int c = 0; c < KMAX; ++c) o[r][c] = (c < kc && i < top) ? C[i + Index(c) * ldc] : 0.0;
  }
  for (int j = int(top) - 1; j >= 0; --j) {
    const double t = tau[j];
    if (t == 0.0) continue;
    double* buf = sh + (j & 1) * (kGroupWarps * KMAX + 2 * KMAX);
    double* redP = buf;
    double* bc = buf + kGroupWarps * KMAX;
    double* wsh = bc + KMAX;
    double v[ROWS];
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {
      const Index i = gt + Index(r) * kGroup;
      v[r] = (i > j && i < nr) ? a[i + Index(j) * lda] : 0.0;
      if (i == j)
#pragma unroll
        for (int c = 0; c < KMAX; ++c) bc[c] = o[r][c];
    }
#pragma unroll
    for (int c = 0; c < KMAX; ++c)
      if (c < kc) {
        double pc = 0.0;
#pragma unroll
        for (int r = 0; r < ROWS; ++r) pc += v[r] * o[r][c];
        pc = warp_sum(pc);
        if (lane == 0) redP[w * KMAX + c] = pc;
      }
    group_sync(bar);
    if (gt < kc) {
      double s = 0;
#pragma unroll
      for (int ww = 0; ww < kGroupWarps; ++ww) s += redP[ww * KMAX + gt];
      wsh[gt] = (bc[gt] + s) * t;
    }
    group_sync(bar);
#pragma unroll
    for (int r = 0; r < ROWS; ++r) {
      const Index i = gt + Index(r) * kGroup;
      if (i > j && i < nr) {
#pragma unroll
        for (int c = 0; c < KMAX; ++c)
          if (c < kc) o[r][c] -= wsh[c] * v[r];
      } else if (i == j) {
#pragma unroll
        for (int c = 0; c < KMAX; ++c)
          if (c < kc) o[r][c] -= wsh[c];
      }
    }
  }
#pragma unroll
  for (int r = 0; r < ROWS; ++r) {
    const Index i = gt + Index(r) * kGroup;
    if (i < nr)
#pragma unroll
      for (int c = 0; c < KMAX; ++c)
        if (c < kc) out[i + Index(c) * ldo] = o[r][c];
  }
}

template <int RMAX, int ROWS>
__global__ void __launch_bounds__(1024) k_round_small(const RoundJob* __restrict__ jobs) {
  extern __shared__ double smem[];
  const RoundJob J = jobs[blockIdx.x];
  const Index m = J.m, n = J.n;
  const int R = J.R;
  const int gid = threadIdx.x / kGroup, gt = threadIdx.x % kGroup;
  double* ax = smem;
  double* ay = ax + m * R;
  double* tx = ay + n * R;
  double* ty = tx + RMAX;
  double* gsh = ty + RMAX;  // 2 groups x (2 * (16*RMAX + 2*RMAX)) doubles
  const int gsz = 2 * (kGroupWarps * RMAX + 2 * RMAX);
  double* work = gsh + 2 * gsz;  // svd: 2 Rp^2 + 2 Rp
  if (J.prof && threadIdx.x == 0) J.prof[0] = clock64();
  for (Index idx = threadIdx.x; idx < m * R; idx += blockDim.x) ax[idx] = J.Xs[idx];
  for (Index idx = threadIdx.x; idx < n * R; idx += blockDim.x) ay[idx] = J.Ys[idx];
  __syncthreads();
  if (J.prof && threadIdx.x == 0) J.prof[1] = clock64();
  if (gid == 0)
    group_qr_rows<RMAX, ROWS>(ax, m, m, R, tx, gsh, 1, gt);
  else
    group_qr_rows<RMAX, ROWS>(ay, n, n, R, ty, gsh + gsz, 2, gt);
  __syncthreads();
  if (J.prof && threadIdx.x == 0) J.prof[2] = clock64();
  cta_svd(ax, m, ay, n, R, J.eps, work, J.A, J.B, J.sigma, J.info);
  __syncthreads();
  if (J.prof && threadIdx.x == 0) J.prof[3] = clock64();
  const int k = int(J.info[0]);
  if (k == 0) {
    for (Index i = threadIdx.x; i < m; i += blockDim.x) J.Xout[i] = 0.0;
    for (Index i = threadIdx.x; i < n; i += blockDim.x) J.Ytout[i] = 0.0;
    return;
  }
  // output columns in chunks of 8 (register-resident rows, no spills for any R <= 16)
  for (int c0 = 0; c0 < k; c0 += 8) {
    if (J.prof && threadIdx.x == 0) J.prof[5] = k;
    const int kc = k - c0 < 8 ? k - c0 : 8;
    if (gid == 0)
      group_apply_rows<8, ROWS>(ax, m, tx, m, R, J.A + Index(c0) * R, R, kc, J.Xout + Index(c0) * m, m, gsh, 1, gt);
    else
      group_apply_rows<8, ROWS>(ay, n, ty, n, R, J.B + Index(c0) * R, R, kc, J.Ytout + Index(c0) * n, n, gsh + gsz,
                                2, gt);
  }
  __syncthreads();
  if (J.prof && threadIdx.x == 0) {
    J.prof[4] = clock64();
    J.prof[6] = R;
    J.prof[7] = (long long)J.info[2];  // Jacobi sweeps
  }
}

size_t fused_round_smem(Index m, Index n, Index R) {
  const Index Rp = R + (R & 1);
  return size_t((m + n) * R + 2 * R + 2 * Rp * Rp + 2 * Rp) * sizeof(double);
}

size_t small_round_smem(Index m, Index n, Index R, int rmax) {
  const Index Rp = R + (R & 1);
  const Index gsz = 2 * (kGroupWarps * rmax + 2 * rmax);
  return size_t((m + n) * R + 2 * rmax + 2 * gsz + 2 * Rp * Rp + 2 * Rp) * sizeof(double);
}

bool small_round_fits(const Context* ctx, Index m, Index n, Index R) {
  if (R > 16 || m > 2 * kGroup || n > 2 * kGroup || m < R || n < R) return false;
  return small_round_smem(m, n, R, R <= 8 ? 8 : 16) + 4096 <= ctx->smem_optin;
}

void launch_gather_jobs(Context* ctx, const RoundJob* jobs, int njobs, Index max_cols, const MapDesc* maps,
                        int nmaps, int max_terms) {
  // one CTA per (panel column, job): max_cols = 2 max R
  dim3 g(unsigned(std::max<Index>(1, max_cols)), unsigned(njobs));
  // a launch too small to fill the device (the single lazy operands of the crosses) splits
  // its columns into row slices: the per-thread chain of dependent loads gets shorter
  const long ctas = long(g.x) * long(g.y);
  if (ctas < 2L * ctx->num_sms) g.z = unsigned(std::min<long>(8, (2L * ctx->num_sms + ctas - 1) / ctas));
  const size_t gs = sizeof(TermDesc) * size_t(max_terms) + sizeof(MapDesc) * size_t(nmaps);
  set_smem(k_gather_cols, gs);
  k_gather_cols<<<g, 256, gs, ctx->stream>>>(jobs, maps, nmaps);
  ctx->launches++;
  TTSW_CUDA(cudaGetLastError());
}

void launch_round_small(Context* ctx, const RoundJob* jobs, int njobs, Index max_elems, const MapDesc* maps,
                        int nmaps, int max_terms, int rmax, int rows, size_t smem) {
  dim3 g(unsigned(std::min<Index>((max_elems + 255) / 256, 148 * 4)), unsigned(njobs));
  const size_t gs = sizeof(TermDesc) * size_t(max_terms) + sizeof(MapDesc) * size_t(nmaps);
  set_smem(k_gather_jobs, gs);
  k_gather_jobs<<<g, 256, gs, ctx->stream>>>(jobs, maps, nmaps);
  ctx->launches++;
  TTSW_CUDA(cudaGetLastError());
#define TTSW_SMALL(RM, RW)                                            \
  if (rmax == RM && rows == RW) {                                     \
    set_smem(k_round_small<RM, RW>, smem);                            \
    k_round_small<RM, RW><<<njobs, 1024, smem, ctx->stream>>>(jobs);  \
  }
  TTSW_SMALL(8, 1) TTSW_SMALL(8, 2) TTSW_SMALL(16, 1) TTSW_SMALL(16, 2)
#undef TTSW_SMALL
  ctx->launches++;
  TTSW_CUDA(cudaGetLastError());
}

void launch_round_fused(Context* ctx, const RoundJob* jobs, int njobs, const MapDesc* maps, size_t smem) {
  set_smem(k_round_fused, smem);
  k_round_fused<<<njobs, 1024, smem, ctx->stream>>>(jobs, maps);
  ctx->launches++;
  TTSW_CUDA(cudaGetLastError());
}

void launch_csr_map(Context* ctx, const double* in, Index ld_in, double* out, Index rows, Index r, const long* rowptr,
                    const long* colidx, const double* vals) {
  if (rows * r == 0) return;
  k_csr_map<<<grid_for(rows * r), kThreads, 0, ctx->stream>>>(in, ld_in, out, rows, r, rowptr, colidx, vals);
  ctx->launches++;
  TTSW_CUDA(cudaGetLastError());
}

void launch_scale_copy(Context* ctx, double* dst, const double* src, Index count, double a) {
  if (count == 0) return;
  k_scale_copy<<<grid_for(count), kThreads, 0, ctx->stream>>>(dst, src, count, a);
  ctx->launches++;
  TTSW_CUDA(cudaGetLastError());
}

void launch_fill(Context* ctx, double* dst, Index count, double v) {
  if (count == 0) return;
  k_fill<<<grid_for(count), kThreads, 0, ctx->stream>>>(dst, count, v);
  ctx->launches++;
  TTSW_CUDA(cudaGetLastError());
}

void launch_hadamard(Context* ctx, const double* x, Index rx, const double* y, Index ry, Index rows, double* out) {
  const Index total = rows * rx * ry;
  if (total == 0) return;
  k_hadamard<<<grid_for(total), kThreads, 0, ctx->stream>>>(x, rx, y, ry, rows, out);
  ctx->launches++;
  TTSW_CUDA(cudaGetLastError());
}

void launch_transpose(Context* ctx, const double* in, Index rows, Index cols, double* out) {
  dim3 grid(unsigned((rows + 31) / 32), unsigned((cols + 31) / 32));
  k_transpose<<<grid, dim3(32, 8), 0, ctx->stream>>>(in, rows, cols, out);
  ctx->launches++;
  TTSW_CUDA(cudaGetLastError());
}

void launch_norm2(Context* ctx, const double* X, Index m, const double* Yt, Index n, Index r, double* work,
                  double* out) {
  k_gram_prod<<<dim3(unsigned(r), unsigned(r)), kThreads, 0, ctx->stream>>>(X, m, Yt, n, r, work);
  k_reduce_final<<<1, 1024, 0, ctx->stream>>>(work, r * r, 0, r, out);
  ctx->launches += 2;
  TTSW_CUDA(cudaGetLastError());
}

void launch_sum_entries(Context* ctx, const double* X, Index m, const double* Yt, Index n, Index r, double* work,
                        double* out) {
  k_colsums<<<unsigned(r), kThreads, 0, ctx->stream>>>(X, m, Yt, n, work, r);
  k_reduce_final<<<1, 1024, 0, ctx->stream>>>(work, 0, 1, r, out);
  ctx->launches += 2;
  TTSW_CUDA(cudaGetLastError());
}

QRPlan plan_tsqr(Context* ctx, Index rows, Index R) {
  QRPlan p;
  p.R = R;
  Index cur = rows;
  // leaves must have >= R rows; small R: 256-row leaves in shared memory; large R:
  // square R-row leaves (more CTAs in flight) processed from L2 by 1024 threads
  const Index leaf = 2 * R * R * 8 + 4096 <= Index(ctx->smem_optin) ? std::max<Index>(2 * R, 256) : R;
  for (int guard = 0; guard < 64; ++guard) {
    QRLevel lv;
    lv.rows = cur;
    // tree levels merge at least two stacked R factors per block so the tree shrinks
    const Index target = p.levels.empty() ? leaf : std::max<Index>(2 * R, leaf);
    lv.L = int(std::max<Index>(1, cur / target));
    lv.V = ctx->alloc(size_t(cur * R));
    lv.tau = ctx->alloc(size_t(lv.L * R));
    lv.Rst = ctx->alloc(size_t(Index(lv.L) * R * R));
    p.levels.push_back(lv);
    if (lv.L == 1) break;
    cur = Index(lv.L) * R;
  }
  if (p.levels.back().L != 1) throw CudaError("plan_tsqr: tree did not reduce");
  return p;
}

void free_tsqr(Context* ctx, QRPlan& p) {
  for (auto& lv : p.levels) {
    ctx->free(lv.V);
    ctx->free(lv.tau);
    ctx->free(lv.Rst);
  }
  p.levels.clear();
}

void tsqr_factor(Context* ctx, QRPlan& p, const double* A, Index lda) {
  const int R = int(p.R);
  const double* in = A;
  Index ldin = lda;
  for (auto& lv : p.levels) {
    const Index maxrows = (lv.rows + lv.L - 1) / lv.L;
    const size_t bytes = size_t(maxrows) * R * sizeof(double);
    if (bytes <= ctx->smem_optin - 1024) {
      set_smem(k_qr_blocks<true>, bytes);
      k_qr_blocks<true><<<lv.L, kThreads, bytes, ctx->stream>>>(in, ldin, lv.rows, R, lv.L, lv.V, lv.tau, lv.Rst);
    } else {
      k_qr_blocks<false><<<lv.L, 1024, 0, ctx->stream>>>(in, ldin, lv.rows, R, lv.L, lv.V, lv.tau, lv.Rst);
    }
    ctx->launches++;
    TTSW_CUDA(cudaGetLastError());
    in = lv.Rst;
    ldin = Index(lv.L) * R;
  }
}

void tsqr_apply(Context* ctx, const QRPlan& p, const double* C, Index ld_c, int kc, double* out, Index ld_out) {
  const int R = int(p.R);
  const double* cin = C;
  Index ldcin = ld_c;
  std::vector<double*> temps;
  for (int li = int(p.levels.size()) - 1; li >= 0; --li) {
    const auto& lv = p.levels[size_t(li)];
    double* cout;
    Index ldcout;
    if (li == 0) {
      cout = out;
      ldcout = ld_out;
    } else {
      cout = ctx->alloc(size_t(lv.rows * kc));
      temps.push_back(cout);
      ldcout = lv.rows;
    }
    const Index maxrows = (lv.rows + lv.L - 1) / lv.L;
    const size_t bytes = size_t(maxrows) * kc * sizeof(double);
    if (bytes <= ctx->smem_optin - 1024) {
      set_smem(k_apply_blocks<true>, bytes);
      k_apply_blocks<true><<<lv.L, kThreads, bytes, ctx->stream>>>(lv.V, lv.tau, lv.rows, R, lv.L, cin, ldcin, kc,
                                                                   cout, ldcout);
    } else {
      k_apply_blocks<false><<<lv.L, 1024, 0, ctx->stream>>>(lv.V, lv.tau, lv.rows, R, lv.L, cin, ldcin, kc, cout,
                                                           ldcout);
    }
    ctx->launches++;
    TTSW_CUDA(cudaGetLastError());
    cin = cout;
    ldcin = ldcout;
  }
  for (double* t : temps) ctx->free(t);
}

/// Cluster size for the pivoted QR of the large-R SVDs (0: the single-CTA path). 8 CTAs
/// (portable) when S fits their shared memory, else 16 (non-portable) when it fits those.
int qrcp_cluster_size(Context* ctx, int R) {
  const size_t cap = size_t(ctx->smem_optin) - 1024;
  // clusters of 16 are non-portable
  allow_nonportable_cluster(reinterpret_cast<const void*>(k_qrcp_cluster));
  allow_nonportable_cluster(reinterpret_cast<const void*>(k_lq_cluster));
  if (qrcp_cluster_smem(R, 8) <= cap) return 8;
  if (qrcp_cluster_smem(R, 16) <= cap) return 16;
  return 0;
}

void launch_svd_batch(Context* ctx, const std::vector<SvdRequest>& reqs) {
  HostRegion hr_(ctx, "launch_svd_batch");
  if (reqs.empty()) return;
  static const bool prof_on = std::getenv("TTSW_PROFILE_TSQR") != nullptr;
  std::vector<SvdJob> big, small;
  std::vector<double*> allocs;
  int maxtiles = 0;
  Index maxR = 0, maxRs = 0;
  for (const auto& q : reqs) maxR = std::max(maxR, q.R);
  const int qc = qrcp_cluster_size(ctx, int(maxR));
  constexpr Index qrcp_min = kQrcpThreshold + 1;
  for (const auto& q : reqs) {
    const Index R = q.R;
    SvdJob J{};
    J.Rx = q.Rx;
    J.Ry = q.Ry;
    J.R = int(R);
    J.eps = q.eps;
    J.A = q.A;
    J.B = q.B;
    J.sigma = q.sigma;
    J.info = q.info;
    J.hidden_rel = q.hidden_rel;
    if (R >= qrcp_min) {
      const Index RR = R * R;
      const Index used = 5 * RR + 3 * R + 2 * (R + 1) * (R + 1) + 2 * (R + 1) + 8 + 8;
      const int tiles = int((R + 31) / 32);
      double* ws = ctx->alloc(size_t(used + R + RR + 3 * tiles * tiles + 16 + 16 + 8));
      allocs.push_back(ws);
      J.ws = ws;
      J.perm = reinterpret_cast<int*>(ws + used);
      J.S = ws + used + R;
      J.part = J.S + RR;
      J.tiles = tiles;
      J.prof = prof_on ? reinterpret_cast<long long*>(J.part + 3 * tiles * tiles) : nullptr;
      if (J.prof) TTSW_CUDA(cudaMemsetAsync(J.prof, 0, 16 * sizeof(long long), ctx->stream));
      J.qinfo = qc ? J.part + 3 * tiles * tiles + 16 : nullptr;
      J.ainfo = (R <= 24 * 32) ? J.part + 3 * tiles * tiles + 20 : nullptr;
      J.cinfo = (qc && J.ainfo) ? J.part + 3 * tiles * tiles + 32 : nullptr;
      maxtiles = std::max(maxtiles, tiles);
      maxR = std::max(maxR, R);
      big.push_back(J);
    } else {
      maxRs = std::max(maxRs, R);
      small.push_back(J);
    }
  }
  // job descriptors: one pinned staging copy (the arena is free between round_batch calls)
  const size_t bytes = sizeof(SvdJob) * (big.size() + small.size());
  ctx->ensure_stage(bytes);
  std::memcpy(ctx->stage_host, big.data(), sizeof(SvdJob) * big.size());
  std::memcpy(static_cast<char*>(ctx->stage_host) + sizeof(SvdJob) * big.size(), small.data(),
              sizeof(SvdJob) * small.size());
  TTSW_CUDA(cudaMemcpyAsync(ctx->stage_dev, ctx->stage_host, bytes, cudaMemcpyHostToDevice, ctx->stream));
  const SvdJob* dbig = static_cast<const SvdJob*>(ctx->stage_dev);
  const SvdJob* dsmall = dbig + big.size();
  // mixed batch: the small SVDs run on the side stream beside the QRCP batch
  const bool fork = !big.empty() && !small.empty();
  if (fork) {
    TTSW_CUDA(cudaEventRecord(ctx->fork_ev, ctx->stream));
    TTSW_CUDA(cudaStreamWaitEvent(ctx->side, ctx->fork_ev, 0));
  }
  if (!big.empty()) {
    k_form_s_batch<<<dim3(maxtiles, maxtiles, unsigned(big.size())), 256, 0, ctx->stream>>>(dbig);
    if (qc) {
      constexpr double first = 1e-3;  // first-pass stop (two-pass QRCP stop)
      const size_t qbytes = qrcp_cluster_smem(int(maxR), qc);
      set_smem(k_qrcp_cluster, qbytes);
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(unsigned(big.size()) * unsigned(qc));
      cfg.blockDim = dim3(kQcThreads);
      cfg.dynamicSmemBytes = qbytes;
      cfg.stream = ctx->stream;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = unsigned(qc);
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      TTSW_CUDA(cudaLaunchKernelEx(&cfg, k_qrcp_cluster, dbig, first, 1e-6));
      ctx->launches++;
      const size_t lbytes = lq_cluster_smem(int(maxR), qc);
      if (lbytes <= size_t(ctx->smem_optin) - 1024) {
        set_smem(k_lq_cluster, lbytes);
        cfg.dynamicSmemBytes = lbytes;
        TTSW_CUDA(cudaLaunchKernelEx(&cfg, k_lq_cluster, dbig));
        ctx->launches++;
      }
    }
    // shared memory: the step reflector (R) and, when they fit, the Jacobi work arrays
    const size_t smem = std::min<size_t>(size_t(ctx->smem_optin) - 2048,
                                         (2 * size_t(maxR + 2) * (maxR + 2) + 2 * size_t(maxR + 2) + size_t(maxR)) *
                                             sizeof(double));
    set_smem(k_svd_qrcp_batch, smem);
    {
      cudaLaunchConfig_t scfg{};
      scfg.gridDim = dim3(2 * unsigned(big.size()));
      scfg.blockDim = dim3(1024);
      scfg.dynamicSmemBytes = smem;
      scfg.stream = ctx->stream;
      cudaLaunchAttribute sat[1];
      sat[0].id = cudaLaunchAttributeClusterDimension;
      sat[0].val.clusterDim.x = 2;
      sat[0].val.clusterDim.y = 1;
      sat[0].val.clusterDim.z = 1;
      scfg.attrs = sat;
      scfg.numAttrs = 1;
      const size_t sb = smem - size_t(maxR) * sizeof(double);
      bool split = qc != 0 && maxR >= kJcMinP;
      for (const auto& J : big) split = split && J.cinfo;
      TTSW_CUDA(cudaLaunchKernelEx(&scfg, k_svd_qrcp_batch, dbig, sb, split ? 1 : 0));
      if (split) {
        const int rpm = int(std::min<Index>(kJcMaxRp, maxR + (maxR & 1)));
        const size_t jb = 2 * size_t((rpm + kJcC - 1) / kJcC) * size_t(rpm) * sizeof(double);
        set_smem(k_jacobi_cluster, jb);
        cudaLaunchConfig_t jcfg{};
        jcfg.gridDim = dim3(unsigned(kJcC) * unsigned(big.size()));
        jcfg.blockDim = dim3(kJcThreads);
        jcfg.dynamicSmemBytes = jb;
        jcfg.stream = ctx->stream;
        cudaLaunchAttribute jat[1];
        jat[0].id = cudaLaunchAttributeClusterDimension;
        jat[0].val.clusterDim.x = unsigned(kJcC);
        jat[0].val.clusterDim.y = 1;
        jat[0].val.clusterDim.z = 1;
        jcfg.attrs = jat;
        jcfg.numAttrs = 1;
        TTSW_CUDA(cudaLaunchKernelEx(&jcfg, k_jacobi_cluster, dbig));
        TTSW_CUDA(cudaLaunchKernelEx(&scfg, k_svd_qrcp_batch, dbig, sb, 2));
        ctx->launches += 2;
      }
    }
    ctx->launches += 2;
    TTSW_CUDA(cudaGetLastError());
    bool deferred = false;  // jobs without ainfo (R > 768) applied Q in their SVD CTA
    for (const auto& J : big) deferred = deferred || J.ainfo;
    if (deferred) {
      const dim3 g(unsigned((maxR + 7) / 8), 2, unsigned(big.size()));
      if (maxR <= 256)
        k_qrcp_apply_batch<8><<<g, 256, 0, ctx->stream>>>(dbig);
      else if (maxR <= 512)
        k_qrcp_apply_batch<16><<<g, 256, 0, ctx->stream>>>(dbig);
      else
        k_qrcp_apply_batch<24><<<g, 256, 0, ctx->stream>>>(dbig);
      ctx->launches++;
      TTSW_CUDA(cudaGetLastError());
    }
  }
  if (!small.empty()) {
    const Index Rp = maxRs + (maxRs & 1);
    const size_t sbytes = size_t(2 * Rp * Rp + 2 * Rp) * sizeof(double);
    set_smem(k_svd_small_batch, sbytes);
    k_svd_small_batch<<<unsigned(small.size()), kSvdSmallThreads, sbytes, fork ? ctx->side : ctx->stream>>>(dsmall);
    ctx->launches++;
    TTSW_CUDA(cudaGetLastError());
  }
  if (fork) {
    TTSW_CUDA(cudaEventRecord(ctx->join_ev, ctx->side));
    TTSW_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->join_ev, 0));
  }
  if (prof_on && !big.empty()) {
    TTSW_CUDA(cudaStreamSynchronize(ctx->stream));
    for (const auto& J : big) {
      long long h[16];
      TTSW_CUDA(cudaMemcpy(h, J.prof, sizeof(h), cudaMemcpyDeviceToHost));
      std::fprintf(stderr,
                   "svd_qrcp R=%d p=%lld sweeps=%lld kcycles: qrcp %lld lq %lld jacobi %lld apply %lld p2=%lld p4=%lld\n",
                   J.R, h[6], h[7], (h[1] - h[0]) / 1000, (h[2] - h[1]) / 1000, (h[3] - h[2]) / 1000,
                   (h[4] - h[3]) / 1000, h[8], h[9]);
    }
  }
  for (double* a : allocs) ctx->free(a);  // stream-ordered: safe after the launches
}

void launch_svd_small(Context* ctx, const double* Rx, const double* Ry, Index R, double eps, double* A, double* B,
                      double* sigma, double* info) {
  launch_svd_batch(ctx, {SvdRequest{Rx, Ry, R, eps, A, B, sigma, info}});
}

}  // namespace ttsw
