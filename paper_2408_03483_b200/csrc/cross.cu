// TT-cross (2-D skeleton / CUR) and maxvol on device: restates
// /root/reference/proj/include/ttsw/cross.hpp:31-254 with
//  * fiber evaluation (CrossSampler, cross.hpp:77-146) as kernels that contract the
//    operand cores and apply a fixed device functor (the host std::function EntryFn of
//    cross.hpp:64-65 becomes an enum; WENO5 / LLF functors of reconstruction.hpp:174-247
//    and swe.hpp:342-347);
//  * FullPivLU row order (cross.hpp:37-45) and the partial-pivot re-solve of every
//    maxvol swap (cross.hpp:48-59) as kernels, argmax ties broken column-major first
//    like Eigen's maxCoeff;
//  * the validation sampler kept bit-compatible on the host: std::mt19937_64 seeded
//    per call + std::uniform_int_distribution (cross.hpp:179-180, :216-217), the
//    non-stable std::sort of residuals (cross.hpp:237-238).
#include <algorithm>
#include <mutex>
#include <cfloat>
#include <cmath>
#include <random>
#include <sstream>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cooperative_groups.h>

#include "kernels.cuh"

namespace ttsw {

namespace cg = cooperative_groups;
constexpr int kMaxvolRank = 128;  // largest maxvol rank swapped on the device in one launch

namespace {

constexpr int kMaxOps = 8;

struct OpSet {
  const double* X[kMaxOps];
  const double* Yt[kMaxOps];
  int r[kMaxOps];
  int nops;
  Index m, n;
};

struct FnParams {
  int fn;
  double a;  // eps_weno or g
  double step1_c[3][3];
  double c[3][3][3];
  double gamma[3][3];
  double gamma_plus[3], gamma_minus[3], weno_d[3];
  double sigma_plus, sigma_minus;
};

FnParams make_fn(int fn, double param) {
  FnParams p{};
  p.fn = fn;
  p.a = param;
  const Tables& t = recon_tables(Scheme::Weno5);
  for (int i = 0; i < 3; ++i) {
    for (int j = 0; j < 3; ++j) {
      p.step1_c[i][j] = t.step1_c[i][j];
      p.gamma[i][j] = t.gamma[i][j];
      for (int l = 0; l < 3; ++l) p.c[i][j][l] = t.c[i][j][l];
    }
    p.gamma_plus[i] = t.gamma_plus[i];
    p.gamma_minus[i] = t.gamma_minus[i];
    p.weno_d[i] = t.weno_d[i];
  }
  p.sigma_plus = t.sigma_plus;
  p.sigma_minus = t.sigma_minus;
  return p;
}

// smoothness_indicators (reconstruction.hpp:174-185); std::pow(x, 2) == x * x.
__device__ inline void smoothness(const double* v, double* b) {
  const double c = 13.0 / 12.0;
  double t1 = v[2] - 2 * v[3] + v[4], t2 = 3 * v[2] - 4 * v[3] + v[4];
  b[0] = c * (t1 * t1) + 0.25 * (t2 * t2);
  t1 = v[1] - 2 * v[2] + v[3];
  t2 = v[1] - v[3];
  b[1] = c * (t1 * t1) + 0.25 * (t2 * t2);
  t1 = v[0] - 2 * v[1] + v[2];
  t2 = v[0] - 4 * v[1] + 3 * v[2];
  b[2] = c * (t1 * t1) + 0.25 * (t2 * t2);
}

// weno_weights (reconstruction.hpp:188-200)
__device__ inline void weno_weights(const double* beta, const double* ideal, double eps, double* w) {
  double total = 0;
  for (int r = 0; r < 3; ++r) {
    const double d = beta[r] + eps;
    w[r] = ideal[r] / (d * d);
    total += w[r];
  }
  for (int r = 0; r < 3; ++r) w[r] /= total;
}

// weno5_step1_value (reconstruction.hpp:205-218)
__device__ inline double weno_step1(const double* v, const FnParams& p) {
  double beta[3], w[3];
  smoothness(v, beta);
  weno_weights(beta, p.weno_d, p.a, w);
  double out = 0;
  for (int r = 0; r < 3; ++r) {
    double cand = 0;
    for (int l = 0; l < 3; ++l) cand += p.step1_c[r][l] * v[2 - r + l];
    out += w[r] * cand;
  }
  return out;
}

// weno5_step2_value (reconstruction.hpp:221-247)
__device__ inline double weno_step2(const double* v, int m, const FnParams& p) {
  double beta[3], cand[3];
  smoothness(v, beta);
  for (int r = 0; r < 3; ++r) {
    cand[r] = 0;
    for (int l = 0; l < 3; ++l) cand[r] += p.c[m][r][l] * v[2 - r + l];
  }
  if (m == 1) {
    double wp[3], wm[3];
    weno_weights(beta, p.gamma_plus, p.a, wp);
    weno_weights(beta, p.gamma_minus, p.a, wm);
    double up = 0, um = 0;
    for (int r = 0; r < 3; ++r) {
      up += wp[r] * cand[r];
      um += wm[r] * cand[r];
    }
    return p.sigma_plus * up - p.sigma_minus * um;
  }
  double w[3];
  weno_weights(beta, p.gamma[m], p.a, w);
  double out = 0;
  for (int r = 0; r < 3; ++r) out += w[r] * cand[r];
  return out;
}

// Returns false on a domain error (the reference functor throws -> EvaluationError).
__device__ inline bool apply_fn(const FnParams& p, const double* v, double& out) {
  switch (p.fn) {
    case FN_IDENTITY: out = v[0]; return true;
    case FN_PRODUCT: out = v[0] * v[1]; return true;
    case FN_SQRT:
      if (v[0] < 0) return false;
      out = sqrt(v[0]);
      return true;
    case FN_AFFINE: out = 2.0 * v[0] + 1.0; return true;
    case FN_SQUARE: out = v[0] * v[0]; return true;
    case FN_WENO5_S1_MINUS: out = weno_step1(v, p); return true;
    case FN_WENO5_S1_PLUS: {
      const double rev[5] = {v[4], v[3], v[2], v[1], v[0]};
      out = weno_step1(rev, p);
      return true;
    }
    case FN_WENO5_S2_QUAD: out = weno_step2(v, int(v[5] + 0.5), p); return true;
    case FN_LLF_LAMBDA:
      if (v[0] <= 0.0 || v[2] <= 0.0) return false;
      out = fmax(fabs(v[1] / v[0]) + sqrt(p.a * v[0]), fabs(v[3] / v[2]) + sqrt(p.a * v[2]));
      return true;
    case FN_WAVE_SPEED:
      if (v[0] <= 0.0) return false;
      out = fabs(v[1] / v[0]) + sqrt(p.a * v[0]);
      return true;
  }
  return false;
}

__device__ inline void operand_values(const OpSet& o, Index i, Index j, double* v) {
  for (int k = 0; k < o.nops; ++k) {
    const double* x = o.X[k];
    const double* y = o.Yt[k];
    double s = 0;
    for (int a = 0; a < o.r[k]; ++a) s += x[i + a * o.m] * y[j + a * o.n];
    v[k] = s;
  }
}

// Column fibers Z(:, cols[c]) -> out (m x nc); error key = c * m + i (evaluation order).
__global__ void k_eval_cols(OpSet o, FnParams p, const long* __restrict__ cols, int nc, double* __restrict__ out,
                            unsigned long long* err) {
  const Index total = o.m * nc;
  for (Index idx = Index(blockIdx.x) * blockDim.x + threadIdx.x; idx < total; idx += Index(gridDim.x) * blockDim.x) {
    const Index i = idx % o.m, c = idx / o.m;
    double v[kMaxOps], z = 0;
    operand_values(o, i, cols[c], v);
    if (!apply_fn(p, v, z)) {
      atomicMin(err, (unsigned long long)idx);
      z = 0;
    }
    out[idx] = z;
  }
}

// Row fibers Z(rows[k], :) written transposed: out (n x nr) = core_y^T of the result.
__global__ void k_eval_rows(OpSet o, FnParams p, const long* __restrict__ rows, int nr, double* __restrict__ out,
                            unsigned long long* err) {
  const Index total = o.n * nr;
  for (Index idx = Index(blockIdx.x) * blockDim.x + threadIdx.x; idx < total; idx += Index(gridDim.x) * blockDim.x) {
    const Index j = idx % o.n, k = idx / o.n;
    double v[kMaxOps], z = 0;
    operand_values(o, rows[k], j, v);
    if (!apply_fn(p, v, z)) {
      atomicMin(err, (unsigned long long)(k * o.n + j));
      z = 0;
    }
    out[idx] = z;
  }
}

// Validation entries: z[s] = f(ops(i_s, j_s)), d[s] = z - basis(i_s,:) . rowvals(:, j_s)
__global__ void k_eval_entries(OpSet o, FnParams p, const long* __restrict__ ij, int ns, const double* __restrict__ bx,
                               const double* __restrict__ by, int rr, double* __restrict__ zd,
                               unsigned long long* err) {
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < ns; s += gridDim.x * blockDim.x) {
    const Index i = ij[2 * s], j = ij[2 * s + 1];
    double v[kMaxOps], z = 0;
    operand_values(o, i, j, v);
    if (!apply_fn(p, v, z)) {
      atomicMin(err, (unsigned long long)s);
      z = 0;
    }
    double zh = 0;
    for (int a = 0; a < rr; ++a) zh += bx[i + a * o.m] * by[j + a * o.n];
    zd[2 * s] = z;
    zd[2 * s + 1] = z - zh;
  }
}

__device__ inline double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Column-major "first index" ordering of (i, j): smaller j first, then smaller i.
__device__ inline bool better(double v, long key, double bv, long bkey) {
  return v > bv || (v == bv && key < bkey);
}

// Full-pivot LU (Eigen::FullPivLU semantics) of W (n x r, in place, ld n) by one CTA.
// Writes orig[k] = original row of pivot k and info = {rank}.
__global__ void __launch_bounds__(1024) k_fullpiv_lu(double* W, Index n, int r, long* orig, long* out_info) {
  __shared__ double sv[32];
  __shared__ long sk[32];
  __shared__ double best_v;
  __shared__ long best_k;
  __shared__ double maxpivot;
  __shared__ int nonzero;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (Index i = threadIdx.x; i < n; i += blockDim.x) orig[i] = i;
  if (threadIdx.x == 0) {
    maxpivot = 0;
    nonzero = r;
  }
  __syncthreads();
  for (int k = 0; k < r; ++k) {
    const Index rows = n - k;
    const Index cnt = rows * (r - k);
    double bv = -1;
    long bk = LONG_MAX;
    (void)cnt;
    // column-major scan of the trailing block; key t = (j - k) rows + (i - k) orders ties
    // as Eigen's maxCoeff (first index in column-major order)
    for (int j = k; j < r; ++j) {
      const double* col = W + Index(j) * n;
      const Index base = Index(j - k) * rows - k;
      for (Index i = k + threadIdx.x; i < n; i += blockDim.x) {
        const double v = fabs(col[i]);
        if (better(v, long(base + i), bv, bk)) {
          bv = v;
          bk = long(base + i);
        }
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const long ok = __shfl_xor_sync(0xffffffffu, bk, o);
      if (better(ov, ok, bv, bk)) {
        bv = ov;
        bk = ok;
      }
    }
    if (lane == 0) {
      sv[warp] = bv;
      sk[warp] = bk;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double v = sv[0];
      long kk = sk[0];
      for (int w = 1; w < nw; ++w)
        if (better(sv[w], sk[w], v, kk)) {
          v = sv[w];
          kk = sk[w];
        }
      best_v = v;
      best_k = kk;
      if (v == 0.0) nonzero = k;
      if (v > maxpivot) maxpivot = v;
    }
    __syncthreads();
    if (best_v == 0.0) break;
    const Index bi = k + best_k % rows, bj = k + best_k / rows;
    if (bi != k)
      for (int j = threadIdx.x; j < r; j += blockDim.x) {
        const double t = W[k + Index(j) * n];
        W[k + Index(j) * n] = W[bi + Index(j) * n];
        W[bi + Index(j) * n] = t;
      }
    if (bi != k && threadIdx.x == 0) {
      const long t = orig[k];
      orig[k] = orig[bi];
      orig[bi] = t;
    }
    __syncthreads();  // row swap and column swap share the pivot entries
    if (bj != k)
      for (Index i = threadIdx.x; i < n; i += blockDim.x) {
        const double t = W[i + k * n];
        W[i + k * n] = W[i + bj * n];
        W[i + bj * n] = t;
      }
    __syncthreads();
    const double d = W[k + k * n];
    for (Index i = k + 1 + threadIdx.x; i < n; i += blockDim.x) W[i + k * n] /= d;
    __syncthreads();
    for (int j = k + 1; j < r; ++j) {
      const double wkj = W[k + Index(j) * n];
      double* col = W + Index(j) * n;
      const double* ck = W + Index(k) * n;
      for (Index i = k + 1 + threadIdx.x; i < n; i += blockDim.x) col[i] -= ck[i] * wkj;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double thr = maxpivot * double(r < n ? r : n) * DBL_EPSILON;
    long rank = 0;
    for (int i = 0; i < nonzero; ++i) rank += fabs(W[i + Index(i) * n]) > thr;
    out_info[0] = rank;
  }
}

// k_fullpiv_lu on a thread-block cluster: the n x r matrix is distributed over the CTAs'
// shared memories by contiguous row blocks (read from M, never written back: maxvol needs
// only the pivot order and the rank). Rows never move: a row swap only exchanges the two
// rows' logical positions (the tie-break key uses logical positions exactly as the
// in-place kernel's), pivot rows are retired, and the column swap and elimination are
// applied to each CTA's live rows with the same per-element arithmetic (a /= d, then
// a -= l * u, no FMA contraction in this file). Per step one cluster barrier: every CTA
// publishes its best (|value|, key) and the owner of logical row k; every warp reduces
// the C candidates with the same total order, so all CTAs take the same pivot.
constexpr int kLuThreads = 512;

__host__ __device__ inline size_t lu_cluster_smem(Index n, int r, int C) {
  const size_t nb = size_t((n + C - 1) / C);
  return nb * size_t(r) * sizeof(double) + nb * (sizeof(int) + 1) + size_t(r) * 2 * sizeof(double) + 512;
}

__global__ void __launch_bounds__(kLuThreads, 1) k_fullpiv_cluster(const double* __restrict__ M, Index n, int r,
                                                                  long* orig, long* out_info) {
  cg::cluster_group cl = cg::this_cluster();
  const int C = int(cl.num_blocks()), rank = int(cl.block_rank());
  const int nb = int((n + C - 1) / C);
  const Index row0 = Index(rank) * nb;
  const int nl = int(max(Index(0), min(Index(nb), n - row0)));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  extern __shared__ double sm[];
  double* A = sm;                               // own rows, column-major: A[j nb + t]
  double* prow = A + size_t(nb) * r;            // pivot row of the current step (r)
  double* pvals = prow + r;                     // |pivot| of every step (rank test)
  double* cand = pvals + r;                     // 2 x {value, key, row of best, row at k}
  int* lpos = reinterpret_cast<int*>(cand + 8);  // logical position of own row t (-1: retired)
  __shared__ double wv[32];
  __shared__ long wk[32];
  __shared__ int wt[32], wkrow[32];
  for (Index idx = threadIdx.x; idx < Index(nl) * r; idx += blockDim.x) {
    const int t = int(idx % nl), j = int(idx / nl);
    A[Index(j) * nb + t] = M[row0 + t + Index(j) * n];
  }
  for (int t = threadIdx.x; t < nl; t += blockDim.x) lpos[t] = int(row0 + t);
  __syncthreads();
  double maxpivot = 0.0;
  int nonzero = r;
  for (int k = 0; k < r; ++k) {
    const Index rows = n - k;
    double bv = -1.0;
    long bk = LONG_MAX;
    int bt = -1, tk = -1;
    for (int t = threadIdx.x; t < nl; t += blockDim.x) {
      const int i = lpos[t];
      if (i < k) continue;  // retired pivot row
      if (i == k) tk = t;
      for (int j = k; j < r; ++j) {
        const double v = fabs(A[Index(j) * nb + t]);
        const long key = long(Index(j - k) * rows + (i - k));
        if (better(v, key, bv, bk)) {
          bv = v;
          bk = key;
          bt = t;
        }
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const long ok = __shfl_xor_sync(0xffffffffu, bk, o);
      const int ot = __shfl_xor_sync(0xffffffffu, bt, o);
      const int otk = __shfl_xor_sync(0xffffffffu, tk, o);
      if (better(ov, ok, bv, bk)) {
        bv = ov;
        bk = ok;
        bt = ot;
      }
      tk = max(tk, otk);
    }
    if (lane == 0) {
      wv[warp] = bv;
      wk[warp] = bk;
      wt[warp] = bt;
      wkrow[warp] = tk;
    }
    __syncthreads();
    double* cb = cand + 4 * (k & 1);
    if (threadIdx.x == 0) {
      for (int w = 1; w < nw; ++w) {
        if (better(wv[w], wk[w], bv, bk)) {
          bv = wv[w];
          bk = wk[w];
          bt = wt[w];
        }
        tk = max(tk, wkrow[w]);
      }
      cb[0] = bv;
      cb[1] = double(bk);
      cb[2] = double(bt);
      cb[3] = double(tk);
    }
    cl.sync();
    // global pivot (every warp, identical): best over the C candidates, owner of row k
    double gv = -1.0;
    long gk = LONG_MAX;
    int gc = -1, gt = -1, kc = -1, kt = -1;
    if (lane < C) {
      const double* rc = cl.map_shared_rank(cb, lane);
      gv = rc[0];
      gk = long(rc[1]);
      gt = int(rc[2]);
      gc = lane;
      if (rc[3] >= 0) {
        kc = lane;
        kt = int(rc[3]);
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, gv, o);
      const long ok = __shfl_xor_sync(0xffffffffu, gk, o);
      const int oc = __shfl_xor_sync(0xffffffffu, gc, o);
      const int ot = __shfl_xor_sync(0xffffffffu, gt, o);
      const int okc = __shfl_xor_sync(0xffffffffu, kc, o);
      const int okt = __shfl_xor_sync(0xffffffffu, kt, o);
      if (better(ov, ok, gv, gk)) {
        gv = ov;
        gk = ok;
        gc = oc;
        gt = ot;
      }
      if (okc > kc) {
        kc = okc;
        kt = okt;
      }
    }
    if (gv == 0.0) {
      nonzero = k;
      break;
    }
    if (gv > maxpivot) maxpivot = gv;
    const int bj = k + int(gk / rows);
    const int bi = k + int(gk % rows);
    // pivot row (retired from now on, so its owner never modifies it again)
    const double* src = cl.map_shared_rank(A, gc);
    for (int j = threadIdx.x; j < r; j += blockDim.x) prow[j] = src[Index(j) * nb + gt];
    __syncthreads();
    if (threadIdx.x == 0) {
      if (bj != k) {
        const double tswap = prow[k];
        prow[k] = prow[bj];
        prow[bj] = tswap;
      }
      pvals[k] = gv;
      if (rank == 0) orig[k] = long(Index(gc) * nb + gt);
      if (rank == kc && !(kc == gc && kt == gt)) lpos[kt] = bi;  // the row at k moves to bi
      if (rank == gc) lpos[gt] = -1;                              // the pivot row retires
    }
    __syncthreads();
    const double d = prow[k];
    for (int t = threadIdx.x; t < nl; t += blockDim.x) {
      if (lpos[t] < 0) continue;
      if (bj != k) {
        const double tswap = A[Index(k) * nb + t];
        A[Index(k) * nb + t] = A[Index(bj) * nb + t];
        A[Index(bj) * nb + t] = tswap;
      }
      const double l = A[Index(k) * nb + t] / d;
      A[Index(k) * nb + t] = l;
      for (int j = k + 1; j < r; ++j) A[Index(j) * nb + t] -= l * prow[j];
    }
    __syncthreads();
  }
  if (rank == 0 && threadIdx.x == 0) {
    const double thr = maxpivot * double(Index(r) < n ? r : n) * DBL_EPSILON;
    long rk = 0;
    for (int i = 0; i < nonzero; ++i) rk += pvals[i] > thr;
    out_info[0] = rk;
  }
  cl.sync();  // no CTA leaves while another may still read its rows or candidates
}

// B = M * P^{-1}, P = M[rows] (r x r): partial-pivot LU of P^T (Eigen PartialPivLU)
// computed per CTA in smem, then each thread solves one row. Per-CTA argmax of |B|
// (column-major first index) to cand[blockIdx] = {value, j, i}.
// (The CTA body is shared by k_solve_right, one swap evaluation per launch, and by
// k_maxvol_loop, the whole swap iteration in one cooperative launch; thread 0 gets the
// CTA's best {value, j, i}.)
__device__ void solve_right_cta(const double* __restrict__ M, Index n, int r, const long* rows,
                                double* __restrict__ B, Index row_block, double& out_v, long& out_j, long& out_i) {
  extern __shared__ double sm[];
  double* lu = sm;                      // r x r, lu[i + j*r]
  int* perm = reinterpret_cast<int*>(lu + r * r);
  double* y = reinterpret_cast<double*>(perm + ((r + 1) & ~1));  // r x T
  __shared__ double s_piv;
  __shared__ int s_pi;
  const int T = blockDim.x;
  // P^T(i, j) = P(j, i) = M[rows[j], i]
  for (int idx = threadIdx.x; idx < r * r; idx += T) {
    const int i = idx % r, j = idx / r;
    lu[i + j * r] = M[rows[j] + Index(i) * n];
  }
  for (int i = threadIdx.x; i < r; i += T) perm[i] = i;
  __syncthreads();
  for (int k = 0; k < r; ++k) {
    if (threadIdx.x == 0) {
      int p = k;
      double b = fabs(lu[k + k * r]);
      for (int i = k + 1; i < r; ++i)
        if (fabs(lu[i + k * r]) > b) {
          b = fabs(lu[i + k * r]);
          p = i;
        }
      s_pi = p;
      if (p != k) {
        const int t = perm[k];
        perm[k] = perm[p];
        perm[p] = t;
      }
    }
    __syncthreads();
    const int p = s_pi;
    if (p != k)
      for (int j = threadIdx.x; j < r; j += T) {
        const double t = lu[k + j * r];
        lu[k + j * r] = lu[p + j * r];
        lu[p + j * r] = t;
      }
    __syncthreads();
    if (threadIdx.x == 0) s_piv = lu[k + k * r];
    __syncthreads();
    const double d = s_piv;
    if (d != 0.0)
      for (int i = k + 1 + threadIdx.x; i < r; i += T) lu[i + k * r] /= d;
    __syncthreads();
    const int tail = (r - k - 1) * (r - k - 1);
    for (int t = threadIdx.x; t < tail; t += T) {
      const int i = k + 1 + t % (r - k - 1), j = k + 1 + t / (r - k - 1);
      lu[i + j * r] -= lu[i + k * r] * lu[k + j * r];
    }
    __syncthreads();
  }
  const Index c = row_block * T + threadIdx.x;
  double bv = -1;
  long bj = LONG_MAX, bi = LONG_MAX;
  if (c < n) {
    double* yc = y + threadIdx.x;
    for (int k = 0; k < r; ++k) {
      double s = M[c + Index(perm[k]) * n];
      for (int l = 0; l < k; ++l) s -= lu[k + l * r] * yc[l * T];
      yc[k * T] = s;
    }
    for (int k = r - 1; k >= 0; --k) {
      double s = yc[k * T];
      for (int l = k + 1; l < r; ++l) s -= lu[k + l * r] * yc[l * T];
      yc[k * T] = s / lu[k + k * r];
    }
    for (int j = 0; j < r; ++j) {
      const double v = yc[j * T];
      if (B) B[c + Index(j) * n] = v;
      const double a = fabs(v);
      if (a > bv) {  // j ascending: first max per row
        bv = a;
        bj = j;
        bi = long(c);
      }
    }
  }
  // CTA argmax, ties -> smaller j then smaller i
  __shared__ double rv[32];
  __shared__ long rj[32], ri[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = T >> 5;
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const long oj = __shfl_xor_sync(0xffffffffu, bj, o);
    const long oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > bv || (ov == bv && (oj < bj || (oj == bj && oi < bi)))) {
      bv = ov;
      bj = oj;
      bi = oi;
    }
  }
  if (lane == 0) {
    rv[warp] = bv;
    rj[warp] = bj;
    ri[warp] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < nw; ++w)
      if (rv[w] > bv || (rv[w] == bv && (rj[w] < bj || (rj[w] == bj && ri[w] < bi)))) {
        bv = rv[w];
        bj = rj[w];
        bi = ri[w];
      }
    out_v = bv;
    out_j = bj;
    out_i = bi;
  }
}

__global__ void k_solve_right(const double* __restrict__ M, Index n, int r, const long* __restrict__ rows,
                              double* __restrict__ B, double* __restrict__ cand) {
  double bv;
  long bj, bi;
  solve_right_cta(M, n, r, rows, B, blockIdx.x, bv, bj, bi);
  if (threadIdx.x == 0) {
    cand[3 * blockIdx.x] = bv;
    cand[3 * blockIdx.x + 1] = double(bj);
    cand[3 * blockIdx.x + 2] = double(bi);
  }
}

// The maxvol swap iteration (cross.hpp:40-58) in one cooperative launch: every iteration
// each CTA evaluates its rows of B = M P^{-1} (solve_right_cta, the arithmetic of
// k_solve_right), publishes its best entry, and after a grid barrier every CTA reduces the
// candidates in CTA order exactly as the host loop did (strict improvement, ties to the
// smaller j then i), so all CTAs take the same swap; the candidates are double-buffered by
// iteration parity. No host round trip per swap. out = {iterations, converged}.
__global__ void k_maxvol_loop(const double* __restrict__ M, Index n, int r, long* rows_g, double* cand,
                              long* out, double growth, int max_iter, const long* lu_info) {
  cg::grid_group grid = cg::this_grid();
  __shared__ long rows_s[kMaxvolRank];
  __shared__ double s_bv;
  __shared__ long s_bj, s_bi;
  if (lu_info[0] < r) {  // rank-deficient start: the host raises DegeneracyError
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      out[0] = 0;
      out[1] = 1;
    }
    return;
  }
  for (int i = threadIdx.x; i < r; i += blockDim.x) rows_s[i] = rows_g[i];
  const int G = int(gridDim.x);
  for (int it = 0; it < max_iter; ++it) {
    __syncthreads();
    double bv;
    long bj, bi;
    solve_right_cta(M, n, r, rows_s, nullptr, blockIdx.x, bv, bj, bi);
    double* cb = cand + size_t(it & 1) * 3 * G;
    if (threadIdx.x == 0) {
      cb[3 * blockIdx.x] = bv;
      cb[3 * blockIdx.x + 1] = double(bj);
      cb[3 * blockIdx.x + 2] = double(bi);
    }
    grid.sync();
    if (threadIdx.x == 0) {
      double v = cb[0], j = cb[1], i = cb[2];
      for (int g = 1; g < G; ++g) {
        const double ov = cb[3 * g], oj = cb[3 * g + 1], oi = cb[3 * g + 2];
        if (ov > v || (ov == v && (oj < j || (oj == j && oi < i)))) {
          v = ov;
          j = oj;
          i = oi;
        }
      }
      s_bv = v;
      s_bj = long(j);
      s_bi = long(i);
    }
    __syncthreads();
    if (s_bv <= growth) {
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        for (int q = 0; q < r; ++q) rows_g[q] = rows_s[q];
        out[0] = it;
        out[1] = 1;
      }
      return;
    }
    if (threadIdx.x == 0) rows_s[s_bj] = s_bi;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    out[0] = max_iter;
    out[1] = 0;
  }
}

__global__ void k_sumsq(const double* __restrict__ a, Index count, double* out) {
  __shared__ double sc[32];
  double s = 0;
  for (Index i = threadIdx.x; i < count; i += blockDim.x) s += a[i] * a[i];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) sc[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) t += sc[w];
    *out = t;
  }
}

}  // namespace

namespace {

struct CrossWork {
  Context* ctx;
  std::vector<void*> bufs;
  double* dbl(size_t n) {
    double* p = ctx->alloc(n);
    bufs.push_back(p);
    return p;
  }
  long* lng(size_t n) {
    double* p = ctx->alloc(n);
    bufs.push_back(p);
    return reinterpret_cast<long*>(p);
  }
  ~CrossWork() {
    for (void* p : bufs) ctx->free(p);
  }
};

int solve_threads(int r, size_t smem_optin, size_t& bytes) {
  const size_t fixed = size_t(r) * r * sizeof(double) + size_t((r + 1) & ~1) * sizeof(int);
  for (int T = 256; T >= 32; T -= 32) {
    bytes = fixed + size_t(r) * T * sizeof(double);
    if (bytes <= smem_optin - 2048) return T;
  }
  throw InputError("maxvol: rank too large for the device solver");
}

/// thin_q (cross.hpp:148-153): Householder TSQR + Q * I.
double* thin_q(Context* ctx, CrossWork& w, const double* M, Index rows, Index cols, Index& q) {
  q = std::min(rows, cols);
  QRPlan p = plan_tsqr(ctx, rows, cols);
  tsqr_factor(ctx, p, M, rows);
  std::vector<double> eye(size_t(cols * q), 0.0);
  for (Index k = 0; k < q; ++k) eye[size_t(k + k * cols)] = 1.0;
  double* I = ctx->alloc(size_t(cols * q));
  TTSW_CUDA(cudaMemcpyAsync(I, eye.data(), sizeof(double) * eye.size(), cudaMemcpyHostToDevice, ctx->stream));
  double* Q = w.dbl(size_t(rows * q));
  tsqr_apply(ctx, p, I, cols, int(q), Q, rows);
  ctx->sync();  // eye lifetime
  ctx->free(I);
  free_tsqr(ctx, p);
  return Q;
}

/// Launch B = M P^{-1}; returns the global argmax {value, j, i}.
void solve_right_dev(Context* ctx, const double* M, Index n, int r, const long* rows_dev, double* B, double* cand,
                     double* host_best) {
  size_t bytes = 0;
  const int T = solve_threads(r, ctx->smem_optin, bytes);
  const int grid = int((n + T - 1) / T);
  allow_dynamic_smem(reinterpret_cast<const void*>(k_solve_right), bytes);
  k_solve_right<<<grid, T, bytes, ctx->stream>>>(M, n, r, rows_dev, B, cand);
  ctx->launches++;
  TTSW_CUDA(cudaGetLastError());
  if (host_best) {
    std::vector<double> c(static_cast<size_t>(3 * grid));
    TTSW_CUDA(cudaMemcpyAsync(c.data(), cand, sizeof(double) * c.size(), cudaMemcpyDeviceToHost, ctx->stream));
    ctx->sync();
    double bv = c[0], bj = c[1], bi = c[2];
    for (int g = 1; g < grid; ++g) {
      const double v = c[size_t(3 * g)], j = c[size_t(3 * g + 1)], i = c[size_t(3 * g + 2)];
      if (v > bv || (v == bv && (j < bj || (j == bj && i < bi)))) {
        bv = v;
        bj = j;
        bi = i;
      }
    }
    host_best[0] = bv;
    host_best[1] = bj;
    host_best[2] = bi;
  }
}

/// maxvol (cross.hpp:31-61) on a device matrix M (n x r).
std::vector<Index> maxvol_dev(Context* ctx, const double* M, Index n, Index r) {
  if (n < r) throw ShapeError("maxvol: matrix must have at least as many rows as columns");
  CrossWork w{ctx};
  double* W = w.dbl(size_t(n * r));
  long* orig = w.lng(size_t(n));
  long* info = w.lng(2);
  int lc = 0;  // cluster size of the full-pivot LU (0: it does not fit, single-CTA kernel)
  for (int c : {8, 16})
    if (lu_cluster_smem(n, int(r), c) <= size_t(ctx->smem_optin) - 1024) {
      lc = c;
      break;
    }
  if (lc) {
    const size_t lb = lu_cluster_smem(n, int(r), lc);
    allow_nonportable_cluster(reinterpret_cast<const void*>(k_fullpiv_cluster));
    allow_dynamic_smem(reinterpret_cast<const void*>(k_fullpiv_cluster), lb);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned(lc));
    cfg.blockDim = dim3(kLuThreads);
    cfg.dynamicSmemBytes = lb;
    cfg.stream = ctx->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = unsigned(lc);
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    TTSW_CUDA(cudaLaunchKernelEx(&cfg, k_fullpiv_cluster, M, n, int(r), orig, info));
  } else {
    TTSW_CUDA(cudaMemcpyAsync(W, M, sizeof(double) * size_t(n * r), cudaMemcpyDeviceToDevice, ctx->stream));
    k_fullpiv_lu<<<1, 1024, 0, ctx->stream>>>(W, n, int(r), orig, info);
  }
  ctx->launches++;
  TTSW_CUDA(cudaGetLastError());
  long* rows_dev = w.lng(size_t(r));
  constexpr double kGrowth = 1.01;
  if (r <= kMaxvolRank) {  // else (and when not co-resident) the host-driven swap loop
    size_t bytes = 0;
    const int Ts = solve_threads(int(r), ctx->smem_optin, bytes);
    const int grid = int((n + Ts - 1) / Ts);
    int per_sm = 0;
    allow_dynamic_smem(reinterpret_cast<const void*>(k_maxvol_loop), bytes);
    TTSW_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_maxvol_loop, Ts, bytes));
    if (per_sm > 0 && grid <= per_sm * 148 / 2) {  // co-resident with room for concurrent work
      // the swap loop starts from the full-pivot rows on the device (no host round trip);
      // a rank-deficient LU is reported through info and the loop does not run
      double* cand2 = w.dbl(size_t(6 * grid));
      long* outd = w.lng(2);
      TTSW_CUDA(cudaMemcpyAsync(rows_dev, orig, sizeof(long) * size_t(r), cudaMemcpyDeviceToDevice, ctx->stream));
      const double* Mp = M;
      Index nn = n;
      int rr = int(r);
      double g = kGrowth;
      int mi = 500;
      const long* infop = info;
      void* args[] = {&Mp, &nn, &rr, &rows_dev, &cand2, &outd, &g, &mi, &infop};
      TTSW_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(k_maxvol_loop), grid, Ts, args, bytes,
                                            ctx->stream));
      ctx->launches++;
      long outh[2], rank = 0;
      std::vector<long> rows_h(static_cast<size_t>(r));
      TTSW_CUDA(cudaMemcpyAsync(rows_h.data(), rows_dev, sizeof(long) * size_t(r), cudaMemcpyDeviceToHost,
                                ctx->stream));
      TTSW_CUDA(cudaMemcpyAsync(outh, outd, sizeof(outh), cudaMemcpyDeviceToHost, ctx->stream));
      TTSW_CUDA(cudaMemcpyAsync(&rank, info, sizeof(long), cudaMemcpyDeviceToHost, ctx->stream));
      ctx->sync();
      if (rank < r) throw DegeneracyError("maxvol: matrix is rank deficient");
      if (!outh[1]) throw ConvergenceError("maxvol: swap iteration failed to settle", 0.0, 500);
      std::vector<Index> rows(rows_h.begin(), rows_h.end());
      std::sort(rows.begin(), rows.end());
      return rows;
    }
  }
  std::vector<long> order(static_cast<size_t>(r));
  long rank = 0;
  TTSW_CUDA(cudaMemcpyAsync(order.data(), orig, sizeof(long) * size_t(r), cudaMemcpyDeviceToHost, ctx->stream));
  TTSW_CUDA(cudaMemcpyAsync(&rank, info, sizeof(long), cudaMemcpyDeviceToHost, ctx->stream));
  ctx->sync();
  if (rank < r) throw DegeneracyError("maxvol: matrix is rank deficient");
  std::vector<Index> rows(order.begin(), order.end());
  double* cand = w.dbl(size_t(3 * ((n + 31) / 32 + 1)));
  for (int iter = 0; iter < 500; ++iter) {
    TTSW_CUDA(cudaMemcpyAsync(rows_dev, rows.data(), sizeof(long) * size_t(r), cudaMemcpyHostToDevice, ctx->stream));
    double best[3];
    solve_right_dev(ctx, M, n, int(r), rows_dev, nullptr, cand, best);
    if (best[0] <= kGrowth) {
      std::sort(rows.begin(), rows.end());
      return rows;
    }
    rows[size_t(best[1])] = Index(best[2]);
  }
  throw ConvergenceError("maxvol: swap iteration failed to settle", 0.0, 500);
}

OpSet make_opset(const std::vector<TT>& ops) {
  if (ops.size() > size_t(kMaxOps)) throw InputError("cross_elementwise: too many operands");
  // operands are materialised by the caller (cross_elementwise)
  OpSet o{};
  o.nops = int(ops.size());
  o.m = ops[0]->m;
  o.n = ops[0]->n;
  for (size_t k = 0; k < ops.size(); ++k) {
    o.X[k] = ops[k]->X;
    o.Yt[k] = ops[k]->Yt;
    o.r[k] = int(ops[k]->r);
  }
  return o;
}

int grid_of(Index total) { return int(std::max<Index>(1, std::min<Index>((total + 255) / 256, 148 * 16))); }

void throw_eval(unsigned long long e, const char* phase, Index m, Index n, const long* cols_h, const long* rows_h,
                const long* ij_h);

void check_eval(Context* ctx, unsigned long long* err, const char* phase, Index m, Index n, const long* cols_h,
                const long* rows_h, const long* ij_h) {
  unsigned long long e = 0;
  TTSW_CUDA(cudaMemcpyAsync(&e, err, sizeof(e), cudaMemcpyDeviceToHost, ctx->stream));
  ctx->sync();
  throw_eval(e, phase, m, n, cols_h, rows_h, ij_h);
}

/// Raise the EvaluationError of a failed fiber evaluation (e = first failing flat index,
/// ~0: none), as check_eval does after its own read.
void throw_eval(unsigned long long e, const char* phase, Index m, Index n, const long* cols_h, const long* rows_h,
                const long* ij_h) {
  if (e == ~0ull) return;
  Index i = 0, j = 0;
  if (phase[0] == 'c') {
    i = Index(e % (unsigned long long)m);
    j = cols_h[e / (unsigned long long)m];
  } else if (phase[0] == 'r') {
    i = rows_h[e / (unsigned long long)n];
    j = Index(e % (unsigned long long)n);
  } else {
    i = ij_h[2 * e];
    j = ij_h[2 * e + 1];
  }
  std::ostringstream os;
  os << "cross_elementwise: function failed at entry (" << i << ", " << j << "): domain error";
  throw EvaluationError(os.str(), i, j);
}

}  // namespace

std::vector<Index> maxvol_host(Context* ctx, Index n, Index r, const double* m_colmajor) {
  double* M = ctx->alloc(size_t(n * r));
  TTSW_CUDA(cudaMemcpyAsync(M, m_colmajor, sizeof(double) * size_t(n * r), cudaMemcpyHostToDevice, ctx->stream));
  try {
    auto rows = maxvol_dev(ctx, M, n, r);
    ctx->free(M);
    return rows;
  } catch (...) {
    ctx->free(M);
    throw;
  }
}

/// cross_elementwise_stats (cross.hpp:162-254).
TT cross_elementwise(int fn, double param, const std::vector<TT>& operands_in, const TT& guess_in,
                     const CrossConfig& cfg, CrossStats* stats) {
  if (operands_in.empty()) throw InputError("cross_elementwise: no operands");
  return cross_elementwise_on(operands_in[0]->ctx, fn, param, operands_in, guess_in, cfg, stats);
}

/// The cross on an explicit context (stream): operands may belong to another context
/// on the same device whose stream the caller has ordered before this one (see
/// Solver::rhs); materialised operands are only read.
TT cross_elementwise_on(Context* ctx, int fn, double param, const std::vector<TT>& operands_in, const TT& guess_in,
                        const CrossConfig& cfg, CrossStats* stats) {
  HostRegion hr_(ctx, "cross");
  if (operands_in.empty()) throw InputError("cross_elementwise: no operands");
  std::vector<TT> operands;
  for (const auto& o : operands_in) operands.push_back(materialize(o));
  const TT guess = materialize(guess_in);
  const Index n_rows = operands[0]->m, n_cols = operands[0]->n;
  for (const auto& op : operands)
    if (op->m != n_rows || op->n != n_cols) throw ShapeError("cross_elementwise: operand shapes differ");
  if (guess->m != n_rows || guess->n != n_cols)
    throw ShapeError("cross_elementwise: guess shape differs from operands");
  if (cfg.eps <= 0) throw InputError("cross_elementwise: eps must be positive");
  static const bool prof_on = std::getenv("TTSW_PROFILE_CROSS") != nullptr;
  const auto t_start = std::chrono::steady_clock::now();
  const long launches0 = ctx->launches;

  const Index rank_cap = std::min({cfg.max_rank, n_rows, n_cols});
  const OpSet o = make_opset(operands);
  const FnParams fp = make_fn(fn, param);
  std::mt19937_64 gen(cfg.seed);
  std::uniform_int_distribution<Index> row_dist(0, n_rows - 1), col_dist(0, n_cols - 1);
  CrossWork w{ctx};
  unsigned long long* err = reinterpret_cast<unsigned long long*>(w.lng(1));
  long evaluations = 0;

  std::vector<Index> cols;
  {
    CrossWork tw{ctx};
    Index q = 0;
    double* Q = thin_q(ctx, tw, guess->Yt, guess->n, guess->r, q);
    cols = maxvol_dev(ctx, Q, guess->n, q);
  }
  if (Index(cols.size()) > rank_cap) cols.resize(size_t(rank_cap));

  TT result = materialize(tt_zero(ctx, n_rows, n_cols));
  double residual = INFINITY;
  const int vs = cfg.validation_sample;
  long* ij_dev = w.lng(size_t(2 * std::max(vs, 1)));
  double* zd = w.dbl(size_t(2 * std::max(vs, 1)));
  std::vector<long> ij(size_t(2 * std::max(vs, 1)));
  std::vector<double> zd_h(size_t(2 * std::max(vs, 1)));

  unsigned long long* err_rows = reinterpret_cast<unsigned long long*>(w.lng(1));
  for (int sweep = 1; sweep <= cfg.max_sweeps; ++sweep) {
    CrossWork sw{ctx};
    std::vector<long> rows_keep;  // host copy of the rows of this sweep (error reports)
    TTSW_CUDA(cudaMemsetAsync(err_rows, 0xff, sizeof(unsigned long long), ctx->stream));
    const int nc = int(cols.size());
    std::vector<long> cols_h(cols.begin(), cols.end());
    long* cols_dev = sw.lng(size_t(nc));
    TTSW_CUDA(cudaMemcpyAsync(cols_dev, cols_h.data(), sizeof(long) * size_t(nc), cudaMemcpyHostToDevice, ctx->stream));
    double* C = sw.dbl(size_t(n_rows * nc));
    TTSW_CUDA(cudaMemsetAsync(err, 0xff, sizeof(unsigned long long), ctx->stream));
    k_eval_cols<<<grid_of(n_rows * nc), 256, 0, ctx->stream>>>(o, fp, cols_dev, nc, C, err);
    ctx->launches++;
    TTSW_CUDA(cudaGetLastError());
    evaluations += long(n_rows) * nc;
    // the evaluation check and the column-norm read share one host round trip
    double* nrm = sw.dbl(1);
    k_sumsq<<<1, 1024, 0, ctx->stream>>>(C, n_rows * nc, nrm);
    ctx->launches++;
    double cn2 = 0;
    unsigned long long ecols = 0;
    TTSW_CUDA(cudaMemcpyAsync(&ecols, err, sizeof(ecols), cudaMemcpyDeviceToHost, ctx->stream));
    TTSW_CUDA(cudaMemcpyAsync(&cn2, nrm, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    ctx->sync();
    throw_eval(ecols, "cols", n_rows, n_cols, cols_h.data(), nullptr, nullptr);

    std::vector<Index> rows;
    if (cn2 == 0.0) {
      result = materialize(tt_zero(ctx, n_rows, n_cols));
    } else {
      Index q = 0;
      double* Q = thin_q(ctx, sw, C, n_rows, nc, q);
      rows = maxvol_dev(ctx, Q, n_rows, q);
      std::vector<long> rows_h(rows.begin(), rows.end());
      long* rows_dev = sw.lng(rows.size());
      TTSW_CUDA(cudaMemcpyAsync(rows_dev, rows_h.data(), sizeof(long) * rows.size(), cudaMemcpyHostToDevice,
                                ctx->stream));
      auto res = make_tt(ctx, n_rows, n_cols, Index(rows.size()));
      double* cand = sw.dbl(size_t(3 * (n_rows / 32 + 2)));
      solve_right_dev(ctx, Q, n_rows, int(q), rows_dev, res->X, cand, nullptr);  // basis = Q Q[rows]^{-1}
      TTSW_CUDA(cudaMemsetAsync(err, 0xff, sizeof(unsigned long long), ctx->stream));
      k_eval_rows<<<grid_of(n_cols * Index(rows.size())), 256, 0, ctx->stream>>>(o, fp, rows_dev, int(rows.size()),
                                                                                 res->Yt, err);
      ctx->launches++;
      TTSW_CUDA(cudaGetLastError());
      evaluations += long(n_cols) * long(rows.size());
      // checked together with the validation entries below (rows first, as in sequence)
      TTSW_CUDA(cudaMemcpyAsync(err_rows, err, sizeof(unsigned long long), cudaMemcpyDeviceToDevice, ctx->stream));
      rows_keep = rows_h;
      result = res;
    }

    // Validation on a fresh seeded sample (cross.hpp:212-231).
    for (int s = 0; s < vs; ++s) {
      const Index i = row_dist(gen), j = col_dist(gen);
      ij[size_t(2 * s)] = i;
      ij[size_t(2 * s + 1)] = j;
    }
    if (vs > 0) {
      TTSW_CUDA(cudaMemcpyAsync(ij_dev, ij.data(), sizeof(long) * size_t(2 * vs), cudaMemcpyHostToDevice, ctx->stream));
      TTSW_CUDA(cudaMemsetAsync(err, 0xff, sizeof(unsigned long long), ctx->stream));
      k_eval_entries<<<grid_of(vs), 256, 0, ctx->stream>>>(o, fp, ij_dev, vs, result->X, result->Yt, int(result->r),
                                                          zd, err);
      ctx->launches++;
      TTSW_CUDA(cudaGetLastError());
      unsigned long long ee[2] = {~0ull, ~0ull};
      TTSW_CUDA(cudaMemcpyAsync(&ee[0], err_rows, sizeof(unsigned long long), cudaMemcpyDeviceToHost, ctx->stream));
      TTSW_CUDA(cudaMemcpyAsync(&ee[1], err, sizeof(unsigned long long), cudaMemcpyDeviceToHost, ctx->stream));
      TTSW_CUDA(cudaMemcpyAsync(zd_h.data(), zd, sizeof(double) * size_t(2 * vs), cudaMemcpyDeviceToHost, ctx->stream));
      ctx->sync();
      throw_eval(ee[0], "rows", n_rows, n_cols, nullptr, rows_keep.data(), nullptr);
      throw_eval(ee[1], "entries", n_rows, n_cols, nullptr, nullptr, ij.data());
    } else {
      unsigned long long e0 = ~0ull;
      TTSW_CUDA(cudaMemcpyAsync(&e0, err_rows, sizeof(unsigned long long), cudaMemcpyDeviceToHost, ctx->stream));
      ctx->sync();
      throw_eval(e0, "rows", n_rows, n_cols, nullptr, rows_keep.data(), nullptr);
    }
    evaluations += vs;
    double err2 = 0, mag2 = 0;
    std::vector<std::pair<double, Index>> column_residuals;
    column_residuals.reserve(size_t(vs));
    for (int s = 0; s < vs; ++s) {
      const double z = zd_h[size_t(2 * s)], d = zd_h[size_t(2 * s + 1)];
      err2 += d * d;
      mag2 += z * z;
      column_residuals.emplace_back(std::fabs(d), ij[size_t(2 * s + 1)]);
    }
    const double rms_err = std::sqrt(err2 / vs);
    const double rms_mag = std::sqrt(mag2 / vs);
    residual = rms_mag == 0 ? (rms_err == 0 ? 0.0 : INFINITY) : rms_err / rms_mag;
    if (stats) {
      stats->sweeps = sweep;
      stats->residual = residual;
      stats->evaluations = evaluations;
    }
    if (residual <= cfg.eps) {
      if (prof_on) {
        ctx->sync();
        const double ms =
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();
        std::fprintf(stderr, "cross fn=%d m=%ld n=%ld ops=%zu rank=%ld sweeps=%d evals=%ld launches=%ld ms=%.3f\n", fn,
                     long(n_rows), long(n_cols), operands.size(), long(result->r), sweep, evaluations,
                     ctx->launches - launches0, ms);
      }
      ctx->cross_calls++;
      if (ctx->ctrace) {
        long h = 0;
        for (Index v : rows) h = h * 1000003 + v;
        for (Index v : cols) h = h * 1000003 + v;
        ctx->ctrace->push_back({result->r, sweep, residual, h});
      }
      return result;
    }

    if (!rows.empty()) {
      CrossWork tw{ctx};
      Index q = 0;
      double* Q = thin_q(ctx, tw, result->Yt, n_cols, result->r, q);
      cols = maxvol_dev(ctx, Q, n_cols, q);
    }
    std::sort(column_residuals.begin(), column_residuals.end(),
              [](const auto& a, const auto& b) { return a.first > b.first; });
    Index added = 0;
    for (const auto& [res, j] : column_residuals) {
      if (Index(cols.size()) >= rank_cap || added >= cfg.rank_increment) break;
      if (res == 0) break;
      if (std::find(cols.begin(), cols.end(), j) == cols.end()) {
        cols.push_back(j);
        ++added;
      }
    }
  }
  std::ostringstream os;
  os << "cross_elementwise: tolerance " << cfg.eps << " not met after " << cfg.max_sweeps
     << " sweeps (achieved relative RMS " << residual << ")";
  throw ConvergenceError(os.str(), residual, cfg.max_sweeps);
}

}  // namespace ttsw
