// Sketched pre-compression of large-rank rounding inputs (round, tt.hpp:120-138).
//
// The flux Hadamard products and the Taylor-reciprocal terms reach R ~ 200-800 while the
// rounded rank k stays at 20-100: the numerical rank of the represented matrix
// M = X Yt^T is far below R although neither core alone is low rank. Instead of
// orthogonalising both m x R / n x R cores (2 (m + n) R^2 flops of 32-column Householder
// panels), the range of M is captured by a Gaussian sketch:
//   G  = Yt^T Omega              (R x L, Omega n x L, L = l + q: l range columns, q probes)
//   Z  = X G = M Omega           (m x L)
//   Qz = orth(Z[:, :l])          (CAQR; the q probe columns ride along as trailing columns,
//                                 so rows >= l of the transformed probes are exactly
//                                 (I - Qz Qz^T) M omega: the captured-energy check)
//   Ct = X^T Qz                  (R x l)
//   Bt = Yt Ct = M^T Qz          (n x l)
// and the rounding continues on the rank-l TT (Qz, Bt) with the estimated uncaptured energy
// carried as hidden tail energy of the truncation decision (the contract of the pivoted-QR
// pre-truncation of the SVD). All products are plain GEMMs with a long or a
// rank-sized inner dimension and run on the FP64 tensor cores (mma.sync m8n8k4 f64, the
// only f64 MMA sm_100a has: DMMA.8x8x4, 37 TFLOP/s measured, scripts/ubench/dmma_ubench.cu).
#include <algorithm>
#include <cstdio>
#include <cstring>

#include "kernels.cuh"

namespace ttsw {

namespace {

constexpr int BM = 64, BN = 64, BK = 16, NST = 3;
constexpr int LDM = BM + 4;  // shared row stride of a k-major A tile  (k rows of BM)
constexpr int LDK = BK + 4;  // shared row stride of an m- or n-major tile (rows of BK)
constexpr int A_TILE = (BK * LDM > BM * LDK) ? BK * LDM : BM * LDK;
constexpr int B_TILE = BN * LDK;
constexpr int GT = 256;  // threads: 8 warps, 4 along M (16 rows) x 2 along N (32 columns)

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}
__device__ __forceinline__ void cp8(double* smem_dst, const double* gsrc, bool valid) {
  const unsigned saddr = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  const int sz = valid ? 8 : 0;  // 0: nothing read, the destination is zero-filled
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(saddr), "l"(gsrc), "r"(sz));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

/// C (M x N) = op(A) B for a batch of jobs; op(A) = A (M x K, TA = false) or A^T (A stored
/// K x M, TA = true); all column-major. One CTA per (job, 64 x 64 tile, K split); a split
/// job writes its partial products to `part` (ksplit x M x N, ld M) for k_gemm_reduce.
template <bool TA>
__global__ void __launch_bounds__(GT) k_gemm(const GemmJob* __restrict__ jobs, int njobs) {
  extern __shared__ double gsm[];
  int jq = 0;
  for (int i = 1; i < njobs; ++i)
    if (jobs[i].block0 <= int(blockIdx.x)) jq = i;
  const GemmJob& J = jobs[jq];
  int loc = int(blockIdx.x) - J.block0;
  const int tm = loc % J.tiles_m;
  loc /= J.tiles_m;
  const int tn = loc % J.tiles_n;
  const int ks = loc / J.tiles_n;
  const int m0 = tm * BM, n0 = tn * BN;
  const int M = J.M, N = J.N;
  const int chunk = ((J.K + J.ksplit - 1) / J.ksplit + BK - 1) / BK * BK;
  const int kb = ks * chunk, ke = min(J.K, kb + chunk);
  const int nt = ke > kb ? (ke - kb + BK - 1) / BK : 0;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 3, wn = warp >> 2;
  const int fr = lane >> 2, fk = lane & 3;
  const double* __restrict__ A = J.A;
  const double* __restrict__ B = J.B;
  const Index lda = J.lda, ldb = J.ldb;

  auto load = [&](int st, int kt) {
    double* As = gsm + st * (A_TILE + B_TILE);
    double* Bs = As + A_TILE;
    const int k0 = kb + kt * BK;
    if (!TA) {
#pragma unroll
      for (int e = tid; e < BM * BK; e += GT) {
        const int mm = e % BM, kk = e / BM;
        const bool ok = m0 + mm < M && k0 + kk < ke;
        cp8(&As[kk * LDM + mm], ok ? A + (m0 + mm) + Index(k0 + kk) * lda : A, ok);
      }
    } else {
#pragma unroll
      for (int e = tid; e < BM * BK; e += GT) {
        const int kk = e % BK, mm = e / BK;
        const bool ok = m0 + mm < M && k0 + kk < ke;
        cp8(&As[mm * LDK + kk], ok ? A + (k0 + kk) + Index(m0 + mm) * lda : A, ok);
      }
    }
#pragma unroll
    for (int e = tid; e < BN * BK; e += GT) {
      const int kk = e % BK, nn = e / BK;
      const bool ok = n0 + nn < N && k0 + kk < ke;
      cp8(&Bs[nn * LDK + kk], ok ? B + (k0 + kk) + Index(n0 + nn) * ldb : B, ok);
    }
  };

  double acc[2][4][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < NST - 1; ++s) {
    if (s < nt) load(s, s);
    cp_commit();
  }
  for (int kt = 0; kt < nt; ++kt) {
    cp_wait<NST - 2>();
    __syncthreads();
    if (kt + NST - 1 < nt) load((kt + NST - 1) % NST, kt + NST - 1);
    cp_commit();
    const double* As = gsm + (kt % NST) * (A_TILE + B_TILE);
    const double* Bs = As + A_TILE;
#pragma unroll
    for (int k4 = 0; k4 < BK; k4 += 4) {
      double a[2], b[4];
#pragma unroll
      for (int i = 0; i < 2; ++i)
        a[i] = TA ? As[(wm * 16 + 8 * i + fr) * LDK + k4 + fk] : As[(k4 + fk) * LDM + wm * 16 + 8 * i + fr];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[(wn * 32 + 8 * j + fr) * LDK + k4 + fk];
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
  }
  cp_wait<0>();
  double* __restrict__ C = J.ksplit > 1 ? J.part + Index(ks) * M * N : J.C;
  const Index ldc = J.ksplit > 1 ? Index(M) : J.ldc;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int r = m0 + wm * 16 + 8 * i + fr;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = n0 + wn * 32 + 8 * j + 2 * fk;
      if (r < M && c < N) C[r + Index(c) * ldc] = acc[i][j][0];
      if (r < M && c + 1 < N) C[r + Index(c + 1) * ldc] = acc[i][j][1];
    }
  }
}

/// C = sum over the K splits of the partial products, in split order.
__global__ void __launch_bounds__(256) k_gemm_reduce(const GemmJob* __restrict__ jobs, int njobs) {
  const GemmJob& J = jobs[blockIdx.y];
  if (J.ksplit <= 1) return;
  const Index MN = Index(J.M) * J.N;
  for (Index e = Index(blockIdx.x) * blockDim.x + threadIdx.x; e < MN; e += Index(gridDim.x) * blockDim.x) {
    double s = 0.0;
    for (int q = 0; q < J.ksplit; ++q) s += J.part[Index(q) * MN + e];
    J.C[e % J.M + (e / J.M) * J.ldc] = s;
  }
}

__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/// Standard normal entries from a counter-based generator (splitmix64 of the element index,
/// Box-Muller): the sketch matrix depends on nothing but (seed, index).
__global__ void k_fill_gauss(double* __restrict__ out, Index count, unsigned long long seed) {
  for (Index e = Index(blockIdx.x) * blockDim.x + threadIdx.x; e < count; e += Index(gridDim.x) * blockDim.x) {
    const unsigned long long a = mix64(seed ^ (2ULL * (unsigned long long)e));
    const unsigned long long b = mix64(seed ^ (2ULL * (unsigned long long)e + 1ULL));
    const double u1 = (double(a >> 11) + 1.0) * (1.0 / 9007199254740992.0);  // (0, 1]
    const double u2 = double(b >> 11) * (1.0 / 9007199254740992.0);
    out[e] = sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
  }
}

__global__ void k_fill_identity(double* __restrict__ out, int n) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n * n; e += gridDim.x * blockDim.x)
    out[e] = (e % n == e / n) ? 1.0 : 0.0;
}

__device__ inline double block_sum256(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < int(blockDim.x >> 5); ++w) s += red[w];
  return s;
}

/// Captured-energy check of one sketch: Zp (rows x q, ld) holds the probe columns after the
/// reflectors of the l range columns were applied; out = {uncaptured / total probe energy,
/// total probe energy / q (an estimate of ||M||_F^2)}.
__global__ void __launch_bounds__(1024) k_probe_energy(const ProbeJob* __restrict__ jobs) {
  __shared__ double red[32];
  const ProbeJob& J = jobs[blockIdx.x];
  double top = 0.0, rest = 0.0;
  for (Index e = threadIdx.x; e < J.rows * J.q; e += blockDim.x) {
    const Index i = e % J.rows, j = e / J.rows;
    const double v = J.Zp[i + j * J.ld];
    if (i < J.l)
      top += v * v;
    else
      rest += v * v;
  }
  top = block_sum256(top, red);
  rest = block_sum256(rest, red);
  if (threadIdx.x == 0) {
    const double total = top + rest;
    J.out[0] = total > 0.0 ? rest / total : 1.0;
    J.out[1] = total / double(J.q);
  }
}

/// Partial sums of squares of a panel (for the cancellation ratio kappa of the record):
/// part[job * nchunk + chunk].
__global__ void __launch_bounds__(256) k_sumsq_part(const SumsqJob* __restrict__ jobs, int nchunk, double* __restrict__ part) {
  __shared__ double red[8];
  const SumsqJob& J = jobs[blockIdx.y];
  const Index per = (J.count + nchunk - 1) / nchunk;
  const Index b = Index(blockIdx.x) * per, e1 = min(J.count, b + per);
  double s = 0.0;
  for (Index e = b + threadIdx.x; e < e1; e += blockDim.x) {
    const double v = J.a[e];
    s += v * v;
  }
  s = block_sum256(s, red);
  if (threadIdx.x == 0) part[Index(blockIdx.y) * nchunk + blockIdx.x] = s;
}

}  // namespace

void launch_gemm_batch(Context* ctx, std::vector<GemmJob>& jobs, bool trans_a) {
  if (jobs.empty()) return;
  // K splits: enough CTAs to fill the device a few times over, never below 8 k-tiles each
  int total = 0;
  for (auto& J : jobs) {
    J.tiles_m = (J.M + BM - 1) / BM;
    J.tiles_n = (J.N + BN - 1) / BN;
    total += J.tiles_m * J.tiles_n;
  }
  const int want = 3 * ctx->num_sms;
  std::vector<double*> parts;
  int blocks = 0;
  for (auto& J : jobs) {
    int ks = 1;
    if (total < want) ks = std::min((want + total - 1) / total, std::max(1, J.K / (8 * BK)));
    J.ksplit = std::max(1, ks);
    J.part = nullptr;
    if (J.ksplit > 1) {
      J.part = ctx->alloc(size_t(J.ksplit) * size_t(J.M) * size_t(J.N));
      parts.push_back(J.part);
    }
    J.block0 = blocks;
    blocks += J.tiles_m * J.tiles_n * J.ksplit;
  }
  const size_t bytes = sizeof(GemmJob) * jobs.size();
  GemmJob* dj = reinterpret_cast<GemmJob*>(ctx->alloc((bytes + 7) / 8));
  // pageable source: the upload has been staged when the call returns
  TTSW_CUDA(cudaMemcpyAsync(dj, jobs.data(), bytes, cudaMemcpyHostToDevice, ctx->stream));
  const size_t smem = size_t(NST) * (A_TILE + B_TILE) * sizeof(double);
  if (trans_a) {
    allow_dynamic_smem(reinterpret_cast<const void*>(k_gemm<true>), smem);
    k_gemm<true><<<blocks, GT, smem, ctx->stream>>>(dj, int(jobs.size()));
  } else {
    allow_dynamic_smem(reinterpret_cast<const void*>(k_gemm<false>), smem);
    k_gemm<false><<<blocks, GT, smem, ctx->stream>>>(dj, int(jobs.size()));
  }
  ctx->launches++;
  TTSW_CUDA(cudaGetLastError());
  if (!parts.empty()) {
    k_gemm_reduce<<<dim3(64, unsigned(jobs.size())), 256, 0, ctx->stream>>>(dj, int(jobs.size()));
    ctx->launches++;
    TTSW_CUDA(cudaGetLastError());
  }
  for (double* p : parts) ctx->free(p);
  ctx->free(dj);
}

const double* sketch_omega(Context* ctx, Index rows, int cols) {
  if (ctx->omega && ctx->omega_rows >= rows && ctx->omega_cols >= cols) return ctx->omega;
  // grown geometrically; the entries depend only on (seed, row, column), so growing keeps
  // the values of the leading block: column-major with a fixed leading dimension
  const Index ld = kSketchOmegaLd;
  if (rows > ld) throw CudaError("sketch_omega: more rows than the sketch matrix holds");
  const int nc = std::max(cols, std::max(ctx->omega_cols * 2, 136));
  double* fresh = ctx->alloc(size_t(ld) * size_t(nc));
  k_fill_gauss<<<4 * ctx->num_sms, 256, 0, ctx->stream>>>(fresh, ld * Index(nc), 0x7454ce5eedULL);
  ctx->launches++;
  TTSW_CUDA(cudaGetLastError());
  if (ctx->omega) ctx->free(ctx->omega);
  ctx->omega = fresh;
  ctx->omega_rows = ld;
  ctx->omega_cols = nc;
  return ctx->omega;
}

void launch_fill_identity(Context* ctx, double* out, int n) {
  k_fill_identity<<<std::max(1, std::min(296, (n * n + 255) / 256)), 256, 0, ctx->stream>>>(out, n);
  ctx->launches++;
  TTSW_CUDA(cudaGetLastError());
}

void launch_probe_energy(Context* ctx, const std::vector<ProbeJob>& jobs) {
  if (jobs.empty()) return;
  const size_t bytes = sizeof(ProbeJob) * jobs.size();
  ProbeJob* dj = reinterpret_cast<ProbeJob*>(ctx->alloc((bytes + 7) / 8));
  TTSW_CUDA(cudaMemcpyAsync(dj, jobs.data(), bytes, cudaMemcpyHostToDevice, ctx->stream));
  k_probe_energy<<<unsigned(jobs.size()), 1024, 0, ctx->stream>>>(dj);
  ctx->launches++;
  TTSW_CUDA(cudaGetLastError());
  ctx->free(dj);
}

void launch_sumsq_batch(Context* ctx, const std::vector<SumsqJob>& jobs, int nchunk, double* part) {
  if (jobs.empty()) return;
  const size_t bytes = sizeof(SumsqJob) * jobs.size();
  SumsqJob* dj = reinterpret_cast<SumsqJob*>(ctx->alloc((bytes + 7) / 8));
  TTSW_CUDA(cudaMemcpyAsync(dj, jobs.data(), bytes, cudaMemcpyHostToDevice, ctx->stream));
  k_sumsq_part<<<dim3(unsigned(nchunk), unsigned(jobs.size())), 256, 0, ctx->stream>>>(dj, nchunk, part);
  ctx->launches++;
  TTSW_CUDA(cudaGetLastError());
  ctx->free(dj);
}

}  // namespace ttsw
