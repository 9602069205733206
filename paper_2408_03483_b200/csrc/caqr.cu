// Communication-avoiding blocked Householder QR (CAQR) for the large-rank roundings.
//
// round (tt.hpp:120-138) needs the R factors of the two cores (m x R, n x R) and, after
// the small SVD, Q * [W; 0] for the truncated outputs. At the ranks the nonlinear and
// WENO configurations reach (R ~ 100-800 on 4097 x 12288 faces) a tree of per-CTA
// Householder factorisations leaves most of the 148 SMs idle and re-reads its blocks
// from L2 once per column. Here every 32-column panel is factored by
//   * k_caqr_leaf  — one CTA per row chunk (256..767 rows, resident in shared memory,
//                    one thread per row); it produces the chunk's reflectors V_i, the
//                    compact-WY factor T_i (Q_i = I - V_i T_i V_i^T) and a 32 x 32 R_i;
//   * k_caqr_top   — one CTA factoring the stack of the R_i (<= 24 x 32 rows) -> V_top,
//                    T_top and the panel's final R rows;
// and the trailing columns are updated by
//   * k_caqr_update_mma3 — one CTA per (chunk, 64-column tile): W = V^T C, W = T^T W,
//                    C -= V W, i.e. a pair of small GEMMs over the chunk on the FP64
//                    tensor cores (mma.sync m8n8k4 f64);
//   * k_caqr_stack  — the same update with the stack reflectors (split over the stack
//                    blocks, then a fixed-order sum).
// The same update kernel with T instead of T^T applies Q to [W; 0] for the outputs
// (panels last to first, the top reflectors before the chunk reflectors).
// Several independent matrices (the X and Y cores of one rounding) run in the same
// launches. Reflector convention as everywhere else (Eigen's makeHouseholder, see
// cta_householder_qr): beta = -sign(c0)||x||, tau = (beta - c0)/beta, v = x/(c0 - beta).
#include <algorithm>
#include <cfloat>
#include <climits>
#include <cstdlib>
#include <cstdio>

#include "kernels.cuh"

namespace ttsw {

namespace {

constexpr int PB = 32;         // panel width
constexpr int PAD = PB + 1;    // shared row stride (doubles) of a panel chunk
constexpr int RPG = 32;        // panel rows per warp in the chunk kernel (one register per row per lane)
constexpr int TOP_RPG = 48;    // panel rows per warp in the stack kernel
constexpr int LEAF_NW = 16;    // warps of the chunk kernel: chunks up to 512 rows
constexpr int TOP_NW = 16;     // warps of the stack kernel: stacks up to 16 x 48 = 768 rows (24 chunks)
constexpr int UT = 256;        // threads of the update kernel
constexpr int CTL = 64;        // column tile of the chunk updates
constexpr int CTT = 16;        // column tile of the (few-CTA) stack updates
constexpr int MAXROWS = TOP_NW * TOP_RPG;

__host__ __device__ inline void chunk_range(Index rows, int L, int i, Index& start, Index& size) {
  const Index base = rows / L, rem = rows % L;
  start = Index(i) * base + (Index(i) < rem ? Index(i) : rem);
  size = base + (Index(i) < rem ? 1 : 0);
}

__device__ inline double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

struct alignas(16) PanelShared {
  double T[PB * PAD];
  double Ys[PB * PAD];     // Ys[c][l] = v_l^T v_c (l < c), the T recurrence inputs
  double red[32 * PB];
  double redn[32];
  double beta[PB], tau[PB], invd[PB];
  double wsum[PB];
  double diag;
  double pad_;
  double vraw[MAXROWS];    // column c (unscaled) for the rows below the diagonal
};

// Householder QR of an nr x bw panel (nr <= NW * RPG) held in registers: warp g owns rows
// [g*RPG, g*RPG + RPG), lane j holds column j of them in ar[]. Per column c: warp 0 turns
// the per-warp tail-norm partials into (beta, tau, 1/(c0 - beta)) while the owner lanes
// publish column c; every lane forms its dot v^T a_j from registers (v = raw / (c0 - beta)
// below the diagonal, 1 on it) and, after the per-warp partials are summed, applies the
// rank-1 update register-locally; the owner lane of column c + 1 computes the next
// tail-norm partial (look-ahead). Lanes keep their column unscaled after its step (the
// scale is applied once at the store, see store_panel), and the compact-WY T is built
// after the loop from the saved V^T v_c columns. Three barriers per column.
template <int NW, int RPG>
__device__ void panel_qr(double (&ar)[RPG], int bw, PanelShared& sh, int lim0 = INT_MAX, int limstep = 0) {
  const int tid = threadIdx.x, lane = tid & 31, g = tid >> 5;
  const int r0 = g * RPG;
  if (lane == 0) {  // tail-norm partial of column 0 (rows > 0) and the first diagonal
    double x = 0.0;
#pragma unroll
    for (int q = 0; q < RPG; ++q)
      if (r0 + q > 0) x += ar[q] * ar[q];
    sh.redn[g] = x;
    if (g == 0) sh.diag = ar[0];
  }
  __syncthreads();
  for (int c = 0; c < bw; ++c) {
    const int qc = c - r0;  // position of row c in this warp (< 0: warp below it, >= RPG: above)
    // rows >= lim0 + (c + 1) limstep are exactly zero in columns <= c (structured stacks):
    // such warps skip the column's arithmetic and contribute zero partials
    const bool act = r0 < lim0 + (c + 1) * limstep;
    const bool act_next = r0 < lim0 + (c + 2) * limstep;
    if (g == 0) {
      double tail2 = lane < NW ? sh.redn[lane] : 0.0;
      tail2 = warp_sum(tail2);
      if (lane == 0) {
        const double c0 = sh.diag;
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
        sh.beta[c] = beta;
        sh.tau[c] = t;
        sh.invd[c] = (t == 0.0) ? 0.0 : 1.0 / d;
      }
    }
    if (act && lane == c && qc < RPG) {  // publish column c below the diagonal (zeros at and above it)
#pragma unroll
      for (int q = 0; q < RPG; ++q) sh.vraw[r0 + q] = (q > qc) ? ar[q] : 0.0;
    }
    __syncthreads();
    const double t = sh.tau[c], invd = sh.invd[c];
    const double2* vb2 = reinterpret_cast<const double2*>(&sh.vraw[r0]);
    double p = 0.0;
    if (!act) {
    } else if (qc < 0) {  // every row of this warp lies below row c
      double pa[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int q = 0; q < RPG; q += 2) {
        const double2 v2 = vb2[q / 2];
        pa[q & 3] += v2.x * ar[q];
        pa[(q + 1) & 3] += v2.y * ar[q + 1];
      }
      p = invd * ((pa[0] + pa[1]) + (pa[2] + pa[3]));
    } else if (qc < RPG) {  // this warp holds row c: the published rows at and above it are zero,
      // so the same vector loop gives the sum over the rows below (adding exact zeros)
      double pa[4] = {0.0, 0.0, 0.0, 0.0};
      double rowc = 0.0;
#pragma unroll
      for (int q = 0; q < RPG; q += 2) {
        const double2 v2 = vb2[q / 2];
        pa[q & 3] += v2.x * ar[q];
        pa[(q + 1) & 3] += v2.y * ar[q + 1];
      }
#pragma unroll
      for (int q = 0; q < RPG; ++q)
        if (q == qc) rowc = ar[q];
      p = rowc + invd * ((pa[0] + pa[1]) + (pa[2] + pa[3]));
    }
    sh.red[g * PB + lane] = p;
    __syncthreads();
    // warp 0 sums the per-warp partials once (the other warps would otherwise each issue
    // NW shared loads per lane: the chain is shared-memory-issue and barrier bound)
    if (g == 0) {
      double wa[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int q = 0; q < NW; ++q) wa[q & 3] += sh.red[q * PB + lane];
      const double ws = (wa[0] + wa[1]) + (wa[2] + wa[3]);
      sh.wsum[lane] = ws;
      // lanes j < c keep column j unscaled: v_j^T v_c = invd_j * (raw_j^T v_c)
      if (lane < c) sh.Ys[c * PAD + lane] = sh.invd[lane] * ws;
    }
    __syncthreads();
    const double w = sh.wsum[lane];
    if (act && lane > c && lane < bw && t != 0.0) {
      const double tw = t * w, twi = tw * invd;
      if (qc < 0) {
#pragma unroll
        for (int q = 0; q < RPG; q += 2) {
          const double2 v2 = vb2[q / 2];
          ar[q] -= twi * v2.x;
          ar[q + 1] -= twi * v2.y;
        }
      } else if (qc < RPG) {
#pragma unroll
        for (int q = 0; q < RPG; q += 2) {
          const double2 v2 = vb2[q / 2];
          ar[q] -= twi * v2.x;
          ar[q + 1] -= twi * v2.y;
        }
#pragma unroll
        for (int q = 0; q < RPG; ++q)
          if (q == qc) ar[q] -= tw;
      }
    }
    if (lane == c + 1) {  // look-ahead: tail-norm partial and diagonal of column c + 1
      const int qn = c + 1 - r0;
      double x = 0.0;
      if (!act_next) {
      } else if (qn < 0) {
        double xa[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int q = 0; q < RPG; ++q) xa[q & 3] += ar[q] * ar[q];
        x = (xa[0] + xa[1]) + (xa[2] + xa[3]);
      } else if (qn < RPG) {
#pragma unroll
        for (int q = 0; q < RPG; ++q) {
          if (q > qn) x += ar[q] * ar[q];
          if (q == qn) sh.diag = ar[q];
        }
      }
      sh.redn[g] = x;
    }
    __syncthreads();
  }
  // compact-WY T (forward): T[c][c] = tau_c, T[0:c, c] = -tau_c T[0:c, 0:c] Ys[c][0:c]
  if (g == 0) {
    for (int i = lane; i < PB * PAD; i += 32) sh.T[i] = 0.0;
    __syncwarp();
    for (int c = 0; c < bw; ++c) {
      double ta[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int l = 0; l < PB; ++l)
        if (l < c) ta[l & 3] += sh.T[lane * PAD + l] * sh.Ys[c * PAD + l];
      const double tc = sh.tau[c];
      if (lane < c) sh.T[lane * PAD + c] = -tc * ((ta[0] + ta[1]) + (ta[2] + ta[3]));
      if (lane == c) sh.T[c * PAD + c] = tc;
      __syncwarp();
    }
  }
  __syncthreads();
}

// Final value of register row q of lane j (column j): R above the diagonal, beta on it,
// v = raw / (c0 - beta) below it.
template <int RPG>
__device__ inline double panel_value(const PanelShared& sh, const double (&ar)[RPG], int q, int r, int j) {
  if (r < j) return ar[q];
  if (r == j) return sh.beta[j];
  return ar[q] * sh.invd[j];
}

__device__ inline int find_prob(const CaqrBatch& B, int kind, int blk, int& local) {
  int p = 0;
  for (int i = 1; i < B.np; ++i)
    if (B.p[i].off[kind] <= blk) p = i;
  local = blk - B.p[p].off[kind];
  return p;
}

template <int NW>
__global__ void __launch_bounds__(NW * 32, 1) k_caqr_leaf(const __grid_constant__ CaqrBatch B) {
  __shared__ PanelShared sh;
  int i;
  const CaqrProb& P = B.p[find_prob(B, 0, blockIdx.x, i)];
  Index start, nr_;
  chunk_range(P.M, P.nblk, i, start, nr_);
  const int nr = int(nr_);
  const int lane = threadIdx.x & 31, r0 = (threadIdx.x >> 5) * RPG;
  const Index row0 = P.j + start;
  double ar[RPG];
  const double* col = P.A + row0 + (P.j + lane) * P.lda;
#pragma unroll
  for (int q = 0; q < RPG; ++q) ar[q] = (lane < P.bw && r0 + q < nr) ? col[r0 + q] : 0.0;
  panel_qr<NW, RPG>(ar, P.bw, sh);
  double* colw = P.A + row0 + (P.j + lane) * P.lda;
  if (lane < P.bw)
#pragma unroll
    for (int q = 0; q < RPG; ++q)
      if (r0 + q < nr) colw[r0 + q] = panel_value(sh, ar, q, r0 + q, lane);
  double* T = P.Tleaf + Index(i) * PB * PB;
  for (int e = threadIdx.x; e < PB * PB; e += NW * 32) T[e] = sh.T[(e % PB) * PAD + e / PB];  // col-major T
}

template <int NW>
__global__ void __launch_bounds__(NW * 32, 1) k_caqr_top(const __grid_constant__ CaqrBatch B) {
  __shared__ PanelShared sh;
  int i;
  const CaqrProb& P = B.p[find_prob(B, 1, blockIdx.x, i)];
  const int bw = P.bw, nrs = P.nblk * bw, nb1 = P.nblk - 1;
  const int lane = threadIdx.x & 31, r0 = (threadIdx.x >> 5) * TOP_RPG;
  __shared__ Index cstart[kCaqrMaxChunks];  // first row of every chunk (relative to j)
  if (threadIdx.x < P.nblk) {
    Index st, sz;
    chunk_range(P.M, P.nblk, int(threadIdx.x), st, sz);
    cstart[threadIdx.x] = st;
  }
  __syncthreads();
  // Rows are factored in the order: chunk 0's rows (its R_0 gives the diagonal), then the
  // other chunks' triangles interleaved by local row (l = 0 of chunks 1.., l = 1 of chunks
  // 1.., ...). Q is the same up to this row order (stored back in stack order), but column c
  // then only involves the first bw + (c + 1)(nblk - 1) rows (the triangles are upper
  // triangular and the reflectors keep them so): warps past that skip the column.
  double ar[TOP_RPG];
  // (chunk, local row) of this warp's first stack position; the following positions step
  // through the interleaved order without a division per element
  int ci0 = 0, l0 = r0;
  if (r0 >= bw && nb1 > 0) {
    const int t = r0 - bw;
    l0 = t / nb1;
    ci0 = 1 + t % nb1;
  }
  auto advance = [&](int sp, int& ci, int& l) {  // (ci, l) of position sp -> of position sp + 1
    if (sp + 1 < bw) {
      l = sp + 1;
    } else if (sp + 1 == bw) {
      ci = 1;
      l = 0;
    } else if (++ci > nb1) {
      ci = 1;
      ++l;
    }
  };
  {
    int ci = ci0, l = l0;
#pragma unroll
    for (int q = 0; q < TOP_RPG; ++q) {
      const int sp = r0 + q;
      double v = 0.0;
      if (sp < nrs && lane < bw && l <= lane) v = P.A[P.j + cstart[ci] + l + (P.j + lane) * P.lda];
      ar[q] = v;
      advance(sp, ci, l);
    }
  }
  panel_qr<NW, TOP_RPG>(ar, bw, sh, bw, nb1);
  if (lane < bw) {
    int ci = ci0, l = l0;
#pragma unroll
    for (int q = 0; q < TOP_RPG; ++q) {
      const int sp = r0 + q;
      const int ci_q = ci, l_q = l;
      advance(sp, ci, l);
      const int s = ci_q * bw + l_q;
      const double v = panel_value(sh, ar, q, sp, lane);
      if (sp < nrs) P.Vtop[s + Index(lane) * nrs] = v;
      // the panel's final R rows (chunk 0 starts at row j)
      if (s < bw && s <= lane) P.A[P.j + s + (P.j + lane) * P.lda] = v;
    }
  }
  for (int e = threadIdx.x; e < PB * PB; e += NW * 32) P.Ttop[e] = sh.T[(e % PB) * PAD + e / PB];
}

// FP64 tensor-core MMA (sm_80+ mma.sync, available on sm_100a; tcgen05 has no f64
// kind): D(8x8) = A(8x4, row) B(4x8, col) + C. Fragments per lane: a = A[lane/4][lane%4],
// b = B[lane%4][lane/4], c/d = C[lane/4][2*(lane%4) + {0,1}].
__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async8(double* smem_dst, const double* gsrc, bool valid) {
  const unsigned saddr = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  const int sz = valid ? 8 : 0;  // 0: no bytes read, the destination is zero-filled
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(saddr), "l"(gsrc), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Chunk update with two warp groups of 8 warps that take alternate 32-row slabs
// (the slab loop is a chain of DMMA accumulations and cp.async round trips; two groups
// halve it). Each group has its own double buffers and synchronises on its own named
// barrier; W = V^T C is the sum of the two groups' partials (fixed order).
struct UpdMma3Shared {
  double Vs[2][2][PB * PAD];
  double Cs[2][2][PB * (CTL + 1)];
  double W[2][PB * (CTL + 1)];
  double T[PB * PAD];
};

__device__ __forceinline__ void group_bar(int id) { asm volatile("bar.sync %0, 256;\n" ::"r"(id)); }

template <bool TRANS>
__global__ void __launch_bounds__(2 * UT) k_caqr_update_mma3(const __grid_constant__ CaqrBatch B) {
  constexpr int CT = CTL, CTP = CT + 1;
  extern __shared__ double sm[];
  UpdMma3Shared& sh = *reinterpret_cast<UpdMma3Shared*>(sm);
  int loc;
  const CaqrProb& P = B.p[find_prob(B, 2, blockIdx.x, loc)];
  const int tid = threadIdx.x, gp = tid >> 8, gt = tid & 255;
  const int lane = tid & 31, warp = gt >> 5;
  const int bw = P.bw;
  const int tile = loc % P.ntile, ci = loc / P.ntile;
  const int col0 = tile * CT;
  const int ncol = min(CT, P.ncols - col0);
  Index start, sz;
  chunk_range(P.M, P.nblk, ci, start, sz);
  const int nr = int(sz);
  const Index row0 = P.j + start;
  const double* V = P.A + row0 + P.j * P.lda;
  const Index ldv = P.lda;
  const double* Tg = P.Tleaf + Index(ci) * PB * PB;
  double* Cb = P.C + Index(P.c0 + col0) * P.ldc + row0;
  const int nslab = (nr + PB - 1) / PB;
  const int nmine = (nslab - gp + 1) / 2;  // slabs gp, gp + 2, ...
  for (int e = tid; e < PB * PB; e += 2 * UT) sh.T[(e % PB) * PAD + e / PB] = Tg[e];
  const int mt = warp & 3, nt0 = (warp >> 2) * 4;
  const int fr = lane >> 2, fk = lane & 3;
  auto issue = [&](int sl, int buf) {
    const int r0 = sl * PB;
    for (int e = gt; e < PB * PB; e += UT) {
      const int rr = e % PB, cc = e / PB, r = r0 + rr;
      const bool ok = r < nr && cc < bw;
      cp_async8(&sh.Vs[gp][buf][rr * PAD + cc], ok ? V + r + Index(cc) * ldv : V, ok);
    }
    for (int e = gt; e < PB * CT; e += UT) {
      const int rr = e % PB, cc = e / PB, r = r0 + rr;
      const bool ok = r < nr && cc < ncol;
      cp_async8(&sh.Cs[gp][buf][rr * CTP + cc], ok ? Cb + r + Index(cc) * P.ldc : Cb, ok);
    }
    cp_async_commit();
  };
  auto vval = [&](int buf, int sl, int rr, int c) -> double {
    const int r = sl * PB + rr;
    if (c >= bw) return 0.0;
    return r > c ? sh.Vs[gp][buf][rr * PAD + c] : (r == c ? 1.0 : 0.0);
  };
  double acc[4][2];
#pragma unroll
  for (int t = 0; t < 4; ++t) acc[t][0] = acc[t][1] = 0.0;
  // W_gp = V^T C over this group's slabs
  if (nmine > 0) issue(gp, 0);
  for (int q = 0; q < nmine; ++q) {
    const int sl = gp + 2 * q, buf = q & 1;
    if (q + 1 < nmine) {
      issue(sl + 2, buf ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    group_bar(1 + gp);
#pragma unroll
    for (int k0 = 0; k0 < PB; k0 += 4) {
      const double a = vval(buf, sl, k0 + fk, 8 * mt + fr);
#pragma unroll
      for (int t = 0; t < 4; ++t)
        dmma_8x8x4(acc[t][0], acc[t][1], a, sh.Cs[gp][buf][(k0 + fk) * CTP + 8 * (nt0 + t) + fr]);
    }
    group_bar(1 + gp);
  }
  // the first slab of the update pass loads while W is finished
  if (nmine > 0) issue(gp, 0);
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    sh.W[gp][(8 * mt + fr) * CTP + 8 * (nt0 + t) + 2 * fk] = acc[t][0];
    sh.W[gp][(8 * mt + fr) * CTP + 8 * (nt0 + t) + 2 * fk + 1] = acc[t][1];
    acc[t][0] = acc[t][1] = 0.0;
  }
  __syncthreads();
  // W = op(T) (W_0 + W_1)
  for (int e = tid; e < PB * CT; e += 2 * UT) {
    const int r = e % PB, cc = e / PB;
    sh.W[0][r * CTP + cc] += sh.W[1][r * CTP + cc];
  }
  __syncthreads();
  if (gp == 0) {
#pragma unroll
    for (int k0 = 0; k0 < PB; k0 += 4) {
      const int m = 8 * mt + fr, k = k0 + fk;
      const double a = TRANS ? sh.T[k * PAD + m] : sh.T[m * PAD + k];
#pragma unroll
      for (int t = 0; t < 4; ++t) dmma_8x8x4(acc[t][0], acc[t][1], a, sh.W[0][(k0 + fk) * CTP + 8 * (nt0 + t) + fr]);
    }
  }
  __syncthreads();
  if (gp == 0) {
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      sh.W[1][(8 * mt + fr) * CTP + 8 * (nt0 + t) + 2 * fk] = acc[t][0];
      sh.W[1][(8 * mt + fr) * CTP + 8 * (nt0 + t) + 2 * fk + 1] = acc[t][1];
    }
  }
  __syncthreads();
  const double* Wf = sh.W[1];
  // C -= V W, this group's slabs (double-buffered), D starts as the C tile, A = -V
  for (int q = 0; q < nmine; ++q) {
    const int sl = gp + 2 * q, buf = q & 1;
    if (q + 1 < nmine) {
      issue(sl + 2, buf ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    group_bar(1 + gp);
    double d[4][2];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      d[t][0] = sh.Cs[gp][buf][(8 * mt + fr) * CTP + 8 * (nt0 + t) + 2 * fk];
      d[t][1] = sh.Cs[gp][buf][(8 * mt + fr) * CTP + 8 * (nt0 + t) + 2 * fk + 1];
    }
#pragma unroll
    for (int k0 = 0; k0 < PB; k0 += 4) {
      const double a = -vval(buf, sl, 8 * mt + fr, k0 + fk);
#pragma unroll
      for (int t = 0; t < 4; ++t) dmma_8x8x4(d[t][0], d[t][1], a, Wf[(k0 + fk) * CTP + 8 * (nt0 + t) + fr]);
    }
    group_bar(1 + gp);
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      sh.Cs[gp][buf][(8 * mt + fr) * CTP + 8 * (nt0 + t) + 2 * fk] = d[t][0];
      sh.Cs[gp][buf][(8 * mt + fr) * CTP + 8 * (nt0 + t) + 2 * fk + 1] = d[t][1];
    }
    group_bar(1 + gp);
    const int r0 = sl * PB;
    for (int e = gt; e < PB * CT; e += UT) {
      const int rr = e % PB, cc = e / PB, r = r0 + rr;
      if (r < nr && cc < ncol) Cb[r + Index(cc) * P.ldc] = sh.Cs[gp][buf][rr * CTP + cc];
    }
    group_bar(1 + gp);
  }
}

// Stack (top-level) update split over the stack blocks: block i holds chunk i's first bw
// rows (global rows j + start_i + l). PARTIAL: Wp[i] = V_i^T C_i for one 16-column tile
// (K = bw). Otherwise: W = sum_i Wp[i] (fixed order, every CTA of a tile sums the same
// partials identically), W = op(T) W, C_i -= V_i W. op = T^T (TRANS, factorisation) or T.
template <bool PARTIAL, bool TRANS>
__global__ void __launch_bounds__(128) k_caqr_stack(const __grid_constant__ CaqrBatch B) {
  __shared__ double Vs[PB][PAD];
  __shared__ double Cs[PB][CTT + 1];
  __shared__ double W[PB][CTT + 1];
  __shared__ double Ts[PB][PAD];
  int loc;
  const CaqrProb& P = B.p[find_prob(B, 3, blockIdx.x, loc)];
  const int tid = threadIdx.x;
  const int bw = P.bw, nrs = P.nblk * bw;
  const int tile = loc % P.ntile, i = loc / P.ntile;
  const int col0 = tile * CTT, ncol = min(CTT, P.ncols - col0);
  Index start, sz;
  chunk_range(P.M, P.nblk, i, start, sz);
  const Index row0 = P.j + start;
  double* Cb = P.C + Index(P.c0 + col0) * P.ldc;
  for (int e = tid; e < PB * PB; e += 128) {
    const int l = e % PB, c = e / PB, srow = i * bw + l;
    double v = 0.0;
    if (l < bw && c < bw) v = srow > c ? P.Vtop[srow + Index(c) * nrs] : (srow == c ? 1.0 : 0.0);
    Vs[l][c] = v;
  }
  for (int e = tid; e < PB * CTT; e += 128) {
    const int l = e % PB, cc = e / PB;
    Cs[l][cc] = (l < bw && cc < ncol) ? Cb[row0 + l + Index(cc) * P.ldc] : 0.0;
  }
  if (!PARTIAL)
    for (int e = tid; e < PB * PB; e += 128) Ts[e % PB][e / PB] = P.Ttop[e];
  __syncthreads();
  const int cc = tid % CTT, g = tid / CTT;  // outputs (g + 8 x, cc), x < 4
  if (PARTIAL) {
    if (cc < ncol) {
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        const int c = g + 8 * x;
        double acc = 0.0;
#pragma unroll 8
        for (int l = 0; l < PB; ++l) acc += Vs[l][c] * Cs[l][cc];
        P.Wp[(Index(i) * P.ncols + col0 + cc) * PB + c] = acc;
      }
    }
    return;
  }
  // W = sum of the partials, fixed order over the stack blocks
  for (int e = tid; e < PB * CTT; e += 128) {
    const int c = e % PB, ccx = e / PB;
    double acc = 0.0;
    if (ccx < ncol)
      for (int ib = 0; ib < P.nblk; ++ib) acc += P.Wp[(Index(ib) * P.ncols + col0 + ccx) * PB + c];
    W[c][ccx] = acc;
  }
  __syncthreads();
  double w2[4];
#pragma unroll
  for (int x = 0; x < 4; ++x) {
    const int c = g + 8 * x;
    double acc = 0.0;
#pragma unroll 8
    for (int l = 0; l < PB; ++l) acc += (TRANS ? Ts[l][c] : Ts[c][l]) * W[l][cc];
    w2[x] = acc;
  }
  __syncthreads();
#pragma unroll
  for (int x = 0; x < 4; ++x) W[g + 8 * x][cc] = w2[x];
  __syncthreads();
#pragma unroll
  for (int x = 0; x < 4; ++x) {
    const int l = g + 8 * x;
    double acc = 0.0;
#pragma unroll 8
    for (int c = 0; c < PB; ++c) acc += Vs[l][c] * W[c][cc];
    if (l < bw && cc < ncol) Cb[row0 + l + Index(cc) * P.ldc] = Cs[l][cc] - acc;
  }
}

__global__ void k_extract_r(const double* __restrict__ A, Index lda, int R, double* __restrict__ Rout) {
  for (Index e = blockIdx.x * blockDim.x + threadIdx.x; e < Index(R) * R; e += Index(gridDim.x) * blockDim.x) {
    const Index i = e % R, j = e / R;
    Rout[e] = i <= j ? A[i + j * lda] : 0.0;
  }
}

// out (rows x k) = [W (R x k, ldw); 0]
__global__ void k_pad_copy(const double* __restrict__ W, Index ldw, int R, Index rows, int k, double* __restrict__ out,
                           Index ldo) {
  for (Index e = blockIdx.x * Index(blockDim.x) + threadIdx.x; e < rows * k; e += Index(gridDim.x) * blockDim.x) {
    const Index i = e % rows, j = e / rows;
    out[i + j * ldo] = i < R ? W[i + j * ldw] : 0.0;
  }
}

template <class K>
void opt_in_smem(K kernel, size_t bytes) {
  allow_dynamic_smem(reinterpret_cast<const void*>(kernel), bytes);
}

int panel_chunks(Index M) {
  // rows per chunk: TTSW_CHUNK_ROWS (A/B switch), default 256
  static const Index rows = [] {
    const char* e = std::getenv("TTSW_CHUNK_ROWS");
    const long v = e ? std::atol(e) : 256;
    return Index(std::clamp<long>(v, 64, LEAF_NW * RPG));
  }();
  const Index n = std::clamp<Index>(rows == 256 ? M / 256 : (M + rows - 1) / rows, 1, kCaqrMaxChunks);
  return int(n);
}

// chunk updates (I - V op(T) V^T) C on the FP64 tensor cores (k_caqr_update_mma3)
template <bool TRANS>
void launch_update(Context* ctx, CaqrBatch& B, int blocks) {
  if (blocks == 0) return;
  const size_t b3 = sizeof(UpdMma3Shared);
  opt_in_smem(k_caqr_update_mma3<TRANS>, b3);
  k_caqr_update_mma3<TRANS><<<blocks, 2 * UT, b3, ctx->stream>>>(B);
  ctx->launches++;
  TTSW_CUDA(cudaGetLastError());
}

template <bool TRANS>
void launch_stack_update(Context* ctx, CaqrBatch& B) {
  int blocks = 0;
  std::vector<double*> ws;
  for (int q = 0; q < B.np; ++q) {
    CaqrProb& P = B.p[q];
    P.ntile = (P.ncols + CTT - 1) / CTT;
    P.off[3] = blocks;
    P.Wp = nullptr;
    if (P.nblk > 1 && P.ncols > 0) {
      blocks += P.nblk * P.ntile;
      P.Wp = ctx->alloc(size_t(P.nblk) * size_t(P.ncols) * PB);
      ws.push_back(P.Wp);
    }
  }
  if (blocks) {
    k_caqr_stack<true, TRANS><<<blocks, 128, 0, ctx->stream>>>(B);
    k_caqr_stack<false, TRANS><<<blocks, 128, 0, ctx->stream>>>(B);
    ctx->launches += 2;
    TTSW_CUDA(cudaGetLastError());
  }
  for (double* w : ws) ctx->free(w);
}

}  // namespace

bool caqr_fits(Index rows, Index R) {
  return R >= 1 && rows >= R && rows <= Index(kCaqrMaxChunks) * LEAF_NW * RPG;
}

void caqr_factor(Context* ctx, const std::vector<CaqrFactor*>& fs) {
  HostRegion hr_(ctx, "caqr_factor");
  if (fs.empty()) return;
  if (int(fs.size()) > kCaqrMaxProbs) throw CudaError("caqr_factor: too many problems in one batch");
  int npanels = 0;
  for (auto* f : fs) {
    if (!caqr_fits(f->rows, f->R)) throw CudaError("caqr_factor: shape outside the CAQR range");
    f->panels.clear();
    npanels = std::max(npanels, (f->R + PB - 1) / PB);
  }
  // workspace: per panel and problem T_leaf (nblk x 32 x 32), V_top (nblk*32 x 32), T_top
  for (auto* f : fs) {
    const int np_f = (f->R + PB - 1) / PB;
    size_t total = 0;
    for (int p = 0; p < np_f; ++p) {
      const int nb = panel_chunks(f->rows - Index(p) * PB);
      total += size_t(nb) * PB * PB * 2 + PB * PB;
    }
    f->ws = ctx->alloc(total);
    double* cur = f->ws;
    for (int p = 0; p < np_f; ++p) {
      CaqrPanel pn;
      pn.j = Index(p) * PB;
      pn.bw = std::min(PB, f->R - p * PB);
      pn.nblk = panel_chunks(f->rows - pn.j);
      pn.Tleaf = cur;
      cur += size_t(pn.nblk) * PB * PB;
      pn.Vtop = cur;
      cur += size_t(pn.nblk) * PB * PB;
      pn.Ttop = cur;
      cur += PB * PB;
      f->panels.push_back(pn);
    }
  }
  for (int p = 0; p < npanels; ++p) {
    // the matrices that still have panel p (mixed ranks in one batch)
    CaqrBatch B{};
    int nleaf = 0, ntop = 0, nupd = 0, nupdtop = 0;
    for (auto* fp : fs) {
      const CaqrFactor& f = *fp;
      if (p >= int(f.panels.size())) continue;
      const CaqrPanel& pn = f.panels[size_t(p)];
      CaqrProb& P = B.p[B.np++];
      P.A = f.A;
      P.lda = f.lda;
      P.j = pn.j;
      P.bw = pn.bw;
      P.M = f.rows - pn.j;
      P.nblk = pn.nblk;
      P.Tleaf = pn.Tleaf;
      P.Vtop = pn.Vtop;
      P.Ttop = pn.Ttop;
      P.C = f.A;
      P.ldc = f.lda;
      P.c0 = int(pn.j) + pn.bw;
      P.ncols = f.R + f.extra - P.c0;
      P.ntile = (P.ncols + CTL - 1) / CTL;
      P.off[0] = nleaf;
      P.off[1] = ntop;
      P.off[2] = nupd;
      nleaf += P.nblk;
      ntop += P.nblk > 1 ? 1 : 0;
      nupd += P.nblk * P.ntile;
    }
    k_caqr_leaf<LEAF_NW><<<nleaf, LEAF_NW * 32, 0, ctx->stream>>>(B);
    ctx->launches++;
    TTSW_CUDA(cudaGetLastError());
    if (ntop) {
      // the stack factorisation needs only the chunk R factors: it runs on the side stream
      // beside the chunk updates (which need only the chunk reflectors); both join before
      // the stack update. Problems without a stack never map to a top block.
      TTSW_CUDA(cudaEventRecord(ctx->fork_ev, ctx->stream));
      TTSW_CUDA(cudaStreamWaitEvent(ctx->side, ctx->fork_ev, 0));
      k_caqr_top<TOP_NW><<<ntop, TOP_NW * 32, 0, ctx->side>>>(B);
      ctx->launches++;
      TTSW_CUDA(cudaGetLastError());
      TTSW_CUDA(cudaEventRecord(ctx->join_ev, ctx->side));
    }
    launch_update<true>(ctx, B, nupd);
    if (ntop) TTSW_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->join_ev, 0));
    launch_stack_update<true>(ctx, B);
  }
  for (auto* f : fs) {
    const int R = f->R;
    f->Rout = ctx->alloc(size_t(R) * R);
    k_extract_r<<<std::max(1, std::min(1184, (R * R + 255) / 256)), 256, 0, ctx->stream>>>(f->A, f->lda, R, f->Rout);
    ctx->launches++;
    TTSW_CUDA(cudaGetLastError());
  }
}

void caqr_apply(Context* ctx, const std::vector<CaqrFactor*>& fs, const std::vector<const double*>& W,
                const std::vector<Index>& ldw, const std::vector<int>& k, const std::vector<double*>& out,
                const std::vector<Index>& ldo) {
  HostRegion hr_(ctx, "caqr_apply");
  const int nf = int(fs.size());
  int npanels = 0;
  for (int q = 0; q < nf; ++q) {
    const CaqrFactor& f = *fs[size_t(q)];
    const int kq = k[size_t(q)];
    if (kq <= 0) continue;
    npanels = std::max(npanels, int(f.panels.size()));
    const Index total = f.rows * kq;
    k_pad_copy<<<int(std::min<Index>(4 * 148, (total + 255) / 256)), 256, 0, ctx->stream>>>(
        W[size_t(q)], ldw[size_t(q)], f.R, f.rows, kq, out[size_t(q)], ldo[size_t(q)]);
    ctx->launches++;
    TTSW_CUDA(cudaGetLastError());
  }
  for (int p = npanels - 1; p >= 0; --p) {
    CaqrBatch B{};
    int nupd = 0, nupdtop = 0;
    for (int q = 0; q < nf; ++q) {
      const CaqrFactor& f = *fs[size_t(q)];
      const int kq = k[size_t(q)];
      if (kq <= 0 || p >= int(f.panels.size())) continue;
      const CaqrPanel& pn = f.panels[size_t(p)];
      CaqrProb& P = B.p[B.np++];
      P.A = f.A;
      P.lda = f.lda;
      P.j = pn.j;
      P.bw = pn.bw;
      P.M = f.rows - pn.j;
      P.nblk = pn.nblk;
      P.Tleaf = pn.Tleaf;
      P.Vtop = pn.Vtop;
      P.Ttop = pn.Ttop;
      P.C = out[size_t(q)];
      P.ldc = ldo[size_t(q)];
      P.c0 = 0;
      P.ncols = kq;
    }
    if (B.np == 0) continue;
    launch_stack_update<false>(ctx, B);
    for (int q = 0; q < B.np; ++q) {
      CaqrProb& P = B.p[q];
      P.ntile = (P.ncols + CTL - 1) / CTL;
      P.off[2] = nupd;
      nupd += P.nblk * P.ntile;
    }
    launch_update<false>(ctx, B, nupd);
  }
}

void caqr_free(Context* ctx, CaqrFactor& f) {
  if (f.ws) ctx->free(f.ws);
  if (f.Rout) ctx->free(f.Rout);
  f.ws = nullptr;
  f.Rout = nullptr;
  f.panels.clear();
}

}  // namespace ttsw
