// Kernel launchers (sm_100a). All fp64; all launches go to the context stream.
#pragma once

#include "ttsw.hpp"

namespace ttsw {

struct TermDesc;
struct MapDesc;

/// One rounding of a lazy TT for the fused single-CTA kernel.
struct RoundJob {
  const TermDesc* terms;
  int nterms;
  Index m, n;
  int R;
  double eps;
  double* Xout;   // m x R capacity (first k columns used)
  double* Ytout;  // n x R capacity
  double* A;      // R x R workspace
  double* B;      // R x R workspace
  double* sigma;  // R
  double* info;   // 4: k, margin, sweeps, kappa
  const double* Xs;  // scratch panels (small path): m x R, n x R
  const double* Ys;
  long long* prof;   // optional phase timestamps (clock64), 8 per job; nullptr = off
};
size_t small_round_smem(Index m, Index n, Index R, int rmax);
bool small_round_fits(const Context* ctx, Index m, Index n, Index R);
void launch_round_small(Context* ctx, const RoundJob* jobs, int njobs, Index max_elems, const MapDesc* maps,
                        int nmaps, int max_terms, int rmax, int rows, size_t smem);
size_t fused_round_smem(Index m, Index n, Index R);
void launch_round_fused(Context* ctx, const RoundJob* jobs, int njobs, const MapDesc* maps, size_t smem);
void launch_gather(Context* ctx, const TermDesc* terms, int nterms, const MapDesc* maps, Index m, Index n, Index r,
                   double* X, double* Yt);
/// Batched gather: every job's lazy term list into its Xs / Ys panels (one launch).
void launch_gather_jobs(Context* ctx, const RoundJob* jobs, int njobs, Index max_cols, const MapDesc* maps,
                        int nmaps, int max_terms);
void launch_band_map(Context* ctx, const double* in, Index ld_in, double* out, Index ld_out, Index r,
                     const BandMap& m);
void launch_scale_copy(Context* ctx, double* dst, const double* src, Index count, double a);
void launch_csr_map(Context* ctx, const double* in, Index ld_in, double* out, Index rows, Index r, const long* rowptr,
                    const long* colidx, const double* vals);
void launch_fill(Context* ctx, double* dst, Index count, double v);
void launch_hadamard(Context* ctx, const double* x, Index rx, const double* y, Index ry, Index rows, double* out);
void launch_transpose(Context* ctx, const double* in, Index rows, Index cols, double* out);

/// v = sum_{a,b} (X^T X)_{ab} (Yt^T Yt)_{ab}  (norm_fro, tt.hpp:105-111) -> *out (device)
void launch_norm2(Context* ctx, const double* X, Index m, const double* Yt, Index n, Index r, double* work,
                  double* out);
/// s = sum_a colsum(X)_a colsum(Yt)_a  (sum_entries, tt.hpp:113-116) -> *out (device)
void launch_sum_entries(Context* ctx, const double* X, Index m, const double* Yt, Index n, Index r, double* work,
                        double* out);

// ---- TSQR ------------------------------------------------------------------------------
struct QRLevel {
  Index rows = 0;  // rows of this level's input
  int L = 1;       // number of row blocks (equal split, every block >= R rows unless L == 1)
  double* V = nullptr;    // reflectors, rows x R (ld = rows)
  double* tau = nullptr;  // L x R
  double* Rst = nullptr;  // stacked R factors (L*R) x R, ld = L*R
};
struct QRPlan {
  Index R = 0;
  std::vector<QRLevel> levels;
};

/// Plan the tree for a rows x R panel (host only).
QRPlan plan_tsqr(Context* ctx, Index rows, Index R);
void free_tsqr(Context* ctx, QRPlan& p);
/// Factor A (rows x R, lda) level by level; the final R factor is levels.back().Rst (R x R, ld R).
void tsqr_factor(Context* ctx, QRPlan& p, const double* A, Index lda);
/// out (rows x kc, ld_out) = Q * [C; 0] with C = R x kc (ld_c), Q the thin TSQR factor.
void tsqr_apply(Context* ctx, const QRPlan& p, const double* C, Index ld_c, int kc, double* out, Index ld_out);

// ---- CAQR (caqr.cu) --------------------------------------------------------------------
constexpr int kCaqrMaxChunks = 24;  // row chunks per panel (the top stack is <= 24 x 32 rows)
constexpr int kCaqrMaxProbs = 24;   // independent matrices per launch (12 roundings)
constexpr Index kCaqrMinR = 1;      // every large-panel rounding batches through CAQR (TSQR: rows > 12288)

/// One matrix of a batched CAQR launch (per panel; host-filled, passed by value).
struct CaqrProb {
  double* A;        // factored matrix (reflectors + R), column-major
  Index lda;
  Index j;          // panel offset (row and column)
  int bw;           // panel width
  Index M;          // active rows (rows - j)
  int nblk;         // row chunks of this panel
  double* Tleaf;    // nblk x (32 x 32) compact-WY factors of the chunks
  double* Vtop;     // (nblk*bw) x bw reflectors of the stacked chunk R factors
  double* Ttop;     // 32 x 32
  double* C;        // update target and its columns [c0, c0 + ncols)
  Index ldc;
  int c0, ncols, ntile;
  int off[4];       // first block of this matrix in the leaf / top / update / top-update grids
  double* Wp;       // stack update: per stack block partial products (nblk x ncols x 32)
};
struct CaqrBatch {
  int np;
  CaqrProb p[kCaqrMaxProbs];
};
struct CaqrPanel {
  Index j;
  int bw, nblk;
  double* Tleaf;
  double* Vtop;
  double* Ttop;
};
struct CaqrFactor {
  double* A = nullptr;  // rows x R working copy, overwritten by the factorisation
  Index lda = 0, rows = 0;
  int R = 0;
  int extra = 0;  // trailing columns [R, R + extra) that receive every panel's update but are not factored
  std::vector<CaqrPanel> panels;
  double* ws = nullptr;    // panel workspace
  double* Rout = nullptr;  // R x R upper-triangular factor (ld R), zero below
};
bool caqr_fits(Index rows, Index R);
/// Factor every matrix of the batch (ranks may differ) panel by panel in the same
/// launches; fills panels and Rout.
void caqr_factor(Context* ctx, const std::vector<CaqrFactor*>& fs);
/// out_q (rows_q x k_q) = Q_q [W_q; 0] for every matrix of the batch (k_q = 0: skipped).
void caqr_apply(Context* ctx, const std::vector<CaqrFactor*>& fs, const std::vector<const double*>& W,
                const std::vector<Index>& ldw, const std::vector<int>& k, const std::vector<double*>& out,
                const std::vector<Index>& ldo);
void caqr_free(Context* ctx, CaqrFactor& f);

/// One SVD of a batch: S = Rx Ry^T (R x R, ld R), outputs as launch_svd_small.
struct SvdRequest {
  const double* Rx;
  const double* Ry;
  Index R;
  double eps;
  double* A;
  double* B;
  double* sigma;
  double* info;  // 5 values: k, margin, sweeps, kappa, ambiguous (only written with hidden_rel)
  // Optional device scalar: energy of the represented matrix that S does not carry, as a
  // fraction of ||S||_F^2 (sketched inputs). It joins the tail sum of the truncation
  // decision; info[4] = 1 when the decision would differ without it.
  const double* hidden_rel = nullptr;
};
/// Independent SVDs in one launch per kind (QRCP path for R > 48, cta_svd below).
void launch_svd_batch(Context* ctx, const std::vector<SvdRequest>& reqs);

/// One-sided Jacobi SVD of S = Rx Ry^T (R x R), descending order, truncation rank on
/// device (double-double tail sums, truncation_rank tt.hpp:61-77).
/// Writes A = S V (columns U_j sigma_j), B = V, sigma (R), and info = {k, margin, sweeps}.
/// k = 0 flags an all-zero input (canonical zero result).
void launch_svd_small(Context* ctx, const double* Rx, const double* Ry, Index R, double eps, double* A, double* B,
                      double* sigma, double* info);

// ---- sketched pre-compression (sketch.cu) ----------------------------------------------
constexpr Index kSketchOmegaLd = Index(kCaqrMaxChunks) * 512;  // rows of the Gaussian test matrix (CAQR row limit)
constexpr int kSketchProbes = 8;

/// C (M x N, ldc) = op(A) B; op(A) = A (M x K) or A^T (A stored K x M); column-major.
struct GemmJob {
  const double* A;
  Index lda;
  const double* B;
  Index ldb;
  double* C;
  Index ldc;
  int M, N, K;
  // filled by launch_gemm_batch
  int ksplit, tiles_m, tiles_n, block0;
  double* part;
};
/// All jobs in one launch on the FP64 tensor cores (plus a fixed-order reduction launch when
/// the inner dimension was split).
void launch_gemm_batch(Context* ctx, std::vector<GemmJob>& jobs, bool trans_a);

struct ProbeJob {
  const double* Zp;  // transformed probe columns, rows x q (ld)
  Index ld, rows;
  int l, q;
  double* out;  // {uncaptured fraction, ||M||_F^2 estimate}
};
void launch_probe_energy(Context* ctx, const std::vector<ProbeJob>& jobs);

struct SumsqJob {
  const double* a;
  Index count;
};
/// part[job * nchunk + chunk] = partial sums of squares (summed on the host in order).
void launch_sumsq_batch(Context* ctx, const std::vector<SumsqJob>& jobs, int nchunk, double* part);

/// The context's Gaussian test matrix (ld kSketchOmegaLd), at least rows x cols.
const double* sketch_omega(Context* ctx, Index rows, int cols);
void launch_fill_identity(Context* ctx, double* out, int n);

}  // namespace ttsw
