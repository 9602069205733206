// Internal C++ runtime of the B200 TT-FV library (host side of the C ABI in
// include/ttsw_capi.h). Exceptions mirror the reference's error types
// (/root/reference/proj/include/ttsw/types.hpp:28-56) and are mapped to status codes
// at the C boundary.
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <array>
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace ttsw {

using Index = long;

struct InputError : std::invalid_argument { using std::invalid_argument::invalid_argument; };
struct ShapeError : std::invalid_argument { using std::invalid_argument::invalid_argument; };
struct StateError : std::runtime_error { using std::runtime_error::runtime_error; };
struct DegeneracyError : std::runtime_error { using std::runtime_error::runtime_error; };
struct ConvergenceError : std::runtime_error {
  ConvergenceError(const std::string& w, double r, int it) : std::runtime_error(w), residual(r), iterations(it) {}
  double residual;
  int iterations;
};
struct EvaluationError : std::runtime_error {
  EvaluationError(const std::string& w, Index i, Index j) : std::runtime_error(w), row(i), col(j) {}
  Index row, col;
};
struct CudaError : std::runtime_error { using std::runtime_error::runtime_error; };

void cuda_check(cudaError_t e, const char* what, const char* file, int line);
#define TTSW_CUDA(x) ::ttsw::cuda_check((x), #x, __FILE__, __LINE__)

enum class Axis { X = 0, Y = 1 };
enum class Scheme { Upwind3 = 0, Upwind5 = 1, Weno5 = 2 };
enum class Side { Minus = 0, Plus = 1 };
enum class Model { Linear = 0, Nonlinear = 1 };
inline constexpr Index kGhost = 3;       // types.hpp:24
inline constexpr double kNoRound = -1.0;  // swe.hpp:41

inline int stencil_radius(Scheme s) { return s == Scheme::Upwind3 ? 1 : 2; }
inline int quadrature_points(Scheme s) { return s == Scheme::Upwind3 ? 2 : 3; }

/// Reconstruction tables (ReconTables, reconstruction.hpp:89-160), generated once
/// per process on the host and passed to kernels by value.
struct Tables {
  int radius = 0, nq = 0;
  double offset[3] = {0, 0, 0}, weight[3] = {0, 0, 0};
  double step1_c[3][3] = {};
  double step1_ideal[3] = {};
  double step1_row[5] = {};
  double c[3][3][3] = {};
  double gamma[3][3] = {};
  double point_row[3][5] = {};
  double gamma_plus[3] = {}, gamma_minus[3] = {};
  double sigma_plus = 107.0 / 40.0, sigma_minus = 67.0 / 40.0;
  double weno_d[3] = {};
};
const Tables& recon_tables(Scheme s);

struct RoundRecord {
  Index m, n, r_in, k_out;
  double margin;  // relative distance of the closest truncation comparison to its budget
  double kappa;   // ||core_x||_F ||core_y||_F / ||X||_F (cancellation ratio of the input)
  long crosses;   // cross calls completed before this rounding (trace alignment)
};

struct BandMap;

/// Per cross call: output rank, sweeps, residual and a hash of the final pivots.
struct CrossRecord {
  Index rank;
  int sweeps;
  double residual;
  long pivot_hash;
};

/// What a rounding call site of the solver step did last time: its output rank, the sketch
/// width that was accepted (0: both cores were factored) and whether that width had margin.
struct SketchHint {
  int k = -1;
  int L = 0;
  bool spare = false;
  int fail = 0;  // widest sketch that failed here (never narrowed back to it)
};

/// One CUDA stream + stream-ordered memory pool + launch counter per context.
struct Context : std::enable_shared_from_this<Context> {
  int device = 0;
  cudaStream_t stream = nullptr;
  // side stream for work that overlaps the main stream inside one operation (CAQR: the
  // stack factorisation runs beside the chunk updates), joined by events
  cudaStream_t side = nullptr;
  cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
  long launches = 0;
  long cross_calls = 0;
  int num_sms = 148;
  size_t smem_optin = 227 * 1024;
  // pinned host staging for small scalars read back at sync points
  void* pinned = nullptr;
  std::vector<RoundRecord>* trace = nullptr;
  std::vector<CrossRecord>* ctrace = nullptr;
  // Optional device timing of every rounding (CUDA events on this stream) with the
  // algorithmic work of SURVEY.md Appendix B, for the bench roofline.
  bool time_rounds = false;
  double round_ms = 0, round_flops = 0, round_bytes = 0;
  long round_count = 0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  // Registry of banded maps referenced by lazy terms (uploaded on change).
  std::vector<std::string> map_keys;
  std::vector<char> map_host;  // MapDesc array bytes
  void* map_dev = nullptr;
  size_t map_dev_count = 0;
  int register_map(const BandMap& m);
  const void* device_maps();  // uploads if needed
  // Staging reused by every batched rounding (each batch ends in a stream sync, so the
  // regions are free again at the next call): pinned host + device descriptor area and
  // a device workspace, grown geometrically.
  void* stage_host = nullptr;
  void* stage_dev = nullptr;
  size_t stage_cap = 0;
  double* work_dev = nullptr;
  size_t work_cap = 0;
  void ensure_stage(size_t bytes);
  double* ensure_work(size_t doubles);

  // Sketched pre-compression of large-rank roundings (sketch.cu): the Gaussian test matrix
  // (grown on demand), the switches, and the per-call-site rank hints of the solver step
  // (hint_pos runs over the CAQR-path roundings of a step in issue order; the last output
  // rank seen there sizes the next sketch).
  double* omega = nullptr;
  Index omega_rows = 0;
  int omega_cols = 0;
  bool sketch_on = std::getenv("TTSW_NO_SKETCH") == nullptr;
  int sketch_min_r = std::getenv("TTSW_SKETCH_MIN_R") ? std::atoi(std::getenv("TTSW_SKETCH_MIN_R")) : 160;
  int sketch_default_l = 64;
  std::vector<SketchHint> sketch_hint;
  size_t hint_pos = 0;
  bool hint_active = false;
  long sketch_used = 0, sketch_fallback = 0;

  // Child contexts (same device and memory pool, own stream) for independent work run
  // concurrently from host threads; see fork_join in swe.cu.
  std::vector<std::shared_ptr<Context>> children;
  Context* child(size_t i);

  // host time per region (diagnostic; TTSW_PROFILE_HOST): inclusive wall ms and sync ms
  bool prof_host = std::getenv("TTSW_PROFILE_HOST") != nullptr;
  std::vector<std::pair<std::string, std::array<double, 3>>> host_regions;  // name -> {ms, sync ms, calls}
  // host time blocked in sync() (diagnostic; TTSW_PROFILE_SYNC)
  bool count_sync = std::getenv("TTSW_PROFILE_SYNC") != nullptr || std::getenv("TTSW_PROFILE_HOST") != nullptr;
  double sync_ms = 0;
  long sync_count = 0;

  explicit Context(int dev);
  ~Context();
  double* alloc(size_t count);   // doubles, stream-ordered
  void free(void* p);
  void sync();
};

/// Scoped host-time accounting for TTSW_PROFILE_HOST (inclusive, nested regions double count),
/// and an NVTX range of the same name (rhs, its phases, round_batch, the CAQR groups, crosses).
struct HostRegion {
  Context* ctx;
  const char* name;
  std::chrono::steady_clock::time_point t0;
  double sync0;
  HostRegion(Context* c, const char* n) : ctx(c), name(n) {
    nvtxRangePushA(n);  // NVTX range per region (no-op without an attached tool)
    if (ctx && ctx->prof_host) {
      t0 = std::chrono::steady_clock::now();
      sync0 = ctx->sync_ms;
    }
  }
  ~HostRegion() {
    nvtxRangePop();
    if (!ctx || !ctx->prof_host) return;
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    for (auto& r : ctx->host_regions)
      if (r.first == name) {
        r.second[0] += ms;
        r.second[1] += ctx->sync_ms - sync0;
        r.second[2] += 1;
        return;
      }
    ctx->host_regions.push_back({name, {ms, ctx->sync_ms - sync0, 1.0}});
  }
};

/// Stream-ordered device buffer shared between TT handles (cores are immutable, so
/// apply_core_map / scale share the untouched core instead of copying it).
struct DBuf {
  std::shared_ptr<Context> owner;  // keeps the stream/pool alive while device data exists
  Context* ctx;
  double* p;
  DBuf(Context* c, size_t count) : owner(c->shared_from_this()), ctx(c), p(c->alloc(count)) {}
  ~DBuf() { ctx->free(p); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
};
using Buf = std::shared_ptr<DBuf>;

/// One side (X or Yt) of a lazy term: a base panel and a chain of one-mode ops
/// (device encoding in expr.cuh).
struct HostSideOp {
  int kind;  // 0 scale, 1 map
  int map;
  double scale;
};
struct HostSide {
  Buf base;
  Index ld = 0;
  std::vector<HostSideOp> ops;
};
struct HostTerm {
  int kind = 0;  // TERM_PLAIN / TERM_HADAMARD / TERM_CONST (expr.cuh)
  Index r = 0;
  HostSide x, y;
  Buf x2, y2;  // Hadamard second operand
  Index ldx2 = 0, ldy2 = 0, r2 = 0;
  double cx = 0, cy = 0;  // constant term values
};

/// Device-resident two-core TT (TTMatrix<double>, tt.hpp:19-53). Materialised form:
/// tall column-major panels X = core_x (m x r) and Yt = core_y^T (n x r), so both axes
/// are handled by the same kernels. Lazy form: a list of terms (concatenation,
/// scalings, banded maps, Hadamard products, constants) evaluated only where a kernel
/// needs real cores (rounding input, norms, cross operands). Immutable.
struct DevTT {
  Context* ctx;
  Index m, n, r;
  std::vector<HostTerm> terms;
  Buf xb, yb;            // set iff materialised
  double* X = nullptr;   // valid iff materialised
  double* Yt = nullptr;
  mutable std::shared_ptr<const DevTT> cache;  // memoised materialisation
  DevTT(Context* c, Index m_, Index n_, Index r_, Buf x, Buf y);  // materialised
  DevTT(Context* c, Index m_, Index n_, std::vector<HostTerm> t);  // lazy
  bool materialised() const { return X != nullptr; }
};
using TT = std::shared_ptr<const DevTT>;
using MutTT = std::shared_ptr<DevTT>;

/// Raise a kernel's dynamic shared memory limit to the device maximum (once per kernel,
/// thread-safe; the limit is process-wide, so it is never lowered while another host
/// thread may be launching the kernel).
void allow_dynamic_smem(const void* kernel, size_t bytes);
void allow_nonportable_cluster(const void* kernel);

/// Re-home a materialised TT made on another context (a child) to `ctx`: its buffers are
/// freed on ctx's stream from now on. The caller orders ctx's stream after the producer.
TT adopt(Context* ctx, const TT& x);

/// Materialise a lazy TT into plain cores (one gather kernel); identity if plain.
TT materialize(const TT& x);

MutTT make_tt(Context* ctx, Index m, Index n, Index r);

// ---- TT algebra (tt.hpp) ---------------------------------------------------------------
TT tt_from_host(Context* ctx, Index m, Index n, Index r, const double* cx, const double* cy);
void tt_to_host(const TT& x, double* cx, double* cy);
TT tt_from_full(Context* ctx, Index m, Index n, const double* a, double eps, RoundRecord* rec = nullptr);
TT tt_zero(Context* ctx, Index rows, Index cols);
TT tt_constant(Context* ctx, Index rows, Index cols, double v);
TT round(const TT& x, double eps, RoundRecord* rec = nullptr);
/// Independent roundings in one batch (fused single-CTA kernel where it fits).
std::vector<TT> round_batch(const std::vector<TT>& xs, const std::vector<double>& eps,
                            std::vector<RoundRecord>* recs = nullptr);
/// round_batch with the records routed to caller-owned slots instead of the trace (the
/// solver places them in the reference's sequential order); nullptr slots are dropped.
std::vector<TT> round_batch_into(const std::vector<TT>& xs, const std::vector<double>& eps,
                                 const std::vector<RoundRecord*>& dst);
TT add(const TT& x, const TT& y);
TT scale(const TT& x, double a);
TT hadamard(const TT& x, const TT& y);
double norm_fro(const TT& x);
double sum_entries(const TT& x);
TT reciprocal_taylor(const TT& x, double eps, int max_iterations = 200, int* iterations = nullptr);
/// reciprocal_taylor of independent fields in lock step (each side's arithmetic and stop
/// rule unchanged); side s's rounding records go to sinks[s] in its own order; the first
/// failing side in input order raises, as the sequential reference would.
std::vector<TT> reciprocal_taylor_batch(const std::vector<TT>& xs, double eps,
                                        const std::vector<std::vector<RoundRecord>*>& sinks,
                                        int max_iterations = 200);

/// Banded one-mode operator descriptor: row i of the output reads input rows
/// base(i) + t, t < taps, with base(i) = (i / period) * stride + off[i % period],
/// optionally wrapped modulo n_in (periodic pad).
struct BandMap {
  Index n_out = 0, n_in = 0;
  int period = 1, stride = 1, taps = 1;
  int off[3] = {0, 0, 0};
  double coef[3][5] = {};
  bool wrap = false;
};
BandMap make_band_map(int op, Scheme scheme, Side side, Index n, Index a0, Index a1);
TT apply_core_map(const TT& x, Axis axis, const BandMap& m, double scale_x = 1.0);

// ---- cross (cross.hpp) -----------------------------------------------------------------
struct CrossConfig {
  double eps = 1e-10;
  Index max_rank = 128;
  int max_sweeps = 30;
  Index rank_increment = 2;
  int validation_sample = 1000;
  std::uint64_t seed = 0x5eed5eedULL;
};
struct CrossStats {
  long evaluations = 0;
  int sweeps = 0;
  double residual = 0;
};
enum FnKind : int {
  FN_IDENTITY = 0, FN_PRODUCT = 1, FN_SQRT = 2, FN_AFFINE = 3, FN_SQUARE = 4,
  FN_WENO5_S1_MINUS = 10, FN_WENO5_S1_PLUS = 11, FN_WENO5_S2_QUAD = 12,
  FN_LLF_LAMBDA = 20, FN_WAVE_SPEED = 21
};
TT cross_elementwise(int fn, double param, const std::vector<TT>& ops, const TT& guess, const CrossConfig& cfg,
                     CrossStats* stats = nullptr);
TT cross_elementwise_on(Context* ctx, int fn, double param, const std::vector<TT>& ops, const TT& guess, const CrossConfig& cfg,
                     CrossStats* stats = nullptr);
std::vector<Index> maxvol_host(Context* ctx, Index n, Index r, const double* m_colmajor);

// ---- reconstruction / SWE (reconstruction.hpp, swe.hpp) ---------------------------------
struct FacePair {
  TT minus, plus;
};
struct ReconContext {
  Scheme scheme{};
  double eps_tt = 1e-12;
  CrossConfig cross;
  double dx = 1.0, dy = 1.0;
};
TT periodic_ghost(const TT& x);
TT ghosted(const TT& x, bool dir_x, bool dir_y, const double* strip_x, const double* strip_y, double eps_tt,
           RoundRecord* rec = nullptr);
FacePair reconstruct_faces(const TT& ghosted, Axis axis, const ReconContext& ctx);

struct PhysParams {
  double g = 10.0, f = 1e-4, H = 1000.0;
};
struct SolverOptions {
  Scheme scheme = Scheme::Upwind3;
  Model model = Model::Linear;
  PhysParams params;
  CrossConfig cross;
  double lambda_eps_floor = 1e-6;
};
struct EpsSchedule {
  std::array<double, 3> var{kNoRound, kNoRound, kNoRound};
  double global = kNoRound;
};
/// Policy-mode tolerances (swe.hpp:134-138): C_eps V^(1/2) dx^(p-1/2) / ||q||_F.
struct EpsPolicy {
  double c_eps = 1.0;
  int order = 3;
  double volume = 1.0;
  double clip = 1e-3;
};
using Triple = std::array<TT, 3>;
/// compute_eps_schedule<TTRep> (swe.hpp:167-183): per component eps_for_variable of its
/// Frobenius norm, global from the largest norm (one host sync for the three norms).
EpsSchedule compute_eps_schedule(const Triple& u, const EpsPolicy& policy, double dx);
std::vector<double> norm_fro_batch(const std::vector<TT>& xs);

struct Solver {
  Context* ctx;
  Index n;
  SolverOptions opt;
  EpsSchedule eps;
  double dt;
  Triple state;
  bool tracing = true;
  bool use_policy = false;  // harness.cpp:108-116: schedule recomputed before every step
  EpsPolicy policy;
  std::vector<RoundRecord> trace;
  std::vector<CrossRecord> ctrace;
  double t = 0;  // advanced by dt per step; stage times reach the hooks
  // RhsHooks (swe.hpp:276-282); empty = both axes periodic, no extra source
  std::function<Triple(const Triple&, double)> fill_ghost;
  std::function<Triple(double)> extra_source;
  Triple rhs(const Triple& u, double t_stage);
  void step();
};

/// Full-tensor DenseRep path (swe.hpp:45-80 with rhs/ssprk3, reconstruction.hpp:253-423):
/// three N x N column-major device fields, periodic or Dirichlet (host strips) ghosts.
struct DenseSolver {
  Context* ctx;
  Index n;
  SolverOptions opt;
  double dt;
  double t = 0;
  int bc_x = 0, bc_y = 0;
  // Dirichlet ghost values of component c at time t (strip_x 6 x (n+6), strip_y (n+6) x 6,
  // the ttsw_ghosted layouts) and the cell-average extra source (3 x n x n); 0 = success
  std::function<int(double, int, double*, double*)> strip_fn;
  std::function<int(double, double*)> source_fn;
  double* q[3];
  double *s1[3], *s2[3], *gh[3], *fx[3], *fy[3];
  double *lam, *strips, *src;
  DenseSolver(Context* c, const SolverOptions& o, Index n, double dt);
  ~DenseSolver();
  DenseSolver(const DenseSolver&) = delete;
  DenseSolver& operator=(const DenseSolver&) = delete;
  void step();
  void rhs(double* const out[3]);
  void rhs_stage(double* const w[3], double* const u[3], double* const out[3], double ts, int mode, double a,
                 double b);
  void check_positive();
};

}  // namespace ttsw
