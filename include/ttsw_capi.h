/* ttsw_capi.h — C ABI of the B200-native TT finite-volume shallow-water hot path.
 *
 * Drop-in boundary for the reference's `Rep` representation plugin
 * (/root/reference/proj/include/ttsw/swe.hpp:84-119) and its step-level callers
 * `rhs<Rep>` (swe.hpp:362-423) / `ssprk3<Rep>` (swe.hpp:428-454). Every entry point
 * below names the reference interface it replaces. Plain pointers and sizes only;
 * all arithmetic is fp64 on the GPU (sm_100a), cores stay resident in HBM.
 *
 * Ownership (reference: TTMatrix is an immutable value type, tt.hpp:19-53): every op
 * returns a NEW caller-owned handle; inputs are never mutated; free with ttsw_tt_free.
 * Errors (reference: exception types, types.hpp:28-56): int status codes below plus
 * ttsw_last_error(). Threading: a context is not thread-safe; contexts are independent.
 */
#ifndef TTSW_CAPI_H
#define TTSW_CAPI_H

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ttsw_ctx ttsw_ctx;
typedef struct ttsw_tt ttsw_tt;
typedef struct ttsw_solver ttsw_solver;
typedef struct ttsw_dense ttsw_dense;
typedef struct ttsw_ensemble ttsw_ensemble;

/* Status codes mirror the reference exception types (types.hpp:28-56). */
enum {
  TTSW_OK = 0,
  TTSW_INPUT = 1,        /* InputError */
  TTSW_SHAPE = 2,        /* ShapeError */
  TTSW_STATE = 3,        /* StateError */
  TTSW_DEGENERACY = 4,   /* DegeneracyError */
  TTSW_CONVERGENCE = 5,  /* ConvergenceError{residual, iterations} */
  TTSW_EVALUATION = 6,   /* EvaluationError{row, col} */
  TTSW_CUDA = 7,         /* CUDA runtime failure (no CPU fallback exists) */
  TTSW_INTERNAL = 8
};

enum { TTSW_AXIS_X = 0, TTSW_AXIS_Y = 1 };                           /* types.hpp:26 */
enum { TTSW_UPWIND3 = 0, TTSW_UPWIND5 = 1, TTSW_WENO5 = 2 };         /* reconstruction.hpp:16 */
enum { TTSW_MINUS = 0, TTSW_PLUS = 1 };                              /* reconstruction.hpp:17 */
enum { TTSW_LINEAR = 0, TTSW_NONLINEAR = 1 };                        /* swe.hpp:15 */

/* One-mode banded operators replacing the dense matrices of reconstruction.hpp:428-501
 * and cases.cpp:302-308 (never materialised). n = interior mode size. */
enum {
  TTSW_MAP_PERIODIC_PAD = 0,  /* periodic_pad_matrix(n)               (n+6) x n     */
  TTSW_MAP_STEP1 = 1,         /* step1_matrix(scheme, side, n)         (n+1) x (n+6) */
  TTSW_MAP_QPOINT = 2,        /* quadrature_point_matrix(scheme, n)    (n nq) x (n+6)*/
  TTSW_MAP_QSUM = 3,          /* quadrature_sum_matrix(scheme, n)      n x (n nq)    */
  TTSW_MAP_DIFF = 4,          /* interface_difference_matrix(n)        n x (n+1)     */
  TTSW_MAP_ROW_SLICE = 5,     /* row_slice_matrix(a0, a1, n+6)         a1 x (n+6)    */
  TTSW_MAP_QSLICE = 6         /* quadrature_slice_matrix(a0, n, nq, k) (n nq) x (n+6)*/
};

/* Fixed device functors replacing the host std::function EntryFn (cross.hpp:64-65). */
enum {
  TTSW_FN_IDENTITY = 0, TTSW_FN_PRODUCT = 1, TTSW_FN_SQRT = 2, TTSW_FN_AFFINE = 3, TTSW_FN_SQUARE = 4,
  TTSW_FN_WENO5_S1_MINUS = 10, /* reconstruction.hpp:546-548, param = eps1 */
  TTSW_FN_WENO5_S1_PLUS = 11,  /* reconstruction.hpp:549-552, param = eps1 */
  TTSW_FN_WENO5_S2_QUAD = 12,  /* reconstruction.hpp:553-556, param = eps2 */
  TTSW_FN_LLF_LAMBDA = 20,     /* swe.hpp:342-347, param = g */
  TTSW_FN_WAVE_SPEED = 21      /* swe.hpp:225-228, param = g */
};

typedef struct {
  double residual;  /* ConvergenceError::residual */
  int iterations;   /* ConvergenceError::iterations */
  long row, col;    /* EvaluationError::row/col */
} ttsw_err_info;

/* CrossConfig (cross.hpp:19-26). */
typedef struct {
  double eps;
  long max_rank;
  int max_sweeps;
  long rank_increment;
  int validation_sample;
  unsigned long long seed;
} ttsw_cross_cfg;

/* CrossResult counters (cross.hpp:67-73). */
typedef struct {
  long evaluations;
  int sweeps;
  double residual;
} ttsw_cross_stats;

/* One rounding decision: truncation_rank (tt.hpp:61-77) plus its margin (relative
 * distance of the closest comparison to the (0.9 eps)^2 ||sigma||^2 budget) and the
 * cancellation ratio kappa = ||core_x||_F ||core_y||_F / ||X||_F of the input. */
typedef struct {
  long m, n, r_in, k_out;
  double margin;
  double kappa;
} ttsw_round_info;

/* Step-level solver: SolverOptions (swe.hpp:285-295) + Grid (nx=ny=n, unit square) +
 * fixed EpsSchedule{var = tol x3, global = tol} (swe.hpp:156-159) + dt. */
typedef struct {
  int model, scheme;
  long n;
  double g, f, H;
  double dt;
  double tol;
  double lambda_eps_floor;  /* SolverOptions::lambda_eps_floor (swe.hpp:294) */
  ttsw_cross_cfg cross;     /* SolverOptions::cross; harness sets seed = RunConfig::seed */
} ttsw_solver_desc;

/* --- context (one stream + stream-ordered pool + error slot per context) --------- */
int ttsw_ctx_create(int device, ttsw_ctx** out);
void ttsw_ctx_destroy(ttsw_ctx* ctx);
int ttsw_last_error(ttsw_ctx* ctx, char* buf, long len, ttsw_err_info* info);
int ttsw_ctx_sync(ttsw_ctx* ctx);
/* cudaStream_t of the context, for event timing by callers. */
void* ttsw_ctx_stream(ttsw_ctx* ctx);
/* Number of kernels this context has launched so far (for launch accounting). */
long ttsw_ctx_launches(ttsw_ctx* ctx);
/* Device timing of every rounding with CUDA events on the context stream (off by
 * default). stats = {ms, algorithmic flops, algorithmic bytes, count}. */
void ttsw_ctx_time_rounds(ttsw_ctx* ctx, int enabled);
void ttsw_ctx_round_stats(ttsw_ctx* ctx, double* stats4, int reset);
/* Sketched pre-compression of large-rank roundings (round, tt.hpp:120-138): a
 * rounding of input rank >= min_rank whose expected output rank is far below it captures the
 * range of the represented matrix from a Gaussian sketch with default_columns columns (the
 * solver sizes later sketches from the output ranks of its previous step) and falls back to
 * factoring both cores when the probes show uncaptured energy above 1e-3 of the truncation
 * budget or the rank decision depends on it. On by default; min_rank/default_columns <= 0
 * keep their values. stats: roundings that used the sketch / fell back since creation. */
void ttsw_ctx_set_sketch(ttsw_ctx* ctx, int enabled, int min_rank, int default_columns);
void ttsw_ctx_sketch_stats(ttsw_ctx* ctx, long* used, long* fallback);

/* --- fields (TTMatrix<double>, tt.hpp:19-53; Eigen column-major core layouts) ----- */
int ttsw_tt_from_host(ttsw_ctx* ctx, long m, long n, long r, const double* cx_colmajor,
                      const double* cy_colmajor, ttsw_tt** out);
/* tt_from_full (tt.hpp:82-97; TTRep::compress, swe.hpp:93-95): dense A (m x n,
 * column-major, host) compressed to a TT with ||A - result||_F <= eps ||A||_F on the device
 * (rounding of the exact rank-min(m,n) TT (A, I) or (I, A)). InputError on non-finite
 * entries or eps < 0; a zero A gives TTMatrix::zero. info (may be NULL) as ttsw_round. */
int ttsw_tt_from_full(ttsw_ctx* ctx, long m, long n, const double* a_colmajor, double eps, ttsw_tt** out,
                      ttsw_round_info* info);
int ttsw_tt_to_host(ttsw_ctx* ctx, const ttsw_tt* x, double* cx_colmajor, double* cy_colmajor);
void ttsw_tt_dims(const ttsw_tt* x, long* m, long* n, long* r);
void ttsw_tt_free(ttsw_tt* x);
int ttsw_tt_constant(ttsw_ctx* ctx, long m, long n, double value, ttsw_tt** out); /* TTMatrix::constant */

/* --- TT algebra (tt.hpp) and the TTRep plugin methods (swe.hpp:84-119) ----------- */
int ttsw_round(ttsw_ctx* ctx, const ttsw_tt* x, double eps, ttsw_tt** out, ttsw_round_info* info); /* round, tt.hpp:120-138 */
int ttsw_add(ttsw_ctx* ctx, const ttsw_tt* x, const ttsw_tt* y, ttsw_tt** out);              /* add, tt.hpp:152-161 */
int ttsw_scale(ttsw_ctx* ctx, const ttsw_tt* x, double a, ttsw_tt** out);                    /* scale, tt.hpp:163-166 */
int ttsw_axpy(ttsw_ctx* ctx, double a, const ttsw_tt* x, double b, const ttsw_tt* y, double eps,
              ttsw_tt** out);                                                                /* TTRep::axpy, swe.hpp:103-105; eps<0 = kNoRound */
int ttsw_hadamard(ttsw_ctx* ctx, const ttsw_tt* x, const ttsw_tt* y, ttsw_tt** out);         /* hadamard, tt.hpp:169-181 */
int ttsw_mul(ttsw_ctx* ctx, const ttsw_tt* x, const ttsw_tt* y, double eps, ttsw_tt** out);  /* TTRep::mul, swe.hpp:106-108 */
int ttsw_core_map(ttsw_ctx* ctx, const ttsw_tt* x, int axis, int op, int scheme, int side, long n, long a0,
                  long a1, ttsw_tt** out);                                                   /* apply_core_map, tt.hpp:185-194 */
/* General one-mode operator given as CSR (rows x cols): dense(out) = M dense(x) (axis X) or
 * dense(x) M^T (axis Y). Lets a drop-in TTRep::lin(Axis, const MatrixXd&, F) (swe.hpp:109-111)
 * pass the reference's own operator matrices (reconstruction.hpp:428-501) by their nonzeros. */
int ttsw_core_map_csr(ttsw_ctx* ctx, const ttsw_tt* x, int axis, long rows, long cols, const long* rowptr,
                      const long* colidx, const double* vals, ttsw_tt** out);            /* apply_core_map, tt.hpp:185-194 */
int ttsw_norm_fro(ttsw_ctx* ctx, const ttsw_tt* x, double* out);                             /* norm_fro, tt.hpp:105-111 */
int ttsw_sum_entries(ttsw_ctx* ctx, const ttsw_tt* x, double* out);                          /* sum_entries, tt.hpp:113-116 */
int ttsw_recip_taylor(ttsw_ctx* ctx, const ttsw_tt* x, double eps, int max_iterations, int* iterations,
                      ttsw_tt** out);                                                        /* reciprocal_taylor, tt.hpp:204-241 */
int ttsw_cross(ttsw_ctx* ctx, int fn, const double* params, const ttsw_tt* const* ops, int nops,
               const ttsw_tt* guess, const ttsw_cross_cfg* cfg, ttsw_tt** out,
               ttsw_cross_stats* stats);                                                     /* cross_elementwise_stats, cross.hpp:162-254 */
int ttsw_maxvol(ttsw_ctx* ctx, long n, long r, const double* m_colmajor, long* rows_out);   /* maxvol, cross.hpp:31-61 */

/* --- reconstruction / ghosting (reconstruction.hpp:611-616, cases.cpp:298-309) ---- */
int ttsw_periodic_ghost(ttsw_ctx* ctx, const ttsw_tt* x, ttsw_tt** out);
/* tt_ghosted (cases.cpp:298-344): bc_x/bc_y 0 = Periodic, 1 = DirichletExact. For a
 * Dirichlet axis the caller passes the exact ghost-cell averages (what the reference's
 * exact_cell_average_at yields): strip_x 6 x (ny+6) column-major (ghost rows 0-2, nx+3..nx+5,
 * every ghosted column), strip_y (nx+6) x 6 (every ghosted row, ghost columns; its corner
 * rows are ignored when both axes are Dirichlet). Interior pad + strips, then round at
 * eps_tt (< 0: no rounding) when a strip was added; all-periodic = ttsw_periodic_ghost. */
int ttsw_ghosted(ttsw_ctx* ctx, const ttsw_tt* x, int bc_x, int bc_y, const double* strip_x, const double* strip_y,
                 double eps_tt, ttsw_tt** out);
int ttsw_reconstruct_faces(ttsw_ctx* ctx, const ttsw_tt* ghosted, int axis, int scheme, double eps_tt,
                           const ttsw_cross_cfg* cfg, double dx, double dy, ttsw_tt** minus, ttsw_tt** plus);

/* --- step level: rhs<Rep> (swe.hpp:362-423) and ssprk3<Rep> (swe.hpp:428-454) ----- */
int ttsw_solver_create(ttsw_ctx* ctx, const ttsw_solver_desc* desc, ttsw_solver** out);
void ttsw_solver_destroy(ttsw_solver* s);
int ttsw_solver_set_state(ttsw_solver* s, int component, const ttsw_tt* x);
int ttsw_solver_get_state(ttsw_solver* s, int component, ttsw_tt** out);
int ttsw_solver_rhs(ttsw_solver* s, ttsw_tt** out3);
int ttsw_solver_step(ttsw_solver* s, long nsteps);
long ttsw_solver_trace_len(const ttsw_solver* s);
/* per rounding: op, m, n, r_in, k_out, crosses-before (6 longs), margin and kappa */
void ttsw_solver_trace(const ttsw_solver* s, long* ints, double* margins, double* kappas);
void ttsw_solver_trace_clear(ttsw_solver* s);
/* per cross call inside the step: output rank, sweeps, pivot hash (3 longs), residual */
long ttsw_solver_cross_trace_len(const ttsw_solver* s);
void ttsw_solver_cross_trace(ttsw_solver* s, long* ints, double* residuals, int clear);
void ttsw_solver_set_tracing(ttsw_solver* s, int enabled);
/* RhsHooks (swe.hpp:276-282), for the Dirichlet/MMS verification cases: fill_ghost gets the
 * stage state q3 (borrowed for the call) and the stage time and returns three ghosted
 * (nx+6) x (ny+6) fields (typically via ttsw_ghosted with exact strips), extra_source
 * returns three cell-average source fields added to the Coriolis source at the flux
 * tolerance (swe.hpp:412-416). Every non-NULL handle a hook writes is taken over by the
 * solver, also when the hook fails (the same handle may fill several slots; it is freed
 * once); a hook returns 0 on success, and the q3 handles are invalid after it returns. NULL restores periodic ghosts / no extra source. Stage times
 * t, t+dt, t+dt/2 (swe.hpp:441-448); the solver time advances by dt per step. */
typedef int (*ttsw_fill_ghost_fn)(void* user, const ttsw_tt* const* q3, double t, ttsw_tt** ghosted3);
typedef int (*ttsw_extra_source_fn)(void* user, double t, ttsw_tt** extra3);
int ttsw_solver_set_hooks(ttsw_solver* s, ttsw_fill_ghost_fn fill_ghost, ttsw_extra_source_fn extra_source,
                          void* user);
int ttsw_solver_set_time(ttsw_solver* s, double t);
/* step size of the following steps (run_impl clips the last step to land on T, harness.cpp:106) */
int ttsw_solver_set_dt(ttsw_solver* s, double dt);
double ttsw_solver_time(const ttsw_solver* s);
/* Policy-mode tolerances (replaces swe.hpp:134-183 + harness.cpp:108-116): before every
   step the schedule is recomputed from the state, eps_var[c] = min(clip, C_eps V^(1/2)
   dx^(p-1/2) / ||q_c||_F) (clip if the component vanishes), eps_global from the largest
   norm (clip only if all vanish). Replaces the fixed tol of the descriptor. */
int ttsw_solver_set_eps_policy(ttsw_solver* s, double c_eps, int order, double volume, double clip);
/* the schedule used by the last step: eps_var[0..2], eps_global */
void ttsw_solver_eps(const ttsw_solver* s, double* out4);

/* --- full-tensor path: DenseRep (swe.hpp:45-80) through rhs<Rep>/ssprk3<Rep> -------
 * The reference's second representation plugin on the device: three N x N column-major
 * cell-average fields resident in HBM, dense reconstruction (reconstruction.hpp:253-423,
 * step1/step2 on stencil blocks), pointwise fluxes, LLF with the scalar dissipation speed
 * max(|m/h| + sqrt(g h)) (swe.hpp:329-339), SSP-RK3. desc->tol and desc->cross are ignored
 * (DenseRep ignores tolerances). Ghosts are periodic unless ttsw_dense_set_hooks makes an
 * axis DirichletExact; then `strips` fills the exact ghost averages of component c at time t
 * in the ttsw_ghosted layouts (strip_x 6 x (n+6), strip_y (n+6) x 6), and `source` (may be
 * NULL) the cell-average extra source, 3 x n x n column-major, component-major. */
typedef int (*ttsw_dense_strip_fn)(void* user, double t, int component, double* strip_x, double* strip_y);
typedef int (*ttsw_dense_source_fn)(void* user, double t, double* source3);
int ttsw_dense_create(ttsw_ctx* ctx, const ttsw_solver_desc* desc, ttsw_dense** out);
void ttsw_dense_destroy(ttsw_dense* s);
int ttsw_dense_set_state(ttsw_dense* s, int component, const double* host_colmajor);
int ttsw_dense_get_state(ttsw_dense* s, int component, double* host_colmajor);
/* the device field (n x n, column-major) of a component, for callers that keep data in HBM */
double* ttsw_dense_device_state(ttsw_dense* s, int component);
int ttsw_dense_set_dt(ttsw_dense* s, double dt);
int ttsw_dense_set_time(ttsw_dense* s, double t);
double ttsw_dense_time(const ttsw_dense* s);
int ttsw_dense_set_hooks(ttsw_dense* s, int bc_x, int bc_y, ttsw_dense_strip_fn strips, ttsw_dense_source_fn source,
                         void* user);
int ttsw_dense_step(ttsw_dense* s, long nsteps);
/* rhs<DenseRep> of the current state at the current time (3 x n x n host, component-major) */
int ttsw_dense_rhs(ttsw_dense* s, double* out3_host);

/* --- ensembles of independent trajectories (BASELINE config 5) -------
 * `members` independent solvers (one descriptor each, e.g. per-member seeded ICs) on one
 * device, advanced by `threads` host worker threads inside the library; every worker owns
 * its own context (stream + pool) and steps its members in turn, so the members' kernels
 * overlap on the GPU (at most 32 workers). Members never exchange data. Errors carry the
 * member index. */
int ttsw_ensemble_create(int device, int members, const ttsw_solver_desc* descs, int threads, ttsw_ensemble** out);
void ttsw_ensemble_destroy(ttsw_ensemble* e);
/* state component c of a member from host cores; round_eps >= 0 rounds it (the IC compression) */
int ttsw_ensemble_set_state_host(ttsw_ensemble* e, int member, int component, long m, long n, long r,
                                 const double* cx_colmajor, const double* cy_colmajor, double round_eps);
/* every member advances nsteps SSP-RK3 steps; returns after the device work finished */
int ttsw_ensemble_step(ttsw_ensemble* e, long nsteps);
/* 10 doubles per member: member, steps, mean h, ranks[3], max ranks[3], host ms of its worker */
int ttsw_ensemble_records(ttsw_ensemble* e, double* out);
int ttsw_ensemble_last_error(ttsw_ensemble* e, char* buf, long len);

#ifdef __cplusplus
}
#endif
#endif
