/* TEST INFRASTRUCTURE ONLY — C ABI of the CPU oracle (restated reference path).
 * Loaded by tests/ (ctypes), __graft_entry__.smoke() and bench.py's CPU legs only.
 * The numeric enums intentionally equal those of include/ttsw_capi.h so that
 * parity tests can drive both libraries with the same arguments. */
#ifndef TTSW_ORACLE_H
#define TTSW_ORACLE_H

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ttor_tt ttor_tt;
typedef struct ttor_solver ttor_solver;
typedef struct ttor_rng ttor_rng;

enum { TTOR_OK = 0, TTOR_INPUT = 1, TTOR_SHAPE = 2, TTOR_STATE = 3, TTOR_DEGENERACY = 4,
       TTOR_CONVERGENCE = 5, TTOR_EVALUATION = 6, TTOR_INTERNAL = 8, TTOR_DEADLINE = 9 };

typedef struct {
  double eps;
  long max_rank;
  int max_sweeps;
  long rank_increment;
  int validation_sample;
  unsigned long long seed;
} ttor_cross_cfg;

typedef struct {
  long evaluations;
  int sweeps;
  double residual;
} ttor_cross_stats;

typedef struct {
  int model;   /* 0 linear, 1 nonlinear */
  int scheme;  /* 0 upwind3, 1 upwind5, 2 weno5 */
  long n;      /* nx = ny = n, unit square */
  double g, f, H;
  double dt;
  double tol;  /* EpsSchedule{var = tol x3, global = tol} */
  double lambda_eps_floor;
  ttor_cross_cfg cross;
} ttor_solver_desc;

int ttor_last_error(char* buf, long len, double* residual, int* iterations, long* row, long* col);

ttor_tt* ttor_tt_new(long m, long n, long r, const double* cx_colmajor, const double* cy_colmajor);
void ttor_tt_free(ttor_tt* x);
void ttor_tt_dims(const ttor_tt* x, long* m, long* n, long* r);
void ttor_tt_get(const ttor_tt* x, double* cx_colmajor, double* cy_colmajor);

int ttor_from_full(long m, long n, const double* a_colmajor, double eps, ttor_tt** out);
int ttor_to_full(const ttor_tt* x, double* out_colmajor);
int ttor_round(const ttor_tt* x, double eps, ttor_tt** out, long* k_out, double* margin, double* kappa);
int ttor_add(const ttor_tt* x, const ttor_tt* y, ttor_tt** out);
int ttor_scale(const ttor_tt* x, double a, ttor_tt** out);
int ttor_axpy(double a, const ttor_tt* x, double b, const ttor_tt* y, double eps, ttor_tt** out);
int ttor_hadamard(const ttor_tt* x, const ttor_tt* y, ttor_tt** out);
int ttor_norm_fro(const ttor_tt* x, double* out);
int ttor_sum_entries(const ttor_tt* x, double* out);
/* op: 0 periodic pad, 1 step1, 2 quadrature point, 3 quadrature sum, 4 difference,
 *     5 row slice (a0=offset, a1=rows), 6 quadrature slice (a0=s) ; n = interior size */
int ttor_core_map(const ttor_tt* x, int axis, int op, int scheme, int side, long n, long a0, long a1,
                  ttor_tt** out);
int ttor_core_map_dense(const ttor_tt* x, int axis, long rows, long cols, const double* m_colmajor,
                        ttor_tt** out);
int ttor_recip(const ttor_tt* x, double eps, int max_iterations, int* iterations, ttor_tt** out);
int ttor_cross(int fn, const double* params, const ttor_tt* const* ops, int nops, const ttor_tt* guess,
               const ttor_cross_cfg* cfg, ttor_tt** out, ttor_cross_stats* stats);
int ttor_maxvol(long n, long r, const double* m_colmajor, long* rows_out);
int ttor_svd_values(long m, long n, const double* a_colmajor, double* s_out);
int ttor_truncation_rank(const double* sv, long n, double eps, long* keep, double* margin);
/* table dump: step1_c(9) step1_ideal(3) step1_row(5) c[3](27) gamma[3](9) point_row[3](15)
 *             gamma_plus(3) gamma_minus(3) weno_d(3) quad offset(3) weight(3) radius nq */
int ttor_tables(int scheme, double* out);
int ttor_weno_step1(const double* v5, double eps, double* out);
int ttor_weno_step2(const double* v5, int m, double eps, double* out);
int ttor_smoothness(const double* v5, double* beta3);
int ttor_weno_weights(const double* beta3, const double* ideal3, double eps, double* out3);

int ttor_periodic_ghost(const ttor_tt* x, ttor_tt** out);
/* tt_ghosted (cases.cpp:298-344); bc 0 = Periodic, 1 = DirichletExact with caller strips */
int ttor_ghosted(const ttor_tt* x, int bc_x, int bc_y, const double* strip_x, const double* strip_y, double eps_tt,
                 ttor_tt** out);
int ttor_reconstruct_faces(const ttor_tt* ghosted, int axis, int scheme, double eps_tt,
                           const ttor_cross_cfg* cfg, double dx, double dy, ttor_tt** minus, ttor_tt** plus);
int ttor_physical_flux(ttor_tt* const* u3, int axis, int model, double g, double f, double H, double eps,
                       ttor_tt** out3);

ttor_solver* ttor_solver_new(const ttor_solver_desc* desc);
void ttor_solver_free(ttor_solver* s);
int ttor_solver_set_state(ttor_solver* s, int c, const ttor_tt* x);
ttor_tt* ttor_solver_get_state(ttor_solver* s, int c);
int ttor_solver_rhs(ttor_solver* s, ttor_tt** out3);
/* RhsHooks (swe.hpp:276-282): q3 are borrowed for the call; the three returned fields
 * become the solver's (a hook returns 0 on success). Stage times per swe.hpp:441-448. */
typedef int (*ttor_fill_ghost_fn)(void* user, const ttor_tt* const* q3, double t, ttor_tt** ghosted3);
typedef int (*ttor_extra_source_fn)(void* user, double t, ttor_tt** extra3);
int ttor_solver_set_hooks(ttor_solver* s, ttor_fill_ghost_fn ghost, ttor_extra_source_fn source, void* user);
int ttor_solver_set_time(ttor_solver* s, double t);
double ttor_solver_time(const ttor_solver* s);
int ttor_solver_step(ttor_solver* s, long nsteps);
/* bench only: stop the calling thread's next rounding after `seconds` of wall time (<= 0 clears);
   the step then returns TTOR_DEADLINE with the completed roundings in the trace */
void ttor_set_sample_deadline(double seconds);
/* policy-mode tolerances (swe.hpp:134-183): schedule recomputed from the state each step */
int ttor_solver_set_eps_policy(ttor_solver* s, double c_eps, int order, double volume, double clip);
int ttor_solver_eps(const ttor_solver* s, double* out4);
long ttor_solver_trace_len(const ttor_solver* s);
/* per record: op, m, n, r_in, k_out, crosses-before (6 longs), margin and kappa = ||cx|| ||cy|| / ||X|| */
void ttor_solver_trace(const ttor_solver* s, long* ints, double* margins, double* kappas);
void ttor_solver_trace_clear(ttor_solver* s);
/* per cross call: rank, sweeps, pivot hash (3 longs) and residual */
long ttor_solver_cross_trace_len(const ttor_solver* s);
void ttor_solver_cross_trace(ttor_solver* s, long* ints, double* residuals, int clear);

ttor_rng* ttor_rng_new(unsigned long long seed);
void ttor_rng_free(ttor_rng* g);
/* std::normal_distribution<double>(0,1) draws, column-major fill order of random_matrix */
void ttor_rng_normal(ttor_rng* g, long count, double* out);
void ttor_rng_uniform_int(ttor_rng* g, long lo, long hi, long count, long* out);
void ttor_rng_uniform_real(ttor_rng* g, double lo, double hi, long count, double* out);
unsigned long long ttor_rng_raw(ttor_rng* g);

#ifdef __cplusplus
}
#endif
#endif
