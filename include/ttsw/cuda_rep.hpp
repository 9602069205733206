// cuda_rep.hpp — C++ drop-in for the reference's TT representation plugin.
//
// `ttsw_cuda::CudaTTRep` provides the static interface of `TTRep`
// (/root/reference/proj/include/ttsw/swe.hpp:84-119) over the C ABI in ttsw_capi.h, so
// the reference's templated consumers `rhs<Rep>` (swe.hpp:362-423) and `ssprk3<Rep>`
// (swe.hpp:428-454) can be instantiated with device-resident fields. Header-only; links
// against paper_2408_03483_b200/libttsw_cuda.so. Matrix arguments are any column-major
// dense type with rows()/cols()/operator()(i,j) (Eigen::MatrixXd in the reference).
//
// Differences a maintainer must wire:
//  * elementwise(): the reference passes a host std::function (cross.hpp:64-65); on the
//    device the functor is one of the fixed kinds (ttsw_capi.h TTSW_FN_*), selected by
//    the two call sites face_wave_speed (swe.hpp:341-352) and tt_recon_weno
//    (reconstruction.hpp:546-556). There is no host fallback.
//  * the two `if constexpr (Rep::is_tt)` free functions get overloads below:
//    reconstruct_faces (reconstruction.hpp:611-616) and tt_ghosted (cases.cpp:298-344; periodic
//    and DirichletExact with caller-evaluated strips).
#pragma once

#include <array>
#include <cstddef>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../ttsw_capi.h"

namespace ttsw_cuda {

using Index = long;
enum class Axis { X = 0, Y = 1 };

/// Error thrown for every non-OK status (message from ttsw_last_error).
struct Error : std::runtime_error {
  int code;
  ttsw_err_info info;
  Error(int c, const std::string& m, ttsw_err_info i) : std::runtime_error(m), code(c), info(i) {}
};

/// Process-wide default context (one device, one stream), like the reference's
/// implicit single-threaded execution.
class Context {
 public:
  explicit Context(int device = 0) {
    ttsw_ctx* c = nullptr;
    const int st = ttsw_ctx_create(device, &c);
    ctx_.reset(c, ttsw_ctx_destroy);
    check(st);
  }
  ttsw_ctx* get() const { return ctx_.get(); }
  void check(int st) const {
    if (st == TTSW_OK) return;
    char buf[1024];
    ttsw_err_info info{};
    ttsw_last_error(ctx_.get(), buf, sizeof(buf), &info);
    throw Error(st, buf, info);
  }
  /// The process-wide context lives on this device (set before its first use).
  static int& default_device() {
    static int d = 0;
    return d;
  }
  static void select_device(int device) { default_device() = device; }
  static Context& instance() {
    static Context c(default_device());
    return c;
  }

 private:
  std::shared_ptr<ttsw_ctx> ctx_;
};

/// Immutable device TT handle: the `Field` of CudaTTRep (TTMatrix<double>, tt.hpp:19-53).
class Field {
 public:
  Field() = default;
  explicit Field(ttsw_tt* h) : h_(h, ttsw_tt_free) {}
  const ttsw_tt* get() const { return h_.get(); }
  Index rows() const { return dims()[0]; }
  Index cols() const { return dims()[1]; }
  Index rank() const { return dims()[2]; }

 private:
  std::vector<long> dims() const {
    std::vector<long> d(3);
    ttsw_tt_dims(h_.get(), &d[0], &d[1], &d[2]);
    return d;
  }
  std::shared_ptr<ttsw_tt> h_;
};

struct CudaTTRep {
  using Field = ttsw_cuda::Field;
  static constexpr bool is_tt = true;

  static Context& ctx() { return Context::instance(); }
  template <class F>
  static Field make(F&& f) {
    ttsw_tt* out = nullptr;
    ctx().check(f(&out));
    return Field(out);
  }

  static Index rows(const Field& x) { return x.rows(); }
  static Index cols(const Field& x) { return x.cols(); }
  static Index rank(const Field& x) { return x.rank(); }
  static double norm(const Field& x) {
    double v = 0;
    ctx().check(ttsw_norm_fro(ctx().get(), x.get(), &v));
    return v;
  }
  /// Dense copy to the host (diagnostics only, like TTRep::dense).
  template <class M>
  static M dense(const Field& x) {
    const Index m = x.rows(), n = x.cols(), r = x.rank();
    std::vector<double> cx(size_t(m * r)), cy(size_t(r * n));
    ctx().check(ttsw_tt_to_host(ctx().get(), x.get(), cx.data(), cy.data()));
    M out(m, n);
    for (Index j = 0; j < n; ++j)
      for (Index i = 0; i < m; ++i) {
        double s = 0;
        for (Index a = 0; a < r; ++a) s += cx[size_t(i + a * m)] * cy[size_t(a + j * r)];
        out(i, j) = s;
      }
    return out;
  }
  /// From host cores (core_x m x r, core_y r x n, column-major) — the IC upload.
  static Field from_cores(Index m, Index n, Index r, const double* cx, const double* cy) {
    return make([&](ttsw_tt** o) { return ttsw_tt_from_host(ctx().get(), m, n, r, cx, cy, o); });
  }
  /// TTRep::compress (swe.hpp:93-95): any matrix type with rows()/cols()/data() in
  /// column-major order (Eigen::MatrixXd); eps < 0 compresses at eps = 0 as the reference.
  template <class M>
  static Field compress(const M& a, double eps) {
    return make([&](ttsw_tt** o) {
      return ttsw_tt_from_full(ctx().get(), a.rows(), a.cols(), a.data(), eps < 0 ? 0.0 : eps, o, nullptr);
    });
  }
  static Field round_to(const Field& x, double eps) {
    if (eps < 0) return x;
    return make([&](ttsw_tt** o) { return ttsw_round(ctx().get(), x.get(), eps, o, nullptr); });
  }
  static Field zero_like(const Field& x) {
    return make([&](ttsw_tt** o) { return ttsw_tt_constant(ctx().get(), x.rows(), x.cols(), 0.0, o); });
  }
  static Field scaled(const Field& x, double a) {
    return make([&](ttsw_tt** o) { return ttsw_scale(ctx().get(), x.get(), a, o); });
  }
  static Field axpy(double a, const Field& x, double b, const Field& y, double eps) {
    return make([&](ttsw_tt** o) { return ttsw_axpy(ctx().get(), a, x.get(), b, y.get(), eps, o); });
  }
  static Field mul(const Field& x, const Field& y, double eps) {
    return make([&](ttsw_tt** o) { return ttsw_mul(ctx().get(), x.get(), y.get(), eps, o); });
  }
  /// TTRep::lin (swe.hpp:109-111): the reference's dense operator is passed by its nonzeros.
  template <class M>
  static Field lin(Axis axis, const M& m, const Field& x) {
    std::vector<long> rowptr(size_t(m.rows()) + 1, 0), colidx;
    std::vector<double> vals;
    for (Index i = 0; i < m.rows(); ++i) {
      for (Index j = 0; j < m.cols(); ++j)
        if (m(i, j) != 0.0) {
          colidx.push_back(j);
          vals.push_back(m(i, j));
        }
      rowptr[size_t(i) + 1] = long(colidx.size());
    }
    if (colidx.empty()) {
      colidx.push_back(0);
      vals.push_back(0.0);
    }
    return make([&](ttsw_tt** o) {
      return ttsw_core_map_csr(ctx().get(), x.get(), int(axis), m.rows(), m.cols(), rowptr.data(), colidx.data(),
                               vals.data(), o);
    });
  }
  /// Banded operator by kind (never materialised): TTSW_MAP_* of ttsw_capi.h.
  static Field lin_banded(Axis axis, int op, int scheme, int side, Index n, const Field& x, Index a0 = 0,
                          Index a1 = 0) {
    return make([&](ttsw_tt** o) {
      return ttsw_core_map(ctx().get(), x.get(), int(axis), op, scheme, side, n, a0, a1, o);
    });
  }
  static Field recip(const Field& x, double eps) {
    return make([&](ttsw_tt** o) { return ttsw_recip_taylor(ctx().get(), x.get(), eps, 200, nullptr, o); });
  }
  /// TTRep::elementwise with a device functor kind (TTSW_FN_*) instead of std::function.
  static Field elementwise(int fn, double param, const std::vector<Field>& ops, const Field& guess, double eps,
                           ttsw_cross_cfg base) {
    base.eps = eps;
    std::vector<const ttsw_tt*> raw;
    for (const auto& f : ops) raw.push_back(f.get());
    return make([&](ttsw_tt** o) {
      return ttsw_cross(ctx().get(), fn, &param, raw.data(), int(raw.size()), guess.get(), &base, o, nullptr);
    });
  }
};

/// Overload for reconstruct_faces(const TT&, Axis, const TTReconContext&) (reconstruction.hpp:611-616).
struct FacePair {
  Field minus, plus;
};
inline FacePair reconstruct_faces(const Field& ghosted, Axis axis, int scheme, double eps_tt,
                                  const ttsw_cross_cfg& cross, double dx, double dy) {
  ttsw_tt *mi = nullptr, *pl = nullptr;
  auto& c = CudaTTRep::ctx();
  c.check(ttsw_reconstruct_faces(c.get(), ghosted.get(), int(axis), scheme, eps_tt, &cross, dx, dy, &mi, &pl));
  return {Field(mi), Field(pl)};
}

/// Overload for detail::tt_ghosted, both axes periodic (cases.cpp:298-309).
inline Field tt_ghosted_periodic(const Field& interior) {
  return CudaTTRep::make(
      [&](ttsw_tt** o) { return ttsw_periodic_ghost(CudaTTRep::ctx().get(), interior.get(), o); });
}

/// detail::tt_ghosted (cases.cpp:298-344) with DirichletExact axes: bc 0 = Periodic,
/// 1 = DirichletExact; the strips are the exact ghost-cell averages the caller evaluates
/// (strip_x 6 x (ny+6), strip_y (nx+6) x 6, column-major; NULL for a periodic axis).
inline Field tt_ghosted(const Field& interior, int bc_x, int bc_y, const double* strip_x, const double* strip_y,
                        double eps_tt) {
  return CudaTTRep::make([&](ttsw_tt** o) {
    return ttsw_ghosted(CudaTTRep::ctx().get(), interior.get(), bc_x, bc_y, strip_x, strip_y, eps_tt, o);
  });
}

/// Step-level driver equivalent to looping ssprk3<Rep>(state, t, dt, rhs, eps) with a
/// fixed EpsSchedule (swe.hpp:156-159, :428-454).
class Solver {
 public:
  Solver(const ttsw_solver_desc& d) {
    ttsw_solver* s = nullptr;
    CudaTTRep::ctx().check(ttsw_solver_create(CudaTTRep::ctx().get(), &d, &s));
    s_.reset(s, ttsw_solver_destroy);
  }
  void set_state(int c, const Field& x) { CudaTTRep::ctx().check(ttsw_solver_set_state(s_.get(), c, x.get())); }
  Field state(int c) const {
    return CudaTTRep::make([&](ttsw_tt** o) { return ttsw_solver_get_state(s_.get(), c, o); });
  }
  void step(long n = 1) { CudaTTRep::ctx().check(ttsw_solver_step(s_.get(), n)); }
  /// step size of the following steps (run_impl clips the last step, harness.cpp:106)
  void set_dt(double dt) { CudaTTRep::ctx().check(ttsw_solver_set_dt(s_.get(), dt)); }
  void set_time(double t) { CudaTTRep::ctx().check(ttsw_solver_set_time(s_.get(), t)); }
  double time() const { return ttsw_solver_time(s_.get()); }
  /// the EpsSchedule of the current / last step: var[0..2], global
  std::array<double, 4> eps() const {
    std::array<double, 4> e{};
    ttsw_solver_eps(s_.get(), e.data());
    return e;
  }
  /// RhsHooks (swe.hpp:276-282) as C callbacks; the solver takes over returned handles.
  void set_hooks(ttsw_fill_ghost_fn ghost, ttsw_extra_source_fn source, void* user) {
    CudaTTRep::ctx().check(ttsw_solver_set_hooks(s_.get(), ghost, source, user));
  }
  ttsw_solver* get() const { return s_.get(); }
  /// EpsPolicy mode (swe.hpp:134-183): the schedule is recomputed from the state before
  /// every step, as run_impl does (harness.cpp:108-116).
  void set_eps_policy(double c_eps, int order = 3, double volume = 1.0, double clip = 1e-3) {
    CudaTTRep::ctx().check(ttsw_solver_set_eps_policy(s_.get(), c_eps, order, volume, clip));
  }

 private:
  std::shared_ptr<ttsw_solver> s_;
};

/// The reference's second representation, DenseRep (swe.hpp:45-80), stepped on the device:
/// three n x n column-major fields in HBM (ttsw_dense_*).
class DenseSolver {
 public:
  explicit DenseSolver(const ttsw_solver_desc& d) {
    ttsw_dense* s = nullptr;
    CudaTTRep::ctx().check(ttsw_dense_create(CudaTTRep::ctx().get(), &d, &s));
    s_.reset(s, ttsw_dense_destroy);
  }
  void set_state(int c, const double* host_colmajor) {
    CudaTTRep::ctx().check(ttsw_dense_set_state(s_.get(), c, host_colmajor));
  }
  void state(int c, double* host_colmajor) const {
    CudaTTRep::ctx().check(ttsw_dense_get_state(s_.get(), c, host_colmajor));
  }
  void step(long n = 1) { CudaTTRep::ctx().check(ttsw_dense_step(s_.get(), n)); }
  void set_dt(double dt) { CudaTTRep::ctx().check(ttsw_dense_set_dt(s_.get(), dt)); }
  void set_time(double t) { CudaTTRep::ctx().check(ttsw_dense_set_time(s_.get(), t)); }
  double time() const { return ttsw_dense_time(s_.get()); }
  void set_hooks(int bc_x, int bc_y, ttsw_dense_strip_fn strips, ttsw_dense_source_fn source, void* user) {
    CudaTTRep::ctx().check(ttsw_dense_set_hooks(s_.get(), bc_x, bc_y, strips, source, user));
  }

 private:
  std::shared_ptr<ttsw_dense> s_;
};

}  // namespace ttsw_cuda
