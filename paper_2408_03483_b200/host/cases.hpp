// The paper's four verification cases on the host side of the B200 build.
//
// Restates the behaviour of /root/reference/proj/include/ttsw/cases.hpp:13-191 and
// /root/reference/proj/src/cases.cpp:11-296: the case table (scales, dimensional
// parameters, boundary kinds, published dt ratios and C_eps per scheme, wave modes),
// the closed-form exact solutions, the manufactured source, and tensor-Gauss cell
// averages. Host evaluation only: the device consumes the results as initial fields
// (ttsw_tt_from_full / ttsw_dense_set_state), Dirichlet ghost strips (ttsw_ghosted /
// the dense strip callback) and the manufactured source (RhsHooks::extra_source).
#pragma once

#include <array>
#include <stdexcept>
#include <optional>
#include <string>
#include <string_view>
#include <vector>

namespace ttswe {

enum class CaseId { Kelvin, InertiaGravity, BarotropicTide, Manufactured };
enum class Boundary { Periodic, DirichletExact };
enum class Model { Linear = 0, Nonlinear = 1 };
enum class Scheme { Upwind3 = 0, Upwind5 = 1, Weno5 = 2 };

inline int scheme_order(Scheme s) { return s == Scheme::Upwind3 ? 3 : 5; }          // reconstruction.hpp:18
inline int quadrature_points(Scheme s) { return s == Scheme::Upwind3 ? 2 : 3; }     // reconstruction.hpp:20

struct InputError : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};

/// g, f, H (dimensional before scaling, nondimensional after): swe.hpp:19-26.
struct Phys {
  double g = 10.0, f = 1e-4, H = 1000.0;
  double wave_speed() const;    // sqrt(g H)
  double rossby_radius() const;  // sqrt(g H) / f
};

/// Characteristic scales (SI) and the scaling they induce (cases.hpp:17-57).
struct Scales {
  double length = 1.0, velocity = 1.0, height = 1.0;
  double time() const { return length / velocity; }
  Phys nondimensional(const Phys& dim) const;  // Nondimensionalizer::params
  double height_nd(double h) const;
  double velocity_nd(double u) const;
};

struct Mode {
  double amp = 0, kx = 0, ky = 0, omega = 0;
};

struct CaseSpec {
  CaseId id = CaseId::Kelvin;
  std::string name;
  Model model = Model::Linear;
  Scales scales;
  Phys dimensional, params;
  double domain_length_m = 1.0;
  double final_time_s = 0.0;
  Boundary bc_x = Boundary::Periodic, bc_y = Boundary::Periodic;
  std::array<double, 3> dt_ratio{}, c_eps{};  // indexed by Scheme
  std::vector<Mode> modes;
  double u_amp = 0.0;
  bool mms_source = false;

  double length() const { return domain_length_m / scales.length; }
  double final_time() const { return final_time_s / scales.time(); }
};

CaseSpec case_spec(CaseId id);
const std::vector<std::pair<std::string, CaseId>>& case_registry();
std::optional<CaseId> parse_case_id(std::string_view name);

/// Uniform grid on [x0, x0 + lx) x [y0, y0 + ly) (swe.hpp:28-38).
struct Grid {
  long nx = 0, ny = 0;
  double x0 = 0, y0 = 0, lx = 1, ly = 1;
  double dx() const { return lx / double(nx); }
  double dy() const { return ly / double(ny); }
};

/// (eta, u, v) at (x, y, t), nondimensional (cases.cpp:143-196).
std::array<double, 3> exact_primitive(const CaseSpec& s, double x, double y, double t);
/// (eta, u, v) for the linear model, (h, hu, hv) for the nonlinear one.
std::array<double, 3> exact_conserved(const CaseSpec& s, double x, double y, double t);
/// Manufactured forcing of the nonlinear system (cases.cpp:198-220); zero when inactive.
std::array<double, 3> mms_source(const CaseSpec& s, double x, double y, double t);

/// n_q-point Gauss rule on [-1/2, 1/2] (reconstruction.hpp:33-49).
void gauss_rule(int nq, double* offset, double* weight);

/// Exact cell average of conserved component c over cell (i, j) — i, j may lie in the
/// ghost layer (negative or >= n) — at time t, by the n_q x n_q tensor Gauss rule.
double exact_cell_average(const CaseSpec& s, const Grid& g, double t, int nq, int c, long i, long j);
/// All nx x ny exact cell averages of component c, column-major.
std::vector<double> exact_cell_averages(const CaseSpec& s, const Grid& g, double t, int nq, int c);
/// Cell averages of the manufactured source, 3 x (nx ny), component-major, column-major.
std::vector<double> mms_source_averages(const CaseSpec& s, const Grid& g, double t, int nq);
/// Exact ghost strips of component c in the ttsw_ghosted layouts: strip_x 6 x (ny+6) (ghost
/// rows 0-2 and nx+3..nx+5, every ghosted column), strip_y (nx+6) x 6, column-major.
void exact_strips(const CaseSpec& s, const Grid& g, double t, int nq, int c, double* strip_x, double* strip_y);

}  // namespace ttswe
