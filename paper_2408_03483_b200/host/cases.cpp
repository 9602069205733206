// Verification cases of the paper (see cases.hpp): table, exact solutions, manufactured
// source, tensor-Gauss cell averages. Reference behaviour: proj/src/cases.cpp:11-296.
#include "cases.hpp"

#include <cmath>

namespace ttswe {

namespace {

constexpr double kPi = 3.14159265358979323846;

// One table row per case (cases.cpp:11-89): SI scales and parameters, domain, final time,
// boundaries, published dt ratios / C_eps per scheme (Upwind3, Upwind5, WENO5), wave
// content. finalize() turns the modes into nondimensional amplitudes and frequencies.
struct Row {
  CaseId id;
  const char* name;
  Model model;
  Scales scales;
  Phys dim;
  double length_m, final_s;
  Boundary bx, by;
  std::array<double, 3> dt_ratio, c_eps;
  std::vector<Mode> modes;  // amp (SI height, or the H-relative Kelvin amplitude), kx, ky
  double u_amp_si;
  bool mms;
};

const std::vector<Row>& table() {
  static const std::vector<Row> rows = {
      {CaseId::Kelvin, "kelvin", Model::Linear, {5e6, 5e-3, 0.1}, {10.0, 1e-4, 1000.0}, 5e6, 3.0 * 3600.0,
       Boundary::DirichletExact, Boundary::Periodic, {5e-5, 2.5e-4, 2.5e-4}, {1.0, 1.0, 1000.0},
       {{1e-4, 0.0, 2.0 * kPi, 0.0}, {2e-4, 0.0, 4.0 * kPi, 0.0}}, 0.0, false},
      {CaseId::InertiaGravity, "inertia-gravity", Model::Linear, {1e7, 1.622e-3, 0.2}, {10.0, 1e-4, 1000.0}, 1e7,
       3.0 * 3600.0, Boundary::Periodic, Boundary::Periodic, {1e-4, 1e-3, 1e-3}, {1.0, 1.0, 500.0},
       {{0.1, 2.0 * kPi, 2.0 * kPi, 0.0}, {0.2, 4.0 * kPi, 4.0 * kPi, 0.0}}, 0.0, false},
      {CaseId::BarotropicTide, "barotropic-tide", Model::Linear, {25e4, 3.163e-3, 0.2}, {10.0, 1e-4, 200.0}, 25e4,
       30.0 * 60.0, Boundary::DirichletExact, Boundary::Periodic, {2.5e-4, 5e-4, 5e-4}, {1.0, 1.0, 1.0},
       {{0.2, 2.5 * kPi, 0.0, 0.0}, {0.4, 4.5 * kPi, 0.0, 0.0}}, 0.0, false},
      {CaseId::Manufactured, "manufactured", Model::Nonlinear, {1e7, 1e-2, 500.0}, {10.0, 1e-4, 1000.0}, 1e7,
       3.0 * 3600.0, Boundary::Periodic, Boundary::Periodic, {5e-5, 5e-3, 5e-3}, {1e-4, 1.0, 1.0},
       {{1e-2, 2.0 * kPi, 2.0 * kPi, 0.0}}, 1e-2, true},
  };
  return rows;
}

}  // namespace

double Phys::wave_speed() const { return std::sqrt(g * H); }
double Phys::rossby_radius() const { return wave_speed() / f; }

Phys Scales::nondimensional(const Phys& d) const {
  if (!(length > 0) || !(velocity > 0) || !(height > 0)) throw InputError("Nondimensionalizer: scale must be positive");
  // gravity scales with U^2 / H*, frequency with U / L, depth with H*
  return {d.g / (velocity * velocity / height), d.f / (velocity / length), d.H / height};
}
double Scales::height_nd(double h) const { return h / height; }
double Scales::velocity_nd(double u) const { return u / velocity; }

CaseSpec case_spec(CaseId id) {
  for (const Row& r : table()) {
    if (r.id != id) continue;
    CaseSpec s;
    s.id = r.id;
    s.name = r.name;
    s.model = r.model;
    s.scales = r.scales;
    s.dimensional = r.dim;
    s.params = r.scales.nondimensional(r.dim);
    s.domain_length_m = r.length_m;
    s.final_time_s = r.final_s;
    s.bc_x = r.bx;
    s.bc_y = r.by;
    s.dt_ratio = r.dt_ratio;
    s.c_eps = r.c_eps;
    s.modes = r.modes;
    s.u_amp = r.u_amp_si;
    s.mms_source = r.mms;
    const double c = s.params.wave_speed(), f = s.params.f;
    switch (id) {
      case CaseId::Kelvin:  // nondispersive: the amplitudes stay relative to H, c enters directly
        break;
      case CaseId::InertiaGravity:
        for (Mode& m : s.modes) {
          m.amp = s.scales.height_nd(m.amp);
          m.omega = std::sqrt(c * c * (m.kx * m.kx + m.ky * m.ky) + f * f);
        }
        break;
      case CaseId::BarotropicTide:
        for (Mode& m : s.modes) {
          m.amp = s.scales.height_nd(m.amp);
          m.omega = std::sqrt(s.params.g * s.params.H * m.kx * m.kx + f * f);
        }
        break;
      case CaseId::Manufactured:
        for (Mode& m : s.modes) {
          m.amp = s.scales.height_nd(m.amp);
          m.omega = std::sqrt(c * c * (m.kx * m.kx + m.ky * m.ky));
        }
        s.u_amp = s.scales.velocity_nd(s.u_amp);
        break;
    }
    return s;
  }
  throw InputError("case_spec: unknown case");
}

const std::vector<std::pair<std::string, CaseId>>& case_registry() {
  static const std::vector<std::pair<std::string, CaseId>> reg = [] {
    std::vector<std::pair<std::string, CaseId>> v;
    for (const Row& r : table()) v.emplace_back(r.name, r.id);
    return v;
  }();
  return reg;
}

std::optional<CaseId> parse_case_id(std::string_view name) {
  for (const auto& [key, id] : case_registry())
    if (key == name) return id;
  return std::nullopt;
}

std::array<double, 3> exact_primitive(const CaseSpec& s, double x, double y, double t) {
  const Phys& p = s.params;
  const double c = p.wave_speed();
  double eta = 0, u = 0, v = 0;
  switch (s.id) {
    case CaseId::Kelvin: {
      // coast at x = 0, propagation towards -y, offshore decay over the Rossby radius
      const double decay = std::exp(-x / p.rossby_radius());
      double wave = 0;
      for (const Mode& m : s.modes) wave += m.amp * std::sin(m.ky * (y + c * t));
      eta = -p.H * wave * decay;
      v = c * wave * decay;
      break;
    }
    case CaseId::InertiaGravity:
      for (const Mode& m : s.modes) {
        const double ph = m.kx * x + m.ky * y - m.omega * t;
        const double cs = std::cos(ph), sn = std::sin(ph);
        const double a = p.g * m.amp / (m.omega * m.omega - p.f * p.f);
        eta += m.amp * cs;
        u += a * (m.omega * m.kx * cs - p.f * m.ky * sn);
        v += a * (m.omega * m.ky * cs + p.f * m.kx * sn);
      }
      break;
    case CaseId::BarotropicTide:
      for (const Mode& m : s.modes) {
        const double a = p.g * m.amp * m.kx / (m.omega * m.omega - p.f * p.f);
        eta += m.amp * std::cos(m.kx * x) * std::cos(m.omega * t);
        u += a * m.omega * std::sin(m.kx * x) * std::sin(m.omega * t);
        v += a * p.f * std::sin(m.kx * x) * std::cos(m.omega * t);
      }
      break;
    case CaseId::Manufactured: {
      const Mode& m = s.modes[0];
      const double ph = m.kx * x + m.ky * y - m.omega * t;
      eta = m.amp * std::sin(ph);
      u = s.u_amp * std::cos(ph);
      break;
    }
  }
  return {eta, u, v};
}

std::array<double, 3> exact_conserved(const CaseSpec& s, double x, double y, double t) {
  const auto w = exact_primitive(s, x, y, t);
  if (s.model == Model::Linear) return w;
  const double h = s.params.H + w[0];
  return {h, h * w[1], h * w[2]};
}

std::array<double, 3> mms_source(const CaseSpec& s, double x, double y, double t) {
  if (!s.mms_source) return {0.0, 0.0, 0.0};
  // residual of the nonlinear equations on h = H + A sin(ph), u = B cos(ph), v = 0
  const Phys& p = s.params;
  const Mode& m = s.modes[0];
  const double A = m.amp, B = s.u_amp;
  const double ph = m.kx * x + m.ky * y - m.omega * t;
  const double cs = std::cos(ph), sn = std::sin(ph);
  const double h = p.H + A * sn;
  const double mass = -m.omega * A * cs + m.kx * B * (A * cs * cs - h * sn);
  const double xmom = B * m.omega * (-A * cs * cs + h * sn) + m.kx * B * B * (A * cs * cs * cs - 2.0 * h * cs * sn) +
                      p.g * h * A * m.kx * cs;
  const double ymom = p.g * h * A * m.ky * cs + p.f * h * B * cs;
  return {mass, xmom, ymom};
}

void gauss_rule(int nq, double* offset, double* weight) {
  if (nq == 2) {
    const double a = 1.0 / (2.0 * std::sqrt(3.0));
    offset[0] = -a;
    offset[1] = a;
    weight[0] = weight[1] = 0.5;
  } else if (nq == 3) {
    const double b = std::sqrt(3.0 / 5.0) / 2.0;
    offset[0] = -b;
    offset[1] = 0.0;
    offset[2] = b;
    weight[0] = weight[2] = 5.0 / 18.0;
    weight[1] = 8.0 / 18.0;
  } else {
    throw InputError("gauss_rule: only 2- and 3-point rules are supported");
  }
}

namespace {

template <class F>
double cell_average(const Grid& g, int nq, long i, long j, F&& f) {
  double off[3], w[3];
  gauss_rule(nq, off, w);
  const double xc = g.x0 + (double(i) + 0.5) * g.dx(), yc = g.y0 + (double(j) + 0.5) * g.dy();
  double acc = 0.0;
  for (int a = 0; a < nq; ++a)
    for (int b = 0; b < nq; ++b) acc += w[a] * w[b] * f(xc + off[a] * g.dx(), yc + off[b] * g.dy());
  return acc;
}

}  // namespace

double exact_cell_average(const CaseSpec& s, const Grid& g, double t, int nq, int c, long i, long j) {
  return cell_average(g, nq, i, j, [&](double x, double y) { return exact_conserved(s, x, y, t)[size_t(c)]; });
}

std::vector<double> exact_cell_averages(const CaseSpec& s, const Grid& g, double t, int nq, int c) {
  std::vector<double> out(size_t(g.nx * g.ny));
  for (long j = 0; j < g.ny; ++j)
    for (long i = 0; i < g.nx; ++i) out[size_t(i + g.nx * j)] = exact_cell_average(s, g, t, nq, c, i, j);
  return out;
}

std::vector<double> mms_source_averages(const CaseSpec& s, const Grid& g, double t, int nq) {
  const size_t nn = size_t(g.nx * g.ny);
  std::vector<double> out(3 * nn);
  for (long j = 0; j < g.ny; ++j)
    for (long i = 0; i < g.nx; ++i)
      for (int c = 0; c < 3; ++c)
        out[size_t(c) * nn + size_t(i + g.nx * j)] =
            cell_average(g, nq, i, j, [&](double x, double y) { return mms_source(s, x, y, t)[size_t(c)]; });
  return out;
}

void exact_strips(const CaseSpec& s, const Grid& g, double t, int nq, int c, double* strip_x, double* strip_y) {
  const long gx = g.nx + 6, gy = g.ny + 6;
  for (int k = 0; k < 6; ++k) {
    const long row = k < 3 ? k : g.nx + 3 + (k - 3);  // ghosted row index
    for (long j = 0; j < gy; ++j) strip_x[k + 6 * j] = exact_cell_average(s, g, t, nq, c, row - 3, j - 3);
    const long col = k < 3 ? k : g.ny + 3 + (k - 3);
    for (long i = 0; i < gx; ++i) strip_y[i + gx * k] = exact_cell_average(s, g, t, nq, c, i - 3, col - 3);
  }
}

}  // namespace ttswe
