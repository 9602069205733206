// ttswe run driver on the device (see harness.hpp). Reference behaviour:
// proj/src/harness.cpp:15-358 (run_impl, convergence, CSV/JSON writers, run_cli).
#include "harness.hpp"

#include <algorithm>
#include <charconv>
#include <chrono>
#include <cmath>
#include <cstring>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>

#include "ttsw/cuda_rep.hpp"

namespace ttswe {

using ttsw_cuda::CudaTTRep;

std::string scheme_name(Scheme s) {
  switch (s) {
    case Scheme::Upwind3: return "upwind3";
    case Scheme::Upwind5: return "upwind5";
    default: return "weno5";
  }
}

std::optional<Scheme> parse_scheme(std::string_view name) {
  if (name == "upwind3") return Scheme::Upwind3;
  if (name == "upwind5") return Scheme::Upwind5;
  if (name == "weno5") return Scheme::Weno5;
  return std::nullopt;
}

std::optional<Representation> parse_representation(std::string_view name) {
  if (name == "tt" || name == "cuda") return Representation::TT;
  if (name == "dense" || name == "cuda-dense") return Representation::Dense;
  return std::nullopt;
}

namespace {

/// Host matrix with the rows()/cols()/data()/operator() surface CudaTTRep expects.
struct HostMat {
  long r = 0, c = 0;
  std::vector<double> a;
  HostMat(long r_, long c_) : r(r_), c(c_), a(size_t(r_ * c_)) {}
  long rows() const { return r; }
  long cols() const { return c; }
  const double* data() const { return a.data(); }
  double operator()(long i, long j) const { return a[size_t(i + r * j)]; }
  double& operator()(long i, long j) { return a[size_t(i + r * j)]; }
};

double nominal_dt(const CaseSpec& spec, const RunConfig& cfg, double dx) {
  const double ratio = cfg.dt_ratio.value_or(spec.dt_ratio[size_t(cfg.scheme)]);
  if (!(ratio > 0)) throw InputError("run: dt ratio must be positive");
  return scheme_order(cfg.scheme) == 3 ? ratio * dx : ratio * std::pow(dx, 5.0 / 3.0);
}

struct Policy {
  double c_eps = 1.0, volume = 1.0, clip = 1e-3;
  int order = 3;
};

/// eps_global / eps_for_variable (swe.hpp:146-163) of the dense initial fields.
double eps_global_of(const Policy& p, double dx, const std::array<std::vector<double>, 3>& q) {
  double mx = 0.0;
  for (const auto& f : q) {
    double s = 0.0;
    for (double v : f) s += v * v;
    mx = std::max(mx, std::sqrt(s));
  }
  if (mx <= 0.0) return p.clip;
  return p.c_eps * std::sqrt(p.volume) * std::pow(dx, p.order - 0.5) / mx;
}

struct Hooks {
  const CaseSpec* spec;
  Grid grid;
  int nq;
  ttsw_cuda::Solver* tt = nullptr;  // current EpsSchedule for the TT hooks
  std::string error;
};

// RhsHooks of make_rhs_hooks (cases.hpp:175-189) for the device TT solver: Dirichlet ghosts
// through ttsw_ghosted with the exact strips, the manufactured source compressed at the
// step's global tolerance (TTRep::compress).
int tt_fill_ghost(void* user, const ttsw_tt* const* q3, double t, ttsw_tt** out) {
  auto* h = static_cast<Hooks*>(user);
  try {
    const double eps = h->tt->eps()[3];
    const long gx = h->grid.nx + 6, gy = h->grid.ny + 6;
    std::vector<double> sx(size_t(6 * gy)), sy(size_t(6 * gx));
    const int bx = h->spec->bc_x == Boundary::DirichletExact, by = h->spec->bc_y == Boundary::DirichletExact;
    for (int c = 0; c < 3; ++c) {
      exact_strips(*h->spec, h->grid, t, h->nq, c, sx.data(), sy.data());
      CudaTTRep::ctx().check(ttsw_ghosted(CudaTTRep::ctx().get(), q3[c], bx, by, bx ? sx.data() : nullptr,
                                          by ? sy.data() : nullptr, eps, &out[c]));
    }
    return 0;
  } catch (const std::exception& e) {
    h->error = e.what();
    return 1;
  }
}

int tt_source(void* user, double t, ttsw_tt** out) {
  auto* h = static_cast<Hooks*>(user);
  try {
    const double eps = h->tt->eps()[3];
    const auto avg = mms_source_averages(*h->spec, h->grid, t, h->nq);
    const size_t nn = size_t(h->grid.nx * h->grid.ny);
    for (int c = 0; c < 3; ++c)
      CudaTTRep::ctx().check(ttsw_tt_from_full(CudaTTRep::ctx().get(), h->grid.nx, h->grid.ny,
                                               avg.data() + size_t(c) * nn, eps < 0 ? 0.0 : eps, &out[c], nullptr));
    return 0;
  } catch (const std::exception& e) {
    h->error = e.what();
    return 1;
  }
}

int dense_strips(void* user, double t, int c, double* sx, double* sy) {
  auto* h = static_cast<Hooks*>(user);
  try {
    exact_strips(*h->spec, h->grid, t, h->nq, c, sx, sy);
    return 0;
  } catch (const std::exception& e) {
    h->error = e.what();
    return 1;
  }
}

int dense_source(void* user, double t, double* out) {
  auto* h = static_cast<Hooks*>(user);
  try {
    const auto avg = mms_source_averages(*h->spec, h->grid, t, h->nq);
    std::copy(avg.begin(), avg.end(), out);
    return 0;
  } catch (const std::exception& e) {
    h->error = e.what();
    return 1;
  }
}

ttsw_solver_desc make_desc(const CaseSpec& spec, const RunConfig& cfg, double dt, double tol) {
  ttsw_solver_desc d{};
  d.model = int(spec.model);
  d.scheme = int(cfg.scheme);
  d.n = cfg.n;
  d.g = spec.params.g;
  d.f = spec.params.f;
  d.H = spec.params.H;
  d.dt = dt;
  d.tol = tol;
  d.lambda_eps_floor = 1e-6;  // SolverOptions::lambda_eps_floor (swe.hpp:294)
  d.cross = ttsw_cross_cfg{1e-10, 128, 30, 2, 1000, cfg.seed};  // CrossConfig defaults, seed = RunConfig::seed
  return d;
}

std::string format_double(double v) {
  char buf[64];
  auto [ptr, ec] = std::to_chars(buf, buf + sizeof(buf), v);
  return std::string(buf, ptr);
}

}  // namespace

std::array<double, 3> l2_error(const std::array<std::vector<double>, 3>& q, const CaseSpec& spec, const Grid& grid,
                               double t, int nq) {
  std::array<double, 3> out{};
  for (int c = 0; c < 3; ++c) {
    const auto ex = exact_cell_averages(spec, grid, t, nq, c);
    double s = 0.0;
    for (size_t e = 0; e < ex.size(); ++e) {
      const double d = q[size_t(c)][e] - ex[e];
      s += d * d;
    }
    out[size_t(c)] = std::sqrt(grid.dx() * grid.dy() * s);
  }
  return out;
}

RunReport run(const RunConfig& cfg) { return run(cfg, case_spec(cfg.case_id)); }

RunReport run(const RunConfig& cfg, const CaseSpec& spec) {
  if (cfg.n < 16) throw InputError("run: grid must have at least 16 cells per axis");
  if (std::abs(spec.length() - 1.0) > 1e-12)
    throw InputError("run: the device solvers take the unit square (all four cases have length 1)");
  Grid grid;
  grid.nx = grid.ny = cfg.n;
  grid.lx = grid.ly = spec.length();
  Policy policy;
  policy.c_eps = cfg.c_eps.value_or(spec.c_eps[size_t(cfg.scheme)]);
  if (!(policy.c_eps > 0)) throw InputError("run: C_eps must be positive");
  policy.order = scheme_order(cfg.scheme);
  policy.volume = grid.lx * grid.ly;
  const int nq = quadrature_points(cfg.scheme);
  const double T = cfg.final_time.value_or(spec.final_time());
  const double dt_nominal = nominal_dt(spec, cfg, grid.dx());

  RunReport rep;
  rep.case_name = spec.name;
  rep.scheme_label = scheme_name(cfg.scheme);
  rep.rep_label = cfg.rep_label;
  rep.n = cfg.n;
  rep.dt = dt_nominal;
  const auto start = std::chrono::steady_clock::now();

  std::array<std::vector<double>, 3> init;
  for (int c = 0; c < 3; ++c) init[size_t(c)] = exact_cell_averages(spec, grid, 0.0, nq, c);
  Hooks hooks{&spec, grid, nq, nullptr, {}};
  const bool dirichlet = spec.bc_x == Boundary::DirichletExact || spec.bc_y == Boundary::DirichletExact;
  const size_t nn = size_t(cfg.n) * size_t(cfg.n);
  std::array<std::vector<double>, 3> final_state;
  double t = 0.0;
  long steps = 0;
  auto step_wrap = [&](auto&& fn) {
    try {
      fn();
    } catch (const std::exception& e) {
      std::ostringstream os;
      os << "run: " << spec.name << " failed at step " << steps << " (t = " << t << "): " << e.what();
      if (!hooks.error.empty()) os << " [hook: " << hooks.error << "]";
      throw std::runtime_error(os.str());
    }
  };

  if (cfg.rep == Representation::TT) {
    // IC compressed at the global tolerance of the initial field norms (harness.cpp:93-95)
    const double eps0 = eps_global_of(policy, grid.dx(), init);
    ttsw_cuda::Solver solver(make_desc(spec, cfg, dt_nominal, eps0));
    solver.set_eps_policy(policy.c_eps, policy.order, policy.volume, policy.clip);
    for (int c = 0; c < 3; ++c) {
      HostMat m(cfg.n, cfg.n);
      m.a = init[size_t(c)];
      solver.set_state(c, CudaTTRep::compress(m, eps0));
    }
    hooks.tt = &solver;
    if (dirichlet || spec.mms_source)
      solver.set_hooks(dirichlet ? tt_fill_ghost : nullptr, spec.mms_source ? tt_source : nullptr, &hooks);
    bool seen = false;
    double cur_dt = dt_nominal;
    while (t < T * (1.0 - 1e-12)) {
      if (cfg.max_steps && steps >= *cfg.max_steps) break;
      const double dt = std::min(dt_nominal, T - t);
      if (dt != cur_dt) {
        solver.set_dt(dt);
        cur_dt = dt;
      }
      step_wrap([&] { solver.step(1); });
      const auto e = solver.eps();  // the schedule this step used (swe.hpp:167-183)
      for (double v : e) {
        rep.eps_min = seen ? std::min(rep.eps_min, v) : v;
        rep.eps_max = seen ? std::max(rep.eps_max, v) : v;
        seen = true;
      }
      if (cfg.debug_log) rep.eps_log.push_back(e[3]);
      t += dt;
      ++steps;
      std::array<long, 3> ranks{};
      for (int c = 0; c < 3; ++c) {
        ranks[size_t(c)] = solver.state(c).rank();
        rep.max_rank[size_t(c)] = std::max(rep.max_rank[size_t(c)], ranks[size_t(c)]);
      }
      if (cfg.debug_log) rep.rank_log.push_back(ranks);
      if (cfg.debug_positivity && spec.model == Model::Nonlinear) {  // once per step (the reference: per rhs)
        const auto h = CudaTTRep::dense<HostMat>(solver.state(0));
        if (*std::min_element(h.a.begin(), h.a.end()) <= 0.0)
          throw std::runtime_error("rhs: nonpositive layer thickness in the interior");
      }
    }
    for (int c = 0; c < 3; ++c) final_state[size_t(c)] = CudaTTRep::dense<HostMat>(solver.state(c)).a;
  } else {
    ttsw_cuda::DenseSolver solver(make_desc(spec, cfg, dt_nominal, 0.0));
    for (int c = 0; c < 3; ++c) solver.set_state(c, init[size_t(c)].data());
    if (dirichlet || spec.mms_source)
      solver.set_hooks(spec.bc_x == Boundary::DirichletExact, spec.bc_y == Boundary::DirichletExact,
                       dirichlet ? dense_strips : nullptr, spec.mms_source ? dense_source : nullptr, &hooks);
    double cur_dt = dt_nominal;
    while (t < T * (1.0 - 1e-12)) {
      if (cfg.max_steps && steps >= *cfg.max_steps) break;
      const double dt = std::min(dt_nominal, T - t);
      if (dt != cur_dt) {
        solver.set_dt(dt);
        cur_dt = dt;
      }
      step_wrap([&] { solver.step(1); });
      t += dt;
      ++steps;
    }
    for (int c = 0; c < 3; ++c) {
      final_state[size_t(c)].resize(nn);
      solver.state(c, final_state[size_t(c)].data());
    }
  }
  rep.steps = steps;
  rep.l2 = l2_error(final_state, spec, grid, t, nq);
  rep.wall_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - start).count();
  return rep;
}

std::vector<RunReport> convergence(const RunConfig& base, const std::vector<int>& grids) {
  return convergence(base, grids, case_spec(base.case_id));
}

std::vector<RunReport> convergence(const RunConfig& base, const std::vector<int>& grids, const CaseSpec& spec) {
  if (grids.size() < 2) throw InputError("convergence: need at least two grids");
  for (size_t i = 1; i < grids.size(); ++i)
    if (grids[i] != 2 * grids[i - 1]) throw InputError("convergence: grids must double between levels");
  // levels run one after another on the device (the reference may overlap them on host
  // threads, TTSWE_THREADS; here each level already uses the whole GPU)
  std::vector<RunReport> reports;
  for (int n : grids) {
    RunConfig cfg = base;
    cfg.n = n;
    reports.push_back(run(cfg, spec));
  }
  for (size_t i = 0; i < reports.size(); ++i) {
    for (int c = 0; c < 3; ++c)
      reports[i].rel_l2[size_t(c)] = reports[0].l2[size_t(c)] > 0 ? reports[i].l2[size_t(c)] / reports[0].l2[size_t(c)] : 1.0;
    if (i > 0 && reports[i].l2[0] > 0) reports[i].order_c1 = std::log2(reports[i - 1].l2[0] / reports[i].l2[0]);
  }
  return reports;
}

void write_csv(std::ostream& os, const std::vector<RunReport>& reports) {
  os << "case,scheme,rep,N,dt,steps,l2_c1,l2_c2,l2_c3,rel_l2_c1,order_c1,max_rank,wall_s,eps_min,eps_max\n";
  for (const auto& r : reports) {
    const long mr = std::max({r.max_rank[0], r.max_rank[1], r.max_rank[2]});
    os << r.case_name << ',' << r.scheme_label << ',' << r.rep_label << ',' << r.n << ',' << format_double(r.dt) << ','
       << r.steps << ',' << format_double(r.l2[0]) << ',' << format_double(r.l2[1]) << ','
       << format_double(r.l2[2]) << ',' << format_double(r.rel_l2[0]) << ','
       << (r.order_c1 ? format_double(*r.order_c1) : std::string()) << ',' << mr << ',' << format_double(r.wall_s)
       << ',' << format_double(r.eps_min) << ',' << format_double(r.eps_max) << '\n';
  }
}

void write_json(std::ostream& os, const std::vector<RunReport>& reports) {
  // one object per report; keys sorted as an ordered JSON object map emits them
  auto str = [](const std::string& s) {
    std::string o = "\"";
    for (char ch : s) {
      if (ch == '"' || ch == '\\') o += '\\';
      o += ch;
    }
    return o + "\"";
  };
  os << "[";
  for (size_t k = 0; k < reports.size(); ++k) {
    const auto& r = reports[k];
    std::map<std::string, std::string> row{
        {"case", str(r.case_name)},
        {"scheme", str(r.scheme_label)},
        {"rep", str(r.rep_label)},
        {"N", std::to_string(r.n)},
        {"dt", format_double(r.dt)},
        {"steps", std::to_string(r.steps)},
        {"l2_c1", format_double(r.l2[0])},
        {"l2_c2", format_double(r.l2[1])},
        {"l2_c3", format_double(r.l2[2])},
        {"rel_l2_c1", format_double(r.rel_l2[0])},
        {"max_rank", std::to_string(std::max({r.max_rank[0], r.max_rank[1], r.max_rank[2]}))},
        {"wall_s", format_double(r.wall_s)},
        {"eps_min", format_double(r.eps_min)},
        {"eps_max", format_double(r.eps_max)},
        {"order_c1", r.order_c1 ? format_double(*r.order_c1) : std::string("null")},
    };
    os << (k ? ",\n  {" : "\n  {");
    size_t i = 0;
    for (const auto& [key, v] : row) os << (i++ ? ",\n    " : "\n    ") << str(key) << ": " << v;
    os << "\n  }";
  }
  os << (reports.empty() ? "]\n" : "\n]\n");
}

namespace {

int emit_reports(const RunConfig& cfg, const std::vector<RunReport>& reports) {
  if (!cfg.out.empty()) {
    std::ofstream file(cfg.out, std::ios::binary);
    if (!file) {
      std::cerr << "error: cannot open output file '" << cfg.out << "'\n";
      return 1;
    }
    write_csv(file, reports);
    if (cfg.json) {
      std::ofstream jf(cfg.out + ".json", std::ios::binary);
      write_json(jf, reports);
    }
  }
  if (cfg.json && cfg.out.empty())
    write_json(std::cout, reports);
  else
    write_csv(std::cout, reports);
  return 0;
}

const char* kUsage =
    "Tensor-train finite volume solver for the shallow water equations (B200)\n"
    "Usage: ttswe SUBCOMMAND [OPTIONS]\n"
    "  run          Integrate one configuration (--n N)\n"
    "  convergence  Grid-doubling convergence study (--grids N1,N2,...)\n"
    "  cases        Print exact cell averages / sources (host only, no GPU)\n"
    "Options: --case {kelvin,inertia-gravity,barotropic-tide,manufactured} --scheme {upwind3,upwind5,weno5}\n"
    "         --rep {dense,tt,cuda,cuda-dense} --dt-ratio R --c-eps C --out PATH --seed S --json\n"
    "         --debug-positivity --device D; testing: --final-time T --max-steps K\n";

int usage_error(const std::string& m) {
  std::cerr << m << "\n" << kUsage;
  return 1;
}

bool to_double(const std::string& s, double& v) {
  const char* b = s.data();
  auto [p, ec] = std::from_chars(b, b + s.size(), v);
  return ec == std::errc() && p == b + s.size();
}

template <class I>
bool to_int(const std::string& s, I& v) {
  const char* b = s.data();
  auto [p, ec] = std::from_chars(b, b + s.size(), v);
  return ec == std::errc() && p == b + s.size();
}

// ttswe cases: values for host-side checks (no device work)
int cases_cmd(const std::map<std::string, std::string>& o) {
  const auto id = parse_case_id(o.count("--case") ? o.at("--case") : "kelvin");
  if (!id) return usage_error("error: --case: unknown case");
  const CaseSpec spec = case_spec(*id);
  long n = 16;
  double t = 0;
  int nq = 3, comp = 0;
  if (o.count("--n") && !to_int(o.at("--n"), n)) return usage_error("error: --n");
  if (o.count("--t") && !to_double(o.at("--t"), t)) return usage_error("error: --t");
  if (o.count("--nq") && !to_int(o.at("--nq"), nq)) return usage_error("error: --nq");
  if (o.count("--component") && !to_int(o.at("--component"), comp)) return usage_error("error: --component");
  const std::string what = o.count("--what") ? o.at("--what") : "exact";
  Grid g;
  g.nx = g.ny = n;
  g.lx = g.ly = spec.length();
  std::vector<double> v;
  if (what == "exact") {
    v = exact_cell_averages(spec, g, t, nq, comp);
  } else if (what == "source") {
    v = mms_source_averages(spec, g, t, nq);
  } else if (what == "strips") {
    v.resize(size_t(12 * (n + 6)));
    exact_strips(spec, g, t, nq, comp, v.data(), v.data() + 6 * (n + 6));
  } else if (what == "spec") {
    std::cout << spec.name << ',' << format_double(spec.params.g) << ',' << format_double(spec.params.f) << ','
              << format_double(spec.params.H) << ',' << format_double(spec.final_time()) << ','
              << format_double(spec.length()) << '\n';
    return 0;
  } else {
    return usage_error("error: --what must be exact, source, strips or spec");
  }
  for (size_t i = 0; i < v.size(); ++i) std::cout << (i ? "," : "") << format_double(v[i]);
  std::cout << '\n';
  return 0;
}

}  // namespace

int run_cli(int argc, const char* const* argv) {
  if (argc < 2) return usage_error("error: a subcommand is required");
  const std::string sub = argv[1];
  if (sub == "--help" || sub == "-h") {
    std::cout << kUsage;
    return 0;
  }
  if (sub != "run" && sub != "convergence" && sub != "cases") return usage_error("error: unknown subcommand " + sub);
  static const std::vector<std::string> with_value = {"--case", "--scheme", "--rep", "--dt-ratio", "--c-eps",
                                                      "--out", "--seed", "--n", "--grids", "--final-time",
                                                      "--max-steps", "--device", "--t", "--nq", "--what",
                                                      "--component"};
  static const std::vector<std::string> flags = {"--json", "--debug-positivity", "--debug-log"};
  std::map<std::string, std::string> opt;
  for (int i = 2; i < argc; ++i) {
    std::string a = argv[i], v;
    if (a == "--help" || a == "-h") {
      std::cout << kUsage;
      return 0;
    }
    const auto eq = a.find('=');
    if (a.rfind("--", 0) == 0 && eq != std::string::npos) {
      v = a.substr(eq + 1);
      a = a.substr(0, eq);
    }
    if (std::find(flags.begin(), flags.end(), a) != flags.end()) {
      opt[a] = "1";
      continue;
    }
    if (std::find(with_value.begin(), with_value.end(), a) == with_value.end())
      return usage_error("error: unknown option " + a);
    if (a == "--n" && sub == "convergence") return usage_error("error: --n is an option of run");
    if (a == "--grids" && sub == "run") return usage_error("error: --grids is an option of convergence");
    if (eq == std::string::npos) {
      if (i + 1 >= argc) return usage_error("error: " + a + " needs a value");
      v = argv[++i];
    }
    opt[a] = v;
  }
  if (sub == "cases") return cases_cmd(opt);

  RunConfig cfg;
  std::string case_name = opt.count("--case") ? opt["--case"] : "kelvin";
  std::string scheme = opt.count("--scheme") ? opt["--scheme"] : "upwind3";
  std::string rep = opt.count("--rep") ? opt["--rep"] : "dense";
  const auto id = parse_case_id(case_name);
  if (!id) return usage_error("error: --case: " + case_name + " not in {kelvin,inertia-gravity,barotropic-tide,manufactured}");
  const auto sc = parse_scheme(scheme);
  if (!sc) return usage_error("error: --scheme: " + scheme + " not in {upwind3,upwind5,weno5}");
  const auto rp = parse_representation(rep);
  if (!rp) return usage_error("error: --rep: " + rep + " not in {dense,tt,cuda,cuda-dense}");
  cfg.case_id = *id;
  cfg.scheme = *sc;
  cfg.rep = *rp;
  cfg.rep_label = rep;
  if (opt.count("--n") && (!to_int(opt["--n"], cfg.n) || cfg.n <= 0))
    return usage_error("error: --n must be a positive number");
  double v = 0;
  if (opt.count("--dt-ratio")) {
    if (!to_double(opt["--dt-ratio"], v)) return usage_error("error: --dt-ratio must be a number");
    if (v != 0.0) cfg.dt_ratio = v;
  }
  if (opt.count("--c-eps")) {
    if (!to_double(opt["--c-eps"], v)) return usage_error("error: --c-eps must be a number");
    if (v != 0.0) cfg.c_eps = v;
  }
  if (opt.count("--seed") && !to_int(opt["--seed"], cfg.seed)) return usage_error("error: --seed must be an integer");
  if (opt.count("--final-time")) {
    if (!to_double(opt["--final-time"], v)) return usage_error("error: --final-time must be a number");
    cfg.final_time = v;
  }
  if (opt.count("--max-steps")) {
    long k = 0;
    if (!to_int(opt["--max-steps"], k)) return usage_error("error: --max-steps must be an integer");
    cfg.max_steps = k;
  }
  if (opt.count("--device") && !to_int(opt["--device"], cfg.device)) return usage_error("error: --device");
  cfg.out = opt.count("--out") ? opt["--out"] : "";
  cfg.json = opt.count("--json") > 0;
  cfg.debug_positivity = opt.count("--debug-positivity") > 0;
  cfg.debug_log = opt.count("--debug-log") > 0;
  std::vector<int> grids;
  if (sub == "convergence") {
    if (!opt.count("--grids")) return usage_error("error: --grids is required");
    std::stringstream ss(opt["--grids"]);
    std::string tok;
    while (std::getline(ss, tok, ',')) {
      int g = 0;
      if (!to_int(tok, g) || g <= 0) {
        std::cerr << "error: invalid grid size '" << tok << "'\n";
        return 1;
      }
      grids.push_back(g);
    }
  }
  try {
    if (cfg.device != 0) ttsw_cuda::Context::select_device(cfg.device);
    if (sub == "run") return emit_reports(cfg, {run(cfg)});
    return emit_reports(cfg, convergence(cfg, grids));
  } catch (const InputError& e) {
    std::cerr << "error: " << e.what() << '\n';
    return 1;
  } catch (const ttsw_cuda::Error& e) {
    if (e.code == TTSW_INPUT) {
      std::cerr << "error: " << e.what() << '\n';
      return 1;
    }
    std::cerr << "solver error: " << e.what() << '\n';
    return 2;
  } catch (const std::exception& e) {
    std::cerr << "solver error: " << e.what() << '\n';
    return 2;
  }
}

}  // namespace ttswe
