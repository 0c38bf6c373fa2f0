// TEST INFRASTRUCTURE ONLY — pins the CPU oracle (cas_oracle.hpp) to the
// reference's own known-answer and property tests for the hot path.  The
// reference ships no golden vectors and cannot be built here (no Eigen), so
// these ported assertions — same inputs, same tolerances — are the pin.
// Each TEST names the reference test it ports (/root/reference/proj/tests/).
#include <cmath>
#include <complex>
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

#include "../cas_oracle.hpp"

using namespace orc;

static int g_fail = 0, g_checks = 0;
static std::string g_test;
#define REQUIRE(cond)                                                                   \
  do {                                                                                  \
    ++g_checks;                                                                         \
    if (!(cond)) {                                                                      \
      ++g_fail;                                                                         \
      std::printf("FAIL [%s] %s:%d: %s\n", g_test.c_str(), __FILE__, __LINE__, #cond); \
    }                                                                                   \
  } while (0)

struct TestReg {
  static std::vector<std::pair<std::string, std::function<void()>>>& all() {
    static std::vector<std::pair<std::string, std::function<void()>>> v;
    return v;
  }
  TestReg(const char* n, std::function<void()> f) { all().emplace_back(n, f); }
};
#define TEST(name)                                 \
  static void name();                              \
  static TestReg reg_##name(#name, name);          \
  static void name()

static Shape cshape(int d, int N, int S = 32) {
  Shape s;
  s.complex_field = true;
  s.d = d;
  s.N = N;
  s.lanes = S;
  return s;
}

static Vec random_test_frame(const Shape& sh, std::uint64_t seed) {  // support.hpp:75-78
  Rng r(seed);
  return random_frame(sh, r);
}

// support.hpp:83-97 — independent coordinate-wise central FD of the value
static Vec fd_gradient(const Shape& sh, const Vec& point, double delta, bool squared = true) {
  Vec g(point.size()), p = point;
  for (size_t i = 0; i < point.size(); ++i) {
    const double h = 5e-8 * (1.0 + std::abs(point[i]));
    const double saved = p[i];
    p[i] = saved + h;
    const double fp = eval_objective(sh, p.data(), nullptr, 0.0, delta, squared).value;
    p[i] = saved - h;
    const double fm = eval_objective(sh, p.data(), nullptr, 0.0, delta, squared).value;
    p[i] = saved;
    g[i] = (fp - fm) / (2.0 * h);
  }
  return g;
}

static double componentwise_rel_error(const Vec& a, const Vec& b) {  // support.hpp:101-108
  double worst = 0.0;
  for (size_t i = 0; i < a.size(); ++i) {
    const double scale = std::max({1.0, std::abs(a[i]), std::abs(b[i])});
    worst = std::max(worst, std::abs(a[i] - b[i]) / scale);
  }
  return worst;
}

static Vec sic_2_4() {  // support.hpp:22-35
  Vec f(16, 0.0);
  f[0] = 1.0;
  const double c = std::sqrt(1.0 / 3.0), s = std::sqrt(2.0 / 3.0);
  for (int k = 0; k < 3; ++k) {
    const double phi = 2.0 * 3.14159265358979323846 * k / 3.0;
    const std::complex<double> e = std::polar(s, phi);
    f[4 * (k + 1) + 0] = c;
    f[4 * (k + 1) + 2] = e.real();
    f[4 * (k + 1) + 3] = e.imag();
  }
  return f;
}

static Vec sic_3_9() {  // support.hpp:39-55
  const std::complex<double> fid[3] = {0.0, 1.0 / std::sqrt(2.0), -1.0 / std::sqrt(2.0)};
  const double w = 2.0 * 3.14159265358979323846 / 3.0;
  Vec f(2 * 3 * 9);
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) {
      const int col = 3 * a + b;
      for (int j = 0; j < 3; ++j) {
        const std::complex<double> v = std::polar(1.0, w * b * j) * fid[(j - a + 3) % 3];
        f[2 * (j + 3 * col)] = v.real();
        f[2 * (j + 3 * col) + 1] = v.imag();
      }
    }
  return f;
}

// smooth_max / lse_partials (smoothing.hpp:46-69), restated on the CAS exp/log
static double smooth_max(const Vec& x, double delta) {
  double s = x[0];
  for (double v : x) s = std::max(s, v);
  double z = 0.0;
  for (double v : x) z += cas_exp((v - s) / delta);
  return s + delta * cas_log(z);
}
static Vec lse_partials(const Vec& x, double delta) {
  double s = x[0];
  for (double v : x) s = std::max(s, v);
  Vec w(x.size());
  double z = 0.0;
  for (size_t i = 0; i < x.size(); ++i) {
    w[i] = cas_exp((x[i] - s) / delta);
    z += w[i];
  }
  for (double& v : w) v /= z;
  return w;
}

// ----------------------------------------------------------- test_smoothing.cpp
TEST(orthogonal_pair_gives_objective_zero) {  // test_smoothing.cpp:16-25
  Vec id = {1, 0, 0, 0, 0, 0, 1, 0};
  for (double delta : {1.0, 1e-2, 1e-6}) {
    EvalResult e = eval_objective(cshape(2, 2), id.data(), nullptr, 0.0, delta);
    REQUIRE(e.s == 0.0);
    REQUIRE(e.value == 0.0);
  }
}

TEST(coincident_pair_gives_objective_one) {  // test_smoothing.cpp:27-34
  Vec f = {1, 0, 0, 0, 1, 0, 0, 0};
  EvalResult e = eval_objective(cshape(2, 2), f.data(), nullptr, 0.0, 0.1);
  REQUIRE(std::abs(e.value - 1.0) <= 1e-15);
}

TEST(sandwich_property_on_random_frames) {  // test_smoothing.cpp:36-46
  for (std::uint64_t seed = 1; seed <= 20; ++seed) {
    Shape sh = cshape(3, 6);
    Vec f = random_test_frame(sh, seed);
    EvalResult e = eval_objective(sh, f.data(), nullptr, 0.0, 1e-3, true, true);
    const double overshoot = 1e-3 * std::log(15.0);
    REQUIRE(e.s <= e.value);
    REQUIRE(e.value <= e.s + overshoot);
    double sum = 0.0;
    for (double w : e.weights) sum += w;
    REQUIRE(std::abs(sum - 1.0) < 1e-12);
  }
}

TEST(lse_partials_matches_closed_forms) {  // test_smoothing.cpp:48-68
  Vec w = lse_partials({0.4, 0.4, 0.4}, 0.05);
  for (double v : w) REQUIRE(std::abs(v - 1.0 / 3.0) <= 1e-15);
  Vec sharp = lse_partials({1.0, 0.0}, 1e-3);
  REQUIRE(std::abs(sharp[0] - 1.0) <= 1e-12);
  REQUIRE(std::abs(sharp[1]) <= 1e-12);
  Vec soft = lse_partials({0.5, 0.3}, 0.1);
  const double e0 = 1.0 / (1.0 + std::exp(-2.0));
  REQUIRE(std::abs(soft[0] - e0) <= 1e-12);
  REQUIRE(std::abs(soft[1] - (1.0 - e0)) <= 1e-12);
}

TEST(stabilized_value_equals_unshifted_form) {  // test_smoothing.cpp:70-81
  Rng rng(5);
  for (int trial = 0; trial < 50; ++trial) {
    Vec x(6);
    for (double& v : x) v = rng.uniform();
    const double delta = 0.25 + rng.uniform();
    double z = 0.0;
    for (double v : x) z += std::exp(v / delta);
    REQUIRE(std::abs(smooth_max(x, delta) - delta * std::log(z)) <= 1e-12);
  }
}

TEST(decreasing_delta_never_increases_value) {  // test_smoothing.cpp:83-95
  Rng rng(11);
  for (int trial = 0; trial < 10; ++trial) {
    Vec x(10);
    for (double& v : x) v = rng.uniform();
    double prev = std::numeric_limits<double>::infinity();
    for (double delta : {1.0, 0.3, 0.1, 0.03, 0.01, 1e-3, 1e-5}) {
      const double v = smooth_max(x, delta);
      REQUIRE(v <= prev + 1e-15);
      prev = v;
    }
  }
}

TEST(objective_invariant_under_column_permutation) {  // test_smoothing.cpp:97-106
  Shape sh = cshape(3, 5);
  Vec f = random_test_frame(sh, 77);
  const double base = eval_objective(sh, f.data(), nullptr, 0.0, 1e-2).value;
  Vec p = f;
  auto swapcol = [&](int a, int b) {
    for (int q = 0; q < 6; ++q) std::swap(p[6 * a + q], p[6 * b + q]);
  };
  swapcol(1, 4);
  swapcol(0, 2);
  REQUIRE(std::abs(base - eval_objective(sh, p.data(), nullptr, 0.0, 1e-2).value) <= 1e-12);
}

TEST(analytic_gradient_matches_central_fd) {  // test_smoothing.cpp:108-123
  const std::pair<int, int> sizes[] = {{2, 4}, {3, 6}, {4, 10}};
  std::uint64_t seed = 100;
  for (auto [d, n] : sizes)
    for (double delta : {1e-1, 1e-3})
      for (int rep = 0; rep < 4; ++rep) {
        Shape sh = cshape(d, n);
        Vec f = random_test_frame(sh, ++seed);
        Vec a = eval_objective(sh, f.data(), nullptr, 0.0, delta).grad;
        REQUIRE(componentwise_rel_error(a, fd_gradient(sh, f, delta)) <= 1e-5);
      }
}

TEST(magnitude_mode_gradient_matches_fd) {  // test_smoothing.cpp:125-132
  Shape sh = cshape(3, 5);
  Vec f = random_test_frame(sh, 4096);
  Vec a = eval_objective(sh, f.data(), nullptr, 0.0, 1e-1, false).grad;
  REQUIRE(componentwise_rel_error(a, fd_gradient(sh, f, 1e-1, false)) <= 1e-5);
}

TEST(gradient_zero_along_column_rescaling) {  // test_smoothing.cpp:134-146
  Shape sh = cshape(3, 4);
  Vec f = random_test_frame(sh, 2024);
  Vec g = eval_objective(sh, f.data(), nullptr, 0.0, 1e-2).grad;
  for (int j = 0; j < 4; ++j) {
    double dot = 0.0;
    for (int q = 0; q < 6; ++q) dot += g[6 * j + q] * f[6 * j + q];
    REQUIRE(std::abs(dot) < 1e-12);
  }
}

TEST(zero_column_propagates_from_evaluation) {  // test_smoothing.cpp:148-153
  Vec p(8, 0.0);
  p[0] = 1.0;
  REQUIRE(eval_objective(cshape(2, 2), p.data(), nullptr, 0.0, 0.1).zero_col == 1);
}

TEST(hvp_on_zero_direction_is_zero) {  // test_smoothing.cpp:155-162
  Shape sh = cshape(2, 4);
  Vec f = random_test_frame(sh, 8);
  HvpResult r = hvp_adapter(sh, f, Vec(f.size(), 0.0), 1e-2, nullptr);
  double nrm = 0.0;
  for (double v : r.hv) nrm += v * v;
  REQUIRE(nrm == 0.0);
}

TEST(hvp_is_symmetric_at_random_frame_points) {  // test_smoothing.cpp:184-197
  Shape sh = cshape(3, 6);
  Vec f = random_test_frame(sh, 55);
  Rng rng(56);
  Vec v(f.size()), w(f.size());
  for (size_t i = 0; i < f.size(); ++i) {
    v[i] = rng.normal();
    w[i] = rng.normal();
  }
  HvpResult hv = hvp_adapter(sh, f, v, 1e-2, nullptr), hw = hvp_adapter(sh, f, w, 1e-2, nullptr);
  double hvw = 0.0, hwv = 0.0;
  for (size_t i = 0; i < f.size(); ++i) {
    hvw += hv.hv[i] * w[i];
    hwv += hw.hv[i] * v[i];
  }
  REQUIRE(hv.path == HVP_CENTRAL && hw.path == HVP_CENTRAL);
  REQUIRE(std::abs(hvw - hwv) <= 1e-4 * std::max(std::abs(hvw), std::abs(hwv)));
}

// ------------------------------------------------------- test_trust_region.cpp
static HvpOperator matrix_op(const std::vector<Vec>& m) {
  return [m](const Vec& v) {
    Vec out(v.size(), 0.0);
    for (size_t i = 0; i < v.size(); ++i)
      for (size_t j = 0; j < v.size(); ++j) out[i] += m[i][j] * v[j];
    return out;
  };
}
static std::vector<Vec> identity(int n) {
  std::vector<Vec> m(n, Vec(n, 0.0));
  for (int i = 0; i < n; ++i) m[i][i] = 1.0;
  return m;
}
static double nrm(const Vec& v) {
  double s = 0.0;
  for (double x : v) s += x * x;
  return std::sqrt(s);
}

TEST(steihaug_returns_zero_on_vanishing_gradient) {  // test_trust_region.cpp:27-34
  auto [step, tr] = steihaug_cg(Vec(5, 0.0), matrix_op(identity(5)), 1.0, 1e-8, 10, 32);
  REQUIRE(nrm(step) == 0.0);
  REQUIRE(tr.exit_reason == CG_ZERO_GRADIENT);
}

TEST(steihaug_recovers_newton_step_on_identity) {  // test_trust_region.cpp:36-45
  Rng rng(1);
  Vec g(6);
  for (double& v : g) v = rng.normal();
  auto [step, tr] = steihaug_cg(g, matrix_op(identity(6)), 10.0 * nrm(g), 1e-10 * nrm(g), 12, 32);
  Vec s(6);
  for (int i = 0; i < 6; ++i) s[i] = step[i] + g[i];
  REQUIRE(nrm(s) <= 1e-8 * nrm(g));
  REQUIRE(tr.exit_reason == CG_SMALL_RESIDUAL);
}

TEST(steihaug_clips_to_boundary_along_steepest_descent) {  // test_trust_region.cpp:47-58
  Rng rng(2);
  Vec g(6);
  for (double& v : g) v = rng.normal();
  const double radius = 0.5 * nrm(g);
  auto [step, tr] = steihaug_cg(g, matrix_op(identity(6)), radius, 1e-10, 12, 32);
  REQUIRE(tr.exit_reason == CG_BOUNDARY_HIT);
  REQUIRE(std::abs(nrm(step) - radius) <= 1e-10 * radius);
  double dot = 0.0;
  for (int i = 0; i < 6; ++i) dot += step[i] * g[i];
  REQUIRE(std::abs(-dot / (nrm(step) * nrm(g)) - 1.0) <= 1e-12);
}

TEST(steihaug_negative_curvature_exits_on_boundary) {  // test_trust_region.cpp:60-72
  std::vector<Vec> b = {{1.0, 0.0}, {0.0, -1.0}};
  for (double radius : {0.3, 1.0, 5.0, 50.0}) {
    auto [step, tr] = steihaug_cg({1.0, 0.1}, matrix_op(b), radius, 1e-12, 100, 32);
    REQUIRE(tr.exit_reason == CG_NEGATIVE_CURVATURE || tr.exit_reason == CG_BOUNDARY_HIT);
    REQUIRE(std::abs(nrm(step) - radius) <= 1e-10 * radius);
  }
}

TEST(steihaug_steps_respect_radius_and_decrease_model) {  // test_trust_region.cpp:88-108
  Rng rng(4);
  const int dim = 8;
  for (int trial = 0; trial < 20; ++trial) {
    std::vector<Vec> b(dim, Vec(dim));
    for (int i = 0; i < dim; ++i)
      for (int j = 0; j < dim; ++j) b[i][j] = rng.normal();
    std::vector<Vec> s(dim, Vec(dim));
    for (int i = 0; i < dim; ++i)
      for (int j = 0; j < dim; ++j) s[i][j] = 0.5 * (b[i][j] + b[j][i]);
    Vec g(dim);
    for (double& v : g) v = rng.normal();
    const double radius = 0.1 + 3.0 * rng.uniform();
    auto [step, tr] = steihaug_cg(g, matrix_op(s), radius, 1e-8, 2 * dim, 32);
    REQUIRE(nrm(step) <= radius * (1.0 + 1e-10));
    REQUIRE(tr.model_value <= 0.0);
    Vec bs = matrix_op(s)(step);
    double direct = 0.0, sbs = 0.0;
    for (int i = 0; i < dim; ++i) {
      direct += g[i] * step[i];
      sbs += step[i] * bs[i];
    }
    direct += 0.5 * sbs;
    REQUIRE(std::abs(direct - tr.model_value) <= 1e-9 * std::max(1.0, std::abs(direct)));
  }
}

TEST(minimize_quadratic_to_zero) {  // test_trust_region.cpp:110-126
  Rng rng(5);
  Vec x0(10);
  for (double& v : x0) v = 2.0 * rng.uniform() - 1.0;
  Objective f = [](const Vec& x) {
    Vec g(x.size());
    double v = 0.0;
    for (size_t i = 0; i < x.size(); ++i) {
      v += x[i] * x[i];
      g[i] = 2.0 * x[i];
    }
    return Evaluation{v, g};
  };
  HvpFactory fac = [](const Vec&) -> HvpOperator {
    return [](const Vec& v) {
      Vec o(v.size());
      for (size_t i = 0; i < v.size(); ++i) o[i] = 2.0 * v[i];
      return o;
    };
  };
  TrustRegionConfig cfg;
  MinimizeResult r = trust_region_minimize(f, fac, x0, cfg, 32);
  REQUIRE(r.status == ST_GRADIENT_TOLERANCE);
  REQUIRE(r.history.size() <= 10);
  REQUIRE(nrm(r.x) <= 1e-9);
}

TEST(minimize_rosenbrock_from_classic_start) {  // test_trust_region.cpp:128-152
  Objective f = [](const Vec& x) {
    const double a = 1.0 - x[0], b = x[1] - x[0] * x[0];
    return Evaluation{a * a + 100.0 * b * b, {-2.0 * a - 400.0 * x[0] * b, 200.0 * b}};
  };
  HvpFactory fac = [&f](const Vec& x) -> HvpOperator {
    return [&f, x](const Vec& dir) {
      const double dn = nrm(dir);
      if (dn == 0.0) return Vec(x.size(), 0.0);
      const double h = kFdBaseStep * (1.0 + nrm(x)) / std::max(dn, 1e-300);
      Vec p(x.size()), m(x.size());
      for (size_t i = 0; i < x.size(); ++i) {
        p[i] = x[i] + h * dir[i];
        m[i] = x[i] - h * dir[i];
      }
      Vec gp = f(p).grad, gm = f(m).grad, o(x.size());
      for (size_t i = 0; i < x.size(); ++i) o[i] = (gp[i] - gm[i]) / (2.0 * h);
      return o;
    };
  };
  TrustRegionConfig cfg;
  cfg.grad_tol = 1e-8;
  cfg.max_outer = 500;
  MinimizeResult r = trust_region_minimize(f, fac, {-1.2, 1.0}, cfg, 32);
  REQUIRE(r.value < 1e-8);
  REQUIRE(std::abs(r.x[0] - 1.0) <= 1e-4);
  REQUIRE(std::abs(r.x[1] - 1.0) <= 1e-4);
}

TEST(minimize_stationary_start_returns_immediately) {  // test_trust_region.cpp:154-168
  Objective f = [](const Vec& x) {
    Vec g(x.size());
    double v = 0.0;
    for (size_t i = 0; i < x.size(); ++i) {
      v += x[i] * x[i];
      g[i] = 2.0 * x[i];
    }
    return Evaluation{v, g};
  };
  HvpFactory fac = [](const Vec&) -> HvpOperator { return [](const Vec& v) { return v; }; };
  TrustRegionConfig cfg;
  cfg.grad_tol = 1e-6;
  MinimizeResult r = trust_region_minimize(f, fac, Vec(4, 0.0), cfg, 32);
  REQUIRE(r.status == ST_GRADIENT_TOLERANCE);
  REQUIRE(r.history.empty());
}

TEST(pole_rejects_and_shrinks) {  // test_trust_region.cpp:202-222
  Objective f = [](const Vec& x) {
    if (x[0] >= 0.9) return Evaluation{std::numeric_limits<double>::infinity(), Vec(1, 0.0)};
    const double s = x[0] - 0.5;
    return Evaluation{s * s, {2.0 * s}};
  };
  HvpFactory fac = [](const Vec&) -> HvpOperator {
    return [](const Vec& v) { return Vec{2.0 * v[0]}; };
  };
  TrustRegionConfig cfg;
  cfg.grad_tol = 1e-10;
  MinimizeResult r = trust_region_minimize(f, fac, {-3.0}, cfg, 32);
  REQUIRE(std::abs(r.x[0] - 0.5) <= 1e-8);
}

TEST(config_invariants_are_validated) {  // test_trust_region.cpp:224-236
  Objective f = [](const Vec& x) { return Evaluation{0.0, Vec(x.size(), 0.0)}; };
  HvpFactory fac = [](const Vec&) -> HvpOperator { return [](const Vec& v) { return v; }; };
  TrustRegionConfig bad;
  bad.eta = 0.3;
  bool threw = false;
  try {
    trust_region_minimize(f, fac, Vec(2, 1.0), bad, 32);
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  REQUIRE(threw);
}

// ---------------------------------------------------------- test_solver.cpp
TEST(default_schedule_ends_at_eps_over_2logN) {  // test_solver.cpp:12-25
  std::vector<double> s = default_delta_schedule(100, 1e-6);
  REQUIRE(std::abs(s.front() - 1e-1) <= 1e-12);
  REQUIRE(std::abs(s.back() - 1.0857e-7) <= 1e-3 * 1.0857e-7);
  std::vector<double> t = default_delta_schedule(2, 1e-6);
  REQUIRE(std::abs(t.back() - 1e-6 / (2.0 * std::log(2.0))) <= 1e-12 * t.back());
}

TEST(default_schedule_strictly_decreasing) {  // test_solver.cpp:27-40
  for (int n : {2, 5, 30, 100, 500})
    for (double eps : {1e-3, 1e-5, 1e-7}) {
      std::vector<double> s = default_delta_schedule(n, eps);
      REQUIRE(s.size() >= 2);
      for (size_t k = 0; k + 1 < s.size(); ++k) REQUIRE(s[k] > s[k + 1] && s[k + 1] > 0.0);
    }
  for (int n = 2; n <= 100; ++n) {
    const double term = default_delta_schedule(n, 1e-7).back();
    REQUIRE(term >= 1e-8 && term <= 1e-7);
  }
}

TEST(random_frames_deterministic_unit_norm) {  // test_solver.cpp:42-51
  Shape sh = cshape(2, 1000);
  Rng a(42), b(42);
  Vec fa = random_frame(sh, a), fb = random_frame(sh, b);
  REQUIRE(fa == fb);
  for (int j = 0; j < 1000; ++j) REQUIRE(std::abs(column_norm(&fa[4 * j], 4) - 1.0) <= 1e-12);
}

TEST(random_pair_overlaps_average_one_over_d) {  // test_solver.cpp:53-71
  Shape sh = cshape(3, 2);
  Rng rng(777);
  double sum = 0.0, sq = 0.0;
  const int pairs = 20000;
  for (int p = 0; p < pairs; ++p) {
    Vec f = random_frame(sh, rng);
    double gr, gi;
    gram_entry(sh, &f[0], &f[6], &gr, &gi);
    const double o = gr * gr + gi * gi;
    sum += o;
    sq += o * o;
  }
  const double mean = sum / pairs, var = (sq - pairs * mean * mean) / (pairs - 1.0);
  REQUIRE(std::abs(mean - 1.0 / 3.0) <= 3.0 * std::sqrt(var / pairs));
}

TEST(anneal_finds_orthogonal_pair) {  // test_solver.cpp:73-84
  SolverConfig cfg;
  cfg.shape = cshape(2, 2);
  cfg.eps_target = 1e-6;
  Rng rng(1);
  Vec start = random_frame(cfg.shape, rng);
  AnnealResult a = anneal(start, cfg, &rng);
  REQUIRE(a.mu <= 1e-6);
  REQUIRE(a.stages.size() >= 2);
}

TEST(solve_one_restart_equals_anneal_on_child_seed) {  // test_solver.cpp:95-110
  SolverConfig cfg;
  cfg.shape = cshape(2, 3);
  cfg.restarts = 1;
  cfg.seed = 9001;
  cfg.eps_target = 1e-5;
  SolveResult r = solve(cfg, 1);
  Rng rng(mix_seed(9001, 0));
  Vec start = random_frame(cfg.shape, rng);
  AnnealResult a = anneal(start, cfg, &rng);
  REQUIRE(r.best_frame == a.frame);
  REQUIRE(r.per_restart[0].stages.size() == a.stages.size());
}

TEST(solve_deterministic_and_thread_count_independent) {  // test_solver.cpp:112-132
  SolverConfig cfg;
  cfg.shape = cshape(2, 4);
  cfg.restarts = 6;
  cfg.seed = 31337;
  cfg.eps_target = 1e-6;
  SolveResult a = solve(cfg, 1), b = solve(cfg, 1), c = solve(cfg, 4);
  REQUIRE(a.best_frame == b.best_frame);
  REQUIRE(a.best_coherence == c.best_coherence);
  REQUIRE(a.best_restart == c.best_restart);
  for (int i = 0; i < 6; ++i) REQUIRE(a.per_restart[i].coherence == c.per_restart[i].coherence);
}

TEST(solve_reaches_known_optimum_2_4) {  // test_solver.cpp:134-149
  SolverConfig cfg;
  cfg.shape = cshape(2, 4);
  cfg.restarts = 5;
  cfg.seed = 7;
  SolveResult r = solve(cfg, 4);
  REQUIRE(r.best_coherence <= 0.5774 + 1e-3);
  CoherenceResult c = coherence(cfg.shape, r.best_frame.data(), false);
  REQUIRE(r.best_coherence == c.mu);
}

TEST(solve_never_beats_welch) {  // test_solver.cpp:151-163
  for (auto [d, n] : {std::pair<int, int>{2, 5}, {3, 7}}) {
    SolverConfig cfg;
    cfg.shape = cshape(d, n);
    cfg.seed = 5;
    cfg.restarts = 2;
    cfg.eps_target = 1e-5;
    SolveResult r = solve(cfg, 2);
    REQUIRE(r.best_coherence >= welch_bound(d, n) - 1e-9);
  }
}

TEST(orthonormal_bases_recovered_for_N_eq_d) {  // test_solver.cpp:165-176
  for (int d : {2, 3, 5, 8}) {
    SolverConfig cfg;
    cfg.shape = cshape(d, d, d * d * 2 > 64 ? 128 : 32);
    cfg.restarts = 5;
    cfg.seed = 11;
    cfg.eps_target = 1e-6;
    REQUIRE(solve(cfg, 5).best_coherence <= 1e-6);
  }
}

TEST(optimized_2_5_is_near_1_over_sqrt2) {  // test_solver.cpp:199-210
  SolverConfig cfg;
  cfg.shape = cshape(2, 5);
  cfg.restarts = 6;
  cfg.seed = 123;
  SolveResult r = solve(cfg, 6);
  REQUIRE(std::abs(r.best_coherence - 1.0 / std::sqrt(2.0)) <= 2e-3);
}

TEST(hvp_one_sided_fallback_at_zero_threshold) {  // test_solver.cpp:212-230
  Shape sh = cshape(1, 2);
  Vec point = {1e-3, 0.0, 1.0, 0.0}, dir = {-1.0, 0.0, 0.0, 0.0};
  for (int i = 0; i < 3; ++i) point[0] = kFdBaseStep * (1.0 + nrm(point)) / nrm(dir);
  HvpResult r = hvp_adapter(sh, point, dir, 1e-1, nullptr);
  REQUIRE(r.path == HVP_FORWARD || r.path == HVP_BACKWARD);
  for (double v : r.hv) REQUIRE(std::isfinite(v));
}

TEST(collapsed_column_redrawn_at_stage_boundary) {  // test_solver.cpp:232-250
  SolverConfig cfg;
  cfg.shape = cshape(2, 3);
  cfg.eps_target = 1e-4;
  Vec start = {1, 0, 0, 0, 0, 0, 1, 0, 0, 0, 0, 0};
  Rng rng(8);
  AnnealResult a = anneal(start, cfg, &rng);
  REQUIRE(a.stages.size() >= 2);
  for (int j = 0; j < 3; ++j) REQUIRE(std::abs(column_norm(&a.frame[4 * j], 4) - 1.0) <= 1e-10);
  bool threw = false;
  try {
    anneal(start, cfg, nullptr);
  } catch (const ZeroColumnFailure& e) {
    threw = e.column == 2;
  }
  REQUIRE(threw);
}

TEST(stage_coherence_non_increasing_in_practice) {  // test_solver.cpp:252-272
  int total = 0, viol = 0;
  for (std::uint64_t seed = 0; seed < 5; ++seed) {
    SolverConfig cfg;
    cfg.shape = cshape(3, 6);
    cfg.restarts = 1;
    cfg.seed = seed;
    cfg.eps_target = 1e-6;
    SolveResult r = solve(cfg, 1);
    const auto& st = r.per_restart[0].stages;
    for (size_t k = 0; k + 1 < st.size(); ++k) {
      ++total;
      if (st[k + 1].coherence > st[k].coherence + 1e-6) ++viol;
    }
  }
  REQUIRE(viol * 20 <= total);
}

// ------------------------------------------------------------ test_frames.cpp
TEST(sic_frames_have_equal_magnitudes) {  // test_frames.cpp:71-81, test_analysis.cpp:24-34
  Shape s24 = cshape(2, 4);
  Vec f = sic_2_4();
  CoherenceResult c = coherence(s24, f.data(), false);
  REQUIRE(std::abs(c.mu - 1.0 / std::sqrt(3.0)) <= 1e-12);
  for (int j = 0; j < 4; ++j)
    for (int k = j + 1; k < 4; ++k) {
      double gr, gi;
      gram_entry(s24, &f[4 * j], &f[4 * k], &gr, &gi);
      REQUIRE(std::abs(std::sqrt(gr * gr + gi * gi) - 1.0 / std::sqrt(3.0)) <= 1e-12);
    }
  Shape s39 = cshape(3, 9);
  Vec g = sic_3_9();
  REQUIRE(std::abs(coherence(s39, g.data(), false).mu - 0.5) <= 1e-12);
}

TEST(coherence_invariant_under_phase_and_permutation) {  // test_frames.cpp:110-134 (unitary part: test_gpu_*)
  Rng rng(314159);
  for (int trial = 0; trial < 8; ++trial) {
    const int d = 2 + trial % 3, n = d + 2 + trial % 4;
    Shape sh = cshape(d, n);
    Vec f = random_frame(sh, rng);
    const double mu = coherence(sh, f.data(), false).mu;
    REQUIRE(mu >= 0.0 && mu <= 1.0);
    Vec ph = f;
    for (int j = 0; j < n; ++j) {
      const std::complex<double> e = std::polar(1.0, 6.28 * rng.uniform());
      for (int i = 0; i < d; ++i) {
        const std::complex<double> v = e * std::complex<double>(f[2 * (i + d * j)], f[2 * (i + d * j) + 1]);
        ph[2 * (i + d * j)] = v.real();
        ph[2 * (i + d * j) + 1] = v.imag();
      }
    }
    REQUIRE(std::abs(coherence(sh, ph.data(), false).mu - mu) < 1e-12);
    Vec pm = f;
    for (int q = 0; q < 2 * d; ++q) std::swap(pm[q], pm[2 * d * (n - 1) + q]);
    REQUIRE(std::abs(coherence(sh, pm.data(), false).mu - mu) < 1e-12);
  }
}

TEST(coherence_zero_for_orthonormal_basis) {  // test_frames.cpp:136-141
  Vec id(50, 0.0);
  for (int j = 0; j < 5; ++j) id[2 * (j + 5 * j)] = 1.0;
  REQUIRE(coherence(cshape(5, 5), id.data(), false).mu == 0.0);
}

TEST(normalize_reports_first_zero_column) {  // test_frames.cpp:39-49
  Vec f(18, 0.0);
  f[0] = 1.0;
  REQUIRE(coherence(cshape(3, 3), f.data(), true).zero_col == 1);
}

TEST(gram_bit_identical_across_calls) {  // test_frames.cpp:157-163
  Shape sh = cshape(4, 9);
  Rng rng(4242);
  Vec f = random_frame(sh, rng);
  CoherenceResult a = coherence(sh, f.data(), false), b = coherence(sh, f.data(), false);
  REQUIRE(a.mu == b.mu && a.argmax == b.argmax);
}

// -------------------------------------------------------- acceptance_main.cpp
TEST(acceptance_criterion_1_known_optima) {  // acceptance_main.cpp:62-87 (kSeed 20250809, 20 restarts)
  struct Case {
    int d, n;
    double target, slack;
  };
  for (Case c : {Case{2, 4, 0.5774, 1e-3}, Case{3, 9, 0.5001, 1e-3}}) {
    SolverConfig cfg;
    cfg.shape = cshape(c.d, c.n, 2 * c.d * c.n > 64 ? 128 : 32);
    cfg.restarts = 20;
    cfg.seed = 20250809;
    cfg.eps_target = 1e-7;
    SolveResult r = solve(cfg, 8);
    REQUIRE(r.best_coherence <= c.target + c.slack);
  }
}

TEST(acceptance_criterion_7_lse_random_instances) {  // acceptance_main.cpp:171-192
  Rng rng(20250809);
  for (int inst = 0; inst < 1000; ++inst) {
    const int n = 2 + static_cast<int>(rng.uniform() * 30);
    Vec x(n);
    for (double& v : x) v = rng.uniform();
    const double delta = std::pow(10.0, -1.0 - 4.0 * rng.uniform());
    const double f = smooth_max(x, delta);
    double s = x[0];
    for (double v : x) s = std::max(s, v);
    REQUIRE(s <= f + 1e-15 && f <= s + delta * std::log(static_cast<double>(n)) + 1e-15);
    Vec w = lse_partials(x, delta);
    double sum = 0.0;
    for (double v : w) sum += v;
    REQUIRE(std::abs(sum - 1.0) < 1e-12);
  }
}

int main(int argc, char** argv) {
  const std::string only = argc > 1 ? argv[1] : "";
  int n = 0;
  for (auto& [name, fn] : TestReg::all()) {
    if (!only.empty() && name.find(only) == std::string::npos) continue;
    g_test = name;
    const int before = g_fail;
    try {
      fn();
    } catch (const std::exception& e) {
      ++g_fail;
      std::printf("FAIL [%s] exception: %s\n", name.c_str(), e.what());
    }
    std::printf("%s %s\n", g_fail == before ? "ok  " : "FAIL", name.c_str());
    ++n;
  }
  std::printf("%d tests, %d checks, %d failures\n", n, g_checks, g_fail);
  return g_fail ? 1 : 0;
}
