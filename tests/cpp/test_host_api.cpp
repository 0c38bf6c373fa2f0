// The reference's hot-path unit tests (proj/tests/test_smoothing.cpp,
// test_trust_region.cpp, test_solver.cpp) re-run against the C++ host mirror
// of the B200 path (paper_2207_06374_b200/csrc/host/trstmi_host.hpp): same
// inputs, same assertions, same tolerances, GPU underneath.
#include <cmath>
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

#include "../../paper_2207_06374_b200/csrc/host/trstmi_host.hpp"

using namespace trstmi::b200;

static int g_fail = 0, g_checks = 0;
static std::string g_test;
#define REQUIRE(c)                                                                       \
  do {                                                                                   \
    ++g_checks;                                                                          \
    if (!(c)) {                                                                          \
      ++g_fail;                                                                          \
      std::printf("FAIL [%s] %s:%d: %s\n", g_test.c_str(), __FILE__, __LINE__, #c);     \
    }                                                                                    \
  } while (0)
#define REQUIRE_THROWS_AS(expr, T) \
  do {                             \
    bool ok_ = false;              \
    try {                          \
      (void)(expr);                \
    } catch (const T&) {           \
      ok_ = true;                  \
    }                              \
    REQUIRE(ok_);                  \
  } while (0)

static std::vector<std::pair<std::string, std::function<void()>>>& reg() {
  static std::vector<std::pair<std::string, std::function<void()>>> v;
  return v;
}
struct Reg {
  Reg(const char* n, std::function<void()> f) { reg().emplace_back(n, f); }
};
#define TEST(name)                   \
  static void name();                \
  static Reg r_##name(#name, name);  \
  static void name()

static VectorXd frame_of(Index d, Index N, std::uint64_t seed, Field f = Field::complex_field) {
  const Index dim = (f == Field::complex_field ? 2 : 1) * d * N;
  VectorXd x(dim);
  trstmi_random_frames((int)f, d, N, seed, 0, 1, x.data(), nullptr);
  return x;
}

TEST(orthogonal_pair_gives_objective_zero) {  // test_smoothing.cpp:16-25
  VectorXd id = {1, 0, 0, 0, 0, 0, 1, 0};
  for (double delta : {1.0, 1e-2, 1e-6}) {
    ObjectiveEval e = eval_objective(id, SmoothObjective{delta, 2, 2, true});
    REQUIRE(e.s == 0.0);
    REQUIRE(e.value == 0.0);
  }
}

TEST(coincident_pair_gives_objective_one) {  // test_smoothing.cpp:27-34
  ObjectiveEval e = eval_objective({1, 0, 0, 0, 1, 0, 0, 0}, SmoothObjective{0.1, 2, 2, true});
  REQUIRE(std::abs(e.value - 1.0) <= 1e-15);
}

TEST(sandwich_property_on_random_frames) {  // test_smoothing.cpp:36-46
  for (std::uint64_t seed = 1; seed <= 20; ++seed) {
    SmoothObjective obj{1e-3, 3, 6, true};
    ObjectiveEval e = eval_objective(frame_of(3, 6, seed), obj);
    REQUIRE(e.s <= e.value);
    REQUIRE(e.value <= e.s + obj.delta * std::log((double)obj.pair_count()));
    double sum = 0.0;
    for (double w : e.softmax_weights) sum += w;
    REQUIRE(std::abs(sum - 1.0) < 1e-12);
  }
}

TEST(analytic_gradient_matches_central_fd) {  // test_smoothing.cpp:108-123 (support.hpp:83-108)
  const std::pair<Index, Index> sizes[] = {{2, 4}, {3, 6}, {4, 10}};
  std::uint64_t seed = 100;
  for (auto [d, n] : sizes)
    for (double delta : {1e-1, 1e-3})
      for (int rep = 0; rep < 4; ++rep) {
        SmoothObjective obj{delta, d, n, true};
        VectorXd p = frame_of(d, n, ++seed);
        VectorXd a = eval_objective(p, obj).grad;
        double worst = 0.0;
        for (size_t i = 0; i < p.size(); ++i) {
          const double h = 5e-8 * (1.0 + std::abs(p[i]));
          VectorXd q = p;
          q[i] = p[i] + h;
          const double fp = eval_objective(q, obj).value;
          q[i] = p[i] - h;
          const double fm = eval_objective(q, obj).value;
          const double fd = (fp - fm) / (2.0 * h);
          worst = std::max(worst, std::abs(a[i] - fd) / std::max({1.0, std::abs(a[i]), std::abs(fd)}));
        }
        REQUIRE(worst <= 1e-5);
      }
}

TEST(gradient_zero_along_column_rescaling) {  // test_smoothing.cpp:134-146
  VectorXd p = frame_of(3, 4, 2024);
  VectorXd g = eval_objective(p, SmoothObjective{1e-2, 3, 4, true}).grad;
  for (int j = 0; j < 4; ++j) {
    double dot = 0.0;
    for (int q = 0; q < 6; ++q) dot += g[6 * j + q] * p[6 * j + q];
    REQUIRE(std::abs(dot) < 1e-12);
  }
}

TEST(zero_column_propagates_from_evaluation) {  // test_smoothing.cpp:148-153
  VectorXd p(8, 0.0);
  p[0] = 1.0;
  REQUIRE_THROWS_AS(eval_objective(p, SmoothObjective{0.1, 2, 2, true}), ZeroColumnError);
}

TEST(hvp_zero_direction_and_symmetry) {  // test_smoothing.cpp:155-162, 184-197
  VectorXd p = frame_of(2, 4, 8);
  VectorXd hv = hessian_vector_product(p, VectorXd(p.size(), 0.0), SmoothObjective{1e-2, 2, 4, true});
  REQUIRE(vec::norm(hv) == 0.0);
  VectorXd q = frame_of(3, 6, 55);
  VectorXd v = frame_of(3, 6, 56), w = frame_of(3, 6, 57);
  SmoothObjective obj{1e-2, 3, 6, true};
  const double hvw = vec::dot(hessian_vector_product(q, v, obj), w);
  const double hwv = vec::dot(hessian_vector_product(q, w, obj), v);
  REQUIRE(std::abs(hvw - hwv) <= 1e-4 * std::max(std::abs(hvw), std::abs(hwv)));
}

TEST(minimize_quadratic_and_rosenbrock) {  // test_trust_region.cpp:110-152
  Objective quad = [](const VectorXd& x) {
    VectorXd g(x.size());
    double v = 0.0;
    for (size_t i = 0; i < x.size(); ++i) {
      v += x[i] * x[i];
      g[i] = 2.0 * x[i];
    }
    return Evaluation{v, g};
  };
  HvpFactory fq = [](const VectorXd&) -> HvpOperator {
    return [](const VectorXd& v) {
      VectorXd o(v.size());
      for (size_t i = 0; i < v.size(); ++i) o[i] = 2.0 * v[i];
      return o;
    };
  };
  VectorXd x0(10);
  for (int i = 0; i < 10; ++i) x0[i] = 0.1 * (i - 4.5);
  MinimizeResult r = trust_region_minimize(quad, fq, x0, TrustRegionConfig{});
  REQUIRE(r.status == MinimizeStatus::gradient_tolerance);
  REQUIRE(r.history.size() <= 10);
  Objective rb = [](const VectorXd& x) {
    const double a = 1.0 - x[0], b = x[1] - x[0] * x[0];
    return Evaluation{a * a + 100.0 * b * b, {-2.0 * a - 400.0 * x[0] * b, 200.0 * b}};
  };
  HvpFactory fr = [&rb](const VectorXd& x) -> HvpOperator {
    return [&rb, x](const VectorXd& dir) {
      const double h = 0x1.965fea53d6e3dp-18 * (1.0 + vec::norm(x)) / std::max(vec::norm(dir), 1e-300);
      VectorXd p = x, m = x, o(x.size());
      for (size_t i = 0; i < x.size(); ++i) {
        p[i] += h * dir[i];
        m[i] -= h * dir[i];
      }
      VectorXd gp = rb(p).grad, gm = rb(m).grad;
      for (size_t i = 0; i < x.size(); ++i) o[i] = (gp[i] - gm[i]) / (2.0 * h);
      return o;
    };
  };
  TrustRegionConfig cfg;
  cfg.grad_tol = 1e-8;
  cfg.max_outer = 500;
  MinimizeResult s = trust_region_minimize(rb, fr, {-1.2, 1.0}, cfg);
  REQUIRE(s.value < 1e-8);
  REQUIRE(std::abs(s.x[0] - 1.0) <= 1e-4 && std::abs(s.x[1] - 1.0) <= 1e-4);
}

TEST(minimize_frame_objective_through_gpu_plugin) {  // the reference seam, solver.hpp:189-191
  SmoothObjective obj{1e-2, 2, 6, true};
  VectorXd x0 = frame_of(2, 6, 3);
  TrustRegionConfig cfg;
  cfg.max_outer = 40;
  MinimizeResult r = trust_region_minimize(detail::make_objective(obj), detail::make_hvp_factory(obj), x0, cfg);
  double last = 1e300;
  for (const OuterRecord& rec : r.history) {
    if (!rec.accepted) continue;
    REQUIRE(rec.value <= last + 1e-15);
    last = rec.value;
  }
  REQUIRE(r.value < eval_objective(x0, obj).value);
}

TEST(config_invariants_are_validated) {  // test_trust_region.cpp:224-236
  Objective f = [](const VectorXd& x) { return Evaluation{0.0, VectorXd(x.size(), 0.0)}; };
  HvpFactory h = [](const VectorXd&) -> HvpOperator { return [](const VectorXd& v) { return v; }; };
  TrustRegionConfig bad;
  bad.eta = 0.3;
  REQUIRE_THROWS_AS(trust_region_minimize(f, h, VectorXd(2, 1.0), bad), std::invalid_argument);
}

TEST(default_schedule_values) {  // test_solver.cpp:12-40
  std::vector<double> s = default_delta_schedule(100, 1e-6);
  REQUIRE(std::abs(s.front() - 1e-1) <= 1e-12);
  REQUIRE(std::abs(s.back() - 1.0857e-7) <= 1e-3 * 1.0857e-7);
  for (Index n = 2; n <= 100; ++n) {
    const double t = default_delta_schedule(n, 1e-7).back();
    REQUIRE(t >= 1e-8 && t <= 1e-7);
  }
}

TEST(anneal_finds_orthogonal_pair) {  // test_solver.cpp:73-84
  SolverConfig cfg;
  cfg.d = 2;
  cfg.N = 2;
  cfg.eps_target = 1e-6;
  Frame start{2, 2, Field::complex_field, frame_of(2, 2, 1)};
  std::uint64_t rng[3] = {1, 0, 0};
  auto [frame, stages] = anneal(start, cfg, rng);
  REQUIRE(coherence(frame) <= 1e-6);
  REQUIRE(stages.size() >= 2);
}

TEST(anneal_rejects_mismatched_start) {  // test_solver.cpp:86-93
  SolverConfig cfg;
  cfg.d = 2;
  cfg.N = 3;
  Frame start{2, 2, Field::complex_field, frame_of(2, 2, 1)};
  REQUIRE_THROWS_AS(anneal(start, cfg), DimensionMismatchError);
}

TEST(solve_deterministic) {  // test_solver.cpp:112-132
  SolverConfig cfg;
  cfg.d = 2;
  cfg.N = 4;
  cfg.restarts = 6;
  cfg.seed = 31337;
  cfg.eps_target = 1e-6;
  SolveResult a = solve(cfg, 1), b = solve(cfg, 4);
  REQUIRE(a.best_frame.packed == b.best_frame.packed);
  REQUIRE(a.best_coherence == b.best_coherence && a.best_restart == b.best_restart);
  for (int i = 0; i < 6; ++i) REQUIRE(a.per_restart[i].coherence == b.per_restart[i].coherence);
}

TEST(solve_reaches_known_optimum_2_4) {  // test_solver.cpp:134-149
  SolverConfig cfg;
  cfg.d = 2;
  cfg.N = 4;
  cfg.restarts = 5;
  cfg.seed = 7;
  SolveResult r = solve(cfg);
  REQUIRE(r.best_coherence <= 0.5774 + 1e-3);
  REQUIRE(r.best_coherence == coherence(r.best_frame));
  double mn = 1e9;
  for (const RestartRecord& rr : r.per_restart) {
    REQUIRE(rr.succeeded);
    mn = std::min(mn, rr.coherence);
  }
  REQUIRE(r.best_coherence == mn);
}

TEST(solve_never_beats_welch_and_onb) {  // test_solver.cpp:151-176
  for (auto [d, n] : {std::pair<Index, Index>{2, 5}, {3, 7}}) {
    SolverConfig cfg;
    cfg.d = d;
    cfg.N = n;
    cfg.seed = 5;
    cfg.restarts = 2;
    cfg.eps_target = 1e-5;
    REQUIRE(solve(cfg).best_coherence >= welch_bound(d, n) - 1e-9);
  }
  for (Index d : {2, 3, 5, 8}) {
    SolverConfig cfg;
    cfg.d = d;
    cfg.N = d;
    cfg.restarts = 5;
    cfg.seed = 11;
    cfg.eps_target = 1e-6;
    REQUIRE(solve(cfg).best_coherence <= 1e-6);
  }
}

TEST(optimized_2_5_near_inverse_sqrt2) {  // test_solver.cpp:199-210
  SolverConfig cfg;
  cfg.d = 2;
  cfg.N = 5;
  cfg.restarts = 6;
  cfg.seed = 123;
  REQUIRE(std::abs(solve(cfg).best_coherence - 1.0 / std::sqrt(2.0)) <= 2e-3);
}

TEST(collapsed_column_redrawn_at_stage_boundary) {  // test_solver.cpp:232-250
  SolverConfig cfg;
  cfg.d = 2;
  cfg.N = 3;
  cfg.eps_target = 1e-4;
  Frame start{2, 3, Field::complex_field, {1, 0, 0, 0, 0, 0, 1, 0, 0, 0, 0, 0}};
  std::uint64_t rng[3] = {8, 0, 0};
  auto [frame, stages] = anneal(start, cfg, rng);
  REQUIRE(stages.size() >= 2);
  REQUIRE_THROWS_AS(anneal(start, cfg), ZeroColumnError);
}

int main() {
  int n = 0;
  for (auto& [name, fn] : reg()) {
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
