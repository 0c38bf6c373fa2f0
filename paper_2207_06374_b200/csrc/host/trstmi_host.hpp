// C++ host mirror of the reference library's solver/objective interface
// (/root/reference/proj/include/trstmi/{frame,smoothing,trust_region,solver}.hpp)
// over the B200 C ABI (include/trstmi_b200.h).  Same names, argument meaning
// and exceptions as the reference, Eigen-free value types:
//
//   trstmi::b200::eval_objective            <- smoothing.hpp:82-162   (GPU)
//   trstmi::b200::hessian_vector_product    <- smoothing.hpp:187-194  (GPU)
//   trstmi::b200::detail::make_objective    <- solver.hpp:104-114     (GPU-backed Objective)
//   trstmi::b200::detail::make_hvp_factory  <- solver.hpp:118-137     (GPU-backed HvpFactory)
//   trstmi::b200::steihaug_cg / trust_region_minimize <- trust_region.hpp:81-295
//        (generic plugin host: any Objective/HvpFactory, as in the reference)
//   trstmi::b200::anneal / solve            <- solver.hpp:164-273     (batched GPU anneal)
//   trstmi::b200::coherence / normalize_columns / welch_bound / default_delta_schedule
//
// Header-only; link with paper_2207_06374_b200/_lib/libtrstmi_b200.so.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <functional>
#include <limits>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../../../include/trstmi_b200.h"

namespace trstmi {
namespace b200 {

using Index = std::int64_t;
using VectorXd = std::vector<double>;

inline constexpr double kZeroColumnTol = 1e-12;

struct ZeroColumnError : std::runtime_error {  // frame.hpp:25-31
  explicit ZeroColumnError(Index column_index)
      : std::runtime_error("column " + std::to_string(column_index) + " has near-zero norm"), column(column_index) {}
  Index column;
};
struct DimensionMismatchError : std::invalid_argument {  // frame.hpp:33-35
  using std::invalid_argument::invalid_argument;
};
struct SolveError : std::runtime_error {  // solver.hpp:56-58
  using std::runtime_error::runtime_error;
};
struct DeviceError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

enum class Field { complex_field = TRSTMI_COMPLEX, real_field = TRSTMI_REAL };

// Frame (frame.hpp:41-49) in its packed form (frame.hpp:165-186): column-major
// d x N, complex entries interleaved (re, im).
struct Frame {
  Index d = 0, N = 0;
  Field field = Field::complex_field;
  VectorXd packed;
  Index dim() const { return d; }
  Index count() const { return N; }
};

// One device context per process by default (a ctx is used by one host thread).
class Context {
 public:
  explicit Context(int device = 0) {
    trstmi_ctx* c = nullptr;
    const int rc = trstmi_ctx_create(device, &c);
    if (rc != TRSTMI_OK) throw DeviceError("trstmi_ctx_create failed (" + std::to_string(rc) + "): no CPU fallback");
    ctx_.reset(c);
  }
  trstmi_ctx* get() const { return ctx_.get(); }
  static Context& instance() {
    static Context c(0);
    return c;
  }

 private:
  struct Del {
    void operator()(trstmi_ctx* c) const { trstmi_ctx_destroy(c); }
  };
  std::unique_ptr<trstmi_ctx, Del> ctx_;
};

inline void check(trstmi_ctx* ctx, int rc) {
  if (rc == TRSTMI_OK) return;
  const std::string msg = trstmi_last_error(ctx);
  switch (rc) {
    case TRSTMI_ERR_INVALID_ARG: throw std::invalid_argument(msg);
    case TRSTMI_ERR_DIM_MISMATCH: throw DimensionMismatchError(msg);
    case TRSTMI_ERR_ALL_FAILED: throw SolveError(msg);
    default: throw DeviceError(msg + " (code " + std::to_string(rc) + ")");
  }
}

// ------------------------------------------------------------------ objective
struct SmoothObjective {  // smoothing.hpp:27-34 (+ field, new)
  double delta = 1e-2;
  Index d = 0;
  Index N = 0;
  bool squared = true;
  Field field = Field::complex_field;
  Index pair_count() const { return N * (N - 1) / 2; }
  Index point_size() const { return (field == Field::complex_field ? 2 : 1) * d * N; }
};

struct ObjectiveEval {  // smoothing.hpp:36-41
  double value = 0.0;
  double s = 0.0;
  VectorXd grad;
  VectorXd softmax_weights;
};

inline ObjectiveEval eval_objective(const VectorXd& point, const SmoothObjective& obj,
                                    Context& ctx = Context::instance()) {
  if (obj.delta <= 0.0) throw std::invalid_argument("eval_objective: delta <= 0");
  if (obj.N < 2) throw std::invalid_argument("eval_objective: need N >= 2");
  if ((Index)point.size() != obj.point_size()) throw DimensionMismatchError("eval_objective: point length mismatch");
  ObjectiveEval e;
  e.grad.resize(point.size());
  e.softmax_weights.resize(obj.pair_count());
  std::int64_t zc = -1;
  check(ctx.get(), trstmi_eval_batch(ctx.get(), (int)obj.field, obj.d, obj.N, 1, point.data(), &obj.delta,
                                     obj.squared ? 1 : 0, &e.value, &e.s, e.grad.data(), e.softmax_weights.data(),
                                     &zc));
  if (zc >= 0) throw ZeroColumnError(zc);
  return e;
}

inline VectorXd hessian_vector_product(const VectorXd& point, const VectorXd& direction, const SmoothObjective& obj,
                                       Context& ctx = Context::instance()) {
  if (direction.size() != point.size()) throw DimensionMismatchError("fd_hessian_vector_product: length mismatch");
  VectorXd hv(point.size());
  std::int32_t path = 0;
  std::int64_t zc = -1;
  check(ctx.get(), trstmi_hvp_batch(ctx.get(), (int)obj.field, obj.d, obj.N, 1, point.data(), direction.data(),
                                    &obj.delta, hv.data(), &path, &zc));
  if (path == TRSTMI_HVP_FORWARD || path == TRSTMI_HVP_BACKWARD || path == TRSTMI_HVP_FAILED)
    throw ZeroColumnError(zc);  // the plain central difference threw
  return hv;
}

// ------------------------------------------------------------- trust region
struct TrustRegionConfig {  // trust_region.hpp:20-30
  double delta0 = 0.0;
  double delta_max = 1e3;
  double eta = 0.05;
  double shrink = 0.25;
  double grow = 2.0;
  double grad_tol = 1e-9;
  int max_outer = 200;
  double cg_force_c = 0.5;
  int max_cg = 0;
};

enum class CgExit { small_residual, negative_curvature, boundary_hit, zero_gradient };
struct CgTrace {
  int iterations = 0;
  CgExit exit_reason = CgExit::small_residual;
  double step_norm = 0.0;
  bool converged = true;
  double model_value = 0.0;
};
struct Evaluation {
  double value = 0.0;
  VectorXd grad;
};
using Objective = std::function<Evaluation(const VectorXd&)>;  // trust_region.hpp:42-49
using HvpOperator = std::function<VectorXd(const VectorXd&)>;
using HvpFactory = std::function<HvpOperator(const VectorXd&)>;

enum class MinimizeStatus { gradient_tolerance, iteration_limit, radius_underflow, stalled };
struct OuterRecord {
  int iteration = 0;
  double value = 0.0, grad_norm = 0.0, radius = 0.0, rho = 0.0;
  bool accepted = false;
  CgExit cg_exit = CgExit::small_residual;
  int cg_iterations = 0;
  double step_norm = 0.0;
};
struct MinimizeResult {
  VectorXd x;
  double value = 0.0, grad_norm = 0.0;
  MinimizeStatus status = MinimizeStatus::iteration_limit;
  std::vector<OuterRecord> history;
};

namespace vec {
inline double dot(const VectorXd& a, const VectorXd& b) {
  double s = 0.0;
  for (size_t i = 0; i < a.size(); ++i) s = std::fma(a[i], b[i], s);
  return s;
}
inline double norm(const VectorXd& a) { return std::sqrt(dot(a, a)); }
inline bool all_finite(const VectorXd& a) {
  for (double v : a)
    if (!std::isfinite(v)) return false;
  return true;
}
}  // namespace vec

namespace detail {
inline std::pair<double, double> boundary_roots(const VectorXd& z, const VectorXd& d, double radius) {
  const double a = vec::dot(d, d);
  const double b = 2.0 * vec::dot(z, d);
  const double c = vec::dot(z, z) - radius * radius;
  if (a <= 0.0) return {0.0, 0.0};
  const double disc = std::sqrt(std::max(b * b - 4.0 * a * c, 0.0));
  const double q = -0.5 * (b + std::copysign(disc, b));
  double r1 = q != 0.0 ? c / q : 0.0;
  double r2 = a != 0.0 ? q / a : 0.0;
  if (r1 > r2) std::swap(r1, r2);
  return {r1, r2};
}
}  // namespace detail

// Generic Steihaug-CG / trust-region host loop for the reference's plugin
// seam (any Objective/HvpFactory, trust_region.hpp:81-295).  The frame
// objective's hot path runs the same algorithm entirely on the GPU (anneal).
inline std::pair<VectorXd, CgTrace> steihaug_cg(const VectorXd& grad, const HvpOperator& hvp, double radius,
                                                double eps_k, int max_cg) {
  if (radius <= 0.0) throw std::invalid_argument("steihaug_cg: radius <= 0");
  if (eps_k < 0.0) throw std::invalid_argument("steihaug_cg: eps_k < 0");
  const size_t n = grad.size();
  VectorXd z(n, 0.0);
  CgTrace tr;
  const double gn = vec::norm(grad);
  if (gn < eps_k || gn == 0.0) {
    tr.exit_reason = CgExit::zero_gradient;
    return {z, tr};
  }
  VectorXd r = grad, d(n);
  for (size_t i = 0; i < n; ++i) d[i] = -grad[i];
  double rr = vec::dot(r, r), model = 0.0;
  VectorXd zn(n);
  for (int j = 0; j < max_cg; ++j) {
    const VectorXd bd = hvp(d);
    const double dbd = vec::dot(d, bd), rd = vec::dot(r, d);
    if (dbd <= 0.0) {
      const auto [lo, hi] = detail::boundary_roots(z, d, radius);
      const double m_lo = model + lo * rd + 0.5 * lo * lo * dbd;
      const double m_hi = model + hi * rd + 0.5 * hi * hi * dbd;
      const double tau = m_lo < m_hi ? lo : hi;
      for (size_t i = 0; i < n; ++i) z[i] = z[i] + tau * d[i];
      tr.iterations = j;
      tr.exit_reason = CgExit::negative_curvature;
      tr.step_norm = vec::norm(z);
      tr.model_value = std::min(m_lo, m_hi);
      return {z, tr};
    }
    const double alpha = rr / dbd;
    for (size_t i = 0; i < n; ++i) zn[i] = z[i] + alpha * d[i];
    if (vec::norm(zn) >= radius) {
      const double tau = detail::boundary_roots(z, d, radius).second;
      for (size_t i = 0; i < n; ++i) z[i] = z[i] + tau * d[i];
      tr.iterations = j;
      tr.exit_reason = CgExit::boundary_hit;
      tr.step_norm = vec::norm(z);
      tr.model_value = model + tau * rd + 0.5 * tau * tau * dbd;
      return {z, tr};
    }
    model += alpha * rd + 0.5 * alpha * alpha * dbd;
    z = zn;
    for (size_t i = 0; i < n; ++i) r[i] = r[i] + alpha * bd[i];
    const double rr_next = vec::dot(r, r);
    tr.iterations = j + 1;
    if (std::sqrt(rr_next) < eps_k) {
      tr.exit_reason = CgExit::small_residual;
      tr.step_norm = vec::norm(z);
      tr.model_value = model;
      return {z, tr};
    }
    const double beta = rr_next / rr;
    rr = rr_next;
    for (size_t i = 0; i < n; ++i) d[i] = -r[i] + beta * d[i];
  }
  tr.exit_reason = CgExit::small_residual;
  tr.converged = false;
  tr.step_norm = vec::norm(z);
  tr.model_value = model;
  return {z, tr};
}

inline MinimizeResult trust_region_minimize(const Objective& objective, const HvpFactory& make_hvp, VectorXd x0,
                                            TrustRegionConfig cfg) {
  const size_t dim = x0.size();
  if (cfg.delta0 == 0.0) cfg.delta0 = 0.1 * std::sqrt(static_cast<double>(dim));
  if (cfg.max_cg == 0) cfg.max_cg = static_cast<int>(2 * dim);
  if (!(cfg.delta0 > 0.0) || cfg.delta0 > cfg.delta_max)
    throw std::invalid_argument("trust_region_minimize: need 0 < delta0 <= delta_max");
  if (!(cfg.eta >= 0.0 && cfg.eta < 0.25)) throw std::invalid_argument("trust_region_minimize: need 0 <= eta < 1/4");
  if (!(cfg.shrink > 0.0 && cfg.shrink < 1.0 && cfg.grow > 1.0))
    throw std::invalid_argument("trust_region_minimize: need 0 < shrink < 1 < grow");
  Evaluation cur = objective(x0);
  if (!std::isfinite(cur.value) || !vec::all_finite(cur.grad))
    throw std::invalid_argument("trust_region_minimize: objective not finite at x0");
  MinimizeResult res;
  res.x = x0;
  res.value = cur.value;
  res.grad_norm = vec::norm(cur.grad);
  VectorXd x = std::move(x0), trial(dim);
  double radius = cfg.delta0;
  for (int iter = 0; iter < cfg.max_outer; ++iter) {
    const double gn = vec::norm(cur.grad);
    if (gn <= cfg.grad_tol) {
      res.status = MinimizeStatus::gradient_tolerance;
      break;
    }
    const double eps_k = std::min(cfg.cg_force_c, std::sqrt(gn)) * gn;
    auto [step, tr] = steihaug_cg(cur.grad, make_hvp(x), radius, eps_k, cfg.max_cg);
    OuterRecord rec;
    rec.iteration = iter;
    rec.value = cur.value;
    rec.grad_norm = gn;
    rec.radius = radius;
    rec.cg_exit = tr.exit_reason;
    rec.cg_iterations = tr.iterations;
    rec.step_norm = tr.step_norm;
    const double predicted = -tr.model_value;
    if (tr.exit_reason == CgExit::zero_gradient || predicted <= 0.0) {
      radius *= cfg.shrink;
      res.history.push_back(rec);
      if (radius < 1e-16) {
        res.status = MinimizeStatus::radius_underflow;
        break;
      }
      continue;
    }
    for (size_t i = 0; i < dim; ++i) trial[i] = x[i] + step[i];
    Evaluation te = objective(trial);
    const bool finite = std::isfinite(te.value) && vec::all_finite(te.grad);
    const double rho = finite ? (cur.value - te.value) / predicted : -std::numeric_limits<double>::infinity();
    rec.rho = rho;
    if (finite && te.value < res.value) {
      res.x = trial;
      res.value = te.value;
      res.grad_norm = vec::norm(te.grad);
    }
    if (rho > cfg.eta) {
      x = trial;
      cur = std::move(te);
      rec.accepted = true;
    }
    if (rho < 0.25) radius *= cfg.shrink;
    else if (rho > 0.75 && tr.step_norm >= (1.0 - 1e-10) * radius) radius = std::min(cfg.grow * radius, cfg.delta_max);
    res.history.push_back(rec);
    if (radius < 1e-16) {
      res.status = MinimizeStatus::radius_underflow;
      break;
    }
  }
  if (cur.value < res.value) {
    res.x = x;
    res.value = cur.value;
    res.grad_norm = vec::norm(cur.grad);
  }
  return res;
}

// ------------------------------------------------------------------ solver
struct SolverConfig {  // solver.hpp:21-29 (+ field)
  Index d = 0;
  Index N = 0;
  std::vector<double> delta_schedule;
  int restarts = 20;
  std::uint64_t seed = 0;
  TrustRegionConfig tr;
  double eps_target = 1e-7;
  Field field = Field::complex_field;
};
struct StageRecord {  // solver.hpp:31-36
  double delta = 0.0, objective = 0.0, coherence = 0.0;
  int outer_iterations = 0;
};
struct RestartRecord {  // solver.hpp:38-45
  int restart_index = 0;
  std::uint64_t seed = 0;
  double coherence = 0.0;
  bool succeeded = false;
  std::string error;
  std::vector<StageRecord> stages;
};
struct SolveResult {  // solver.hpp:47-54
  Frame best_frame;
  double best_coherence = 0.0;
  int best_restart = -1;
  std::vector<RestartRecord> per_restart;
  SolverConfig config;
  double wall_time_seconds = 0.0;
};

inline double welch_bound(Index d, Index N) { return trstmi_welch_bound(d, N); }

inline std::vector<double> default_delta_schedule(Index N, double eps_target) {
  double buf[TRSTMI_MAX_STAGES];
  const int n = trstmi_default_schedule(N, eps_target, buf, TRSTMI_MAX_STAGES);
  if (n < 0) throw std::invalid_argument("default_delta_schedule: invalid input");
  return std::vector<double>(buf, buf + std::min(n, TRSTMI_MAX_STAGES));
}

inline trstmi_cfg to_cfg(const SolverConfig& c) {
  trstmi_cfg k;
  trstmi_cfg_defaults(&k, (int)c.field, (int)c.d, (int)c.N);
  if (c.delta_schedule.size() > TRSTMI_MAX_STAGES) throw std::invalid_argument("anneal: schedule too long");
  k.n_stages = (int)c.delta_schedule.size();
  for (size_t i = 0; i < c.delta_schedule.size(); ++i) k.schedule[i] = c.delta_schedule[i];
  k.eps_target = c.eps_target;
  k.delta0 = c.tr.delta0;
  k.delta_max = c.tr.delta_max;
  k.eta = c.tr.eta;
  k.shrink = c.tr.shrink;
  k.grow = c.tr.grow;
  k.grad_tol = c.tr.grad_tol;
  k.max_outer = c.tr.max_outer;
  k.max_cg = c.tr.max_cg;
  k.cg_force_c = c.tr.cg_force_c;
  return k;
}

inline std::string trial_error(const trstmi_trial_out& t) {
  if (t.status == TRSTMI_TRIAL_ZERO_COLUMN) return "column " + std::to_string(t.zero_col) + " has near-zero norm";
  if (t.status == TRSTMI_TRIAL_NONFINITE_X0) return "trust_region_minimize: objective not finite at x0";
  return "trial failed";
}

// anneal (solver.hpp:164-204) of one start frame on the GPU.  rescue_state:
// nullable SplitMix64 state {state, has_spare, spare-bits} (the reference's
// rescue generator), updated in place.
inline std::pair<Frame, std::vector<StageRecord>> anneal(const Frame& start, const SolverConfig& cfg,
                                                          std::uint64_t* rescue_state = nullptr,
                                                          Context& ctx = Context::instance()) {
  if (start.d != cfg.d || start.N != cfg.N || start.field != cfg.field)
    throw DimensionMismatchError("anneal: start frame does not match config");
  trstmi_cfg k = to_cfg(cfg);
  const int ns = k.n_stages ? k.n_stages : (int)default_delta_schedule(cfg.N, cfg.eps_target).size();
  VectorXd params = start.packed, frame(start.packed.size());
  trstmi_trial_out to;
  std::vector<trstmi_stage_out> so(ns);
  check(ctx.get(), trstmi_solve_batch(ctx.get(), &k, 1, params.data(), rescue_state, frame.data(), &to, so.data(),
                                      nullptr));
  if (to.status == TRSTMI_TRIAL_ZERO_COLUMN) throw ZeroColumnError(to.zero_col);
  if (to.status != TRSTMI_TRIAL_OK) throw std::invalid_argument(trial_error(to));
  std::vector<StageRecord> stages(ns);
  for (int s = 0; s < ns; ++s) stages[s] = {so[s].delta, so[s].objective, so[s].coherence, so[s].outer_iterations};
  Frame f{cfg.d, cfg.N, cfg.field, frame};
  return {f, stages};
}

// solve (solver.hpp:210-273): all restarts as one batched GPU anneal.
// `threads` is accepted for API compatibility (the reference's CPU workers).
inline SolveResult solve(const SolverConfig& cfg, int threads = 1, Context& ctx = Context::instance()) {
  (void)threads;
  if (cfg.d < 1 || cfg.N < 1) throw std::invalid_argument("solve: need d, N >= 1");
  if (cfg.restarts < 1) throw std::invalid_argument("solve: need restarts >= 1");
  SolveResult res;
  res.config = cfg;
  trstmi_cfg k = to_cfg(cfg);
  const int ns = k.n_stages ? k.n_stages : (int)default_delta_schedule(cfg.N, cfg.eps_target).size();
  const Index dim = (cfg.field == Field::complex_field ? 2 : 1) * cfg.d * cfg.N;
  VectorXd best(dim);
  double bc = 0.0;
  std::int64_t bi = -1;
  std::vector<trstmi_trial_out> to(cfg.restarts);
  std::vector<trstmi_stage_out> so((size_t)cfg.restarts * ns);
  const int rc = trstmi_solve(ctx.get(), &k, cfg.restarts, cfg.seed, 0, best.data(), &bc, &bi, to.data(), so.data());
  for (int i = 0; i < cfg.restarts; ++i) {
    RestartRecord r;
    r.restart_index = i;
    std::uint64_t z = cfg.seed + (std::uint64_t)(i + 1) * 0x9E3779B97F4A7C15ULL;  // mix_seed, rng.hpp:13-18
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    r.seed = z ^ (z >> 31);
    r.succeeded = to[i].status == TRSTMI_TRIAL_OK;
    r.coherence = to[i].coherence;
    if (!r.succeeded) r.error = trial_error(to[i]);
    for (int s = 0; s < ns && s < to[i].stages_done; ++s) {
      const trstmi_stage_out& o = so[(size_t)i * ns + s];
      r.stages.push_back({o.delta, o.objective, o.coherence, o.outer_iterations});
    }
    res.per_restart.push_back(r);
  }
  check(ctx.get(), rc);
  res.best_restart = (int)bi;
  res.best_coherence = bc;
  res.best_frame = Frame{cfg.d, cfg.N, cfg.field, best};
  return res;
}

// coherence (frame.hpp:138-145) of an already-normalised frame; the argmax
// pair is the build's addition.
inline double coherence(const Frame& f, Index* argmax_pair = nullptr, Context& ctx = Context::instance()) {
  double mu = 0.0;
  std::int64_t arg = -1, zc = -1;
  check(ctx.get(), trstmi_coherence_batch(ctx.get(), (int)f.field, f.d, f.N, 1, f.packed.data(), 0, &mu, &arg, &zc));
  if (argmax_pair) *argmax_pair = arg;
  return mu;
}

// normalize_columns (frame.hpp:60-69): throws ZeroColumnError on the first
// column with norm < 1e-12; CAS column norm.
inline Frame normalize_columns(const Frame& f) {
  const Index L = (f.field == Field::complex_field ? 2 : 1) * f.d;
  Frame out = f;
  for (Index j = 0; j < f.N; ++j) {
    double acc = 0.0;
    for (Index q = 0; q < L; ++q) acc = std::fma(f.packed[j * L + q], f.packed[j * L + q], acc);
    const double nrm = std::sqrt(acc);
    if (nrm < kZeroColumnTol) throw ZeroColumnError(j);
    for (Index q = 0; q < L; ++q) out.packed[j * L + q] = f.packed[j * L + q] / nrm;
  }
  return out;
}

namespace detail {
// make_objective (solver.hpp:104-114): zero column -> +inf, zero gradient.
inline Objective make_objective(const SmoothObjective& obj, Context& ctx = Context::instance()) {
  return [obj, &ctx](const VectorXd& p) -> Evaluation {
    double F = 0.0, s = 0.0;
    VectorXd g(p.size());
    std::int64_t zc = -1;
    check(ctx.get(), trstmi_eval_batch(ctx.get(), (int)obj.field, obj.d, obj.N, 1, p.data(), &obj.delta,
                                       obj.squared ? 1 : 0, &F, &s, g.data(), nullptr, &zc));
    return {F, std::move(g)};
  };
}
// make_hvp_factory (solver.hpp:118-137): central difference with the
// one-sided fallback, evaluated on the GPU.
inline HvpFactory make_hvp_factory(const SmoothObjective& obj, Context& ctx = Context::instance()) {
  return [obj, &ctx](const VectorXd& x) -> HvpOperator {
    return [obj, x, &ctx](const VectorXd& dir) -> VectorXd {
      VectorXd hv(x.size());
      std::int32_t path = 0;
      std::int64_t zc = -1;
      check(ctx.get(), trstmi_hvp_batch(ctx.get(), (int)obj.field, obj.d, obj.N, 1, x.data(), dir.data(), &obj.delta,
                                        hv.data(), &path, &zc));
      if (path == TRSTMI_HVP_FAILED) throw ZeroColumnError(zc);
      return hv;
    };
  };
}
}  // namespace detail

}  // namespace b200
}  // namespace trstmi
