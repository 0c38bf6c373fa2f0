// TEST INFRASTRUCTURE ONLY — C ABI over the CPU oracle (cas_oracle.hpp) so
// the pytest suite and bench.py's cpu_baseline / --impl reference arm can
// drive it.  Mirrors include/trstmi_b200.h entry by entry (orc_ prefix) and
// reuses its POD structs; it never calls into the CUDA product.
#include <chrono>
#include <cstring>

#include "../include/trstmi_b200.h"
#include "cas_oracle.hpp"
#include "altproj_oracle.hpp"

using namespace orc;

namespace {

// CAS shape parameters: the oracle takes the lane count S from
// the caller and derives the gradient chunk count K from (N, d, S) by the
// same rule as trstmi_kchunks().
int kchunks_for(std::int64_t d, std::int64_t N, int S) {
  (void)d;
  const std::int64_t K = S / N;
  return (int)(K < 1 ? 1 : (K > 8 ? 8 : K));
}

Shape make_shape(int field, std::int64_t d, std::int64_t N, int lanes) {
  Shape sh;
  sh.complex_field = (field == TRSTMI_COMPLEX);
  sh.d = d;
  sh.N = N;
  sh.lanes = lanes;
  sh.kchunks = kchunks_for(d, N, lanes);
  sh.zrows = (lanes == 32768) ? 16 : 0;  // large-frame path (trstmi_lanes == 32768)
  return sh;
}

SolverConfig make_solver_cfg(const trstmi_cfg* c, int lanes) {
  SolverConfig cfg;
  cfg.shape = make_shape(c->field, c->d, c->N, lanes);
  for (int k = 0; k < c->n_stages; ++k) cfg.delta_schedule.push_back(c->schedule[k]);
  cfg.eps_target = c->eps_target;
  cfg.tr.delta0 = c->delta0;
  cfg.tr.delta_max = c->delta_max;
  cfg.tr.eta = c->eta;
  cfg.tr.shrink = c->shrink;
  cfg.tr.grow = c->grow;
  cfg.tr.grad_tol = c->grad_tol;
  cfg.tr.max_outer = c->max_outer;
  cfg.tr.max_cg = c->max_cg;
  cfg.tr.cg_force_c = c->cg_force_c;
  return cfg;
}

void pack_rng(const Rng& r, std::uint64_t* st) {
  st[0] = r.state;
  st[1] = r.has_spare ? 1 : 0;
  std::memcpy(&st[2], &r.spare, 8);
}
Rng unpack_rng(const std::uint64_t* st) {
  Rng r(st[0]);
  r.has_spare = st[1] != 0;
  std::memcpy(&r.spare, &st[2], 8);
  return r;
}

void run_trial(const SolverConfig& cfg, const trstmi_cfg* c, std::int64_t t, double* params, std::uint64_t* rng_state,
               double* frames, trstmi_trial_out* to, trstmi_stage_out* so, int n_stages, trstmi_outer_out* oo) {
  const std::int64_t dim = cfg.shape.dim();
  Vec start(params + t * dim, params + (t + 1) * dim);
  Rng rng;
  Rng* rp = nullptr;
  if (rng_state) {
    rng = unpack_rng(rng_state + 3 * t);
    rp = &rng;
  }
  AnnealResult a;
  int stage_at = 0;
  trstmi_trial_out& r = to[t];
  std::memset(&r, 0, sizeof(r));
  r.zero_col = -1;
  r.fail_stage = -1;
  r.argmax_pair = -1;
  try {
    anneal_into(start, cfg, rp, oo != nullptr && c->record_cap > 0, a, &stage_at);
    r.status = TRSTMI_TRIAL_OK;
    r.coherence = a.mu;
    r.argmax_pair = a.argmax;
    std::memcpy(params + t * dim, a.param.data(), dim * sizeof(double));
    if (frames) std::memcpy(frames + t * dim, a.frame.data(), dim * sizeof(double));
  } catch (const ZeroColumnFailure& e) {
    r.status = TRSTMI_TRIAL_ZERO_COLUMN;
    r.zero_col = e.column;
    r.fail_stage = stage_at;
  } catch (const HvpFailure& e) {
    r.status = TRSTMI_TRIAL_ZERO_COLUMN;
    r.zero_col = e.column;
    r.fail_stage = stage_at;
  } catch (const std::invalid_argument&) {
    r.status = TRSTMI_TRIAL_NONFINITE_X0;
    r.fail_stage = stage_at;
  }
  r.stages_done = static_cast<int>(a.stages.size());
  r.outer_iterations = a.counters.outer;
  r.evals = a.counters.evals;
  r.hvps = a.counters.cg;
  if (rng_state) pack_rng(rng, rng_state + 3 * t);
  for (int k = 0; k < n_stages && k < (int)a.stages.size(); ++k) {
    trstmi_stage_out& s = so[t * n_stages + k];
    s.delta = a.stages[k].delta;
    s.objective = a.stages[k].objective;
    s.coherence = a.stages[k].coherence;
    s.argmax_pair = a.stages[k].argmax;
    s.outer_iterations = a.stages[k].outer_iterations;
    s.status = a.stages[k].status;
  }
  if (oo && c->record_cap > 0) {
    const std::int64_t cap = c->record_cap;
    const std::int64_t nrec = std::min<std::int64_t>(cap, (std::int64_t)a.history.size());
    for (std::int64_t i = 0; i < nrec; ++i) {
      const OuterRecord& h = a.history[i];
      trstmi_outer_out& o = oo[t * cap + i];
      o.stage = a.history_stage[i];
      o.iteration = h.iteration;
      o.cg_exit = h.cg_exit;
      o.cg_iterations = h.cg_iterations;
      o.accepted = h.accepted ? 1 : 0;
      o.pad = 0;
      o.value = h.value;
      o.grad_norm = h.grad_norm;
      o.radius = h.radius;
      o.rho = h.rho;
      o.step_norm = h.step_norm;
    }
    r.records = nrec;
  }
}

}  // namespace

extern "C" {

int orc_kchunks(std::int64_t d, std::int64_t N, int S) { return kchunks_for(d, N, S); }
double orc_exp(double x) { return cas_exp(x); }
double orc_log(double x) { return cas_log(x); }
void orc_exp_array(const double* x, double* y, std::int64_t n) {
  for (std::int64_t i = 0; i < n; ++i) y[i] = cas_exp(x[i]);
}
void orc_log_array(const double* x, double* y, std::int64_t n) {
  for (std::int64_t i = 0; i < n; ++i) y[i] = cas_log(x[i]);
}
double orc_hypot(double x, double y) { return cas_hypot(x, y); }
double orc_cas_sum(const double* v, std::int64_t n, int S) { return cas_sum(v, n, S); }
double orc_cas_dot(const double* a, const double* b, std::int64_t n, int S) { return cas_dot(a, b, n, S); }
std::uint64_t orc_mix_seed(std::uint64_t seed, std::uint64_t index) { return mix_seed(seed, index); }
double orc_welch_bound(std::int64_t d, std::int64_t N) { return welch_bound(d, N); }

int orc_default_schedule(std::int64_t N, double eps, double* out, int cap) {
  try {
    std::vector<double> s = default_delta_schedule(N, eps);
    const int n = (int)s.size();
    for (int i = 0; i < n && i < cap; ++i) out[i] = s[i];
    return n;
  } catch (...) {
    return -1;
  }
}

// Uniform stream helpers for porting the reference's property tests.
void orc_rng_uniform(std::uint64_t seed, double* out, std::int64_t n) {
  Rng r(seed);
  for (std::int64_t i = 0; i < n; ++i) out[i] = r.uniform();
}
void orc_rng_normal(std::uint64_t seed, double* out, std::int64_t n) {
  Rng r(seed);
  for (std::int64_t i = 0; i < n; ++i) out[i] = r.normal();
}

int orc_random_frames(int field, std::int64_t d, std::int64_t N, std::uint64_t seed, std::int64_t first,
                      std::int64_t count, double* frames, std::uint64_t* rng_state) {
  if (d < 1 || N < 1) return TRSTMI_ERR_INVALID_ARG;
  Shape sh = make_shape(field, d, N, 32);
  for (std::int64_t t = 0; t < count; ++t) {
    Rng rng(mix_seed(seed, (std::uint64_t)(first + t)));
    Vec f = random_frame(sh, rng);
    std::memcpy(frames + t * sh.dim(), f.data(), sh.dim() * sizeof(double));
    if (rng_state) pack_rng(rng, rng_state + 3 * t);
  }
  return TRSTMI_OK;
}

// Plain-seed frame (testsupport::random_test_frame, tests/support.hpp:75-78).
int orc_random_test_frame(int field, std::int64_t d, std::int64_t N, std::uint64_t seed, double* frame) {
  Shape sh = make_shape(field, d, N, 32);
  Rng rng(seed);
  Vec f = random_frame(sh, rng);
  std::memcpy(frame, f.data(), sh.dim() * sizeof(double));
  return TRSTMI_OK;
}

// eval_objective at x + sc*dir (dir may be NULL when sc == 0).
std::int64_t orc_eval(int field, std::int64_t d, std::int64_t N, int lanes, const double* x, const double* dir,
                      double sc, double delta, int squared, double* F, double* s, double* grad, double* weights) {
  Shape sh = make_shape(field, d, N, lanes);
  EvalResult e = eval_objective(sh, x, dir, sc, delta, squared != 0, weights != nullptr);
  if (e.zero_col >= 0) {
    *F = std::numeric_limits<double>::infinity();
    *s = 0.0;
    std::memset(grad, 0, sh.dim() * sizeof(double));
    return e.zero_col;
  }
  *F = e.value;
  *s = e.s;
  std::memcpy(grad, e.grad.data(), sh.dim() * sizeof(double));
  if (weights) std::memcpy(weights, e.weights.data(), sh.pairs() * sizeof(double));
  return -1;
}

std::int64_t orc_hvp(int field, std::int64_t d, std::int64_t N, int lanes, const double* x, const double* dir,
                     double delta, double* hv, int* path) {
  Shape sh = make_shape(field, d, N, lanes);
  Vec xv(x, x + sh.dim()), dv(dir, dir + sh.dim());
  HvpResult r = hvp_adapter(sh, xv, dv, delta, nullptr);
  *path = r.path;
  if (r.path == HVP_FAILED) {
    std::memset(hv, 0, sh.dim() * sizeof(double));
    return r.zero_col;
  }
  std::memcpy(hv, r.hv.data(), sh.dim() * sizeof(double));
  return -1;
}

// distortion_mc (beamforming.hpp:78-163) restated with the CAS orders (the
// checker of trstmi_distortion_mc): blocks of 4096 samples, SplitMix64 per
// block, overlaps |conj(phi_i) . h|^2 by ascending fma chains, moments summed
// sequentially per block and then in block order.
int orc_distortion_mc(std::int64_t d, std::int64_t N, const double* book, std::uint64_t samples,
                      std::uint64_t seed, double* estimate, double* std_error) {
  if (samples < 1 || N < 1) return 1;
  const std::uint64_t B = 4096, nblocks = (samples + B - 1) / B;
  double sum = 0.0, sum_sq = 0.0;
  std::vector<double> h(2 * d);
  for (std::uint64_t b = 0; b < nblocks; ++b) {
    Rng rng(mix_seed(seed, b));
    const std::uint64_t count = std::min(B, samples - b * B);
    double bs = 0.0, bq = 0.0;
    for (std::uint64_t s = 0; s < count; ++s) {
      double norm_sq = 0.0;
      do {
        for (std::int64_t i = 0; i < d; ++i) rng.complex_normal(&h[2 * i], &h[2 * i + 1]);
        norm_sq = 0.0;
        for (std::int64_t q = 0; q < 2 * d; ++q) norm_sq = std::fma(h[q], h[q], norm_sq);
      } while (norm_sq < kZeroColumnTol * kZeroColumnTol);
      double best = 0.0;
      for (std::int64_t i = 0; i < N; ++i) {
        const double* col = book + i * 2 * d;
        double re = 0.0, im = 0.0;
        for (std::int64_t q = 0; q < d; ++q) {
          const double ar = col[2 * q], ai = col[2 * q + 1], hr = h[2 * q], hi = h[2 * q + 1];
          re = std::fma(ar, hr, re);
          re = std::fma(ai, hi, re);
          im = std::fma(ar, hi, im);
          im = std::fma(-ai, hr, im);
        }
        const double ov = re * re + im * im;
        if (ov > best) best = ov;
      }
      const double dsq = std::max(0.0, 1.0 - best / norm_sq);
      bs += dsq;
      bq += dsq * dsq;
    }
    sum += bs;
    sum_sq += bq;
  }
  const double n = static_cast<double>(samples);
  *estimate = sum / n;
  *std_error = 0.0;
  if (samples > 1) *std_error = std::sqrt(std::max(0.0, (sum_sq - n * *estimate * *estimate) / (n - 1.0)) / n);
  return 0;
}

// offdiagonal_magnitudes (frame.hpp:80-91) of a frame, CAS |G| (the checker
// of trstmi_offdiag_magnitudes)
void orc_offdiag_magnitudes(int field, std::int64_t d, std::int64_t N, const double* frame, double* mags) {
  Shape sh = make_shape(field, d, N, 32);
  const std::int64_t L = sh.col_len();
  for (std::int64_t j = 0, p = 0; j < N; ++j)
    for (std::int64_t k = j + 1; k < N; ++k, ++p) {
      double gr, gi;
      gram_entry(sh, frame + j * L, frame + k * L, &gr, &gi);
      mags[p] = cas_hypot(gr, gi);
    }
}

std::int64_t orc_coherence(int field, std::int64_t d, std::int64_t N, const double* frame, int normalize, double* mu,
                           std::int64_t* argmax) {
  Shape sh = make_shape(field, d, N, 32);
  CoherenceResult c = coherence(sh, frame, normalize != 0);
  *mu = c.mu;
  *argmax = c.argmax;
  return c.zero_col;
}

int orc_solve_batch(const trstmi_cfg* c, int lanes, std::int64_t trials, double* params, std::uint64_t* rng_state,
                    double* frames, trstmi_trial_out* trial_out, trstmi_stage_out* stage_out,
                    trstmi_outer_out* outer_out, int threads) {
  SolverConfig cfg = make_solver_cfg(c, lanes);
  int n_stages = c->n_stages;
  if (n_stages == 0) {
    try {
      n_stages = (int)default_delta_schedule(c->N, c->eps_target).size();
    } catch (...) {
      return TRSTMI_ERR_INVALID_ARG;
    }
  }
  const int workers = std::max(1, std::min<int>(threads, (int)trials));
  std::atomic<std::int64_t> next{0};
  auto work = [&] {
    for (std::int64_t t = next.fetch_add(1); t < trials; t = next.fetch_add(1))
      run_trial(cfg, c, t, params, rng_state, frames, trial_out, stage_out, n_stages, outer_out);
  };
  if (workers == 1) {
    work();
  } else {
    std::vector<std::thread> pool;
    for (int w = 0; w < workers; ++w) pool.emplace_back(work);
    for (auto& th : pool) th.join();
  }
  return TRSTMI_OK;
}

// Bounded CPU sample for bench.py: runs `trials` anneals (threads workers) and
// returns the wall seconds; outer iterations / evals are summed into *outer,
// *evals.
double orc_time_solve_batch(const trstmi_cfg* c, int lanes, std::int64_t trials, double* params,
                            std::uint64_t* rng_state, int threads, std::int64_t* outer, std::int64_t* evals) {
  int n_stages = c->n_stages ? c->n_stages : (int)default_delta_schedule(c->N, c->eps_target).size();
  std::vector<trstmi_trial_out> to(trials);
  std::vector<trstmi_stage_out> so(trials * n_stages);
  const auto t0 = std::chrono::steady_clock::now();
  orc_solve_batch(c, lanes, trials, params, rng_state, nullptr, to.data(), so.data(), nullptr, threads);
  const double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  std::int64_t o = 0, e = 0;
  for (auto& r : to) {
    o += r.outer_iterations;
    e += r.evals;
  }
  *outer = o;
  *evals = e;
  return sec;
}

// alternating_projection (baseline.hpp:68-167) for `restarts` start frames (restarts x 2dN doubles, each the
// random_frame of its own child generator): the checker of trstmi_altproj_batch.  iterations[r] > 0: converged
// after that many iterations, < 0: the best iterate after -iterations[r] (StageRecord::outer_iterations).
int orc_altproj_batch(std::int64_t d, std::int64_t N, int max_iters, double mu_target, double tol, std::int64_t restarts,
                      const double* starts, double* frames, double* coherences, std::int32_t* iterations,
                      std::int32_t* sweeps) {
  if (d < 1 || N < 1 || d > N || max_iters < 1) return TRSTMI_ERR_INVALID_ARG;
  AltProjCfg cfg;
  cfg.max_iters = max_iters;
  cfg.mu_target = mu_target;
  cfg.tol = tol;
  const std::int64_t dim = 2 * d * N;
  for (std::int64_t r = 0; r < restarts; ++r) {
    const AltProjOut o = altproj_run((int)d, (int)N, cfg, starts + r * dim);
    std::memcpy(frames + r * dim, o.frame.data(), dim * sizeof(double));
    coherences[r] = o.coherence;
    iterations[r] = o.iterations;
    if (sweeps) sweeps[r] = o.jacobi_sweeps;
  }
  return TRSTMI_OK;
}

}  // extern "C"
