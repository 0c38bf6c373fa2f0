// TEST INFRASTRUCTURE ONLY — the reference's own hot-path headers
// (/root/reference/proj/include/trstmi/{rng,frame,smoothing,trust_region,
// solver}.hpp), compiled UNCHANGED against oracle/eigen_shim (Eigen is absent
// from this image), behind a small C ABI.  Built by oracle/Makefile into
// oracle/_ref/libtrstmi_ref.so only where /root/reference exists; the built
// .so travels to the GPU box.  Used by tests/ (to pin the CAS oracle to the
// reference at the north-star tolerances) and by bench.py's cpu_baseline and
// --impl reference arms (cpu_baseline.kind = "reference").  Never linked into
// the product.
//
// Everything numeric below is the reference's code; this file only adapts
// buffers, catches the reference's exceptions into status codes, counts
// evaluator calls, and runs restarts on a thread pool the way solve() does
// (solver.hpp:239-254).
#include <atomic>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <limits>
#include <thread>
#include <vector>

#include "trstmi/frame.hpp"
#include "trstmi/rng.hpp"
#include "trstmi/smoothing.hpp"
#include "trstmi/solver.hpp"
#include "trstmi/trust_region.hpp"

using namespace trstmi;

namespace {

// Real frames (BASELINE configs 1 and 4) run through the reference's complex
// code with Im == 0 (exact: zeros propagate as exact zeros; SURVEY.md App. B
// item 7); `field` 1 = real input/output of length d*N.
VectorXd embed(int field, Index d, Index N, const double* p) {
  VectorXd v(2 * d * N);
  if (field == 0) {
    std::memcpy(v.data(), p, sizeof(double) * 2 * d * N);
  } else {
    for (Index i = 0; i < d * N; ++i) {
      v[2 * i] = p[i];
      v[2 * i + 1] = 0.0;
    }
  }
  return v;
}

void extract(int field, Index d, Index N, const VectorXd& v, double* out) {
  if (field == 0) {
    std::memcpy(out, v.data(), sizeof(double) * 2 * d * N);
  } else {
    for (Index i = 0; i < d * N; ++i) out[i] = v[2 * i];
  }
}

struct Counters {
  std::int64_t evals = 0, hvps = 0;
};

// make_objective / make_hvp_factory (solver.hpp:104-137) wrapped to count
// evaluator calls: x0 + trial evaluations, and 2 per Hessian-vector product
// (the central difference; the rare one-sided fallback is not counted).
Objective counting(Objective f, Counters* c) {
  return [f, c](const VectorXd& p) {
    ++c->evals;
    return f(p);
  };
}
HvpFactory counting(HvpFactory f, Counters* c) {
  return [f, c](const VectorXd& x) -> HvpOperator {
    HvpOperator op = f(x);
    return [op, c](const VectorXd& dir) {
      ++c->hvps;
      c->evals += 2;
      return op(dir);
    };
  };
}

TrustRegionConfig tr_cfg(int field, Index d, Index N, const double* tr6, const int* tri) {
  TrustRegionConfig t;
  t.delta0 = tr6[0];
  t.delta_max = tr6[1];
  t.eta = tr6[2];
  t.shrink = tr6[3];
  t.grow = tr6[4];
  t.grad_tol = tr6[5];
  t.cg_force_c = tr6[6];
  t.max_outer = tri[0];
  t.max_cg = tri[1];
  if (field == 1) {  // real mode: the dim-dependent defaults on dim = dN (trust_region.hpp:194-195)
    if (t.delta0 == 0.0) t.delta0 = 0.1 * std::sqrt(static_cast<double>(d * N));
    if (t.max_cg == 0) t.max_cg = static_cast<int>(2 * d * N);
  }
  return t;
}

// One anneal in flight: the trial's raw parameter vector and its rescue
// generator (solver.hpp:221-237).
struct Trial {
  SplitMix64 rng{0};
  VectorXd param;
  Counters cnt;
  std::int64_t outer = 0;
  int status = 0;  // 0 ok, 1 zero column escaped, 2 other exception
  std::vector<OuterRecord> history;  // kept when the batch records (ref_batch_keep_history)
  std::vector<int> history_stage;
};

struct Batch {
  int field;
  Index d, N;
  std::vector<Trial> trials;
  bool keep_history = false;
};

template <class F>
void pool(std::int64_t n, int threads, F&& fn) {
  const int workers = std::max<int>(1, std::min<std::int64_t>(threads, n));
  std::atomic<std::int64_t> next{0};
  auto work = [&] {
    for (std::int64_t i = next.fetch_add(1); i < n; i = next.fetch_add(1)) fn(i);
  };
  if (workers == 1) {
    work();
    return;
  }
  std::vector<std::thread> th;
  for (int w = 0; w < workers; ++w) th.emplace_back(work);
  for (auto& t : th) t.join();
}

}  // namespace

extern "C" {

// eval_objective (smoothing.hpp:82-162) through make_objective semantics:
// returns -1, or the zero column (F = +inf, grad = 0).  weights nullable.
std::int64_t ref_eval(int field, std::int64_t d, std::int64_t N, const double* point, double delta, int squared,
                      double* F, double* s, double* grad, double* weights) {
  const VectorXd p = embed(field, d, N, point);
  SmoothObjective obj{delta, d, N, squared != 0};
  try {
    ObjectiveEval e = eval_objective(p, obj);
    *F = e.value;
    *s = e.s;
    extract(field, d, N, e.grad, grad);
    if (weights) std::memcpy(weights, e.softmax_weights.data(), sizeof(double) * obj.pair_count());
    return -1;
  } catch (const ZeroColumnError& z) {
    *F = std::numeric_limits<double>::infinity();
    *s = 0.0;
    std::memset(grad, 0, sizeof(double) * (field == 0 ? 2 : 1) * d * N);
    return z.column;
  }
}

// detail::make_hvp_factory(obj)(x)(dir) (solver.hpp:118-137): central FD with
// the one-sided fallback.  Returns -1, or the zero column that escaped.
std::int64_t ref_hvp(int field, std::int64_t d, std::int64_t N, const double* x, const double* dir, double delta,
                     double* hv) {
  SmoothObjective obj{delta, d, N, true};
  try {
    const VectorXd r = detail::make_hvp_factory(obj)(embed(field, d, N, x))(embed(field, d, N, dir));
    extract(field, d, N, r, hv);
    return -1;
  } catch (const ZeroColumnError& z) {
    return z.column;
  }
}

// offdiagonal_magnitudes (frame.hpp:80-91), std::abs = hypot.
void ref_offdiag_magnitudes(int field, std::int64_t d, std::int64_t N, const double* frame, double* mags) {
  const std::vector<double> m = offdiagonal_magnitudes(unpack_frame(embed(field, d, N, frame), d, N));
  std::memcpy(mags, m.data(), sizeof(double) * m.size());
}

// coherence (frame.hpp:138-145), optionally of normalize_columns(frame); the
// argmax is the first strict maximum in the same pair order.
std::int64_t ref_coherence(int field, std::int64_t d, std::int64_t N, const double* frame, int normalize, double* mu,
                           std::int64_t* argmax) {
  try {
    Frame f = unpack_frame(embed(field, d, N, frame), d, N);
    if (normalize) f = normalize_columns(f);
    *mu = coherence(f);
    const std::vector<double> m = offdiagonal_magnitudes(f);
    double best = 0.0;
    std::int64_t arg = -1;
    for (std::size_t i = 0; i < m.size(); ++i)
      if (m[i] > best) {
        best = m[i];
        arg = (std::int64_t)i;
      }
    *argmax = arg;
    return -1;
  } catch (const ZeroColumnError& z) {
    *mu = 0.0;
    *argmax = -1;
    return z.column;
  }
}

// default_delta_schedule (solver.hpp:64-82)
int ref_default_schedule(std::int64_t N, double eps, double* out, int cap) {
  try {
    const std::vector<double> s = default_delta_schedule(N, eps);
    for (int i = 0; i < (int)s.size() && i < cap; ++i) out[i] = s[i];
    return (int)s.size();
  } catch (...) {
    return -1;
  }
}

// ---- batched anneals, stage by stage --------------------------------------
// ref_batch_create: trials [first, first+count) of `seed`.  Complex field:
// the reference's own run_restart prologue (solver.hpp:224-226): generator
// SplitMix64(mix_seed(seed, i)), start = random_frame(d, N, rng).  Real field:
// start frames come from the caller (`starts`, count x dN) and are embedded.
void* ref_batch_create(int field, std::int64_t d, std::int64_t N, std::uint64_t seed, std::int64_t first,
                       std::int64_t count, const double* starts) {
  Batch* b = new Batch{field, d, N, std::vector<Trial>(count)};
  for (std::int64_t t = 0; t < count; ++t) {
    Trial& tr = b->trials[t];
    tr.rng = SplitMix64(mix_seed(seed, (std::uint64_t)(first + t)));
    if (field == 0 && !starts) {
      tr.param = pack_frame(random_frame(d, N, tr.rng));
    } else {
      tr.param = embed(field, d, N, starts + t * (field == 0 ? 2 : 1) * d * N);
    }
  }
  return b;
}

void ref_batch_destroy(void* h) { delete static_cast<Batch*>(h); }

// Stages [k0, k1) of anneal() (solver.hpp:182-200) for every trial of the
// batch on `threads` workers: rescue, SmoothObjective{delta_k}, cap
// max_outer + 50k, trust_region_minimize, param <- best-seen x, stage record.
// tr6 = {delta0, delta_max, eta, shrink, grow, grad_tol, cg_force_c};
// tri = {max_outer, max_cg}.  stage_rec (nullable): count x n_stages x 4
// doubles {delta, objective, coherence, outer_iterations}.  Returns the wall
// seconds of the run; *outer / *evals / *hvps receive this call's totals.
double ref_batch_run_stages(void* h, const double* schedule, int n_stages, int k0, int k1, const double* tr6,
                            const int* tri, int threads, double* stage_rec, std::int64_t* outer, std::int64_t* evals,
                            std::int64_t* hvps) {
  Batch* b = static_cast<Batch*>(h);
  const TrustRegionConfig base = tr_cfg(b->field, b->d, b->N, tr6, tri);
  const std::int64_t T = (std::int64_t)b->trials.size();
  std::vector<Counters> before(T);
  std::vector<std::int64_t> outer0(T);
  for (std::int64_t t = 0; t < T; ++t) {
    before[t] = b->trials[t].cnt;
    outer0[t] = b->trials[t].outer;
  }
  const auto t0 = std::chrono::steady_clock::now();
  pool(T, threads, [&](std::int64_t t) {
    Trial& tr = b->trials[t];
    if (tr.status) return;
    try {
      for (int k = k0; k < k1; ++k) {
        detail::rescue_zero_columns(tr.param, b->d, b->N, &tr.rng);
        SmoothObjective obj{schedule[k], b->d, b->N, true};
        TrustRegionConfig trc = base;
        trc.max_outer = base.max_outer + 50 * k;
        MinimizeResult res = trust_region_minimize(counting(detail::make_objective(obj), &tr.cnt),
                                                   counting(detail::make_hvp_factory(obj), &tr.cnt),
                                                   std::move(tr.param), trc);
        tr.param = std::move(res.x);
        tr.outer += (std::int64_t)res.history.size();
        if (b->keep_history)
          for (const OuterRecord& r : res.history) {
            tr.history.push_back(r);
            tr.history_stage.push_back(k);
          }
        if (stage_rec) {
          double* r = stage_rec + (t * n_stages + k) * 4;
          r[0] = schedule[k];
          r[1] = res.value;
          r[2] = coherence(normalize_columns(unpack_frame(tr.param, b->d, b->N)));
          r[3] = (double)res.history.size();
        }
      }
    } catch (const ZeroColumnError&) {
      tr.status = 1;
    } catch (const std::exception&) {
      tr.status = 2;
    }
  });
  const double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  std::int64_t o = 0, e = 0, hv = 0;
  for (std::int64_t t = 0; t < T; ++t) {
    o += b->trials[t].outer - outer0[t];
    e += b->trials[t].cnt.evals - before[t].evals;
    hv += b->trials[t].cnt.hvps - before[t].hvps;
  }
  if (outer) *outer = o;
  if (evals) *evals = e;
  if (hvps) *hvps = hv;
  return sec;
}

void ref_batch_keep_history(void* h, int on) { static_cast<Batch*>(h)->keep_history = on != 0; }

// OuterRecords (trust_region.hpp:163-173) of trial t, at most cap, as
// trstmi_outer_out-shaped rows: {stage, iteration, cg_exit, cg_iterations,
// accepted} ints + {value, grad_norm, radius, rho, step_norm} doubles.
// Returns the number of records the trial has.
std::int64_t ref_batch_history(void* h, std::int64_t t, std::int64_t cap, int* ints5, double* dbl5) {
  const Trial& tr = static_cast<Batch*>(h)->trials[t];
  const std::int64_t n = (std::int64_t)tr.history.size();
  for (std::int64_t i = 0; i < n && i < cap; ++i) {
    const OuterRecord& r = tr.history[i];
    int* o = ints5 + 5 * i;
    o[0] = tr.history_stage[i];
    o[1] = r.iteration;
    o[2] = static_cast<int>(r.cg_exit);
    o[3] = r.cg_iterations;
    o[4] = r.accepted ? 1 : 0;
    double* v = dbl5 + 5 * i;
    v[0] = r.value;
    v[1] = r.grad_norm;
    v[2] = r.radius;
    v[3] = r.rho;
    v[4] = r.step_norm;
  }
  return n;
}

// Raw parameters (count x dim) and per-trial status of the batch.
void ref_batch_params(void* h, double* params, int* status) {
  Batch* b = static_cast<Batch*>(h);
  const std::int64_t dim = (b->field == 0 ? 2 : 1) * b->d * b->N;
  for (std::size_t t = 0; t < b->trials.size(); ++t) {
    extract(b->field, b->d, b->N, b->trials[t].param, params + t * dim);
    if (status) status[t] = b->trials[t].status;
  }
}

// The reference's own anneal() (solver.hpp:164-204) on one complex start
// frame (with the run_restart generator when seed_index >= 0): final
// normalised frame and stage records (n_stages x 4 as above).  Returns 0, or
// 1 when an exception escaped.
int ref_anneal(std::int64_t d, std::int64_t N, const double* schedule, int n_stages, const double* tr6,
               const int* tri, std::uint64_t seed, std::int64_t seed_index, const double* start, double* frame_out,
               double* stage_rec) {
  SolverConfig cfg;
  cfg.d = d;
  cfg.N = N;
  cfg.delta_schedule.assign(schedule, schedule + n_stages);
  cfg.tr = tr_cfg(0, d, N, tr6, tri);
  try {
    SplitMix64 rng(mix_seed(seed, (std::uint64_t)std::max<std::int64_t>(seed_index, 0)));
    Frame st = start ? unpack_frame(embed(0, d, N, start), d, N) : random_frame(d, N, rng);
    auto [frame, stages] = anneal(st, cfg, seed_index >= 0 ? &rng : nullptr);
    if (frame_out) extract(0, d, N, pack_frame(frame), frame_out);
    for (int k = 0; k < (int)stages.size() && stage_rec; ++k) {
      stage_rec[4 * k] = stages[k].delta;
      stage_rec[4 * k + 1] = stages[k].objective;
      stage_rec[4 * k + 2] = stages[k].coherence;
      stage_rec[4 * k + 3] = stages[k].outer_iterations;
    }
    return 0;
  } catch (const std::exception&) {
    return 1;
  }
}

// The reference's solve() (solver.hpp:210-273), complex field.  per_restart
// (nullable): restarts coherences (NaN where a restart failed).  Returns 0,
// or 1 on SolveError / invalid argument.
int ref_solve(std::int64_t d, std::int64_t N, int restarts, std::uint64_t seed, double eps_target, const double* tr6,
              const int* tri, int threads, double* best_frame, double* best_coherence, int* best_restart,
              double* per_restart, double* wall_s) {
  SolverConfig cfg;
  cfg.d = d;
  cfg.N = N;
  cfg.restarts = restarts;
  cfg.seed = seed;
  cfg.eps_target = eps_target;
  cfg.tr = tr_cfg(0, d, N, tr6, tri);
  try {
    SolveResult r = solve(cfg, threads);
    *best_coherence = r.best_coherence;
    *best_restart = r.best_restart;
    if (best_frame) extract(0, d, N, pack_frame(r.best_frame), best_frame);
    for (int i = 0; per_restart && i < restarts; ++i)
      per_restart[i] = r.per_restart[i].succeeded ? r.per_restart[i].coherence : std::nan("");
    if (wall_s) *wall_s = r.wall_time_seconds;
    return 0;
  } catch (const std::exception&) {
    return 1;
  }
}

}  // extern "C"
