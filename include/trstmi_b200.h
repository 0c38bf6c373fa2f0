/*
 * trstmi_b200.h — C ABI of the B200-native TRST-MI hot path.
 *
 * Plain pointers and sizes only (no C++ / torch types).  Every entry point
 * returns an int status (TRSTMI_OK == 0); no exception crosses the ABI.  The
 * C++ host mirror of the reference API (paper_2207_06374_b200/csrc/host/
 * trstmi_host.hpp) rethrows the reference's exception types from these codes.
 *
 * Reference interfaces replaced (paths under /root/reference/proj/include/trstmi):
 *   trstmi_eval_batch       <- eval_objective            smoothing.hpp:82-162
 *                              + detail::make_objective   solver.hpp:104-114
 *   trstmi_hvp_batch        <- hessian_vector_product    smoothing.hpp:167-194
 *                              + detail::make_hvp_factory solver.hpp:118-137
 *   trstmi_coherence_batch  <- coherence / normalize_columns  frame.hpp:60-69,138-145
 *   trstmi_welch_bound      <- welch_bound               analysis.hpp:27-31
 *   trstmi_default_schedule <- default_delta_schedule    solver.hpp:64-82
 *   trstmi_solve_batch      <- anneal (per trial)        solver.hpp:164-204
 *                              driving trust_region_minimize trust_region.hpp:189-295
 *                              and steihaug_cg            trust_region.hpp:81-154
 *   trstmi_solve            <- solve (multistart)        solver.hpp:210-273
 *   trstmi_random_frames    <- random_frame + mix_seed   solver.hpp:87-98, rng.hpp:13-64
 *
 * Layout of a frame / point (frame.hpp:37-40,165-186): column-major d x N;
 * complex entries interleaved (re, im), so column j is the contiguous run
 * [j*2d, (j+1)*2d).  Real frames (new mode) store column j at [j*d, (j+1)*d).
 * dim = 2dN (complex) or dN (real).  Pair p enumerates j<k in row-major
 * upper-triangular order: p(j,k) = j*N - j(j+1)/2 + (k-j-1)  (frame.hpp:80-91).
 *
 * Host pointers everywhere except the *_dev variants, which take device
 * pointers and a cudaStream_t passed as void* (used verbatim: NULL is the
 * legacy default stream).
 */
#ifndef TRSTMI_B200_H
#define TRSTMI_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (map to the reference's exception types) ---- */
#define TRSTMI_OK 0
#define TRSTMI_ERR_INVALID_ARG 1      /* std::invalid_argument                          */
#define TRSTMI_ERR_DIM_MISMATCH 2     /* DimensionMismatchError (frame.hpp:33-35)       */
#define TRSTMI_ERR_ZERO_COLUMN 3      /* ZeroColumnError (frame.hpp:25-31)              */
#define TRSTMI_ERR_ALL_FAILED 4       /* SolveError "solve: all restarts failed"        */
#define TRSTMI_ERR_CUDA 5
#define TRSTMI_ERR_NCCL 6
#define TRSTMI_ERR_UNSUPPORTED 7      /* shape outside the compiled kernel families     */
#define TRSTMI_ERR_NO_DEVICE 8

/* ---- field ---- */
#define TRSTMI_COMPLEX 0              /* reference field                  */
#define TRSTMI_REAL 1                 /* real lines (new; BASELINE configs 1 and 4)     */

/* ---- HVP path (make_hvp_factory fallback, solver.hpp:118-137) ---- */
#define TRSTMI_HVP_CENTRAL 0
#define TRSTMI_HVP_FORWARD 1
#define TRSTMI_HVP_BACKWARD 2
#define TRSTMI_HVP_ZERO_DIR 3
#define TRSTMI_HVP_FAILED (-1)        /* ZeroColumnError escapes the adapter            */

/* ---- MinimizeStatus (trust_region.hpp:156-161) ---- */
#define TRSTMI_ST_GRADIENT_TOLERANCE 0
#define TRSTMI_ST_ITERATION_LIMIT 1
#define TRSTMI_ST_RADIUS_UNDERFLOW 2

/* ---- per-trial status (RestartRecord::succeeded / error, solver.hpp:225-236) ---- */
#define TRSTMI_TRIAL_OK 0
#define TRSTMI_TRIAL_ZERO_COLUMN 1    /* rescue failed / hvp fallback failed            */
#define TRSTMI_TRIAL_NONFINITE_X0 2   /* "trust_region_minimize: objective not finite"  */
#define TRSTMI_TRIAL_NEED_RESCUE 3    /* internal: stage start found a zero column      */
#define TRSTMI_TRIAL_INVALID 4

/* ---- CgExit (trust_region.hpp:32) ---- */
#define TRSTMI_CG_SMALL_RESIDUAL 0
#define TRSTMI_CG_NEGATIVE_CURVATURE 1
#define TRSTMI_CG_BOUNDARY_HIT 2
#define TRSTMI_CG_ZERO_GRADIENT 3

#define TRSTMI_MAX_STAGES 32

/* SolverConfig (solver.hpp:21-29) + TrustRegionConfig (trust_region.hpp:20-30). */
typedef struct trstmi_cfg {
  int32_t field;                  /* TRSTMI_COMPLEX / TRSTMI_REAL                    */
  int32_t d, N;
  int32_t n_stages;               /* 0 -> default_delta_schedule(N, eps_target)      */
  double schedule[TRSTMI_MAX_STAGES];
  double eps_target;              /* 1e-7                                            */
  /* TrustRegionConfig */
  double delta0;                  /* 0 -> 0.1*sqrt(dim)                              */
  double delta_max;               /* 1e3 */
  double eta;                     /* 0.05 */
  double shrink;                  /* 0.25 */
  double grow;                    /* 2.0 */
  double grad_tol;                /* 1e-9 */
  int32_t max_outer;              /* 200; stage k runs max_outer + 50k (solver.hpp:187) */
  int32_t max_cg;                 /* 0 -> 2*dim */
  double cg_force_c;              /* 0.5 */
  int32_t record_cap;             /* OuterRecords kept per trial (0: none)           */
  int32_t reserved;
} trstmi_cfg;

/* RestartRecord (solver.hpp:38-45) without the strings. */
typedef struct trstmi_trial_out {
  double coherence;               /* mu of the final normalised frame                */
  int64_t argmax_pair;            /* first maximising pair (row-major upper-tri)     */
  int32_t status;                 /* TRSTMI_TRIAL_*                                  */
  int32_t stages_done;
  int32_t zero_col;               /* column of a ZeroColumnError, else -1            */
  int32_t fail_stage;             /* stage of the failure / rescue request, else -1  */
  int64_t outer_iterations;       /* sum of OuterRecord counts over stages           */
  int64_t evals;                  /* evaluator calls (x0 + trials + 2/hvp + fallback)*/
  int64_t hvps;                   /* CG Hessian-vector products                      */
  int64_t records;                /* OuterRecords written (<= record_cap)            */
} trstmi_trial_out;

/* StageRecord (solver.hpp:31-36) + the stage's MinimizeStatus and argmax. */
typedef struct trstmi_stage_out {
  double delta;
  double objective;
  double coherence;
  int64_t argmax_pair;
  int32_t outer_iterations;
  int32_t status;
} trstmi_stage_out;

/* OuterRecord (trust_region.hpp:163-173) + stage index. */
typedef struct trstmi_outer_out {
  int32_t stage;
  int32_t iteration;
  int32_t cg_exit;
  int32_t cg_iterations;
  int32_t accepted;
  int32_t pad;
  double value;
  double grad_norm;
  double radius;
  double rho;
  double step_norm;
} trstmi_outer_out;

typedef struct trstmi_ctx trstmi_ctx;

/* ---- context ---- */
int trstmi_ctx_create(int device, trstmi_ctx** out);
int trstmi_ctx_destroy(trstmi_ctx* ctx);
const char* trstmi_last_error(const trstmi_ctx* ctx);
int trstmi_version(void);
/* Number of kernels this library has launched (all contexts, all threads). */
long long trstmi_launch_count(void);
/* FP64 roofline denominator: measured DFMA throughput of the device (TFLOP/s). */
int trstmi_measure_dfma_peak(trstmi_ctx* ctx, int iters, double* tflops);

/* Self tests: device CAS exp (which = 0) / log (1) on host arrays (hypot (2):
 * x holds n (re, im) pairs, y receives n magnitudes), and the
 * Markstein division used by the kernels vs IEEE division on n seeded pairs. */
int trstmi_selftest_cas_math(trstmi_ctx* ctx, int which, const double* x, double* y, int64_t n);
int trstmi_selftest_division(trstmi_ctx* ctx, int64_t n, uint64_t seed, uint64_t* mismatches);

/* ---- single-frame row-block sharding (large-frame path) ----
 * The frame's Gram rows are split into 64-row blocks over `world` ranks; each
 * rank computes the tiles touching its rows, its z-block partials and its
 * gradient columns; the exchanges (max s, z partials, gradient slices) are
 * NCCL collectives.  Results are bit-identical for every world size.
 * nccl_id == NULL with world > 1 runs `world` virtual ranks on this device
 * (each with its own workspace) — the single-GPU test of the partitioning. */
int trstmi_nccl_unique_id(char* out128);
int trstmi_set_shard(trstmi_ctx* ctx, int world, int rank, const char* nccl_id);

/* CAS reduction width S used for a shape: the lane count of
 * every dot / norm / z-sum.  The oracle takes the same S. */
int trstmi_lanes(int field, int64_t d, int64_t N);
/* CAS gradient k-chunk count K for a shape. */
int trstmi_kchunks(int field, int64_t d, int64_t N);
/* Kernel layout chosen for a shape (does not change any result bit):
 * -1 large-frame path, 0 small path with the Gram recomputed in the
 * gradient, 1 small path with stored Gram, 2 stored Gram in bank-padded rows. */
int trstmi_small_layout(int field, int64_t d, int64_t N);
/* Fills cfg with the reference defaults (trust_region.hpp:20-30, solver.hpp:21-29). */
void trstmi_cfg_defaults(trstmi_cfg* cfg, int field, int d, int N);
double trstmi_welch_bound(int64_t d, int64_t N);
/* Returns the number of stages (<= cap) or -1 on invalid input. */
int trstmi_default_schedule(int64_t N, double eps_target, double* out, int cap);
/* Seeded start frames of trials [first, first+count): trial i uses
 * SplitMix64(mix_seed(seed, i)) and random_frame (real: normal() entries).
 * rng_state (nullable) receives {state, has_spare, spare-bits} per trial for
 * the stage-boundary rescue. Host-only (Box-Muller uses libm). */
int trstmi_random_frames(int field, int64_t d, int64_t N, uint64_t seed, int64_t first, int64_t count,
                         double* frames, uint64_t* rng_state);
/* random_frame (solver.hpp:87-98) from the plain generator SplitMix64(rng_seed)
 * (no child-seed mixing): the start of alternating_projection(d, N, cfg, rng),
 * baseline.hpp:84, and of the reference's tests that seed a generator directly. */
int trstmi_random_frame_seeded(int field, int64_t d, int64_t N, uint64_t rng_seed, double* frame);

/* ---- objective / gradient (eval_objective at B points) ----
 * pts: B x dim.  delta: B values.  squared: 1 (solver mode) or 0 (magnitude).
 * F, s: B values.  grad: B x dim.  weights: nullable, B x N(N-1)/2 softmax
 * weights.  zero_col: B values, -1 or the first zero column (the point's F is
 * +inf and its gradient zero, as make_objective returns).  Status is OK even
 * when some points hit a zero column. */
int trstmi_eval_batch(trstmi_ctx* ctx, int field, int64_t d, int64_t N, int64_t B, const double* pts,
                      const double* delta, int squared, double* F, double* s, double* grad, double* weights,
                      int64_t* zero_col);
int trstmi_eval_batch_dev(trstmi_ctx* ctx, int field, int64_t d, int64_t N, int64_t B, const double* pts,
                          const double* delta, int squared, double* F, double* s, double* grad, double* weights,
                          int64_t* zero_col, void* stream);

/* ---- Hessian-vector products (make_hvp_factory semantics) ----
 * hv: B x dim; path: B values (TRSTMI_HVP_*); zero_col: B values. */
int trstmi_hvp_batch(trstmi_ctx* ctx, int field, int64_t d, int64_t N, int64_t B, const double* pts,
                     const double* dirs, const double* delta, double* hv, int32_t* path, int64_t* zero_col);

/* ---- exact coherence + argmax pair ----
 * normalize = 1: normalize_columns first (zero columns reported in zero_col);
 * normalize = 0: the frame is used as given (coherence() semantics). */
int trstmi_coherence_batch(trstmi_ctx* ctx, int field, int64_t d, int64_t N, int64_t B, const double* frames,
                           int normalize, double* mu, int64_t* argmax_pair, int64_t* zero_col);

/* ---- batched anneal: the hot path ----
 * Runs anneal() for `trials` independent start frames, one trust-region
 * state machine per trial on the GPU.  params (trials x dim, in/out): start
 * frames in, best-seen raw parameters out.  frames (out, nullable): the
 * normalised final frames.  rng_state (in/out, nullable): per-trial
 * SplitMix64 state for the stage-boundary rescue (NULL == anneal(start, cfg)
 * without a rescue generator).  stage_out: trials x n_stages.  outer_out
 * (nullable): trials x cfg->record_cap. */
int trstmi_solve_batch(trstmi_ctx* ctx, const trstmi_cfg* cfg, int64_t trials, double* params,
                       uint64_t* rng_state, double* frames, trstmi_trial_out* trial_out,
                       trstmi_stage_out* stage_out, trstmi_outer_out* outer_out);
/* Device-pointer variant (params/frames/outputs on the device; rng_state on
 * the host).  Synchronises the stream before returning. */
int trstmi_solve_batch_dev(trstmi_ctx* ctx, const trstmi_cfg* cfg, int64_t trials, double* params_dev,
                           uint64_t* rng_state, double* frames_dev, trstmi_trial_out* trial_out_dev,
                           trstmi_stage_out* stage_out_dev, trstmi_outer_out* outer_out_dev, void* stream);

/* ---- multistart solve (solve(), solver.hpp:210-273) over restarts
 * [first, first+restarts) of `seed`'s child-seed sequence.  best_frame: dim
 * doubles.  trial_out / stage_out (nullable) as above.  best_restart is the
 * lowest index among the minimum coherences. */
int trstmi_solve(trstmi_ctx* ctx, const trstmi_cfg* cfg, int64_t restarts, uint64_t seed, int64_t first,
                 double* best_frame, double* best_coherence, int64_t* best_restart, trstmi_trial_out* trial_out,
                 trstmi_stage_out* stage_out);

/* ---- multi-GPU trial scheduler (solve()'s restart pool and
 * best-of selection, solver.hpp:210-273, across one process per GPU) ----
 * Restart i runs on rank floor(i * world / restarts): rank r owns the
 * contiguous block [first, first + count). */
int trstmi_shard_range(int64_t restarts, int world, int rank, int64_t* first, int64_t* count);
/* Best-of rule of solve() (solver.hpp:256-263): the minimum mu over entries
 * with ok != 0 (ok nullable = all) and mu not NaN, lowest index (index
 * nullable = position) on ties.  ALL_FAILED when there is none. */
int trstmi_select_best(int64_t n, const double* mu, const int64_t* index, const int32_t* ok, int64_t* best_pos);
/* Attach an NCCL communicator (128-byte ncclUniqueId from
 * trstmi_nccl_unique_id on rank 0, shared by the caller) to the context;
 * world == 1 needs no id. */
int trstmi_comm_init(trstmi_ctx* ctx, int world, int rank, const char* nccl_id);
/* Cross-rank best-of: NCCL allgather of every rank's (local_mu, local_index)
 * (NaN mu = no successful trial on that rank), selection by
 * trstmi_select_best, then the owner broadcasts its frame (device pointers,
 * dim doubles) into best_frame_dev on every rank. */
int trstmi_best_of_ranks(trstmi_ctx* ctx, int64_t dim, double local_mu, int64_t local_index,
                         const double* local_frame_dev, double* best_frame_dev, double* best_mu,
                         int64_t* best_index, void* stream);
/* solve() over the context's ranks: this rank's block of restarts
 * (trstmi_shard_range) annealed on its GPU, then trstmi_best_of_ranks.  Every
 * rank returns the same best frame / coherence / restart.  local_trial_out
 * (nullable): the block's records (local_count entries). */
int trstmi_solve_sharded(trstmi_ctx* ctx, const trstmi_cfg* cfg, int64_t restarts, uint64_t seed, double* best_frame,
                         double* best_coherence, int64_t* best_restart, trstmi_trial_out* local_trial_out,
                         int64_t* local_first, int64_t* local_count);
/* solve() over several GPUs of one process (the reference's restart pool with
 * one worker per GPU, solver.hpp:239-254): one host thread and one context per
 * entry of `devices` (a device may repeat for small frames; the large-frame
 * engine sizes its lanes to the device's free memory, so list each GPU once
 * there), restart blocks by
 * trstmi_shard_range, best-of on the host in restart order (strict <), no NCCL.
 * The result equals trstmi_solve's bit for bit for any device list.  trial_out
 * (restarts entries) / stage_out (restarts x stages) nullable. */
int trstmi_solve_devices(const int* devices, int ndev, const trstmi_cfg* cfg, int64_t restarts, uint64_t seed,
                         double* best_frame, double* best_coherence, int64_t* best_restart,
                         trstmi_trial_out* trial_out, trstmi_stage_out* stage_out);

/* Child seed of restart `index` (mix_seed, rng.hpp:13-18): RestartRecord::seed. */
uint64_t trstmi_mix_seed(uint64_t seed, uint64_t index);

/* ---- post-solve analysis (csrc/analysis.cu).  Host
 * buffers; run on the default stream and synchronise.  No context needed. */
/* offdiagonal_magnitudes (frame.hpp:80-91): n = N(N-1)/2 magnitudes |G(j,k)|
 * in row-major upper-triangular order into mags (nullable); sorted_mags
 * (nullable) receives them in ascending order (device sort).  normalize != 0
 * first applies normalize_columns (frame.hpp:60-69): ZERO_COLUMN + *zero_col. */
int trstmi_offdiag_magnitudes(int field, int64_t d, int64_t N, const double* frame, int normalize, double* mags,
                              double* sorted_mags, int64_t* zero_col);
/* normalize_columns (frame.hpp:60-69) in place (CAS norm, IEEE-exact division);
 * ZERO_COLUMN with *zero_col = the first column whose norm is < 1e-12. */
int trstmi_normalize_columns(int field, int64_t d, int64_t N, double* frame, int64_t* zero_col);
/* cluster_magnitudes (frame.hpp:96-118) over an ascending array: means of the
 * single-linkage clusters (gap > cluster_tol), sequential sums; *count means. */
int trstmi_cluster_sorted(const double* sorted, int64_t n, double cluster_tol, double* means, int64_t* count);
/* distortion_mc (beamforming.hpp:78-163): Monte-Carlo quantisation
 * distortion E[1 - max_i |<phi_i, h>|^2 / |h|^2] of a complex d x N codebook
 * (interleaved, unit columns) over samples channels h ~ CN(0, I), blocks of
 * 4096 samples each with SplitMix64(mix_seed(seed, block)).  GPU Box-Muller
 * (CUDA log/sin/cos): within an ulp of the reference's draws. */
int trstmi_distortion_mc(int64_t d, int64_t N, const double* codebook, uint64_t samples, uint64_t seed,
                         double* estimate, double* std_error);
/* check_tight's deviation (analysis.hpp:76-84): max |(Phi Phi*)(r,s) - (N/d) I| */
int trstmi_frame_operator_deviation(int field, int64_t d, int64_t N, const double* frame, double* deviation);

/* ---- alternating-projection baseline (csrc/altproj.cu).
 * alternating_projection (baseline.hpp:68-167) for `restarts` complex d x N start
 * frames (restarts x 2dN doubles, interleaved column-major; restart i of
 * solve_altproj, baseline.hpp:172-199, starts from random_frame of the child
 * generator mix_seed(seed, i): trstmi_random_frames(TRSTMI_COMPLEX, ...)).
 * One CTA per restart.  mu_target 0 -> max(welch_bound(d, N), 1e-12); tol =
 * AltProjConfig::tol (max-entry change of the Gram).  Outputs per restart: the
 * result frame (the converged iterate, else the best seen), its coherence,
 * iterations (> 0: converged after that many, < 0: best of -iterations, the
 * sign convention of StageRecord::outer_iterations, baseline.hpp:156) and the
 * Jacobi sweeps spent (nullable).  INVALID_ARG where the reference throws
 * std::invalid_argument (d > N, max_iters < 1, mu_target >= 1) and for N > 256. */
int trstmi_altproj_batch(int64_t d, int64_t N, int32_t max_iters, double mu_target, double tol, int64_t restarts,
                         const double* starts, double* frames, double* coherence, int32_t* iterations,
                         int32_t* sweeps);

#ifdef __cplusplus
}
#endif

#endif /* TRSTMI_B200_H */
