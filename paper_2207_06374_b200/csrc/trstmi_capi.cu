// C ABI (include/trstmi_b200.h) over the B200 kernels.  Host logic only:
// argument validation with the reference's error semantics, device
// workspaces, kernel-family dispatch, the rescue loop of the batched anneal
// and the multistart best-of selection (solver.hpp:256-267).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <map>
#include <mutex>
#include <thread>
#include <string>
#include <vector>

#include "../../include/trstmi_b200.h"
#include "batch_kernels.cuh"
#include "host/host_common.hpp"
#include "kernel_table.hpp"
#include "large_engine.hpp"
#include "ctx.hpp"

using namespace trstmi_dev;

static long long g_launches = 0;  // kernels launched by this library (bench.py gpu_launches)

// DFMA throughput probe (bench.py's FP64 roofline denominator): each thread
// runs 8 independent fma chains.
__global__ void dfma_peak_kernel(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  const double r = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (r == 12345.678) out[0] = r;
}

// Self-test kernels: device CAS transcendentals on caller data, and the
// Markstein division against the hardware IEEE division on a seeded stream.
__global__ void cas_math_kernel(const double* x, double* y, long long n, int which) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    y[i] = which == 0 ? cas_exp(x[i]) : which == 1 ? cas_log(x[i]) : cas_hypot(x[2 * i], x[2 * i + 1]);
}

__device__ __forceinline__ unsigned long long sm64(unsigned long long& s) {
  unsigned long long z = (s += 0x9E3779B97F4A7C15ULL);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

__global__ void div_selftest_kernel(long long n, unsigned long long seed, unsigned long long* bad) {
  unsigned long long s = seed ^ (0x632BE59BD9B4E019ULL * (blockIdx.x * (long long)blockDim.x + threadIdx.x + 1));
  unsigned long long nb = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    // numerators: random significand, exponent in [-80, 20]; sign random;
    // denominators: random significand, exponent in [-45, 15] (covers delta, z, alpha)
    const unsigned long long r1 = sm64(s), r2 = sm64(s), r3 = sm64(s);
    const double a = __longlong_as_double((long long)((r1 & 0x800fffffffffffffULL) |
                                                      ((unsigned long long)(1023 - 80 + (r3 % 101)) << 52)));
    const double b = __longlong_as_double((long long)((r2 & 0x000fffffffffffffULL) |
                                                      ((unsigned long long)(1023 - 45 + ((r3 >> 20) % 61)) << 52)));
    const double q = div_rn(a, b, __drcp_rn(b));
    if (__double_as_longlong(q) != __double_as_longlong(__ddiv_rn(a, b))) ++nb;
  }
  if (nb) atomicAdd(bad, nb);
}

// ------------------------------------------------------------------ path rule
// Small-frame kernel choice for a shape: CTA width S (= the CAS reduction
// width) and pair layout.  Candidates in order; the first whose anneal
// shared memory fits one SM (227 KB) wins, none -> the large-frame path.
//   dim <= 64      S = 64   stored Gram (padded / unpadded)
//   dim <= 256     S = 128  stored Gram, else Gram recomputed
//   larger         S = 512  stored Gram when even S = 256 leaves one CTA per
//                           SM (16 warps instead of 8); S = 128 stored Gram
//                           when there are <= 2048 pairs (4 trials per SM hide
//                           the fixed per-evaluation costs); else S = 256
//                           stored Gram, else recomputed
struct SmallMode {
  bool ok;
  int S, gs, pad;
};

static long long small_bytes(int field, long long d, long long N, int S, int gs, int pad) {
  const Prob P = make_small_prob(field == TRSTMI_COMPLEX, (int)d, (int)N, kchunks_for((int)d, (int)N, S), gs, pad);
  return anneal_smem_doubles(P, S, field == TRSTMI_COMPLEX) * 8;
}

static SmallMode small_mode(int field, long long d, long long N) {
  SmallMode m{false, 0, 0, 0};
  if (d > 16 || N > 4096) return m;
  const long long dim = (field == TRSTMI_COMPLEX ? 2 : 1) * d * N;
  const long long kMax = 227LL * 1024;
  const bool gs_ok = N <= 256 && gs_phys_slots((int)N, 1) <= 65536;  // packed pair table limits
  int cand[8][3];
  int nc = 0;
  auto add = [&](int S, int gs, int pad) {
    if (gs && !gs_ok) return;
    cand[nc][0] = S;
    cand[nc][1] = gs;
    cand[nc][2] = pad;
    ++nc;
  };
  if (dim <= 64) {
    add(64, 1, 1);  // tiny frames: per-trial latency binds (config 1 runs 64 trials on 148 SMs)
    add(64, 1, 0);
  } else if (dim <= 256) {
    add(128, 1, 1);
    add(128, 1, 0);
    add(128, 0, 0);
  } else {
    if (gs_ok && small_bytes(field, d, N, 256, 1, 1) > kMax / 2) {
      add(512, 1, 1);
      add(512, 1, 0);
    }
    if (N * (N - 1) / 2 <= 2048) {  // few pairs: fixed per-evaluation costs bind -> 4 trials per SM
      add(128, 1, 1);
      add(128, 1, 0);
    }
    add(256, 1, 1);
    add(256, 1, 0);
    add(256, 0, 0);
  }
  for (int i = 0; i < nc; ++i) {
    if (small_bytes(field, d, N, cand[i][0], cand[i][1], cand[i][2]) <= kMax) {
      m.ok = true;
      m.S = cand[i][0];
      m.gs = cand[i][1];
      m.pad = cand[i][2];
      return m;
    }
  }
  return m;
}

static int small_lanes(int field, long long d, long long N) { return small_mode(field, d, N).S; }

static bool small_fits(int field, long long d, long long N) { return small_mode(field, d, N).ok; }

bool trstmi_large::use_large(int field, long long d, long long N) { return !small_fits(field, d, N); }

namespace {

int fail(trstmi_ctx* ctx, int code, const std::string& msg) {
  if (ctx) ctx->err = msg;
  return code;
}

#define CUDA_TRY(ctx, expr)                                                                \
  do {                                                                                     \
    cudaError_t e_ = (expr);                                                               \
    if (e_ != cudaSuccess) return fail((ctx), TRSTMI_ERR_CUDA, std::string(#expr ": ") + cudaGetErrorString(e_)); \
  } while (0)

Prob make_prob(int field, long long d, long long N) {
  const SmallMode m = small_mode(field, d, N);
  if (!m.ok) {  // large path shapes: the fields the host code reads
    Prob P = make_small_prob(field == TRSTMI_COMPLEX, (int)d, (int)N, 1, 0, 0);
    P.K = kchunks_for(P.d, P.N, trstmi_lanes(field, d, N));
    return P;
  }
  return make_small_prob(field == TRSTMI_COMPLEX, (int)d, (int)N, kchunks_for((int)d, (int)N, m.S), m.gs, m.pad);
}

int check_shape(trstmi_ctx* ctx, int field, long long d, long long N, const char* who) {
  if (field != TRSTMI_COMPLEX && field != TRSTMI_REAL) return fail(ctx, TRSTMI_ERR_INVALID_ARG, std::string(who) + ": bad field");
  if (d < 1) return fail(ctx, TRSTMI_ERR_INVALID_ARG, std::string(who) + ": need d >= 1");
  if (N < 2) return fail(ctx, TRSTMI_ERR_INVALID_ARG, std::string(who) + ": need N >= 2");
  if (N > 16384 || d > 4096) return fail(ctx, TRSTMI_ERR_UNSUPPORTED, std::string(who) + ": N > 16384 or d > 4096");
  return TRSTMI_OK;
}

// Device buffer RAII for the host-pointer entry points.
struct DBuf {
  void* p = nullptr;
  ~DBuf() {
    if (p) cudaFree(p);
  }
};

}  // namespace

extern "C" {

int trstmi_version(void) { return 1; }

long long trstmi_launch_count(void) { return g_launches + trstmi_large::launches() + trstmi_bde_host::launches(); }

// Measured FP64 FMA peak of the device (TFLOP/s, 2 flops per fma), timed with
// CUDA events over `iters` x 128 fma per thread on a full-occupancy grid.
int trstmi_measure_dfma_peak(trstmi_ctx* ctx, int iters, double* tflops) {
  if (!ctx) return TRSTMI_ERR_INVALID_ARG;
  cudaSetDevice(ctx->device);
  double* out = nullptr;
  CUDA_TRY(ctx, cudaMalloc(&out, 8));
  const int threads = 256;
  const int blocks = ctx->sm_count * 8;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  dfma_peak_kernel<<<blocks, threads, 0, ctx->stream>>>(out, iters / 4 + 1, 0.999999, 1e-7);  // warm-up
  cudaEventRecord(e0, ctx->stream);
  dfma_peak_kernel<<<blocks, threads, 0, ctx->stream>>>(out, iters, 0.999999, 1e-7);
  cudaEventRecord(e1, ctx->stream);
  CUDA_TRY(ctx, cudaEventSynchronize(e1));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  const double flops = 2.0 * 8 * 16 * (double)iters * threads * blocks;
  *tflops = flops / (ms * 1e-3) / 1e12;
  return TRSTMI_OK;
}

int trstmi_selftest_cas_math(trstmi_ctx* ctx, int which, const double* x, double* y, int64_t n) {
  if (!ctx || n < 0) return TRSTMI_ERR_INVALID_ARG;
  cudaSetDevice(ctx->device);
  DBuf dx, dy;
  const int64_t nin = which == 2 ? 2 * n : n;  // hypot: n (x, y) pairs
  CUDA_TRY(ctx, cudaMalloc(&dx.p, std::max<int64_t>(nin, 1) * 8));
  CUDA_TRY(ctx, cudaMalloc(&dy.p, std::max<int64_t>(n, 1) * 8));
  // every copy on the context's (non-blocking) stream: a legacy-stream
  // cudaMemcpy is not ordered with it and may still be in flight
  CUDA_TRY(ctx, cudaMemcpyAsync(dx.p, x, nin * 8, cudaMemcpyHostToDevice, ctx->stream));
  cas_math_kernel<<<ctx->sm_count * 4, 256, 0, ctx->stream>>>((const double*)dx.p, (double*)dy.p, n, which);
  CUDA_TRY(ctx, cudaGetLastError());
  CUDA_TRY(ctx, cudaMemcpyAsync(y, dy.p, n * 8, cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  return TRSTMI_OK;
}

int trstmi_selftest_division(trstmi_ctx* ctx, int64_t n, uint64_t seed, uint64_t* mismatches) {
  if (!ctx) return TRSTMI_ERR_INVALID_ARG;
  cudaSetDevice(ctx->device);
  DBuf db;
  CUDA_TRY(ctx, cudaMalloc(&db.p, 8));
  CUDA_TRY(ctx, cudaMemsetAsync(db.p, 0, 8, ctx->stream));
  div_selftest_kernel<<<ctx->sm_count * 8, 256, 0, ctx->stream>>>(n, seed, (unsigned long long*)db.p);
  CUDA_TRY(ctx, cudaGetLastError());
  CUDA_TRY(ctx, cudaMemcpyAsync(mismatches, db.p, 8, cudaMemcpyDeviceToHost, ctx->stream));
  CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  return TRSTMI_OK;
}

static trstmi_large::Engine* large_engine(trstmi_ctx* ctx, cudaStream_t st);

int trstmi_nccl_unique_id(char* out128) {
  std::string e;
  return trstmi_large::nccl_unique_id(out128, &e);
}

int trstmi_set_shard(trstmi_ctx* ctx, int world, int rank, const char* nccl_id) {
  if (!ctx || world < 1 || rank < 0 || rank >= world) return TRSTMI_ERR_INVALID_ARG;
  cudaSetDevice(ctx->device);
  trstmi_large::Engine* E = large_engine(ctx, ctx->stream);
  const int rc = trstmi_large::engine_set_shard(E, world, rank, nccl_id, &ctx->err);
  if (rc == TRSTMI_OK) ctx->shard_world = world;
  return rc;
}

uint64_t trstmi_mix_seed(uint64_t seed, uint64_t index) { return trstmi_host::mix_seed(seed, index); }

int trstmi_small_layout(int field, int64_t d, int64_t N) {
  const SmallMode m = small_mode(field, d, N);
  if (!m.ok) return -1;
  return m.gs ? 1 + m.pad : 0;
}

int trstmi_kchunks(int field, int64_t d, int64_t N) { return kchunks_for((int)d, (int)N, trstmi_lanes(field, d, N)); }

int trstmi_lanes(int field, int64_t d, int64_t N) {
  if (trstmi_large::use_large(field, d, N)) return trstmi_large::kLanes;
  return small_lanes(field, d, N);
}

void trstmi_cfg_defaults(trstmi_cfg* c, int field, int d, int N) {
  std::memset(c, 0, sizeof(*c));
  c->field = field;
  c->d = d;
  c->N = N;
  c->n_stages = 0;
  c->eps_target = 1e-7;
  c->delta0 = 0.0;
  c->delta_max = 1e3;
  c->eta = 0.05;
  c->shrink = 0.25;
  c->grow = 2.0;
  c->grad_tol = 1e-9;
  c->max_outer = 200;
  c->max_cg = 0;
  c->cg_force_c = 0.5;
  c->record_cap = 0;
}

double trstmi_welch_bound(int64_t d, int64_t N) { return trstmi_host::welch_bound(d, N); }

int trstmi_default_schedule(int64_t N, double eps_target, double* out, int cap) {
  try {
    std::vector<double> s = trstmi_host::default_delta_schedule(N, eps_target);
    for (int i = 0; i < (int)s.size() && i < cap; ++i) out[i] = s[i];
    return (int)s.size();
  } catch (...) {
    return -1;
  }
}

int trstmi_random_frames(int field, int64_t d, int64_t N, uint64_t seed, int64_t first, int64_t count, double* frames,
                         uint64_t* rng_state) {
  if (d < 1 || N < 1 || count < 0) return TRSTMI_ERR_INVALID_ARG;
  const int64_t dim = (field == TRSTMI_COMPLEX ? 2 : 1) * d * N;
  for (int64_t t = 0; t < count; ++t) {
    trstmi_host::SplitMix64 rng(trstmi_host::mix_seed(seed, (uint64_t)(first + t)));
    trstmi_host::random_frame(field == TRSTMI_COMPLEX, d, N, rng, frames + t * dim);
    if (rng_state) rng.save(rng_state + 3 * t);
  }
  return TRSTMI_OK;
}

int trstmi_random_frame_seeded(int field, int64_t d, int64_t N, uint64_t rng_seed, double* frame) {
  if (d < 1 || N < 1 || !frame) return TRSTMI_ERR_INVALID_ARG;
  trstmi_host::SplitMix64 rng(rng_seed);
  trstmi_host::random_frame(field == TRSTMI_COMPLEX, d, N, rng, frame);
  return TRSTMI_OK;
}

int trstmi_ctx_create(int device, trstmi_ctx** out) {
  *out = nullptr;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    return TRSTMI_ERR_NO_DEVICE;
  }
  if (device < 0 || device >= n) return TRSTMI_ERR_INVALID_ARG;
  trstmi_ctx* ctx = new trstmi_ctx();
  ctx->device = device;
  if (cudaSetDevice(device) != cudaSuccess) {
    delete ctx;
    return TRSTMI_ERR_CUDA;
  }
  cudaDeviceGetAttribute(&ctx->sm_count, cudaDevAttrMultiProcessorCount, device);
  if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaMalloc(&ctx->counter, 64 * sizeof(int)) != cudaSuccess) {
    delete ctx;
    return TRSTMI_ERR_CUDA;
  }
  *out = ctx;
  return TRSTMI_OK;
}

int trstmi_ctx_destroy(trstmi_ctx* ctx) {
  if (!ctx) return TRSTMI_OK;
  cudaSetDevice(ctx->device);
  if (ctx->counter) cudaFree(ctx->counter);
  if (ctx->comm) ncclCommDestroy(ctx->comm);
  if (ctx->large) trstmi_large::engine_destroy(ctx->large);
  if (ctx->bde) trstmi_bde_host::destroy(ctx->bde);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
  return TRSTMI_OK;
}

const char* trstmi_last_error(const trstmi_ctx* ctx) { return ctx ? ctx->err.c_str() : "no context"; }

// concurrent large-path trials (host worker + stream + workspace each);
// TRSTMI_LARGE_WORKERS overrides the context default
static int large_workers(const trstmi_ctx* ctx) {
  const char* e = std::getenv("TRSTMI_LARGE_WORKERS");
  const int v = e ? std::atoi(e) : 0;
  return v > 0 ? v : ctx->large_workers;
}

// The context's large-frame engine, bound to the stream of the current call
// (every entry point passes its own: the caller's for *_dev, else ctx->stream,
// which also carries that call's H2D copies).
static trstmi_large::Engine* large_engine(trstmi_ctx* ctx, cudaStream_t st) {
  if (!ctx->large) ctx->large = trstmi_large::engine_create(ctx->device, st);
  trstmi_large::engine_set_stream(ctx->large, st);
  return ctx->large;
}

static trstmi_bde_host::Engine* bde_engine(trstmi_ctx* ctx) {
  if (!ctx->bde) ctx->bde = trstmi_bde_host::create(ctx->device);
  return ctx->bde;
}

// Dynamic shared-memory opt-in of a kernel: the attribute is per function and device and shared by every host thread,
// so it is only ever raised (a launch of a smaller shape from another thread must not lower it under a launch in
// flight: trstmi_solve_devices, multi-threaded callers).
static cudaError_t raise_smem_optin(int device, const void* fn, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> have;
  std::lock_guard<std::mutex> lock(mu);
  size_t& cur = have[{device, fn}];
  if (bytes <= cur) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) cur = bytes;
  return e;
}

// ------------------------------------------------------------------ eval / hvp / coherence
static int batch_launch(trstmi_ctx* ctx, int kind, int field, int64_t d, int64_t N, BatchArgs& A, cudaStream_t st) {
  const int S = trstmi_lanes(field, d, N);
  const KernelSet* ks = find_kernels(field == TRSTMI_COMPLEX, (int)d, S, A.P.gs);
  if (!ks) return fail(ctx, TRSTMI_ERR_UNSUPPORTED, "no kernel family for this shape");
  const void* fn = kind == 0 ? ks->eval : kind == 1 ? ks->hvp : ks->coherence;
  A.P.dual = 0;
  if (kind == 1 && A.P.gs && A.P.dim <= kGsDualElems * S && !std::getenv("TRSTMI_NO_DUAL")) {
    Prob Pd = A.P;  // fused central difference (hvp_cta_gs) where its second set of columns fits
    Pd.dual = 1;
    if (smem_doubles(Pd, S, field == TRSTMI_COMPLEX, 3) * (long long)sizeof(double) <= 227 * 1024) A.P.dual = 1;
  }
  const long long dbl = smem_doubles(A.P, S, field == TRSTMI_COMPLEX, kind == 2 ? 0 : 3);
  const size_t bytes = (size_t)dbl * sizeof(double);
  if (bytes > 227 * 1024) return fail(ctx, TRSTMI_ERR_UNSUPPORTED, "frame too large for the small-frame kernels");
  CUDA_TRY(ctx, raise_smem_optin(ctx->device, fn, bytes));
  const long long grid = std::min<long long>(A.B, 65535LL);
  if (grid <= 0) return TRSTMI_OK;
  void* args[] = {&A};
  CUDA_TRY(ctx, cudaLaunchKernel(fn, dim3((unsigned)grid), dim3(S), args, bytes, st));
  CUDA_TRY(ctx, cudaGetLastError());
  ++g_launches;
  return TRSTMI_OK;
}

int trstmi_eval_batch_dev(trstmi_ctx* ctx, int field, int64_t d, int64_t N, int64_t B, const double* pts,
                          const double* delta, int squared, double* F, double* s, double* grad, double* weights,
                          int64_t* zero_col, void* stream) {
  if (!ctx) return TRSTMI_ERR_INVALID_ARG;
  int rc = check_shape(ctx, field, d, N, "eval_objective");
  if (rc) return rc;
  cudaSetDevice(ctx->device);
  if (trstmi_large::use_large(field, d, N) && ctx->shard_world == 1) {  // batched engine: all B points at once
    cudaStream_t st = (cudaStream_t)stream;
    std::vector<double> hd(B), hF(B), hs(B);
    std::vector<long long> hz(B);
    CUDA_TRY(ctx, cudaMemcpyAsync(hd.data(), delta, B * sizeof(double), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(ctx, cudaStreamSynchronize(st));
    const int r2 = trstmi_bde_host::eval_points(bde_engine(ctx), st, field, (int)d, (int)N, (int)B, pts, nullptr, nullptr,
                                                hd.data(), squared, grad, weights, hF.data(), hs.data(), hz.data(),
                                                &ctx->err);
    if (r2) return r2;
    CUDA_TRY(ctx, cudaMemcpyAsync(F, hF.data(), B * sizeof(double), cudaMemcpyHostToDevice, st));
    CUDA_TRY(ctx, cudaMemcpyAsync(s, hs.data(), B * sizeof(double), cudaMemcpyHostToDevice, st));
    CUDA_TRY(ctx, cudaMemcpyAsync(zero_col, hz.data(), B * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    CUDA_TRY(ctx, cudaStreamSynchronize(st));
    return TRSTMI_OK;
  }
  if (trstmi_large::use_large(field, d, N)) {
    const trstmi_large::Shape sh = trstmi_large::make_shape(field, (int)d, (int)N);
    cudaStream_t st = (cudaStream_t)stream;
    trstmi_large::Engine* E = large_engine(ctx, st);
    std::vector<double> hd(B), hF(B), hs(B);
    std::vector<int64_t> hz(B);
    CUDA_TRY(ctx, cudaMemcpyAsync(hd.data(), delta, B * sizeof(double), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(ctx, cudaStreamSynchronize(st));
    for (int64_t b = 0; b < B; ++b) {
      long long zc;
      int r2 = trstmi_large::eval(E, sh, pts + b * sh.dim, nullptr, 0.0, hd[b], squared, grad + b * sh.dim, &hF[b],
                                  &hs[b], weights ? weights + b * sh.n : nullptr, &zc, &ctx->err);
      if (r2) return r2;
      hz[b] = zc;
    }
    CUDA_TRY(ctx, cudaMemcpyAsync(F, hF.data(), B * sizeof(double), cudaMemcpyHostToDevice, st));
    CUDA_TRY(ctx, cudaMemcpyAsync(s, hs.data(), B * sizeof(double), cudaMemcpyHostToDevice, st));
    CUDA_TRY(ctx, cudaMemcpyAsync(zero_col, hz.data(), B * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    CUDA_TRY(ctx, cudaStreamSynchronize(st));
    return TRSTMI_OK;
  }
  BatchArgs A{};
  A.P = make_prob(field, d, N);
  A.B = B;
  A.pts = pts;
  A.delta = delta;
  A.squared = squared;
  A.F = F;
  A.s = s;
  A.out = grad;
  A.weights = weights;
  A.zero_col = reinterpret_cast<long long*>(zero_col);
  cudaSetDevice(ctx->device);
  return batch_launch(ctx, 0, field, d, N, A, (cudaStream_t)stream);
}

int trstmi_eval_batch(trstmi_ctx* ctx, int field, int64_t d, int64_t N, int64_t B, const double* pts,
                      const double* delta, int squared, double* F, double* s, double* grad, double* weights,
                      int64_t* zero_col) {
  if (!ctx) return TRSTMI_ERR_INVALID_ARG;
  int rc = check_shape(ctx, field, d, N, "eval_objective");
  if (rc) return rc;
  for (int64_t b = 0; b < B; ++b)
    if (!(delta[b] > 0.0)) return fail(ctx, TRSTMI_ERR_INVALID_ARG, "eval_objective: delta <= 0");
  cudaSetDevice(ctx->device);
  const Prob P = make_prob(field, d, N);
  const size_t vb = (size_t)B * P.dim * sizeof(double);
  DBuf dp, dd, dF, ds, dg, dw, dz;
  CUDA_TRY(ctx, cudaMalloc(&dp.p, vb));
  CUDA_TRY(ctx, cudaMalloc(&dd.p, B * sizeof(double)));
  CUDA_TRY(ctx, cudaMalloc(&dF.p, B * sizeof(double)));
  CUDA_TRY(ctx, cudaMalloc(&ds.p, B * sizeof(double)));
  CUDA_TRY(ctx, cudaMalloc(&dg.p, vb));
  CUDA_TRY(ctx, cudaMalloc(&dz.p, B * sizeof(int64_t)));
  if (weights) CUDA_TRY(ctx, cudaMalloc(&dw.p, (size_t)B * P.n * sizeof(double)));
  cudaStream_t st = ctx->stream;
  CUDA_TRY(ctx, cudaMemcpyAsync(dp.p, pts, vb, cudaMemcpyHostToDevice, st));
  CUDA_TRY(ctx, cudaMemcpyAsync(dd.p, delta, B * sizeof(double), cudaMemcpyHostToDevice, st));
  rc = trstmi_eval_batch_dev(ctx, field, d, N, B, (double*)dp.p, (double*)dd.p, squared, (double*)dF.p, (double*)ds.p,
                             (double*)dg.p, (double*)dw.p, (int64_t*)dz.p, st);
  if (rc) return rc;
  CUDA_TRY(ctx, cudaMemcpyAsync(F, dF.p, B * sizeof(double), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(ctx, cudaMemcpyAsync(s, ds.p, B * sizeof(double), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(ctx, cudaMemcpyAsync(grad, dg.p, vb, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(ctx, cudaMemcpyAsync(zero_col, dz.p, B * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  if (weights) CUDA_TRY(ctx, cudaMemcpyAsync(weights, dw.p, (size_t)B * P.n * sizeof(double), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(ctx, cudaStreamSynchronize(st));
  return TRSTMI_OK;
}

int trstmi_hvp_batch(trstmi_ctx* ctx, int field, int64_t d, int64_t N, int64_t B, const double* pts,
                     const double* dirs, const double* delta, double* hv, int32_t* path, int64_t* zero_col) {
  if (!ctx) return TRSTMI_ERR_INVALID_ARG;
  int rc = check_shape(ctx, field, d, N, "hessian_vector_product");
  if (rc) return rc;
  for (int64_t b = 0; b < B; ++b)
    if (!(delta[b] > 0.0)) return fail(ctx, TRSTMI_ERR_INVALID_ARG, "eval_objective: delta <= 0");
  cudaSetDevice(ctx->device);
  const Prob P = make_prob(field, d, N);
  const size_t vb = (size_t)B * P.dim * sizeof(double);
  DBuf dp, dr, dd, dh, dpa, dz;
  CUDA_TRY(ctx, cudaMalloc(&dp.p, vb));
  CUDA_TRY(ctx, cudaMalloc(&dr.p, vb));
  CUDA_TRY(ctx, cudaMalloc(&dd.p, B * sizeof(double)));
  CUDA_TRY(ctx, cudaMalloc(&dh.p, vb));
  CUDA_TRY(ctx, cudaMalloc(&dpa.p, B * sizeof(int32_t)));
  CUDA_TRY(ctx, cudaMalloc(&dz.p, B * sizeof(int64_t)));
  cudaStream_t st = ctx->stream;
  CUDA_TRY(ctx, cudaMemcpyAsync(dp.p, pts, vb, cudaMemcpyHostToDevice, st));
  CUDA_TRY(ctx, cudaMemcpyAsync(dr.p, dirs, vb, cudaMemcpyHostToDevice, st));
  CUDA_TRY(ctx, cudaMemcpyAsync(dd.p, delta, B * sizeof(double), cudaMemcpyHostToDevice, st));
  if (trstmi_large::use_large(field, d, N) && ctx->shard_world == 1) {
    std::vector<int> hp(B);
    std::vector<long long> hz(B);
    const int r2 = trstmi_bde_host::hvp_points(bde_engine(ctx), st, field, (int)d, (int)N, (int)B, (double*)dp.p,
                                               (double*)dr.p, delta, (double*)dh.p, hp.data(), hz.data(), &ctx->err);
    if (r2) return r2;
    for (int64_t b = 0; b < B; ++b) {
      path[b] = hp[b];
      zero_col[b] = hz[b];
    }
    CUDA_TRY(ctx, cudaMemcpyAsync(hv, dh.p, vb, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(ctx, cudaStreamSynchronize(st));
    return TRSTMI_OK;
  }
  if (trstmi_large::use_large(field, d, N)) {
    const trstmi_large::Shape sh = trstmi_large::make_shape(field, (int)d, (int)N);
    trstmi_large::Engine* E = large_engine(ctx, st);
    for (int64_t b = 0; b < B; ++b) {
      int pth;
      long long zc;
      int r2 = trstmi_large::hvp(E, sh, (double*)dp.p + b * sh.dim, (double*)dr.p + b * sh.dim, delta[b],
                                 (double*)dh.p + b * sh.dim, &pth, &zc, &ctx->err);
      if (r2) return r2;
      path[b] = pth;
      zero_col[b] = zc;
    }
    CUDA_TRY(ctx, cudaMemcpyAsync(hv, dh.p, vb, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(ctx, cudaStreamSynchronize(st));
    return TRSTMI_OK;
  }
  BatchArgs A{};
  A.P = P;
  A.B = B;
  A.pts = (double*)dp.p;
  A.dirs = (double*)dr.p;
  A.delta = (double*)dd.p;
  A.squared = 1;
  A.out = (double*)dh.p;
  A.path = (int*)dpa.p;
  A.zero_col = (long long*)dz.p;
  rc = batch_launch(ctx, 1, field, d, N, A, st);
  if (rc) return rc;
  CUDA_TRY(ctx, cudaMemcpyAsync(hv, dh.p, vb, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(ctx, cudaMemcpyAsync(path, dpa.p, B * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(ctx, cudaMemcpyAsync(zero_col, dz.p, B * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(ctx, cudaStreamSynchronize(st));
  return TRSTMI_OK;
}

int trstmi_coherence_batch(trstmi_ctx* ctx, int field, int64_t d, int64_t N, int64_t B, const double* frames,
                           int normalize, double* mu, int64_t* argmax_pair, int64_t* zero_col) {
  if (!ctx) return TRSTMI_ERR_INVALID_ARG;
  int rc = check_shape(ctx, field, d, N, "coherence");
  if (rc) return rc;
  cudaSetDevice(ctx->device);
  const Prob P = make_prob(field, d, N);
  const size_t vb = (size_t)B * P.dim * sizeof(double);
  DBuf dp, dm, da, dz;
  CUDA_TRY(ctx, cudaMalloc(&dp.p, vb));
  CUDA_TRY(ctx, cudaMalloc(&dm.p, B * sizeof(double)));
  CUDA_TRY(ctx, cudaMalloc(&da.p, B * sizeof(int64_t)));
  CUDA_TRY(ctx, cudaMalloc(&dz.p, B * sizeof(int64_t)));
  cudaStream_t st = ctx->stream;
  CUDA_TRY(ctx, cudaMemcpyAsync(dp.p, frames, vb, cudaMemcpyHostToDevice, st));
  if (trstmi_large::use_large(field, d, N) && ctx->shard_world == 1) {
    std::vector<long long> ha(B), hz(B);
    const int r2 = trstmi_bde_host::coherence_points(bde_engine(ctx), st, field, (int)d, (int)N, (int)B, (double*)dp.p,
                                                     normalize, mu, ha.data(), hz.data(), &ctx->err);
    if (r2) return r2;
    for (int64_t b = 0; b < B; ++b) {
      argmax_pair[b] = ha[b];
      zero_col[b] = hz[b];
    }
    return TRSTMI_OK;
  }
  if (trstmi_large::use_large(field, d, N)) {
    const trstmi_large::Shape sh = trstmi_large::make_shape(field, (int)d, (int)N);
    trstmi_large::Engine* E = large_engine(ctx, st);
    for (int64_t b = 0; b < B; ++b) {
      long long a, zc;
      int r2 = trstmi_large::coherence(E, sh, (double*)dp.p + b * sh.dim, normalize, &mu[b], &a, &zc, &ctx->err);
      if (r2) return r2;
      argmax_pair[b] = a;
      zero_col[b] = zc;
      if (zc >= 0) mu[b] = 0.0;
    }
    return TRSTMI_OK;
  }
  BatchArgs A{};
  A.P = P;
  A.B = B;
  A.pts = (double*)dp.p;
  A.normalize = normalize;
  A.mu = (double*)dm.p;
  A.argmax = (long long*)da.p;
  A.zero_col = (long long*)dz.p;
  rc = batch_launch(ctx, 2, field, d, N, A, st);
  if (rc) return rc;
  CUDA_TRY(ctx, cudaMemcpyAsync(mu, dm.p, B * sizeof(double), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(ctx, cudaMemcpyAsync(argmax_pair, da.p, B * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(ctx, cudaMemcpyAsync(zero_col, dz.p, B * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(ctx, cudaStreamSynchronize(st));
  return TRSTMI_OK;
}

// ------------------------------------------------------------------ batched anneal
static int resolve_cfg(trstmi_ctx* ctx, const trstmi_cfg* c, AnnealArgs& A, std::vector<double>& sched) {
  int rc = check_shape(ctx, c->field, c->d, c->N, "anneal");
  if (rc) return rc;
  A.P = make_prob(c->field, c->d, c->N);
  if (c->n_stages < 0 || c->n_stages > TRSTMI_MAX_STAGES) return fail(ctx, TRSTMI_ERR_INVALID_ARG, "anneal: bad n_stages");
  if (c->n_stages == 0) {
    try {
      sched = trstmi_host::default_delta_schedule(c->N, c->eps_target);
    } catch (const std::exception& e) {
      return fail(ctx, TRSTMI_ERR_INVALID_ARG, e.what());
    }
  } else {
    sched.assign(c->schedule, c->schedule + c->n_stages);
  }
  if ((int)sched.size() > TRSTMI_MAX_STAGES) return fail(ctx, TRSTMI_ERR_INVALID_ARG, "anneal: schedule too long");
  for (size_t k = 0; k + 1 < sched.size(); ++k)  // solver.hpp:172-176
    if (!(sched[k] > sched[k + 1]) || sched[k + 1] <= 0.0)
      return fail(ctx, TRSTMI_ERR_INVALID_ARG, "anneal: schedule must be strictly decreasing and positive");
  if (!sched.empty() && !(sched[0] > 0.0)) return fail(ctx, TRSTMI_ERR_INVALID_ARG, "eval_objective: delta <= 0");
  A.n_stages = (int)sched.size();
  for (int k = 0; k < A.n_stages; ++k) A.schedule[k] = sched[k];
  TrCfg& t = A.tr;
  const double dim = (double)A.P.dim;
  t.delta0 = c->delta0 == 0.0 ? 0.1 * std::sqrt(dim) : c->delta0;  // trust_region.hpp:194-195
  t.max_cg = c->max_cg == 0 ? (int)(2 * A.P.dim) : c->max_cg;
  t.delta_max = c->delta_max;
  t.eta = c->eta;
  t.shrink = c->shrink;
  t.grow = c->grow;
  t.grad_tol = c->grad_tol;
  t.cg_force_c = c->cg_force_c;
  t.max_outer = c->max_outer;
  if (!(t.delta0 > 0.0) || t.delta0 > t.delta_max)  // trust_region.hpp:196-204
    return fail(ctx, TRSTMI_ERR_INVALID_ARG, "trust_region_minimize: need 0 < delta0 <= delta_max");
  if (!(t.eta >= 0.0 && t.eta < 0.25)) return fail(ctx, TRSTMI_ERR_INVALID_ARG, "trust_region_minimize: need 0 <= eta < 1/4");
  if (!(t.shrink > 0.0 && t.shrink < 1.0 && t.grow > 1.0))
    return fail(ctx, TRSTMI_ERR_INVALID_ARG, "trust_region_minimize: need 0 < shrink < 1 < grow");
  A.record_cap = c->record_cap < 0 ? 0 : c->record_cap;
  return TRSTMI_OK;
}

static int launch_anneal(trstmi_ctx* ctx, const trstmi_cfg* c, AnnealArgs& A, cudaStream_t st) {
  const int S = trstmi_lanes(c->field, c->d, c->N);
  const KernelSet* ks = find_kernels(c->field == TRSTMI_COMPLEX, c->d, S, A.P.gs);
  if (!ks) return fail(ctx, TRSTMI_ERR_UNSUPPORTED, "no kernel family for this shape");
  A.P.dual = 0;
  size_t bytes = (size_t)anneal_smem_doubles(A.P, S, c->field == TRSTMI_COMPLEX) * sizeof(double);
  if (bytes > 227 * 1024) return fail(ctx, TRSTMI_ERR_UNSUPPORTED, "trial state exceeds one SM's shared memory");
  // dual layout (both points of a central difference normalised side by side, hvp_cta_gs): taken when its extra
  // shared memory costs no resident trial; results are bit-identical either way
  size_t bytes_d = 0;
  if (A.P.gs && A.P.dim <= kGsDualElems * S && !std::getenv("TRSTMI_NO_DUAL")) {
    Prob Pd = A.P;
    Pd.dual = 1;
    bytes_d = (size_t)anneal_smem_doubles(Pd, S, c->field == TRSTMI_COMPLEX) * sizeof(double);
    if (bytes_d > 227 * 1024) bytes_d = 0;
  }
  CUDA_TRY(ctx, raise_smem_optin(ctx->device, ks->anneal, std::max(bytes, bytes_d)));
  int per_sm = 0;
  CUDA_TRY(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ks->anneal, S, bytes));
  if (per_sm < 1) return fail(ctx, TRSTMI_ERR_UNSUPPORTED, "anneal kernel cannot be resident");
  if (bytes_d) {
    int per_sm_d = 0;
    CUDA_TRY(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_d, ks->anneal, S, bytes_d));
    if (per_sm_d >= per_sm) {
      A.P.dual = 1;
      bytes = bytes_d;
    }
  }
  const long long grid = std::min<long long>(A.n_list, (long long)per_sm * ctx->sm_count);
  A.counter = ctx->counter;
  CUDA_TRY(ctx, cudaMemsetAsync(ctx->counter, 0, sizeof(int), st));
  if (grid <= 0) return TRSTMI_OK;
  void* args[] = {&A};
  CUDA_TRY(ctx, cudaLaunchKernel(ks->anneal, dim3((unsigned)grid), dim3(S), args, bytes, st));
  CUDA_TRY(ctx, cudaGetLastError());
  ++g_launches;
  return TRSTMI_OK;
}

int trstmi_solve_batch_dev(trstmi_ctx* ctx, const trstmi_cfg* cfg, int64_t trials, double* params_dev,
                           uint64_t* rng_state, double* frames_dev, trstmi_trial_out* trial_out_dev,
                           trstmi_stage_out* stage_out_dev, trstmi_outer_out* outer_out_dev, void* stream) {
  if (!ctx || !cfg) return TRSTMI_ERR_INVALID_ARG;
  if (trials < 0 || trials > (1LL << 30)) return fail(ctx, TRSTMI_ERR_INVALID_ARG, "bad trial count");
  AnnealArgs A;
  std::memset(&A, 0, sizeof(A));
  std::vector<double> sched;
  int rc = resolve_cfg(ctx, cfg, A, sched);
  if (rc) return rc;
  cudaSetDevice(ctx->device);
  cudaStream_t st = (cudaStream_t)stream;
  if (trstmi_large::use_large(cfg->field, cfg->d, cfg->N) && ctx->shard_world == 1) {
    // batched engine: every trial's trust-region state machine on the device, one
    // launch per pipeline kernel per tick for all trials in flight
    const trstmi_bde_host::TrCfg tr{A.tr.delta0, A.tr.delta_max, A.tr.eta,      A.tr.shrink, A.tr.grow,
                                    A.tr.grad_tol, A.tr.cg_force_c, A.tr.max_outer, A.tr.max_cg};
    const int cap = A.record_cap;
    if (stage_out_dev)
      CUDA_TRY(ctx, cudaMemsetAsync(stage_out_dev, 0, (size_t)trials * A.n_stages * sizeof(trstmi_stage_out), st));
    if (outer_out_dev && cap)
      CUDA_TRY(ctx, cudaMemsetAsync(outer_out_dev, 0, (size_t)trials * cap * sizeof(trstmi_outer_out), st));
    return trstmi_bde_host::anneal(bde_engine(ctx), st, cfg->field, cfg->d, cfg->N, tr, sched, cap, trials, params_dev,
                                   frames_dev, rng_state, trial_out_dev, stage_out_dev, outer_out_dev, &ctx->err);
  }
  if (trstmi_large::use_large(cfg->field, cfg->d, cfg->N)) {
    const trstmi_large::Shape sh = trstmi_large::make_shape(cfg->field, cfg->d, cfg->N);
    trstmi_large::TrCfg tr{A.tr.delta0, A.tr.delta_max, A.tr.eta, A.tr.shrink, A.tr.grow, A.tr.grad_tol,
                           A.tr.cg_force_c, A.tr.max_outer, A.tr.max_cg};
    const int cap = A.record_cap;
    std::vector<trstmi_trial_out> to(trials);
    std::vector<trstmi_stage_out> so((size_t)trials * A.n_stages);
    std::vector<trstmi_outer_out> oo(outer_out_dev && cap ? (size_t)trials * cap : 0);
    std::memset(so.data(), 0, so.size() * sizeof(trstmi_stage_out));
    // Trial scheduler (the reference's restart thread pool, solver.hpp:239-254):
    // host workers, one CUDA stream + engine each, pull trial ids from an
    // atomic counter; each drives its trial's trust-region loop.
    CUDA_TRY(ctx, cudaStreamSynchronize(st));
    const int workers =
        ctx->shard_world > 1 ? 1 : (int)std::max<int64_t>(1, std::min<int64_t>(trials, large_workers(ctx)));
    std::atomic<int64_t> next{0};
    std::vector<int> rcs(workers, TRSTMI_OK);
    std::vector<std::string> errs(workers);
    auto work = [&](int wi) {
      cudaSetDevice(ctx->device);
      cudaStream_t ws = nullptr;
      trstmi_large::Engine* E = nullptr;
      if (ctx->shard_world > 1) {  // the sharded engine (NCCL communicator / virtual ranks) of the context
        E = large_engine(ctx, st);
      } else {
        cudaStreamCreateWithFlags(&ws, cudaStreamNonBlocking);
        E = trstmi_large::engine_create(ctx->device, ws);
      }
      for (int64_t t = next.fetch_add(1); t < trials && rcs[wi] == TRSTMI_OK; t = next.fetch_add(1)) {
        std::memset(&to[t], 0, sizeof(trstmi_trial_out));
        rcs[wi] = trstmi_large::anneal_trial(E, sh, tr, sched, 0, cap, params_dev + t * sh.dim,
                                             frames_dev ? frames_dev + t * sh.dim : nullptr,
                                             rng_state ? rng_state + 3 * t : nullptr, &to[t],
                                             so.data() + t * A.n_stages, oo.empty() ? nullptr : oo.data() + t * cap,
                                             &errs[wi]);
      }
      if (ws) {
        trstmi_large::engine_destroy(E);
        cudaStreamDestroy(ws);
      }
    };
    if (workers == 1) {
      work(0);
    } else {
      std::vector<std::thread> pool;
      for (int wi = 0; wi < workers; ++wi) pool.emplace_back(work, wi);
      for (auto& th : pool) th.join();
    }
    for (int wi = 0; wi < workers; ++wi)
      if (rcs[wi]) return fail(ctx, rcs[wi], errs[wi]);
    CUDA_TRY(ctx, cudaMemcpyAsync(trial_out_dev, to.data(), trials * sizeof(trstmi_trial_out), cudaMemcpyHostToDevice, st));
    if (stage_out_dev)
      CUDA_TRY(ctx, cudaMemcpyAsync(stage_out_dev, so.data(), so.size() * sizeof(trstmi_stage_out), cudaMemcpyHostToDevice, st));
    if (!oo.empty())
      CUDA_TRY(ctx, cudaMemcpyAsync(outer_out_dev, oo.data(), oo.size() * sizeof(trstmi_outer_out), cudaMemcpyHostToDevice, st));
    CUDA_TRY(ctx, cudaStreamSynchronize(st));
    return TRSTMI_OK;
  }
  A.n_list = (int)trials;
  A.params = params_dev;
  A.frames = frames_dev;
  A.tout = trial_out_dev;
  A.sout = stage_out_dev;
  A.oout = outer_out_dev;
  rc = launch_anneal(ctx, cfg, A, st);
  if (rc) return rc;
  // Stage-boundary rescue loop (solver.hpp:139-156, 183): flagged trials get
  // their collapsed columns redrawn from their own generator on the host and
  // resume at the flagged stage.
  std::vector<trstmi_trial_out> to((size_t)trials);
  const bool cplx = cfg->field == TRSTMI_COMPLEX;
  const int dim = A.P.dim;
  for (int round = 0; trials > 0; ++round) {
    CUDA_TRY(ctx, cudaMemcpyAsync(to.data(), trial_out_dev, trials * sizeof(trstmi_trial_out), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(ctx, cudaStreamSynchronize(st));
    std::vector<int> list, start(trials, 0);
    for (int64_t t = 0; t < trials; ++t) {
      if (to[t].status != TRSTMI_TRIAL_NEED_RESCUE) continue;
      std::vector<double> p(dim);
      CUDA_TRY(ctx, cudaMemcpyAsync(p.data(), params_dev + t * dim, dim * sizeof(double), cudaMemcpyDeviceToHost, st));
      CUDA_TRY(ctx, cudaStreamSynchronize(st));
      int bad;
      if (rng_state) {
        trstmi_host::SplitMix64 rng = trstmi_host::SplitMix64::load(rng_state + 3 * t);
        bad = trstmi_host::rescue_zero_columns(cplx, cfg->d, cfg->N, p.data(), &rng);
        rng.save(rng_state + 3 * t);
      } else {
        bad = trstmi_host::rescue_zero_columns(cplx, cfg->d, cfg->N, p.data(), nullptr);
      }
      if (bad >= 0) {  // ZeroColumnError escapes anneal: the restart fails
        to[t].status = TRSTMI_TRIAL_ZERO_COLUMN;
        to[t].zero_col = bad;
        CUDA_TRY(ctx, cudaMemcpyAsync(trial_out_dev + t, &to[t], sizeof(trstmi_trial_out), cudaMemcpyHostToDevice, st));
        CUDA_TRY(ctx, cudaStreamSynchronize(st));
        continue;
      }
      CUDA_TRY(ctx, cudaMemcpyAsync(params_dev + t * dim, p.data(), dim * sizeof(double), cudaMemcpyHostToDevice, st));
      CUDA_TRY(ctx, cudaStreamSynchronize(st));
      list.push_back((int)t);
      start[t] = to[t].fail_stage;
    }
    if (list.empty()) break;
    if (round > 64 * A.n_stages) return fail(ctx, TRSTMI_ERR_INVALID_ARG, "rescue loop did not converge");
    DBuf dl, ds;
    CUDA_TRY(ctx, cudaMalloc(&dl.p, list.size() * sizeof(int)));
    CUDA_TRY(ctx, cudaMalloc(&ds.p, trials * sizeof(int)));
    CUDA_TRY(ctx, cudaMemcpyAsync(dl.p, list.data(), list.size() * sizeof(int), cudaMemcpyHostToDevice, st));
    CUDA_TRY(ctx, cudaMemcpyAsync(ds.p, start.data(), trials * sizeof(int), cudaMemcpyHostToDevice, st));
    CUDA_TRY(ctx, cudaStreamSynchronize(st));
    A.list = (const int*)dl.p;
    A.start_stage = (const int*)ds.p;
    A.n_list = (int)list.size();
    rc = launch_anneal(ctx, cfg, A, st);
    if (rc) return rc;
    CUDA_TRY(ctx, cudaStreamSynchronize(st));
    A.list = nullptr;
    A.start_stage = nullptr;
  }
  return TRSTMI_OK;
}

int trstmi_solve_batch(trstmi_ctx* ctx, const trstmi_cfg* cfg, int64_t trials, double* params, uint64_t* rng_state,
                       double* frames, trstmi_trial_out* trial_out, trstmi_stage_out* stage_out,
                       trstmi_outer_out* outer_out) {
  if (!ctx || !cfg) return TRSTMI_ERR_INVALID_ARG;
  AnnealArgs A;
  std::memset(&A, 0, sizeof(A));
  std::vector<double> sched;
  int rc = resolve_cfg(ctx, cfg, A, sched);
  if (rc) return rc;
  cudaSetDevice(ctx->device);
  const size_t vb = (size_t)trials * A.P.dim * sizeof(double);
  const size_t cap = (size_t)A.record_cap;
  DBuf dp, df, dt, ds, dout;
  CUDA_TRY(ctx, cudaMalloc(&dp.p, std::max<size_t>(vb, 8)));
  if (frames) CUDA_TRY(ctx, cudaMalloc(&df.p, std::max<size_t>(vb, 8)));
  CUDA_TRY(ctx, cudaMalloc(&dt.p, std::max<size_t>(trials * sizeof(trstmi_trial_out), 8)));
  CUDA_TRY(ctx, cudaMalloc(&ds.p, std::max<size_t>(trials * A.n_stages * sizeof(trstmi_stage_out), 8)));
  if (outer_out && cap) CUDA_TRY(ctx, cudaMalloc(&dout.p, trials * cap * sizeof(trstmi_outer_out)));
  cudaStream_t st = ctx->stream;
  CUDA_TRY(ctx, cudaMemcpyAsync(dp.p, params, vb, cudaMemcpyHostToDevice, st));
  CUDA_TRY(ctx, cudaMemsetAsync(ds.p, 0, trials * A.n_stages * sizeof(trstmi_stage_out), st));
  rc = trstmi_solve_batch_dev(ctx, cfg, trials, (double*)dp.p, rng_state, (double*)df.p, (trstmi_trial_out*)dt.p,
                              (trstmi_stage_out*)ds.p, (trstmi_outer_out*)dout.p, st);
  if (rc) return rc;
  CUDA_TRY(ctx, cudaMemcpyAsync(params, dp.p, vb, cudaMemcpyDeviceToHost, st));
  if (frames) CUDA_TRY(ctx, cudaMemcpyAsync(frames, df.p, vb, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(ctx, cudaMemcpyAsync(trial_out, dt.p, trials * sizeof(trstmi_trial_out), cudaMemcpyDeviceToHost, st));
  if (stage_out)
    CUDA_TRY(ctx, cudaMemcpyAsync(stage_out, ds.p, trials * A.n_stages * sizeof(trstmi_stage_out), cudaMemcpyDeviceToHost, st));
  if (outer_out && cap)
    CUDA_TRY(ctx, cudaMemcpyAsync(outer_out, dout.p, trials * cap * sizeof(trstmi_outer_out), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(ctx, cudaStreamSynchronize(st));
  return TRSTMI_OK;
}

int trstmi_solve(trstmi_ctx* ctx, const trstmi_cfg* cfg, int64_t restarts, uint64_t seed, int64_t first,
                 double* best_frame, double* best_coherence, int64_t* best_restart, trstmi_trial_out* trial_out,
                 trstmi_stage_out* stage_out) {
  if (!ctx || !cfg) return TRSTMI_ERR_INVALID_ARG;
  if (cfg->d < 1 || cfg->N < 1) return fail(ctx, TRSTMI_ERR_INVALID_ARG, "solve: need d, N >= 1");
  if (restarts < 1) return fail(ctx, TRSTMI_ERR_INVALID_ARG, "solve: need restarts >= 1");
  const int64_t dim = (cfg->field == TRSTMI_COMPLEX ? 2 : 1) * (int64_t)cfg->d * cfg->N;
  std::vector<double> params(restarts * dim), frames(restarts * dim);
  std::vector<uint64_t> rng(restarts * 3);
  int rc = trstmi_random_frames(cfg->field, cfg->d, cfg->N, seed, first, restarts, params.data(), rng.data());
  if (rc) return fail(ctx, rc, "random_frame failed");
  std::vector<trstmi_trial_out> to(restarts);
  int n_stages = cfg->n_stages;
  if (n_stages == 0) n_stages = std::max(0, trstmi_default_schedule(cfg->N, cfg->eps_target, nullptr, 0));
  std::vector<trstmi_stage_out> so(restarts * std::max(n_stages, 1));
  rc = trstmi_solve_batch(ctx, cfg, restarts, params.data(), rng.data(), frames.data(), to.data(), so.data(), nullptr);
  if (rc) return rc;
  int64_t best = -1;
  double bc = 0.0;
  for (int64_t i = 0; i < restarts; ++i) {  // solver.hpp:256-263
    if (to[i].status != TRSTMI_TRIAL_OK) continue;
    if (best < 0 || to[i].coherence < bc) {
      best = i;
      bc = to[i].coherence;
    }
  }
  if (trial_out) std::memcpy(trial_out, to.data(), restarts * sizeof(trstmi_trial_out));
  if (stage_out) std::memcpy(stage_out, so.data(), restarts * n_stages * sizeof(trstmi_stage_out));
  if (best < 0) return fail(ctx, TRSTMI_ERR_ALL_FAILED, "solve: all restarts failed");
  *best_restart = best;
  *best_coherence = bc;
  std::memcpy(best_frame, frames.data() + best * dim, dim * sizeof(double));
  return TRSTMI_OK;
}

}  // extern "C"
