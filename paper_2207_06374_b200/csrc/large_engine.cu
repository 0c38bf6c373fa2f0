// Host engine of the large-frame path.  See large_engine.hpp.
#include "large_engine.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <atomic>
#include <map>
#include <mutex>

#include <nccl.h>

#include "host/host_common.hpp"
#include "large_path.cuh"

using namespace trstmi_dev;

namespace trstmi_large {

std::atomic<long long> g_large_launches{0};  // kernels launched by the large-frame engine

namespace {

struct Work {
  Shape sh{};
  bool valid = false;
  double *phiT = nullptr, *alpha = nullptr, *X = nullptr, *GR = nullptr, *GI = nullptr, *zpart = nullptr,
         *scal = nullptr, *PR = nullptr, *PI = nullptr, *CU = nullptr, *part = nullptr, *tpart = nullptr,
         *tile_mu = nullptr;
  long long* tile_arg = nullptr;
  unsigned long long* smax = nullptr;
  int* zero_col = nullptr;
  // trust-region vectors
  double *x = nullptr, *g = nullptr, *zs = nullptr, *r = nullptr, *dv = nullptr, *bd = nullptr, *xt = nullptr,
         *gt = nullptr, *xb = nullptr, *zn = nullptr, *gp = nullptr, *gm = nullptr;
};

}  // namespace

struct Engine {
  int device = 0;
  cudaStream_t st = nullptr;
  Work w;
  // single-frame row-block sharding: world ranks; virtual ranks
  // run every rank's share on this device in sequence (each with its own
  // workspace, exchanges by device copies); otherwise one rank per process
  // with NCCL collectives on st.
  int world = 1, rank = 0;
  bool virtual_ranks = false;
  ncclComm_t nccl = nullptr;
  std::vector<Work> vw;
  double* dots_cta = nullptr;
  double* dots_out = nullptr;
  int* flag = nullptr;
  double* h_scal = nullptr;  // pinned: [0..3] dots / scalars, [4] zero col
};

long long launches() { return g_large_launches.load(); }

Shape make_shape(int field, int d, int N) {
  Shape s;
  s.cplx = field == TRSTMI_COMPLEX;
  s.d = d;
  s.N = N;
  s.L = (s.cplx ? 2 : 1) * d;
  s.dim = s.L * N;
  s.n = (long long)N * (N - 1) / 2;
  s.K = kchunks_for(d, N, kLanes);
  return s;
}

#define LCHK(expr)                                          \
  do {                                                      \
    cudaError_t e_ = (expr);                                \
    if (e_ != cudaSuccess) {                                \
      if (err) *err = std::string(#expr ": ") + cudaGetErrorString(e_); \
      return TRSTMI_ERR_CUDA;                               \
    }                                                       \
  } while (0)

Engine* engine_create(int device, cudaStream_t stream) {
  Engine* E = new Engine();
  E->device = device;
  E->st = stream;
  cudaMalloc(&E->dots_cta, 3 * LS_CTAS * sizeof(double));
  cudaMalloc(&E->dots_out, 8 * sizeof(double));
  cudaMalloc(&E->flag, sizeof(int));
  cudaMallocHost(&E->h_scal, 16 * sizeof(double));
  return E;
}

void engine_set_stream(Engine* E, cudaStream_t stream) { E->st = stream; }

static void free_work(Work& w) {
  double** ptrs[] = {&w.phiT, &w.alpha, &w.X, &w.GR, &w.GI, &w.zpart, &w.scal, &w.PR, &w.PI, &w.CU,
                     &w.part, &w.tpart, &w.tile_mu, &w.x, &w.g, &w.zs, &w.r, &w.dv, &w.bd, &w.xt,
                     &w.gt, &w.xb, &w.zn, &w.gp, &w.gm};
  for (double** p : ptrs) {
    if (*p) cudaFree(*p);
    *p = nullptr;
  }
  if (w.tile_arg) cudaFree(w.tile_arg);
  if (w.smax) cudaFree(w.smax);
  if (w.zero_col) cudaFree(w.zero_col);
  w.tile_arg = nullptr;
  w.smax = nullptr;
  w.zero_col = nullptr;
  w.valid = false;
}

void engine_destroy(Engine* E) {
  if (!E) return;
  free_work(E->w);
  for (Work& w : E->vw) free_work(w);
  if (E->nccl) ncclCommDestroy(E->nccl);
  cudaFree(E->dots_cta);
  cudaFree(E->dots_out);
  cudaFree(E->flag);
  cudaFreeHost(E->h_scal);
  delete E;
}

static int alloc_work(Work& w, const Shape& sh, std::string* err) {
  if (w.valid && w.sh.cplx == sh.cplx && w.sh.d == sh.d && w.sh.N == sh.N) return TRSTMI_OK;
  free_work(w);
  const size_t N2 = (size_t)sh.N * sh.N;
  const int nt = (sh.N + GT - 1) / GT;
  const size_t tiles = (size_t)nt * (nt + 1) / 2;
  LCHK(cudaMalloc(&w.phiT, (size_t)sh.dim * 8));
  LCHK(cudaMalloc(&w.alpha, (size_t)sh.N * 8));
  LCHK(cudaMalloc(&w.X, (size_t)std::max<long long>(sh.n, 1) * 8));
  LCHK(cudaMalloc(&w.GR, (size_t)std::max<long long>(sh.n, 1) * 8));
  LCHK(cudaMalloc(&w.GI, sh.cplx ? (size_t)std::max<long long>(sh.n, 1) * 8 : 8));
  LCHK(cudaMalloc(&w.zpart, (size_t)((sh.N + ZROWS - 1) / ZROWS) * 8));
  LCHK(cudaMemset(w.zpart, 0, (size_t)((sh.N + ZROWS - 1) / ZROWS) * 8));
  LCHK(cudaMalloc(&w.scal, 8 * 8));
  LCHK(cudaMalloc(&w.PR, N2 * 8));
  LCHK(cudaMalloc(&w.PI, sh.cplx ? N2 * 8 : 8));
  LCHK(cudaMalloc(&w.CU, N2 * 8));
  LCHK(cudaMemset(w.PR, 0, N2 * 8));  // diagonals stay zero
  if (sh.cplx) LCHK(cudaMemset(w.PI, 0, N2 * 8));
  LCHK(cudaMemset(w.CU, 0, N2 * 8));
  LCHK(cudaMalloc(&w.part, (size_t)sh.K * sh.dim * 8));
  LCHK(cudaMalloc(&w.tpart, (size_t)sh.K * sh.N * 8));
  LCHK(cudaMalloc(&w.tile_mu, tiles * 8));
  LCHK(cudaMalloc(&w.tile_arg, tiles * 8));
  LCHK(cudaMalloc(&w.smax, 8));
  LCHK(cudaMalloc(&w.zero_col, 4));
  double** vecs[] = {&w.x, &w.g, &w.zs, &w.r, &w.dv, &w.bd, &w.xt, &w.gt, &w.xb, &w.zn, &w.gp, &w.gm};
  for (double** v : vecs) LCHK(cudaMalloc(v, (size_t)sh.dim * 8));
  // the memsets above ran on the legacy stream, which the engine's
  // non-blocking streams do not wait for
  LCHK(cudaDeviceSynchronize());
  w.sh = sh;
  w.valid = true;
  return TRSTMI_OK;
}

static int ensure(Engine* E, const Shape& sh, std::string* err) { return alloc_work(E->w, sh, err); }

static LargeEval make_eval_w(Work& w, const Shape& sh, const double* x, const double* dir, double sc, double delta,
                             int squared, double* grad, double* weights) {
  LargeEval L;
  L.cplx = sh.cplx;
  L.d = sh.d;
  L.N = sh.N;
  L.L = sh.L;
  L.dim = sh.dim;
  L.K = sh.K;
  L.squared = squared;
  L.n = sh.n;
  L.x = x;
  L.dir = dir;
  L.sc = sc;
  L.delta = delta;
  L.phiT = w.phiT;
  L.alpha = w.alpha;
  L.zero_col = w.zero_col;
  L.X = w.X;
  L.GR = w.GR;
  L.GI = w.GI;
  L.smax_bits = w.smax;
  L.zpart = w.zpart;
  L.scal = w.scal;
  L.PR = w.PR;
  L.PI = w.PI;
  L.CU = w.CU;
  L.part = w.part;
  L.tpart = w.tpart;
  L.gout = grad;
  L.wout = weights;
  L.m0 = 0;
  L.m1 = sh.N;
  return L;
}

// Dynamic shared-memory opt-in of `fn` on the current device (the attribute is
// per function and per device; cached per (function, device), failures are
// not cached).
static cudaError_t ensure_smem(const void* fn, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  size_t& have = done[{fn, dev}];
  if (bytes <= have) return cudaSuccess;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) have = bytes;
  return e;
}

// K1 with its staging buffer (norm_smem(L) bytes of dynamic shared memory)
static cudaError_t launch_normalize(const LargeEval& L, cudaStream_t st) {
  const size_t bytes = norm_smem(L.L);
  const cudaError_t e = ensure_smem((const void*)large_normalize, bytes);
  if (e != cudaSuccess) return e;
  const int nc = norm_cols(L.L);
  large_normalize<<<(L.N + nc - 1) / nc, NORM_THREADS, bytes, st>>>(L);
  return cudaGetLastError();
}

// K6 with its two cp.async pipeline buffers (gg_smem(GMT) bytes, > 48 KB opt-in);
// 32-column CTAs for small frames (twice the CTAs of a single-wave grid)
template <bool CPLX, int GMT>
static cudaError_t launch_grad_gemm_t(const LargeEval& L, int cols, int d, int K, cudaStream_t st) {
  const cudaError_t attr = ensure_smem((const void*)large_grad_gemm<CPLX, GMT>, gg_smem(GMT));
  if (attr != cudaSuccess) return attr;
  dim3 gg((cols + GMT - 1) / GMT, (d + GRB - 1) / GRB, K);
  large_grad_gemm<CPLX, GMT><<<gg, 256, gg_smem(GMT), st>>>(L);
  return cudaGetLastError();
}
template <bool CPLX>
static cudaError_t launch_grad_gemm(const LargeEval& L, int cols, int d, int K, cudaStream_t st) {
  if (L.N <= 2048) return launch_grad_gemm_t<CPLX, 32>(L, cols, d, K, st);
  return launch_grad_gemm_t<CPLX, 64>(L, cols, d, K, st);
}

// K5 over the upper-triangular pair tiles
template <bool CPLX>
static void launch_coef(const LargeEval& L, cudaStream_t st) {
  const int nt = (L.N + GT - 1) / GT;
  large_coef<CPLX><<<dim3(nt * (nt + 1) / 2, GT / 16), 256, 0, st>>>(L);
}

// K3a + K3b: the weights over the owned rows with a full grid, then the z chains
static int launch_weights(const LargeEval& L, int nzb, cudaStream_t st) {  // returns the launch count
  const long long p0 = (long long)L.m0 * L.N - (long long)L.m0 * (L.m0 + 1) / 2;
  const long long p1 = (long long)L.m1 * L.N - (long long)L.m1 * (L.m1 + 1) / 2;
  const long long n = p1 - p0;
  if (n < (1LL << 21)) {  // small frames (config 4): one fused kernel, a launch fewer per evaluation
    large_weights<true><<<nzb, ZLANES, 0, st>>>(L);
    return 1;
  }
  large_exp<<<(unsigned)std::min<long long>((n + 511) / 512, 148LL * 16), 256, 0, st>>>(L);
  large_weights<false><<<nzb, ZLANES, 0, st>>>(L);
  return 2;
}

static LargeEval make_eval(Engine* E, const Shape& sh, const double* x, const double* dir, double sc, double delta,
                           int squared, double* grad, double* weights) {
  return make_eval_w(E->w, sh, x, dir, sc, delta, squared, grad, weights);
}

static int eval_sharded(Engine* E, const Shape& sh, const double* x, const double* dir, double sc, double delta,
                        int squared, double* grad, double* F, double* s, long long* zero_col, std::string* err);

int eval(Engine* E, const Shape& sh, const double* x, const double* dir, double sc, double delta, int squared,
         double* grad, double* F, double* s, double* weights, long long* zero_col, std::string* err) {
  if (E->world > 1 && !weights) return eval_sharded(E, sh, x, dir, sc, delta, squared, grad, F, s, zero_col, err);
  int rc = ensure(E, sh, err);
  if (rc) return rc;
  Work& w = E->w;
  cudaStream_t st = E->st;
  LargeEval L = make_eval(E, sh, x, dir, sc, delta, squared, grad, weights);
  LCHK(cudaMemsetAsync(w.zero_col, 0x7f, 4, st));
  LCHK(launch_normalize(L, st));
  const int nt = (sh.N + GT - 1) / GT;
  const int tiles = nt * (nt + 1) / 2;
  if (sh.cplx) large_gram<true, 0><<<tiles, 256, 0, st>>>(L, nullptr, nullptr);
  else large_gram<false, 0><<<tiles, 256, 0, st>>>(L, nullptr, nullptr);
  const int nzb = (sh.N + ZROWS - 1) / ZROWS;
  const int wl = launch_weights(L, nzb, st);
  large_zreduce<<<1, 32, 0, st>>>(L, nzb);
  if (sh.cplx) launch_coef<true>(L, st);
  else launch_coef<false>(L, st);
  if (sh.cplx) LCHK(launch_grad_gemm<true>(L, sh.N, sh.d, sh.K, st));
  else LCHK(launch_grad_gemm<false>(L, sh.N, sh.d, sh.K, st));
  large_finalize<<<(sh.dim + 255) / 256, 256, 0, st>>>(L);
  g_large_launches += 7 + wl;
  LCHK(cudaGetLastError());
  LCHK(cudaMemcpyAsync(E->h_scal, w.scal, 3 * 8, cudaMemcpyDeviceToHost, st));
  LCHK(cudaMemcpyAsync(E->h_scal + 4, w.zero_col, 4, cudaMemcpyDeviceToHost, st));
  LCHK(cudaStreamSynchronize(st));
  int zc;
  std::memcpy(&zc, E->h_scal + 4, 4);
  if (zc >= 0 && zc < sh.N) {
    LCHK(cudaMemsetAsync(grad, 0, (size_t)sh.dim * 8, st));
    if (weights) LCHK(cudaMemsetAsync(weights, 0, (size_t)sh.n * 8, st));
    *zero_col = zc;
    *F = std::numeric_limits<double>::infinity();
    *s = 0.0;
    return TRSTMI_OK;
  }
  *zero_col = -1;
  *s = E->h_scal[0];
  *F = E->h_scal[2];
  return TRSTMI_OK;
}

#define NCHK(expr)                                                        \
  do {                                                                    \
    ncclResult_t r_ = (expr);                                             \
    if (r_ != ncclSuccess) {                                              \
      if (err) *err = std::string(#expr ": ") + ncclGetErrorString(r_);   \
      return TRSTMI_ERR_NCCL;                                             \
    }                                                                     \
  } while (0)

// Rank r of `world` owns the 64-row blocks [r*NB/world, (r+1)*NB/world).
static void shard_rows(const Shape& sh, int world, int r, int* m0, int* m1) {
  const int NB = (sh.N + GT - 1) / GT;
  *m0 = std::min(sh.N, GT * (int)((long long)r * NB / world));
  *m1 = std::min(sh.N, GT * (int)((long long)(r + 1) * NB / world));
}

// One evaluation with the frame's Gram rows sharded over E->world ranks:
// each rank computes the Gram tiles touching its rows/columns, its 16-row z
// blocks and the gradient columns it owns; exchanges are a max of s, the
// z-block partials and the gradient column slices (all pure data movement, so
// the result is bit-identical for every world size).
static int eval_sharded(Engine* E, const Shape& sh, const double* x, const double* dir, double sc, double delta,
                        int squared, double* grad, double* F, double* s, long long* zero_col, std::string* err) {
  int rc = ensure(E, sh, err);
  if (rc) return rc;
  cudaStream_t st = E->st;
  const int G = E->world;
  std::vector<int> ranks;
  if (E->virtual_ranks) {
    if ((int)E->vw.size() != G) E->vw.resize(G);
    for (int r = 0; r < G; ++r) {
      if ((rc = alloc_work(E->vw[r], sh, err))) return rc;
      ranks.push_back(r);
    }
  } else {
    ranks.push_back(E->rank);
  }
  auto work = [&](int r) -> Work& { return E->virtual_ranks ? E->vw[r] : E->w; };
  std::vector<LargeEval> Ls(G);
  for (int r : ranks) {
    LargeEval L = make_eval_w(work(r), sh, x, dir, sc, delta, squared, grad, nullptr);
    shard_rows(sh, G, r, &L.m0, &L.m1);
    Ls[r] = L;
  }
  const int nt = (sh.N + GT - 1) / GT;
  const int tiles = nt * (nt + 1) / 2;
  const int nzb = (sh.N + ZROWS - 1) / ZROWS;
  // phase A: normalise, Gram of the shard's tiles, local max
  for (int r : ranks) {
    LCHK(cudaMemsetAsync(work(r).zero_col, 0x7f, 4, st));
    LCHK(launch_normalize(Ls[r], st));
    if (sh.cplx) large_gram<true, 0><<<tiles, 256, 0, st>>>(Ls[r], nullptr, nullptr);
    else large_gram<false, 0><<<tiles, 256, 0, st>>>(Ls[r], nullptr, nullptr);
  }
  LCHK(cudaGetLastError());
  // exchange: s = max over ranks (x >= 0, so the bit patterns order like the values)
  if (E->virtual_ranks) {
    unsigned long long mx = 0, v = 0;
    for (int r : ranks) {
      LCHK(cudaMemcpyAsync(&v, work(r).smax, 8, cudaMemcpyDeviceToHost, st));
      LCHK(cudaStreamSynchronize(st));
      mx = std::max(mx, v);
    }
    for (int r : ranks) LCHK(cudaMemcpyAsync(work(r).smax, &mx, 8, cudaMemcpyHostToDevice, st));
    LCHK(cudaStreamSynchronize(st));
  } else {
    NCHK(ncclAllReduce(E->w.smax, E->w.smax, 1, ncclUint64, ncclMax, E->nccl, st));
  }
  // phase B: weights of the shard's pairs, z partials of its 16-row blocks
  int wl = 0;
  for (int r : ranks) wl += launch_weights(Ls[r], nzb, st);
  LCHK(cudaGetLastError());
  // exchange: every rank's z-block partials to every rank
  auto zslice = [&](int r, int* b0, int* cnt) {
    int m0, m1;
    shard_rows(sh, G, r, &m0, &m1);
    *b0 = m0 / ZROWS;
    *cnt = (m1 + ZROWS - 1) / ZROWS - *b0;
  };
  if (E->virtual_ranks) {
    for (int r : ranks) {
      int b0, cnt;
      zslice(r, &b0, &cnt);
      for (int q : ranks)
        if (q != r && cnt > 0)
          LCHK(cudaMemcpyAsync(work(q).zpart + b0, work(r).zpart + b0, (size_t)cnt * 8, cudaMemcpyDeviceToDevice, st));
    }
  } else {
    NCHK(ncclGroupStart());
    for (int r = 0; r < G; ++r) {
      int b0, cnt;
      zslice(r, &b0, &cnt);
      if (cnt > 0) NCHK(ncclBroadcast(E->w.zpart + b0, E->w.zpart + b0, (size_t)cnt, ncclDouble, r, E->nccl, st));
    }
    NCHK(ncclGroupEnd());
  }
  // phase C: z, coefficients, gradient columns of the shard
  for (int r : ranks) {
    const LargeEval& L = Ls[r];
    large_zreduce<<<1, 32, 0, st>>>(L, nzb);
    if (sh.cplx) launch_coef<true>(L, st);
    else launch_coef<false>(L, st);
    const int cols = L.m1 - L.m0;
    if (cols > 0) {
      if (sh.cplx) LCHK(launch_grad_gemm<true>(L, cols, sh.d, sh.K, st));
      else LCHK(launch_grad_gemm<false>(L, cols, sh.d, sh.K, st));
      large_finalize<<<(int)(((long long)cols * sh.L + 255) / 256), 256, 0, st>>>(L);
    }
  }
  LCHK(cudaGetLastError());
  g_large_launches += (long long)ranks.size() * 7 + wl;
  if (!E->virtual_ranks) {  // gradient column slices to every rank
    NCHK(ncclGroupStart());
    for (int r = 0; r < G; ++r) {
      int m0, m1;
      shard_rows(sh, G, r, &m0, &m1);
      const size_t cnt = (size_t)(m1 - m0) * sh.L;
      if (cnt) NCHK(ncclBroadcast(grad + (size_t)m0 * sh.L, grad + (size_t)m0 * sh.L, cnt, ncclDouble, r, E->nccl, st));
    }
    NCHK(ncclGroupEnd());
  }
  Work& w0 = work(ranks[0]);
  LCHK(cudaMemcpyAsync(E->h_scal, w0.scal, 3 * 8, cudaMemcpyDeviceToHost, st));
  LCHK(cudaMemcpyAsync(E->h_scal + 4, w0.zero_col, 4, cudaMemcpyDeviceToHost, st));
  LCHK(cudaStreamSynchronize(st));
  int zc;
  std::memcpy(&zc, E->h_scal + 4, 4);
  if (zc >= 0 && zc < sh.N) {
    LCHK(cudaMemsetAsync(grad, 0, (size_t)sh.dim * 8, st));
    *zero_col = zc;
    *F = std::numeric_limits<double>::infinity();
    *s = 0.0;
    return TRSTMI_OK;
  }
  *zero_col = -1;
  *s = E->h_scal[0];
  *F = E->h_scal[2];
  return TRSTMI_OK;
}

int engine_set_shard(Engine* E, int world, int rank, const void* nccl_id, std::string* err) {
  if (E->nccl) {
    ncclCommDestroy(E->nccl);
    E->nccl = nullptr;
  }
  E->world = world < 1 ? 1 : world;
  E->rank = rank;
  E->virtual_ranks = nccl_id == nullptr && world > 1;
  if (!E->virtual_ranks && world > 1) {
    ncclUniqueId id;
    std::memcpy(&id, nccl_id, sizeof(id));
    cudaSetDevice(E->device);
    NCHK(ncclCommInitRank(&E->nccl, world, id, rank));
  }
  return TRSTMI_OK;
}

int nccl_unique_id(void* out, std::string* err) {
  ncclUniqueId id;
  NCHK(ncclGetUniqueId(&id));
  std::memcpy(out, &id, sizeof(id));
  return TRSTMI_OK;
}

// CAS dots (width 32768) of up to three pairs; blocking.
static int dots(Engine* E, long long n, int nd, const double* a0, const double* b0, const double* a1, const double* b1,
                const double* a2, const double* b2, double* out, std::string* err) {
  large_dots<<<LS_CTAS, LS_THREADS, 0, E->st>>>(a0, b0, a1 ? a1 : a0, b1 ? b1 : b0, a2 ? a2 : a0, b2 ? b2 : b0, nd,
                                                n, E->dots_cta);
  large_dots_reduce<<<1, LS_CTAS, 0, E->st>>>(E->dots_cta, nd, E->dots_out);
  g_large_launches += 2;
  LCHK(cudaGetLastError());
  LCHK(cudaMemcpyAsync(E->h_scal, E->dots_out, nd * 8, cudaMemcpyDeviceToHost, E->st));
  LCHK(cudaStreamSynchronize(E->st));
  for (int q = 0; q < nd; ++q) out[q] = E->h_scal[q];
  return TRSTMI_OK;
}

static int grid_for(long long n) { return (int)std::max<long long>(1, std::min<long long>((n + 255) / 256, 148LL * 8)); }

static int all_finite(Engine* E, const double* v, long long n, bool* ok, std::string* err) {
  LCHK(cudaMemsetAsync(E->flag, 0, 4, E->st));
  large_nonfinite<<<grid_for(n), 256, 0, E->st>>>(v, n, E->flag);
  int f = 0;
  LCHK(cudaMemcpyAsync(E->h_scal + 6, E->flag, 4, cudaMemcpyDeviceToHost, E->st));
  LCHK(cudaStreamSynchronize(E->st));
  std::memcpy(&f, E->h_scal + 6, 4);
  *ok = f == 0;
  return TRSTMI_OK;
}

int hvp(Engine* E, const Shape& sh, const double* x, const double* dir, double delta, double* hv, int* path,
        long long* zero_col, std::string* err) {
  int rc = ensure(E, sh, err);
  if (rc) return rc;
  Work& w = E->w;
  double nn[2];
  rc = dots(E, sh.dim, 2, dir, dir, x, x, nullptr, nullptr, nn, err);
  if (rc) return rc;
  const double dn = std::sqrt(nn[0]);
  *zero_col = -1;
  if (dn == 0.0) {
    LCHK(cudaMemsetAsync(hv, 0, (size_t)sh.dim * 8, E->st));
    *path = TRSTMI_HVP_ZERO_DIR;
    return TRSTMI_OK;
  }
  const double h = trstmi_dev::kFdBaseStep * (1.0 + std::sqrt(nn[1])) / std::max(dn, 1e-300);
  double F, s;
  long long zp, zm;
  if ((rc = eval(E, sh, x, dir, h, delta, 1, w.gp, &F, &s, nullptr, &zp, err))) return rc;
  if (zp < 0) {
    if ((rc = eval(E, sh, x, dir, -h, delta, 1, w.gm, &F, &s, nullptr, &zm, err))) return rc;
    if (zm < 0) {
      large_fd<<<grid_for(sh.dim), 256, 0, E->st>>>(hv, w.gp, w.gm, 2.0 * h, sh.dim);
      *path = TRSTMI_HVP_CENTRAL;
    } else {
      if ((rc = eval(E, sh, x, nullptr, 0.0, delta, 1, w.gt, &F, &s, nullptr, &zm, err))) return rc;
      large_fd<<<grid_for(sh.dim), 256, 0, E->st>>>(hv, w.gp, w.gt, h, sh.dim);
      *path = TRSTMI_HVP_FORWARD;
    }
  } else {
    if ((rc = eval(E, sh, x, nullptr, 0.0, delta, 1, w.gt, &F, &s, nullptr, &zm, err))) return rc;
    if ((rc = eval(E, sh, x, dir, -h, delta, 1, w.gm, &F, &s, nullptr, &zm, err))) return rc;
    if (zm < 0) {
      large_fd<<<grid_for(sh.dim), 256, 0, E->st>>>(hv, w.gt, w.gm, h, sh.dim);
      *path = TRSTMI_HVP_BACKWARD;
    } else {
      LCHK(cudaMemsetAsync(hv, 0, (size_t)sh.dim * 8, E->st));
      *path = TRSTMI_HVP_FAILED;
      *zero_col = zm;
    }
  }
  LCHK(cudaStreamSynchronize(E->st));
  return TRSTMI_OK;
}

int coherence(Engine* E, const Shape& sh, const double* frame, int normalize, double* mu, long long* argmax,
              long long* zero_col, std::string* err) {
  int rc = ensure(E, sh, err);
  if (rc) return rc;
  Work& w = E->w;
  cudaStream_t st = E->st;
  LargeEval L = make_eval(E, sh, frame, nullptr, 0.0, 1.0, 1, nullptr, nullptr);
  LCHK(cudaMemsetAsync(w.zero_col, 0x7f, 4, st));
  if (normalize) LCHK(launch_normalize(L, st));
  std::vector<double> hframe;
  if (!normalize) {
    hframe.resize(sh.dim);
    LCHK(cudaMemcpyAsync(hframe.data(), frame, (size_t)sh.dim * 8, cudaMemcpyDeviceToHost, st));
    LCHK(cudaStreamSynchronize(st));
    std::vector<double> t((size_t)sh.dim);
    for (int j = 0; j < sh.N; ++j)
      for (int q = 0; q < sh.L; ++q) t[(size_t)q * sh.N + j] = hframe[(size_t)j * sh.L + q];
    LCHK(cudaMemcpyAsync(w.phiT, t.data(), (size_t)sh.dim * 8, cudaMemcpyHostToDevice, st));
  }
  const int nt = (sh.N + GT - 1) / GT;
  const int tiles = nt * (nt + 1) / 2;
  if (sh.cplx) large_gram<true, 1><<<tiles, 256, 0, st>>>(L, w.tile_mu, w.tile_arg);
  else large_gram<false, 1><<<tiles, 256, 0, st>>>(L, w.tile_mu, w.tile_arg);
  LCHK(cudaGetLastError());
  std::vector<double> tm(tiles);
  std::vector<long long> ta(tiles);
  int zc = INT_MAX;
  LCHK(cudaMemcpyAsync(tm.data(), w.tile_mu, tiles * 8, cudaMemcpyDeviceToHost, st));
  LCHK(cudaMemcpyAsync(ta.data(), w.tile_arg, tiles * 8, cudaMemcpyDeviceToHost, st));
  LCHK(cudaMemcpyAsync(&zc, w.zero_col, 4, cudaMemcpyDeviceToHost, st));
  LCHK(cudaStreamSynchronize(st));
  if (normalize && zc >= 0 && zc < sh.N) {
    *zero_col = zc;
    *mu = 0.0;
    *argmax = -1;
    return TRSTMI_OK;
  }
  double best = 0.0;
  long long arg = LLONG_MAX;
  for (int t = 0; t < tiles; ++t)
    if (tm[t] > best || (tm[t] == best && tm[t] > 0.0 && ta[t] < arg)) {
      best = tm[t];
      arg = ta[t];
    }
  *zero_col = -1;
  *mu = best;
  *argmax = arg == LLONG_MAX ? -1 : arg;
  return TRSTMI_OK;
}

// --------------------------------------------------------------- anneal driver
// trust_region_minimize / steihaug_cg / make_hvp_factory / anneal, line for
// line as oracle/cas_oracle.hpp (which restates trust_region.hpp:56-295 and
// solver.hpp:118-204), with the vectors on the device.
int anneal_trial(Engine* E, const Shape& sh, const TrCfg& tr, const std::vector<double>& schedule, int start_stage,
                 int record_cap, double* params, double* frame, uint64_t* rng_state, trstmi_trial_out* TO,
                 trstmi_stage_out* SO, trstmi_outer_out* OO, std::string* err) {
  int rc = ensure(E, sh, err);
  if (rc) return rc;
  Work& w = E->w;
  cudaStream_t st = E->st;
  const long long dim = sh.dim;
  const int G = grid_for(dim);
  auto axpy = [&](double* y, const double* a, double s, const double* b) {
    large_axpy<<<G, 256, 0, st>>>(y, a, s, b, dim);
  };
  auto copy = [&](double* dst, const double* src) {
    return cudaMemcpyAsync(dst, src, (size_t)dim * 8, cudaMemcpyDeviceToDevice, st);
  };
  auto dot1 = [&](const double* a, const double* b, double* out) { return dots(E, dim, 1, a, b, nullptr, nullptr, nullptr, nullptr, out, err); };

  long long outer = 0, evals = 0, hvps = 0, nrec = 0;
  if (start_stage > 0) {
    outer = TO->outer_iterations;
    evals = TO->evals;
    hvps = TO->hvps;
    nrec = TO->records;
  }
  int status = TRSTMI_TRIAL_OK, zero_col = -1, fail_stage = -1, stages_done = start_stage;
  double mu = 0.0;
  long long argmax = -1;
  double* x = w.x;
  double* g = w.g;
  double* xt = w.xt;
  double* gt = w.gt;
  double* xb = w.xb;
  LCHK(copy(x, params));
  std::vector<double> host((size_t)dim);
  trstmi_host::SplitMix64 rng;
  if (rng_state) rng = trstmi_host::SplitMix64::load(rng_state);
  const int n_stages = (int)schedule.size();
  for (int k = start_stage; k < n_stages; ++k) {
    // rescue_zero_columns (solver.hpp:139-156)
    LCHK(cudaMemcpyAsync(host.data(), x, (size_t)dim * 8, cudaMemcpyDeviceToHost, st));
    LCHK(cudaStreamSynchronize(st));
    bool any_zero = false;
    for (int j = 0; j < sh.N && !any_zero; ++j)
      any_zero = !(trstmi_host::column_norm(&host[(size_t)j * sh.L], sh.L) >= trstmi_host::kZeroColumnTol);
    if (any_zero) {
      const int bad = trstmi_host::rescue_zero_columns(sh.cplx, sh.d, sh.N, host.data(), rng_state ? &rng : nullptr);
      if (bad >= 0) {
        status = TRSTMI_TRIAL_ZERO_COLUMN;
        zero_col = bad;
        fail_stage = k;
        break;
      }
      LCHK(cudaMemcpyAsync(x, host.data(), (size_t)dim * 8, cudaMemcpyHostToDevice, st));
    }
    const double delta = schedule[k];
    const int max_outer = tr.max_outer + 50 * k;
    double Fcur, s;
    long long zc;
    ++evals;
    if ((rc = eval(E, sh, x, nullptr, 0.0, delta, 1, g, &Fcur, &s, nullptr, &zc, err))) return rc;
    bool fin;
    if ((rc = all_finite(E, g, dim, &fin, err))) return rc;
    if (!std::isfinite(Fcur) || !fin) {
      status = TRSTMI_TRIAL_NONFINITE_X0;
      fail_stage = k;
      break;
    }
    double bestv = Fcur;
    LCHK(copy(xb, x));
    double radius = tr.delta0;
    int mstatus = TRSTMI_ST_ITERATION_LIMIT;
    int hist = 0;
    bool failed = false;
    for (int iter = 0; iter < max_outer; ++iter) {
      double gv[2];
      if ((rc = dots(E, dim, 2, g, g, x, x, nullptr, nullptr, gv, err))) return rc;
      const double grad_norm = std::sqrt(gv[0]);
      const double xnorm = std::sqrt(gv[1]);
      if (grad_norm <= tr.grad_tol) {
        mstatus = TRSTMI_ST_GRADIENT_TOLERANCE;
        break;
      }
      const double eps_k = std::min(tr.cg_force_c, std::sqrt(grad_norm)) * grad_norm;
      int cg_iters = 0, cg_exit = TRSTMI_CG_SMALL_RESIDUAL;
      double step_norm = 0.0, model_value = 0.0;
      LCHK(cudaMemsetAsync(w.zs, 0, (size_t)dim * 8, st));
      if (grad_norm < eps_k || grad_norm == 0.0) {
        cg_exit = TRSTMI_CG_ZERO_GRADIENT;
      } else {
        LCHK(copy(w.r, g));
        large_neg<<<G, 256, 0, st>>>(w.dv, g, dim);
        double rr = gv[0], model = 0.0;
        bool done = false;
        for (int j = 0; j < tr.max_cg; ++j) {
          ++hvps;
          double dn2;
          if ((rc = dot1(w.dv, w.dv, &dn2))) return rc;
          const double dn = std::sqrt(dn2);
          if (dn == 0.0) {
            LCHK(cudaMemsetAsync(w.bd, 0, (size_t)dim * 8, st));
          } else {
            const double h = trstmi_dev::kFdBaseStep * (1.0 + xnorm) / std::max(dn, 1e-300);
            double Fx, sx;
            long long zp, zm;
            evals += 2;
            if ((rc = eval(E, sh, x, w.dv, h, delta, 1, w.gp, &Fx, &sx, nullptr, &zp, err))) return rc;
            if (zp < 0) {
              if ((rc = eval(E, sh, x, w.dv, -h, delta, 1, w.gm, &Fx, &sx, nullptr, &zm, err))) return rc;
              if (zm < 0) {
                large_fd<<<G, 256, 0, st>>>(w.bd, w.gp, w.gm, 2.0 * h, dim);
              } else {  // forward fallback: g0 and g(x + h d) again (solver.hpp:129-130), reused values
                evals += 2;
                large_fd<<<G, 256, 0, st>>>(w.bd, w.gp, g, h, dim);
              }
            } else {
              evals += 2;
              if ((rc = eval(E, sh, x, w.dv, -h, delta, 1, w.gm, &Fx, &sx, nullptr, &zm, err))) return rc;
              if (zm >= 0) {
                status = TRSTMI_TRIAL_ZERO_COLUMN;
                zero_col = (int)zm;
                fail_stage = k;
                failed = true;
                break;
              }
              large_fd<<<G, 256, 0, st>>>(w.bd, g, w.gm, h, dim);
            }
          }
          double dd[2];
          if ((rc = dots(E, dim, 2, w.dv, w.bd, w.r, w.dv, nullptr, nullptr, dd, err))) return rc;
          const double dbd = dd[0], rd = dd[1];
          if (dbd <= 0.0) {
            double br[3];
            if ((rc = dots(E, dim, 3, w.dv, w.dv, w.zs, w.dv, w.zs, w.zs, br, err))) return rc;
            const double a = br[0], b = 2.0 * br[1], c = br[2] - radius * radius;
            double tau_lo = 0.0, tau_hi = 0.0;
            if (!(a <= 0.0)) {
              const double disc = std::sqrt(std::max(b * b - 4.0 * a * c, 0.0));
              const double q = -0.5 * (b + std::copysign(disc, b));
              double r1 = q != 0.0 ? c / q : 0.0;
              double r2 = a != 0.0 ? q / a : 0.0;
              if (r1 > r2) std::swap(r1, r2);
              tau_lo = r1;
              tau_hi = r2;
            }
            const double m_lo = model + tau_lo * rd + 0.5 * tau_lo * tau_lo * dbd;
            const double m_hi = model + tau_hi * rd + 0.5 * tau_hi * tau_hi * dbd;
            const double tau = m_lo < m_hi ? tau_lo : tau_hi;
            axpy(w.zs, w.zs, tau, w.dv);
            double zz;
            if ((rc = dot1(w.zs, w.zs, &zz))) return rc;
            step_norm = std::sqrt(zz);
            cg_iters = j;
            cg_exit = TRSTMI_CG_NEGATIVE_CURVATURE;
            model_value = std::min(m_lo, m_hi);
            done = true;
            break;
          }
          const double alpha = rr / dbd;
          axpy(w.zn, w.zs, alpha, w.dv);
          double zn2;
          if ((rc = dot1(w.zn, w.zn, &zn2))) return rc;
          if (std::sqrt(zn2) >= radius) {
            double br[3];
            if ((rc = dots(E, dim, 3, w.dv, w.dv, w.zs, w.dv, w.zs, w.zs, br, err))) return rc;
            const double a = br[0], b = 2.0 * br[1], c = br[2] - radius * radius;
            double tau = 0.0;
            if (!(a <= 0.0)) {
              const double disc = std::sqrt(std::max(b * b - 4.0 * a * c, 0.0));
              const double q = -0.5 * (b + std::copysign(disc, b));
              double r1 = q != 0.0 ? c / q : 0.0;
              double r2 = a != 0.0 ? q / a : 0.0;
              tau = (r1 > r2) ? r1 : r2;
            }
            axpy(w.zs, w.zs, tau, w.dv);
            double zz;
            if ((rc = dot1(w.zs, w.zs, &zz))) return rc;
            step_norm = std::sqrt(zz);
            cg_iters = j;
            cg_exit = TRSTMI_CG_BOUNDARY_HIT;
            model_value = model + tau * rd + 0.5 * tau * tau * dbd;
            done = true;
            break;
          }
          model += alpha * rd + 0.5 * alpha * alpha * dbd;
          std::swap(w.zs, w.zn);  // z = z_next
          axpy(w.r, w.r, alpha, w.bd);
          double rr_next;
          if ((rc = dot1(w.r, w.r, &rr_next))) return rc;
          cg_iters = j + 1;
          if (std::sqrt(rr_next) < eps_k) {
            cg_exit = TRSTMI_CG_SMALL_RESIDUAL;
            double zz;
            if ((rc = dot1(w.zs, w.zs, &zz))) return rc;
            step_norm = std::sqrt(zz);
            model_value = model;
            done = true;
            break;
          }
          const double beta = rr_next / rr;
          rr = rr_next;
          large_cg_dir<<<G, 256, 0, st>>>(w.dv, w.r, beta, dim);
        }
        if (failed) break;
        if (!done) {
          cg_exit = TRSTMI_CG_SMALL_RESIDUAL;
          double zz;
          if ((rc = dot1(w.zs, w.zs, &zz))) return rc;
          step_norm = std::sqrt(zz);
          model_value = model;
        }
      }
      trstmi_outer_out rec;
      std::memset(&rec, 0, sizeof(rec));
      rec.stage = k;
      rec.iteration = iter;
      rec.cg_exit = cg_exit;
      rec.cg_iterations = cg_iters;
      rec.value = Fcur;
      rec.grad_norm = grad_norm;
      rec.radius = radius;
      rec.step_norm = step_norm;
      const double predicted = -model_value;
      bool underflow = false;
      if (cg_exit == TRSTMI_CG_ZERO_GRADIENT || predicted <= 0.0) {
        radius *= tr.shrink;
        underflow = radius < 1e-16;
      } else {
        axpy(xt, x, 1.0, w.zs);
        ++evals;
        double Ft, st2;
        long long zt;
        if ((rc = eval(E, sh, xt, nullptr, 0.0, delta, 1, gt, &Ft, &st2, nullptr, &zt, err))) return rc;
        bool gfin;
        if ((rc = all_finite(E, gt, dim, &gfin, err))) return rc;
        const bool finite = std::isfinite(Ft) && gfin;
        const double rho = finite ? (Fcur - Ft) / predicted : -std::numeric_limits<double>::infinity();
        rec.rho = rho;
        if (finite && Ft < bestv) {
          LCHK(copy(xb, xt));
          bestv = Ft;
        }
        if (rho > tr.eta) {
          std::swap(x, xt);
          std::swap(g, gt);
          Fcur = Ft;
          rec.accepted = 1;
        }
        if (rho < 0.25) {
          radius *= tr.shrink;
        } else if (rho > 0.75 && step_norm >= (1.0 - 1e-10) * radius) {
          radius = std::min(tr.grow * radius, tr.delta_max);
        }
        underflow = radius < 1e-16;
      }
      if (OO && nrec < record_cap) OO[nrec] = rec;
      if (OO && nrec < record_cap) ++nrec;
      ++hist;
      if (underflow) {
        mstatus = TRSTMI_ST_RADIUS_UNDERFLOW;
        break;
      }
    }
    if (failed) break;
    outer += hist;
    if (Fcur < bestv) {
      LCHK(copy(xb, x));
      bestv = Fcur;
    }
    std::swap(x, xb);
    double smu;
    long long sarg, szc;
    if ((rc = coherence(E, sh, x, 1, &smu, &sarg, &szc, err))) return rc;
    if (szc >= 0) {
      status = TRSTMI_TRIAL_ZERO_COLUMN;
      zero_col = (int)szc;
      fail_stage = k;
      break;
    }
    trstmi_stage_out so;
    so.delta = delta;
    so.objective = bestv;
    so.coherence = smu;
    so.argmax_pair = sarg;
    so.outer_iterations = hist;
    so.status = mstatus;
    SO[k] = so;
    mu = smu;
    argmax = sarg;
    stages_done = k + 1;
  }
  // restore the canonical buffer assignment (pointer swaps above)
  LCHK(copy(params, x));
  if (status == TRSTMI_TRIAL_OK && frame) {
    LCHK(cudaMemcpyAsync(host.data(), x, (size_t)dim * 8, cudaMemcpyDeviceToHost, st));
    LCHK(cudaStreamSynchronize(st));
    for (int j = 0; j < sh.N; ++j) {
      double* c = &host[(size_t)j * sh.L];
      const double a = trstmi_host::column_norm(c, sh.L);
      for (int q = 0; q < sh.L; ++q) c[q] = c[q] / a;
    }
    LCHK(cudaMemcpyAsync(frame, host.data(), (size_t)dim * 8, cudaMemcpyHostToDevice, st));
  }
  LCHK(cudaStreamSynchronize(st));
  if (rng_state) rng.save(rng_state);
  TO->coherence = mu;
  TO->argmax_pair = argmax;
  TO->status = status;
  TO->stages_done = stages_done;
  TO->zero_col = zero_col;
  TO->fail_stage = fail_stage;
  TO->outer_iterations = outer;
  TO->evals = evals;
  TO->hvps = hvps;
  TO->records = nrec;
  return TRSTMI_OK;
}

}  // namespace trstmi_large
