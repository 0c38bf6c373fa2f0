// Host side of the batched device engine (csrc/bde_engine.hpp).
#include "bde_engine.hpp"

#include <algorithm>
#include <atomic>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>

#include "bde_tr.cuh"
#include "host/host_common.hpp"

namespace trstmi_bde_host {

using namespace trstmi_bde;

static std::atomic<long long> g_launches{0};
long long launches() { return g_launches.load(); }

#define BCHK(expr)                                                                      \
  do {                                                                                  \
    cudaError_t e_ = (expr);                                                            \
    if (e_ != cudaSuccess) {                                                            \
      if (err) *err = std::string(#expr ": ") + cudaGetErrorString(e_);                 \
      return TRSTMI_ERR_CUDA;                                                           \
    }                                                                                   \
  } while (0)

namespace {

int kchunks(int N) {  // CAS gradient chunks of the large path: K = clamp(32768 / N, 1, 8)
  const int K = 32768 / N;
  return K < 1 ? 1 : (K > 8 ? 8 : K);
}

Shape make_shape(int field, int d, int N) {
  Shape s;
  s.cplx = field == TRSTMI_COMPLEX;
  s.d = d;
  s.N = N;
  s.L = (s.cplx ? 2 : 1) * d;
  s.dim = s.L * N;
  s.K = kchunks(N);
  s.n = (long long)N * (N - 1) / 2;
  s.nt = (N + BT - 1) / BT;
  s.tiles = s.nt * (s.nt + 1) / 2;
  s.nzb = (N + BZROWS - 1) / BZROWS;
  return s;
}

template <class T>
void dfree(T*& p) {
  if (p) cudaFree(p);
  p = nullptr;
}

cudaError_t ensure_smem(const void* fn, size_t bytes) {
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

// point layout per point: HVP preparation (CAS norms of dir and x) and combine
__global__ void __launch_bounds__(TR_T, 1) bde_hvp_prep(const double* pts, const double* dirs, long long dim,
                                                        double* nn) {
  __shared__ double tot[2 * CAS_G];
  const double* x = pts + blockIdx.x * dim;
  const double* v = dirs + blockIdx.x * dim;
  const double* a[2] = {v, x};
  double o[2];
  cas_dots<2>(a, a, dim, o, tot);
  if (threadIdx.x == 0) {
    nn[2 * blockIdx.x] = o[0];
    nn[2 * blockIdx.x + 1] = o[1];
  }
}

// mode: 0 central (gp - gm)/(2h), 1 forward (gp - g0)/h, 2 backward (g0 - gm)/h, 3 zero
__global__ void bde_hvp_combine(double* hv, const double* gp, const double* gm, const double* g0, const int* mode,
                                const double* hh, long long dim) {
  const int b = blockIdx.y;
  const long long off = (long long)b * dim;
  const int md = mode[b];
  const double h = hh[b];
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < dim; i += (long long)gridDim.x * blockDim.x) {
    double v = 0.0;
    if (md == 0) v = __ddiv_rn(__dsub_rn(gp[off + i], gm[off + i]), 2.0 * h);
    else if (md == 1) v = __ddiv_rn(__dsub_rn(gp[off + i], g0[off + i]), h);
    else if (md == 2) v = __ddiv_rn(__dsub_rn(g0[off + i], gm[off + i]), h);
    hv[off + i] = v;
  }
}

}  // namespace

struct Engine {
  int device = 0;
  Shape sh{};
  bool valid = false;
  int slots = 0;   // workspace slots
  int lanes = 0;   // trust-region lanes
  Ws ws{};
  Req* reqs = nullptr;
  ReqOut* outs = nullptr;
  int* act_obj = nullptr;
  int* act_coh = nullptr;
  int* counters = nullptr;
  int* paused = nullptr;
  int* next = nullptr;
  Lane* lanevec = nullptr;
  double* vecs = nullptr;
  int* h_counters = nullptr;  // pinned
  // scratch for the single-point entry points
  double* scratch = nullptr;
  size_t scratch_bytes = 0;
};

Engine* create(int device) {
  Engine* E = new Engine();
  E->device = device;
  cudaSetDevice(device);
  cudaMallocHost(&E->h_counters, 8 * sizeof(int));
  return E;
}

static void free_all(Engine* E) {
  dfree(E->ws.phi);
  dfree(E->ws.alpha);
  dfree(E->ws.G);
  dfree(E->ws.W);
  dfree(E->ws.zpart);
  dfree(E->ws.part);
  dfree(E->ws.tpart);
  dfree(E->ws.tmu);
  dfree(E->ws.targ);
  dfree(E->reqs);
  dfree(E->outs);
  dfree(E->act_obj);
  dfree(E->act_coh);
  dfree(E->counters);
  dfree(E->paused);
  dfree(E->next);
  dfree(E->lanevec);
  dfree(E->vecs);
  dfree(E->scratch);
  E->scratch_bytes = 0;
  E->valid = false;
  E->slots = E->lanes = 0;
}

void destroy(Engine* E) {
  if (!E) return;
  cudaSetDevice(E->device);
  free_all(E);
  if (E->h_counters) cudaFreeHost(E->h_counters);
  delete E;
}

static size_t slot_doubles(const Shape& s) {
  return (size_t)s.dim + s.N + (size_t)s.n * (s.cplx ? 2 : 1) + (size_t)s.n + s.nzb + (size_t)s.K * s.dim +
         (size_t)s.K * s.N + 2 * (size_t)s.tiles;
}

// Workspaces for `slots` evaluation slots and `lanes` trust-region lanes.
static int ensure(Engine* E, const Shape& sh, int slots, int lanes, std::string* err) {
  const bool same = E->valid && E->sh.cplx == sh.cplx && E->sh.d == sh.d && E->sh.N == sh.N;
  if (same && E->slots >= slots && E->lanes >= lanes) return TRSTMI_OK;
  slots = std::max(slots, same ? E->slots : 0);
  lanes = std::max(lanes, same ? E->lanes : 0);
  free_all(E);
  E->sh = sh;
  Ws& w = E->ws;
  w.s_phi = sh.dim;
  w.s_alpha = sh.N;
  w.s_G = sh.n * (sh.cplx ? 2 : 1);
  w.s_W = sh.n;
  w.s_zpart = sh.nzb;
  w.s_part = (long long)sh.K * sh.dim;
  w.s_tpart = (long long)sh.K * sh.N;
  w.s_tile = sh.tiles;
  const size_t S = (size_t)std::max(slots, 1);
  BCHK(cudaMalloc(&w.phi, S * w.s_phi * 8));
  BCHK(cudaMalloc(&w.alpha, S * w.s_alpha * 8));
  BCHK(cudaMalloc(&w.G, S * std::max<long long>(w.s_G, 1) * 8));
  BCHK(cudaMalloc(&w.W, S * std::max<long long>(w.s_W, 1) * 8));
  BCHK(cudaMalloc(&w.zpart, S * w.s_zpart * 8));
  BCHK(cudaMalloc(&w.part, S * w.s_part * 8));
  BCHK(cudaMalloc(&w.tpart, S * w.s_tpart * 8));
  BCHK(cudaMalloc(&w.tmu, S * w.s_tile * 8));
  BCHK(cudaMalloc(&w.targ, S * w.s_tile * 8));
  BCHK(cudaMalloc(&E->reqs, S * sizeof(Req)));
  BCHK(cudaMalloc(&E->outs, S * sizeof(ReqOut)));
  BCHK(cudaMalloc(&E->act_obj, S * sizeof(int)));
  BCHK(cudaMalloc(&E->act_coh, S * sizeof(int)));
  BCHK(cudaMalloc(&E->counters, 8 * sizeof(int)));
  BCHK(cudaMalloc(&E->next, sizeof(int)));
  if (lanes > 0) {
    BCHK(cudaMalloc(&E->paused, (size_t)lanes * sizeof(int)));
    BCHK(cudaMalloc(&E->lanevec, (size_t)lanes * sizeof(Lane)));
    BCHK(cudaMalloc(&E->vecs, (size_t)lanes * NVEC * sh.dim * 8));
  }
  E->slots = (int)S;
  E->lanes = lanes;
  E->valid = true;
  return TRSTMI_OK;
}

// Lanes / slots that fit a memory budget (a share of the free device memory).
static int lanes_for_memory(const Shape& sh, long long want) {
  size_t fr = 0, tot = 0;
  cudaMemGetInfo(&fr, &tot);
  const double budget = std::min<double>(0.55 * (double)fr, 96e9);
  const double per_lane = 8.0 * (2.0 * slot_doubles(sh) + (double)NVEC * sh.dim) + sizeof(Lane) + 2 * sizeof(Req);
  const long long cap = std::max<long long>(1, (long long)(budget / per_lane));
  return (int)std::max<long long>(1, std::min<long long>(want, std::min<long long>(cap, 4096)));
}
static int slots_for_memory(const Shape& sh, long long want) {
  size_t fr = 0, tot = 0;
  cudaMemGetInfo(&fr, &tot);
  const double budget = std::min<double>(0.5 * (double)fr, 64e9);
  const long long cap = std::max<long long>(1, (long long)(budget / (8.0 * slot_doubles(sh))));
  return (int)std::max<long long>(1, std::min<long long>(want, std::min<long long>(cap, 8192)));
}

static int ib_for(const Shape& sh) {
  if (sh.cplx) return sh.d > 64 ? 128 : (sh.d > 32 ? 64 : 32);
  return sh.d > 32 ? 64 : 32;
}

// Chunk groups per request: a CTA walks K / KS consecutive CAS chunks (one software pipeline over all of
// them); the k range is split only as far as the grid needs to fill the GPU (~3 CTAs per SM).
static int chunk_groups(const Shape& sh, int ib, int nreq) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  const long long per = (long long)((sh.N + BT - 1) / BT) * ((sh.d + ib - 1) / ib) * nreq;
  long long ks = (3LL * sms + per - 1) / per;
  if (ks < 1) ks = 1;
  if (ks > sh.K) ks = sh.K;
  return (int)ks;
}

template <bool CPLX, int IB>
static cudaError_t launch_grad(const Pipe& P, int nreq, int KS, cudaStream_t st) {
  using C = GradWsCfg<CPLX, IB>;
  const cudaError_t e = ensure_smem((const void*)bde_grad_ws<CPLX, IB>, C::smem);
  if (e != cudaSuccess) return e;
  dim3 grid((P.sh.N + BT - 1) / BT, (P.sh.d + IB - 1) / IB, KS * nreq);
  bde_grad_ws<CPLX, IB><<<grid, C::NTHR, C::smem, st>>>(P, KS);
  return cudaGetLastError();
}

// Gram tiles.  Operand staging: 8-byte cp.async (default) or TMA bulk copies of the 256-byte row segments
// (TRSTMI_GRAM_TMA=1, needs L % 4 == 0).  Measured on B200 (profiles/r2_gram_tma_vs_cpasync.txt): the bulk
// variant is bit-identical and 28-38 % slower — 128 copies of 256 bytes per stage are bound by the copy
// engine's per-request rate, not by bytes; a 2-D tensor map (one box per operand per stage) would need a
// 16-byte swizzle that the f64 m16n8k4 fragment pattern turns into 2-way bank conflicts.
static bool gram_tma_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("TRSTMI_GRAM_TMA");
    return e && e[0] == '1';
  }();
  return on;
}

template <int MODE>
static cudaError_t launch_gram(const Pipe& P, int nreq, cudaStream_t st) {
  const Shape& sh = P.sh;
  const bool tma = gram_tma_enabled() && sh.L % 4 == 0;
  const void* fn = sh.cplx ? (tma ? (const void*)bde_gram<true, MODE, true> : (const void*)bde_gram<true, MODE, false>)
                           : (tma ? (const void*)bde_gram<false, MODE, true> : (const void*)bde_gram<false, MODE, false>);
  const cudaError_t e = ensure_smem(fn, bde_gram_smem());
  if (e != cudaSuccess) return e;
  Pipe Pc = P;
  void* args[] = {&Pc};
  return cudaLaunchKernel(fn, dim3(sh.tiles, nreq), dim3(256), args, bde_gram_smem(), st);
}

// The evaluation pipeline over the requests listed in act (device), nreq of them.
static int run_obj(Engine* E, const int* act, int nreq, bool any_wout, cudaStream_t st, std::string* err) {
  if (nreq <= 0) return TRSTMI_OK;
  const Shape& sh = E->sh;
  Pipe P{sh, E->reqs, E->outs, act, E->ws};
  const int nc = bde_norm_cols(sh.L);
  BCHK(ensure_smem((const void*)bde_normalize, bde_norm_smem(sh.L)));
  bde_normalize<<<dim3((sh.N + nc - 1) / nc, nreq), NORM_T, bde_norm_smem(sh.L), st>>>(P);
  BCHK((launch_gram<0>(P, nreq, st)));
  if (sh.cplx) bde_weights<true><<<dim3(sh.nzb, nreq), BZLANES, 0, st>>>(P);
  else bde_weights<false><<<dim3(sh.nzb, nreq), BZLANES, 0, st>>>(P);
  bde_zreduce<<<nreq, 32, 0, st>>>(P);
  const int ib = ib_for(sh);
  const int KS = chunk_groups(sh, ib, nreq);
  cudaError_t e;
  if (sh.cplx) e = ib == 128 ? launch_grad<true, 128>(P, nreq, KS, st) : ib == 64 ? launch_grad<true, 64>(P, nreq, KS, st)
                                                                                  : launch_grad<true, 32>(P, nreq, KS, st);
  else e = ib == 64 ? launch_grad<false, 64>(P, nreq, KS, st) : launch_grad<false, 32>(P, nreq, KS, st);
  BCHK(e);
  bde_finalize<<<dim3((unsigned)((sh.dim + 255) / 256), nreq), 256, 0, st>>>(P);
  g_launches += 6;
  if (any_wout) {
    bde_wout<<<dim3(256, nreq), 256, 0, st>>>(P);
    ++g_launches;
  }
  BCHK(cudaGetLastError());
  return TRSTMI_OK;
}

static int run_coh(Engine* E, const int* act, int nreq, cudaStream_t st, std::string* err) {
  if (nreq <= 0) return TRSTMI_OK;
  const Shape& sh = E->sh;
  Pipe P{sh, E->reqs, E->outs, act, E->ws};
  const int nc = bde_norm_cols(sh.L);
  BCHK(ensure_smem((const void*)bde_normalize, bde_norm_smem(sh.L)));
  bde_normalize<<<dim3((sh.N + nc - 1) / nc, nreq), NORM_T, bde_norm_smem(sh.L), st>>>(P);
  BCHK((launch_gram<1>(P, nreq, st)));
  bde_coh_reduce<<<nreq, 256, 0, st>>>(P);
  g_launches += 3;
  BCHK(cudaGetLastError());
  return TRSTMI_OK;
}

static Req make_req(const double* x, const double* dir, double sc, double delta, double* grad, double* wout, int kind,
                    int squared, int slot) {
  Req r;
  r.x = x;
  r.dir = dir;
  r.sc = sc;
  r.delta = delta;
  r.grad = grad;
  r.wout = wout;
  r.kind = kind;
  r.squared = squared;
  r.slot = slot;
  r.pad = 0;
  return r;
}

static ReqOut fresh_out() {
  ReqOut o;
  std::memset(&o, 0, sizeof(o));
  o.argmax = -1;
  o.zc = INT_MAX;
  return o;
}

// Upload B requests (slots 0..B-1), run, read the outputs back.
static int run_requests(Engine* E, const std::vector<Req>& rq, bool coh, bool any_wout, std::vector<ReqOut>& out,
                        cudaStream_t st, std::string* err) {
  const int B = (int)rq.size();
  std::vector<ReqOut> init(B, fresh_out());
  std::vector<int> act(B);
  for (int b = 0; b < B; ++b) act[b] = b;
  BCHK(cudaMemcpyAsync(E->reqs, rq.data(), B * sizeof(Req), cudaMemcpyHostToDevice, st));
  BCHK(cudaMemcpyAsync(E->outs, init.data(), B * sizeof(ReqOut), cudaMemcpyHostToDevice, st));
  BCHK(cudaMemcpyAsync(E->act_obj, act.data(), B * sizeof(int), cudaMemcpyHostToDevice, st));
  int rc = coh ? run_coh(E, E->act_obj, B, st, err) : run_obj(E, E->act_obj, B, any_wout, st, err);
  if (rc) return rc;
  out.resize(B);
  BCHK(cudaMemcpyAsync(out.data(), E->outs, B * sizeof(ReqOut), cudaMemcpyDeviceToHost, st));
  BCHK(cudaStreamSynchronize(st));
  return TRSTMI_OK;
}

int eval_points(Engine* E, cudaStream_t st, int field, int d, int N, int B, const double* pts, const double* dirs,
                const double* sc, const double* delta, int squared, double* grads, double* weights, double* F,
                double* s, long long* zc, std::string* err) {
  cudaSetDevice(E->device);
  const Shape sh = make_shape(field, d, N);
  const int chunk = slots_for_memory(sh, B);
  int rc = ensure(E, sh, chunk, 0, err);
  if (rc) return rc;
  for (int b0 = 0; b0 < B; b0 += chunk) {
    const int nb = std::min(chunk, B - b0);
    std::vector<Req> rq(nb);
    for (int i = 0; i < nb; ++i) {
      const int b = b0 + i;
      rq[i] = make_req(pts + (long long)b * sh.dim, dirs ? dirs + (long long)b * sh.dim : nullptr, sc ? sc[b] : 0.0,
                       delta[b], grads + (long long)b * sh.dim, weights ? weights + (long long)b * sh.n : nullptr,
                       REQ_OBJ, squared, i);
    }
    std::vector<ReqOut> out;
    if ((rc = run_requests(E, rq, false, weights != nullptr, out, st, err))) return rc;
    for (int i = 0; i < nb; ++i) {
      const int b = b0 + i;
      const bool z = out[i].zc != INT_MAX;
      F[b] = out[i].F;
      s[b] = z ? 0.0 : out[i].s;
      zc[b] = z ? out[i].zc : -1;
    }
  }
  return TRSTMI_OK;
}

int hvp_points(Engine* E, cudaStream_t st, int field, int d, int N, int B, const double* pts, const double* dirs,
               const double* delta, double* hv, int* path, long long* zc, std::string* err) {
  cudaSetDevice(E->device);
  const Shape sh = make_shape(field, d, N);
  const long long dim = sh.dim;
  const int chunk = std::max(1, slots_for_memory(sh, 3LL * B) / 3);
  int rc = ensure(E, sh, 3 * chunk, 0, err);
  if (rc) return rc;
  // scratch: gp, gm, g0 (3 x chunk x dim), norms, modes, h
  const size_t need = (size_t)3 * chunk * dim * 8 + (size_t)chunk * (2 * 8 + 8 + 8);
  if (E->scratch_bytes < need) {
    dfree(E->scratch);
    BCHK(cudaMalloc(&E->scratch, need));
    E->scratch_bytes = need;
  }
  double* gp = E->scratch;
  double* gm = gp + (size_t)chunk * dim;
  double* g0 = gm + (size_t)chunk * dim;
  double* nn = g0 + (size_t)chunk * dim;
  double* hh = nn + 2 * (size_t)chunk;
  int* mode = reinterpret_cast<int*>(hh + chunk);
  for (int b0 = 0; b0 < B; b0 += chunk) {
    const int nb = std::min(chunk, B - b0);
    const double* P0 = pts + (long long)b0 * dim;
    const double* D0 = dirs + (long long)b0 * dim;
    bde_hvp_prep<<<nb, TR_T, 0, st>>>(P0, D0, dim, nn);
    ++g_launches;
    std::vector<double> hn(2 * nb);
    BCHK(cudaMemcpyAsync(hn.data(), nn, 2 * nb * 8, cudaMemcpyDeviceToHost, st));
    BCHK(cudaStreamSynchronize(st));
    std::vector<double> h(nb, 0.0);
    std::vector<int> md(nb, 3);
    std::vector<Req> rq;
    std::vector<int> who;  // point of each request (+ kind: 0 plus, 1 minus, 2 base)
    for (int i = 0; i < nb; ++i) {
      const double dn = std::sqrt(hn[2 * i]);
      if (dn == 0.0) {
        path[b0 + i] = TRSTMI_HVP_ZERO_DIR;
        zc[b0 + i] = -1;
        continue;
      }
      h[i] = trstmi_dev::kFdBaseStep * (1.0 + std::sqrt(hn[2 * i + 1])) / std::max(dn, 1e-300);
      const double* x = P0 + (long long)i * dim;
      const double* v = D0 + (long long)i * dim;
      rq.push_back(make_req(x, v, h[i], delta[b0 + i], gp + (long long)i * dim, nullptr, REQ_OBJ, 1, (int)rq.size()));
      who.push_back(3 * i);
      rq.push_back(make_req(x, v, -h[i], delta[b0 + i], gm + (long long)i * dim, nullptr, REQ_OBJ, 1, (int)rq.size()));
      who.push_back(3 * i + 1);
    }
    std::vector<ReqOut> out;
    if (!rq.empty() && (rc = run_requests(E, rq, false, false, out, st, err))) return rc;
    std::vector<int> zp(nb, INT_MAX), zm(nb, INT_MAX);
    for (size_t r = 0; r < rq.size(); ++r) (who[r] % 3 == 0 ? zp : zm)[who[r] / 3] = out[r].zc;
    // the one-sided fallbacks need g0 = eval(x) (solver.hpp:128)
    std::vector<Req> rq0;
    std::vector<int> who0;
    for (int i = 0; i < nb; ++i) {
      if (h[i] == 0.0) continue;
      if (zp[i] == INT_MAX && zm[i] == INT_MAX) {
        md[i] = 0;
        path[b0 + i] = TRSTMI_HVP_CENTRAL;
        zc[b0 + i] = -1;
        continue;
      }
      rq0.push_back(make_req(P0 + (long long)i * dim, nullptr, 0.0, delta[b0 + i], g0 + (long long)i * dim, nullptr,
                             REQ_OBJ, 1, (int)rq0.size()));
      who0.push_back(i);
      if (zp[i] == INT_MAX) {
        md[i] = 1;
        path[b0 + i] = TRSTMI_HVP_FORWARD;
        zc[b0 + i] = -1;
      } else if (zm[i] == INT_MAX) {
        md[i] = 2;
        path[b0 + i] = TRSTMI_HVP_BACKWARD;
        zc[b0 + i] = -1;
      } else {
        md[i] = 3;
        path[b0 + i] = TRSTMI_HVP_FAILED;
        zc[b0 + i] = zm[i];
      }
    }
    if (!rq0.empty() && (rc = run_requests(E, rq0, false, false, out, st, err))) return rc;
    BCHK(cudaMemcpyAsync(hh, h.data(), nb * 8, cudaMemcpyHostToDevice, st));
    BCHK(cudaMemcpyAsync(mode, md.data(), nb * sizeof(int), cudaMemcpyHostToDevice, st));
    bde_hvp_combine<<<dim3((unsigned)std::min<long long>((dim + 255) / 256, 1024), nb), 256, 0, st>>>(
        hv + (long long)b0 * dim, gp, gm, g0, mode, hh, dim);
    ++g_launches;
    BCHK(cudaGetLastError());
  }
  BCHK(cudaStreamSynchronize(st));
  return TRSTMI_OK;
}

int coherence_points(Engine* E, cudaStream_t st, int field, int d, int N, int B, const double* frames, int normalize,
                     double* mu, long long* argmax, long long* zc, std::string* err) {
  cudaSetDevice(E->device);
  const Shape sh = make_shape(field, d, N);
  const int chunk = slots_for_memory(sh, B);
  int rc = ensure(E, sh, chunk, 0, err);
  if (rc) return rc;
  for (int b0 = 0; b0 < B; b0 += chunk) {
    const int nb = std::min(chunk, B - b0);
    std::vector<Req> rq(nb);
    for (int i = 0; i < nb; ++i)
      rq[i] = make_req(frames + (long long)(b0 + i) * sh.dim, nullptr, 0.0, 1.0, nullptr, nullptr,
                       normalize ? REQ_COH_NORM : REQ_COH_RAW, 1, i);
    std::vector<ReqOut> out;
    if ((rc = run_requests(E, rq, true, false, out, st, err))) return rc;
    for (int i = 0; i < nb; ++i) {
      const bool z = normalize && out[i].zc != INT_MAX;
      mu[b0 + i] = z ? 0.0 : out[i].mu;
      argmax[b0 + i] = z ? -1 : out[i].argmax;
      zc[b0 + i] = z ? out[i].zc : -1;
    }
  }
  return TRSTMI_OK;
}

int anneal(Engine* E, cudaStream_t st, int field, int d, int N, const TrCfg& tr, const std::vector<double>& schedule,
           int record_cap, long long trials, double* params, double* frames, uint64_t* rng_state,
           trstmi_trial_out* tout, trstmi_stage_out* sout, trstmi_outer_out* oout, std::string* err) {
  if (trials <= 0) return TRSTMI_OK;
  cudaSetDevice(E->device);
  const Shape sh = make_shape(field, d, N);
  const int nl = lanes_for_memory(sh, trials);
  int rc = ensure(E, sh, 2 * nl, nl, err);
  if (rc) return rc;
  TrArgs A;
  std::memset(&A, 0, sizeof(A));
  A.sh = sh;
  A.tr = TrCfgD{tr.delta0, tr.delta_max, tr.eta, tr.shrink, tr.grow, tr.grad_tol, tr.cg_force_c, tr.max_outer, tr.max_cg};
  A.n_stages = (int)schedule.size();
  A.stage_end = A.n_stages;
  for (int k = 0; k < A.n_stages; ++k) A.schedule[k] = schedule[k];
  A.record_cap = record_cap;
  A.n_list = (int)trials;
  A.next = E->next;
  A.lanes = E->lanevec;
  A.vecs = E->vecs;
  A.params = params;
  A.frames = frames;
  A.tout = tout;
  A.sout = sout;
  A.oout = oout;
  A.reqs = E->reqs;
  A.outs = E->outs;
  A.act_obj = E->act_obj;
  A.act_coh = E->act_coh;
  A.counters = E->counters;
  A.paused = E->paused;
  std::vector<Lane> init(nl);
  std::memset(init.data(), 0, nl * sizeof(Lane));
  for (auto& l : init) {
    l.phase = PH_START;
    l.trial = -1;
  }
  BCHK(cudaMemcpyAsync(E->lanevec, init.data(), nl * sizeof(Lane), cudaMemcpyHostToDevice, st));
  BCHK(cudaMemsetAsync(E->next, 0, sizeof(int), st));
  const long long dim = sh.dim;
  std::vector<double> host;
  for (long long tick = 0;; ++tick) {
    BCHK(cudaMemsetAsync(E->counters, 0, 4 * sizeof(int), st));
    bde_advance<<<nl, TR_T, 0, st>>>(A);
    ++g_launches;
    BCHK(cudaGetLastError());
    BCHK(cudaMemcpyAsync(E->h_counters, E->counters, 4 * sizeof(int), cudaMemcpyDeviceToHost, st));
    BCHK(cudaStreamSynchronize(st));
    const int nobj = E->h_counters[0], ncoh = E->h_counters[1], npause = E->h_counters[2], busy = E->h_counters[3];
    if (npause > 0) {  // rescue_zero_columns (solver.hpp:139-156) from the trial's own generator, on the host
      std::vector<int> pl(npause);
      BCHK(cudaMemcpyAsync(pl.data(), E->paused, npause * sizeof(int), cudaMemcpyDeviceToHost, st));
      BCHK(cudaStreamSynchronize(st));
      host.resize(dim);
      for (int l : pl) {
        Lane L;
        BCHK(cudaMemcpyAsync(&L, E->lanevec + l, sizeof(Lane), cudaMemcpyDeviceToHost, st));
        BCHK(cudaStreamSynchronize(st));
        double* x = E->vecs + ((long long)l * NVEC + L.ix[V_X]) * dim;
        BCHK(cudaMemcpyAsync(host.data(), x, dim * 8, cudaMemcpyDeviceToHost, st));
        BCHK(cudaStreamSynchronize(st));
        int bad;
        if (rng_state) {
          trstmi_host::SplitMix64 rng = trstmi_host::SplitMix64::load(rng_state + 3 * L.trial);
          bad = trstmi_host::rescue_zero_columns(sh.cplx, d, N, host.data(), &rng);
          rng.save(rng_state + 3 * L.trial);
        } else {
          bad = trstmi_host::rescue_zero_columns(sh.cplx, d, N, host.data(), nullptr);
        }
        if (bad >= 0) {
          L.status = TRSTMI_TRIAL_ZERO_COLUMN;
          L.zero_col = bad;
          L.fail_stage = L.stage;
          L.phase = PH_FINISH;
        } else {
          BCHK(cudaMemcpyAsync(x, host.data(), dim * 8, cudaMemcpyHostToDevice, st));
          L.status = TRSTMI_TRIAL_OK;
          L.zero_col = -1;
          L.fail_stage = -1;
          L.phase = PH_STAGE_GO;
        }
        BCHK(cudaMemcpyAsync(E->lanevec + l, &L, sizeof(Lane), cudaMemcpyHostToDevice, st));
        BCHK(cudaStreamSynchronize(st));
      }
    }
    if (nobj == 0 && ncoh == 0 && busy == 0 && npause == 0) break;
    if ((rc = run_obj(E, E->act_obj, nobj, false, st, err))) return rc;
    if ((rc = run_coh(E, E->act_coh, ncoh, st, err))) return rc;
  }
  BCHK(cudaStreamSynchronize(st));
  return TRSTMI_OK;
}

}  // namespace trstmi_bde_host
