// Multi-GPU trial scheduler (replaces solve()'s restart pool
// and best-of selection, solver.hpp:210-273, across one process per GPU).
//
// Trials are independent, so the data path has no collective: restart i runs
// on rank floor(i * world / restarts) (contiguous blocks), each rank anneals
// its block with the single-GPU batched kernels, and the only exchange is the
// final best-of: an NCCL allgather of every rank's (best mu, restart index)
// followed by a broadcast of the winning frame from its owner.  Selection
// compares mu with a strict < in restart-index order (solver.hpp:256-263), so
// the result is bit-identical for every world size.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/trstmi_b200.h"
#include "ctx.hpp"

namespace {

int fail(trstmi_ctx* ctx, int code, const std::string& msg) {
  if (ctx) ctx->err = msg;
  return code;
}

#define SH_CUDA(expr)                                                                              \
  do {                                                                                             \
    cudaError_t e_ = (expr);                                                                       \
    if (e_ != cudaSuccess) return fail(ctx, TRSTMI_ERR_CUDA, std::string(#expr ": ") + cudaGetErrorString(e_)); \
  } while (0)
#define SH_NCCL(expr)                                                                              \
  do {                                                                                             \
    ncclResult_t r_ = (expr);                                                                      \
    if (r_ != ncclSuccess) return fail(ctx, TRSTMI_ERR_NCCL, std::string(#expr ": ") + ncclGetErrorString(r_)); \
  } while (0)

struct DevBuf {
  void* p = nullptr;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
};

}  // namespace

extern "C" {

int trstmi_shard_range(int64_t restarts, int world, int rank, int64_t* first, int64_t* count) {
  if (restarts < 0 || world < 1 || rank < 0 || rank >= world || !first || !count) return TRSTMI_ERR_INVALID_ARG;
  // {i : floor(i * world / restarts) == r} = [ceil(r T / G), ceil((r+1) T / G))
  auto lo = [&](int64_t r) { return (r * restarts + world - 1) / world; };
  *first = lo(rank);
  *count = lo(rank + 1) - *first;
  return TRSTMI_OK;
}

int trstmi_select_best(int64_t n, const double* mu, const int64_t* index, const int32_t* ok, int64_t* best_pos) {
  if (n < 0 || !mu || !best_pos) return TRSTMI_ERR_INVALID_ARG;
  int64_t best = -1;
  for (int64_t i = 0; i < n; ++i) {
    if (ok && !ok[i]) continue;
    if (std::isnan(mu[i])) continue;
    const int64_t id = index ? index[i] : i;
    if (best < 0 || mu[i] < mu[best] || (mu[i] == mu[best] && id < (index ? index[best] : best))) best = i;
  }
  *best_pos = best;
  return best < 0 ? TRSTMI_ERR_ALL_FAILED : TRSTMI_OK;
}

int trstmi_comm_init(trstmi_ctx* ctx, int world, int rank, const char* nccl_id) {
  if (!ctx || world < 1 || rank < 0 || rank >= world) return TRSTMI_ERR_INVALID_ARG;
  cudaSetDevice(ctx->device);
  if (ctx->comm) {
    ncclCommDestroy(ctx->comm);
    ctx->comm = nullptr;
  }
  ctx->world = world;
  ctx->rank = rank;
  if (world == 1) return TRSTMI_OK;
  if (!nccl_id) return fail(ctx, TRSTMI_ERR_INVALID_ARG, "comm_init: world > 1 needs an NCCL unique id");
  ncclUniqueId id;
  std::memcpy(&id, nccl_id, sizeof(id));
  SH_NCCL(ncclCommInitRank(&ctx->comm, world, id, rank));
  return TRSTMI_OK;
}

int trstmi_best_of_ranks(trstmi_ctx* ctx, int64_t dim, double local_mu, int64_t local_index,
                         const double* local_frame_dev, double* best_frame_dev, double* best_mu,
                         int64_t* best_index, void* stream) {
  if (!ctx || dim < 1 || !best_frame_dev || !best_mu || !best_index) return TRSTMI_ERR_INVALID_ARG;
  cudaSetDevice(ctx->device);
  cudaStream_t st = stream ? (cudaStream_t)stream : ctx->stream;
  const int W = ctx->world;
  // (mu, index) of every rank; a rank without a successful trial sends NaN.
  std::vector<double> all(2 * (size_t)W);
  if (W == 1) {
    all[0] = local_mu;
    all[1] = (double)local_index;
  } else {
    if (!ctx->comm) return fail(ctx, TRSTMI_ERR_INVALID_ARG, "best_of_ranks: call trstmi_comm_init first");
    DevBuf d;
    SH_CUDA(cudaMalloc(&d.p, sizeof(double) * 2 * (W + 1)));
    double* mine = (double*)d.p + 2 * W;
    const double h[2] = {local_mu, (double)local_index};
    SH_CUDA(cudaMemcpyAsync(mine, h, sizeof(h), cudaMemcpyHostToDevice, st));
    SH_NCCL(ncclAllGather(mine, d.p, 2, ncclDouble, ctx->comm, st));
    SH_CUDA(cudaMemcpyAsync(all.data(), d.p, sizeof(double) * 2 * W, cudaMemcpyDeviceToHost, st));
    SH_CUDA(cudaStreamSynchronize(st));
  }
  std::vector<double> mus(W);
  std::vector<int64_t> ids(W);
  for (int r = 0; r < W; ++r) {
    mus[r] = all[2 * r];
    ids[r] = (int64_t)all[2 * r + 1];
  }
  int64_t owner = -1;
  const int rc = trstmi_select_best(W, mus.data(), ids.data(), nullptr, &owner);
  if (rc) return fail(ctx, rc, "solve: all restarts failed");
  *best_mu = mus[owner];
  *best_index = ids[owner];
  if (W == 1) {
    if (best_frame_dev != local_frame_dev)
      SH_CUDA(cudaMemcpyAsync(best_frame_dev, local_frame_dev, sizeof(double) * dim, cudaMemcpyDeviceToDevice, st));
  } else {
    if (ctx->rank == owner && best_frame_dev != local_frame_dev)
      SH_CUDA(cudaMemcpyAsync(best_frame_dev, local_frame_dev, sizeof(double) * dim, cudaMemcpyDeviceToDevice, st));
    SH_NCCL(ncclBroadcast(best_frame_dev, best_frame_dev, (size_t)dim, ncclDouble, (int)owner, ctx->comm, st));
  }
  SH_CUDA(cudaStreamSynchronize(st));
  return TRSTMI_OK;
}

int trstmi_solve_sharded(trstmi_ctx* ctx, const trstmi_cfg* cfg, int64_t restarts, uint64_t seed, double* best_frame,
                         double* best_coherence, int64_t* best_restart, trstmi_trial_out* local_trial_out,
                         int64_t* local_first, int64_t* local_count) {
  if (!ctx || !cfg || !best_frame || !best_coherence || !best_restart) return TRSTMI_ERR_INVALID_ARG;
  if (cfg->d < 1 || cfg->N < 1) return fail(ctx, TRSTMI_ERR_INVALID_ARG, "solve: need d, N >= 1");
  if (restarts < 1) return fail(ctx, TRSTMI_ERR_INVALID_ARG, "solve: need restarts >= 1");
  int64_t first = 0, count = 0;
  int rc = trstmi_shard_range(restarts, ctx->world, ctx->rank, &first, &count);
  if (rc) return rc;
  if (local_first) *local_first = first;
  if (local_count) *local_count = count;
  const int64_t dim = (cfg->field == TRSTMI_COMPLEX ? 2 : 1) * (int64_t)cfg->d * cfg->N;
  std::vector<double> params((size_t)std::max<int64_t>(count, 1) * dim), frames(params.size());
  std::vector<uint64_t> rng((size_t)std::max<int64_t>(count, 1) * 3);
  std::vector<trstmi_trial_out> to((size_t)std::max<int64_t>(count, 1));
  double mu = std::nan("");
  int64_t idx = -1, pos = -1;
  if (count > 0) {
    rc = trstmi_random_frames(cfg->field, cfg->d, cfg->N, seed, first, count, params.data(), rng.data());
    if (rc) return fail(ctx, rc, "random_frame failed");
    int n_stages = cfg->n_stages ? cfg->n_stages : trstmi_default_schedule(cfg->N, cfg->eps_target, nullptr, 0);
    std::vector<trstmi_stage_out> so((size_t)count * std::max(n_stages, 1));
    rc = trstmi_solve_batch(ctx, cfg, count, params.data(), rng.data(), frames.data(), to.data(), so.data(), nullptr);
    if (rc) return rc;
    std::vector<double> mus(count);
    std::vector<int32_t> ok(count);
    for (int64_t t = 0; t < count; ++t) {
      mus[t] = to[t].coherence;
      ok[t] = to[t].status == TRSTMI_TRIAL_OK;
    }
    if (trstmi_select_best(count, mus.data(), nullptr, ok.data(), &pos) == TRSTMI_OK) {
      mu = mus[pos];
      idx = first + pos;
    }
    if (local_trial_out) std::memcpy(local_trial_out, to.data(), sizeof(trstmi_trial_out) * count);
  }
  cudaSetDevice(ctx->device);
  DevBuf dl, db;
  SH_CUDA(cudaMalloc(&dl.p, sizeof(double) * dim));
  SH_CUDA(cudaMalloc(&db.p, sizeof(double) * dim));
  if (pos >= 0)
    SH_CUDA(cudaMemcpyAsync(dl.p, frames.data() + pos * dim, sizeof(double) * dim, cudaMemcpyHostToDevice, ctx->stream));
  else
    SH_CUDA(cudaMemsetAsync(dl.p, 0, sizeof(double) * dim, ctx->stream));
  rc = trstmi_best_of_ranks(ctx, dim, mu, idx, (const double*)dl.p, (double*)db.p, best_coherence, best_restart,
                            ctx->stream);
  if (rc) return rc;
  SH_CUDA(cudaMemcpyAsync(best_frame, db.p, sizeof(double) * dim, cudaMemcpyDeviceToHost, ctx->stream));
  SH_CUDA(cudaStreamSynchronize(ctx->stream));
  return TRSTMI_OK;
}

// solve() (solver.hpp:210-273) over several GPUs of ONE process — the drop-in for a caller that today passes
// `threads` to solve(): one host thread per listed device (the reference's restart pool, one worker per GPU) anneals
// the contiguous block trstmi_shard_range gives it on a context of its own; the best-of scan then runs over the
// blocks in restart order with a strict <, so the result is the single-GPU one bit for bit whatever the device list
// (a device may be listed more than once).  No NCCL: the exchange is host memory.
int trstmi_solve_devices(const int* devices, int ndev, const trstmi_cfg* cfg, int64_t restarts, uint64_t seed,
                         double* best_frame, double* best_coherence, int64_t* best_restart,
                         trstmi_trial_out* trial_out, trstmi_stage_out* stage_out) {
  if (!devices || ndev < 1 || !cfg || !best_frame || !best_coherence || !best_restart) return TRSTMI_ERR_INVALID_ARG;
  if (cfg->d < 1 || cfg->N < 1 || restarts < 1) return TRSTMI_ERR_INVALID_ARG;
  const int64_t dim = (cfg->field == TRSTMI_COMPLEX ? 2 : 1) * (int64_t)cfg->d * cfg->N;
  const int n_stages = cfg->n_stages ? cfg->n_stages : trstmi_default_schedule(cfg->N, cfg->eps_target, nullptr, 0);
  struct Shard {
    int rc = TRSTMI_OK;
    int64_t first = 0, count = 0, best = -1;
    double mu = 0.0;
    std::vector<double> frame;
  };
  std::vector<Shard> sh(ndev);
  std::vector<std::thread> pool;
  for (int r = 0; r < ndev; ++r) {
    trstmi_shard_range(restarts, ndev, r, &sh[r].first, &sh[r].count);
    sh[r].frame.resize(dim);
    pool.emplace_back([&, r]() {
      Shard& S = sh[r];
      if (S.count == 0) return;
      trstmi_ctx* c = nullptr;
      S.rc = trstmi_ctx_create(devices[r], &c);
      if (S.rc) return;
      S.rc = trstmi_solve(c, cfg, S.count, seed, S.first, S.frame.data(), &S.mu, &S.best,
                          trial_out ? trial_out + S.first : nullptr,
                          stage_out ? stage_out + S.first * std::max(n_stages, 1) : nullptr);
      trstmi_ctx_destroy(c);
    });
  }
  for (auto& t : pool) t.join();
  int64_t win = -1;
  for (int r = 0; r < ndev; ++r) {
    if (sh[r].count == 0 || sh[r].rc == TRSTMI_ERR_ALL_FAILED) continue;  // a block without a successful restart
    if (sh[r].rc) return sh[r].rc;
    if (win < 0 || sh[r].mu < sh[win].mu) win = r;  // strict <: the lowest restart index wins ties (solver.hpp:259)
  }
  if (win < 0) return TRSTMI_ERR_ALL_FAILED;
  *best_coherence = sh[win].mu;
  *best_restart = sh[win].first + sh[win].best;
  std::memcpy(best_frame, sh[win].frame.data(), sizeof(double) * dim);
  return TRSTMI_OK;
}

}  // extern "C"
