// Host engine of the large-frame path (csrc/large_path.cuh): per-shape device
// workspaces, the evaluation pipeline, CAS dot products, coherence, and the
// trust-region / Steihaug-CG / anneal driver (trust_region.hpp:81-295,
// solver.hpp:118-204) running on the host over device vectors.  Every scalar
// decision is made by the host from CAS-exact device reductions, so the
// trajectory is bit-identical to the oracle with S = 32768 lanes.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/trstmi_b200.h"

namespace trstmi_large {

constexpr int kLanes = 32768;

long long launches();  // kernels launched by the large-frame engine so far

struct Shape {
  int cplx, d, N, L, dim, K;
  long long n;
};

Shape make_shape(int field, int d, int N);

// Path rule: the small-frame family covers d <= 16 when one
// trial's anneal state fits one SM's shared memory; everything else is large.
bool use_large(int field, long long d, long long N);

struct Engine;
Engine* engine_create(int device, cudaStream_t stream);
void engine_destroy(Engine*);
void engine_set_stream(Engine* E, cudaStream_t stream);

// Row-block sharding of a single frame over `world` ranks.
// nccl_id == NULL: virtual ranks, all shares computed on this device (tests);
// else this process is `rank` of a NCCL communicator (128-byte ncclUniqueId).
int engine_set_shard(Engine* E, int world, int rank, const void* nccl_id, std::string* err);
int nccl_unique_id(void* out128, std::string* err);

// All pointers are device pointers.  Returns TRSTMI_* status; *zero_col = -1
// or the first zero column (then *F = +inf and grad = 0).
int eval(Engine* E, const Shape& sh, const double* x, const double* dir, double sc, double delta, int squared,
         double* grad, double* F, double* s, double* weights, long long* zero_col, std::string* err);
int hvp(Engine* E, const Shape& sh, const double* x, const double* dir, double delta, double* hv, int* path,
        long long* zero_col, std::string* err);
int coherence(Engine* E, const Shape& sh, const double* frame, int normalize, double* mu, long long* argmax,
              long long* zero_col, std::string* err);

struct TrCfg {
  double delta0, delta_max, eta, shrink, grow, grad_tol, cg_force_c;
  int max_outer, max_cg;
};
// anneal() of one trial; params (device, in/out), frame (device, out, nullable).
int anneal_trial(Engine* E, const Shape& sh, const TrCfg& tr, const std::vector<double>& schedule, int start_stage,
                 int record_cap, double* params, double* frame, uint64_t* rng_state, trstmi_trial_out* tout,
                 trstmi_stage_out* sout, trstmi_outer_out* oout, std::string* err);

}  // namespace trstmi_large
