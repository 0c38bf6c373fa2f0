// Host side of the batched device engine for large frames (csrc/bde.cuh,
// csrc/bde_tr.cuh): workspaces, the per-tick launch sequence, the rare
// host-side column rescue, and the single-point entry points (objective,
// Hessian-vector product, coherence) batched over their B points.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/trstmi_b200.h"

namespace trstmi_bde_host {

long long launches();

struct Engine;
Engine* create(int device);
void destroy(Engine* E);

struct TrCfg {
  double delta0, delta_max, eta, shrink, grow, grad_tol, cg_force_c;
  int max_outer, max_cg;
};

// All array pointers are device pointers unless noted; st is the stream of
// the call (every launch and copy of the call is ordered on it).
// Objective at pts[b] (+ sc[b] * dirs[b]); sc / delta / F / s / zc on the host.
int eval_points(Engine* E, cudaStream_t st, int field, int d, int N, int B, const double* pts, const double* dirs,
                const double* sc, const double* delta, int squared, double* grads, double* weights, double* F,
                double* s, long long* zc, std::string* err);
// make_hvp_factory semantics (solver.hpp:118-137); path / zc on the host.
int hvp_points(Engine* E, cudaStream_t st, int field, int d, int N, int B, const double* pts, const double* dirs,
               const double* delta, double* hv, int* path, long long* zc, std::string* err);
// coherence (frame.hpp:138-145), optionally of normalize_columns; host outputs.
int coherence_points(Engine* E, cudaStream_t st, int field, int d, int N, int B, const double* frames, int normalize,
                     double* mu, long long* argmax, long long* zc, std::string* err);
// anneal() of `trials` trials, stages [0, n_stages): params (in/out), frames
// (out, nullable), tout / sout / oout device arrays; rng_state host (nullable).
int anneal(Engine* E, cudaStream_t st, int field, int d, int N, const TrCfg& tr, const std::vector<double>& schedule,
           int record_cap, long long trials, double* params, double* frames, uint64_t* rng_state,
           trstmi_trial_out* tout, trstmi_stage_out* sout, trstmi_outer_out* oout, std::string* err);

}  // namespace trstmi_bde_host
