// Single-point entry kernels (one CTA per batch point) behind the plugin seam
// of the reference (trust_region.hpp:42-49): eval_objective, the
// make_hvp_factory Hessian-vector product and coherence.  They reuse the
// small-path CTA building blocks, so a batch point is evaluated with exactly
// the arithmetic the batched anneal uses.
#pragma once
#include "anneal_small.cuh"

namespace trstmi_dev {

struct BatchArgs {
  Prob P;
  long long B;
  const double* pts;     // B x dim
  const double* dirs;    // B x dim (hvp)
  const double* delta;   // B
  int squared;
  int normalize;         // coherence
  double* F;             // B
  double* s;             // B
  double* out;           // B x dim: gradient / hv
  double* weights;       // nullable B x n
  long long* zero_col;   // B
  int* path;             // B (hvp)
  double* mu;            // B (coherence)
  long long* argmax;     // B (coherence)
};

template <bool CPLX, int DMAX, bool EXACT, int S, bool GS>
__global__ void __launch_bounds__(S, (S >= 512 ? 1 : 512 / S)) eval_batch_kernel(const BatchArgs A) {
  extern __shared__ __align__(16) double smem_raw[];
  Smem sm;
  double* v[3];
  carve<CPLX>(A.P, S, smem_raw, sm, v, 3);
  build_tables<S, CPLX, GS>(A.P, sm);
  int rbuf = 0;
  for (long long b = blockIdx.x; b < A.B; b += gridDim.x) {
    const double* x = A.pts + b * A.P.dim;
    double F, s;
    double* wo = A.weights ? A.weights + b * A.P.n : nullptr;
    const int zc = A.squared
                       ? eval_any<CPLX, DMAX, EXACT, S, GS, true>(A.P, x, nullptr, 0.0, A.delta[b], sm, rbuf,
                                                              A.out + b * A.P.dim, &sm.scal[0], &sm.scal[1], wo)
                       : eval_any<CPLX, DMAX, EXACT, S, GS, false>(A.P, x, nullptr, 0.0, A.delta[b], sm, rbuf,
                                                               A.out + b * A.P.dim, &sm.scal[0], &sm.scal[1], wo);
    F = sm.scal[0];
    s = sm.scal[1];
    if (threadIdx.x == 0) {
      A.F[b] = F;
      A.s[b] = s;
      A.zero_col[b] = zc;
    }
    __syncthreads();
  }
}

// make_hvp_factory(obj)(x)(dir) (solver.hpp:118-137) around
// fd_hessian_vector_product (smoothing.hpp:167-181).
template <bool CPLX, int DMAX, bool EXACT, int S, bool GS>
__global__ void __launch_bounds__(S, (S >= 512 ? 1 : 512 / S)) hvp_batch_kernel(const BatchArgs A) {
  extern __shared__ __align__(16) double smem_raw[];
  Smem sm;
  double* v[3];
  carve<CPLX>(A.P, S, smem_raw, sm, v, 3);
  build_tables<S, CPLX, GS>(A.P, sm);
  double* gp = v[0];
  double* gm = v[1];
  double* g0 = v[2];
  int rbuf = 0;
  const int dim = A.P.dim;
  for (long long b = blockIdx.x; b < A.B; b += gridDim.x) {
    const double* x = A.pts + b * dim;
    const double* dir = A.dirs + b * dim;
    double* hv = A.out + b * dim;
    const double delta = A.delta[b];
    double nn[2] = {dot_partial<S>(dir, dir, dim), dot_partial<S>(x, x, dim)};
    block_sum<S, 2>(nn, sm.red, rbuf);
    const double dn = sqrt(nn[0]);
    int path, zc = -1;
    if (dn == 0.0) {
      for (int i = threadIdx.x; i < dim; i += S) hv[i] = 0.0;
      path = TRSTMI_HVP_ZERO_DIR;
    } else {
      const double h = kFdBaseStep * (1.0 + sqrt(nn[1])) / fmax(dn, 1e-300);
      int zp = INT_MAX - 1;
      if constexpr (GS) {  // both points in one pass (hvp_cta_gs); a vanishing column falls through to the steps below
        if (A.P.dual) zp = hvp_cta_gs<CPLX, DMAX, EXACT, S>(A.P, x, dir, h, delta, sm, rbuf, hv);
      }
      if (zp == -1) {
        path = TRSTMI_HVP_CENTRAL;
      } else if ((zp = eval_any<CPLX, DMAX, EXACT, S, GS>(A.P, x, dir, h, delta, sm, rbuf, gp, nullptr, nullptr,
                                                          nullptr)) < 0) {
        const int zm = eval_any<CPLX, DMAX, EXACT, S, GS>(A.P, x, dir, -h, delta, sm, rbuf, gm, nullptr, nullptr, nullptr);
        if (zm < 0) {
          const double h2 = 2.0 * h;
          for (int i = threadIdx.x; i < dim; i += S) hv[i] = (gp[i] - gm[i]) / h2;
          path = TRSTMI_HVP_CENTRAL;
        } else {
          eval_any<CPLX, DMAX, EXACT, S, GS>(A.P, x, nullptr, 0.0, delta, sm, rbuf, g0, nullptr, nullptr, nullptr);
          for (int i = threadIdx.x; i < dim; i += S) hv[i] = (gp[i] - g0[i]) / h;
          path = TRSTMI_HVP_FORWARD;
        }
      } else {
        eval_any<CPLX, DMAX, EXACT, S, GS>(A.P, x, nullptr, 0.0, delta, sm, rbuf, g0, nullptr, nullptr, nullptr);
        const int zm = eval_any<CPLX, DMAX, EXACT, S, GS>(A.P, x, dir, -h, delta, sm, rbuf, gm, nullptr, nullptr, nullptr);
        if (zm < 0) {
          for (int i = threadIdx.x; i < dim; i += S) hv[i] = (g0[i] - gm[i]) / h;
          path = TRSTMI_HVP_BACKWARD;
        } else {
          for (int i = threadIdx.x; i < dim; i += S) hv[i] = 0.0;
          path = TRSTMI_HVP_FAILED;
          zc = zm;
        }
      }
    }
    if (threadIdx.x == 0) {
      A.path[b] = path;
      A.zero_col[b] = zc;
    }
    __syncthreads();
  }
}

template <bool CPLX, int DMAX, bool EXACT, int S, bool GS>
__global__ void __launch_bounds__(S, (S >= 512 ? 1 : 512 / S)) coherence_batch_kernel(const BatchArgs A) {
  extern __shared__ __align__(16) double smem_raw[];
  Smem sm;
  double* v[1];
  carve<CPLX>(A.P, S, smem_raw, sm, v, 0);
  build_tables<S, CPLX, GS>(A.P, sm);
  int rbuf = 0;
  for (long long b = blockIdx.x; b < A.B; b += gridDim.x) {
    double mu = 0.0;
    long long arg = -1;
    const int zc = coherence_cta<CPLX, DMAX, EXACT, S, GS>(A.P, A.pts + b * A.P.dim, A.normalize != 0, sm, rbuf, &mu, &arg);
    if (threadIdx.x == 0) {
      A.mu[b] = zc >= 0 ? 0.0 : mu;
      A.argmax[b] = zc >= 0 ? -1 : arg;
      A.zero_col[b] = zc;
    }
    __syncthreads();
  }
}

}  // namespace trstmi_dev
