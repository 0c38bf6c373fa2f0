// Small-frame path: one CTA owns one trial (or one batch point) and keeps the
// whole trust-region state in shared memory.  Used for BASELINE configs 1-3
// (real d=4 N=10; complex d=2 N=100; complex d=6 N=36) and any shape whose
// state fits in one SM's shared memory.
//
// Every floating-point operation follows the Canonical Arithmetic Spec
// so results are bit-identical to the CPU oracle: the file is
// compiled with -fmad=false and fuses only at explicit fma() sites; all CTA
// reductions use the CAS lane-strided / xor-butterfly / warp-sequential order.
//
// Reference functions restated here (paths under /root/reference/proj/include/trstmi):
//   eval_cta            eval_objective           smoothing.hpp:82-162
//   hvp (in tr loop)    make_hvp_factory         solver.hpp:118-137
//                       fd_hessian_vector_product smoothing.hpp:167-181
//   steihaug (inline)   steihaug_cg              trust_region.hpp:81-154
//   tr loop             trust_region_minimize    trust_region.hpp:189-295
//   stage loop          anneal                   solver.hpp:164-204
//   coherence_cta       coherence/normalize      frame.hpp:60-69,138-145
#pragma once
#include <climits>
#include <cstdint>

#include "cas_math.cuh"
#include "../../include/trstmi_b200.h"

namespace trstmi_dev {

constexpr double kZeroColumnTol = 1e-12;               // frame.hpp:20
constexpr double kFdBaseStep = 0x1.965fea53d6e3dp-18;  // smoothing.hpp:16-17 (glibc cbrt(DBL_EPSILON))
constexpr double kUnderflowCut = -746.0;               // exp((x-s)/delta) == 0 below this * delta
constexpr unsigned FULL = 0xffffffffu;

struct Prob {
  int d, N, L, dim, n;  // L = doubles per column (2d complex, d real); n = pairs
};

// ------------------------------------------------------------------ CTA reductions
// CAS sum: lanes already hold their strided partials; xor butterfly inside
// each warp, then the S/32 warp totals left to right.  Result is identical in
// every thread.  Two alternating scratch buffers make one __syncthreads per
// reduction sufficient.
template <int S, int K>
__device__ __forceinline__ void block_sum(double (&v)[K], double* red, int& rbuf) {
  constexpr int W = S / 32;
#pragma unroll
  for (int k = 0; k < K; ++k)
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) v[k] = __dadd_rn(v[k], __shfl_xor_sync(FULL, v[k], off));
  if constexpr (W > 1) {
    double* buf = red + rbuf * (4 * W);
    const int warp = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
#pragma unroll
      for (int k = 0; k < K; ++k) buf[k * W + warp] = v[k];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double t = buf[k * W];
#pragma unroll
      for (int w = 1; w < W; ++w) t = __dadd_rn(t, buf[k * W + w]);
      v[k] = t;
    }
    rbuf ^= 1;
  } else {
    __syncwarp();
  }
}

template <int S>
__device__ __forceinline__ double block_sum1(double v, double* red, int& rbuf) {
  double a[1] = {v};
  block_sum<S, 1>(a, red, rbuf);
  return a[0];
}

template <int S>
__device__ __forceinline__ double block_max(double v, double* red, int& rbuf) {
  constexpr int W = S / 32;
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) v = fmax(v, __shfl_xor_sync(FULL, v, off));
  if constexpr (W > 1) {
    double* buf = red + rbuf * (4 * W);
    if ((threadIdx.x & 31) == 0) buf[threadIdx.x >> 5] = v;
    __syncthreads();
    v = buf[0];
#pragma unroll
    for (int w = 1; w < W; ++w) v = fmax(v, buf[w]);
    rbuf ^= 1;
  } else {
    __syncwarp();
  }
  return v;
}

// int min over the CTA (first zero column).
template <int S>
__device__ __forceinline__ int block_min_int(int v, int* ired, int& ibuf) {
  constexpr int W = S / 32;
  v = static_cast<int>(__reduce_min_sync(FULL, static_cast<unsigned>(v)));
  if constexpr (W > 1) {
    int* buf = ired + ibuf * W;
    if ((threadIdx.x & 31) == 0) buf[threadIdx.x >> 5] = v;
    __syncthreads();
    v = buf[0];
#pragma unroll
    for (int w = 1; w < W; ++w) v = min(v, buf[w]);
    ibuf ^= 1;
  } else {
    __syncwarp();
  }
  return v;
}

// (value, index) max with the lowest index on ties: the first strict maximum
// in pair order (frame.hpp:141-143).
template <int S>
__device__ __forceinline__ void block_argmax(double& v, long long& idx, double* red, int& rbuf) {
  constexpr int W = S / 32;
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    const double ov = __shfl_xor_sync(FULL, v, off);
    const long long oi = __shfl_xor_sync(FULL, idx, off);
    if (ov > v || (ov == v && oi < idx)) {
      v = ov;
      idx = oi;
    }
  }
  if constexpr (W > 1) {
    double* buf = red + rbuf * (4 * W);
    if ((threadIdx.x & 31) == 0) {
      buf[threadIdx.x >> 5] = v;
      buf[W + (threadIdx.x >> 5)] = __longlong_as_double(idx);
    }
    __syncthreads();
    v = buf[0];
    idx = __double_as_longlong(buf[W]);
#pragma unroll
    for (int w = 1; w < W; ++w) {
      const double ov = buf[w];
      const long long oi = __double_as_longlong(buf[W + w]);
      if (ov > v || (ov == v && oi < idx)) {
        v = ov;
        idx = oi;
      }
    }
    rbuf ^= 1;
  } else {
    __syncwarp();
  }
}

// CAS dot of two length-n vectors in shared/global memory (lane = i mod S).
template <int S>
__device__ __forceinline__ double dot_partial(const double* a, const double* b, int n) {
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += S) acc = fma(a[i], b[i], acc);
  return acc;
}

// ------------------------------------------------------------------ pair walk
// Row-major upper-triangular pair p -> (j, k); advancing by S stays O(1).
__device__ __forceinline__ void pair_first(int N, int p, int& j, int& k) {
  j = 0;
  int row = N - 1;
  while (p >= row) {
    p -= row;
    ++j;
    --row;
  }
  k = j + 1 + p;
}
__device__ __forceinline__ void pair_advance(int N, int step, int& j, int& k) {
  k += step;
  while (k >= N && j < N - 1) {
    k = k - N + (j + 2);
    ++j;
  }
}

// ------------------------------------------------------------------ workspace
// Shared-memory carve for one CTA.  phiS is component-major (phiS[q*N + j])
// so consecutive pairs read consecutive columns without bank conflicts.
struct Smem {
  double* phiS;   // L*N
  double* alpha;  // N
  double* cw;     // n   (x_p, then w_p, then c_p = w_p / z)
  double* red;    // 2 * 4 * W
  double* scal;   // 4 scalars (F of the last evaluation, ...)
  int* ired;      // 2 * W
};

// ------------------------------------------------------------------ evaluation
// eval_objective (smoothing.hpp:82-162) at p = x + sc*dir (sc == 0: p = x),
// CTA-wide.  Returns -1 or the first zero column (then *F = +inf and gout = 0,
// the make_objective convention, solver.hpp:108-112).  gout may alias nothing
// that is read here.  Ends with a __syncthreads().
template <bool CPLX, int DMAX, bool EXACT, int S>
__device__ int eval_cta(const Prob& P, const double* __restrict__ x, const double* __restrict__ dir, double sc,
                        double delta, bool squared, const Smem& sm, int& rbuf, double* __restrict__ gout,
                        double* F_out, double* s_out, double* __restrict__ wout) {
  constexpr int C = CPLX ? 2 : 1;
  const int d = EXACT ? DMAX : P.d;
  const int N = P.N, L = P.L, n = P.n;
  const int tid = threadIdx.x;

  // ---- phase 1: column norms, normalisation (smoothing.hpp:95-102)
  int zc = INT_MAX;
  for (int j = tid; j < N; j += S) {
    double col[C * DMAX];
    double acc = 0.0;
#pragma unroll
    for (int q = 0; q < C * DMAX; ++q) {
      if (q < C * d) {
        const double xv = x[j * L + q];
        const double pv = (sc == 0.0) ? xv : __dadd_rn(xv, __dmul_rn(sc, dir[j * L + q]));
        col[q] = pv;
        acc = fma(pv, pv, acc);
      }
    }
    const double a = sqrt(acc);
    sm.alpha[j] = a;
    if (a < kZeroColumnTol) zc = min(zc, j);
#pragma unroll
    for (int q = 0; q < C * DMAX; ++q)
      if (q < C * d) sm.phiS[q * N + j] = __ddiv_rn(col[q], a);
  }
  zc = block_min_int<S>(zc, sm.ired, rbuf);  // also publishes phiS / alpha
  if (zc != INT_MAX) {
    for (int i = tid; i < P.dim; i += S) gout[i] = 0.0;
    if (F_out) *F_out = __longlong_as_double(0x7ff0000000000000LL);
    if (s_out) *s_out = 0.0;
    __syncthreads();
    return zc;
  }

  // ---- phase 2: Gram upper triangle, x_p, s = max x_p (smoothing.hpp:104-118)
  double smax = -__longlong_as_double(0x7ff0000000000000LL);
  if (tid < n) {
    int j, k;
    pair_first(N, tid, j, k);
    for (int p = tid; p < n; p += S) {
      double re = 0.0, im = 0.0;
#pragma unroll
      for (int i = 0; i < DMAX; ++i) {
        if (i < d) {
          if constexpr (CPLX) {
            const double ar = sm.phiS[(2 * i) * N + j], ai = sm.phiS[(2 * i + 1) * N + j];
            const double br = sm.phiS[(2 * i) * N + k], bi = sm.phiS[(2 * i + 1) * N + k];
            re = fma(ar, br, re);
            re = fma(ai, bi, re);
            im = fma(ar, bi, im);
            im = fma(-ai, br, im);
          } else {
            re = fma(sm.phiS[i * N + j], sm.phiS[i * N + k], re);
          }
        }
      }
      const double u = CPLX ? __dadd_rn(__dmul_rn(re, re), __dmul_rn(im, im)) : __dmul_rn(re, re);
      const double xv = squared ? u : sqrt(u);
      sm.cw[p] = xv;
      smax = fmax(smax, xv);
      pair_advance(N, S, j, k);
    }
  }
  const double s = block_max<S>(smax, sm.red, rbuf);

  // ---- phase 3: w_p = exp((x_p - s)/delta), z = CAS sum (smoothing.hpp:119-126)
  const double cut = __dmul_rn(kUnderflowCut, delta);
  double zp = 0.0;
  for (int p = tid; p < n; p += S) {
    const double diff = __dsub_rn(sm.cw[p], s);
    const double w = (diff < cut) ? 0.0 : cas_exp(__ddiv_rn(diff, delta));
    sm.cw[p] = w;
    zp = __dadd_rn(zp, w);
  }
  const double z = block_sum1<S>(zp, sm.red, rbuf);
  for (int p = tid; p < n; p += S) {
    const double w = sm.cw[p];
    const double c = (w == 0.0) ? 0.0 : __ddiv_rn(w, z);
    sm.cw[p] = c;
    if (wout) wout[p] = c;
  }
  if (F_out && tid == 0) *F_out = __dadd_rn(s, __dmul_rn(delta, cas_log(z)));
  if (s_out && tid == 0) *s_out = s;
  __syncthreads();

  // ---- phase 4: gradient (smoothing.hpp:130-160), column m per thread,
  // k ascending, pairs with c == 0 skipped; G(k,m) = conj(G(m,k)) for k > m.
  for (int m = tid; m < N; m += S) {
    double pm[C * DMAX], acc[C * DMAX];
#pragma unroll
    for (int q = 0; q < C * DMAX; ++q) {
      acc[q] = 0.0;
      pm[q] = (q < C * d) ? sm.phiS[q * N + m] : 0.0;
    }
    double t = 0.0;
    int plo = m - 1;                         // p(k, m) for k = 0: m - 1
    const int prow = m * N - m * (m + 1) / 2 - m - 1;  // p(m, k) = prow + k
    for (int k = 0; k < N; ++k) {
      if (k == m) continue;
      const bool lower = k < m;
      const int p = lower ? plo : prow + k;
      if (lower) plo += N - k - 2;
      double c = sm.cw[p];
      if (c == 0.0) continue;
      double re = 0.0, im = 0.0;
#pragma unroll
      for (int i = 0; i < DMAX; ++i) {
        if (i < d) {
          if constexpr (CPLX) {
            const double kr = sm.phiS[(2 * i) * N + k], ki = sm.phiS[(2 * i + 1) * N + k];
            const double mr = pm[2 * i], mi = pm[2 * i + 1];
            // G(a,b) with a = min(k,m), b = max(k,m) (CAS gram_entry order)
            const double ar = lower ? kr : mr, ai = lower ? ki : mi;
            const double br = lower ? mr : kr, bi = lower ? mi : ki;
            re = fma(ar, br, re);
            re = fma(ai, bi, re);
            im = fma(ar, bi, im);
            im = fma(-ai, br, im);
          } else {
            re = fma(sm.phiS[i * N + k], pm[i], re);
          }
        }
      }
      const double Gr = re;
      const double Gi = lower ? im : -im;  // G(k,m)
      const double u = CPLX ? __dadd_rn(__dmul_rn(Gr, Gr), __dmul_rn(Gi, Gi)) : __dmul_rn(Gr, Gr);
      if (!squared) c = __dmul_rn(c, __ddiv_rn(0.5, fmax(sqrt(u), 1e-150)));
      t = __dadd_rn(t, __dmul_rn(c, u));
      const double cr = __dmul_rn(c, Gr);
      const double ci = __dmul_rn(c, Gi);
#pragma unroll
      for (int i = 0; i < DMAX; ++i) {
        if (i < d) {
          if constexpr (CPLX) {
            const double pr = sm.phiS[(2 * i) * N + k], pi = sm.phiS[(2 * i + 1) * N + k];
            acc[2 * i] = fma(pr, cr, acc[2 * i]);
            acc[2 * i] = fma(-pi, ci, acc[2 * i]);
            acc[2 * i + 1] = fma(pr, ci, acc[2 * i + 1]);
            acc[2 * i + 1] = fma(pi, cr, acc[2 * i + 1]);
          } else {
            acc[i] = fma(sm.phiS[i * N + k], cr, acc[i]);
          }
        }
      }
    }
    const double am = sm.alpha[m];
#pragma unroll
    for (int q = 0; q < C * DMAX; ++q)
      if (q < C * d) gout[m * L + q] = __dmul_rn(__ddiv_rn(__dsub_rn(acc[q], __dmul_rn(t, pm[q])), am), 2.0);
  }
  __syncthreads();
  return -1;
}

// ------------------------------------------------------------------ coherence
// coherence(normalize_columns(frame)) (frame.hpp:60-69,138-145) when
// normalize, else coherence(frame).  |G| = sqrt(re*re + im*im) (CAS).
// Returns -1 or the first zero column.  Leaves phiS holding the normalised
// frame (component-major).
template <bool CPLX, int DMAX, bool EXACT, int S>
__device__ int coherence_cta(const Prob& P, const double* __restrict__ f, bool normalize, const Smem& sm, int& rbuf,
                             double* mu_out, long long* arg_out) {
  constexpr int C = CPLX ? 2 : 1;
  const int d = EXACT ? DMAX : P.d;
  const int N = P.N, L = P.L, n = P.n;
  const int tid = threadIdx.x;
  int zc = INT_MAX;
  for (int j = tid; j < N; j += S) {
    double a = 1.0;
    if (normalize) {
      double acc = 0.0;
#pragma unroll
      for (int q = 0; q < C * DMAX; ++q)
        if (q < C * d) acc = fma(f[j * L + q], f[j * L + q], acc);
      a = sqrt(acc);
      if (a < kZeroColumnTol) zc = min(zc, j);
    }
    sm.alpha[j] = a;
#pragma unroll
    for (int q = 0; q < C * DMAX; ++q)
      if (q < C * d) sm.phiS[q * N + j] = normalize ? __ddiv_rn(f[j * L + q], a) : f[j * L + q];
  }
  zc = block_min_int<S>(zc, sm.ired, rbuf);
  if (zc != INT_MAX) return zc;
  double best = 0.0;
  long long arg = LLONG_MAX;
  if (tid < n) {
    int j, k;
    pair_first(N, tid, j, k);
    for (int p = tid; p < n; p += S) {
      double re = 0.0, im = 0.0;
#pragma unroll
      for (int i = 0; i < DMAX; ++i) {
        if (i < d) {
          if constexpr (CPLX) {
            const double ar = sm.phiS[(2 * i) * N + j], ai = sm.phiS[(2 * i + 1) * N + j];
            const double br = sm.phiS[(2 * i) * N + k], bi = sm.phiS[(2 * i + 1) * N + k];
            re = fma(ar, br, re);
            re = fma(ai, bi, re);
            im = fma(ar, bi, im);
            im = fma(-ai, br, im);
          } else {
            re = fma(sm.phiS[i * N + j], sm.phiS[i * N + k], re);
          }
        }
      }
      const double m = sqrt(CPLX ? __dadd_rn(__dmul_rn(re, re), __dmul_rn(im, im)) : __dmul_rn(re, re));
      if (m > best) {
        best = m;
        arg = p;
      }
      pair_advance(N, S, j, k);
    }
  }
  block_argmax<S>(best, arg, sm.red, rbuf);
  if (arg == LLONG_MAX) arg = -1;  // mu == 0 (or N < 2): no strict maximum above 0
  *mu_out = best;
  *arg_out = arg;
  return -1;
}

}  // namespace trstmi_dev
