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

// ------------------------------------------------------------------ division
// Correctly rounded a/b from yb = RN(1/b) (Markstein's quotient correction:
// q0 = RN(a*yb), r = a - b*q0 exact by fma, RN(q0 + r*yb) == RN(a/b) when
// no intermediate under/overflows).  Bit-identical to IEEE division — the
// oracle's '/' — and checked against __ddiv_rn in tests/test_gpu_parity.py.
// Tiny numerators take the hardware division path.
__device__ __forceinline__ double div_rn(double a, double b, double yb) {
  if (fabs(a) < 0x1.0p-900) return __ddiv_rn(a, b);
  const double q0 = __dmul_rn(a, yb);
  const double r = fma(-q0, b, a);
  return fma(r, yb, q0);
}

// ------------------------------------------------------------------ workspace
// Shared-memory carve for one CTA.  phiS is component-major (phiS[q*N + j])
// so a warp reading consecutive columns is bank-conflict free.  Per pair p:
//   X[p]  : x_p (phase 2) -> w_p (phase 3) -> c_p*u_p, or -1 when c_p == 0
//   GR[p] : Re G(j,k)     -> c_p * Re G(j,k)
//   GI[p] : Im G(j,k)     -> c_p * Im G(j,k)      (complex frames only)
struct Smem {
  double* phiS;   // L*N
  double* alpha;  // N
  double* X;      // n
  double* GR;     // n
  double* GI;     // n (complex) / 0 (real)
  double* red;    // 2 * 4 * W
  double* scal;   // 4 scalars (F of the last evaluation, ...)
  int* ired;      // 2 * W
};

__host__ __device__ inline long long pair_smem_doubles(const Prob& P, bool cplx) {
  return (long long)P.n * (cplx ? 3 : 2);
}

// Gram of the upper triangle, row by row: warp w takes row pairs (a, N-2-a)
// (N pairs per row pair), lanes walk k.  Calls f(p, re, im) per pair.
template <bool CPLX, int DMAX, bool EXACT, int S, class F>
__device__ __forceinline__ void gram_rows(const Prob& P, const double* __restrict__ phiS, F&& f) {
  constexpr int W = S / 32;
  const int d = EXACT ? DMAX : P.d;
  const int N = P.N;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nrp = N / 2;
  for (int rp = warp; rp < nrp; rp += W) {
#pragma unroll 1
    for (int side = 0; side < 2; ++side) {
      const int j = side == 0 ? rp : N - 2 - rp;
      if (side == 1 && j <= rp) break;
      double a[(CPLX ? 2 : 1) * DMAX];
#pragma unroll
      for (int q = 0; q < (CPLX ? 2 : 1) * DMAX; ++q)
        a[q] = (q < (CPLX ? 2 : 1) * d) ? phiS[q * N + j] : 0.0;
      const int base = j * N - j * (j + 1) / 2 - j - 1;
      for (int k = j + 1 + lane; k < N; k += 32) {
        double re = 0.0, im = 0.0;
#pragma unroll
        for (int i = 0; i < DMAX; ++i) {
          if (i < d) {
            if constexpr (CPLX) {
              const double br = phiS[(2 * i) * N + k], bi = phiS[(2 * i + 1) * N + k];
              re = fma(a[2 * i], br, re);
              re = fma(a[2 * i + 1], bi, re);
              im = fma(a[2 * i], bi, im);
              im = fma(-a[2 * i + 1], br, im);
            } else {
              re = fma(a[i], phiS[i * N + k], re);
            }
          }
        }
        f(base + k, re, im);
      }
    }
  }
}

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
    if (a < kZeroColumnTol) {
      zc = min(zc, j);
    } else {
      const double ya = __drcp_rn(a);
#pragma unroll
      for (int q = 0; q < C * DMAX; ++q)
        if (q < C * d) sm.phiS[q * N + j] = div_rn(col[q], a, ya);
    }
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
  gram_rows<CPLX, DMAX, EXACT, S>(P, sm.phiS, [&](int p, double re, double im) {
    const double u = CPLX ? __dadd_rn(__dmul_rn(re, re), __dmul_rn(im, im)) : __dmul_rn(re, re);
    const double xv = squared ? u : sqrt(u);
    sm.X[p] = xv;
    sm.GR[p] = re;
    if constexpr (CPLX) sm.GI[p] = im;
    smax = fmax(smax, xv);
  });
  const double s = block_max<S>(smax, sm.red, rbuf);

  // ---- phase 3: w_p = exp((x_p - s)/delta), z = CAS sum (smoothing.hpp:119-126)
  const double cut = __dmul_rn(kUnderflowCut, delta);
  const double ydelta = __drcp_rn(delta);
  double zp = 0.0;
  for (int p = tid; p < n; p += S) {
    const double diff = __dsub_rn(sm.X[p], s);
    double w = 0.0;
    if (diff >= cut) w = cas_exp(div_rn(diff, delta, ydelta));
    sm.X[p] = w;
    zp = __dadd_rn(zp, w);
  }
  const double z = block_sum1<S>(zp, sm.red, rbuf);
  // ---- phase 3b: c_p = w_p / z and the pair coefficients of the gradient
  // (smoothing.hpp:125, 136-142): c*u, c*Re G, c*Im G; c == 0 flagged -1.
  const double yz = __drcp_rn(z);
  for (int p = tid; p < n; p += S) {
    const double w = sm.X[p];
    const double c = (w == 0.0) ? 0.0 : div_rn(w, z, yz);
    if (wout) wout[p] = c;
    if (c == 0.0) {
      sm.X[p] = -1.0;
    } else {
      const double gr = sm.GR[p];
      const double gi = CPLX ? sm.GI[p] : 0.0;
      const double u = CPLX ? __dadd_rn(__dmul_rn(gr, gr), __dmul_rn(gi, gi)) : __dmul_rn(gr, gr);
      double cc = c;
      if (!squared) cc = __dmul_rn(cc, __ddiv_rn(0.5, fmax(sqrt(u), 1e-150)));
      sm.X[p] = __dmul_rn(cc, u);
      sm.GR[p] = __dmul_rn(cc, gr);
      if constexpr (CPLX) sm.GI[p] = __dmul_rn(cc, gi);
    }
  }
  if (F_out && tid == 0) *F_out = __dadd_rn(s, __dmul_rn(delta, cas_log(z)));
  if (s_out && tid == 0) *s_out = s;
  __syncthreads();

  // ---- phase 4: gradient (smoothing.hpp:147-160).  One thread per output
  // component (m, i): k ascending, pairs with c == 0 skipped, G(k,m) =
  // conj(G(m,k)) for k > m.  t_m is recomputed by each of column m's threads.
  for (int unit = tid; unit < N * d; unit += S) {
    const int m = unit / d;
    const int i = unit - m * d;
    double acc_re = 0.0, acc_im = 0.0, t = 0.0;
    int plo = m - 1;                                   // p(k, m) for k = 0
    const int prow = m * N - m * (m + 1) / 2 - m - 1;  // p(m, k) = prow + k
    const double* pkr = sm.phiS + (C * i) * N;
    const double* pki = sm.phiS + (C * i + 1) * N;
    for (int k = 0; k < N; ++k) {
      if (k == m) continue;
      const bool lower = k < m;
      const int p = lower ? plo : prow + k;
      if (lower) plo += N - k - 2;
      const double cu = sm.X[p];
      if (cu < 0.0) continue;  // c == 0
      t = __dadd_rn(t, cu);
      const double cr = sm.GR[p];
      const double pr = pkr[k];
      if constexpr (CPLX) {
        const double gi = sm.GI[p];
        const double ci = lower ? gi : -gi;
        const double pi = pki[k];
        acc_re = fma(pr, cr, acc_re);
        acc_re = fma(-pi, ci, acc_re);
        acc_im = fma(pr, ci, acc_im);
        acc_im = fma(pi, cr, acc_im);
      } else {
        acc_re = fma(pr, cr, acc_re);
      }
    }
    const double am = sm.alpha[m];
    const double ya = __drcp_rn(am);
    const double pmr = sm.phiS[(C * i) * N + m];
    gout[m * L + C * i] = __dmul_rn(div_rn(__dsub_rn(acc_re, __dmul_rn(t, pmr)), am, ya), 2.0);
    if constexpr (CPLX) {
      const double pmi = sm.phiS[(C * i + 1) * N + m];
      gout[m * L + C * i + 1] = __dmul_rn(div_rn(__dsub_rn(acc_im, __dmul_rn(t, pmi)), am, ya), 2.0);
    }
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
  const int N = P.N, L = P.L;
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
    const double ya = __drcp_rn(a);
#pragma unroll
    for (int q = 0; q < C * DMAX; ++q)
      if (q < C * d) sm.phiS[q * N + j] = normalize ? div_rn(f[j * L + q], a, ya) : f[j * L + q];
  }
  zc = block_min_int<S>(zc, sm.ired, rbuf);
  if (zc != INT_MAX) return zc;
  double best = 0.0;
  long long arg = LLONG_MAX;
  gram_rows<CPLX, DMAX, EXACT, S>(P, sm.phiS, [&](int p, double re, double im) {
    const double m = sqrt(CPLX ? __dadd_rn(__dmul_rn(re, re), __dmul_rn(im, im)) : __dmul_rn(re, re));
    if (m > best || (m == best && m > 0.0 && p < arg)) {
      best = m;
      arg = p;
    }
  });
  block_argmax<S>(best, arg, sm.red, rbuf);
  if (arg == LLONG_MAX) arg = -1;  // mu == 0 (or N < 2): no strict maximum above 0
  *mu_out = best;
  *arg_out = arg;
  return -1;
}

}  // namespace trstmi_dev
