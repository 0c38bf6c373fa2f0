// Small-frame path: one CTA owns one trial (or one batch point) and keeps the
// whole trust-region state in shared memory.  Used for BASELINE configs 1-3
// (real d=4 N=10; complex d=2 N=100; complex d=6 N=36) and any shape whose
// state fits in one SM's shared memory.
//
// Every floating-point operation follows the Canonical Arithmetic Spec
// so results are bit-identical to the CPU oracle: the file is
// compiled with -fmad=false and fuses only at explicit fma() sites; all CTA
// reductions use the CAS lane-strided / xor-butterfly order.
//
// Reference functions restated here (paths under /root/reference/proj/include/trstmi):
//   eval_cta            eval_objective           smoothing.hpp:82-162
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

#ifndef TRSTMI_EXP
#define TRSTMI_EXP cas_exp  // experiments may substitute a stub (scripts/phase_timers.sh)
#endif
#ifndef TRSTMI_EXP_CORE
#define TRSTMI_EXP_CORE cas_exp_core
#endif

#ifdef TRSTMI_PHASE_TIMERS
__device__ unsigned long long g_phase_cycles[8];
#define PHASE_MARK(i)                                                        \
  do {                                                                       \
    if (threadIdx.x == 0) {                                                  \
      const long long now_ = clock64();                                      \
      atomicAdd(&g_phase_cycles[i], (unsigned long long)(now_ - t_phase_)); \
      t_phase_ = now_;                                                       \
    }                                                                        \
  } while (0)
#define PHASE_START long long t_phase_ = clock64()
#else
#define PHASE_MARK(i) \
  do {                \
  } while (0)
#define PHASE_START
#endif

template <bool B>
struct BoolTag {
  static constexpr bool value = B;
};

struct Prob {
  int d, N, L, dim, n;  // L = doubles per column (2d complex, d real); n = pairs
  int K;                // CAS gradient k-chunks (trstmi_kchunks)
  int gs;               // 1: stored-Gram layout (small_gs.cuh), 0: Gram recomputed in the gradient
  int pad;              // gs: pair rows padded so both gradient orientations are bank-conflict free
  int np;               // gs: physical pair slots (padded rows + one zero slot)
  int dual;             // gs anneal: room for a second set of normalised columns (fused central difference, hvp_cta_gs)
};

// Stored-Gram layout (small_gs.cuh): pair (a, b), a < b, lives in slot
// rsp[a] + b - a - 1.  Every row is preceded by at least one zero slot, so
// slot rsp[m] - 1 (what the k == m term of the gradient reads) is 0.  With
// padding, f(a) = rsp[a] - a - 1 == a (mod 16), so the slot of (k, m) is
// == k + m (mod 16) in both orientations: a warp reading pair (k, m) for 16
// consecutive m hits 16 distinct 8-byte banks whether k < m (consecutive
// slots of row k) or k > m (one slot in each of 16 rows).
__host__ __device__ inline int gs_row_step(int N, int a, int pad) {
  const int len = N - a - 1;
  return pad ? len + (((1 - len) & 15) + 1) : len + 1;  // gap >= 1; step == 2 (mod 16) when padded
}
__host__ __device__ inline int gs_phys_slots(int N, int pad) {  // = rsp[N-1]
  int r = 1;
  for (int a = 0; a + 1 < N; ++a) r += gs_row_step(N, a, pad);
  return r;
}
// column stride of the column-major phi copy: conflict-free 16-byte loads
// for consecutive columns (and 8-byte loads when L is odd)
__host__ __device__ inline int gs_col_stride(int L) { return (L % 4 == 0) ? L + 2 : L; }
__host__ __device__ inline Prob make_small_prob(bool cplx, int d, int N, int K, int gs, int pad) {
  Prob P;
  P.d = d;
  P.N = N;
  P.L = (cplx ? 2 : 1) * d;
  P.dim = P.L * N;
  P.n = N * (N - 1) / 2;
  P.K = K;
  P.gs = gs;
  P.pad = gs ? pad : 0;
  P.np = gs ? gs_phys_slots(N, pad) : 0;
  P.dual = 0;
  return P;
}

// CAS gradient chunk count K for a CTA of S threads: one
// thread per (chunk, column), K = clamp(S / N, 1, 8).
__host__ __device__ inline int kchunks_for(int d, int N, int S) {
  (void)d;
  const int K = S / N;
  return K < 1 ? 1 : (K > 8 ? 8 : K);
}

// ------------------------------------------------------------------ CTA reductions
// CAS sum: lanes hold their strided partials; xor butterfly inside each warp
// (16,8,4,2,1), then the same butterfly across the S/32 warp totals (1,2,4,..)
// — a pairwise tree in warp order.  Every thread ends with the identical sum.
// Two alternating scratch buffers make one __syncthreads per reduction enough.
template <int S>
__device__ __forceinline__ double warp_tree_sum(const double* buf) {
  constexpr int W = S / 32;
  const int lane = threadIdx.x & 31;
  double t = lane < W ? buf[lane] : 0.0;
#pragma unroll
  for (int off = 1; off < W; off <<= 1) t = __dadd_rn(t, __shfl_xor_sync(FULL, t, off));
  return __shfl_sync(FULL, t, 0);
}

template <int S, int K>
__device__ __forceinline__ void block_sum(double (&v)[K], double* red, int& rbuf) {
  constexpr int W = S / 32;
  if constexpr (K == 2 && W <= 16) {
    // Two sums at once, transposed (the CTA reductions are bound by shuffle throughput): at the xor-16 level lanes
    // 0-15 keep the first value and lanes 16-31 the second, each trading the other with its partner, and the four
    // remaining levels run in both halves at once; the warp totals are combined the same way.  11 shuffles per warp
    // instead of 20, every add with the operands of the plain butterfly (own + partner's value of the same sum).
    const int lane = threadIdx.x & 31;
    const bool hi = (lane & 16) != 0;
    double t = __dadd_rn(hi ? v[1] : v[0], __shfl_xor_sync(FULL, hi ? v[0] : v[1], 16));
#pragma unroll
    for (int off = 8; off >= 1; off >>= 1) t = __dadd_rn(t, __shfl_xor_sync(FULL, t, off));
    if constexpr (W > 1) {
      double* buf = red + rbuf * (4 * W);
      if ((lane & 15) == 0) buf[(hi ? W : 0) + (threadIdx.x >> 5)] = t;
      __syncthreads();
      t = (lane & 15) < W ? buf[(hi ? W : 0) + (lane & 15)] : 0.0;
#pragma unroll
      for (int off = 1; off < W; off <<= 1) t = __dadd_rn(t, __shfl_xor_sync(FULL, t, off));
      rbuf ^= 1;
    } else {
      __syncwarp();
    }
    v[0] = __shfl_sync(FULL, t, 0);
    v[1] = __shfl_sync(FULL, t, 16);
  } else {
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
      for (int k = 0; k < K; ++k) v[k] = warp_tree_sum<S>(buf + k * W);
      rbuf ^= 1;
    } else {
      __syncwarp();
    }
  }
}

template <int S>
__device__ __forceinline__ double block_sum1(double v, double* red, int& rbuf) {
  double a[1] = {v};
  block_sum<S, 1>(a, red, rbuf);
  return a[0];
}

// WS: warps the scratch buffers are strided for (the CAS lane count / 32 when
// the CTA has fewer threads than CAS lanes, small_rt.cuh) — every reduction
// of a kernel must use the same stride, or the two alternating buffers overlap.
// Max of doubles that are never NaN and, when negative, only -inf (the x_p of an evaluation: squared magnitudes, or
// the -inf a thread without pairs starts from): as signed 64-bit integers they order like the doubles, so the warp
// maximum is two integer REDUX steps (high words, then the low words of the lanes that hold the highest high word)
// instead of a five-step shuffle butterfly.  Order-free, hence bit-identical to any fmax tree.
__device__ __forceinline__ double warp_max_nonneg(double v) {
  const int hi = __double2hiint(v);
  const int mh = __reduce_max_sync(FULL, hi);
  const unsigned lo = hi == mh ? (unsigned)__double2loint(v) : 0u;
  const unsigned ml = __reduce_max_sync(FULL, lo);
  return __hiloint2double(mh, (int)ml);
}

template <int S, int WS = S / 32>
__device__ __forceinline__ double block_max(double v, double* red, int& rbuf) {
  constexpr int W = S / 32;
  v = warp_max_nonneg(v);
  if constexpr (W > 1) {
    double* buf = red + rbuf * (4 * WS);
    if ((threadIdx.x & 31) == 0) buf[threadIdx.x >> 5] = v;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    v = warp_max_nonneg(lane < W ? buf[lane] : buf[0]);
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
    const int lane = threadIdx.x & 31;
    v = static_cast<int>(__reduce_min_sync(FULL, static_cast<unsigned>(lane < W ? buf[lane] : buf[0])));
    ibuf ^= 1;
  } else {
    __syncwarp();
  }
  return v;
}

// (value, index) max with the lowest index on ties: the first strict maximum
// in pair order (frame.hpp:141-143).
template <int S, int WS = S / 32>
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
    double* buf = red + rbuf * (4 * WS);
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
// Row-major upper-triangular pair p = rowstart(j) + (k - j - 1).
__device__ __forceinline__ int rowstart(int N, int j) { return j * N - j * (j + 1) / 2; }

__device__ __forceinline__ void pair_of(int N, int p, int& j, int& k) {
  const double b = 2.0 * N - 1.0;
  int jj = (int)floor(0.5 * (b - sqrt(fmax(b * b - 8.0 * p, 0.0))));
  jj = max(0, min(jj, N - 2));
  while (jj < N - 2 && rowstart(N, jj + 1) <= p) ++jj;
  while (jj > 0 && rowstart(N, jj) > p) --jj;
  j = jj;
  k = p - rowstart(N, jj) + jj + 1;
}

// Warp-contiguous walk over all pairs: warp w owns the contiguous range
// [w*chunk, (w+1)*chunk), lanes step by 32 (consecutive k within a row, so
// the k-column reads are bank-conflict free).  f(p, j, k).
template <int S, class F>
__device__ __forceinline__ void for_pairs(int N, int n, F&& f) {
  constexpr int W = S / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int chunk = (n + W - 1) / W;
  const int pend = min(n, (warp + 1) * chunk);
  int p = warp * chunk + lane;
  if (p >= pend) return;
  int j, k;
  pair_of(N, p, j, k);
  for (; p < pend; p += 32) {
    f(p, j, k);
    k += 32;
    while (k >= N && j < N - 2) {
      k = k - N + j + 2;
      ++j;
    }
  }
}

// Same walk, four pairs per step (p, p+32, p+64, p+96) so the four
// independent dependency chains interleave.  f(p[4], j[4], k[4], valid[4]).
__device__ __forceinline__ void adv32(int N, int& j, int& k) {
  k += 32;
  while (k >= N && j < N - 2) {
    k = k - N + j + 2;
    ++j;
  }
}
template <int S, class F>
__device__ __forceinline__ void for_pairs4(int N, int n, F&& f) {
  constexpr int W = S / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int chunk = (n + W - 1) / W;
  const int pend = min(n, (warp + 1) * chunk);
  int p0 = warp * chunk + lane;
  if (p0 >= pend) return;
  int j0, k0;
  pair_of(N, p0, j0, k0);
  for (; p0 < pend; p0 += 128) {
    int p[4], j[4], k[4];
    bool v[4];
    p[0] = p0;
    j[0] = j0;
    k[0] = k0;
#pragma unroll
    for (int u = 1; u < 4; ++u) {
      j[u] = j[u - 1];
      k[u] = k[u - 1];
      adv32(N, j[u], k[u]);
      p[u] = p[u - 1] + 32;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      v[u] = p[u] < pend;
      if (!v[u]) {  // keep indices in range; results are discarded
        p[u] = p[0];
        j[u] = j[0];
        k[u] = k[0];
      }
    }
    f(p, j, k, v);
    j0 = j[3];
    k0 = k[3];
    adv32(N, j0, k0);
  }
}

// Table-driven walk (the (j,k) of every pair is precomputed once per kernel
// in Smem::jk as j | k << 16): warp-contiguous ranges, lanes step by 32,
// four pairs per step.  f(p[4], j[4], k[4], valid[4]).
template <int S, bool NEED_JK, bool GS = false, class F>
__device__ __forceinline__ void pairs4(int n, const unsigned* __restrict__ jk, F&& f) {
  constexpr int W = S / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int chunk = (n + W - 1) / W;
  const int pbeg = warp * chunk;
  const int pend = min(n, pbeg + chunk);
  for (int p0 = pbeg + lane; p0 < pend; p0 += 128) {
    int p[4], j[4], k[4];
    bool v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      v[u] = p0 + 32 * u < pend;
      p[u] = v[u] ? p0 + 32 * u : p0;
      if constexpr (NEED_JK) {
        const unsigned t = jk[p[u]];
        if constexpr (GS) {  // stored-Gram table: phys | j << 16 | k << 24
          j[u] = (int)((t >> 16) & 0xffu);
          k[u] = (int)(t >> 24);
        } else {
          j[u] = (int)(t & 0xffffu);
          k[u] = (int)(t >> 16);
        }
      } else {
        j[u] = k[u] = 0;
      }
    }
    f(p, j, k, v);
  }
}

// CAS Gram entry G(j,k), j<k, from component-major phiS.
template <bool CPLX, int DMAX, bool EXACT>
__device__ __forceinline__ void gram_jk(const double* __restrict__ phiS, int N, int d_rt, int j, int k, double& re,
                                        double& im) {
  const int d = EXACT ? DMAX : d_rt;
  re = 0.0;
  im = 0.0;
#pragma unroll
  for (int i = 0; i < DMAX; ++i) {
    if (i < d) {
      if constexpr (CPLX) {
        const double ar = phiS[(2 * i) * N + j], ai = phiS[(2 * i + 1) * N + j];
        const double br = phiS[(2 * i) * N + k], bi = phiS[(2 * i + 1) * N + k];
        re = fma(ar, br, re);
        re = fma(ai, bi, re);
        im = fma(ar, bi, im);
        im = fma(-ai, br, im);
      } else {
        re = fma(phiS[i * N + j], phiS[i * N + k], re);
      }
    }
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
// Branch-free Markstein quotient, valid when |a| >= 2^-900 or a == 0; the
// caller fixes up the (rare) tiny numerators with div_needs_ieee().
__device__ __forceinline__ double div_fast(double a, double b, double yb) {
  const double q0 = __dmul_rn(a, yb);
  const double r = fma(-q0, b, a);
  return fma(r, yb, q0);
}
__device__ __forceinline__ bool div_needs_ieee(double a) { return a != 0.0 && fabs(a) < 0x1.0p-900; }

// ------------------------------------------------------------------ workspace
// Shared-memory carve for one CTA.  phiS is component-major (phiS[q*N + j])
// so a warp reading consecutive columns is bank-conflict free; a warp whose
// lanes all read the same column gets a broadcast.
//   U[p]  : x_p (phase 2) -> w_p (phase 3a) -> c_p = w_p / z (phase 3b)
//   part  : K x N x (L+1) chunk partials of the gradient GEMM and of t
//   mask  : N x NW words, bit k of column m set iff c(m,k) != 0 (sparse only)
struct Smem {
  double* phiS;      // L*N
  double* alpha;     // N
  double* alpha2;    // dual: N, norms of the second point (its columns live in phiS, unused by the gs evaluation)
  double* U;         // n (gs: np)
  double* GRI;       // gs: np x C, (Re G, Im G) -> (c Re G, c Im G) per pair slot
  double* phiC;      // gs: N x LP column-major copy of phi (LP = gs_col_stride(L))
  int* fk;           // gs: N, f(a) = rsp[a] - a - 1 (slot of (k, m) = k < m ? f(k) + m : f(m) + k)
  double* part;      // K*N*(L+1)
  unsigned* mask;    // N*NW
  unsigned* jk;      // n: pair p -> j | k << 16
  double* red;       // 2 * 4 * W
  double* scal;      // 4 scalars (F of the last evaluation, ...)
  int* ired;         // 2 * W
  // gs Gram sweep, per thread (build_gs_tables): this thread's column k and its rows [gj0, gj1) (gj1 <= k); gk < 0: none
  int gk, gj0, gj1;
};

__host__ __device__ inline int mask_words(int N) { return (N + 31) / 32; }
__host__ __device__ inline long long pair_smem_doubles(const Prob& P, bool cplx) {
  const long long common = (long long)P.K * P.N * (P.L + 1) + ((long long)P.N * mask_words(P.N) + 1) / 2 +
                           ((long long)P.n + 1) / 2;
  if (!P.gs) return (long long)P.n + common;
  return (long long)P.np * (cplx ? 3 : 2) + (long long)gs_col_stride(P.L) * P.N + (P.N + 1) / 2 + 2 + common;
}

// Fills Smem::jk (once per kernel; ends with a barrier).
template <int S>
__device__ __forceinline__ void build_pair_table(const Prob& P, unsigned* jk) {
  for_pairs<S>(P.N, P.n, [&](int p, int j, int k) { jk[p] = (unsigned)j | ((unsigned)k << 16); });
  __syncthreads();
}

// ------------------------------------------------------------------ evaluation
// eval_objective (smoothing.hpp:82-162) at p = x + sc*dir (sc == 0: p = x),
// CTA-wide.  Returns -1 or the first zero column (then *F = +inf and gout = 0,
// the make_objective convention, solver.hpp:108-112).  gout may alias nothing
// that is read here.  Ends with a __syncthreads().
//
// Data movement: the only per-pair value kept in shared memory is one double
// (x -> w -> c); the gradient recomputes G(k,m) in registers from phi_m
// (registers) and phi_k (a shared-memory broadcast: every lane of a warp is at
// the same k), so the FP64 pipe, not shared-memory bandwidth, sets the pace.
// Pairs with c == 0 contribute exactly nothing (accumulators start at +0 and
// never become -0), so skipping them is bit-identical to including them.
template <bool CPLX, int DMAX, bool EXACT, int S, bool SQ = true>
__device__ int eval_cta(const Prob& P, const double* __restrict__ x, const double* __restrict__ dir, double sc,
                        double delta, const Smem& sm, int& rbuf, double* __restrict__ gout, double* F_out,
                        double* s_out, double* __restrict__ wout) {
  constexpr int C = CPLX ? 2 : 1;
  constexpr int LM = C * DMAX;
  const int d = EXACT ? DMAX : P.d;
  const int N = P.N, L = P.L, n = P.n;
  const int tid = threadIdx.x;
  const int NW = mask_words(N);
  PHASE_START;

  // ---- phase 1: column norms, normalisation (smoothing.hpp:95-102)
  int zc = INT_MAX;
  for (int j = tid; j < N; j += S) {
    double col[LM];
    double acc = 0.0;
#pragma unroll
    for (int q = 0; q < LM; ++q) {
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
      for (int q = 0; q < LM; ++q)
        if (q < C * d) sm.phiS[q * N + j] = div_rn(col[q], a, ya);
    }
  }
  zc = block_min_int<S>(zc, sm.ired, rbuf);  // also publishes phiS / alpha
  PHASE_MARK(0);
  if (zc != INT_MAX) {
    for (int i = tid; i < P.dim; i += S) gout[i] = 0.0;
    if (F_out) *F_out = __longlong_as_double(0x7ff0000000000000LL);
    if (s_out) *s_out = 0.0;
    __syncthreads();
    return zc;
  }

  // ---- phase 2: Gram upper triangle, x_p, s = max x_p (smoothing.hpp:104-118)
  double smax = -__longlong_as_double(0x7ff0000000000000LL);
  pairs4<S, true>(n, sm.jk, [&](const int* p, const int* j, const int* k, const bool* v) {
    double re[4], im[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) gram_jk<CPLX, DMAX, EXACT>(sm.phiS, N, d, j[u], k[u], re[u], im[u]);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double uu = CPLX ? __dadd_rn(__dmul_rn(re[u], re[u]), __dmul_rn(im[u], im[u])) : __dmul_rn(re[u], re[u]);
      double xv = uu;
      if constexpr (!SQ) xv = sqrt(uu);
      if (v[u]) {
        sm.U[p[u]] = xv;
        smax = xv > smax ? xv : smax;
      }
    }
  });
  const double s = block_max<S>(smax, sm.red, rbuf);
  PHASE_MARK(1);

  // ---- phase 3a: w_p = exp((x_p - s)/delta) (smoothing.hpp:119-124), any
  // order; count the nonzero weights.  Clears the sparse-pattern mask.
  for (int i = tid; i < N * NW; i += S) sm.mask[i] = 0u;
  const double cut = __dmul_rn(kUnderflowCut, delta);
  const double ydelta = __drcp_rn(delta);
  double nnz = 0.0;
  pairs4<S, false>(n, sm.jk, [&](const int* p, const int*, const int*, const bool* v) {
    double diff[4], w[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) diff[u] = __dsub_rn(sm.U[p[u]], s);
    const bool any = !((diff[0] < cut) & (diff[1] < cut) & (diff[2] < cut) & (diff[3] < cut));
    if (any) {
      double y[4];
      bool fix = false;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        y[u] = div_fast(diff[u], delta, ydelta);
        fix |= div_needs_ieee(diff[u]);
      }
      if (fix) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (div_needs_ieee(diff[u])) y[u] = __ddiv_rn(diff[u], delta);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) w[u] = (diff[u] < cut) ? 0.0 : TRSTMI_EXP(y[u]);
    } else {
#pragma unroll
      for (int u = 0; u < 4; ++u) w[u] = 0.0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (v[u]) {
        sm.U[p[u]] = w[u];
        if (w[u] != 0.0) nnz += 1.0;
      }
    }
  });
  __syncthreads();
  PHASE_MARK(2);
  // ---- phase 3z: z = CAS sum of w in lane-strided pair order (smoothing.hpp:121-124)
  double zz[2] = {0.0, nnz};
  for (int p = tid; p < n; p += S) zz[0] = __dadd_rn(zz[0], sm.U[p]);
  block_sum<S, 2>(zz, sm.red, rbuf);
  PHASE_MARK(3);
  const double z = zz[0];
  const bool sparse = zz[1] * 4.0 < (double)n;
  // ---- phase 3b: c_p = w_p / z (smoothing.hpp:125); sparse pattern mask
  const double yz = __drcp_rn(z);
  auto coef = [&](const int* p, const int* j, const int* k, const bool* v) {
    double w[4], cq[4];
    bool fix = false;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      w[u] = sm.U[p[u]];
      cq[u] = div_fast(w[u], z, yz);
      fix |= div_needs_ieee(w[u]);
    }
    if (fix) {
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (div_needs_ieee(w[u])) cq[u] = __ddiv_rn(w[u], z);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double c = cq[u];
      if (v[u]) {
        if (wout) wout[p[u]] = c;
        if (w[u] != 0.0) sm.U[p[u]] = c;
        if (sparse && c != 0.0) {
          atomicOr(&sm.mask[j[u] * NW + (k[u] >> 5)], 1u << (k[u] & 31));
          atomicOr(&sm.mask[k[u] * NW + (j[u] >> 5)], 1u << (j[u] & 31));
        }
      }
    }
  };
  if (sparse) pairs4<S, true>(n, sm.jk, coef);
  else pairs4<S, false>(n, sm.jk, coef);
  if (F_out && tid == 0) *F_out = __dadd_rn(s, __dmul_rn(delta, cas_log(z)));
  if (s_out && tid == 0) *s_out = s;
  __syncthreads();
  PHASE_MARK(4);

  // ---- phase 4: gradient (smoothing.hpp:130-160), CAS chunked order.
  // Thread (chunk ch, column m): ascending k in [ch*N/K, (ch+1)*N/K):
  // G(k,m) recomputed (CAS gram order on (min, max), conjugated for k > m),
  // t += c*u, acc += phi_k * (c G).  Partials go to part[], then each output
  // adds its K partials left to right.
  const int K = P.K;
  for (int unit = tid; unit < K * N; unit += S) {
    const int ch = unit / N;
    const int m = unit - ch * N;
    const int k_lo = (ch * N) / K, k_hi = ((ch + 1) * N) / K;
    double pm[LM], acc[LM];
#pragma unroll
    for (int q = 0; q < LM; ++q) {
      pm[q] = (q < C * d) ? sm.phiS[q * N + m] : 0.0;
      acc[q] = 0.0;
    }
    double tp = 0.0;
    auto term = [&](int k, double c, auto lower_tag) {
      constexpr bool lower = decltype(lower_tag)::value;
      double pk[LM];
#pragma unroll
      for (int q = 0; q < LM; ++q) pk[q] = (q < C * d) ? sm.phiS[q * N + k] : 0.0;
      double re = 0.0, im = 0.0;
#pragma unroll
      for (int i = 0; i < DMAX; ++i) {
        if (i < d) {
          if constexpr (CPLX) {
            const double ar = lower ? pk[2 * i] : pm[2 * i], ai = lower ? pk[2 * i + 1] : pm[2 * i + 1];
            const double br = lower ? pm[2 * i] : pk[2 * i], bi = lower ? pm[2 * i + 1] : pk[2 * i + 1];
            re = fma(ar, br, re);
            re = fma(ai, bi, re);
            im = fma(ar, bi, im);
            im = fma(-ai, br, im);
          } else {
            re = fma(pk[i], pm[i], re);
          }
        }
      }
      const double gr = re;
      const double gi = lower ? im : -im;  // G(k,m)
      const double uu = CPLX ? __dadd_rn(__dmul_rn(gr, gr), __dmul_rn(gi, gi)) : __dmul_rn(gr, gr);
      double cc = c;
      if constexpr (!SQ) cc = __dmul_rn(cc, __ddiv_rn(0.5, fmax(sqrt(uu), 1e-150)));
      tp = __dadd_rn(tp, __dmul_rn(cc, uu));
      const double cr = __dmul_rn(cc, gr);
      const double ci = __dmul_rn(cc, gi);
#pragma unroll
      for (int i = 0; i < DMAX; ++i) {
        if (i < d) {
          if constexpr (CPLX) {
            acc[2 * i] = fma(pk[2 * i], cr, acc[2 * i]);
            acc[2 * i] = fma(-pk[2 * i + 1], ci, acc[2 * i]);
            acc[2 * i + 1] = fma(pk[2 * i], ci, acc[2 * i + 1]);
            acc[2 * i + 1] = fma(pk[2 * i + 1], cr, acc[2 * i + 1]);
          } else {
            acc[i] = fma(pk[i], cr, acc[i]);
          }
        }
      }
    };
    if (sparse) {
      const unsigned* mrow = sm.mask + m * NW;
      for (int wi = k_lo >> 5; wi <= ((k_hi - 1) >> 5); ++wi) {
        unsigned wd = mrow[wi];
        const int base = wi << 5;
        if (base < k_lo) wd &= ~0u << (k_lo - base);
        if (k_hi - base < 32) wd &= (1u << (k_hi - base)) - 1u;
        while (wd) {
          const int k = base + __ffs(wd) - 1;
          wd &= wd - 1;
          if (k < m) term(k, sm.U[rowstart(N, k) + (m - k - 1)], BoolTag<true>{});
          else term(k, sm.U[rowstart(N, m) + (k - m - 1)], BoolTag<false>{});
        }
      }
    } else {
      const int kA = min(k_hi, m);
      if (k_lo < kA) {
        // dense: branch-free (a c == 0 term adds exactly nothing)
        int plo = rowstart(N, k_lo) + (m - k_lo - 1);
#pragma unroll 2
        for (int k = k_lo; k < kA; ++k) {
          const double c = sm.U[plo];
          plo += N - k - 2;
          term(k, c, BoolTag<true>{});
        }
      }
      const int kB = max(k_lo, m + 1);
      const int prow = rowstart(N, m) - m - 1;  // p(m, k) = prow + k
#pragma unroll 2
      for (int k = kB; k < k_hi; ++k) term(k, sm.U[prow + k], BoolTag<false>{});
    }
    double* pp = sm.part + (long long)unit * (L + 1);
#pragma unroll
    for (int q = 0; q < LM; ++q)
      if (q < C * d) pp[q] = acc[q];
    pp[L] = tp;
  }
  __syncthreads();
  for (int mq = tid; mq < N * L; mq += S) {
    const int m = mq / L;
    const int q = mq - m * L;
    double a = 0.0, t = 0.0;
    for (int ch = 0; ch < K; ++ch) {
      const double* pp = sm.part + (long long)(ch * N + m) * (L + 1);
      a = ch == 0 ? pp[q] : __dadd_rn(a, pp[q]);
      t = ch == 0 ? pp[L] : __dadd_rn(t, pp[L]);
    }
    const double am = sm.alpha[m];
    gout[m * L + q] =
        __dmul_rn(div_rn(__dsub_rn(a, __dmul_rn(t, sm.phiS[q * N + m])), am, __drcp_rn(am)), 2.0);
  }
  __syncthreads();
  PHASE_MARK(5);
  return -1;
}

// ------------------------------------------------------------------ coherence
// coherence(normalize_columns(frame)) (frame.hpp:60-69,138-145) when
// normalize, else coherence(frame).  |G| = sqrt(re*re + im*im) (CAS).
// Returns -1 or the first zero column.  Leaves phiS holding the normalised
// frame (component-major).
template <bool CPLX, int DMAX, bool EXACT, int S, bool GS = false>
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
  pairs4<S, true, GS>(P.n, sm.jk, [&](const int* p, const int* j, const int* k, const bool* v) {
    double re[4], im[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) gram_jk<CPLX, DMAX, EXACT>(sm.phiS, N, d, j[u], k[u], re[u], im[u]);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double m = cas_hypot(re[u], CPLX ? im[u] : 0.0);  // std::abs = hypot (frame.hpp:87)
      if (v[u] && m > best) {  // pairs ascend within a thread: first strict maximum
        best = m;
        arg = p[u];
      }
    }
  });
  block_argmax<S>(best, arg, sm.red, rbuf);
  if (arg == LLONG_MAX) arg = -1;  // mu == 0 (or N < 2): no strict maximum above 0
  *mu_out = best;
  *arg_out = arg;
  return -1;
}

}  // namespace trstmi_dev
