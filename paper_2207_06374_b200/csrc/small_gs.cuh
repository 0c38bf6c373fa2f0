// Stored-Gram evaluation for the small-frame path (one CTA per trial, state
// in shared memory).  Same arithmetic as eval_cta (small_path.cuh) and the
// oracle — bit-identical results — with a different data movement, chosen
// to minimise issued instructions per pair (the binding resource at small d:
// measured, profiles/README.md):
//
//   phase 2  G(j,k) of every pair -> slot (Re, Im) and x_p -> U
//   phase 3a w_p = exp((x_p - s)/delta) in place, z lane partials
//   phase 3b c_p = w_p / z, slot <- (c Re G, c Im G), U <- c u
//   phase 4  gradient: thread (chunk, column m) walks k ascending and reads
//            slot(k, m); the orientation is only the sign of c Im G, so every
//            lane of a warp runs the same branch-free k loop.
//
// Slot layout (gs_row_step, small_path.cuh): a zero slot before every row
// (the k == m term reads it and adds exactly nothing) and, when padded,
// slot(k, m) == k + m (mod 16) in both orientations (bank-conflict free).
// phi lives in a column-major copy with stride gs_col_stride(L) (16-byte
// conflict-free vector loads).
//
// Pair sweeps are lane-strided in the logical (row-major upper-triangular)
// pair order: thread l visits pairs l, l+S, l+2S, ... so the CAS z sum
// (DESIGN.md §3 item 5) accumulates inside the exp sweep.  The pair table jk
// holds phys | j << 16 | k << 24 (N <= 256, np <= 65536 in this mode).
//
// Reference: eval_objective, smoothing.hpp:82-162 (paths under
// /root/reference/proj/include/trstmi).
#pragma once
#include <type_traits>

#include "small_path.cuh"

#ifndef TRSTMI_GS_UNROLL
#define TRSTMI_GS_UNROLL 4
#endif

namespace trstmi_dev {

constexpr int kGsUnroll = TRSTMI_GS_UNROLL;  // k steps of the branch-free gradient loop in flight

// Slot tables and zeroed pair arrays.  Once per kernel; ends with a barrier.
template <int S, bool CPLX>
__device__ __forceinline__ void build_gs_tables(const Prob& P, const Smem& sm) {
  constexpr int C = CPLX ? 2 : 1;
  for (int i = threadIdx.x; i < P.np; i += S) {
    sm.U[i] = 0.0;
#pragma unroll
    for (int c = 0; c < C; ++c) sm.GRI[C * i + c] = 0.0;
  }
  if (threadIdx.x == 0) {
    sm.scal[3] = 0.0;  // mask prediction (eval_cta_gs)
    int r = 1;
    for (int a = 0; a < P.N; ++a) {
      sm.fk[a] = r - a - 1;
      if (a + 1 < P.N) r += gs_row_step(P.N, a, P.pad);
    }
  }
  __syncthreads();
  for_pairs<S>(P.N, P.n, [&](int p, int j, int k) {
    sm.jk[p] = (unsigned)(sm.fk[j] + k) | ((unsigned)j << 16) | ((unsigned)k << 24);
  });
  __syncthreads();
}

// IEEE division for the rare operands where the Markstein quotient may be
// off (|a| < 2^-900).  Not inlined so the compiler cannot if-convert it into
// every iteration of the pair sweeps.
static __device__ __noinline__ double ieee_div(double a, double b) { return __ddiv_rn(a, b); }

// LM doubles of one column from the column-major copy (16-byte loads when
// the count is even; the column stride keeps them aligned and conflict-free).
template <int LM, bool EXACT>
__device__ __forceinline__ void load_col(const double* __restrict__ src, double (&v)[LM], int len) {
  if constexpr (!EXACT) {  // runtime d: the len doubles of the column only (stride may be odd)
#pragma unroll
    for (int q = 0; q < LM; ++q) v[q] = q < len ? src[q] : 0.0;
  } else if constexpr (LM % 2 == 0) {
#pragma unroll
    for (int q = 0; q < LM; q += 2) {
      const double2 t = *reinterpret_cast<const double2*>(src + q);
      v[q] = t.x;
      v[q + 1] = t.y;
    }
  } else {
#pragma unroll
    for (int q = 0; q < LM; ++q) v[q] = src[q];
  }
}

// CAS Gram entry G(j,k), j < k, from columns in registers.
template <bool CPLX, int DMAX, bool EXACT>
__device__ __forceinline__ void gram_regs(const double* a, const double* b, int d_rt, double& re, double& im) {
  const int d = EXACT ? DMAX : d_rt;
  re = 0.0;
  im = 0.0;
#pragma unroll
  for (int i = 0; i < DMAX; ++i) {
    if (i < d) {
      if constexpr (CPLX) {
        re = fma(a[2 * i], b[2 * i], re);
        re = fma(a[2 * i + 1], b[2 * i + 1], re);
        im = fma(a[2 * i], b[2 * i + 1], im);
        im = fma(-a[2 * i + 1], b[2 * i], im);
      } else {
        re = fma(a[i], b[i], re);
      }
    }
  }
}

template <bool CPLX, int DMAX, bool EXACT, int S, bool SQ = true>
__device__ int eval_cta_gs(const Prob& P, const double* __restrict__ x, const double* __restrict__ dir, double sc,
                           double delta, const Smem& sm, int& rbuf, double* __restrict__ gout, double* F_out,
                           double* s_out, double* __restrict__ wout) {
  constexpr int C = CPLX ? 2 : 1;
  constexpr int LM = C * DMAX;
  const int d = EXACT ? DMAX : P.d;
  const int N = P.N, L = P.L, n = P.n;
  const int LP = EXACT ? gs_col_stride(LM) : gs_col_stride(L);
  const int tid = threadIdx.x;
  const int NW = mask_words(N);
  double* __restrict__ U = sm.U;
  double* __restrict__ GRI = sm.GRI;
  double* __restrict__ phiC = sm.phiC;
  const unsigned* __restrict__ tab = sm.jk;
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
        if (q < C * d) phiC[j * LP + q] = div_rn(col[q], a, ya);
    }
  }
  zc = block_min_int<S>(zc, sm.ired, rbuf);  // also publishes phiC / alpha
  PHASE_MARK(0);
  if (zc != INT_MAX) {
    for (int i = tid; i < P.dim; i += S) gout[i] = 0.0;
    if (F_out) *F_out = __longlong_as_double(0x7ff0000000000000LL);
    if (s_out) *s_out = 0.0;
    __syncthreads();
    return zc;
  }

  // ---- phase 2: Gram upper triangle (smoothing.hpp:104-118): slot <- (re,
  // im), U <- x_p; s = max x_p (fmax skips NaNs like the reference's std::max)
  double smax = -__longlong_as_double(0x7ff0000000000000LL);  // (xv > smax) skips NaNs like std::max
#pragma unroll 2
  for (int p = tid; p < n; p += S) {
    const unsigned t = tab[p];
    const int ph = (int)(t & 0xffffu);
    const int j = (int)((t >> 16) & 0xffu), k = (int)(t >> 24);
    double a[LM], b[LM];
    load_col<LM, EXACT>(phiC + j * LP, a, C * d);
    load_col<LM, EXACT>(phiC + k * LP, b, C * d);
    double re, im;
    gram_regs<CPLX, DMAX, EXACT>(a, b, d, re, im);
    const double uu = CPLX ? __dadd_rn(__dmul_rn(re, re), __dmul_rn(im, im)) : __dmul_rn(re, re);
    double xv = uu;
    if constexpr (!SQ) xv = sqrt(uu);
    U[ph] = xv;
    if constexpr (CPLX) {
      *reinterpret_cast<double2*>(GRI + 2 * ph) = make_double2(re, im);
    } else {
      GRI[ph] = re;
    }
    smax = xv > smax ? xv : smax;
  }
  if (sm.scal[3] != 0.0)
    for (int i = tid; i < N * NW; i += S) sm.mask[i] = 0u;  // published by block_max's barrier
  const double s = block_max<S>(smax, sm.red, rbuf);
  PHASE_MARK(1);

  // ---- phase 3a: w = exp((x - s)/delta) (smoothing.hpp:118-124); 0 where
  // (x - s) < cut (exactly where exp underflows to 0); z lane partials in CAS
  // order.  When the previous evaluation of this CTA was sparse, also the
  // nonzero pattern (mask words cleared in phase 2); any choice of gradient
  // loop gives the same bits, so a stale prediction only costs time.
  const bool build_mask = sm.scal[3] != 0.0;
  const double cut = __dmul_rn(kUnderflowCut, delta);
  const double ydelta = __drcp_rn(delta);
  // s >= 2^-800: every nonzero |x - s| >= 2^-854, the Markstein quotient is exact
  const bool chk = !(s >= 0x1.0p-800);
  double zl = 0.0;
  int nnz = 0, tiny = 0;
  // UW pairs (p, p + S, ...) per step inside ONE conditional region, so their
  // exp chains interleave (a branch per pair serialises them); z accumulates in
  // the CAS lane order p, p + S, ...
  auto exp_sweep = [&](auto uw_tag) {
    constexpr int UW = decltype(uw_tag)::value;
    for (int p0 = tid; p0 < n; p0 += UW * S) {
      unsigned t[UW];
      int ph[UW];
      double dd[UW], w[UW];
      bool kk[UW];
      bool any = false;
#pragma unroll
      for (int u = 0; u < UW; ++u) {
        const int p = p0 + u * S;
        t[u] = tab[p < n ? p : p0];
        ph[u] = (int)(t[u] & 0xffffu);
        dd[u] = __dsub_rn(U[ph[u]], s);
        kk[u] = p < n && !(dd[u] < cut);  // NaN propagates like cas_exp
        any |= kk[u];
        w[u] = 0.0;
      }
      if (any) {
        double y[UW];
#pragma unroll
        for (int u = 0; u < UW; ++u) y[u] = div_fast(dd[u], delta, ydelta);
        if (chk) {
#pragma unroll
          for (int u = 0; u < UW; ++u)
            if (dd[u] < 0.0 && dd[u] > -0x1.0p-900) y[u] = ieee_div(dd[u], delta);
        }
#pragma unroll
        for (int u = 0; u < UW; ++u) {
          const double e = TRSTMI_EXP_CORE(y[u]);  // |y| <= 746 (+1 ulp) where taken
          w[u] = kk[u] ? e : 0.0;
          nnz += (int)kk[u];                        // upper bound: only picks the gradient loop
          tiny |= (int)(kk[u] && y[u] < -620.0);    // w may be < 2^-900: phase 4 checks its quotients
        }
        if (build_mask) {
#pragma unroll
          for (int u = 0; u < UW; ++u) {
            if (kk[u]) {
              const int j = (int)((t[u] >> 16) & 0xffu), k = (int)(t[u] >> 24);
              atomicOr(&sm.mask[j * NW + (k >> 5)], 1u << (k & 31));
              atomicOr(&sm.mask[k * NW + (j >> 5)], 1u << (j & 31));
            }
          }
        }
      }
#pragma unroll
      for (int u = 0; u < UW; ++u) {
        if (p0 + u * S < n) {
          U[ph[u]] = w[u];
          zl = __dadd_rn(zl, w[u]);
        }
      }
    }
  };
  {
    // five pairs per step where a thread owns several (config 2: 9.7, config 3: 4.9); the 64-lane layout of
    // tiny frames (a pair or two per thread) keeps two.  One width per kernel: a run-time choice of widths
    // triples the sweep's code and slowed every phase by 15 % (profiles/r2_c2_occupancy_experiments.md)
    exp_sweep(std::integral_constant<int, (S <= 64 ? 2 : 5)>{});
  }
  double zz[3] = {zl, (double)nnz, (double)tiny};
  block_sum<S, 3>(zz, sm.red, rbuf);
  PHASE_MARK(2);
  const double z = zz[0];
  const bool sparse = zz[1] * 4.0 < (double)n;
  const bool use_mask = build_mask && sparse;
  const bool chkdiv = zz[2] != 0.0;
  const double yz = __drcp_rn(z);
  // c_p = w_p / z (smoothing.hpp:125), computed where it is used (phase 4);
  // the softmax weights are written only when asked for (batch eval API)
  if (wout) {
    for (int p = tid; p < n; p += S) {
      const double w = U[tab[p] & 0xffffu];
      wout[p] = (w > 0.0 && w < 0x1.0p-900) ? ieee_div(w, z) : div_fast(w, z, yz);
    }
  }
  PHASE_MARK(3);

  // ---- phase 4: gradient (smoothing.hpp:130-160), CAS chunked order.
  // Thread (chunk ch, column m), ascending k in [ch*N/K, (ch+1)*N/K):
  // slot(k, m) = k < m ? f(k) + m : f(m) + k (k == m: the zero slot before
  // row m), t += c u, acc += phi_k * (c G(k,m)) with c Im G(k,m) = +-slot.im.
  const int K = P.K;
  const int* __restrict__ fk = sm.fk;
  for (int unit = tid; unit < K * N; unit += S) {
    const int ch = unit / N;
    const int m = unit - ch * N;
    const int k_lo = (ch * N) / K, k_hi = ((ch + 1) * N) / K;
    const int fm = fk[m];
    double acc[LM];
#pragma unroll
    for (int q = 0; q < LM; ++q) acc[q] = 0.0;
    double tp = 0.0;
    auto term = [&](int k, int slot, bool lower, auto chk_tag) {
      const double w = U[slot];
      double re, im = 0.0;
      if constexpr (CPLX) {
        const double2 g = *reinterpret_cast<const double2*>(GRI + 2 * slot);
        re = g.x;
        im = g.y;
      } else {
        re = GRI[slot];
      }
      double c = div_fast(w, z, yz);
      if constexpr (decltype(chk_tag)::value)  // some w may be < 2^-900: its Markstein quotient is not exact
        if (w > 0.0 && w < 0x1.0p-900) c = ieee_div(w, z);
      const double uu = CPLX ? __dadd_rn(__dmul_rn(re, re), __dmul_rn(im, im)) : __dmul_rn(re, re);
      if constexpr (!SQ) c = __dmul_rn(c, __ddiv_rn(0.5, fmax(sqrt(uu), 1e-150)));
      tp = __dadd_rn(tp, __dmul_rn(c, uu));
      const double cr = __dmul_rn(c, re);
      double pk[LM];
      load_col<LM, EXACT>(phiC + k * LP, pk, C * d);
      if constexpr (CPLX) {
        // c Im G(k,m) = +-(c Im G(min, max)): flip the sign bit for k > m
        const double cim = __dmul_rn(c, im);
        const double ci = __hiloint2double(__double2hiint(cim) ^ (lower ? 0 : (int)0x80000000), __double2loint(cim));
#pragma unroll
        for (int i = 0; i < DMAX; ++i) {
          if (i < d) {
            acc[2 * i] = fma(pk[2 * i], cr, acc[2 * i]);
            acc[2 * i] = fma(-pk[2 * i + 1], ci, acc[2 * i]);
            acc[2 * i + 1] = fma(pk[2 * i], ci, acc[2 * i + 1]);
            acc[2 * i + 1] = fma(pk[2 * i + 1], cr, acc[2 * i + 1]);
          }
        }
      } else {
#pragma unroll
        for (int i = 0; i < DMAX; ++i)
          if (i < d) acc[i] = fma(pk[i], cr, acc[i]);
      }
    };
    if (use_mask) {
      const unsigned* mrow = sm.mask + m * NW;
      for (int wi = k_lo >> 5; wi <= ((k_hi - 1) >> 5); ++wi) {
        unsigned wd = mrow[wi];
        const int base = wi << 5;
        if (base < k_lo) wd &= ~0u << (k_lo - base);
        if (k_hi - base < 32) wd &= (1u << (k_hi - base)) - 1u;
        while (wd) {
          const int k = base + __ffs(wd) - 1;
          wd &= wd - 1;
          const bool lower = k < m;
          term(k, lower ? fk[k] + m : fm + k, lower, BoolTag<true>{});
        }
      }
    } else if (chkdiv) {
#pragma unroll 2
      for (int k = k_lo; k < k_hi; ++k) {
        const bool lower = k < m;
        term(k, lower ? fk[k] + m : fm + k, lower, BoolTag<true>{});
      }
    } else {  // the common case, branch-free: consecutive k steps interleave
#pragma unroll kGsUnroll
      for (int k = k_lo; k < k_hi; ++k) {
        const bool lower = k < m;
        term(k, lower ? fk[k] + m : fm + k, lower, BoolTag<false>{});
      }
    }
    double* pp = sm.part + (long long)unit * (L + 1);
#pragma unroll
    for (int q = 0; q < LM; ++q)
      if (q < C * d) pp[q] = acc[q];
    pp[L] = tp;
  }
  if (tid == S - 1) {  // off the critical path when K*N < S (this thread has no unit)
    if (F_out) *F_out = __dadd_rn(s, __dmul_rn(delta, cas_log(z)));
    if (s_out) *s_out = s;
    sm.scal[3] = sparse ? 1.0 : 0.0;  // mask prediction for the next evaluation
  }
  __syncthreads();
  PHASE_MARK(4);
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
    gout[m * L + q] = __dmul_rn(div_rn(__dsub_rn(a, __dmul_rn(t, phiC[m * LP + q])), am, __drcp_rn(am)), 2.0);
  }
  __syncthreads();
  PHASE_MARK(5);
  return -1;
}

// Mode dispatch used by the anneal and batch kernels.
template <bool CPLX, int DMAX, bool EXACT, int S, bool GS, bool SQ = true>
__device__ __forceinline__ int eval_any(const Prob& P, const double* __restrict__ x, const double* __restrict__ dir,
                                        double sc, double delta, const Smem& sm, int& rbuf, double* __restrict__ gout,
                                        double* F_out, double* s_out, double* __restrict__ wout) {
  if constexpr (GS)
    return eval_cta_gs<CPLX, DMAX, EXACT, S, SQ>(P, x, dir, sc, delta, sm, rbuf, gout, F_out, s_out, wout);
  else
    return eval_cta<CPLX, DMAX, EXACT, S, SQ>(P, x, dir, sc, delta, sm, rbuf, gout, F_out, s_out, wout);
}

template <int S, bool CPLX, bool GS>
__device__ __forceinline__ void build_tables(const Prob& P, const Smem& sm) {
  if constexpr (GS)
    build_gs_tables<S, CPLX>(P, sm);
  else
    build_pair_table<S>(P, sm.jk);
}

}  // namespace trstmi_dev
