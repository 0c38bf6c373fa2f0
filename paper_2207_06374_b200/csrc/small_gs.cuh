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
#ifndef TRSTMI_GS_GRAM_COLS
#define TRSTMI_GS_GRAM_COLS 1  // Gram sweep by (row chunk, column) units; 0: lane-strided pair-table sweep
#endif

namespace trstmi_dev {

constexpr int kGsUnroll = TRSTMI_GS_UNROLL;  // k steps of the branch-free gradient loop in flight
#ifndef TRSTMI_GS_EXP_WIDE
#define TRSTMI_GS_EXP_WIDE 5
#endif
constexpr int kGsExpWide = TRSTMI_GS_EXP_WIDE;  // pairs per step of the exp sweep (S > 64)
#ifndef TRSTMI_GS_GRAM_UNROLL
#define TRSTMI_GS_GRAM_UNROLL 1
#endif
constexpr int kGsGramUnroll = TRSTMI_GS_GRAM_UNROLL;  // Gram sweep unroll: 1 measured best in the anneal kernel (registers, code size; profiles/r2_c2_session5.md)
#ifndef TRSTMI_GS_DUAL_ELEMS
#define TRSTMI_GS_DUAL_ELEMS 2
#endif
constexpr int kGsDualElems = TRSTMI_GS_DUAL_ELEMS;              // gradient elements per thread the fused central difference keeps in registers

// Slot tables and zeroed pair arrays.  Once per kernel; ends with a barrier.
template <int S, bool CPLX>
__device__ __forceinline__ void build_gs_tables(const Prob& P, Smem& sm) {
  constexpr int C = CPLX ? 2 : 1;
  {
    // Gram sweep units (gs_gram_sweep): rows in chunks of c, chunk ch = rows [c ch, c ch + c) against every column
    // k > c ch; c is the smallest length whose unit count fits the CTA, so each thread owns at most one unit.
    // (Two columns per thread — half the row loads per pair — measured slower: profiles/r2_c2_session5.md.)
    const int R = P.N - 1;
    int c = 1;
    for (;; ++c) {
      const int nch = (R + c - 1) / c;
      if (nch * R - c * (nch * (nch - 1) / 2) <= S) break;
    }
    int u = threadIdx.x, ch = 0;
    while (c * ch < R && u >= R - c * ch) {
      u -= R - c * ch;
      ++ch;
    }
    if (c * ch < R) {
      sm.gk = c * ch + 1 + u;
      sm.gj0 = c * ch;
      sm.gj1 = min(c * ch + c, sm.gk);
    } else {
      sm.gk = -1;
      sm.gj0 = sm.gj1 = 0;
    }
  }
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

// ---- the phases of one evaluation, shared by eval_cta_gs and hvp_cta_gs.  phiC / alpha are parameters so the two
// points of a central difference can keep their normalised columns side by side.

// phase 1, one column: alpha_j = ||p_j||, phi_j = p_j / alpha_j (smoothing.hpp:95-102), p = x + sc dir.
// Returns true when the column is (numerically) zero; phi_j is then left unwritten.
template <bool CPLX, int DMAX, bool EXACT>
__device__ __forceinline__ bool gs_norm_col(const Prob& P, const double* __restrict__ x, const double* __restrict__ dir,
                                            double sc, int j, double* __restrict__ phiC, double* __restrict__ alpha,
                                            int LP) {
  constexpr int C = CPLX ? 2 : 1;
  constexpr int LM = C * DMAX;
  const int d = EXACT ? DMAX : P.d;
  const int L = P.L;
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
  alpha[j] = a;
  if (a < kZeroColumnTol) return true;
  const double ya = __drcp_rn(a);
#pragma unroll
  for (int q = 0; q < LM; ++q)
    if (q < C * d) phiC[j * LP + q] = div_rn(col[q], a, ya);
  return false;
}

// phase 2: Gram upper triangle (smoothing.hpp:104-118): slot <- (re, im), U <- x_p; returns the thread's max x_p
// ((xv > smax) skips NaNs like the reference's std::max).
template <bool CPLX, int DMAX, bool EXACT, int S, bool SQ>
__device__ __forceinline__ double gs_gram_sweep(const Prob& P, const Smem& sm, const double* __restrict__ phiC, int LP) {
  constexpr int C = CPLX ? 2 : 1;
  constexpr int LM = C * DMAX;
  const int d = EXACT ? DMAX : P.d;
  const int n = P.n;
  double* __restrict__ U = sm.U;
  double* __restrict__ GRI = sm.GRI;
  const unsigned* __restrict__ tab = sm.jk;
  double smax = -__longlong_as_double(0x7ff0000000000000LL);
#if TRSTMI_GS_GRAM_COLS
  // Thread = (row chunk, column k): column k stays in registers, the rows j of the chunk arrive as warp-wide
  // loads of one address (every lane of a chunk is at the same j), and the stores of a warp go to consecutive
  // slots f(j) + k — two thirds of the shared-memory traffic of a pair-table sweep, and no table.
  if (sm.gk >= 0) {
    const int k = sm.gk;
    const int* __restrict__ fk = sm.fk;
    double b[LM];
    load_col<LM, EXACT>(phiC + k * LP, b, C * d);
#pragma unroll kGsGramUnroll
    for (int j = sm.gj0; j < sm.gj1; ++j) {
      double a[LM];
      load_col<LM, EXACT>(phiC + j * LP, a, C * d);
      double re, im;
      gram_regs<CPLX, DMAX, EXACT>(a, b, d, re, im);
      const double uu = CPLX ? __dadd_rn(__dmul_rn(re, re), __dmul_rn(im, im)) : __dmul_rn(re, re);
      double xv = uu;
      if constexpr (!SQ) xv = sqrt(uu);
      const int ph = fk[j] + k;
      U[ph] = xv;
      if constexpr (CPLX) {
        *reinterpret_cast<double2*>(GRI + 2 * ph) = make_double2(re, im);
      } else {
        GRI[ph] = re;
      }
      smax = xv > smax ? xv : smax;
    }
  }
  (void)n;
  (void)tab;
#else
#pragma unroll 2
  for (int p = threadIdx.x; p < n; p += S) {
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
#endif
  if (sm.scal[3] != 0.0)
    for (int i = threadIdx.x; i < P.N * mask_words(P.N); i += S) sm.mask[i] = 0u;  // published by block_max's barrier
  return smax;
}

struct GsZ {
  double z, yz;
  bool sparse, use_mask, chkdiv;
};

// phase 3a: w = exp((x - s)/delta) (smoothing.hpp:118-124); 0 where (x - s) < cut (exactly where exp underflows
// to 0); z lane partials in CAS order, then the CTA sum.  When the previous evaluation of this CTA was sparse, also
// the nonzero pattern (mask words cleared in phase 2); any choice of gradient loop gives the same bits, so a stale
// prediction only costs time.
template <int S>
__device__ __forceinline__ GsZ gs_exp_z(const Prob& P, const Smem& sm, double s, double delta, int& rbuf) {
  const int n = P.n;
  const int tid = threadIdx.x;
  const int NW = mask_words(P.N);
  double* __restrict__ U = sm.U;
  const unsigned* __restrict__ tab = sm.jk;
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
    exp_sweep(std::integral_constant<int, (S <= 64 ? 2 : kGsExpWide)>{});
  }
  // one CTA reduction: z by the CAS tree; the two integer flags ride on the same barrier through REDUX (order-free)
  int flags = __reduce_add_sync(FULL, nnz) | (__reduce_or_sync(FULL, (unsigned)(tiny != 0)) ? (1 << 24) : 0);
  {
    constexpr int W = S / 32;
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) zl = __dadd_rn(zl, __shfl_xor_sync(FULL, zl, off));
    if constexpr (W > 1) {
      double* buf = sm.red + rbuf * (4 * W);
      int* ibuf = sm.ired + rbuf * W;
      if ((tid & 31) == 0) {
        buf[tid >> 5] = zl;
        ibuf[tid >> 5] = flags;
      }
      __syncthreads();
      zl = warp_tree_sum<S>(buf);
      const int f = (tid & 31) < W ? ibuf[tid & 31] : 0;
      flags = __reduce_add_sync(FULL, f & 0xffffff) | (__reduce_or_sync(FULL, (unsigned)(f >> 24)) ? (1 << 24) : 0);
      rbuf ^= 1;
    } else {
      __syncwarp();
    }
  }
  GsZ r;
  r.z = zl;
  r.sparse = (long long)(flags & 0xffffff) * 4 < (long long)n;
  r.use_mask = build_mask && r.sparse;
  r.chkdiv = (flags >> 24) != 0;
  r.yz = __drcp_rn(r.z);
  return r;
}

// phase 4: gradient (smoothing.hpp:130-160), CAS chunked order.
// Thread (chunk ch, column m), ascending k in [ch*N/K, (ch+1)*N/K):
// slot(k, m) = k < m ? f(k) + m : f(m) + k (k == m: the zero slot before
// row m), t += c u, acc += phi_k * (c G(k,m)) with c Im G(k,m) = +-slot.im;
// c_p = w_p / z (smoothing.hpp:125) is computed where it is used.  Chunk partials -> sm.part (no barrier here).
template <bool CPLX, int DMAX, bool EXACT, int S, bool SQ>
__device__ __forceinline__ void gs_grad_loop(const Prob& P, const Smem& sm, const double* __restrict__ phiC, int LP,
                                             const GsZ& Z) {
  constexpr int C = CPLX ? 2 : 1;
  constexpr int LM = C * DMAX;
  const int d = EXACT ? DMAX : P.d;
  const int N = P.N, L = P.L;
  const int NW = mask_words(N);
  const double* __restrict__ U = sm.U;
  const double* __restrict__ GRI = sm.GRI;
  const double z = Z.z, yz = Z.yz;
  const int K = P.K;
  const int* __restrict__ fk = sm.fk;
  for (int unit = threadIdx.x; unit < K * N; unit += S) {
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
    if (Z.use_mask) {
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
    } else if (Z.chkdiv) {
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
}

// phase 5, one output element mq = m L + q: chunk partials left to right, ((acc - t phi)/alpha) * 2.
__device__ __forceinline__ double gs_combine_elem(const Prob& P, const Smem& sm, const double* __restrict__ phiC,
                                                  const double* __restrict__ alpha, int LP, int mq) {
  const int N = P.N, L = P.L, K = P.K;
  const int m = mq / L;
  const int q = mq - m * L;
  double a = 0.0, t = 0.0;
  for (int ch = 0; ch < K; ++ch) {
    const double* pp = sm.part + (long long)(ch * N + m) * (L + 1);
    a = ch == 0 ? pp[q] : __dadd_rn(a, pp[q]);
    t = ch == 0 ? pp[L] : __dadd_rn(t, pp[L]);
  }
  const double am = alpha[m];
  return __dmul_rn(div_rn(__dsub_rn(a, __dmul_rn(t, phiC[m * LP + q])), am, __drcp_rn(am)), 2.0);
}

template <bool CPLX, int DMAX, bool EXACT, int S, bool SQ = true>
__device__ int eval_cta_gs(const Prob& P, const double* __restrict__ x, const double* __restrict__ dir, double sc,
                           double delta, const Smem& sm, int& rbuf, double* __restrict__ gout, double* F_out,
                           double* s_out, double* __restrict__ wout) {
  constexpr int C = CPLX ? 2 : 1;
  constexpr int LM = C * DMAX;
  const int N = P.N, L = P.L, n = P.n;
  const int LP = EXACT ? gs_col_stride(LM) : gs_col_stride(L);
  const int tid = threadIdx.x;
  double* __restrict__ phiC = sm.phiC;
  PHASE_START;

  // ---- phase 1: column norms, normalisation (smoothing.hpp:95-102)
  int zc = INT_MAX;
  for (int j = tid; j < N; j += S)
    if (gs_norm_col<CPLX, DMAX, EXACT>(P, x, dir, sc, j, phiC, sm.alpha, LP)) zc = min(zc, j);
  zc = block_min_int<S>(zc, sm.ired, rbuf);  // also publishes phiC / alpha
  PHASE_MARK(0);
  if (zc != INT_MAX) {
    for (int i = tid; i < P.dim; i += S) gout[i] = 0.0;
    if (F_out) *F_out = __longlong_as_double(0x7ff0000000000000LL);
    if (s_out) *s_out = 0.0;
    __syncthreads();
    return zc;
  }

  // ---- phase 2
  const double smax = gs_gram_sweep<CPLX, DMAX, EXACT, S, SQ>(P, sm, phiC, LP);
  const double s = block_max<S>(smax, sm.red, rbuf);
  PHASE_MARK(1);

  // ---- phase 3a
  const GsZ Z = gs_exp_z<S>(P, sm, s, delta, rbuf);
  PHASE_MARK(2);
  // the softmax weights are written only when asked for (batch eval API)
  if (wout) {
    for (int p = tid; p < n; p += S) {
      const double w = sm.U[sm.jk[p] & 0xffffu];
      wout[p] = (w > 0.0 && w < 0x1.0p-900) ? ieee_div(w, Z.z) : div_fast(w, Z.z, Z.yz);
    }
  }
  PHASE_MARK(3);

  // ---- phase 4
  gs_grad_loop<CPLX, DMAX, EXACT, S, SQ>(P, sm, phiC, LP, Z);
  if (tid == S - 1) {  // off the critical path when K*N < S (this thread has no unit)
    if (F_out) *F_out = __dadd_rn(s, __dmul_rn(delta, cas_log(Z.z)));
    if (s_out) *s_out = s;
    sm.scal[3] = Z.sparse ? 1.0 : 0.0;  // mask prediction for the next evaluation
  }
  __syncthreads();
  PHASE_MARK(4);
  for (int mq = tid; mq < N * L; mq += S) gout[mq] = gs_combine_elem(P, sm, phiC, sm.alpha, LP, mq);
  __syncthreads();
  PHASE_MARK(5);
  return -1;
}

// Central finite difference (g(x + h dir) - g(x - h dir)) / (2h) (smoothing.hpp:167-181, solver.hpp:118-137) as
// ONE pass over the phases of the two evaluations: both points are normalised in one phase (the + point into
// phiC / alpha, the - point into phiS / alpha2 — the dual layout), the + point's combine runs inside the - point's
// Gram phase (the latency chains of one hide behind the sweep of the other), and the - point's combine forms the
// quotient directly.  Every value is computed by the operations of eval_cta_gs in the same order, so bd is
// bit-identical to two eval_cta_gs calls followed by (g+ - g-) / (2h).  Returns -1, or INT_MAX - 1 when either
// point has a zero column: nothing but scratch has been written then and the caller takes the step-by-step path.
// Needs P.dual.  No barrier at the end: each thread has written the bd elements mq = tid, tid + S, ... it owns.
template <bool CPLX, int DMAX, bool EXACT, int S>
__device__ int hvp_cta_gs(const Prob& P, const double* __restrict__ x, const double* __restrict__ dir, double h,
                          double delta, const Smem& sm, int& rbuf, double* __restrict__ bd) {
  constexpr int C = CPLX ? 2 : 1;
  constexpr int LM = C * DMAX;
  const int N = P.N, L = P.L;
  const int LP = EXACT ? gs_col_stride(LM) : gs_col_stride(L);
  const int tid = threadIdx.x;
  double* __restrict__ phiA = sm.phiC;
  double* __restrict__ phiB = sm.phiS;
  PHASE_START;

  // ---- phase 1 of both points: warps [0, NR/32) take the + point, the next NR/32 warps the - point
  const int NR = (N + 31) & ~31;
  int zc = INT_MAX;
  for (int u = tid; u < 2 * NR; u += S) {
    const int side = u >= NR;
    const int j = u - side * NR;
    if (j < N) {
      const bool zero = side ? gs_norm_col<CPLX, DMAX, EXACT>(P, x, dir, -h, j, phiB, sm.alpha2, LP)
                             : gs_norm_col<CPLX, DMAX, EXACT>(P, x, dir, h, j, phiA, sm.alpha, LP);
      if (zero) zc = min(zc, j);
    }
  }
  zc = block_min_int<S>(zc, sm.ired, rbuf);
  PHASE_MARK(0);
  if (zc != INT_MAX) return INT_MAX - 1;

  // ---- + point: phases 2-4
  double s = block_max<S>(gs_gram_sweep<CPLX, DMAX, EXACT, S, true>(P, sm, phiA, LP), sm.red, rbuf);
  PHASE_MARK(1);
  GsZ Z = gs_exp_z<S>(P, sm, s, delta, rbuf);
  PHASE_MARK(2);
  gs_grad_loop<CPLX, DMAX, EXACT, S, true>(P, sm, phiA, LP, Z);
  if (tid == S - 1) sm.scal[3] = Z.sparse ? 1.0 : 0.0;
  __syncthreads();
  PHASE_MARK(4);

  // ---- + point: combine (reads part, phiA, alpha) inside the - point's Gram phase (writes the pair slots, reads phiB)
  double gp[kGsDualElems];  // the dual layout is only chosen when dim <= kGsDualElems * S
#pragma unroll
  for (int e = 0; e < kGsDualElems; ++e) {
    const int mq = tid + e * S;
    gp[e] = mq < N * L ? gs_combine_elem(P, sm, phiA, sm.alpha, LP, mq) : 0.0;
  }
  s = block_max<S>(gs_gram_sweep<CPLX, DMAX, EXACT, S, true>(P, sm, phiB, LP), sm.red, rbuf);
  PHASE_MARK(1);
  Z = gs_exp_z<S>(P, sm, s, delta, rbuf);
  PHASE_MARK(2);
  gs_grad_loop<CPLX, DMAX, EXACT, S, true>(P, sm, phiB, LP, Z);
  if (tid == S - 1) sm.scal[3] = Z.sparse ? 1.0 : 0.0;
  __syncthreads();
  PHASE_MARK(4);

  // ---- - point: combine, and the quotient (solver.hpp:127)
  {
    const double h2 = 2.0 * h;
#pragma unroll
    for (int e = 0; e < kGsDualElems; ++e) {
      const int mq = tid + e * S;
      if (mq < N * L) bd[mq] = (gp[e] - gs_combine_elem(P, sm, phiB, sm.alpha2, LP, mq)) / h2;
    }
  }
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
__device__ __forceinline__ void build_tables(const Prob& P, Smem& sm) {
  if constexpr (GS)
    build_gs_tables<S, CPLX>(P, sm);
  else
    build_pair_table<S>(P, sm.jk);
}

}  // namespace trstmi_dev
