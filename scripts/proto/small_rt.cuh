// Register-tiled evaluation for the small-frame path (layout 3, "rt"): the
// same arithmetic as eval_cta / eval_cta_gs and the oracle — bit-identical
// results — organised around the resource that binds at small d on B200,
// shared-memory wavefronts (measured: the stored-Gram Gram sweep moves 92 B per
// pair through shared memory and runs at 81 % of the 128 B/clk/SM limit,
// profiles/r2_phase_timers_c2_gs512.txt):
//
//   * the only per-pair shared-memory state is one double (x -> w) in pair
//     order, no pair table: 40 KB at N = 100 instead of 139 KB, so TWO trials
//     are resident per SM and each hides the other's barriers, reduction trees
//     and dependent FP64 chains;
//   * the CTA has T = S / V threads and carries the S CAS lanes V per thread
//     (virtual lanes t, t + T, ...): the CAS reduction shapes, and with them
//     every bit of every result, stay those of the S-lane layouts;
//   * phase 2 (Gram, x, max) is register-tiled: a warp owns 32 consecutive
//     columns k (one per lane, in registers) and walks rows j four at a time;
//     phi_j is a shared-memory broadcast: 4.5 wavefronts per 32 pairs instead
//     of 23;
//   * phase 3a (exp, z) walks p = t, t + T, ... four pairs per step (four
//     independent exp chains), z accumulating per virtual lane in CAS order;
//   * phase 4 (gradient) recomputes G(k, m) from phi_m (registers) and the
//     broadcast phi_k, with the (chunk, column) units ordered so that a warp's
//     lanes share the orientation k < m / k > m (no divergence outside the
//     diagonal blocks).
//
// Reference: eval_objective, smoothing.hpp:82-162; coherence, frame.hpp:138-145
// (paths under /root/reference/proj/include/trstmi).
#pragma once
#include "small_gs.cuh"

namespace trstmi_dev {

// ------------------------------------------------------------------ CAS reductions, V lanes per thread
// v[k][vv] is the partial of virtual lane threadIdx.x + vv * T.  Butterfly
// inside each 32-lane group, then the tree over the S/32 group totals in lane
// order — the order of block_sum<S, K>.  The sums come back in v[k][0].
template <int S, int V, int K>
__device__ __forceinline__ void block_sum_v(double (&v)[K][V], double* red, int& rbuf) {
  constexpr int T = S / V, W = S / 32, WT = T / 32;
#pragma unroll
  for (int k = 0; k < K; ++k)
#pragma unroll
    for (int vv = 0; vv < V; ++vv)
#pragma unroll
      for (int off = 16; off >= 1; off >>= 1) v[k][vv] = __dadd_rn(v[k][vv], __shfl_xor_sync(FULL, v[k][vv], off));
  if constexpr (W > 1) {
    double* buf = red + rbuf * (4 * W);
    const int warp = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
#pragma unroll
      for (int k = 0; k < K; ++k)
#pragma unroll
        for (int vv = 0; vv < V; ++vv) buf[k * W + vv * WT + warp] = v[k][vv];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < K; ++k) v[k][0] = warp_tree_sum<S>(buf + k * W);
    rbuf ^= 1;
  } else {
    __syncwarp();
  }
}

// CAS dot partials: virtual lane l = t + vv * T sums elements l, l + S, ...
template <int S, int V>
__device__ __forceinline__ void dot_lanes(const double* a, const double* b, int n, double (&acc)[V]) {
  constexpr int T = S / V;
#pragma unroll
  for (int vv = 0; vv < V; ++vv) {
    double s = 0.0;
    for (int i = threadIdx.x + vv * T; i < n; i += S) s = fma(a[i], b[i], s);
    acc[vv] = s;
  }
}

template <int S, int V>
__device__ __forceinline__ double block_dot(const double* a, const double* b, int n, double* red, int& rbuf) {
  double v[1][V];
  dot_lanes<S, V>(a, b, n, v[0]);
  block_sum_v<S, V, 1>(v, red, rbuf);
  return v[0][0];
}

// ------------------------------------------------------------------ tiled pair sweep
// Every pair (j, k), j < k, exactly once: a warp owns 32 consecutive columns k
// (one per lane, in registers; segments anchored at the right edge,
// k = khi - 32 + lane) and walks the rows j < khi - 1 RB at a time, warps taking
// the row blocks of all segments round-robin.  f(j[RB], rowvalid[RB], k, pk) —
// lane-level validity is rowvalid[u] && k > j[u].
template <int S, int RB, bool CPLX, int DMAX, bool EXACT, class F>
__device__ __forceinline__ void tiled_pairs(int N, int len, int LP, const double* __restrict__ phiC, F&& f) {
  constexpr int LM = (CPLX ? 2 : 1) * DMAX;
  constexpr int NWP = S / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int g = 0;
  for (int khi = N; khi > 1; khi -= 32) {
    const int rows = khi - 1;  // j = 0 .. khi - 2
    const int nb = (rows + RB - 1) / RB;
    const int k = khi - 32 + lane;
    int b = warp - (g % NWP);
    if (b < 0) b += NWP;
    if (b < nb) {
      double pk[LM];
      load_col<LM, EXACT>(phiC + max(k, 0) * LP, pk, len);
      for (; b < nb; b += NWP) {
        int j[RB];
        bool rv[RB];
#pragma unroll
        for (int u = 0; u < RB; ++u) {
          j[u] = RB * b + u;
          rv[u] = j[u] < rows;
          if (!rv[u]) j[u] = rows - 1;
        }
        f(j, rv, k, pk);
      }
    }
    g += nb;
  }
}

// ------------------------------------------------------------------ gradient units
// Unit u of the K x N (chunk, column) units, ordered: every unit whose chunk
// lies entirely below its column (k < m for all k), then those entirely above
// (k > m), then the diagonal blocks.
__device__ __forceinline__ void rt_unit(int u, int N, int K, int& ch, int& m) {
  int base = 0;
  for (int c = 0; c < K; ++c) {
    const int khi = ((c + 1) * N) / K;
    const int cnt = N - khi;
    if (u < base + cnt) {
      ch = c;
      m = khi + (u - base);
      return;
    }
    base += cnt;
  }
  for (int c = 0; c < K; ++c) {
    const int cnt = (c * N) / K;
    if (u < base + cnt) {
      ch = c;
      m = u - base;
      return;
    }
    base += cnt;
  }
  for (int c = 0; c < K; ++c) {
    const int klo = (c * N) / K, khi = ((c + 1) * N) / K;
    const int cnt = khi - klo;
    if (u < base + cnt) {
      ch = c;
      m = klo + (u - base);
      return;
    }
    base += cnt;
  }
  ch = K - 1;
  m = N - 1;
}

// ------------------------------------------------------------------ workspace
// Shared-memory carve of the rt layout (S = CAS lanes; the CTA has S / V
// threads): phiC (N x LP), alpha, U (n doubles, pair order), part, mask, the
// reduction scratch (strided for S / 32 warps), scalars, nvec vectors of dim.
__host__ __device__ inline long long rt_smem_doubles(const Prob& P, int S, int nvec) {
  const int W = S / 32;
  return (((long long)gs_col_stride(P.L) * P.N + 1) & ~1LL) + P.N + P.n + (long long)P.K * P.N * (P.L + 1) +
         ((long long)P.N * mask_words(P.N) + 1) / 2 + 2LL * 4 * W + 4 + (long long)nvec * P.dim + W + 2;
}

__device__ __forceinline__ void carve_rt(const Prob& P, int S, double* base, Smem& sm, double** vecs, int nvec) {
  const int W = S / 32;
  double* p = base;
  sm.GRI = nullptr;
  sm.fk = nullptr;
  sm.jk = nullptr;
  sm.phiS = nullptr;
  sm.phiC = p;
  p += ((long long)gs_col_stride(P.L) * P.N + 1) & ~1LL;
  sm.alpha = p;
  p += P.N;
  sm.U = p;
  p += P.n;
  sm.part = p;
  p += (long long)P.K * P.N * (P.L + 1);
  sm.mask = reinterpret_cast<unsigned*>(p);
  p += ((long long)P.N * mask_words(P.N) + 1) / 2;
  sm.red = p;
  p += 2 * 4 * W;
  sm.scal = p;
  p += 4;
  for (int v = 0; v < nvec; ++v) {
    vecs[v] = p;
    p += P.dim;
  }
  sm.ired = reinterpret_cast<int*>(p);
}

// ------------------------------------------------------------------ evaluation
// Smem fields used: phiC (N x LP), alpha, U (n, pair order), part, mask, red,
// scal, ired.
template <bool CPLX, int DMAX, bool EXACT, int S, int V, bool SQ = true>
__device__ int eval_cta_rt(const Prob& P, const double* __restrict__ x, const double* __restrict__ dir, double sc,
                           double delta, const Smem& sm, int& rbuf, double* __restrict__ gout, double* F_out,
                           double* s_out, double* __restrict__ wout) {
  constexpr int T = S / V;
  constexpr int C = CPLX ? 2 : 1;
  constexpr int LM = C * DMAX;
  const int d = EXACT ? DMAX : P.d;
  const int N = P.N, L = P.L, n = P.n;
  const int LP = EXACT ? gs_col_stride(LM) : gs_col_stride(L);
  const int tid = threadIdx.x;
  const int NW = mask_words(N);
  double* __restrict__ W = sm.U;
  double* __restrict__ phiC = sm.phiC;
  PHASE_START;

  // ---- phase 1: column norms, normalisation (smoothing.hpp:95-102)
  int zc = INT_MAX;
  for (int j = tid; j < N; j += T) {
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
  zc = block_min_int<T>(zc, sm.ired, rbuf);  // also publishes phiC / alpha
  PHASE_MARK(0);
  if (zc != INT_MAX) {
    for (int i = tid; i < P.dim; i += T) gout[i] = 0.0;
    if (F_out) *F_out = __longlong_as_double(0x7ff0000000000000LL);
    if (s_out) *s_out = 0.0;
    __syncthreads();
    return zc;
  }

  // ---- phase 2: Gram upper triangle (smoothing.hpp:104-118): W <- x_p,
  // s = max x_p ((xv > smax) skips NaNs like the reference's std::max)
  double smax = -__longlong_as_double(0x7ff0000000000000LL);
  tiled_pairs<T, 4, CPLX, DMAX, EXACT>(N, C * d, LP, phiC, [&](const int* j, const bool* rv, int k, const double* pk) {
    double re[4], im[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      double a[LM];
      load_col<LM, EXACT>(phiC + j[u] * LP, a, C * d);
      gram_regs<CPLX, DMAX, EXACT>(a, pk, d, re[u], im[u]);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double uu = CPLX ? __dadd_rn(__dmul_rn(re[u], re[u]), __dmul_rn(im[u], im[u])) : __dmul_rn(re[u], re[u]);
      double xv = uu;
      if constexpr (!SQ) xv = sqrt(uu);
      if (rv[u] && k > j[u]) {
        W[rowstart(N, j[u]) + k - j[u] - 1] = xv;
        smax = xv > smax ? xv : smax;
      }
    }
  });
  if (sm.scal[3] != 0.0)
    for (int i = tid; i < N * NW; i += T) sm.mask[i] = 0u;  // published by block_max's barrier
  const double s = block_max<T, S / 32>(smax, sm.red, rbuf);
  PHASE_MARK(1);

  // ---- phase 3a: w = exp((x - s)/delta) (smoothing.hpp:118-124), 0 where
  // (x - s) < cut (exactly where exp underflows to 0); thread t walks
  // p = t + T q, q ascending: virtual lane q mod V, CAS order inside each lane
  const bool build_mask = sm.scal[3] != 0.0;
  const double cut = __dmul_rn(kUnderflowCut, delta);
  const double ydelta = __drcp_rn(delta);
  const bool chk = !(s >= 0x1.0p-800);  // else every nonzero |x - s| >= 2^-854: the Markstein quotient is exact
  double zz[3][V];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int vv = 0; vv < V; ++vv) zz[a][vv] = 0.0;
  int nnz = 0, tiny = 0;
  constexpr int U4 = (4 % V == 0) ? 4 : 4 * V;  // pairs per step: a multiple of V (lanes stay aligned)
  for (int p0 = tid; p0 < n; p0 += U4 * T) {
    double dd[U4], w[U4];
    bool kk[U4];
    bool any = false;
#pragma unroll
    for (int u = 0; u < U4; ++u) {
      const int p = p0 + u * T;
      dd[u] = __dsub_rn(W[p < n ? p : p0], s);
      kk[u] = p < n && !(dd[u] < cut);  // NaN propagates like cas_exp
      any |= kk[u];
      w[u] = 0.0;
    }
    if (any) {
      double y[U4];
#pragma unroll
      for (int u = 0; u < U4; ++u) {
        y[u] = div_fast(dd[u], delta, ydelta);
        if (chk && dd[u] < 0.0 && dd[u] > -0x1.0p-900) y[u] = ieee_div(dd[u], delta);
      }
#pragma unroll
      for (int u = 0; u < U4; ++u) {
        const double e = TRSTMI_EXP_CORE(y[u]);  // |y| <= 746 (+1 ulp) where taken
        w[u] = kk[u] ? e : 0.0;
        nnz += (int)kk[u];
        tiny |= (int)(kk[u] && y[u] < -620.0);  // w may be < 2^-900: phase 4 checks its quotients
      }
      if (build_mask) {
#pragma unroll
        for (int u = 0; u < U4; ++u) {
          if (kk[u]) {
            int j, k;
            pair_of(N, p0 + u * T, j, k);
            atomicOr(&sm.mask[j * NW + (k >> 5)], 1u << (k & 31));
            atomicOr(&sm.mask[k * NW + (j >> 5)], 1u << (j & 31));
          }
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U4; ++u) {
      const int p = p0 + u * T;
      if (p < n) {
        W[p] = w[u];
        zz[0][u % V] = __dadd_rn(zz[0][u % V], w[u]);
      }
    }
  }
  zz[1][0] = (double)nnz;
  zz[2][0] = (double)tiny;
  block_sum_v<S, V, 3>(zz, sm.red, rbuf);
  PHASE_MARK(2);
  const double z = zz[0][0];
  const bool sparse = zz[1][0] * 4.0 < (double)n;
  const bool use_mask = build_mask && sparse;
  const bool chkdiv = zz[2][0] != 0.0;
  const double yz = __drcp_rn(z);
  if (wout) {  // c_p = w_p / z (smoothing.hpp:125): the softmax weights, when asked for
    for (int p = tid; p < n; p += T) {
      const double w = W[p];
      wout[p] = (w > 0.0 && w < 0x1.0p-900) ? ieee_div(w, z) : div_fast(w, z, yz);
    }
  }
  PHASE_MARK(3);

  // ---- phase 4: gradient (smoothing.hpp:130-160), CAS chunked order: thread
  // (chunk ch, column m), ascending k in [ch*N/K, (ch+1)*N/K): c = w/z,
  // G(k, m) recomputed in the CAS Gram order on (min, max) and conjugated for
  // k > m, t += c u, acc += phi_k (c G(k, m)).
  const int K = P.K;
  const int KN = K * N;
  for (int ubase = 0; ubase < KN; ubase += T) {
    if (ubase + (tid & ~31) >= KN) break;  // whole warp past the end
    const int unit = min(ubase + tid, KN - 1);
    const bool active = ubase + tid < KN;
    int ch, m;
    rt_unit(unit, N, K, ch, m);
    const int k_lo = (ch * N) / K, k_hi = active ? ((ch + 1) * N) / K : k_lo;
    double pm[LM], acc[LM];
    load_col<LM, EXACT>(phiC + m * LP, pm, C * d);
#pragma unroll
    for (int q = 0; q < LM; ++q) acc[q] = 0.0;
    double tp = 0.0;
    auto term = [&](int k, double w, auto lower_tag) {
      constexpr bool lower = decltype(lower_tag)::value;
      double pk[LM];
      load_col<LM, EXACT>(phiC + k * LP, pk, C * d);
      double re, im;
      if constexpr (lower) gram_regs<CPLX, DMAX, EXACT>(pk, pm, d, re, im);
      else gram_regs<CPLX, DMAX, EXACT>(pm, pk, d, re, im);
      const double gi = lower ? im : -im;  // G(k, m) = conj(G(m, k)) for k > m
      double c = div_fast(w, z, yz);
      if (chkdiv && w > 0.0 && w < 0x1.0p-900) c = ieee_div(w, z);
      const double uu = CPLX ? __dadd_rn(__dmul_rn(re, re), __dmul_rn(gi, gi)) : __dmul_rn(re, re);
      if constexpr (!SQ) c = __dmul_rn(c, __ddiv_rn(0.5, fmax(sqrt(uu), 1e-150)));
      tp = __dadd_rn(tp, __dmul_rn(c, uu));
      const double cr = __dmul_rn(c, re);
      if constexpr (CPLX) {
        const double ci = __dmul_rn(c, gi);
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
    const int prow = rowstart(N, m) - m - 1;  // p(m, k) = prow + k
    if (use_mask) {
      const unsigned* mrow = sm.mask + m * NW;
      if (k_lo < k_hi) {
        for (int wi = k_lo >> 5; wi <= ((k_hi - 1) >> 5); ++wi) {
          unsigned wd = mrow[wi];
          const int base = wi << 5;
          if (base < k_lo) wd &= ~0u << (k_lo - base);
          if (k_hi - base < 32) wd &= (1u << (k_hi - base)) - 1u;
          while (wd) {
            const int k = base + __ffs(wd) - 1;
            wd &= wd - 1;
            if (k < m) term(k, W[rowstart(N, k) + (m - k - 1)], BoolTag<true>{});
            else term(k, W[prow + k], BoolTag<false>{});
          }
        }
      }
    } else {
      const int kA = min(k_hi, m);
      if (k_lo < kA) {
        int plo = rowstart(N, k_lo) + (m - k_lo - 1);
#pragma unroll 2
        for (int k = k_lo; k < kA; ++k) {
          const double w = W[plo];
          plo += N - k - 2;
          term(k, w, BoolTag<true>{});
        }
      }
      const int kB = max(k_lo, m + 1);
#pragma unroll 2
      for (int k = kB; k < k_hi; ++k) term(k, W[prow + k], BoolTag<false>{});
    }
    if (active) {
      double* pp = sm.part + (long long)(ch * N + m) * (L + 1);
#pragma unroll
      for (int q = 0; q < LM; ++q)
        if (q < C * d) pp[q] = acc[q];
      pp[L] = tp;
    }
  }
  if (tid == T - 1) {
    if (F_out) *F_out = __dadd_rn(s, __dmul_rn(delta, cas_log(z)));
    if (s_out) *s_out = s;
    sm.scal[3] = sparse ? 1.0 : 0.0;  // mask prediction for the next evaluation
  }
  __syncthreads();
  PHASE_MARK(4);
  for (int mq = tid; mq < N * L; mq += T) {
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

// coherence(normalize_columns(frame)) / coherence(frame) (frame.hpp:60-69,
// 138-145) with the tiled sweep; leaves the (normalised) frame in phiC.
template <bool CPLX, int DMAX, bool EXACT, int T, int WS = T / 32>
__device__ int coherence_cta_rt(const Prob& P, const double* __restrict__ f, bool normalize, const Smem& sm, int& rbuf,
                                double* mu_out, long long* arg_out) {
  constexpr int C = CPLX ? 2 : 1;
  constexpr int LM = C * DMAX;
  const int d = EXACT ? DMAX : P.d;
  const int N = P.N, L = P.L;
  const int LP = EXACT ? gs_col_stride(LM) : gs_col_stride(L);
  const int tid = threadIdx.x;
  int zc = INT_MAX;
  for (int j = tid; j < N; j += T) {
    double a = 1.0;
    if (normalize) {
      double acc = 0.0;
#pragma unroll
      for (int q = 0; q < LM; ++q)
        if (q < C * d) acc = fma(f[j * L + q], f[j * L + q], acc);
      a = sqrt(acc);
      if (a < kZeroColumnTol) zc = min(zc, j);
    }
    sm.alpha[j] = a;
    const double ya = __drcp_rn(a);
#pragma unroll
    for (int q = 0; q < LM; ++q)
      if (q < C * d) sm.phiC[j * LP + q] = normalize ? div_rn(f[j * L + q], a, ya) : f[j * L + q];
  }
  zc = block_min_int<T>(zc, sm.ired, rbuf);
  if (zc != INT_MAX) return zc;
  double best = 0.0;
  long long arg = LLONG_MAX;
  tiled_pairs<T, 4, CPLX, DMAX, EXACT>(N, C * d, LP, sm.phiC, [&](const int* j, const bool* rv, int k, const double* pk) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      double a[LM];
      load_col<LM, EXACT>(sm.phiC + j[u] * LP, a, C * d);
      double re, im;
      gram_regs<CPLX, DMAX, EXACT>(a, pk, d, re, im);
      const double m = cas_hypot(re, CPLX ? im : 0.0);  // std::abs = hypot (frame.hpp:87)
      const long long p = rowstart(N, j[u]) + k - j[u] - 1;
      if (rv[u] && k > j[u] && (m > best || (m == best && m > 0.0 && p < arg))) {  // first strict maximum in pair order
        best = m;
        arg = p;
      }
    }
  });
  block_argmax<T, WS>(best, arg, sm.red, rbuf);
  if (arg == LLONG_MAX) arg = -1;
  *mu_out = best;
  *arg_out = arg;
  return -1;
}

}  // namespace trstmi_dev
