// Large-frame path (BASELINE configs 4-5: real d=64 N=1024, complex d=128
// N=4096, and any shape whose trial state does not fit one SM): one
// evaluation is a short pipeline of grid-wide kernels over state in HBM/L2.
//
//   K1 large_normalize   alpha_j, phi = p/alpha (component-major), first zero column
//   K2 large_gram        upper-triangular 64x64 register-tiled Gram (SYRK) ->
//                        x_p, G(j,k) packed; s = max x_p (atomicMax on the bits)
//   K3 large_weights     w_p = exp((x_p - s)/delta); z partial per 16-row block
//   K4 large_zreduce     z = block partials in row order; F = s + delta log z
//   K5 large_coef        c = w/z; dense coefficient matrices P = c G (k,m) and c u
//   K6 large_grad_gemm   chunked D = Phi P (register-tiled DGEMM, CAS k-chunks)
//                        and, in its rb == 0 CTAs, the t chunk partials
//   K7 large_finalize    chunk combine, grad = ((acc - t phi)/alpha) * 2
//
// Arithmetic is the Canonical Arithmetic Spec with S = 32768
// reduction lanes for dots (128 CTAs x 256 threads), z summed per 16-row block
// (so a row-block sharding across GPUs reproduces it exactly) and
// K = clamp(S/N, 1, 8) gradient chunks: every value is bit-identical to the
// oracle run with the same parameters.
// FP64 tensor cores are not used: sm_100a has no FP64 tcgen05 kind, and the
// legacy DMMA peak equals the DFMA peak on B200 while its internal summation
// order is unspecified — SIMT DFMA tiles keep the CAS order exact.
#pragma once
#include <climits>
#include <cstdint>

#include "small_path.cuh"

namespace trstmi_dev {

constexpr int LS_CTAS = 128;
constexpr int LS_THREADS = 256;
constexpr int LS_LANES = LS_CTAS * LS_THREADS;  // 32768 CAS lanes
constexpr int GT = 64;                           // Gram tile (pairs per side)
constexpr int GIC = 8;                           // Gram i-rows staged per step
constexpr int GNBUF = 3;                         // Gram stage buffers (two in flight)

struct LargeEval {
  int cplx, d, N, L, dim, K, squared;
  long long n;
  const double* x;
  const double* dir;
  double sc, delta;
  double* phiT;                    // L x N component-major
  double* alpha;                   // N
  int* zero_col;                   // 1
  double* X;                       // n: x -> w
  double* GR;                      // n
  double* GI;                      // n
  unsigned long long* smax_bits;   // 1
  double* zpart;                   // LS_CTAS
  double* scal;                    // [0] s, [1] z, [2] F
  double* PR;                      // N x N
  double* PI;                      // N x N
  double* CU;                      // N x N
  double* part;                    // K x dim
  double* tpart;                   // K x N
  double* gout;                    // dim
  double* wout;                    // n or null
  int m0, m1;                      // owned rows / gradient columns [m0, m1) (row-block shard; full = [0, N))
};

// ---- K1: a CTA normalises NC consecutive columns: the columns' NC*L
// doubles (one contiguous run of the point) are staged through shared memory
// with coalesced loads, then thread c runs column c's CAS norm chain
// (ascending fma) and divides by Markstein quotients (== IEEE division).
constexpr int NORM_THREADS = 128;
__host__ __device__ inline int norm_cols(int L) { return max(1, min(32, 2048 / (L + 1))); }
__host__ __device__ inline size_t norm_smem(int L) { return (size_t)norm_cols(L) * (L + 1) * sizeof(double); }
__global__ void __launch_bounds__(NORM_THREADS) large_normalize(LargeEval E) {
  extern __shared__ double ncol[];  // NC x (L + 1)
  if (blockIdx.x == 0 && threadIdx.x == 0) *E.smax_bits = 0ull;
  const int L = E.L, LP = L + 1, NC = norm_cols(L);
  const int j0 = blockIdx.x * NC;
  const int nc = min(NC, E.N - j0);
  const long long base = (long long)j0 * L;
  for (int e0 = 0; e0 < nc * L; e0 += 8 * NORM_THREADS) {  // eight loads in flight per thread
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * NORM_THREADS + threadIdx.x;
      double xv = 0.0;
      if (e < nc * L) {
        xv = E.x[base + e];
        if (E.sc != 0.0) xv = __dadd_rn(xv, __dmul_rn(E.sc, E.dir[base + e]));
      }
      v[u] = xv;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * NORM_THREADS + threadIdx.x;
      if (e < nc * L) {
        const int c = e / L, q = e - c * L;
        ncol[c * LP + q] = v[u];
      }
    }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < nc; c += NORM_THREADS) {
    const double* col = ncol + c * LP;
    const int j = j0 + c;
    double acc = 0.0;
    for (int q = 0; q < L; ++q) acc = fma(col[q], col[q], acc);
    const double a = sqrt(acc);
    E.alpha[j] = a;
    if (a < kZeroColumnTol) {
      atomicMin(E.zero_col, j);
      continue;
    }
    const double ya = __drcp_rn(a);
    for (int q = 0; q < L; ++q) E.phiT[(long long)q * E.N + j] = div_rn(col[q], a, ya);
  }
}

__device__ __forceinline__ void tile_of(int t, int nt, int& jb, int& kb) {  // upper-triangular tile index
  int row = 0, rem = t;
  while (rem >= nt - row) {
    rem -= nt - row;
    ++row;
  }
  jb = row;
  kb = row + rem;
}

// cp.async (global -> shared, 8 bytes, zero-fill when !valid) for the
// double-buffered operand streams of the Gram and gradient GEMMs
__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(src), "r"(valid ? 8 : 0) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int NPEND>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(NPEND) : "memory"); }

// ---- K2: tile (jb <= kb) of GT x GT pairs, 256 threads x (4 j x 4 k).
// mode 0: objective (store x, G, max); mode 1: coherence (per-tile max |G| and first argmax).
template <bool CPLX, int MODE>
__global__ void __launch_bounds__(256) large_gram(LargeEval E, double* tile_mu, long long* tile_arg) {
  // [buffer][re a, re b, (im a, im b)][i][column], cp.async-filled; three
  // buffers so two stages stream in while one computes (48 KB complex).
  __shared__ double gbuf[GNBUF][CPLX ? 4 : 2][GIC][GT];
  double* red_v = &gbuf[0][0][0][0];  // reused after the last stage's barrier
  long long* red_i = reinterpret_cast<long long*>(&gbuf[0][0][1][0]);
  const int N = E.N, d = E.d;
  const int nt = (N + GT - 1) / GT;
  int jb, kb;
  tile_of(blockIdx.x, nt, jb, kb);
  if (MODE == 0) {  // shard: tiles touching the owned rows (as row block) or columns (as column block)
    const int b0 = E.m0 / GT, b1 = (E.m1 + GT - 1) / GT;
    if (!((jb >= b0 && jb < b1) || (kb >= b0 && kb < b1))) return;
  }
  const int tid = threadIdx.x;
  const int tj = tid >> 4, tk = tid & 15;  // 16 x 16 threads, each 4 j x 4 k (strided by 16)
  double re[4][4], im[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) re[a][b] = im[a][b] = 0.0;
  auto issue = [&](int i0, int bsel) {
    if (i0 < d) {
      for (int e = tid; e < GIC * GT; e += 256) {
        const int ii = e / GT, c = e - ii * GT;
        const int i = i0 + ii;
        const int j = jb * GT + c, k = kb * GT + c;
        const bool iv = i < d, vj = iv && j < N, vk = iv && k < N;
        const long long rr = (long long)(CPLX ? 2 * i : i) * N;
        cp_async8(&gbuf[bsel][0][ii][c], E.phiT + (vj ? rr + j : 0), vj);
        cp_async8(&gbuf[bsel][1][ii][c], E.phiT + (vk ? rr + k : 0), vk);
        if (CPLX) {
          cp_async8(&gbuf[bsel][CPLX ? 2 : 0][ii][c], E.phiT + (vj ? rr + N + j : 0), vj);
          cp_async8(&gbuf[bsel][CPLX ? 3 : 1][ii][c], E.phiT + (vk ? rr + N + k : 0), vk);
        }
      }
    }
    cp_async_commit();  // always one group per stage index (empty past d) so the wait counts stay uniform
  };
  const int nst = (d + GIC - 1) / GIC;
  issue(0, 0);
  issue(GIC, 1);
  for (int stg = 0; stg < nst; ++stg) {
    const int i0 = stg * GIC, bsel = stg % GNBUF;
    cp_async_wait<1>();  // stage stg landed (stage stg + 1 may still be in flight)
    __syncthreads();     // ... for every thread, and every thread is done computing stage stg - 1
    issue(i0 + 2 * GIC, (stg + 2) % GNBUF);  // refills the buffer of stage stg - 1
    const int imax = min(GIC, d - i0);
    auto step = [&](int ii) {
      double ar[4], ai[4], br[4], bi[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        ar[a] = gbuf[bsel][0][ii][tj + 16 * a];
        br[a] = gbuf[bsel][1][ii][tk + 16 * a];
        if (CPLX) {
          ai[a] = gbuf[bsel][CPLX ? 2 : 0][ii][tj + 16 * a];
          bi[a] = gbuf[bsel][CPLX ? 3 : 1][ii][tk + 16 * a];
        }
      }
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          if (CPLX) {
            re[a][b] = fma(ar[a], br[b], re[a][b]);
            re[a][b] = fma(ai[a], bi[b], re[a][b]);
            im[a][b] = fma(ar[a], bi[b], im[a][b]);
            im[a][b] = fma(-ai[a], br[b], im[a][b]);
          } else {
            re[a][b] = fma(ar[a], br[b], re[a][b]);
          }
        }
    };
    if (imax == GIC) {  // full stage: compile-time trip count
#pragma unroll 4
      for (int ii = 0; ii < GIC; ++ii) step(ii);
    } else {
      for (int ii = 0; ii < imax; ++ii) step(ii);
    }
  }
  cp_async_wait<0>();
  __syncthreads();  // gbuf is reused by the reduction below
  double best = MODE == 0 ? 0.0 : 0.0;
  long long barg = LLONG_MAX;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int j = jb * GT + tj + 16 * a, k = kb * GT + tk + 16 * b;
      if (j < k && k < N) {
        const long long p = (long long)j * N - (long long)j * (j + 1) / 2 + (k - j - 1);
        const double u = CPLX ? __dadd_rn(__dmul_rn(re[a][b], re[a][b]), __dmul_rn(im[a][b], im[a][b]))
                              : __dmul_rn(re[a][b], re[a][b]);
        if (MODE == 0) {
          const double xv = E.squared ? u : sqrt(u);
          E.X[p] = xv;
          E.GR[p] = re[a][b];
          if (CPLX) E.GI[p] = im[a][b];
          best = fmax(best, xv);
        } else {
          const double m = cas_hypot(re[a][b], CPLX ? im[a][b] : 0.0);  // std::abs (frame.hpp:87)
          if (m > best || (m == best && m > 0.0 && p < barg)) {
            best = m;
            barg = p;
          }
        }
      }
    }
  // CTA reduction
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    const double ov = __shfl_xor_sync(FULL, best, off);
    const long long oi = __shfl_xor_sync(FULL, barg, off);
    if (ov > best || (ov == best && oi < barg)) {
      best = ov;
      barg = oi;
    }
  }
  if ((tid & 31) == 0) {
    red_v[tid >> 5] = best;
    red_i[tid >> 5] = barg;
  }
  __syncthreads();
  if (tid == 0) {
    double v = red_v[0];
    long long ix = red_i[0];
    for (int w = 1; w < 8; ++w)
      if (red_v[w] > v || (red_v[w] == v && red_i[w] < ix)) {
        v = red_v[w];
        ix = red_i[w];
      }
    if (MODE == 0) {
      atomicMax(E.smax_bits, (unsigned long long)__double_as_longlong(v));  // x >= 0: bit order == value order
    } else {
      tile_mu[blockIdx.x] = v;
      tile_arg[blockIdx.x] = ix;
    }
  }
}

// ---- K3b: z partial of each block of ZROWS rows (one CTA per block, 256
// CAS lanes over the block's contiguous pair range); rows before a shard's
// first row: the weights of its owned columns
constexpr int ZROWS = 16;
constexpr int ZLANES = 256;
// ---- K3a: w = exp((x - s)/delta) in place over the pairs of the owned rows
// [m0, m1) (a contiguous pair range), all threads of the grid; Markstein
// quotients and the branch-free exp core (== IEEE division + cas_exp).
__global__ void __launch_bounds__(256) large_exp(LargeEval E) {
  const double s = __longlong_as_double((long long)*E.smax_bits);
  const double cut = __dmul_rn(kUnderflowCut, E.delta);
  const double yd = __drcp_rn(E.delta);
  const bool chk = !(s >= 0x1.0p-800);  // else every nonzero |x - s| >= 2^-854 (Markstein exact)
  const long long N = E.N, m0 = E.m0, m1 = E.m1;
  const long long p0 = m0 * N - m0 * (m0 + 1) / 2, p1 = m1 * N - m1 * (m1 + 1) / 2;
  double* __restrict__ X = E.X;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long p = p0 + blockIdx.x * (long long)blockDim.x + threadIdx.x; p < p1; p += 2 * stride) {
    const long long q = p + stride;
    const bool v2 = q < p1;
    const double d1 = __dsub_rn(X[p], s), d2 = v2 ? __dsub_rn(X[q], s) : 0.0;
    double y1 = div_fast(d1, E.delta, yd), y2 = div_fast(d2, E.delta, yd);
    if (chk) {
      if (d1 < 0.0 && d1 > -0x1.0p-900) y1 = __ddiv_rn(d1, E.delta);
      if (d2 < 0.0 && d2 > -0x1.0p-900) y2 = __ddiv_rn(d2, E.delta);
    }
    const double e1 = cas_exp_core(y1), e2 = cas_exp_core(y2);  // the core domain wherever !(diff < cut)
    X[p] = (d1 < cut) ? 0.0 : e1;
    if (v2) X[q] = (d2 < cut) ? 0.0 : e2;
  }
}

template <bool FUSED>
__global__ void __launch_bounds__(ZLANES) large_weights(LargeEval E) {
  __shared__ double wt[ZLANES / 32];
  const double s = __longlong_as_double((long long)*E.smax_bits);
  const double cut = __dmul_rn(kUnderflowCut, E.delta);
  const long long N = E.N;
  const long long r0 = (long long)blockIdx.x * ZROWS, r1 = min(N, r0 + ZROWS);
  if (r0 >= E.m1) return;
  if (r0 < E.m0) {  // rows before the shard: only the pairs in owned columns (no z)
    for (long long r = r0; r < r1; ++r) {
      const long long base = r * N - r * (r + 1) / 2 - r - 1;
      for (long long k = max(r + 1, (long long)E.m0) + threadIdx.x; k < E.m1; k += ZLANES) {
        const long long p = base + k;
        const double diff = __dsub_rn(E.X[p], s);
        E.X[p] = (diff < cut) ? 0.0 : cas_exp(__ddiv_rn(diff, E.delta));
      }
    }
    return;
  }
  const long long p0 = r0 * N - r0 * (r0 + 1) / 2, p1 = r1 * N - r1 * (r1 + 1) / 2;
  double* __restrict__ X = E.X;
  double zp = 0.0;
  if (FUSED) {  // weights computed here (small frames: one launch fewer per evaluation)
    const double yd = __drcp_rn(E.delta);
    const bool chk = !(s >= 0x1.0p-800);  // else every nonzero |x - s| >= 2^-854 (Markstein exact)
    for (long long p = p0 + threadIdx.x; p < p1; p += 4 * ZLANES) {
      double xv[4], w[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) xv[u] = (p + u * ZLANES < p1) ? X[p + u * ZLANES] : 0.0;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double diff = __dsub_rn(xv[u], s);
        double y = div_fast(diff, E.delta, yd);
        if (chk && diff < 0.0 && diff > -0x1.0p-900) y = __ddiv_rn(diff, E.delta);
        const double e = cas_exp_core(y);  // the core domain wherever !(diff < cut)
        w[u] = (diff < cut) ? 0.0 : e;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (p + u * ZLANES < p1) {
          X[p + u * ZLANES] = w[u];
          zp = __dadd_rn(zp, w[u]);
        }
      }
    }
  } else {
    // w written by large_exp; lane l sums its pairs l, l+256, ... in order (the
    // CAS z order), four loads in flight
    for (long long p = p0 + threadIdx.x; p < p1; p += 4 * ZLANES) {
      double w[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) w[u] = (p + u * ZLANES < p1) ? X[p + u * ZLANES] : 0.0;
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (p + u * ZLANES < p1) zp = __dadd_rn(zp, w[u]);
    }
  }
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) zp = __dadd_rn(zp, __shfl_xor_sync(FULL, zp, off));
  if ((threadIdx.x & 31) == 0) wt[threadIdx.x >> 5] = zp;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < ZLANES / 32 ? wt[threadIdx.x] : 0.0;
#pragma unroll
    for (int off = 1; off < ZLANES / 32; off <<= 1) v = __dadd_rn(v, __shfl_xor_sync(FULL, v, off));
    if (threadIdx.x == 0) E.zpart[blockIdx.x] = v;
  }
  if (threadIdx.x == 0 && r0 == E.m0) E.scal[0] = s;
}

// ---- K4: z = block sums added in row order; F = s + delta log z
__global__ void large_zreduce(LargeEval E, int nblocks) {
  __shared__ double zs[1024];
  const bool staged = nblocks <= 1024;
  if (staged)
    for (int b = threadIdx.x; b < nblocks; b += blockDim.x) zs[b] = E.zpart[b];  // loads in parallel
  __syncthreads();
  if (threadIdx.x != 0) return;
  E.scal[0] = __longlong_as_double((long long)*E.smax_bits);
  const double* zp = staged ? zs : E.zpart;
  double z = zp[0];
  for (int b = 1; b < nblocks; ++b) z = __dadd_rn(z, zp[b]);
  E.scal[1] = z;
  E.scal[2] = __dadd_rn(E.scal[0], __dmul_rn(E.delta, cas_log(z)));
}

// ---- K5: coefficients into dense P (row k, column m): P(k,m) = c G(k,m),
// one CTA per upper-triangular 64x64 pair tile: the packed rows are read
// coalesced, P(j,k) written row-major and P(k,j) through a shared-memory
// transpose (both coalesced).  c = w / z by Markstein quotients (== IEEE).
template <bool CPLX>
__global__ void __launch_bounds__(256) large_coef(LargeEval E) {
  constexpr int HR = 16;  // tile rows per pass (4 elements per thread: few registers, high occupancy)
  __shared__ double tv[3][HR][GT + 1];
  const int N = E.N;
  const int nt = (N + GT - 1) / GT;
  int jb, kb;
  tile_of(blockIdx.x, nt, jb, kb);
  if (jb * GT >= E.m1) return;  // rows >= m1 are not owned
  const double z = E.scal[1];
  const double yz = __drcp_rn(z);
  {  // pass h = rows [h, h + HR) of the tile (gridDim.y = GT / HR passes)
    const int h = blockIdx.y * HR;
#pragma unroll
    for (int i = 0; i < HR * GT / 256; ++i) {
      const int e = threadIdx.x + 256 * i;
      const int r = e / GT, c = e - r * GT;
      const int j = jb * GT + h + r, k = kb * GT + c;
      // shard: rows >= m0, plus the owned columns of the rows before m0
      const bool ok = j < k && k < N && j < E.m1 && (j >= E.m0 || (k >= E.m0 && k < E.m1));
      double vr = 0.0, vi = 0.0, vu = 0.0;
      if (ok) {
        const long long p = (long long)j * N - (long long)j * (j + 1) / 2 + (k - j - 1);
        const double w = E.X[p];
        const double cq = (w == 0.0) ? 0.0 : div_rn(w, z, yz);
        if (E.wout) E.wout[p] = cq;
        if (cq != 0.0) {
          const double gr = E.GR[p];
          const double gi = CPLX ? E.GI[p] : 0.0;
          const double u = CPLX ? __dadd_rn(__dmul_rn(gr, gr), __dmul_rn(gi, gi)) : __dmul_rn(gr, gr);
          double cc = cq;
          if (!E.squared) cc = __dmul_rn(cc, __ddiv_rn(0.5, fmax(sqrt(u), 1e-150)));
          vr = __dmul_rn(cc, gr);
          vi = __dmul_rn(cc, gi);
          vu = __dmul_rn(cc, u);
        }
        const long long o = (long long)j * N + k;
        E.PR[o] = vr;
        E.CU[o] = vu;
        if (CPLX) E.PI[o] = vi;
      }
      tv[0][r][c] = vr;
      tv[1][r][c] = vu;
      tv[2][r][c] = -vi;  // P(k,j) = c conj(G(j,k))
    }
    __syncthreads();
    // transposed: row k = kb*GT + c2 (64 rows), columns j = jb*GT + h + r2 (16 per row)
#pragma unroll
    for (int i = 0; i < HR * GT / 256; ++i) {
      const int e = threadIdx.x + 256 * i;
      const int c2 = e / HR, r2 = e - c2 * HR;
      const int j = jb * GT + h + r2, k = kb * GT + c2;
      const bool ok = j < k && k < N && j < E.m1 && (j >= E.m0 || (k >= E.m0 && k < E.m1));
      if (ok) {
        const long long o = (long long)k * N + j;
        E.PR[o] = tv[0][r2][c2];
        E.CU[o] = tv[1][r2][c2];
        if (CPLX) E.PI[o] = tv[2][r2][c2];
      }
    }
  }
}

// ---- K6: chunked gradient GEMM D(q, m) = sum_k phi(q, k) (x) P(k, m)
// over k in chunk c (ascending), register tile 4 m x 4 rows per thread.
// Operand tiles stream global -> shared with cp.async into two buffers, so
// the next k-step's loads overlap this step's FMAs.  The rb == 0 CTAs also
// sum the c*u tile into the t chunk partials (ascending k, add).
constexpr int GM = 64, GK = 16, GRB = 64;  // columns, k-step, rows per CTA
#ifndef GG_UNROLL
#define GG_UNROLL 4
#endif
constexpr int GFS = GRB + 1;  // phi tile row stride: the k-major cp.async writes hit distinct banks
__host__ __device__ constexpr size_t gg_smem(int gmt) { return 2 * (size_t)(GK * gmt * 3 + GK * GFS * 2) * sizeof(double); }


template <bool CPLX, int GMT>
__global__ void __launch_bounds__(256) large_grad_gemm(LargeEval E) {
  constexpr int CW = GMT / 16;                                      // columns per thread
  constexpr int BUF = GK * GMT * 3 + GK * GFS * 2;                  // doubles per pipeline buffer
  constexpr int RT = 4;  // complex rows / real rows per thread
  extern __shared__ double gsm[];
  const int N = E.N, d = E.d, K = E.K;
  const int mb = blockIdx.x + E.m0 / GMT, rb = blockIdx.y, ch = blockIdx.z;
  const int k_lo = (ch * N) / K, k_hi = ((ch + 1) * N) / K;
  const int tid = threadIdx.x;
  const int tm = tid & 15, tr = tid >> 4;
  const bool tsum = rb == 0 && tr == 0;  // threads 0..15: t of columns tm + 16c, ascending k (c*u add)
  auto issue = [&](int k0, int b) {
    double* base = gsm + b * BUF;
    for (int e = tid; e < GK * GMT; e += 256) {
      const int kk = e / GMT, c = e - kk * GMT;
      const int k = k0 + kk, m = mb * GMT + c;
      const bool v = k < k_hi && m < E.m1;
      const long long o = v ? (long long)k * N + m : 0;
      cp_async8(base + e, E.PR + o, v);
      if (CPLX) cp_async8(base + GK * GMT + e, E.PI + o, v);
      if (rb == 0) cp_async8(base + 2 * GK * GMT + e, E.CU + o, v);
    }
    for (int e = tid; e < GK * GRB; e += 256) {  // lanes along k: 128-byte runs of phi rows
      const int kk = e % GK, r = e / GK;
      const int k = k0 + kk, row = rb * GRB + r;
      const bool v = k < k_hi && row < d;
      double* dst = base + 3 * GK * GMT + kk * GFS + r;
      if (CPLX) {
        cp_async8(dst, E.phiT + (v ? (long long)(2 * row) * N + k : 0), v);
        cp_async8(dst + GK * GFS, E.phiT + (v ? (long long)(2 * row + 1) * N + k : 0), v);
      } else {
        cp_async8(dst, E.phiT + (v ? (long long)row * N + k : 0), v);
      }
    }
    cp_async_commit();
  };
  double ar[RT][CW], ai[RT][CW];
#pragma unroll
  for (int r = 0; r < RT; ++r)
#pragma unroll
    for (int c = 0; c < CW; ++c) ar[r][c] = ai[r][c] = 0.0;
  double tc[CW];
#pragma unroll
  for (int c = 0; c < CW; ++c) tc[c] = 0.0;
  const int nsteps = (k_hi - k_lo + GK - 1) / GK;
  if (nsteps > 0) issue(k_lo, 0);
  for (int st = 0; st < nsteps; ++st) {
    const int b = st & 1, k0 = k_lo + st * GK;
    if (st + 1 < nsteps) {
      issue(k0 + GK, b ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double* sPr = gsm + b * BUF;
    const double* sPi = sPr + GK * GMT;
    const double* sCU = sPr + 2 * GK * GMT;
    const double* sFr = sPr + 3 * GK * GMT;
    const double* sFi = sFr + GK * GFS;
    const int kmax = min(GK, k_hi - k0);
    if (tsum) {
      for (int kk = 0; kk < kmax; ++kk)
#pragma unroll
        for (int c = 0; c < CW; ++c) tc[c] = __dadd_rn(tc[c], sCU[kk * GMT + tm + 16 * c]);
    }
    auto step = [&](int kk) {
      double pr[CW], pi[CW], fr[RT], fi[RT];
#pragma unroll
      for (int c = 0; c < CW; ++c) {
        pr[c] = sPr[kk * GMT + tm + 16 * c];
        if (CPLX) pi[c] = sPi[kk * GMT + tm + 16 * c];
      }
#pragma unroll
      for (int r = 0; r < RT; ++r) {
        fr[r] = sFr[kk * GFS + tr + 16 * r];
        if (CPLX) fi[r] = sFi[kk * GFS + tr + 16 * r];
      }
#pragma unroll
      for (int r = 0; r < RT; ++r)
#pragma unroll
        for (int c = 0; c < CW; ++c) {
          if (CPLX) {
            ar[r][c] = fma(fr[r], pr[c], ar[r][c]);
            ar[r][c] = fma(-fi[r], pi[c], ar[r][c]);
            ai[r][c] = fma(fr[r], pi[c], ai[r][c]);
            ai[r][c] = fma(fi[r], pr[c], ai[r][c]);
          } else {
            ar[r][c] = fma(fr[r], pr[c], ar[r][c]);
          }
        }
    };
    if (kmax == GK) {  // full step: a compile-time trip count lets loads run ahead of the FMAs
#pragma unroll 4
      for (int kk = 0; kk < GK; ++kk) step(kk);
    } else {
      for (int kk = 0; kk < kmax; ++kk) step(kk);
    }
    __syncthreads();  // buffer b is refilled by the issue two steps on
  }
  if (tsum) {
#pragma unroll
    for (int c = 0; c < CW; ++c) {
      const int m = mb * GMT + tm + 16 * c;
      if (m < E.m1) E.tpart[(long long)ch * N + m] = tc[c];
    }
  }
#pragma unroll
  for (int r = 0; r < RT; ++r)
#pragma unroll
    for (int c = 0; c < CW; ++c) {
      const int row = rb * GRB + tr + 16 * r, m = mb * GMT + tm + 16 * c;
      if (row < d && m < E.m1) {
        double* out = E.part + (long long)ch * E.dim + (long long)m * E.L;
        if (CPLX) {
          out[2 * row] = ar[r][c];
          out[2 * row + 1] = ai[r][c];
        } else {
          out[row] = ar[r][c];
        }
      }
    }
}

// ---- K7: chunk partials added left to right; grad = ((acc - t phi)/alpha)*2
__global__ void large_finalize(LargeEval E) {
  const long long e = (long long)E.m0 * E.L + blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= (long long)E.m1 * E.L) return;
  const int m = (int)(e / E.L), q = (int)(e - (long long)m * E.L);
  double a = E.part[e], t = E.tpart[m];
  for (int ch = 1; ch < E.K; ++ch) {
    a = __dadd_rn(a, E.part[(long long)ch * E.dim + e]);
    t = __dadd_rn(t, E.tpart[(long long)ch * E.N + m]);
  }
  const double phi = E.phiT[(long long)q * E.N + m];
  E.gout[e] = __dmul_rn(__ddiv_rn(__dsub_rn(a, __dmul_rn(t, phi)), E.alpha[m]), 2.0);
}

// ---- vector kernels (trust-region state in HBM)
// CAS dots of width LS_LANES: up to 3 dots at once, per-CTA tree totals.
__global__ void __launch_bounds__(LS_THREADS) large_dots(const double* a0, const double* b0, const double* a1,
                                                          const double* b1, const double* a2, const double* b2, int nd,
                                                          long long n, double* cta_out) {
  __shared__ double wt[3][LS_THREADS / 32];
  const long long t = (long long)blockIdx.x * LS_THREADS + threadIdx.x;
  double v[3] = {0.0, 0.0, 0.0};
  for (long long i = t; i < n; i += LS_LANES) {
    v[0] = fma(a0[i], b0[i], v[0]);
    if (nd > 1) v[1] = fma(a1[i], b1[i], v[1]);
    if (nd > 2) v[2] = fma(a2[i], b2[i], v[2]);
  }
#pragma unroll
  for (int q = 0; q < 3; ++q) {
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) v[q] = __dadd_rn(v[q], __shfl_xor_sync(FULL, v[q], off));
    if ((threadIdx.x & 31) == 0) wt[q][threadIdx.x >> 5] = v[q];
  }
  __syncthreads();
  if (threadIdx.x < 32) {
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      double u = threadIdx.x < LS_THREADS / 32 ? wt[q][threadIdx.x] : 0.0;
#pragma unroll
      for (int off = 1; off < LS_THREADS / 32; off <<= 1) u = __dadd_rn(u, __shfl_xor_sync(FULL, u, off));
      if (threadIdx.x == 0) cta_out[q * LS_CTAS + blockIdx.x] = u;
    }
  }
}

__global__ void large_dots_reduce(const double* cta_out, int nd, double* out) {
  __shared__ double wt[3][LS_CTAS / 32];
  for (int q = 0; q < nd; ++q) {
    double v = cta_out[q * LS_CTAS + threadIdx.x];
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) v = __dadd_rn(v, __shfl_xor_sync(FULL, v, off));
    if ((threadIdx.x & 31) == 0) wt[q][threadIdx.x >> 5] = v;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    for (int q = 0; q < nd; ++q) {
      double u = threadIdx.x < LS_CTAS / 32 ? wt[q][threadIdx.x] : 0.0;
#pragma unroll
      for (int off = 1; off < LS_CTAS / 32; off <<= 1) u = __dadd_rn(u, __shfl_xor_sync(FULL, u, off));
      if (threadIdx.x == 0) out[q] = u;
    }
  }
}

// y = a + s*b elementwise (mul then add)
__global__ void large_axpy(double* y, const double* a, double s, const double* b, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    y[i] = __dadd_rn(a[i], __dmul_rn(s, b[i]));
}
// d = -r + beta*d
__global__ void large_cg_dir(double* d, const double* r, double beta, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    d[i] = __dadd_rn(-r[i], __dmul_rn(beta, d[i]));
}
// hv = (gp - gm) / den
__global__ void large_fd(double* hv, const double* gp, const double* gm, double den, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    hv[i] = __ddiv_rn(__dsub_rn(gp[i], gm[i]), den);
}
__global__ void large_neg(double* y, const double* a, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    y[i] = -a[i];
}
__global__ void large_nonfinite(const double* a, long long n, int* flag) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    if (!isfinite(a[i])) atomicExch(flag, 1);
}

}  // namespace trstmi_dev
