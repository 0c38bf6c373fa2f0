// Batched device engine (BDE) for large frames (BASELINE configs 4-5 and any
// shape whose trial state does not fit one SM): many evaluation requests —
// the trust-region points of every trial in flight, or the B points of an
// eval/hvp/coherence batch — run through ONE launch per pipeline kernel
// (request index in the grid), and the trust-region / Steihaug-CG / anneal
// control of every trial runs on the device (bde_tr.cuh).
//
// Pipeline (one launch each, all requests of a tick):
//   bde_normalize   alpha_j, phi = p / alpha in the point layout (column j =
//                   L contiguous doubles), first zero column
//   bde_gram        upper-triangular 64x64 Gram tiles on the FP64 tensor
//                   cores (mma.sync m16n8k4 .f64 = DMMA): complex products as
//                   one real GEMM over the interleaved K = 2d with operands
//                   R and J R; the epilogue keeps only G(j,k), j < k, packed
//                   (interleaved re, im) and the block max of x = |G|^2
//   bde_weights     w = exp((x - s)/delta) (x recomputed from G), z partial
//                   per 16-row block
//   bde_zreduce     z in block order, F = s + delta log z
//   bde_grad_ws     D^T = P^T Phi on DMMA with the coefficient matrix
//                   P(k, m) = (w/z) G(k, m) (conjugated below the diagonal)
//                   formed tile by tile in shared memory from the packed
//                   (w, G) by producer warps while consumer warps run the
//                   MMAs — the N x N coefficient matrix never exists in HBM
//                   (north star: W o G fused into the contraction) — plus the
//                   t chunk partials sum_k (w/z) u
//   bde_finalize    chunk partials left to right, grad = ((acc - t phi)/alpha) 2
//
// Arithmetic: the Canonical Arithmetic Spec of the large path,
// bit for bit.  DMMA computes each output as the ascending fma chain over its
// k inputs (measured: profiles/r2_dmma_probe.txt — 0 mismatches against
// std::fma chains on 1.8 M outputs), so a DMMA GEMM over the interleaved
// complex layout reproduces the CAS Gram order (re: ar br, ai bi; im: ar bi,
// -ai br per i ascending) and gradient order (re: fr pr, -fi pi; im: fr pi,
// fi pr per k ascending within a chunk) exactly; every other operation is the
// same IEEE operation as in large_path.cuh / the oracle.
#pragma once
#include <climits>
#include <cstdint>

#include "small_path.cuh"

namespace trstmi_bde {
using namespace trstmi_dev;

constexpr int BT = 64;            // Gram tile edge / gradient m-block
constexpr int BZROWS = 16;        // CAS z blocks (rows) — as large_path.cuh ZROWS
constexpr int BZLANES = 256;      // CAS z lanes per block
constexpr int GKS = 32;           // Gram: K (interleaved) per pipeline stage
constexpr int GSA = GKS + 4;      // Gram smem row stride (== 4 mod 16: conflict-free fragments)
constexpr int NORM_T = 128;

struct Shape {
  int cplx, d, N, L, dim, K;  // L = 2d (complex) / d (real); K = CAS gradient chunks
  long long n;                // pairs
  int nt, tiles, nzb;         // 64-tiles per side, upper tiles, z blocks
};

enum ReqKind { REQ_OBJ = 0, REQ_COH_NORM = 1, REQ_COH_RAW = 2 };

// One evaluation request: the point x + sc * dir (dir nullable).
struct Req {
  const double* x;
  const double* dir;
  double sc;
  double delta;
  double* grad;   // REQ_OBJ: dim doubles out
  double* wout;   // nullable: softmax weights (n) out
  int kind;
  int squared;
  int slot;       // workspace slot
  int pad;
};

struct ReqOut {
  double F, s, z, mu;
  long long argmax;
  unsigned long long smax;  // bits of max x (x >= 0)
  int zc;                   // first zero column (INT_MAX: none)
  int pad;
};

// Slot-strided workspace.
struct Ws {
  double* phi;    // dim per slot, point layout
  double* alpha;  // N
  double* G;      // n (real) / 2n (complex, interleaved)
  double* W;      // n
  double* zpart;  // nzb
  double* part;   // K x dim
  double* tpart;  // K x N
  double* tmu;    // tiles
  long long* targ;
  long long s_phi, s_alpha, s_G, s_W, s_zpart, s_part, s_tpart, s_tile;
};

struct Pipe {
  Shape sh;
  const Req* reqs;
  ReqOut* outs;   // indexed by request
  const int* active;  // request ids of this launch (blockIdx.y / .z -> active[.])
  Ws ws;
};

__device__ __forceinline__ long long pair_index(long long j, long long k, long long N) {
  return j * N - j * (j + 1) / 2 + (k - j - 1);
}

__device__ __forceinline__ void tile_coords(int t, int nt, int& jb, int& kb) {
  // upper-triangular tile t (row-major over jb <= kb)
  int row = 0, rem = t;
  while (rem >= nt - row) {
    rem -= nt - row;
    ++row;
  }
  jb = row;
  kb = row + rem;
}

__device__ __forceinline__ void cpa8(double* dst, const double* src, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(src), "r"(valid ? 8 : 0) : "memory");
}
__device__ __forceinline__ void cpa16(double* dst, const double* src, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(src), "r"(valid ? 16 : 0) : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int NP>
__device__ __forceinline__ void cpa_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(NP) : "memory"); }

// TMA bulk copies (cp.async.bulk, the copy engine — no tensor map needed for a
// contiguous run) completing on an mbarrier.
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@p bra DONE_%=;\n"
      "bra WAIT_%=;\n"
      "DONE_%=:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// D (m16 x n8, f64) += A (m16 x k4) B (k4 x n8): one DMMA, the ascending fma
// chain over k per output.  a0 = A[g][t], a1 = A[g+8][t], b = B[t][g];
// c0,c1 = C[g][2t, 2t+1], c2,c3 = C[g+8][2t, 2t+1]  (g = lane/4, t = lane%4).
__device__ __forceinline__ void dmma(double (&c)[4], double a0, double a1, double b) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
               : "d"(a0), "d"(a1), "d"(b));
}

// ---------------------------------------------------------------- K1
// A CTA normalises NC consecutive columns (one contiguous run of NC*L doubles
// of the point), CAS norm chain per column, Markstein quotients (== IEEE).
__host__ __device__ inline int bde_norm_cols(int L) { return max(1, min(32, 2048 / (L + 1))); }
__host__ __device__ inline size_t bde_norm_smem(int L) {
  return ((size_t)bde_norm_cols(L) * (L + 1) + 2 * (size_t)bde_norm_cols(L)) * sizeof(double);
}

__global__ void __launch_bounds__(NORM_T) bde_normalize(Pipe P) {
  extern __shared__ double ncol[];  // NC x (L + 1), then alpha[NC], 1/alpha[NC]
  const Shape& sh = P.sh;
  const int r = P.active[blockIdx.y];
  const Req q = P.reqs[r];
  const int L = sh.L, LP = L + 1, NC = bde_norm_cols(L);
  double* sal = ncol + NC * LP;
  double* sya = sal + NC;
  const int j0 = blockIdx.x * NC;
  const int nc = min(NC, sh.N - j0);
  const long long base = (long long)j0 * L;
  double* phi = P.ws.phi + (long long)q.slot * P.ws.s_phi;
  const bool raw = q.kind == REQ_COH_RAW;
  for (int e0 = 0; e0 < nc * L; e0 += 8 * NORM_T) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * NORM_T + threadIdx.x;
      double xv = 0.0;
      if (e < nc * L) {
        xv = q.x[base + e];
        if (q.sc != 0.0) xv = __dadd_rn(xv, __dmul_rn(q.sc, q.dir[base + e]));
      }
      v[u] = xv;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * NORM_T + threadIdx.x;
      if (e < nc * L) {
        if (raw) {
          phi[base + e] = v[u];
        } else {
          const int c = e / L, qq = e - c * L;
          ncol[c * LP + qq] = v[u];
        }
      }
    }
  }
  if (raw) return;
  __syncthreads();
  double* alpha = P.ws.alpha + (long long)q.slot * P.ws.s_alpha;
  for (int c = threadIdx.x; c < nc; c += NORM_T) {
    const double* col = ncol + c * LP;
    double acc = 0.0;
    for (int qq = 0; qq < L; ++qq) acc = fma(col[qq], col[qq], acc);
    const double a = sqrt(acc);
    alpha[j0 + c] = a;
    sal[c] = a;
    sya[c] = __drcp_rn(a);
    if (a < kZeroColumnTol) atomicMin(&P.outs[r].zc, j0 + c);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < nc * L; e += NORM_T) {  // coalesced point-layout stores
    const int c = e / L, qq = e - c * L;
    phi[base + e] = div_rn(ncol[c * LP + qq], sal[c], sya[c]);
  }
}

// ---------------------------------------------------------------- K2
// Upper-triangular 64x64 tile (jb <= kb) of G = Phi* Phi on DMMA.  8 warps:
// warp (wj, wk) = (w / 4, w % 4) owns rows 32 wj .. +32 and columns 16 wk ..
// +16: two m16 x two n8 MMA tiles, re (and im) accumulators.  Operands are
// the columns of phi (rows of R^T), staged through shared memory in GKS-wide
// K stages, two buffers.  TMA = true (L a multiple of 4): each stage is 128
// bulk copies of one 256-byte row segment (cp.async.bulk, issued by warp 0,
// four per lane) completing on the buffer's mbarrier — 128 copy instructions
// per stage instead of 4096 8-byte cp.async; rows past N re-read row N - 1
// (their products are never stored).  TMA = false: 8-byte cp.async with
// zero fill, any L.
// MODE 0: objective (packed G, block max of x); MODE 1: coherence (|G| by
// hypot, first argmax of the tile).
__host__ __device__ constexpr size_t bde_gram_smem() { return 2 * 2 * (size_t)BT * GSA * sizeof(double); }

template <bool CPLX, int MODE, bool TMA>
__global__ void __launch_bounds__(256, CPLX ? 2 : 3) bde_gram(Pipe P) {  // real: 32 accumulator registers, three CTAs per SM

  extern __shared__ __align__(16) double gsm[];  // [buf][A | B][64][GSA]
  __shared__ double red_v[8];
  __shared__ long long red_i[8];
  __shared__ __align__(8) unsigned long long full_bar[2];
  const Shape& sh = P.sh;
  const int r = P.active[blockIdx.y];
  const Req q = P.reqs[r];
  if (P.outs[r].zc != INT_MAX && q.kind != REQ_COH_RAW) return;  // zero column: nothing to compute
  const int N = sh.N, L = sh.L;
  int jb, kb;
  tile_coords(blockIdx.x, sh.nt, jb, kb);
  const double* phi = P.ws.phi + (long long)q.slot * P.ws.s_phi;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wj = warp >> 2, wk = warp & 3;
  double re[2][2][4], im[2][2][4];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int e = 0; e < 4; ++e) re[a][b][e] = im[a][b][e] = 0.0;
  const int nst = (L + GKS - 1) / GKS;
  if (TMA) {
    if (tid == 0) {
      mbar_init(&full_bar[0], 1);
      mbar_init(&full_bar[1], 1);
      fence_proxy_async();
    }
    __syncthreads();
  }
  auto issue = [&](int s, int buf) {
    if (TMA) {
      if (warp == 0 && s < nst) {
        double* As = gsm + buf * (2 * BT * GSA);
        const int q0 = s * GKS;
        const unsigned bytes = (unsigned)min(GKS, L - q0) * 8u;  // a multiple of 32 (L % 4 == 0)
        if (lane == 0) mbar_expect_tx(&full_bar[buf], 2u * BT * bytes);
        __syncwarp();
#pragma unroll
        for (int u = 0; u < 2 * BT / 32; ++u) {
          const int rr = lane + 32 * u;  // 0..63: A rows (jb), 64..127: B rows (kb)
          const int row = rr & (BT - 1);
          const int col = min((rr < BT ? jb : kb) * BT + row, N - 1);
          bulk_g2s(As + rr * GSA, phi + (long long)col * L + q0, bytes, &full_bar[buf]);
        }
      }
      return;
    }
    if (s < nst) {
      double* As = gsm + buf * (2 * BT * GSA);
      double* Bs = As + BT * GSA;
      const int q0 = s * GKS;
      for (int e = tid; e < BT * GKS; e += 256) {
        const int row = e / GKS, c = e - row * GKS;
        const int qq = q0 + c;
        const int j = jb * BT + row, k = kb * BT + row;
        const bool vq = qq < L;
        cpa8(As + row * GSA + c, phi + (vq && j < N ? (long long)j * L + qq : 0), vq && j < N);
        cpa8(Bs + row * GSA + c, phi + (vq && k < N ? (long long)k * L + qq : 0), vq && k < N);
      }
    }
    cpa_commit();
  };
  issue(0, 0);
  for (int s = 0; s < nst; ++s) {
    issue(s + 1, (s + 1) & 1);
    if (TMA) {
      mbar_wait(&full_bar[s & 1], (s >> 1) & 1);  // the stage's bytes have landed
    } else {
      cpa_wait<1>();
      __syncthreads();
    }
    const double* As = gsm + (s & 1) * (2 * BT * GSA);
    const double* Bs = As + BT * GSA;
    const int kq = min(GKS, L - s * GKS);  // valid K in this stage (zero-filled beyond)
#pragma unroll 2
    for (int q4 = 0; q4 < GKS; q4 += 4) {
      if (q4 >= kq) break;
      double a0[2], a1[2];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        const int row = 32 * wj + 16 * mt + g;
        a0[mt] = As[row * GSA + q4 + t];
        a1[mt] = As[(row + 8) * GSA + q4 + t];
      }
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        const int col = 16 * wk + 8 * nt + g;
        const double b = Bs[col * GSA + q4 + t];
        double bj = 0.0;
        if (CPLX) {  // (J R): (b_im, -b_re) per complex entry
          const double v = Bs[col * GSA + q4 + (t ^ 1)];
          bj = (t & 1) ? -v : v;
        }
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          dmma(re[mt][nt], a0[mt], a1[mt], b);
          if (CPLX) dmma(im[mt][nt], a0[mt], a1[mt], bj);
        }
      }
    }
    __syncthreads();
  }
  if (!TMA) cpa_wait<0>();
  // epilogue
  double best = 0.0;
  long long barg = LLONG_MAX;
  double* G = P.ws.G + (long long)q.slot * P.ws.s_G;
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int j = jb * BT + 32 * wj + 16 * mt + g + 8 * (e >> 1);
        const int k = kb * BT + 16 * wk + 8 * nt + 2 * t + (e & 1);
        if (j < k && k < N) {
          const long long p = pair_index(j, k, N);
          const double gr = re[mt][nt][e], gi = CPLX ? im[mt][nt][e] : 0.0;
          if (MODE == 0) {
            const double u = CPLX ? __dadd_rn(__dmul_rn(gr, gr), __dmul_rn(gi, gi)) : __dmul_rn(gr, gr);
            const double xv = q.squared ? u : sqrt(u);
            if (CPLX) {
              *reinterpret_cast<double2*>(G + 2 * p) = make_double2(gr, gi);
            } else {
              G[p] = gr;
            }
            best = fmax(best, xv);
          } else {
            const double m = cas_hypot(gr, gi);  // std::abs = hypot (frame.hpp:87)
            if (m > best || (m == best && m > 0.0 && p < barg)) {
              best = m;
              barg = p;
            }
          }
        }
      }
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    const double ov = __shfl_xor_sync(FULL, best, off);
    const long long oi = __shfl_xor_sync(FULL, barg, off);
    if (ov > best || (ov == best && oi < barg)) {
      best = ov;
      barg = oi;
    }
  }
  if (lane == 0) {
    red_v[warp] = best;
    red_i[warp] = barg;
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
      atomicMax(&P.outs[r].smax, (unsigned long long)__double_as_longlong(v));  // x >= 0: bits order like values
    } else {
      P.ws.tmu[(long long)q.slot * P.ws.s_tile + blockIdx.x] = v;
      P.ws.targ[(long long)q.slot * P.ws.s_tile + blockIdx.x] = ix;
    }
  }
}

// ---------------------------------------------------------------- K3
// w_p = exp((x_p - s)/delta), x_p recomputed from G exactly as K2 formed it;
// the pairs of 16 consecutive rows (a contiguous range) summed over 256 CAS
// lanes (lane l: pairs l, l+256, ... in order), xor butterfly, warp tree.
template <bool CPLX>
__global__ void __launch_bounds__(BZLANES) bde_weights(Pipe P) {
  __shared__ double wt[BZLANES / 32];
  const Shape& sh = P.sh;
  const int r = P.active[blockIdx.y];
  const Req q = P.reqs[r];
  if (P.outs[r].zc != INT_MAX) return;
  const double s = __longlong_as_double((long long)P.outs[r].smax);
  const double cut = __dmul_rn(kUnderflowCut, q.delta);
  const double yd = __drcp_rn(q.delta);
  const bool chk = !(s >= 0x1.0p-800);  // else every nonzero |x - s| >= 2^-854 (Markstein exact)
  const long long N = sh.N;
  const long long r0 = (long long)blockIdx.x * BZROWS, r1 = min(N, r0 + BZROWS);
  const long long p0 = r0 * N - r0 * (r0 + 1) / 2, p1 = r1 * N - r1 * (r1 + 1) / 2;
  const double* G = P.ws.G + (long long)q.slot * P.ws.s_G;
  double* W = P.ws.W + (long long)q.slot * P.ws.s_W;
  double zp = 0.0;
  for (long long p = p0 + threadIdx.x; p < p1; p += 4 * BZLANES) {
    double xv[4], w[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const long long pp = p + u * BZLANES;
      double uu = 0.0;
      if (pp < p1) {
        if (CPLX) {
          const double2 gg = *reinterpret_cast<const double2*>(G + 2 * pp);
          uu = __dadd_rn(__dmul_rn(gg.x, gg.x), __dmul_rn(gg.y, gg.y));
        } else {
          const double gr = G[pp];
          uu = __dmul_rn(gr, gr);
        }
      }
      xv[u] = q.squared ? uu : sqrt(uu);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double diff = __dsub_rn(xv[u], s);
      double y = div_fast(diff, q.delta, yd);
      if (chk && diff < 0.0 && diff > -0x1.0p-900) y = __ddiv_rn(diff, q.delta);
      const double e = cas_exp_core(y);  // the core domain wherever !(diff < cut)
      w[u] = (diff < cut) ? 0.0 : e;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (p + u * BZLANES < p1) {
        W[p + u * BZLANES] = w[u];
        zp = __dadd_rn(zp, w[u]);
      }
    }
  }
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) zp = __dadd_rn(zp, __shfl_xor_sync(FULL, zp, off));
  if ((threadIdx.x & 31) == 0) wt[threadIdx.x >> 5] = zp;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < BZLANES / 32 ? wt[threadIdx.x] : 0.0;
#pragma unroll
    for (int off = 1; off < BZLANES / 32; off <<= 1) v = __dadd_rn(v, __shfl_xor_sync(FULL, v, off));
    if (threadIdx.x == 0) P.ws.zpart[(long long)q.slot * P.ws.s_zpart + blockIdx.x] = v;
  }
}

// ---------------------------------------------------------------- K4
__global__ void bde_zreduce(Pipe P) {
  const int r = P.active[blockIdx.x];
  const Req q = P.reqs[r];
  if (threadIdx.x != 0) return;
  ReqOut& o = P.outs[r];
  if (o.zc != INT_MAX) {
    o.F = __longlong_as_double(0x7ff0000000000000LL);
    o.s = 0.0;
    return;
  }
  const double* zp = P.ws.zpart + (long long)q.slot * P.ws.s_zpart;
  const double s = __longlong_as_double((long long)o.smax);
  double z = zp[0];
  for (int b = 1; b < P.sh.nzb; ++b) z = __dadd_rn(z, zp[b]);
  o.s = s;
  o.z = z;
  o.F = __dadd_rn(s, __dmul_rn(q.delta, cas_log(z)));
}

// ---------------------------------------------------------------- K5
// D^T(m, i) = sum_k P(k, m) phi(i, k) over the k of a CAS chunk (ascending),
// register-blocked on DMMA.  Complex: one accumulator pair per (m, i); A = P^T
// interleaved (pr, pi) per k, read as (pr, pi) for re and (pi, pr) for im;
// B = phi interleaved, (fr, -fi) for re and (fr, fi) for im.  The work is split
// by warp role, so the tensor pipe never waits for the coefficient tiles:
//   * producer warps gather the packed (w, G) of a stage from HBM / L2, form
//     c = w/z, P = c G (conjugated below the diagonal) and c u, store the P^T
//     tile, and stream the phi tile in by 16-byte cp.async one stage ahead;
//     they also carry the t chunk partials sum_k c u (ascending k, plain adds);
//   * consumer warps (WM (m) x WI (i)) run the DMMA loop; accumulators are
//     MT x NT m16n8 tiles per warp (complex d = 128: 16 warps of 16 x 32, 64
//     accumulator registers each, four warps per scheduler).
// NST stage buffers cycle through named barriers (full[b]: producers arrive,
// consumers sync; empty[b]: consumers arrive, producers sync).  A CTA walks
// CPG consecutive CAS chunks of k (grid.z = requests x chunk groups): at a
// chunk end the consumers store that chunk's partial and restart from +0 —
// per output the ascending-k fma chain of its chunk, as before.
template <bool CPLX, int IB>
struct GradWsCfg {
  static constexpr int KK = CPLX ? 16 : 32;
  static constexpr int KP = 32;
  // P^T tile rows: complex 36 doubles (== 4 mod 16: conflict-free fragment loads); real 32 doubles with the
  // column index XOR-swizzled by the row (aswz) — conflict-free for the fragment loads AND for the producers'
  // stores in both tile orientations (lanes along k, or along m: a padded stride is 4-way conflicted there)
  static constexpr int SA = CPLX ? KP + 4 : KP;
  static constexpr int FW = CPLX ? 2 * IB : IB;
  static constexpr int SF = CPLX ? FW + 8 : FW + 4;
  static constexpr int WI = 4;                                 // consumer warps along i
  static constexpr int WM = (CPLX && IB >= 128) ? 4 : 2;       // ... along m
  static constexpr int MT = BT / (16 * WM), NT = IB / (8 * WI);
  static constexpr int SU = KK + 1;  // c u row stride: the t sums read one row per lane (odd: conflict-free)
  static constexpr int A_D = BT * SA, F_D = KK * SF, CU_D = BT * SU;
  static constexpr int NST = 3;
  static constexpr int NPROD = CPLX ? 128 : 256;  // real stages hold twice the k
  static constexpr int NCONS = 32 * WM * WI;
  // real frames (a P element feeds only d MMAs' worth of work): the producers are the critical path, so the
  // t sums move to two warps of their own — they consume the c u tile of a stage like the MMA warps consume
  // the P^T tile (1054 -> 902 us per 108 requests at config 4; gathering (w, G) two stages ahead into a second
  // register set was slower: 1167 us, profiles/r2_bde_grad_ws.txt)
  static constexpr int NTW = CPLX ? 0 : BT;
  static constexpr int NTHR = NPROD + NCONS + NTW;
  static constexpr int NCU = NTW ? NST : 2;  // c u tiles: one per stage buffer when the t warps consume them
  static constexpr size_t smem = (size_t)(NST * (A_D + F_D) + NCU * CU_D) * sizeof(double);
  static constexpr int EPT = BT * KK / NPROD;
};

// XOR swizzle of the real P^T tile: row bits 0-1 into column bits 2-3, row bits 2-3 into column bits 0-1
__device__ __forceinline__ int aswz(int row) { return ((row & 3) << 2) | ((row >> 2) & 3); }

__device__ __forceinline__ void nbar_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void nbar_arrive(int id, int count) {
  asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}

template <bool CPLX, int IB>
__global__ void __launch_bounds__(GradWsCfg<CPLX, IB>::NTHR, 1) bde_grad_ws(Pipe P, int KS) {
  using C = GradWsCfg<CPLX, IB>;
  constexpr int KK = C::KK, SA = C::SA, SF = C::SF, SU = C::SU, FW = C::FW, MT = C::MT, NT = C::NT, EPT = C::EPT, NST = C::NST;
  constexpr int NPROD = C::NPROD, NTHR = C::NTHR, WM = C::WM, WI = C::WI;
  constexpr int BAR_FULL = 1, BAR_EMPTY = 1 + NST, BAR_PROD = 1 + 2 * NST;
  extern __shared__ __align__(16) double smem[];
  double* Abuf = smem;                       // NST x A_D
  double* Fbuf = smem + NST * C::A_D;        // NST x F_D
  double* CUbuf = Fbuf + NST * C::F_D;       // NCU x CU_D
  const Shape& sh = P.sh;
  const int K = sh.K;
  const int r = P.active[blockIdx.z / KS], cg = blockIdx.z % KS;
  const Req q = P.reqs[r];
  if (P.outs[r].zc != INT_MAX) return;
  const int N = sh.N, L = sh.L, d = sh.d;
  const int m0 = blockIdx.x * BT, i0 = blockIdx.y * IB;
  const int CPG = (K + KS - 1) / KS;
  const int ch_lo = cg * CPG, ch_hi = min(K, ch_lo + CPG);
  if (ch_lo >= ch_hi) return;
  const int tid = threadIdx.x;
  const double* phi = P.ws.phi + (long long)q.slot * P.ws.s_phi;
  auto chunk_lo = [&](int ch) { return (int)(((long long)ch * N) / K); };

  if (tid < NPROD) {
    // ======================================================= producers
    const double* Gp = P.ws.G + (long long)q.slot * P.ws.s_G;
    const double* Wp = P.ws.W + (long long)q.slot * P.ws.s_W;
    const double z = P.outs[r].z;
    const double yz = __drcp_rn(z);
    const bool tsum = blockIdx.y == 0 && tid < BT;
    struct RegSet {
      double w[EPT], gr[EPT], gi[EPT];
    };
    RegSet setA;  // the packed (w, G) of the stage to convert next
    auto elem = [&](int k0, int u, int& mm, int& kk) {
      // rows of a stage tile above the diagonal read along m, else along k (coalesced both ways)
      const bool upper = k0 + KK <= m0;
      const int e = tid + NPROD * u;
      mm = upper ? (e & (BT - 1)) : (e / KK);
      kk = upper ? (e / BT) : (e % KK);
    };
    auto gather = [&](int k0, int k_hi, RegSet& R) {
#pragma unroll
      for (int u = 0; u < EPT; ++u) {
        int mm, kk;
        elem(k0, u, mm, kk);
        const int k = k0 + kk, m = m0 + mm;
        double w = 0.0, gr = 0.0, gi = 0.0;
        if (k < k_hi && m < N && k != m) {
          const int lo = min(k, m), hi = max(k, m);
          const int p = lo * N - ((lo * (lo + 1)) >> 1) + (hi - lo - 1);  // pair index: 32 bits up to N = 16384
          w = Wp[p];
          if (CPLX) {  // raw loads only: nothing here waits for the data (the conjugation is applied in convert)
            const double2 gg = *reinterpret_cast<const double2*>(Gp + 2 * p);
            gr = gg.x;
            gi = gg.y;
          } else {
            gr = Gp[p];
          }
        }
        R.w[u] = w;
        R.gr[u] = gr;
        R.gi[u] = gi;
      }
    };
    auto convert = [&](int k0, const RegSet& R, double* As, double* CUs) {
      if constexpr (!CPLX) {
        // real frames hold twice the k per stage and feed half the MMAs per element: the conversion is the
        // producers' critical path, so it is branch-free (the EPT quotient chains interleave); the rare
        // operands the Markstein quotient cannot take (0 < |w| < 2^-900) and the magnitude mode take the
        // general loop below
        bool plain = q.squared != 0;
#pragma unroll
        for (int u = 0; u < EPT; ++u) plain &= !(R.w[u] != 0.0 && fabs(R.w[u]) < 0x1.0p-900);
        if (plain) {
#pragma unroll
          for (int u = 0; u < EPT; ++u) {
            int mm, kk;
            elem(k0, u, mm, kk);
            const double cq = div_fast(R.w[u], z, yz);  // w == 0 -> +0
            const double gr = R.gr[u];
            const double uu = __dmul_rn(gr, gr);
            const bool nz = cq != 0.0;  // an underflowed quotient contributes exact zeros
            As[mm * SA + (kk ^ aswz(mm))] = nz ? __dmul_rn(cq, gr) : 0.0;
            CUs[mm * SU + kk] = nz ? __dmul_rn(cq, uu) : 0.0;
          }
          return;
        }
      }
#pragma unroll
      for (int u = 0; u < EPT; ++u) {
        int mm, kk;
        elem(k0, u, mm, kk);
        double vr = 0.0, vi = 0.0, vu = 0.0;
        const double w = R.w[u];
        if (w != 0.0) {
          const double cq = div_rn(w, z, yz);
          if (cq != 0.0) {
            // G(k, m) = conj(G(m, k)) below the diagonal (k > m: the packed entry is G(m, k))
            const double gr = R.gr[u], gi = (k0 + kk < m0 + mm) ? R.gi[u] : -R.gi[u];
            const double uu = CPLX ? __dadd_rn(__dmul_rn(gr, gr), __dmul_rn(gi, gi)) : __dmul_rn(gr, gr);
            double cc = cq;
            if (!q.squared) cc = __dmul_rn(cc, __ddiv_rn(0.5, fmax(sqrt(uu), 1e-150)));
            vr = __dmul_rn(cc, gr);
            vi = __dmul_rn(cc, gi);
            vu = __dmul_rn(cc, uu);
          }
        }
        if (CPLX) {
          *reinterpret_cast<double2*>(As + mm * SA + 2 * kk) = make_double2(vr, vi);
        } else {
          As[mm * SA + (kk ^ aswz(mm))] = vr;
        }
        CUs[mm * SU + kk] = vu;
      }
    };
    auto issue_phi = [&](int k0, int k_hi, double* Fs) {
      // rows kk: phi column k0 + kk, components [c0, c0 + FW); 16-byte copies (complex: c0, FW, SF, L all even;
      // a real frame with odd d copies 8 bytes at a time)
      const int c0 = CPLX ? 2 * i0 : i0;
      if (CPLX || (L % 2 == 0)) {
        for (int e = tid; e < KK * (FW / 2); e += NPROD) {
          const int kk = e / (FW / 2), c = 2 * (e - kk * (FW / 2));
          const int k = k0 + kk;
          const bool v = k < k_hi && c0 + c < L;
          cpa16(Fs + kk * SF + c, phi + (v ? (long long)k * L + c0 + c : 0), v);
        }
      } else {
        for (int e = tid; e < KK * FW; e += NPROD) {
          const int kk = e / FW, c = e - kk * FW;
          const int k = k0 + kk;
          const bool v = k < k_hi && c0 + c < L;
          cpa8(Fs + kk * SF + c, phi + (v ? (long long)k * L + c0 + c : 0), v);
        }
      }
    };
    // stage iterator over the chunks of this CTA
    struct It {
      int ch, s;
    };
    auto nst_of = [&](int ch) { return (chunk_lo(ch + 1) - chunk_lo(ch) + KK - 1) / KK; };
    auto advance = [&](It it) {
      ++it.s;
      if (it.s >= nst_of(it.ch)) {
        ++it.ch;
        it.s = 0;
      }
      return it;
    };
    auto valid = [&](It it) { return it.ch < ch_hi; };
    auto k0_of = [&](It it) { return chunk_lo(it.ch) + it.s * KK; };
    auto khi_of = [&](It it) { return chunk_lo(it.ch + 1); };
    // prologue: the first stage's phi tile and packed (w, G) in flight
    It cur{ch_lo, 0};
    issue_phi(k0_of(cur), khi_of(cur), Fbuf);
    cpa_commit();
    gather(k0_of(cur), khi_of(cur), setA);
    double tacc = 0.0;
    for (int gs = 0; valid(cur); ++gs) {
      const It n1 = advance(cur);
      const int k0 = k0_of(cur), k_hi = khi_of(cur);
      const int b = gs % NST, b2 = (gs + 1) % NST;
      const bool more = valid(n1);
      auto stage = [&](RegSet& R) {
        // the next stage's phi tile streams in while this stage is converted
        if (more) {
          if (gs + 1 >= NST) nbar_sync(BAR_EMPTY + b2, NTHR);  // its readers are done with buffer b2
          issue_phi(k0_of(n1), khi_of(n1), Fbuf + b2 * C::F_D);
        }
        cpa_commit();
        double* CUs = CUbuf + (C::NTW ? b : (gs & 1)) * C::CU_D;
        convert(k0, R, Abuf + b * C::A_D, CUs);
        cpa_wait<1>();  // this stage's phi tile (committed one iteration ago) has landed
        __threadfence_block();
        nbar_arrive(BAR_FULL + b, NTHR);
        if (more) gather(k0_of(n1), khi_of(n1), R);  // the next stage's (w, G): lands during the MMAs
        if constexpr (C::NTW == 0) {
          nbar_sync(BAR_PROD, NPROD);  // CUs complete (and the previous stage's t sums read)
          if (tsum) {  // t chunk partial: ascending k, plain adds (c u of this stage); loads first, then the chain
            const int kmax = min(KK, k_hi - k0);
            double cu[KK];
#pragma unroll
            for (int kk = 0; kk < KK; ++kk) cu[kk] = CUs[tid * SU + kk];
#pragma unroll
            for (int kk = 0; kk < KK; ++kk)
              if (kk < kmax) tacc = __dadd_rn(tacc, cu[kk]);
          }
        }
      };
      stage(setA);
      if constexpr (C::NTW == 0) {
        if (!more || n1.ch != cur.ch) {  // chunk end
          if (tsum && m0 + tid < N)
            P.ws.tpart[(long long)q.slot * P.ws.s_tpart + (long long)cur.ch * N + m0 + tid] = tacc;
          tacc = 0.0;
        }
      }
      cur = n1;
    }
    cpa_wait<0>();
  } else if (C::NTW > 0 && tid >= NPROD + C::NCONS) {
    // ======================================================= t warps (real frames)
    // t_m = sum_k c u over each chunk, ascending k, plain adds: thread ttid owns row m0 + ttid and consumes the
    // c u tile of every stage buffer like the MMA warps consume the P^T tile
    const int ttid = tid - NPROD - C::NCONS;
    const bool tsum = blockIdx.y == 0;
    int gs = 0;
    for (int ch = ch_lo; ch < ch_hi; ++ch) {
      const int k_lo = chunk_lo(ch), k_hi = chunk_lo(ch + 1);
      const int nst = (k_hi - k_lo + KK - 1) / KK;
      double tacc = 0.0;
      for (int s = 0; s < nst; ++s, ++gs) {
        const int b = gs % NST;
        nbar_sync(BAR_FULL + b, NTHR);
        if (tsum) {
          const double* CUs = CUbuf + b * C::CU_D;
          const int kmax = min(KK, k_hi - (k_lo + s * KK));
          double cu[KK];
#pragma unroll
          for (int kk = 0; kk < KK; ++kk) cu[kk] = CUs[ttid * SU + kk];
#pragma unroll
          for (int kk = 0; kk < KK; ++kk)
            if (kk < kmax) tacc = __dadd_rn(tacc, cu[kk]);
        }
        nbar_arrive(BAR_EMPTY + b, NTHR);
      }
      if (tsum && m0 + ttid < N) P.ws.tpart[(long long)q.slot * P.ws.s_tpart + (long long)ch * N + m0 + ttid] = tacc;
    }
  } else {
    // ======================================================= consumers
    const int ctid = tid - NPROD, lane = ctid & 31, warp = ctid >> 5;
    const int g = lane >> 2, t = lane & 3;
    const int wm = warp / WI, wi = warp % WI;
    const int rbase = (BT / WM) * wm, cbase = (IB / WI) * wi;
    double re[MT][NT][4], im[MT][NT][4];
    int gs = 0;
    for (int ch = ch_lo; ch < ch_hi; ++ch) {
      const int k_lo = chunk_lo(ch), k_hi = chunk_lo(ch + 1);
      const int nst = (k_hi - k_lo + KK - 1) / KK;
#pragma unroll
      for (int a = 0; a < MT; ++a)
#pragma unroll
        for (int b2 = 0; b2 < NT; ++b2)
#pragma unroll
          for (int e = 0; e < 4; ++e) re[a][b2][e] = im[a][b2][e] = 0.0;
      for (int s = 0; s < nst; ++s, ++gs) {
        const int b = gs % NST;
        nbar_sync(BAR_FULL + b, NTHR);
        const double* As = Abuf + b * C::A_D;
        const double* Fs = Fbuf + b * C::F_D;
#pragma unroll 2
        for (int q4 = 0; q4 < C::KP; q4 += 4) {
          double ar0[MT], ar1[MT], ai0[MT], ai1[MT];
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) {
            const int row = rbase + 16 * mt + g;
            if (CPLX) {
              ar0[mt] = As[row * SA + q4 + t];
              ar1[mt] = As[(row + 8) * SA + q4 + t];
            } else {
              ar0[mt] = As[row * SA + ((q4 + t) ^ aswz(row))];
              ar1[mt] = As[(row + 8) * SA + ((q4 + t) ^ aswz(row + 8))];
            }
            if (CPLX) {
              ai0[mt] = As[row * SA + q4 + (t ^ 1)];
              ai1[mt] = As[(row + 8) * SA + q4 + (t ^ 1)];
            }
          }
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            const int col = cbase + 8 * nt + g;  // i within the block
            double br, bi = 0.0;
            if (CPLX) {
              const int qq = q4 + t;  // interleaved K': k = qq / 2, component qq & 1
              const double v = Fs[(qq >> 1) * SF + 2 * col + (qq & 1)];
              br = (qq & 1) ? -v : v;
              bi = v;
            } else {
              br = Fs[(q4 + t) * SF + col];
            }
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) {
              dmma(re[mt][nt], ar0[mt], ar1[mt], br);
              if (CPLX) dmma(im[mt][nt], ai0[mt], ai1[mt], bi);
            }
          }
        }
        nbar_arrive(BAR_EMPTY + b, NTHR);
      }
      // ---- this chunk's partial, point layout.  (Folding the chunk partials left to right into one array
      // here — a read-modify-write at every chunk end — was measured: finalize 117 -> 61 us but this kernel
      // 5580 -> 6067 us per 8 config-5 requests; the K partials stay separate.)
      double* part = P.ws.part + (long long)q.slot * P.ws.s_part + (long long)ch * sh.dim;
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int m = m0 + rbase + 16 * mt + g + 8 * h;
            const int i = i0 + cbase + 8 * nt + 2 * t;
            if (m >= N) continue;
            if (CPLX) {
              double* o = part + (long long)m * L + 2 * i;  // 16-byte aligned (L and 2i even)
              if (i < d) *reinterpret_cast<double2*>(o) = make_double2(re[mt][nt][2 * h], im[mt][nt][2 * h]);
              if (i + 1 < d)
                *reinterpret_cast<double2*>(o + 2) = make_double2(re[mt][nt][2 * h + 1], im[mt][nt][2 * h + 1]);
            } else {
              double* o = part + (long long)m * L + i;
              if (i < d) o[0] = re[mt][nt][2 * h];
              if (i + 1 < d) o[1] = re[mt][nt][2 * h + 1];
            }
          }
    }
  }
}

// ---------------------------------------------------------------- K6
__global__ void bde_finalize(Pipe P) {
  const Shape& sh = P.sh;
  const int r = P.active[blockIdx.y];
  const Req q = P.reqs[r];
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= sh.dim) return;
  if (P.outs[r].zc != INT_MAX) {
    q.grad[e] = 0.0;
    return;
  }
  const int m = (int)(e / sh.L);
  const double* part = P.ws.part + (long long)q.slot * P.ws.s_part;
  const double* tpart = P.ws.tpart + (long long)q.slot * P.ws.s_tpart;
  double a = part[e], tt = tpart[m];
  for (int ch = 1; ch < sh.K; ++ch) {
    a = __dadd_rn(a, part[(long long)ch * sh.dim + e]);
    tt = __dadd_rn(tt, tpart[(long long)ch * sh.N + m]);
  }
  const double ph = P.ws.phi[(long long)q.slot * P.ws.s_phi + e];
  const double alpha = P.ws.alpha[(long long)q.slot * P.ws.s_alpha + m];
  q.grad[e] = __dmul_rn(__ddiv_rn(__dsub_rn(a, __dmul_rn(tt, ph)), alpha), 2.0);
}

// softmax weights c_p = w_p / z (ObjectiveEval::softmax_weights), when asked
__global__ void bde_wout(Pipe P) {
  const int r = P.active[blockIdx.y];
  const Req q = P.reqs[r];
  if (!q.wout) return;
  const long long n = P.sh.n;
  const bool zc = P.outs[r].zc != INT_MAX;
  const double z = P.outs[r].z, yz = __drcp_rn(z);
  const double* W = P.ws.W + (long long)q.slot * P.ws.s_W;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x) {
    const double w = zc ? 0.0 : W[p];
    q.wout[p] = (w == 0.0) ? 0.0 : div_rn(w, z, yz);
  }
}

// coherence: the tile maxima in (mu desc, pair asc) order
__global__ void bde_coh_reduce(Pipe P) {
  __shared__ double sv[256];
  __shared__ long long si[256];
  const int r = P.active[blockIdx.x];
  const Req q = P.reqs[r];
  ReqOut& o = P.outs[r];
  const double* tm = P.ws.tmu + (long long)q.slot * P.ws.s_tile;
  const long long* ta = P.ws.targ + (long long)q.slot * P.ws.s_tile;
  double best = 0.0;
  long long arg = LLONG_MAX;
  for (int tt = threadIdx.x; tt < P.sh.tiles; tt += blockDim.x) {
    const double v = tm[tt];
    const long long a = ta[tt];
    if (v > best || (v == best && v > 0.0 && a < arg)) {
      best = v;
      arg = a;
    }
  }
  sv[threadIdx.x] = best;
  si[threadIdx.x] = arg;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int u = 1; u < (int)blockDim.x; ++u)
      if (sv[u] > best || (sv[u] == best && sv[u] > 0.0 && si[u] < arg)) {
        best = sv[u];
        arg = si[u];
      }
    const bool bad = q.kind == REQ_COH_NORM && o.zc != INT_MAX;
    o.mu = bad ? 0.0 : best;
    o.argmax = bad || arg == LLONG_MAX ? -1 : arg;
  }
}

}  // namespace trstmi_bde
