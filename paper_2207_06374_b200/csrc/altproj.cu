// Alternating-projection baseline on the GPU: the reference's comparison method,
// /root/reference/proj/include/trstmi/baseline.hpp:68-167 (alternating_projection) — projections of the Gram matrix
// between the structural set (unit diagonal, off-diagonal magnitudes clipped to mu_target, phases kept) and the
// PSD matrices of rank <= d — batched over restarts: one CTA per restart, its N x N complex matrices (Gram,
// rotated copy, eigenvectors, projection) in an L2-resident workspace.
//
// The Hermitian eigendecomposition the reference delegates to Eigen::SelfAdjointEigenSolver (baseline.hpp:110) is a
// two-sided cyclic Jacobi method in round-robin order: the N/2 disjoint rotations of a round are formed from the
// matrix at the start of the round by N/2 threads, then the whole CTA applies them to the columns of W and V and to
// the rows of W.  Every arithmetic step is one rounding in the order oracle/altproj_oracle.hpp states it (this file
// is compiled with -fmad=false), so frames, coherences and iteration counts equal the CPU oracle's bit for bit.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <vector>

#include "../../include/trstmi_b200.h"
#include "small_path.cuh"

namespace {

using namespace trstmi_dev;

constexpr int kApThreads = 256;
constexpr int kApMaxN = 256;
constexpr int kJacobiMaxSweeps = 60;
constexpr double kJacobiRelTol2 = 1e-30;

struct ApArgs {
  int d, N, max_iters;
  double mu_target, tol;
  const double* starts;  // restarts x 2dN
  double* frames;        // restarts x 2dN
  double* coherence;     // restarts
  int* iterations;       // restarts: +converged / -best-seen (StageRecord::outer_iterations)
  int* sweeps;           // restarts (nullable)
  double* ws;            // restarts x ws_stride doubles
  long long ws_stride;
};

__device__ __forceinline__ double ap_block_max(double v, double* red) {
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) v = fmax(v, __shfl_xor_sync(FULL, v, off));
  __syncthreads();  // red may still be read from the previous reduction
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double m = red[0];
#pragma unroll
  for (int w = 1; w < kApThreads / 32; ++w) m = fmax(m, red[w]);
  return m;
}

// mu of a frame with unit columns: max over j < k of |<f_j, f_k>| (coherence, frame.hpp:138-145; CAS Gram entry, hypot)
__device__ double ap_coherence(const double* __restrict__ f, int d, int N, double* red) {
  const int L = 2 * d;
  double best = 0.0;
  for (long long e = threadIdx.x; e < (long long)N * N; e += kApThreads) {
    const int j = (int)(e / N), k = (int)(e - (long long)j * N);
    if (j >= k) continue;
    double re = 0.0, im = 0.0;
    for (int i = 0; i < d; ++i) {
      const double ar = f[j * L + 2 * i], ai = f[j * L + 2 * i + 1];
      const double br = f[k * L + 2 * i], bi = f[k * L + 2 * i + 1];
      re = fma(ar, br, re);
      re = fma(ai, bi, re);
      im = fma(ar, bi, im);
      im = fma(-ai, br, im);
    }
    best = fmax(best, cas_hypot(re, im));
  }
  return ap_block_max(best, red);
}

__global__ void __launch_bounds__(kApThreads) altproj_kernel(const ApArgs A) {
  const int d = A.d, N = A.N, L = 2 * d, dim = L * N;
  const int M = (N + 1) & ~1, H = M / 2;
  const int tid = threadIdx.x;
  const long long NN = (long long)N * N;
  double* G = A.ws + (long long)blockIdx.x * A.ws_stride;
  double* W = G + 2 * NN;
  double* V = W + 2 * NN;
  double* Pm = V + 2 * NN;
  double* fac = Pm + 2 * NN;
  double* last = fac + dim;
  double* best = last + dim;
  double* nrm = best + dim;  // N
  const double* start = A.starts + (long long)blockIdx.x * dim;
  __shared__ double red[kApThreads / 32];
  __shared__ double rc[kApMaxN / 2], rsr[kApMaxN / 2], rsi[kApMaxN / 2];
  __shared__ int rp[kApMaxN / 2], rq[kApMaxN / 2];
  __shared__ int top[kApMaxN];
  __shared__ int s_zero;

  // gram_matrix(current) (frame.hpp:73-75) and the start as best / last iterate
  for (int i = tid; i < dim; i += kApThreads) best[i] = last[i] = start[i];
  for (long long e = tid; e < NN; e += kApThreads) {
    const int j = (int)(e / N), k = (int)(e - (long long)j * N);
    if (j > k) continue;
    double re = 0.0, im = 0.0;
    for (int i = 0; i < d; ++i) {
      const double ar = start[j * L + 2 * i], ai = start[j * L + 2 * i + 1];
      const double br = start[k * L + 2 * i], bi = start[k * L + 2 * i + 1];
      re = fma(ar, br, re);
      re = fma(ai, bi, re);
      im = fma(ar, bi, im);
      im = fma(-ai, br, im);
    }
    if (j == k) im = 0.0;
    G[2 * ((long long)j * N + k)] = re;
    G[2 * ((long long)j * N + k) + 1] = im;
    G[2 * ((long long)k * N + j)] = re;
    G[2 * ((long long)k * N + j) + 1] = -im;
  }
  double best_mu = ap_coherence(start, d, N, red), last_mu = best_mu;
  bool converged = false;
  int iterations = 0, total_sweeps = 0;

  for (int it = 0; it < A.max_iters; ++it) {
    iterations = it + 1;
    // (a) structural projection (baseline.hpp:96-106); W <- the projected Gram, V <- I
    __syncthreads();
    for (long long e = tid; e < NN; e += kApThreads) {
      const int j = (int)(e / N), k = (int)(e - (long long)j * N);
      if (j > k) continue;
      double re = G[2 * e], im = G[2 * e + 1];
      if (j == k) {
        re = 1.0;
        im = 0.0;
      } else {
        const double mag = cas_hypot(re, im);
        if (mag > A.mu_target) {
          const double f = A.mu_target / mag;
          re *= f;
          im *= f;
        } else {  // untouched entries keep both stored halves (they are conjugates by construction)
          re = G[2 * e];
          im = G[2 * e + 1];
        }
      }
      const long long et = (long long)k * N + j;
      G[2 * e] = W[2 * e] = re;
      G[2 * e + 1] = W[2 * e + 1] = im;
      G[2 * et] = W[2 * et] = re;
      G[2 * et + 1] = W[2 * et + 1] = j == k ? 0.0 : -im;
    }
    for (long long e = tid; e < NN; e += kApThreads) {
      V[2 * e] = (e / N == e % N) ? 1.0 : 0.0;
      V[2 * e + 1] = 0.0;
    }
    __syncthreads();

    // (b) eigendecomposition: cyclic Jacobi, round-robin order
    for (int sweep = 0; sweep < kJacobiMaxSweeps; ++sweep) {
      double off2 = 0.0, diag2 = 0.0;
      for (long long e = tid; e < NN; e += kApThreads) {
        const double m2 = W[2 * e] * W[2 * e] + W[2 * e + 1] * W[2 * e + 1];
        if (e / N == e % N)
          diag2 = fmax(diag2, m2);
        else
          off2 = fmax(off2, m2);
      }
      off2 = ap_block_max(off2, red);
      diag2 = ap_block_max(diag2, red);
      if (off2 <= kJacobiRelTol2 * diag2) break;
      ++total_sweeps;
      for (int r = 0; r < M - 1; ++r) {
        if (tid < H) {
          const int i = tid;
          const int a = i == 0 ? M - 1 : (r + i) % (M - 1);
          const int b = i == 0 ? r : (r + M - 1 - i) % (M - 1);
          const int p = min(a, b), q = max(a, b);
          double c = 1.0, sr = 0.0, si = 0.0;
          if (q < N) {
            const double re = W[2 * ((long long)p * N + q)], im = W[2 * ((long long)p * N + q) + 1];
            const double bm = sqrt(re * re + im * im);
            if (bm != 0.0) {
              const double tau = (W[2 * ((long long)q * N + q)] - W[2 * ((long long)p * N + p)]) / (2.0 * bm);
              const double t = (tau < 0.0 ? -1.0 : 1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
              c = 1.0 / sqrt(1.0 + t * t);
              const double s = t * c;
              sr = s * (re / bm);
              si = s * (im / bm);
            }
          }
          rp[i] = p;
          rq[i] = (q < N && (sr != 0.0 || si != 0.0)) ? q : -1;
          rc[i] = c;
          rsr[i] = sr;
          rsi[i] = si;
        }
        __syncthreads();
        // columns p, q of W and V
        for (int item = tid; item < H * 2 * N; item += kApThreads) {
          const int i = item / (2 * N);
          const int rem = item - i * 2 * N;
          const int q = rq[i];
          if (q < 0) continue;
          const int p = rp[i];
          double* Mx = rem >= N ? V : W;
          const int row = rem >= N ? rem - N : rem;
          double* x = Mx + 2 * ((long long)row * N + p);
          double* y = Mx + 2 * ((long long)row * N + q);
          const double c = rc[i], sr = rsr[i], si = rsi[i];
          const double xr = x[0], xi = x[1], yr = y[0], yi = y[1];
          x[0] = (xr * c - yr * sr) - yi * si;
          x[1] = (xi * c + yr * si) - yi * sr;
          y[0] = (xr * sr - xi * si) + yr * c;
          y[1] = (xr * si + xi * sr) + yi * c;
        }
        __syncthreads();
        // rows p, q of W
        for (int item = tid; item < H * N; item += kApThreads) {
          const int i = item / N;
          const int col = item - i * N;
          const int q = rq[i];
          if (q < 0) continue;
          const int p = rp[i];
          double* x = W + 2 * ((long long)p * N + col);
          double* y = W + 2 * ((long long)q * N + col);
          const double c = rc[i], sr = rsr[i], si = rsi[i];
          const double xr = x[0], xi = x[1], yr = y[0], yi = y[1];
          x[0] = (c * xr - sr * yr) + si * yi;
          x[1] = (c * xi - sr * yi) - si * yr;
          y[0] = (sr * xr + si * xi) + c * yr;
          y[1] = (sr * xi - si * xr) + c * yi;
        }
        __syncthreads();
        if (tid < H && rq[tid] >= 0) {
          const int p = rp[tid], q = rq[tid];
          W[2 * ((long long)p * N + q)] = W[2 * ((long long)p * N + q) + 1] = 0.0;
          W[2 * ((long long)q * N + p)] = W[2 * ((long long)q * N + p) + 1] = 0.0;
          W[2 * ((long long)p * N + p) + 1] = 0.0;
          W[2 * ((long long)q * N + q) + 1] = 0.0;
        }
        __syncthreads();
      }
    }
    // the d largest eigenvalues, ties by the lower index (a stable descending sort)
    for (int e = tid; e < N; e += kApThreads) {
      const double le = W[2 * ((long long)e * N + e)];
      int rank = 0;
      for (int f = 0; f < N; ++f) {
        const double lf = W[2 * ((long long)f * N + f)];
        rank += (lf > le || (lf == le && f < e)) ? 1 : 0;
      }
      if (rank < d) top[rank] = e;
    }
    if (tid == 0) s_zero = 0;
    __syncthreads();
    // projected = sum lambda v v^* (baseline.hpp:112-118), factor rows sqrt(lambda) v^* (:119-120)
    for (long long e = tid; e < NN; e += kApThreads) {
      const int j = (int)(e / N), k = (int)(e - (long long)j * N);
      if (j > k) continue;
      double ar = 0.0, ai = 0.0;
      for (int i = 0; i < d; ++i) {
        const int ev = top[i];
        const double lam = fmax(W[2 * ((long long)ev * N + ev)], 0.0);
        const double vjr = V[2 * ((long long)j * N + ev)], vji = V[2 * ((long long)j * N + ev) + 1];
        const double vkr = V[2 * ((long long)k * N + ev)], vki = V[2 * ((long long)k * N + ev) + 1];
        const double pr = vjr * vkr + vji * vki;
        const double pi = vji * vkr - vjr * vki;
        ar = ar + lam * pr;
        ai = ai + lam * pi;
      }
      const long long et = (long long)k * N + j;
      Pm[2 * e] = ar;
      Pm[2 * e + 1] = ai;
      Pm[2 * et] = ar;
      Pm[2 * et + 1] = -ai;
    }
    for (int e = tid; e < d * N; e += kApThreads) {
      const int i = e / N, j = e - i * N;
      const int ev = top[i];
      const double sl = sqrt(fmax(W[2 * ((long long)ev * N + ev)], 0.0));
      fac[j * L + 2 * i] = sl * V[2 * ((long long)j * N + ev)];
      fac[j * L + 2 * i + 1] = sl * (-V[2 * ((long long)j * N + ev) + 1]);
    }
    __syncthreads();
    // normalize_columns (frame.hpp:60-69) + coherence (baseline.hpp:123-132); a zero column skips the update
    for (int j = tid; j < N; j += kApThreads) {
      double acc = 0.0;
      for (int q = 0; q < L; ++q) acc = fma(fac[j * L + q], fac[j * L + q], acc);
      const double a = sqrt(acc);
      nrm[j] = a;
      if (a < kZeroColumnTol) s_zero = 1;
    }
    __syncthreads();
    const bool zero = s_zero != 0;
    double change = 0.0;
    for (long long e = tid; e < NN; e += kApThreads)
      change = fmax(change, cas_hypot(Pm[2 * e] - G[2 * e], Pm[2 * e + 1] - G[2 * e + 1]));
    change = ap_block_max(change, red);
    if (!zero) {
      for (int i = tid; i < dim; i += kApThreads) fac[i] = fac[i] / nrm[i / L];
      __syncthreads();
      const double mu = ap_coherence(fac, d, N, red);
      for (int i = tid; i < dim; i += kApThreads) last[i] = fac[i];
      last_mu = mu;
      if (last_mu < best_mu) {
        best_mu = last_mu;
        for (int i = tid; i < dim; i += kApThreads) best[i] = fac[i];
      }
    }
    __syncthreads();
    for (long long e = tid; e < 2 * NN; e += kApThreads) G[e] = Pm[e];
    if (change <= A.tol) {
      converged = true;
      break;
    }
  }
  __syncthreads();
  const double* res = converged ? last : best;
  double* out = A.frames + (long long)blockIdx.x * dim;
  for (int i = tid; i < dim; i += kApThreads) out[i] = res[i];
  if (tid == 0) {
    A.coherence[blockIdx.x] = converged ? last_mu : best_mu;
    A.iterations[blockIdx.x] = converged ? iterations : -iterations;
    if (A.sweeps) A.sweeps[blockIdx.x] = total_sweeps;
  }
}

struct DevMem {
  void* p = nullptr;
  ~DevMem() {
    if (p) cudaFree(p);
  }
};

}  // namespace

extern "C" int trstmi_altproj_batch(int64_t d, int64_t N, int32_t max_iters, double mu_target, double tol,
                                    int64_t restarts, const double* starts, double* frames, double* coherence,
                                    int32_t* iterations, int32_t* sweeps) {
  // validation as alternating_projection (baseline.hpp:72-82)
  if (d < 1 || N < 1 || d > N || max_iters < 1 || restarts < 0 || N > kApMaxN) return TRSTMI_ERR_INVALID_ARG;
  if (!starts || !frames || !coherence || !iterations) return TRSTMI_ERR_INVALID_ARG;
  const double welch = N > d ? std::sqrt((double)(N - d) / ((double)d * (double)(N - 1))) : 0.0;  // analysis.hpp:27-31
  const double target = mu_target > 0.0 ? mu_target : std::max(welch, 1e-12);
  if (target >= 1.0) return TRSTMI_ERR_INVALID_ARG;
  if (restarts == 0) return TRSTMI_OK;
  const long long dim = 2 * d * N, NN = (long long)N * N;
  const long long stride = 8 * NN + 3 * dim + N;
  DevMem ds, df, dc, di, dsw, dws;
  const size_t fb = (size_t)restarts * dim * sizeof(double);
  if (cudaMalloc(&ds.p, fb) != cudaSuccess || cudaMalloc(&df.p, fb) != cudaSuccess ||
      cudaMalloc(&dc.p, restarts * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&di.p, restarts * sizeof(int)) != cudaSuccess ||
      cudaMalloc(&dsw.p, restarts * sizeof(int)) != cudaSuccess ||
      cudaMalloc(&dws.p, (size_t)restarts * stride * sizeof(double)) != cudaSuccess)
    return TRSTMI_ERR_CUDA;
  if (cudaMemcpy(ds.p, starts, fb, cudaMemcpyHostToDevice) != cudaSuccess) return TRSTMI_ERR_CUDA;
  ApArgs A;
  A.d = (int)d;
  A.N = (int)N;
  A.max_iters = max_iters;
  A.mu_target = target;
  A.tol = tol;
  A.starts = (const double*)ds.p;
  A.frames = (double*)df.p;
  A.coherence = (double*)dc.p;
  A.iterations = (int*)di.p;
  A.sweeps = (int*)dsw.p;
  A.ws = (double*)dws.p;
  A.ws_stride = stride;
  altproj_kernel<<<(unsigned)restarts, kApThreads>>>(A);
  if (cudaGetLastError() != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) return TRSTMI_ERR_CUDA;
  if (cudaMemcpy(frames, df.p, fb, cudaMemcpyDeviceToHost) != cudaSuccess ||
      cudaMemcpy(coherence, dc.p, restarts * sizeof(double), cudaMemcpyDeviceToHost) != cudaSuccess ||
      cudaMemcpy(iterations, di.p, restarts * sizeof(int), cudaMemcpyDeviceToHost) != cudaSuccess)
    return TRSTMI_ERR_CUDA;
  if (sweeps && cudaMemcpy(sweeps, dsw.p, restarts * sizeof(int), cudaMemcpyDeviceToHost) != cudaSuccess)
    return TRSTMI_ERR_CUDA;
  return TRSTMI_OK;
}
