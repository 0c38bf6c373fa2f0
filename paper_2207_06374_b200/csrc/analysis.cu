// Post-solve analysis on the GPU: the quantities the
// reference's run records and certificates are built from, at any N.
//
//   trstmi_offdiag_magnitudes  offdiagonal_magnitudes  frame.hpp:80-91
//                              (row-major upper-triangular |G(j,k)|), optional
//                              ascending device sort for the angle spectrum
//   trstmi_cluster_sorted      cluster_magnitudes      frame.hpp:96-118
//                              (sequential, host: the reference's sum order)
//   trstmi_frame_operator_deviation  check_tight     analysis.hpp:76-84
//                              (max |Phi Phi* - (N/d) I| entry)
//   trstmi_distortion_mc       distortion_mc           beamforming.hpp:78-163
//                              (Monte-Carlo quantisation distortion of a codebook:
//                              one warp per 4096-sample block, the block's own
//                              SplitMix64 stream, codeword overlaps across lanes)
//
// |z| = sqrt(re*re + im*im) throughout (the CAS coherence, DESIGN.md §3 item
// 10; the reference's std::abs is hypot — at most an ulp apart, far inside
// any certificate tolerance).  Gram entries and frame-operator entries are
// fma chains in ascending index (the CAS order).
#include <cuda_runtime.h>
#include <thrust/device_ptr.h>
#include <thrust/execution_policy.h>
#include <thrust/sort.h>

#include <algorithm>
#include <climits>
#include <cstdint>
#include <cstring>
#include <cmath>
#include <string>
#include <vector>

#include "../../include/trstmi_b200.h"
#include "small_path.cuh"

namespace {

using namespace trstmi_dev;

// columns of a frame normalised in place (normalize_columns, frame.hpp:60-69);
// the first zero column goes to *zero_col
__global__ void an_normalize(double* f, int L, int N, int* zero_col) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= N) return;
  double* col = f + (long long)j * L;
  double acc = 0.0;
  for (int q = 0; q < L; ++q) acc = fma(col[q], col[q], acc);
  const double a = sqrt(acc);
  if (a < kZeroColumnTol) {
    atomicMin(zero_col, j);
    return;
  }
  const double ya = __drcp_rn(a);
  for (int q = 0; q < L; ++q) col[q] = div_rn(col[q], a, ya);
}

// |G(j,k)| for every pair, row-major upper-triangular index p; thread per pair
__global__ void an_magnitudes(const double* __restrict__ f, int cplx, int d, int N, long long n, double* mags) {
  const int L = cplx ? 2 * d : d;
  const double b = 2.0 * N - 1.0;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x) {
    long long j = (long long)floor(0.5 * (b - sqrt(fmax(b * b - 8.0 * (double)p, 0.0))));
    j = max(0LL, min(j, (long long)N - 2));
    while (j < N - 2 && (j + 1) * N - (j + 1) * (j + 2) / 2 <= p) ++j;
    while (j > 0 && j * N - j * (j + 1) / 2 > p) --j;
    const long long k = p - (j * N - j * (j + 1) / 2) + j + 1;
    const double* a = f + j * L;
    const double* c = f + k * L;
    double re = 0.0, im = 0.0;
    if (cplx) {
      for (int i = 0; i < d; ++i) {
        const double ar = a[2 * i], ai = a[2 * i + 1], br = c[2 * i], bi = c[2 * i + 1];
        re = fma(ar, br, re);
        re = fma(ai, bi, re);
        im = fma(ar, bi, im);
        im = fma(-ai, br, im);
      }
    } else {
      for (int i = 0; i < d; ++i) re = fma(a[i], c[i], re);
    }
    mags[p] = cas_hypot(re, im);  // std::abs = hypot (frame.hpp:87)
  }
}

// max |(Phi Phi*)(r,s) - (N/d) delta_rs| over the d x d frame operator; entry
// (r,s) = sum_j phi(r,j) conj(phi(s,j)), ascending j
__global__ void an_frame_operator(const double* __restrict__ f, int cplx, int d, int N,
                                  unsigned long long* dev_bits) {
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  double m = 0.0;
  if (e < (long long)d * d) {
    const int r = (int)(e / d), s = (int)(e - (long long)r * d);
    const int L = cplx ? 2 * d : d;
    double re = 0.0, im = 0.0;
    for (int j = 0; j < N; ++j) {
      const double* col = f + (long long)j * L;
      if (cplx) {
        const double ar = col[2 * r], ai = col[2 * r + 1], br = col[2 * s], bi = col[2 * s + 1];
        re = fma(ar, br, re);
        re = fma(ai, bi, re);
        im = fma(ai, br, im);
        im = fma(-ar, bi, im);
      } else {
        re = fma(col[r], col[s], re);
      }
    }
    if (r == s) re = __dsub_rn(re, (double)N / (double)d);
    m = cas_hypot(re, im);
  }
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, off));
  if ((threadIdx.x & 31) == 0) atomicMax(dev_bits, (unsigned long long)__double_as_longlong(m));
}

// SplitMix64 (rng.hpp:13-64) on the device: the integer stream is exact; the
// Box-Muller normals use CUDA's log/sqrt/sin/cos, within an ulp or two of glibc.
struct DevRng {
  unsigned long long state;
  bool has_spare;
  double spare;
  __device__ unsigned long long next_u64() {
    unsigned long long z = (state += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
  }
  __device__ double uniform() { return (double)(next_u64() >> 11) * 0x1.0p-53; }
  __device__ double normal() {
    if (has_spare) {
      has_spare = false;
      return spare;
    }
    double u1 = uniform();
    if (u1 <= 0.0) u1 = 0x1.0p-53;
    const double u2 = uniform();
    const double r = sqrt(__dmul_rn(-2.0, log(u1)));
    const double theta = __dmul_rn(2.0 * 3.14159265358979323846, u2);
    spare = __dmul_rn(r, sin(theta));
    has_spare = true;
    return __dmul_rn(r, cos(theta));
  }
};

__device__ __forceinline__ unsigned long long dev_mix_seed(unsigned long long seed, unsigned long long index) {
  unsigned long long z = seed + (index + 1) * 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

constexpr unsigned long long kDistortionBlock = 4096;  // beamforming.hpp:61

// one warp per block b: lane 0 draws h (d complex normals, rejection as the
// reference), every lane scores codewords lane, lane+32, ... (|<phi_i, h>|^2,
// ascending-index fma chain), warp max, lane 0 accumulates the block moments
// sequentially (sum, sum of squares) like distortion_block.
__global__ void an_distortion(const double* __restrict__ book, int d, int N, unsigned long long samples,
                              unsigned long long seed, double* __restrict__ moments) {
  extern __shared__ double hs[];  // 2d per warp
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const unsigned long long b = (unsigned long long)blockIdx.x * (blockDim.x >> 5) + wib;
  const unsigned long long nblocks = (samples + kDistortionBlock - 1) / kDistortionBlock;
  if (b >= nblocks) return;
  double* h = hs + (size_t)wib * 2 * d;
  const unsigned long long start = b * kDistortionBlock;
  const unsigned long long count = min(kDistortionBlock, samples - start);
  DevRng rng{dev_mix_seed(seed, b), false, 0.0};
  double sum = 0.0, sum_sq = 0.0;
  for (unsigned long long s = 0; s < count; ++s) {
    double norm_sq = 0.0;
    if (lane == 0) {
      do {
        for (int i = 0; i < d; ++i) {
          const double a = rng.normal(), c = rng.normal();
          h[2 * i] = __dmul_rn(a, 0.70710678118654752440);
          h[2 * i + 1] = __dmul_rn(c, 0.70710678118654752440);
        }
        norm_sq = 0.0;
        for (int q = 0; q < 2 * d; ++q) norm_sq = fma(h[q], h[q], norm_sq);
      } while (norm_sq < kZeroColumnTol * kZeroColumnTol);
    }
    __syncwarp();
    double best = 0.0;
    for (int i = lane; i < N; i += 32) {
      const double* col = book + (long long)i * 2 * d;
      double re = 0.0, im = 0.0;
      for (int q = 0; q < d; ++q) {  // conj(phi_i) . h
        const double ar = col[2 * q], ai = col[2 * q + 1], hr = h[2 * q], hi = h[2 * q + 1];
        re = fma(ar, hr, re);
        re = fma(ai, hi, re);
        im = fma(ar, hi, im);
        im = fma(-ai, hr, im);
      }
      const double ov = __dadd_rn(__dmul_rn(re, re), __dmul_rn(im, im));
      best = ov > best ? ov : best;
    }
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) best = fmax(best, __shfl_xor_sync(0xffffffffu, best, off));
    if (lane == 0) {
      const double dsq = fmax(0.0, __dsub_rn(1.0, __ddiv_rn(best, norm_sq)));
      sum = __dadd_rn(sum, dsq);
      sum_sq = __dadd_rn(sum_sq, __dmul_rn(dsq, dsq));
    }
    __syncwarp();
  }
  if (lane == 0) {
    moments[2 * b] = sum;
    moments[2 * b + 1] = sum_sq;
  }
}

struct DevBuf {
  void* p = nullptr;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
};

int frame_on_device(int field, int64_t d, int64_t N, const double* frame, int normalize, DevBuf& df,
                    int64_t* zero_col) {
  const int L = (field == TRSTMI_COMPLEX ? 2 : 1) * (int)d;
  const size_t bytes = (size_t)L * N * sizeof(double);
  if (cudaMalloc(&df.p, bytes) != cudaSuccess) return TRSTMI_ERR_CUDA;
  if (cudaMemcpy(df.p, frame, bytes, cudaMemcpyHostToDevice) != cudaSuccess) return TRSTMI_ERR_CUDA;
  *zero_col = -1;
  if (normalize) {
    DevBuf dz;
    if (cudaMalloc(&dz.p, sizeof(int)) != cudaSuccess) return TRSTMI_ERR_CUDA;
    const int big = INT_MAX;
    cudaMemcpy(dz.p, &big, sizeof(int), cudaMemcpyHostToDevice);
    an_normalize<<<(int)((N + 127) / 128), 128>>>((double*)df.p, L, (int)N, (int*)dz.p);
    int zc = INT_MAX;
    if (cudaMemcpy(&zc, dz.p, sizeof(int), cudaMemcpyDeviceToHost) != cudaSuccess) return TRSTMI_ERR_CUDA;
    if (zc != INT_MAX) {
      *zero_col = zc;
      return TRSTMI_ERR_ZERO_COLUMN;
    }
  }
  return TRSTMI_OK;
}

}  // namespace

extern "C" {

// All calls run on the legacy default stream and synchronise before returning.
int trstmi_offdiag_magnitudes(int field, int64_t d, int64_t N, const double* frame, int normalize, double* mags,
                              double* sorted_mags, int64_t* zero_col) {
  if ((field != TRSTMI_COMPLEX && field != TRSTMI_REAL) || d < 1 || N < 1 || !frame || !zero_col)
    return TRSTMI_ERR_INVALID_ARG;
  DevBuf df, dm;
  int rc = frame_on_device(field, d, N, frame, normalize, df, zero_col);
  if (rc) return rc;
  const long long n = (long long)N * (N - 1) / 2;
  if (n == 0) return TRSTMI_OK;
  if (cudaMalloc(&dm.p, (size_t)n * sizeof(double)) != cudaSuccess) return TRSTMI_ERR_CUDA;
  const long long grid = std::min<long long>((n + 255) / 256, 148LL * 64);
  an_magnitudes<<<(unsigned)grid, 256>>>((const double*)df.p, field == TRSTMI_COMPLEX, (int)d, (int)N, n,
                                         (double*)dm.p);
  if (cudaGetLastError() != cudaSuccess) return TRSTMI_ERR_CUDA;
  if (mags && cudaMemcpy(mags, dm.p, (size_t)n * sizeof(double), cudaMemcpyDeviceToHost) != cudaSuccess)
    return TRSTMI_ERR_CUDA;
  if (sorted_mags) {
    thrust::device_ptr<double> t((double*)dm.p);
    thrust::sort(thrust::device, t, t + n);
    if (cudaMemcpy(sorted_mags, dm.p, (size_t)n * sizeof(double), cudaMemcpyDeviceToHost) != cudaSuccess)
      return TRSTMI_ERR_CUDA;
  }
  return cudaDeviceSynchronize() == cudaSuccess ? TRSTMI_OK : TRSTMI_ERR_CUDA;
}

int trstmi_normalize_columns(int field, int64_t d, int64_t N, double* frame, int64_t* zero_col) {
  if ((field != TRSTMI_COMPLEX && field != TRSTMI_REAL) || d < 1 || N < 1 || !frame || !zero_col)
    return TRSTMI_ERR_INVALID_ARG;
  DevBuf df;
  const int rc = frame_on_device(field, d, N, frame, 1, df, zero_col);
  if (rc) return rc;
  const size_t bytes = (size_t)(field == TRSTMI_COMPLEX ? 2 : 1) * d * N * sizeof(double);
  return cudaMemcpy(frame, df.p, bytes, cudaMemcpyDeviceToHost) == cudaSuccess ? TRSTMI_OK : TRSTMI_ERR_CUDA;
}

int trstmi_distortion_mc(int64_t d, int64_t N, const double* codebook, uint64_t samples, uint64_t seed,
                         double* estimate, double* std_error) {
  if (d < 1 || N < 1 || !codebook || !estimate || !std_error) return TRSTMI_ERR_INVALID_ARG;
  if (samples < 1) return TRSTMI_ERR_INVALID_ARG;  // distortion_mc: samples >= 1
  const unsigned long long nblocks = (samples + kDistortionBlock - 1) / kDistortionBlock;
  DevBuf db, dm;
  const size_t bytes = (size_t)2 * d * N * sizeof(double);
  if (cudaMalloc(&db.p, bytes) != cudaSuccess || cudaMalloc(&dm.p, (size_t)2 * nblocks * sizeof(double)) != cudaSuccess)
    return TRSTMI_ERR_CUDA;
  if (cudaMemcpy(db.p, codebook, bytes, cudaMemcpyHostToDevice) != cudaSuccess) return TRSTMI_ERR_CUDA;
  constexpr int WPB = 4;  // warps (sample blocks) per CTA
  const size_t smem = (size_t)WPB * 2 * d * sizeof(double);
  if (smem > 48 * 1024 &&
      cudaFuncSetAttribute(an_distortion, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return TRSTMI_ERR_UNSUPPORTED;
  an_distortion<<<(unsigned)((nblocks + WPB - 1) / WPB), 32 * WPB, smem>>>((const double*)db.p, (int)d, (int)N,
                                                                          samples, seed, (double*)dm.p);
  std::vector<double> m((size_t)2 * nblocks);
  if (cudaMemcpy(m.data(), dm.p, m.size() * sizeof(double), cudaMemcpyDeviceToHost) != cudaSuccess)
    return TRSTMI_ERR_CUDA;
  double sum = 0.0, sum_sq = 0.0;  // block moments in block order (beamforming.hpp:142-147)
  for (unsigned long long b = 0; b < nblocks; ++b) {
    sum += m[2 * b];
    sum_sq += m[2 * b + 1];
  }
  const double n = static_cast<double>(samples);
  *estimate = sum / n;
  *std_error = 0.0;
  if (samples > 1) {
    const double var = std::max(0.0, (sum_sq - n * *estimate * *estimate) / (n - 1.0));
    *std_error = std::sqrt(var / n);
  }
  return TRSTMI_OK;
}

int trstmi_cluster_sorted(const double* sorted, int64_t n, double cluster_tol, double* means, int64_t* count) {
  if (!(cluster_tol > 0.0) || !count || (n > 0 && (!sorted || !means))) return TRSTMI_ERR_INVALID_ARG;
  int64_t c = 0, k = 0;
  double sum = 0.0, last = 0.0;
  for (int64_t i = 0; i < n; ++i) {  // cluster_magnitudes, frame.hpp:96-118: sequential sums
    const double v = sorted[i];
    if (k > 0 && v - last > cluster_tol) {
      means[c++] = sum / static_cast<double>(k);
      sum = 0.0;
      k = 0;
    }
    sum += v;
    last = v;
    ++k;
  }
  if (k > 0) means[c++] = sum / static_cast<double>(k);
  *count = c;
  return TRSTMI_OK;
}

int trstmi_frame_operator_deviation(int field, int64_t d, int64_t N, const double* frame, double* deviation) {
  if ((field != TRSTMI_COMPLEX && field != TRSTMI_REAL) || d < 1 || N < 1 || !frame || !deviation)
    return TRSTMI_ERR_INVALID_ARG;
  DevBuf df, db;
  int64_t zc;
  int rc = frame_on_device(field, d, N, frame, 0, df, &zc);
  if (rc) return rc;
  if (cudaMalloc(&db.p, 8) != cudaSuccess) return TRSTMI_ERR_CUDA;
  cudaMemset(db.p, 0, 8);
  const long long e = d * d;
  an_frame_operator<<<(unsigned)((e + 255) / 256), 256>>>((const double*)df.p, field == TRSTMI_COMPLEX, (int)d,
                                                          (int)N, (unsigned long long*)db.p);
  unsigned long long bits = 0;
  if (cudaMemcpy(&bits, db.p, 8, cudaMemcpyDeviceToHost) != cudaSuccess) return TRSTMI_ERR_CUDA;
  std::memcpy(deviation, &bits, 8);
  return TRSTMI_OK;
}

}  // extern "C"
