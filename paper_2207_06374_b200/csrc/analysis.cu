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
#include <string>

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
    mags[p] = sqrt(__dadd_rn(__dmul_rn(re, re), __dmul_rn(im, im)));
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
    m = sqrt(__dadd_rn(__dmul_rn(re, re), __dmul_rn(im, im)));
  }
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, off));
  if ((threadIdx.x & 31) == 0) atomicMax(dev_bits, (unsigned long long)__double_as_longlong(m));
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
