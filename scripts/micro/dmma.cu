// FP64 tensor-core (DMMA, mma.sync .f64) probe on sm_100a:
//  (1) bit-exactness: does D = mma(A, B, C) equal the sequential fma chain
//      d = fma(a_{K-1}, b_{K-1}, ... fma(a_0, b_0, c)) in ascending k?  (If yes,
//      DMMA reproduces the CAS Gram / gradient orders exactly.)
//  (2) throughput of m8n8k4 / m16n8k4 / m16n8k8 / m16n8k16 vs the DFMA loop.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma dmma.cu
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#define CK(x)                                                                            \
  do {                                                                                   \
    cudaError_t e = (x);                                                                 \
    if (e != cudaSuccess) {                                                              \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);           \
      exit(1);                                                                           \
    }                                                                                    \
  } while (0)

// ---- fragments: one MMA per warp; A (M x K, row-major), B (K x N, col), C/D (M x N)
template <int M, int N, int K>
__device__ void mma_op(const double* a, const double* b, double* c);

// m8n8k4: a0 = A[g][t], b0 = B[t][g], c{0,1} = C[g][2t+i]   (g = lane>>2, t = lane&3)
template <>
__device__ void mma_op<8, 8, 4>(const double* A, const double* B, double* C) {
  const int l = threadIdx.x & 31, g = l >> 2, t = l & 3;
  double a0 = A[g * 4 + t], b0 = B[t * 8 + g];
  double c0 = C[g * 8 + 2 * t], c1 = C[g * 8 + 2 * t + 1];
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a0), "d"(b0));
  C[g * 8 + 2 * t] = c0;
  C[g * 8 + 2 * t + 1] = c1;
}
// m16n8k4: a0 = A[g][t], a1 = A[g+8][t]; b0 = B[t][g]; c0,c1 = C[g][2t+i], c2,c3 = C[g+8][2t+i]
template <>
__device__ void mma_op<16, 8, 4>(const double* A, const double* B, double* C) {
  const int l = threadIdx.x & 31, g = l >> 2, t = l & 3;
  double a0 = A[g * 4 + t], a1 = A[(g + 8) * 4 + t], b0 = B[t * 8 + g];
  double c0 = C[g * 8 + 2 * t], c1 = C[g * 8 + 2 * t + 1], c2 = C[(g + 8) * 8 + 2 * t], c3 = C[(g + 8) * 8 + 2 * t + 1];
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
               : "+d"(c0), "+d"(c1), "+d"(c2), "+d"(c3)
               : "d"(a0), "d"(a1), "d"(b0));
  C[g * 8 + 2 * t] = c0;
  C[g * 8 + 2 * t + 1] = c1;
  C[(g + 8) * 8 + 2 * t] = c2;
  C[(g + 8) * 8 + 2 * t + 1] = c3;
}
// m16n8k8: a_i: row g + 8*(i&1), col t + 4*(i>>1); b_i: row t + 4*i, col g
template <>
__device__ void mma_op<16, 8, 8>(const double* A, const double* B, double* C) {
  const int l = threadIdx.x & 31, g = l >> 2, t = l & 3;
  double a[4], b[2];
  for (int i = 0; i < 4; ++i) a[i] = A[(g + 8 * (i & 1)) * 8 + t + 4 * (i >> 1)];
  for (int i = 0; i < 2; ++i) b[i] = B[(t + 4 * i) * 8 + g];
  double c0 = C[g * 8 + 2 * t], c1 = C[g * 8 + 2 * t + 1], c2 = C[(g + 8) * 8 + 2 * t], c3 = C[(g + 8) * 8 + 2 * t + 1];
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+d"(c0), "+d"(c1), "+d"(c2), "+d"(c3)
      : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
  C[g * 8 + 2 * t] = c0;
  C[g * 8 + 2 * t + 1] = c1;
  C[(g + 8) * 8 + 2 * t] = c2;
  C[(g + 8) * 8 + 2 * t + 1] = c3;
}
// m16n8k16: a_i: row g + 8*(i&1), col t + 4*(i>>1) (i < 8); b_i: row t + 4*i (i < 4)
template <>
__device__ void mma_op<16, 8, 16>(const double* A, const double* B, double* C) {
  const int l = threadIdx.x & 31, g = l >> 2, t = l & 3;
  double a[8], b[4];
  for (int i = 0; i < 8; ++i) a[i] = A[(g + 8 * (i & 1)) * 16 + t + 4 * (i >> 1)];
  for (int i = 0; i < 4; ++i) b[i] = B[(t + 4 * i) * 8 + g];
  double c0 = C[g * 8 + 2 * t], c1 = C[g * 8 + 2 * t + 1], c2 = C[(g + 8) * 8 + 2 * t], c3 = C[(g + 8) * 8 + 2 * t + 1];
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
      "{%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
      : "+d"(c0), "+d"(c1), "+d"(c2), "+d"(c3)
      : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]), "d"(b[0]),
        "d"(b[1]), "d"(b[2]), "d"(b[3]));
  C[g * 8 + 2 * t] = c0;
  C[g * 8 + 2 * t + 1] = c1;
  C[(g + 8) * 8 + 2 * t] = c2;
  C[(g + 8) * 8 + 2 * t + 1] = c3;
}

template <int M, int N, int K>
__global__ void exact_kernel(const double* A, const double* B, double* C, int reps) {
  const int w = blockIdx.x;  // one warp per problem
  mma_op<M, N, K>(A + (size_t)w * M * K, B + (size_t)w * K * N, C + (size_t)w * M * N);
}

static unsigned long long rs = 88172645463325252ull;
static double rnd() {
  rs ^= rs << 13;
  rs ^= rs >> 7;
  rs ^= rs << 17;
  const int e = (int)(rs % 40) - 20;
  const double m = (double)(rs >> 11) * 0x1.0p-53 * 2.0 - 1.0;
  return std::ldexp(m, e);
}

template <int M, int N, int K>
void check_exact(int problems) {
  std::vector<double> A((size_t)problems * M * K), B((size_t)problems * K * N), C((size_t)problems * M * N), D(C.size());
  for (auto& v : A) v = rnd();
  for (auto& v : B) v = rnd();
  for (auto& v : C) v = rnd();
  double *dA, *dB, *dC;
  CK(cudaMalloc(&dA, A.size() * 8));
  CK(cudaMalloc(&dB, B.size() * 8));
  CK(cudaMalloc(&dC, C.size() * 8));
  CK(cudaMemcpy(dA, A.data(), A.size() * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size() * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dC, C.data(), C.size() * 8, cudaMemcpyHostToDevice));
  exact_kernel<M, N, K><<<problems, 32>>>(dA, dB, dC, 1);
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(D.data(), dC, D.size() * 8, cudaMemcpyDeviceToHost));
  long long fwd = 0, rev = 0, once = 0, n = 0;
  for (int p = 0; p < problems; ++p)
    for (int i = 0; i < M; ++i)
      for (int j = 0; j < N; ++j) {
        const double* a = &A[(size_t)p * M * K + i * K];
        double f = C[(size_t)p * M * N + i * N + j], r = f;
        long double ex = f;
        for (int k = 0; k < K; ++k) f = std::fma(a[k], B[(size_t)p * K * N + k * N + j], f);
        for (int k = K - 1; k >= 0; --k) r = std::fma(a[k], B[(size_t)p * K * N + k * N + j], r);
        for (int k = 0; k < K; ++k) ex += (long double)a[k] * (long double)B[(size_t)p * K * N + k * N + j];
        const double d = D[(size_t)p * M * N + i * N + j];
        fwd += d != f;
        rev += d != r;
        once += d != (double)ex;
        ++n;
      }
  printf("m%dn%dk%d: %lld outputs; != ascending fma chain: %lld; != descending chain: %lld; != long-double sum: %lld\n",
         M, N, K, n, fwd, rev, once);
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dC);
}

// ---- throughput: each warp keeps 8 independent accumulator sets
template <int M, int N, int K>
__global__ void tput_kernel(double* out, int iters, double s) {
  const int NA = (M * K) / 32, NB = (K * N) / 32;
  double a[8], b[4], c[8][4];
  for (int i = 0; i < 8; ++i) a[i] = s * (threadIdx.x + i);
  for (int i = 0; i < 4; ++i) b[i] = s * (threadIdx.x - i);
  for (int u = 0; u < 8; ++u)
    for (int i = 0; i < 4; ++i) c[u][i] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if constexpr (M == 8) {
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[u][0]), "+d"(c[u][1])
                     : "d"(a[u & 7]), "d"(b[u & 3]));
      } else if constexpr (K == 4) {
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                     : "+d"(c[u][0]), "+d"(c[u][1]), "+d"(c[u][2]), "+d"(c[u][3])
                     : "d"(a[0]), "d"(a[1]), "d"(b[0]));
      } else if constexpr (K == 8) {
        asm volatile(
            "mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
            : "+d"(c[u][0]), "+d"(c[u][1]), "+d"(c[u][2]), "+d"(c[u][3])
            : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
      } else {
        asm volatile(
            "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
            "{%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
            : "+d"(c[u][0]), "+d"(c[u][1]), "+d"(c[u][2]), "+d"(c[u][3])
            : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]), "d"(b[0]),
              "d"(b[1]), "d"(b[2]), "d"(b[3]));
      }
    }
  }
  double r = 0.0;
  for (int u = 0; u < 8; ++u)
    for (int i = 0; i < 4; ++i) r += c[u][i];
  if (r == 1234.5) out[0] = r;
  (void)NA;
  (void)NB;
}

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int u = 0; u < 16; ++u)
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  double r = 0;
  for (int i = 0; i < 8; ++i) r += x[i];
  if (r == 1234.5) out[0] = r;
}

template <int M, int N, int K>
void tput(int sms, int warps_per_cta, int ctas_per_sm) {
  double* out;
  CK(cudaMalloc(&out, 8));
  const int iters = 4000;
  const int grid = sms * ctas_per_sm;
  tput_kernel<M, N, K><<<grid, 32 * warps_per_cta>>>(out, 10, 1e-3);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  tput_kernel<M, N, K><<<grid, 32 * warps_per_cta>>>(out, iters, 1e-3);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flops = 2.0 * M * N * K * 8.0 * iters * (double)grid * warps_per_cta;
  printf("m%dn%dk%d  %2d warps/CTA x %d CTAs/SM: %.2f TFLOP/s\n", M, N, K, warps_per_cta, ctas_per_sm,
         flops / (ms * 1e-3) / 1e12);
  cudaFree(out);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  check_exact<8, 8, 4>(4096);
  check_exact<16, 8, 4>(4096);
  check_exact<16, 8, 8>(4096);
  check_exact<16, 8, 16>(4096);
  {
    double* out;
    CK(cudaMalloc(&out, 8));
    const int iters = 20000;
    dfma_kernel<<<sms * 8, 256>>>(out, 100, 0.999, 1e-7);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    dfma_kernel<<<sms * 8, 256>>>(out, iters, 0.999, 1e-7);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("DFMA loop: %.2f TFLOP/s\n", 2.0 * 8 * 16 * (double)iters * sms * 8 * 256 / (ms * 1e-3) / 1e12);
  }
  for (int w : {4, 8, 16})
    for (int c : {1, 2, 4}) {
      tput<8, 8, 4>(sms, w, c);
      tput<16, 8, 4>(sms, w, c);
      tput<16, 8, 8>(sms, w, c);
      tput<16, 8, 16>(sms, w, c);
    }
  return 0;
}
