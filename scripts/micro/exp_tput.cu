#include <cstdio>
#include "../../paper_2207_06374_b200/csrc/cas_math.cuh"
using namespace trstmi_dev;
__global__ void k_exp(const double* __restrict__ x, double* y, int n, int reps) {
  double acc = 0;
  for (int r = 0; r < reps; ++r)
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x * 4) {
      double a0 = x[i], a1 = x[(i + blockDim.x) % n], a2 = x[(i + 2 * blockDim.x) % n], a3 = x[(i + 3 * blockDim.x) % n];
      acc += cas_exp(a0 - r) + cas_exp(a1 - r) + cas_exp(a2 - r) + cas_exp(a3 - r);
    }
  y[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void k_exp_lib(const double* __restrict__ x, double* y, int n, int reps) {
  double acc = 0;
  for (int r = 0; r < reps; ++r)
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x * 4) {
      double a0 = x[i], a1 = x[(i + blockDim.x) % n], a2 = x[(i + 2 * blockDim.x) % n], a3 = x[(i + 3 * blockDim.x) % n];
      acc += exp(a0 - r) + exp(a1 - r) + exp(a2 - r) + exp(a3 - r);
    }
  y[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
  const int n = 148 * 512 * 4; double *x, *y; cudaMalloc(&x, n * 8); cudaMalloc(&y, n * 8);
  double* h = new double[n]; for (int i = 0; i < n; ++i) h[i] = -(i % 1000) * 0.3; cudaMemcpy(x, h, n * 8, cudaMemcpyHostToDevice);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int which = 0; which < 2; ++which) {
    for (int threads : {256, 512}) {
      auto f = which == 0 ? k_exp : k_exp_lib;
      f<<<148, threads>>>(x, y, n, 2);
      cudaEventRecord(a); f<<<148, threads>>>(x, y, n, 50); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      double exps = 50.0 * n;  // each thread loop covers 4 per iteration over n/4 iterations
      printf("%s threads=%d: %.3f ms -> %.2f exps/clk/SM (at 1.965GHz)\n", which ? "libdevice exp" : "cas_exp", threads, ms,
             exps / (ms * 1e-3) / 148 / 1.965e9);
    }
  }
}
