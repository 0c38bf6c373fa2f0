// FP64 / smem latency and throughput microbenchmarks on one SM.
#include <cstdio>
__global__ void dfma_lat(double* out, long long* cyc, int iters, double a, double b) {
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) x = fma(x, a, b);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; }
  if (x == 1.2345) out[0] = x;
}
__global__ void dadd_lat(double* out, long long* cyc, int iters, double a) {
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) x = __dadd_rn(x, a);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; }
  if (x == 1.2345) out[0] = x;
}
__global__ void dfma_tput(double* out, long long* cyc, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; }
  if (x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7 == 1.2345) out[0] = x0;
}
__global__ void lds_lat(double* out, long long* cyc, int iters) {
  __shared__ int idx[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) idx[i] = (i + 1) & 1023;
  __syncthreads();
  int j = threadIdx.x & 1023;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) j = idx[j];
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  if (j == -1) out[0] = j;
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 8); cudaMalloc(&cyc, 8);
  long long c;
  const int it = 1000;
  for (int w : {1, 4, 16, 32}) {
    dfma_lat<<<1, 32 * w>>>(out, cyc, it, 0.999, 1e-3); cudaDeviceSynchronize();
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("DFMA dependent chain, %2d warps: %.2f cycles/op\n", w, c / (16.0 * it));
  }
  dadd_lat<<<1, 32>>>(out, cyc, it, 1e-3); cudaDeviceSynchronize(); cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("DADD dependent chain, 1 warp: %.2f cycles/op\n", c / (16.0 * it));
  for (int w : {1, 2, 4, 8, 16, 32}) {
    dfma_tput<<<1, 32 * w>>>(out, cyc, it, 0.999, 1e-3); cudaDeviceSynchronize();
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("DFMA 8 chains/thread, %2d warps: %.2f cycles per warp-instr per SM -> %.1f FMA/clk/SM\n", w, c / (32.0 * it * w),
           32.0 * it * w * 32 / c);
  }
  lds_lat<<<1, 32>>>(out, cyc, it); cudaDeviceSynchronize(); cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("LDS.32 dependent chain: %.1f cycles\n", c / (double)it);
  return 0;
}
