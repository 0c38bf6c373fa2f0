// DFMA throughput with distinct register operands (no operand-reuse) vs shared constants.
#include <cstdio>
__global__ void shared_ops(double* out, int iters, double a, double b) {
  double x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int u = 0; u < 8; ++u) x[u] = fma(x[u], a, b);
  double s = 0; for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 1.2345) out[0] = s;
}
__global__ void distinct_ops(double* out, int iters) {
  double x[8], p[8], q[8];
  for (int i = 0; i < 8; ++i) { x[i] = threadIdx.x + i; p[i] = 1.0 + 1e-9 * i; q[i] = 1e-9 * (i + threadIdx.x); }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) x[u] = fma(p[u], x[(u + 1) & 7], q[(u + 3) & 7]);
#pragma unroll
    for (int u = 0; u < 8; ++u) { double t = p[u]; p[u] = q[u]; q[u] = t; }
  }
  double s = 0; for (int i = 0; i < 8; ++i) s += x[i] + p[i];
  if (s == 1.2345) out[0] = s;
}
__global__ void mixed_ops(double* out, int iters) {  // fma + mul + add mix like the eval
  double x[8], p[8];
  for (int i = 0; i < 8; ++i) { x[i] = threadIdx.x + i; p[i] = 1.0 + 1e-9 * i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const double m = __dmul_rn(x[u], p[(u + 1) & 7]);
      x[u] = __dadd_rn(fma(x[u], p[u], m), -m);
    }
  }
  double s = 0; for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 1.2345) out[0] = s;
}
int main() {
  double* out; cudaMalloc(&out, 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int iters = 4000, blocks = 148 * 4, threads = 256;
  float ms;
  shared_ops<<<blocks, threads>>>(out, 10, 0.99, 1e-3);
  cudaEventRecord(a); shared_ops<<<blocks, threads>>>(out, iters, 0.99, 1e-3); cudaEventRecord(b); cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  printf("shared-constant DFMA: %.1f DP ops/clk/SM\n", 8.0 * iters * blocks * threads / (ms * 1e-3) / 148 / 1.965e9);
  distinct_ops<<<blocks, threads>>>(out, 10);
  cudaEventRecord(a); distinct_ops<<<blocks, threads>>>(out, iters); cudaEventRecord(b); cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  printf("distinct-operand DFMA: %.1f DP ops/clk/SM\n", 8.0 * iters * blocks * threads / (ms * 1e-3) / 148 / 1.965e9);
  mixed_ops<<<blocks, threads>>>(out, 10);
  cudaEventRecord(a); mixed_ops<<<blocks, threads>>>(out, iters); cudaEventRecord(b); cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  printf("mul/fma/add mix: %.1f DP ops/clk/SM\n", 24.0 * iters * blocks * threads / (ms * 1e-3) / 148 / 1.965e9);
}
