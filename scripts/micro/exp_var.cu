#include <cstdio>
#include "../../paper_2207_06374_b200/csrc/cas_math.cuh"
using namespace trstmi_dev;
// B: magic-number rounding, bit-built powers
__device__ __forceinline__ double exp_b(double x) {
  const double xc = fmin(fmax(x, -745.25), 709.8);
  const double t = fma(xc, 1.4426950408889634, 0x1.8p52);
  const double kd = __dsub_rn(t, 0x1.8p52);
  const int k = __double2loint(t);
  double r = fma(-kd, 6.93147180369123816490e-01, xc);
  r = fma(-kd, 1.90821492927058770002e-10, r);
  double p = 1.6059043836821613e-10;
  p = fma(p, r, 2.08767569878680989792e-09); p = fma(p, r, 2.50521083854417187751e-08);
  p = fma(p, r, 2.75573192239858906526e-07); p = fma(p, r, 2.75573192239858906526e-06);
  p = fma(p, r, 2.48015873015873015873e-05); p = fma(p, r, 1.98412698412698412698e-04);
  p = fma(p, r, 1.38888888888888888889e-03); p = fma(p, r, 8.33333333333333333333e-03);
  p = fma(p, r, 4.16666666666666666667e-02); p = fma(p, r, 1.66666666666666666667e-01);
  p = fma(p, r, 0.5); p = fma(p, r, 1.0); p = fma(p, r, 1.0);
  const int k1 = k >> 1;
  const double s1 = __hiloint2double((k1 + 1023) << 20, 0), s2 = __hiloint2double((k - k1 + 1023) << 20, 0);
  double res = __dmul_rn(__dmul_rn(p, s1), s2);
  res = (x > 709.782712893383973096) ? __longlong_as_double(0x7ff0000000000000LL) : res;
  res = (x < -745.2) ? 0.0 : res;
  return (x == x) ? res : x;
}
// D: B without clamp/special cases (upper bound on speed)
__device__ __forceinline__ double exp_d(double x) {
  const double t = fma(x, 1.4426950408889634, 0x1.8p52);
  const double kd = __dsub_rn(t, 0x1.8p52);
  const int k = __double2loint(t);
  double r = fma(-kd, 6.93147180369123816490e-01, x);
  r = fma(-kd, 1.90821492927058770002e-10, r);
  double p = 1.6059043836821613e-10;
  p = fma(p, r, 2.08767569878680989792e-09); p = fma(p, r, 2.50521083854417187751e-08);
  p = fma(p, r, 2.75573192239858906526e-07); p = fma(p, r, 2.75573192239858906526e-06);
  p = fma(p, r, 2.48015873015873015873e-05); p = fma(p, r, 1.98412698412698412698e-04);
  p = fma(p, r, 1.38888888888888888889e-03); p = fma(p, r, 8.33333333333333333333e-03);
  p = fma(p, r, 4.16666666666666666667e-02); p = fma(p, r, 1.66666666666666666667e-01);
  p = fma(p, r, 0.5); p = fma(p, r, 1.0); p = fma(p, r, 1.0);
  const int k1 = k >> 1;
  const double s1 = __hiloint2double((k1 + 1023) << 20, 0), s2 = __hiloint2double((k - k1 + 1023) << 20, 0);
  return __dmul_rn(__dmul_rn(p, s1), s2);
}
template <int V>
__global__ void k_exp(const double* __restrict__ x, double* y, int n, int reps) {
  double acc = 0;
  for (int r = 0; r < reps; ++r)
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x * 4) {
      const double base = -(double)(i & 1023) * 0.3 - r;
      double a[4] = {base, base - 0.11, base - 0.37, base - 0.71};
#pragma unroll
      for (int u = 0; u < 4; ++u) acc += V == 0 ? cas_exp(a[u]) : V == 1 ? exp_b(a[u]) : exp_d(a[u]);
    }
  y[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
int main() {
  const int n = 148 * 512 * 4; double *x, *y; cudaMalloc(&x, n * 8); cudaMalloc(&y, n * 8);
  double* h = new double[n]; for (int i = 0; i < n; ++i) h[i] = -(i % 1000) * 0.3; cudaMemcpy(x, h, n * 8, cudaMemcpyHostToDevice);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  void (*fs[3])(const double*, double*, int, int) = {k_exp<0>, k_exp<1>, k_exp<2>};
  const char* names[3] = {"cas_exp (rint)", "magic-round", "magic no-special"};
  for (int v = 0; v < 3; ++v)
    for (int threads : {256, 512, 1024}) {
      fs[v]<<<148, threads>>>(x, y, n, 2);
      cudaEventRecord(a); fs[v]<<<148, threads>>>(x, y, n, 50); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("%-18s threads=%4d: %.2f exps/clk/SM\n", names[v], threads, 50.0 * n / (ms * 1e-3) / 148 / 1.965e9);
    }
}
