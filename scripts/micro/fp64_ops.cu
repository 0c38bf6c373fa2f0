// FP64-pipe instruction throughput on B200 (ops per clock per SM) for the
// instructions the CAS exp / division / pair walk use: DFMA, DADD, DMUL,
// fmax (DSETP+FSEL), rint (FRND), double->int (F2I), int->double (I2F),
// compares, and whole exp variants.  8 independent chains per thread,
// 148 x 8 CTAs x 256 threads, cycles from clock64 on each CTA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o fp64_ops fp64_ops.cu
#include <cstdio>
#include "../../paper_2207_06374_b200/csrc/cas_math.cuh"
using namespace trstmi_dev;

constexpr int U = 8;
__device__ unsigned long long g_cyc[148 * 64];

template <int OP>
__device__ __forceinline__ void step(double (&a)[U], int it) {
#pragma unroll
  for (int u = 0; u < U; ++u) {
    double x = a[u];
    if constexpr (OP == 0) x = fma(x, 0.999999, 1e-7);
    if constexpr (OP == 1) x = __dadd_rn(x, 1e-9);
    if constexpr (OP == 2) x = __dmul_rn(x, 0.9999999);
    if constexpr (OP == 3) x = fmax(x, 1e-3 * u);
    if constexpr (OP == 4) x = rint(x) + 0.25;  // FRND + DADD
    if constexpr (OP == 5) x = (double)(__double2int_rn(x) + it);  // F2I + I2F
    if constexpr (OP == 6) x = (x > 0.5) ? x * 0.5 : x + 1.0;     // DSETP + sel + 2 ops
    if constexpr (OP == 7) x = cas_exp(-x) + 0.5;                 // CAS exp + DADD
    if constexpr (OP == 8) x = __ddiv_rn(1.0, x) + 0.5;           // IEEE division
    if constexpr (OP == 9) x = sqrt(x) + 0.5;                      // sqrt
    a[u] = x;
  }
}

template <int OP>
__global__ void k(double* out, int iters) {
  double a[U];
#pragma unroll
  for (int u = 0; u < U; ++u) a[u] = 0.5 + 0.01 * u + 1e-6 * threadIdx.x;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) step<OP>(a, it);
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) g_cyc[blockIdx.x] = (unsigned long long)(t1 - t0);
  double s = 0;
#pragma unroll
  for (int u = 0; u < U; ++u) s += a[u];
  if (s == 12345.678) out[0] = s;
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  const char* names[] = {"DFMA", "DADD", "DMUL", "fmax", "rint+DADD", "F2I+I2F", "cmp+sel+op", "cas_exp+DADD",
                         "ddiv+DADD", "sqrt+DADD"};
  void (*fs[])(double*, int) = {k<0>, k<1>, k<2>, k<3>, k<4>, k<5>, k<6>, k<7>, k<8>, k<9>};
  for (int threads : {256, 512}) {
    for (int op = 0; op < 10; ++op) {
      int per_sm = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fs[op], threads, 0);
      const int ctas = 148 * per_sm;
      const int iters = op >= 7 ? 256 : 4096;
      fs[op]<<<ctas, threads>>>(out, iters);
      cudaDeviceSynchronize();
      fs[op]<<<ctas, threads>>>(out, iters);
      cudaError_t e = cudaDeviceSynchronize();
      unsigned long long c[148 * 64];
      cudaMemcpyFromSymbol(c, g_cyc, sizeof(unsigned long long) * ctas);
      double mx = 0;
      for (int i = 0; i < ctas; ++i) mx = c[i] > mx ? c[i] : mx;
      // one wave, all CTAs resident: ops per SM per clock
      const double ops = (double)per_sm * threads * iters * U;
      printf("%-14s threads=%d x %d/SM  %6.2f ops/clk/SM  (%s)\n", names[op], threads, per_sm, ops / mx,
             cudaGetErrorString(e));
    }
  }
  return 0;
}
