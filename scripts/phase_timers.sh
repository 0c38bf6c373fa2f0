#!/bin/bash
# Builds a side copy of the eval kernel with per-phase clock64 timers and
# prints cycles per phase per eval.  usage: scripts/phase_timers.sh FIELD D N DELTA [S] [GS] [PAD]
# (GS=1: stored-Gram layout, small_gs.cuh; default 1, PAD default 1)
set -e
cd "$(dirname "$0")/.."
mkdir -p /tmp/phase && cat > /tmp/phase/pt.cu <<'CU'
#define TRSTMI_PHASE_TIMERS 1
#include "batch_kernels.cuh"
#include <cstdio>
#include <vector>
#include <cstdlib>
using namespace trstmi_dev;
int main(int argc, char** argv) {
  int field = atoi(argv[1]), d = atoi(argv[2]), N = atoi(argv[3]); double delta = atof(argv[4]);
  const bool cplx = field == 0;
  Prob P = make_small_prob(cplx, d, N, kchunks_for(d, N, SS), GSM, PADM);
  const int B = 148 * 4;
  std::vector<double> h((size_t)B * P.dim); srand(1); for (auto& v : h) v = rand() / (double)RAND_MAX - 0.5;
  double *x, *dl, *F, *s, *g; long long* zc;
  cudaMalloc(&x, h.size() * 8); cudaMemcpy(x, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  cudaMalloc(&dl, B * 8); std::vector<double> hd(B, delta); cudaMemcpy(dl, hd.data(), B * 8, cudaMemcpyHostToDevice);
  cudaMalloc(&F, B * 8); cudaMalloc(&s, B * 8); cudaMalloc(&g, h.size() * 8); cudaMalloc(&zc, B * 8);
  BatchArgs A{}; A.P = P; A.B = B; A.pts = x; A.delta = dl; A.squared = 1; A.F = F; A.s = s; A.out = g; A.zero_col = zc;
  auto fn = cplx ? (const void*)&eval_batch_kernel<true, DD, true, SS, (GSM != 0)> : (const void*)&eval_batch_kernel<false, DD, true, SS, (GSM != 0)>;
  size_t bytes = smem_doubles(P, SS, cplx, 3) * 8;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  void* args[] = {&A};
  cudaLaunchKernel(fn, dim3(B), dim3(SS), args, bytes, 0);
  cudaDeviceSynchronize();
  unsigned long long z[8] = {0}; cudaMemcpyToSymbol(g_phase_cycles, z, sizeof(z));
  cudaLaunchKernel(fn, dim3(B), dim3(SS), args, bytes, 0);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long c[8]; cudaMemcpyFromSymbol(c, g_phase_cycles, sizeof(c));
  const char* names[6] = {"normalize", "gram+max", "exp", "zsum", "grad-loop", "combine"};
  unsigned long long tot = 0; for (int i = 0; i < 6; ++i) tot += c[i];
  printf("%s field=%d d=%d N=%d delta=%g S=%d gs=%d pad=%d smem=%zu: total %.0f cycles/eval\n", cudaGetErrorString(e), field, d, N, delta, SS, GSM, PADM, bytes, tot / (double)B);
  for (int i = 0; i < 6; ++i) printf("  %-10s %8.0f\n", names[i], c[i] / (double)B);
}
CU
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -fmad=false --expt-relaxed-constexpr -DDD=$2 -DSS=${5:-512} -DGSM=${6:-1} -DPADM=${7:-1} $EXTRA \
  -I paper_2207_06374_b200/csrc -I include -o /tmp/phase/pt /tmp/phase/pt.cu
/tmp/phase/pt "$1" "$2" "$3" "$4"
