// Prototype harness: eval_cta_rt (T = S/V threads, two CTAs per SM) against eval_cta_gs (S threads) —
// bitwise comparison of F, s and the gradient, then throughput of both.
#ifdef PT
#define TRSTMI_PHASE_TIMERS 1
#endif
#include "batch_kernels.cuh"
#include "small_rt.cuh"
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
using namespace trstmi_dev;

#ifndef DD
#define DD 2
#endif
#ifndef SS
#define SS 512
#endif
#ifndef VV
#define VV 2
#endif
#ifndef MINB
#define MINB (SS / VV >= 512 ? 1 : 512 / (SS / VV))
#endif
#ifndef NVEC
#define NVEC 9
#endif

template <bool CPLX, int DMAX, bool EXACT, int S, int V>
__global__ void __launch_bounds__(S / V, MINB) eval_rt_kernel(const BatchArgs A) {
  extern __shared__ __align__(16) double smem_raw[];
  Smem sm;
  double* v[1];
  carve_rt(A.P, S, smem_raw, sm, v, 0);
  if (threadIdx.x == 0) sm.scal[3] = 0.0;
  __syncthreads();
  int rbuf = 0;
  for (long long b = blockIdx.x; b < A.B; b += gridDim.x) {
    const double* x = A.pts + b * A.P.dim;
    const int zc = eval_cta_rt<CPLX, DMAX, EXACT, S, V, true>(A.P, x, nullptr, 0.0, A.delta[b], sm, rbuf,
                                                             A.out + b * A.P.dim, &sm.scal[0], &sm.scal[1], nullptr);
    if (threadIdx.x == 0) {
      A.F[b] = sm.scal[0];
      A.s[b] = sm.scal[1];
      A.zero_col[b] = zc;
    }
    __syncthreads();
  }
}

int main(int argc, char** argv) {
  const int field = atoi(argv[1]), d = DD, N = atoi(argv[2]);
  const double delta = atof(argv[3]);
  const int reps = argc > 4 ? atoi(argv[4]) : 20;
  const bool cplx = field == 0;
  const int B = 148 * 8;
  Prob Pg = make_small_prob(cplx, d, N, kchunks_for(d, N, SS), 1, 1);
  Prob Pr = make_small_prob(cplx, d, N, kchunks_for(d, N, SS), 0, 0);
  std::vector<double> h((size_t)B * Pg.dim);
  srand(1);
  for (auto& v : h) v = rand() / (double)RAND_MAX - 0.5;
  double *x, *dl, *F, *s, *g, *F2, *s2, *g2;
  long long *zc, *zc2;
  size_t nb = h.size() * 8;
  cudaMalloc(&x, nb); cudaMemcpy(x, h.data(), nb, cudaMemcpyHostToDevice);
  std::vector<double> hd(B, delta);
  cudaMalloc(&dl, B * 8); cudaMemcpy(dl, hd.data(), B * 8, cudaMemcpyHostToDevice);
  cudaMalloc(&F, B * 8); cudaMalloc(&s, B * 8); cudaMalloc(&g, nb); cudaMalloc(&zc, B * 8);
  cudaMalloc(&F2, B * 8); cudaMalloc(&s2, B * 8); cudaMalloc(&g2, nb); cudaMalloc(&zc2, B * 8);
  BatchArgs A{}; A.P = Pg; A.B = B; A.pts = x; A.delta = dl; A.squared = 1; A.F = F; A.s = s; A.out = g; A.zero_col = zc;
  BatchArgs R = A; R.P = Pr; R.F = F2; R.s = s2; R.out = g2; R.zero_col = zc2;
  const void* fg = cplx ? (const void*)&eval_batch_kernel<true, DD, true, SS, true> : (const void*)&eval_batch_kernel<false, DD, true, SS, true>;
  const void* fr = cplx ? (const void*)&eval_rt_kernel<true, DD, true, SS, VV> : (const void*)&eval_rt_kernel<false, DD, true, SS, VV>;
  const size_t bg = smem_doubles(Pg, SS, cplx, 3) * 8, br = rt_smem_doubles(Pr, SS, NVEC) * 8;  // rt: anneal-sized (9 vectors) for occupancy realism
  cudaFuncSetAttribute(fg, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bg);
  cudaFuncSetAttribute(fr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)br);
  int og = 0, orr = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&og, fg, SS, bg);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&orr, fr, SS / VV, br);
  printf("field=%d d=%d N=%d delta=%g S=%d V=%d: gs smem %zu (%d CTA/SM), rt smem %zu (%d CTA/SM)\n", field, d, N, delta, SS, VV, bg, og, br, orr);
  void* ag[] = {&A};
  void* ar[] = {&R};
  const int gridg = 148 * og, gridr = 148 * orr;
  cudaLaunchKernel(fg, dim3(gridg), dim3(SS), ag, bg, 0);
  cudaLaunchKernel(fr, dim3(gridr), dim3(SS / VV), ar, br, 0);
  cudaError_t e = cudaDeviceSynchronize();
  printf("run: %s\n", cudaGetErrorString(e));
  std::vector<double> hg(h.size()), hg2(h.size()), hF(B), hF2(B), hs(B), hs2(B);
  cudaMemcpy(hg.data(), g, nb, cudaMemcpyDeviceToHost); cudaMemcpy(hg2.data(), g2, nb, cudaMemcpyDeviceToHost);
  cudaMemcpy(hF.data(), F, B * 8, cudaMemcpyDeviceToHost); cudaMemcpy(hF2.data(), F2, B * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(hs.data(), s, B * 8, cudaMemcpyDeviceToHost); cudaMemcpy(hs2.data(), s2, B * 8, cudaMemcpyDeviceToHost);
  long long badg = 0, badF = 0;
  for (size_t i = 0; i < hg.size(); ++i) badg += memcmp(&hg[i], &hg2[i], 8) != 0;
  for (int b = 0; b < B; ++b) badF += (memcmp(&hF[b], &hF2[b], 8) != 0) + (memcmp(&hs[b], &hs2[b], 8) != 0);
  printf("bitwise mismatches: grad %lld of %zu, F/s %lld of %d   (F[0] = %.17g vs %.17g)\n", badg, hg.size(), badF, 2 * B, hF[0], hF2[0]);
#ifdef PT
  unsigned long long z[8] = {0};
  cudaMemcpyToSymbol(g_phase_cycles, z, sizeof(z));
  cudaLaunchKernel(fr, dim3(gridr), dim3(SS / VV), ar, br, 0);
  cudaDeviceSynchronize();
  unsigned long long c[8];
  cudaMemcpyFromSymbol(c, g_phase_cycles, sizeof(c));
  const char* names[6] = {"normalize", "gram+max", "exp+z", "wout", "grad-loop", "combine"};
  unsigned long long tot = 0;
  for (int i = 0; i < 6; ++i) tot += c[i];
  printf("rt phases (cycles/eval, %d CTA/SM co-resident): total %.0f\n", orr, tot / (double)B);
  for (int i = 0; i < 6; ++i) printf("  %-10s %8.0f\n", names[i], c[i] / (double)B);
#endif
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) cudaLaunchKernel(fg, dim3(gridg), dim3(SS), ag, bg, 0);
  cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
  const double evg = (double)B * reps / (ms * 1e-3);
  printf("gs : %.3f ms/launch, %.4g evals/s, %.0f SM-cycles/eval\n", ms / reps, evg, 148 * 1.965e9 / evg);
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) cudaLaunchKernel(fr, dim3(gridr), dim3(SS / VV), ar, br, 0);
  cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
  const double evr = (double)B * reps / (ms * 1e-3);
  printf("rt : %.3f ms/launch, %.4g evals/s, %.0f SM-cycles/eval  (x%.2f)\n", ms / reps, evr, 148 * 1.965e9 / evr, evr / evg);
  return badg || badF;
}
