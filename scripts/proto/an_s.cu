// Config-2 anneal harness (complex d=2, N=100, S=512, stored Gram): runs anneal_small_kernel on seeded Gaussian
// start frames and prints throughput, a hash of every output, and (with -DTRSTMI_PHASE_TIMERS) where the cycles go.
// usage: an_s TRIALS STAGES [MAX_OUTER]
#include "anneal_small.cuh"
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
using namespace trstmi_dev;
#ifndef SS
#define SS 512
#endif
#ifndef NN
#define NN 100
#endif
#ifndef DD
#define DD 2
#endif
int main(int argc, char** argv) {
  const int T = atoi(argv[1]), ns = atoi(argv[2]), mo = argc > 3 ? atoi(argv[3]) : 500;
  const int N = NN, d = DD;
  AnnealArgs A; memset(&A, 0, sizeof(A));
  A.P = make_small_prob(true, d, N, kchunks_for(d, N, SS), 1, 1);
#ifdef DUAL
  A.P.dual = DUAL;
#endif
  const int dim = A.P.dim;
  std::vector<double> sched;
  const double term = 1e-7 / (2.0 * log((double)N));
  for (double dl = 0.1; dl > term * (1 + 1e-12); dl /= 10) sched.push_back(dl);
  sched.push_back(term);
  A.n_stages = ns < (int)sched.size() ? ns : (int)sched.size();
  for (int k = 0; k < A.n_stages; ++k) A.schedule[k] = sched[k];
  A.tr.delta0 = 0.1 * sqrt((double)dim); A.tr.delta_max = 1e3; A.tr.eta = 0.05; A.tr.shrink = 0.25; A.tr.grow = 2.0;
  A.tr.grad_tol = 1e-9; A.tr.cg_force_c = 0.5; A.tr.max_outer = mo; A.tr.max_cg = 2 * dim;
  A.n_list = T;
  std::vector<double> h((size_t)T * dim);
  unsigned long long st = 88172645463325252ULL;
  auto u01 = [&]() { st ^= st << 13; st ^= st >> 7; st ^= st << 17; return ((st >> 11) + 0.5) / 9007199254740992.0; };
  for (auto& v : h) v = sqrt(-2.0 * log(u01())) * cos(6.283185307179586 * u01()) * 0.7071067811865476;
  for (int t = 0; t < T; ++t) for (int j = 0; j < N; ++j) {
    double a = 0; for (int q = 0; q < A.P.L; ++q) a += h[(size_t)t * dim + j * A.P.L + q] * h[(size_t)t * dim + j * A.P.L + q];
    a = sqrt(a); for (int q = 0; q < A.P.L; ++q) h[(size_t)t * dim + j * A.P.L + q] /= a;
  }
  cudaMalloc(&A.params, h.size() * 8); cudaMemcpy(A.params, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  cudaMalloc(&A.frames, h.size() * 8);
  cudaMalloc(&A.tout, T * sizeof(trstmi_trial_out)); cudaMalloc(&A.sout, (size_t)T * A.n_stages * sizeof(trstmi_stage_out));
  cudaMalloc(&A.counter, 4); cudaMemset(A.counter, 0, 4);
  const void* fn = (const void*)&anneal_small_kernel<true, DD, true, SS, true>;
  const size_t bytes = anneal_smem_doubles(A.P, SS, true) * 8;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  void* args[] = {&A};
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  cudaEventRecord(e0);
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, SS, bytes);
  const int grid = T < 148 * per_sm ? T : 148 * per_sm;
  printf("CTAs per SM %d, grid %d\n", per_sm, grid);
  cudaLaunchKernel(fn, dim3(grid), dim3(SS), args, bytes, 0);
  cudaEventRecord(e1); cudaError_t e2 = cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
  std::vector<trstmi_trial_out> to(T); cudaMemcpy(to.data(), A.tout, T * sizeof(trstmi_trial_out), cudaMemcpyDeviceToHost);
  std::vector<double> fr(h.size()); cudaMemcpy(fr.data(), A.frames, h.size() * 8, cudaMemcpyDeviceToHost);
  long long outer = 0, evals = 0, bad = 0;
  unsigned long long hash = 1469598103934665603ULL;
  auto mix = [&](unsigned long long b) { hash = (hash ^ b) * 1099511628211ULL; };
  for (auto& o : to) { outer += o.outer_iterations; evals += o.evals; bad += o.status != 0; unsigned long long b; memcpy(&b, &o.coherence, 8); mix(b); mix(o.outer_iterations); mix(o.evals); mix(o.argmax_pair); }
  for (double v : fr) { unsigned long long b; memcpy(&b, &v, 8); mix(b); }
  printf("anneal S=%d N=%d T=%d stages=%d smem %zu (%s / %s): %.3f s, outer %lld (%.4g it/s), evals %lld (%.4g /s), bad %lld, hash %016llx\n",
         SS, N, T, A.n_stages, bytes, cudaGetErrorString(e), cudaGetErrorString(e2), ms * 1e-3, outer, outer / (ms * 1e-3), evals, evals / (ms * 1e-3), bad, hash);
#ifdef TRSTMI_PHASE_TIMERS
  unsigned long long c[8]; cudaMemcpyFromSymbol(c, g_phase_cycles, sizeof(c));
  const char* names[6] = {"normalize", "gram+max", "exp", "zsum", "grad-loop", "combine"};
  unsigned long long tot = 0; for (int i = 0; i < 6; ++i) tot += c[i];
  printf("  cycles/eval: trial total %.0f, eval phases %.0f, outside eval %.0f\n", c[7] / (double)evals, tot / (double)evals, (c[7] - tot) / (double)evals);
  for (int i = 0; i < 6; ++i) printf("  %-10s %8.0f\n", names[i], c[i] / (double)evals);
#endif
}
