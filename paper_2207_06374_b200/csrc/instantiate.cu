// Instantiates the small-frame kernel families for one (field, S, layout),
// selected by -DINST_CPLX=0/1 -DINST_S=32/128/256/512 -DINST_GS=0/1 (see
// build.py; GS = stored-Gram layout, small_gs.cuh).
#include "batch_kernels.cuh"
#include "kernel_table.hpp"

#ifndef INST_CPLX
#error "define INST_CPLX"
#endif
#ifndef INST_S
#error "define INST_S"
#endif
#ifndef INST_GS
#error "define INST_GS"
#endif

#define CAT2(a, b) a##b
#define CAT(a, b) CAT2(a, b)
#if INST_GS
#define LAYOUT _g
#else
#define LAYOUT _r
#endif
#if INST_CPLX
#define TABLE_FN CAT(CAT(trstmi_kernels_c_, INST_S), LAYOUT)
#else
#define TABLE_FN CAT(CAT(trstmi_kernels_r_, INST_S), LAYOUT)
#endif

using namespace trstmi_dev;

template <int D, bool EXACT>
static KernelSet make_set() {
  KernelSet k;
  k.anneal = (const void*)&anneal_small_kernel<(INST_CPLX != 0), D, EXACT, INST_S, (INST_GS != 0)>;
  k.eval = (const void*)&eval_batch_kernel<(INST_CPLX != 0), D, EXACT, INST_S, (INST_GS != 0)>;
  k.hvp = (const void*)&hvp_batch_kernel<(INST_CPLX != 0), D, EXACT, INST_S, (INST_GS != 0)>;
  k.coherence = (const void*)&coherence_batch_kernel<(INST_CPLX != 0), D, EXACT, INST_S, (INST_GS != 0)>;
  return k;
}

const KernelSet* TABLE_FN(int d) {
  static const KernelSet table[9] = {make_set<1, true>(), make_set<2, true>(), make_set<3, true>(),
                                     make_set<4, true>(), make_set<5, true>(), make_set<6, true>(),
                                     make_set<7, true>(), make_set<8, true>(), make_set<16, false>()};
  if (d >= 1 && d <= 8) return &table[d - 1];
  if (d >= 9 && d <= 16) return &table[8];
  return nullptr;
}
