// Instantiates the small-frame kernel families for one (field, S), selected
// by -DINST_CPLX=0/1 -DINST_S=32/128/256 (see build.py).
#include "batch_kernels.cuh"
#include "kernel_table.hpp"

#ifndef INST_CPLX
#error "define INST_CPLX"
#endif
#ifndef INST_S
#error "define INST_S"
#endif

#define CAT2(a, b) a##b
#define CAT(a, b) CAT2(a, b)
#if INST_CPLX
#define TABLE_FN CAT(trstmi_kernels_c_, INST_S)
#else
#define TABLE_FN CAT(trstmi_kernels_r_, INST_S)
#endif

using namespace trstmi_dev;

template <int D, bool EXACT>
static KernelSet make_set() {
  KernelSet k;
  k.anneal = (const void*)&anneal_small_kernel<(INST_CPLX != 0), D, EXACT, INST_S>;
  k.eval = (const void*)&eval_batch_kernel<(INST_CPLX != 0), D, EXACT, INST_S>;
  k.hvp = (const void*)&hvp_batch_kernel<(INST_CPLX != 0), D, EXACT, INST_S>;
  k.coherence = (const void*)&coherence_batch_kernel<(INST_CPLX != 0), D, EXACT, INST_S>;
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
