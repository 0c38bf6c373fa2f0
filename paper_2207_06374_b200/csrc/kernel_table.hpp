// Kernel-family dispatch: one instantiation per (field, d, S) for d = 1..8
// (exact, fully unrolled) and a runtime-d family for 9 <= d <= 16.  The
// instantiations live in instantiate.cu, compiled once per (field, S).
#pragma once

struct KernelSet {
  const void* anneal;
  const void* eval;
  const void* hvp;
  const void* coherence;
};

const KernelSet* trstmi_kernels_c_32(int d);
const KernelSet* trstmi_kernels_c_128(int d);
const KernelSet* trstmi_kernels_c_256(int d);
const KernelSet* trstmi_kernels_r_32(int d);
const KernelSet* trstmi_kernels_r_128(int d);
const KernelSet* trstmi_kernels_r_256(int d);

inline const KernelSet* find_kernels(bool cplx, int d, int S) {
  if (cplx) {
    if (S == 32) return trstmi_kernels_c_32(d);
    if (S == 128) return trstmi_kernels_c_128(d);
    if (S == 256) return trstmi_kernels_c_256(d);
  } else {
    if (S == 32) return trstmi_kernels_r_32(d);
    if (S == 128) return trstmi_kernels_r_128(d);
    if (S == 256) return trstmi_kernels_r_256(d);
  }
  return nullptr;
}
