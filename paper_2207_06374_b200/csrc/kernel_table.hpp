// Kernel-family dispatch: one instantiation per (field, d, S, layout) for
// d = 1..8 (exact, fully unrolled) and a runtime-d family for 9 <= d <= 16.
// Layout g = stored Gram (small_gs.cuh), r = Gram recomputed in the gradient
// (small_path.cuh eval_cta).  The instantiations live in instantiate.cu,
// compiled once per (field, S, layout); build.py lists the compiled set.
#pragma once

struct KernelSet {
  const void* anneal;
  const void* eval;
  const void* hvp;
  const void* coherence;
};

#define TRSTMI_DECL(f, s, l) const KernelSet* trstmi_kernels_##f##_##s##_##l(int d);
TRSTMI_DECL(c, 64, g)
TRSTMI_DECL(c, 128, g)
TRSTMI_DECL(c, 128, r)
TRSTMI_DECL(c, 256, g)
TRSTMI_DECL(c, 256, r)
TRSTMI_DECL(c, 512, g)
TRSTMI_DECL(r, 64, g)
TRSTMI_DECL(r, 128, g)
TRSTMI_DECL(r, 128, r)
TRSTMI_DECL(r, 256, g)
TRSTMI_DECL(r, 256, r)
TRSTMI_DECL(r, 512, g)
#undef TRSTMI_DECL

inline const KernelSet* find_kernels(bool cplx, int d, int S, int gs) {
  if (cplx) {
    if (S == 64 && gs) return trstmi_kernels_c_64_g(d);
    if (S == 128) return gs ? trstmi_kernels_c_128_g(d) : trstmi_kernels_c_128_r(d);
    if (S == 256) return gs ? trstmi_kernels_c_256_g(d) : trstmi_kernels_c_256_r(d);
    if (S == 512 && gs) return trstmi_kernels_c_512_g(d);
  } else {
    if (S == 64 && gs) return trstmi_kernels_r_64_g(d);
    if (S == 128) return gs ? trstmi_kernels_r_128_g(d) : trstmi_kernels_r_128_r(d);
    if (S == 256) return gs ? trstmi_kernels_r_256_g(d) : trstmi_kernels_r_256_r(d);
    if (S == 512 && gs) return trstmi_kernels_r_512_g(d);
  }
  return nullptr;
}
