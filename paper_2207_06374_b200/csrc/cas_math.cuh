// Canonical Arithmetic Spec (CAS) transcendentals on the device.
//
// The reference calls std::exp / std::log (smoothing.hpp:122,126).  glibc and
// libdevice differ by an ulp on some inputs, and the FD Hessian-vector product
// (smoothing.hpp:176-180) amplifies such differences ~1e5x, so decision parity
// with the CPU oracle needs ONE exp/log definition on both sides.  These are
// operation-for-operation the same as cas_exp / cas_log in the oracle
// (oracle/cas_oracle.hpp); the file is compiled with -fmad=false so only the
// explicit fma() sites fuse.  Accuracy vs correctly rounded: exp <= 0.85 ulp,
// log <= 1.8 ulp (tests/test_oracle_math.py).
#pragma once
#include <cstdint>
#include <limits>

namespace trstmi_dev {

// |re + i im| exactly as the reference computes it: std::abs(std::complex)
// (frame.hpp:87, coherence / offdiagonal_magnitudes) is glibc's hypot.  This
// restates glibc 2.39's __hypot (sysdeps/ieee754/dbl-64/e_hypot.c: the
// correction kernel of Borges, "An Improved Algorithm for hypot(a,b)",
// without FMA, with the 2^-600 scaling of huge / tiny inputs) operation for
// operation — bit-identical to the host libm on 4e5 random inputs spanning the
// exponent range (tests/test_oracle_cpu.py::test_cas_hypot_matches_libm).
// Compiled with -fmad=false: every product and sum below rounds separately.
__host__ __device__ inline double cas_hypot_kernel(double ax, double ay) {
  double h = sqrt(ax * ax + ay * ay);
  double t1, t2;
  if (h <= 2.0 * ay) {
    const double delta = h - ay;
    t1 = ax * (2.0 * delta - ax);
    t2 = (delta - 2.0 * (ax - ay)) * delta;
  } else {
    const double delta = h - ax;
    t1 = 2.0 * delta * (ax - 2.0 * ay);
    t2 = (4.0 * delta - ay) * ay + delta * delta;
  }
  h -= (t1 + t2) / (2.0 * h);
  return h;
}

__host__ __device__ inline double cas_hypot(double x, double y) {
  x = fabs(x);
  y = fabs(y);
  if (isinf(x) || isinf(y)) return std::numeric_limits<double>::infinity();
  if (isnan(x) || isnan(y)) return x + y;
  const double ax = x < y ? y : x, ay = x < y ? x : y;
  const double kScale = 0x1p-600, kLarge = 0x1p+511, kTiny = 0x1p-511, kEps = 0x1p-54;
  if (ax > kLarge) {
    if (ay <= ax * kEps) return ax + ay;
    return cas_hypot_kernel(ax * kScale, ay * kScale) / kScale;
  }
  if (ay < kTiny) {
    if (ax >= ay / kEps) return ax + ay;
    return cas_hypot_kernel(ax / kScale, ay / kScale) * kScale;
  }
  if (ay <= ax * kEps) return ax + ay;
  return cas_hypot_kernel(ax, ay);
}

__device__ __forceinline__ double pow2i(int k) {  // 2^k, -1022 <= k <= 1023
  return __longlong_as_double(static_cast<long long>(k + 1023) << 52);
}

// k = RNE(x log2 e) by the fma magic-constant trick (no FRND / F2I: both run
// at 1/4 of the DFMA rate on B200, scripts/micro/fp64_ops.cu); the scaling
// (p * 2^(k>>1)) * 2^(k-(k>>1)) is exact in the first product and rounds once,
// so every result (normal, subnormal or overflowing) is RN(p * 2^k).
// cas_exp_core is the formula on [-746.25, 709.78] — no compares, so several
// independent exps interleave; cas_exp adds the NaN / overflow / underflow
// cases.  Operation-for-operation the oracle's cas_exp_core / cas_exp.
// Polynomial / reduction constants in the constant bank: the DFMAs take them
// as c[][] operands instead of two UMOVs per constant inside a large kernel.
static __constant__ double kCasExpC[16] = {
    1.6059043836821613e-10,  2.08767569878680989792e-09, 2.50521083854417187751e-08,
    2.75573192239858906526e-07, 2.75573192239858906526e-06, 2.48015873015873015873e-05,
    1.98412698412698412698e-04, 1.38888888888888888889e-03, 8.33333333333333333333e-03,
    4.16666666666666666667e-02, 1.66666666666666666667e-01, 0.5, 1.0, 1.0,
    6.93147180369123816490e-01, 1.90821492927058770002e-10};

__device__ __forceinline__ double cas_exp_core(double x) {
  const double t = fma(x, 1.4426950408889634, 0x1.8p52);
  const double kd = __dsub_rn(t, 0x1.8p52);
  const int k = __double2loint(t);  // low word of t = k (two's complement)
  double r = fma(-kd, kCasExpC[14], x);
  r = fma(-kd, kCasExpC[15], r);
  double p = kCasExpC[0];
#pragma unroll
  for (int i = 1; i < 14; ++i) p = fma(p, r, kCasExpC[i]);
  const int k1 = k >> 1;
  return __dmul_rn(__dmul_rn(p, pow2i(k1)), pow2i(k - k1));
}

__device__ __forceinline__ double cas_exp(double x) {
  const double res = cas_exp_core(fmin(fmax(x, -746.25), 709.79));  // identity on the core domain
  if (!(x == x)) return x;
  if (x > 709.782712893383973096) return __longlong_as_double(0x7ff0000000000000LL);
  if (x < -746.25) return 0.0;
  return res;
}

__device__ __forceinline__ double cas_log(double x) {
  if (!(x == x) || x < 0.0) return __longlong_as_double(0x7ff8000000000000LL);
  if (x == 0.0) return __longlong_as_double(0xfff0000000000000LL);
  if (x == __longlong_as_double(0x7ff0000000000000LL)) return x;
  int e = 0;
  if (x < 0x1.0p-1022) {
    x = __dmul_rn(x, 0x1.0p54);
    e = -54;
  }
  unsigned long long bits = static_cast<unsigned long long>(__double_as_longlong(x));
  e += static_cast<int>((bits >> 52) & 0x7ff) - 1023;
  bits = (bits & 0x000fffffffffffffULL) | 0x3ff0000000000000ULL;
  double m = __longlong_as_double(static_cast<long long>(bits));
  if (m > 1.4142135623730951) {
    m = __dmul_rn(m, 0.5);
    e += 1;
  }
  const double f = __dsub_rn(m, 1.0);
  const double s = __ddiv_rn(f, __dadd_rn(2.0, f));
  const double s2 = __dmul_rn(s, s);
  double p = 1.0 / 25.0;
  p = fma(p, s2, 1.0 / 23.0);
  p = fma(p, s2, 1.0 / 21.0);
  p = fma(p, s2, 1.0 / 19.0);
  p = fma(p, s2, 1.0 / 17.0);
  p = fma(p, s2, 1.0 / 15.0);
  p = fma(p, s2, 1.0 / 13.0);
  p = fma(p, s2, 1.0 / 11.0);
  p = fma(p, s2, 1.0 / 9.0);
  p = fma(p, s2, 1.0 / 7.0);
  p = fma(p, s2, 1.0 / 5.0);
  p = fma(p, s2, 1.0 / 3.0);
  const double t = __dmul_rn(__dmul_rn(s, s2), p);
  const double logm = __dadd_rn(__dmul_rn(2.0, s), __dmul_rn(2.0, t));
  const double ed = static_cast<double>(e);
  return fma(ed, 6.93147180369123816490e-01, fma(ed, 1.90821492927058770002e-10, logm));
}

}  // namespace trstmi_dev
