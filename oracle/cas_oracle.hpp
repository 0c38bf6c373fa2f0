// ============================================================================
//  TEST INFRASTRUCTURE ONLY — CPU oracle for the TRST-MI hot path.
//
//  This header is a restatement, in plain C++ (no Eigen), of the reference
//  library's hot path (/root/reference/proj/include/trstmi/*.hpp), written to
//  the Canonical Arithmetic Spec (CAS) that fixes every
//  floating-point order the reference leaves to Eigen.  It is the CHECKER for
//  the CUDA product and the CPU baseline arm of bench.py; nothing in the
//  product path (paper_2207_06374_b200/) includes, links or calls it.
//
//  Compile with -ffp-contract=off (oracle/Makefile): every fused multiply-add
//  below is an explicit std::fma at a CAS-named site; every other a*b+c is two
//  roundings, exactly like the device code compiled with -fmad=false.
//
//  Parity pins: the reference cannot be built here (Eigen 3 absent, see
//  DESIGN.md §5), and it ships no golden vectors.  The oracle is pinned by
//  the reference's own known-answer and property tests for this path, ported
//  in oracle/tests/oracle_tests.cpp (test_smoothing.cpp, test_trust_region.cpp,
//  test_solver.cpp, test_frames.cpp, acceptance_main.cpp criteria 1/7/8/9/11).
// ============================================================================
#pragma once

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <functional>
#include <limits>
#include <stdexcept>
#include <string>
#include <thread>
#include <utility>
#include <vector>

namespace orc {

using Vec = std::vector<double>;

// ---------------------------------------------------------------- RNG
// rng.hpp:13-18
inline std::uint64_t mix_seed(std::uint64_t seed, std::uint64_t index) {
  std::uint64_t z = seed + (index + 1) * 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

// rng.hpp:22-64 (SplitMix64 + Box-Muller, cos first, sin cached)
struct Rng {
  std::uint64_t state = 0;
  bool has_spare = false;
  double spare = 0.0;
  explicit Rng(std::uint64_t seed = 0) : state(seed) {}
  std::uint64_t next_u64() {
    std::uint64_t z = (state += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
  }
  double uniform() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
  double normal() {
    if (has_spare) {
      has_spare = false;
      return spare;
    }
    double u1 = uniform();
    if (u1 <= 0.0) u1 = 0x1.0p-53;
    const double u2 = uniform();
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double theta = 2.0 * 3.14159265358979323846 * u2;
    spare = r * std::sin(theta);
    has_spare = true;
    return r * std::cos(theta);
  }
  void complex_normal(double* re, double* im) {
    constexpr double inv_sqrt2 = 0.70710678118654752440;
    const double a = normal();
    const double b = normal();
    *re = a * inv_sqrt2;
    *im = b * inv_sqrt2;
  }
};

// ---------------------------------------------------------------- constants
constexpr double kZeroColumnTol = 1e-12;               // frame.hpp:20
constexpr double kFdBaseStep = 0x1.965fea53d6e3dp-18;  // smoothing.hpp:16-17, glibc cbrt(DBL_EPSILON)
// exp((u-s)/delta) is exactly 0 once (u-s)/delta < -745.2; the CAS skips the
// pair when u - s < kUnderflowCut * delta (a superset test).
constexpr double kUnderflowCut = -746.0;

// ---------------------------------------------------------------- CAS math
// CAS exp: k = round-to-nearest-even(x log2 e) by the fma magic-constant
// trick (t = fma(x, log2e, 1.5*2^52), kd = t - 1.5*2^52, k = low word of t),
// Cody-Waite reduction with an fma split of ln2, degree-13 Taylor in
// Horner/fma form, scaling (p * 2^(k>>1)) * 2^(k-(k>>1)) (the first product
// exact, one rounding, also for subnormal results).  cas_exp_core is the
// formula on [-746.25, 709.78]; cas_exp adds NaN / overflow / underflow.
// No rint/float<->int conversion and no compares in the core: those run at
// 1/4 of the FP64 rate on B200 (scripts/micro/fp64_ops.cu).  Bit-identical to
// the device cas_exp in paper_2207_06374_b200/csrc/cas_math.cuh; <= 1 ulp
// from glibc exp in the tests (tests/test_oracle_cpu.py).
inline double pow2i(int k) {  // 2^k for -1022 <= k <= 1023, exact
  std::uint64_t bits = static_cast<std::uint64_t>(k + 1023) << 52;
  double r;
  std::memcpy(&r, &bits, 8);
  return r;
}

inline double cas_exp_core(double x) {
  const double t = std::fma(x, 1.4426950408889634, 0x1.8p52);
  const double kd = t - 0x1.8p52;
  std::uint64_t tb;
  std::memcpy(&tb, &t, 8);
  const int k = static_cast<int>(static_cast<std::uint32_t>(tb));  // low word = k (two's complement)
  double r = std::fma(-kd, 6.93147180369123816490e-01, x);
  r = std::fma(-kd, 1.90821492927058770002e-10, r);
  double p = 1.6059043836821613e-10;            // 1/13!
  p = std::fma(p, r, 2.08767569878680989792e-09);  // 1/12!
  p = std::fma(p, r, 2.50521083854417187751e-08);  // 1/11!
  p = std::fma(p, r, 2.75573192239858906526e-07);  // 1/10!
  p = std::fma(p, r, 2.75573192239858906526e-06);  // 1/9!
  p = std::fma(p, r, 2.48015873015873015873e-05);  // 1/8!
  p = std::fma(p, r, 1.98412698412698412698e-04);  // 1/7!
  p = std::fma(p, r, 1.38888888888888888889e-03);  // 1/6!
  p = std::fma(p, r, 8.33333333333333333333e-03);  // 1/5!
  p = std::fma(p, r, 4.16666666666666666667e-02);  // 1/4!
  p = std::fma(p, r, 1.66666666666666666667e-01);  // 1/3!
  p = std::fma(p, r, 0.5);
  p = std::fma(p, r, 1.0);
  p = std::fma(p, r, 1.0);
  const int k1 = k >> 1;  // arithmetic shift: floor(k / 2)
  return (p * pow2i(k1)) * pow2i(k - k1);  // exact, then one rounding
}

inline double cas_exp(double x) {
  if (!(x == x)) return x;
  if (x > 709.782712893383973096) return std::numeric_limits<double>::infinity();
  if (x < -746.25) return 0.0;
  return cas_exp_core(x);
}

// CAS log (used once per evaluation, for F = s + delta*log z with z >= 1):
// x = 2^e m, m in [sqrt(1/2), sqrt(2)), log m = 2 atanh(f/(2+f)) by an odd
// series in Horner/fma form, plus e*ln2 split hi/lo.
// |re + i im| for coherence / offdiagonal_magnitudes: std::abs(complex) is
// glibc's hypot (frame.hpp:87).  Restatement of glibc 2.39 __hypot
// (sysdeps/ieee754/dbl-64/e_hypot.c, the non-FMA correction kernel of Borges,
// "An Improved Algorithm for hypot(a,b)", with the 2^-600 scaling);
// -ffp-contract=off keeps every operation separately rounded.  Mirrors
// cas_hypot in csrc/cas_math.cuh.
inline double cas_hypot_kernel(double ax, double ay) {
  double h = std::sqrt(ax * ax + ay * ay);
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

inline double cas_hypot(double x, double y) {
  x = std::fabs(x);
  y = std::fabs(y);
  if (std::isinf(x) || std::isinf(y)) return std::numeric_limits<double>::infinity();
  if (std::isnan(x) || std::isnan(y)) return x + y;
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

inline double cas_log(double x) {
  if (!(x == x) || x < 0.0) return std::numeric_limits<double>::quiet_NaN();
  if (x == 0.0) return -std::numeric_limits<double>::infinity();
  if (x == std::numeric_limits<double>::infinity()) return x;
  int e = 0;
  if (x < 0x1.0p-1022) {
    x *= 0x1.0p54;
    e = -54;
  }
  std::uint64_t bits;
  std::memcpy(&bits, &x, 8);
  e += static_cast<int>((bits >> 52) & 0x7ff) - 1023;
  bits = (bits & 0x000fffffffffffffULL) | 0x3ff0000000000000ULL;
  double m;
  std::memcpy(&m, &bits, 8);
  if (m > 1.4142135623730951) {
    m = m * 0.5;
    e += 1;
  }
  const double f = m - 1.0;
  const double s = f / (2.0 + f);
  const double s2 = s * s;
  double p = 1.0 / 25.0;
  p = std::fma(p, s2, 1.0 / 23.0);
  p = std::fma(p, s2, 1.0 / 21.0);
  p = std::fma(p, s2, 1.0 / 19.0);
  p = std::fma(p, s2, 1.0 / 17.0);
  p = std::fma(p, s2, 1.0 / 15.0);
  p = std::fma(p, s2, 1.0 / 13.0);
  p = std::fma(p, s2, 1.0 / 11.0);
  p = std::fma(p, s2, 1.0 / 9.0);
  p = std::fma(p, s2, 1.0 / 7.0);
  p = std::fma(p, s2, 1.0 / 5.0);
  p = std::fma(p, s2, 1.0 / 3.0);
  const double t = s * s2 * p;          // s^3 (1/3 + s^2/5 + ...)
  const double logm = 2.0 * s + 2.0 * t;
  const double ed = static_cast<double>(e);
  return std::fma(ed, 6.93147180369123816490e-01,
                  std::fma(ed, 1.90821492927058770002e-10, logm));
}

// ---------------------------------------------------------------- CAS sums
// Lane-strided reduction of width S (a power of two >= 32): lane l
// accumulates elements l, l+S, l+2S, ... in ascending order starting from +0;
// each group of 32 lanes is combined by an xor butterfly (offsets
// 16,8,4,2,1); the S/32 group totals are then combined by the same butterfly
// across groups (group offsets 1,2,4,...), i.e. a pairwise tree in group
// order.  This is the order a CTA of S threads produces with
// __shfl_xor_sync inside each warp and again across the warp totals.
inline double butterfly_combine(std::vector<double>& lane, int S) {
  const int W = S / 32;
  std::vector<double> tot(W);
  for (int w = 0; w < W; ++w) {
    double a[32];
    for (int l = 0; l < 32; ++l) a[l] = lane[w * 32 + l];
    for (int off = 16; off >= 1; off >>= 1) {
      double b[32];
      for (int l = 0; l < 32; ++l) b[l] = a[l] + a[l ^ off];
      for (int l = 0; l < 32; ++l) a[l] = b[l];
    }
    tot[w] = a[0];
  }
  for (int off = 1; off < W; off <<= 1) {
    std::vector<double> b(W);
    for (int w = 0; w < W; ++w) b[w] = tot[w] + tot[w ^ off];
    tot = b;
  }
  return tot[0];
}

inline double cas_sum(const double* v, std::int64_t n, int S) {
  std::vector<double> lane(S, 0.0);
  for (std::int64_t p = 0; p < n; ++p) lane[p % S] = lane[p % S] + v[p];
  return butterfly_combine(lane, S);
}

inline double cas_dot(const double* a, const double* b, std::int64_t n, int S) {
  std::vector<double> lane(S, 0.0);
  for (std::int64_t p = 0; p < n; ++p) lane[p % S] = std::fma(a[p], b[p], lane[p % S]);
  return butterfly_combine(lane, S);
}

inline double cas_norm(const Vec& v, int S) { return std::sqrt(cas_dot(v.data(), v.data(), (std::int64_t)v.size(), S)); }
inline double cas_sqnorm(const Vec& v, int S) { return cas_dot(v.data(), v.data(), (std::int64_t)v.size(), S); }
inline double cas_vdot(const Vec& a, const Vec& b, int S) { return cas_dot(a.data(), b.data(), (std::int64_t)a.size(), S); }

// ---------------------------------------------------------------- problem
struct Shape {
  bool complex_field = true;  // false: real lines (new mode)
  std::int64_t d = 0, N = 0;
  int lanes = 32;             // CAS reduction width S (trstmi_lanes())
  int kchunks = 1;            // CAS gradient k-chunks K (trstmi_kchunks())
  int zrows = 0;              // large path: z over row blocks of zrows rows (0: one lane-strided sum)
  std::int64_t comps() const { return complex_field ? 2 : 1; }
  std::int64_t col_len() const { return comps() * d; }  // doubles per column
  std::int64_t dim() const { return col_len() * N; }
  std::int64_t pairs() const { return N * (N - 1) / 2; }
};

// Column norm (Eigen col(j).norm(), frame.hpp:64 / smoothing.hpp:97):
// CAS = sqrt of an fma chain over the column's doubles in ascending order.
inline double column_norm(const double* col, std::int64_t len) {
  double acc = 0.0;
  for (std::int64_t q = 0; q < len; ++q) acc = std::fma(col[q], col[q], acc);
  return std::sqrt(acc);
}

// Gram entry G(j,k) = <phi_j, phi_k> (conjugate-linear in the first argument,
// frame.hpp:73-75).  CAS: ascending i, fma in the order below.  G(k,j) is
// defined as conj(G(j,k)) for j < k.
inline void gram_entry(const Shape& sh, const double* a, const double* b, double* gre, double* gim) {
  double re = 0.0, im = 0.0;
  if (sh.complex_field) {
    for (std::int64_t i = 0; i < sh.d; ++i) {
      const double ar = a[2 * i], ai = a[2 * i + 1], br = b[2 * i], bi = b[2 * i + 1];
      re = std::fma(ar, br, re);
      re = std::fma(ai, bi, re);
      im = std::fma(ar, bi, im);
      im = std::fma(-ai, br, im);
    }
  } else {
    for (std::int64_t i = 0; i < sh.d; ++i) re = std::fma(a[i], b[i], re);
  }
  *gre = re;
  *gim = im;
}

inline std::int64_t pair_index(std::int64_t N, std::int64_t j, std::int64_t k) {  // j < k
  return j * N - j * (j + 1) / 2 + (k - j - 1);
}

struct EvalResult {
  int zero_col = -1;  // first zero column (ZeroColumnError), -1 if none
  double value = 0.0, s = 0.0;
  Vec grad;
  Vec weights;        // softmax weights (ObjectiveEval::softmax_weights)
};

// eval_objective (smoothing.hpp:82-162) at p = x + sc*dir (sc == 0: p = x).
inline EvalResult eval_objective(const Shape& sh, const double* x, const double* dir, double sc,
                                 double delta, bool squared = true, bool want_weights = false) {
  EvalResult out;
  const std::int64_t N = sh.N, L = sh.col_len(), n = sh.pairs();
  Vec phi(sh.dim()), alpha(N);
  for (std::int64_t j = 0; j < N; ++j) {
    double col[2 * 4096];
    double* c = (L <= 2 * 4096) ? col : nullptr;
    Vec big;
    if (!c) {
      big.resize(L);
      c = big.data();
    }
    for (std::int64_t q = 0; q < L; ++q) {
      const double xv = x[j * L + q];
      c[q] = (sc == 0.0) ? xv : xv + sc * dir[j * L + q];
    }
    alpha[j] = column_norm(c, L);
    if (alpha[j] < kZeroColumnTol) {  // smoothing.hpp:98
      out.zero_col = static_cast<int>(j);
      return out;
    }
    for (std::int64_t q = 0; q < L; ++q) phi[j * L + q] = c[q] / alpha[j];
  }
  // Gram (upper triangle, row-major pair order), x_p, s
  Vec gre(n), gim(n), xv(n);
  for (std::int64_t j = 0, p = 0; j < N; ++j)
    for (std::int64_t k = j + 1; k < N; ++k, ++p) {
      gram_entry(sh, &phi[j * L], &phi[k * L], &gre[p], &gim[p]);
      const double u = gre[p] * gre[p] + gim[p] * gim[p];
      xv[p] = squared ? u : std::sqrt(u);
    }
  double s = -std::numeric_limits<double>::infinity();
  for (std::int64_t p = 0; p < n; ++p) s = std::max(s, xv[p]);
  // weights, z, F (smoothing.hpp:118-126)
  Vec w(n);
  const double cut = kUnderflowCut * delta;
  for (std::int64_t p = 0; p < n; ++p) {
    const double diff = xv[p] - s;
    w[p] = (diff < cut) ? 0.0 : cas_exp(diff / delta);
  }
  // z (smoothing.hpp:121-124) in the CAS order: small path — one lane-strided
  // sum of width S over all pairs; large path — the pairs of each block of
  // zrows consecutive rows (a contiguous pair range) summed with 256 lanes,
  // block sums added in row order (so any row-block sharding is exact).
  double z;
  if (sh.zrows > 0) {
    z = 0.0;
    for (std::int64_t r0 = 0, b = 0; r0 < N; r0 += sh.zrows, ++b) {
      const std::int64_t r1 = std::min<std::int64_t>(N, r0 + sh.zrows);
      const std::int64_t p0 = r0 * N - r0 * (r0 + 1) / 2, p1 = r1 * N - r1 * (r1 + 1) / 2;
      const double zb = cas_sum(w.data() + p0, p1 - p0, 256);
      z = (b == 0) ? zb : z + zb;
    }
  } else {
    z = cas_sum(w.data(), n, sh.lanes);
  }
  for (std::int64_t p = 0; p < n; ++p) w[p] = w[p] / z;
  out.s = s;
  out.value = s + delta * cas_log(z);
  // gradient (smoothing.hpp:130-160): per column m, k ascending, c == 0 skipped
  out.grad.assign(sh.dim(), 0.0);
  std::vector<double> acc(L);
  // Gradient (smoothing.hpp:130-160) in the CAS order: for each column m the
  // k-range is split into K = sh.kchunks contiguous chunks
  // [c*N/K, (c+1)*N/K); inside a chunk t_m and the GEMM sums Phi * coeff
  // (Eigen, smoothing.hpp:147) are ascending-k chains from +0 (t by add of
  // c*u, the GEMM by fma); chunk partials are added left to right.
  const int K = sh.kchunks;
  std::vector<double> part(L);
  for (std::int64_t m = 0; m < N; ++m) {
    double t = 0.0;
    std::fill(acc.begin(), acc.end(), 0.0);
    for (int ch = 0; ch < K; ++ch) {
      double tp = 0.0;
      std::fill(part.begin(), part.end(), 0.0);
      const std::int64_t k_lo = (ch * N) / K, k_hi = ((ch + 1) * N) / K;
      for (std::int64_t k = k_lo; k < k_hi; ++k) {
        if (k == m) continue;
        const std::int64_t p = (k < m) ? pair_index(N, k, m) : pair_index(N, m, k);
        double c = w[p];
        if (c == 0.0) continue;
        const double Gr = gre[p];
        const double Gi = (k < m) ? gim[p] : -gim[p];  // G(k,m)
        const double u = Gr * Gr + Gi * Gi;
        if (!squared) c = c * (0.5 / std::max(std::sqrt(u), 1e-150));
        tp = tp + c * u;
        const double cr = c * Gr, ci = c * Gi;
        const double* pk = &phi[k * L];
        if (sh.complex_field) {
          for (std::int64_t i = 0; i < sh.d; ++i) {
            const double pr = pk[2 * i], pi = pk[2 * i + 1];
            part[2 * i] = std::fma(pr, cr, part[2 * i]);
            part[2 * i] = std::fma(-pi, ci, part[2 * i]);
            part[2 * i + 1] = std::fma(pr, ci, part[2 * i + 1]);
            part[2 * i + 1] = std::fma(pi, cr, part[2 * i + 1]);
          }
        } else {
          for (std::int64_t i = 0; i < sh.d; ++i) part[i] = std::fma(pk[i], cr, part[i]);
        }
      }
      t = (ch == 0) ? tp : t + tp;
      for (std::int64_t q = 0; q < L; ++q) acc[q] = (ch == 0) ? part[q] : acc[q] + part[q];
    }
    const double* pm = &phi[m * L];
    for (std::int64_t q = 0; q < L; ++q) out.grad[m * L + q] = ((acc[q] - t * pm[q]) / alpha[m]) * 2.0;
  }
  if (want_weights) out.weights = std::move(w);
  return out;
}

// -------------------------------------------------------------- coherence
// coherence (frame.hpp:138-145) with the argmax pair (first strict maximum in
// row-major upper-triangular order).  |G| := sqrt(re*re + im*im) (CAS).
struct CoherenceResult {
  int zero_col = -1;
  double mu = 0.0;
  std::int64_t argmax = -1;
};

inline CoherenceResult coherence(const Shape& sh, const double* frame, bool normalize) {
  CoherenceResult r;
  const std::int64_t N = sh.N, L = sh.col_len();
  Vec phi(frame, frame + sh.dim());
  if (normalize) {  // normalize_columns (frame.hpp:60-69)
    for (std::int64_t j = 0; j < N; ++j) {
      const double a = column_norm(&frame[j * L], L);
      if (a < kZeroColumnTol) {
        r.zero_col = static_cast<int>(j);
        return r;
      }
      for (std::int64_t q = 0; q < L; ++q) phi[j * L + q] = frame[j * L + q] / a;
    }
  }
  for (std::int64_t j = 0, p = 0; j < N; ++j)
    for (std::int64_t k = j + 1; k < N; ++k, ++p) {
      double gr, gi;
      gram_entry(sh, &phi[j * L], &phi[k * L], &gr, &gi);
      const double m = cas_hypot(gr, gi);  // std::abs = hypot (frame.hpp:87)
      if (m > r.mu) {
        r.mu = m;
        r.argmax = p;
      }
    }
  return r;
}

inline double welch_bound(std::int64_t d, std::int64_t N) {  // analysis.hpp:27-31
  if (N <= d) return 0.0;
  return std::sqrt(static_cast<double>(N - d) / (static_cast<double>(d) * static_cast<double>(N - 1)));
}

// ---------------------------------------------------------------- HVP
enum HvpPath { HVP_CENTRAL = 0, HVP_FORWARD = 1, HVP_BACKWARD = 2, HVP_ZERO_DIR = 3, HVP_FAILED = -1 };

// make_hvp_factory (solver.hpp:118-137) around fd_hessian_vector_product
// (smoothing.hpp:167-181).  g0 is the gradient at x (the TR driver passes its
// current gradient, bit-identical to eval_objective(x).grad).
struct HvpResult {
  int path = HVP_CENTRAL;
  int zero_col = -1;
  int evals = 0;
  Vec hv;
};

inline HvpResult hvp_adapter(const Shape& sh, const Vec& x, const Vec& dir, double delta, const Vec* g0_in) {
  HvpResult r;
  const std::int64_t dim = sh.dim();
  const double dn = cas_norm(dir, sh.lanes);
  if (dn == 0.0) {
    r.path = HVP_ZERO_DIR;
    r.hv.assign(dim, 0.0);
    return r;
  }
  const double h = kFdBaseStep * (1.0 + cas_norm(x, sh.lanes)) / std::max(dn, 1e-300);
  EvalResult gp = eval_objective(sh, x.data(), dir.data(), h, delta);
  r.evals++;
  if (gp.zero_col < 0) {
    EvalResult gm = eval_objective(sh, x.data(), dir.data(), -h, delta);
    r.evals++;
    r.hv.resize(dim);
    if (gm.zero_col < 0) {
      const double h2 = 2.0 * h;
      for (std::int64_t i = 0; i < dim; ++i) r.hv[i] = (gp.grad[i] - gm.grad[i]) / h2;
      r.path = HVP_CENTRAL;
      return r;
    }
    Vec g0;
    if (g0_in) g0 = *g0_in; else { g0 = eval_objective(sh, x.data(), nullptr, 0.0, delta).grad; r.evals++; }
    r.evals++;  // solver.hpp:130 re-evaluates x + h*dir (the value of gp)
    for (std::int64_t i = 0; i < dim; ++i) r.hv[i] = (gp.grad[i] - g0[i]) / h;
    r.path = HVP_FORWARD;
    return r;
  }
  // forward point failed: g0, retry forward (fails identically), then backward
  Vec g0;
  if (g0_in) g0 = *g0_in; else { g0 = eval_objective(sh, x.data(), nullptr, 0.0, delta).grad; r.evals++; }
  r.evals++;  // solver.hpp:131 re-evaluates x + h*dir, which fails again
  EvalResult gm = eval_objective(sh, x.data(), dir.data(), -h, delta);
  r.evals++;
  if (gm.zero_col >= 0) {
    r.path = HVP_FAILED;
    r.zero_col = gm.zero_col;
    return r;
  }
  r.hv.resize(dim);
  for (std::int64_t i = 0; i < dim; ++i) r.hv[i] = (g0[i] - gm.grad[i]) / h;
  r.path = HVP_BACKWARD;
  return r;
}

// ---------------------------------------------------------- trust region
struct TrustRegionConfig {  // trust_region.hpp:20-30
  double delta0 = 0.0;
  double delta_max = 1e3;
  double eta = 0.05;
  double shrink = 0.25;
  double grow = 2.0;
  double grad_tol = 1e-9;
  int max_outer = 200;
  double cg_force_c = 0.5;
  int max_cg = 0;
};

enum CgExit { CG_SMALL_RESIDUAL = 0, CG_NEGATIVE_CURVATURE = 1, CG_BOUNDARY_HIT = 2, CG_ZERO_GRADIENT = 3 };

struct CgTrace {
  int iterations = 0;
  int exit_reason = CG_SMALL_RESIDUAL;
  double step_norm = 0.0;
  bool converged = true;
  double model_value = 0.0;
};

struct Evaluation {
  double value = 0.0;
  Vec grad;
};

// Callable seam, trust_region.hpp:42-49.  The hvp callable may throw
// HvpFailure (a ZeroColumnError escaping make_hvp_factory's fallback).
struct HvpFailure : std::runtime_error {
  int column;
  explicit HvpFailure(int c) : std::runtime_error("column " + std::to_string(c) + " has near-zero norm"), column(c) {}
};
using Objective = std::function<Evaluation(const Vec&)>;
using HvpOperator = std::function<Vec(const Vec&)>;
using HvpFactory = std::function<HvpOperator(const Vec&)>;

// detail::boundary_roots (trust_region.hpp:56-69)
inline std::pair<double, double> boundary_roots(const Vec& z, const Vec& d, double radius, int S) {
  const double a = cas_sqnorm(d, S);
  const double b = 2.0 * cas_vdot(z, d, S);
  const double c = cas_sqnorm(z, S) - radius * radius;
  if (a <= 0.0) return {0.0, 0.0};
  const double disc = std::sqrt(std::max(b * b - 4.0 * a * c, 0.0));
  const double q = -0.5 * (b + std::copysign(disc, b));
  double r1 = q != 0.0 ? c / q : 0.0;
  double r2 = a != 0.0 ? q / a : 0.0;
  if (r1 > r2) std::swap(r1, r2);
  return {r1, r2};
}

// steihaug_cg (trust_region.hpp:81-154)
inline std::pair<Vec, CgTrace> steihaug_cg(const Vec& grad, const HvpOperator& hvp, double radius, double eps_k,
                                           int max_cg, int S) {
  if (radius <= 0.0) throw std::invalid_argument("steihaug_cg: radius <= 0");
  if (eps_k < 0.0) throw std::invalid_argument("steihaug_cg: eps_k < 0");
  const std::size_t dim = grad.size();
  Vec z(dim, 0.0);
  CgTrace trace;
  const double grad_norm = cas_norm(grad, S);
  if (grad_norm < eps_k || grad_norm == 0.0) {
    trace.exit_reason = CG_ZERO_GRADIENT;
    return {z, trace};
  }
  Vec r = grad, d(dim);
  for (std::size_t i = 0; i < dim; ++i) d[i] = -grad[i];
  double rr = cas_sqnorm(r, S);
  double model = 0.0;
  Vec zn(dim);
  for (int j = 0; j < max_cg; ++j) {
    const Vec bd = hvp(d);
    const double dbd = cas_vdot(d, bd, S);
    const double rd = cas_vdot(r, d, S);
    if (dbd <= 0.0) {
      const auto [tau_lo, tau_hi] = boundary_roots(z, d, radius, S);
      const double m_lo = model + tau_lo * rd + 0.5 * tau_lo * tau_lo * dbd;
      const double m_hi = model + tau_hi * rd + 0.5 * tau_hi * tau_hi * dbd;
      const double tau = m_lo < m_hi ? tau_lo : tau_hi;
      for (std::size_t i = 0; i < dim; ++i) z[i] = z[i] + tau * d[i];
      trace.iterations = j;
      trace.exit_reason = CG_NEGATIVE_CURVATURE;
      trace.step_norm = cas_norm(z, S);
      trace.model_value = std::min(m_lo, m_hi);
      return {z, trace};
    }
    const double alpha = rr / dbd;
    for (std::size_t i = 0; i < dim; ++i) zn[i] = z[i] + alpha * d[i];
    if (cas_norm(zn, S) >= radius) {
      const double tau = boundary_roots(z, d, radius, S).second;
      for (std::size_t i = 0; i < dim; ++i) z[i] = z[i] + tau * d[i];
      trace.iterations = j;
      trace.exit_reason = CG_BOUNDARY_HIT;
      trace.step_norm = cas_norm(z, S);
      trace.model_value = model + tau * rd + 0.5 * tau * tau * dbd;
      return {z, trace};
    }
    model += alpha * rd + 0.5 * alpha * alpha * dbd;
    z = zn;
    for (std::size_t i = 0; i < dim; ++i) r[i] = r[i] + alpha * bd[i];
    const double rr_next = cas_sqnorm(r, S);
    trace.iterations = j + 1;
    if (std::sqrt(rr_next) < eps_k) {
      trace.exit_reason = CG_SMALL_RESIDUAL;
      trace.step_norm = cas_norm(z, S);
      trace.model_value = model;
      return {z, trace};
    }
    const double beta = rr_next / rr;
    rr = rr_next;
    for (std::size_t i = 0; i < dim; ++i) d[i] = -r[i] + beta * d[i];
  }
  trace.exit_reason = CG_SMALL_RESIDUAL;
  trace.converged = false;
  trace.step_norm = cas_norm(z, S);
  trace.model_value = model;
  return {z, trace};
}

enum MinimizeStatus { ST_GRADIENT_TOLERANCE = 0, ST_ITERATION_LIMIT = 1, ST_RADIUS_UNDERFLOW = 2, ST_STALLED = 3 };

struct OuterRecord {  // trust_region.hpp:163-173
  int iteration = 0;
  double value = 0.0, grad_norm = 0.0, radius = 0.0, rho = 0.0;
  bool accepted = false;
  int cg_exit = CG_SMALL_RESIDUAL;
  int cg_iterations = 0;
  double step_norm = 0.0;
};

struct MinimizeResult {
  Vec x;
  double value = 0.0, grad_norm = 0.0;
  int status = ST_ITERATION_LIMIT;
  std::vector<OuterRecord> history;
};

inline bool all_finite(const Vec& v) {
  for (double a : v)
    if (!std::isfinite(a)) return false;
  return true;
}

// trust_region_minimize (trust_region.hpp:189-295)
inline MinimizeResult trust_region_minimize(const Objective& objective, const HvpFactory& make_hvp, Vec x0,
                                            TrustRegionConfig cfg, int S) {
  const std::size_t dim = x0.size();
  if (cfg.delta0 == 0.0) cfg.delta0 = 0.1 * std::sqrt(static_cast<double>(dim));
  if (cfg.max_cg == 0) cfg.max_cg = static_cast<int>(2 * dim);
  if (!(cfg.delta0 > 0.0) || cfg.delta0 > cfg.delta_max)
    throw std::invalid_argument("trust_region_minimize: need 0 < delta0 <= delta_max");
  if (!(cfg.eta >= 0.0 && cfg.eta < 0.25)) throw std::invalid_argument("trust_region_minimize: need 0 <= eta < 1/4");
  if (!(cfg.shrink > 0.0 && cfg.shrink < 1.0 && cfg.grow > 1.0))
    throw std::invalid_argument("trust_region_minimize: need 0 < shrink < 1 < grow");
  Evaluation current = objective(x0);
  if (!std::isfinite(current.value) || !all_finite(current.grad))
    throw std::invalid_argument("trust_region_minimize: objective not finite at x0");
  MinimizeResult result;
  result.x = x0;
  result.value = current.value;
  result.grad_norm = cas_norm(current.grad, S);
  result.status = ST_ITERATION_LIMIT;
  Vec x = std::move(x0);
  double radius = cfg.delta0;
  Vec trial(dim);
  for (int iter = 0; iter < cfg.max_outer; ++iter) {
    const double grad_norm = cas_norm(current.grad, S);
    if (grad_norm <= cfg.grad_tol) {
      result.status = ST_GRADIENT_TOLERANCE;
      break;
    }
    const double eps_k = std::min(cfg.cg_force_c, std::sqrt(grad_norm)) * grad_norm;
    const HvpOperator hvp = make_hvp(x);
    auto [step, trace] = steihaug_cg(current.grad, hvp, radius, eps_k, cfg.max_cg, S);
    OuterRecord rec;
    rec.iteration = iter;
    rec.value = current.value;
    rec.grad_norm = grad_norm;
    rec.radius = radius;
    rec.cg_exit = trace.exit_reason;
    rec.cg_iterations = trace.iterations;
    rec.step_norm = trace.step_norm;
    const double predicted = -trace.model_value;
    if (trace.exit_reason == CG_ZERO_GRADIENT || predicted <= 0.0) {
      radius *= cfg.shrink;
      rec.rho = 0.0;
      result.history.push_back(rec);
      if (radius < 1e-16) {
        result.status = ST_RADIUS_UNDERFLOW;
        break;
      }
      continue;
    }
    for (std::size_t i = 0; i < dim; ++i) trial[i] = x[i] + step[i];
    Evaluation trial_eval = objective(trial);
    const bool finite = std::isfinite(trial_eval.value) && all_finite(trial_eval.grad);
    const double rho = finite ? (current.value - trial_eval.value) / predicted : -std::numeric_limits<double>::infinity();
    rec.rho = rho;
    if (finite && trial_eval.value < result.value) {
      result.x = trial;
      result.value = trial_eval.value;
      result.grad_norm = cas_norm(trial_eval.grad, S);
    }
    if (rho > cfg.eta) {
      x = trial;
      current = std::move(trial_eval);
      rec.accepted = true;
    }
    if (rho < 0.25) {
      radius *= cfg.shrink;
    } else if (rho > 0.75 && trace.step_norm >= (1.0 - 1e-10) * radius) {
      radius = std::min(cfg.grow * radius, cfg.delta_max);
    }
    result.history.push_back(rec);
    if (radius < 1e-16) {
      result.status = ST_RADIUS_UNDERFLOW;
      break;
    }
  }
  if (current.value < result.value) {
    result.x = x;
    result.value = current.value;
    result.grad_norm = cas_norm(current.grad, S);
  }
  return result;
}

// ------------------------------------------------------------- solver
// default_delta_schedule (solver.hpp:64-82)
inline std::vector<double> default_delta_schedule(std::int64_t N, double eps_target) {
  if (N < 2) throw std::invalid_argument("default_delta_schedule: need N >= 2");
  if (eps_target <= 0.0) throw std::invalid_argument("default_delta_schedule: eps_target <= 0");
  const double terminal = eps_target / (2.0 * std::log(static_cast<double>(N)));
  std::vector<double> schedule;
  if (terminal >= 1e-1) return {10.0 * terminal, terminal};
  for (double delta = 1e-1; delta > terminal * (1.0 + 1e-12); delta /= 10.0) schedule.push_back(delta);
  schedule.push_back(terminal);
  return schedule;
}

// random_frame (solver.hpp:87-98); real mode draws normal() per entry.
inline Vec random_frame(const Shape& sh, Rng& rng) {
  const std::int64_t L = sh.col_len();
  Vec f(sh.dim());
  for (std::int64_t j = 0; j < sh.N; ++j) {
    double* c = &f[j * L];
    double nrm;
    do {
      if (sh.complex_field) {
        for (std::int64_t i = 0; i < sh.d; ++i) rng.complex_normal(&c[2 * i], &c[2 * i + 1]);
      } else {
        for (std::int64_t i = 0; i < sh.d; ++i) c[i] = rng.normal();
      }
      nrm = column_norm(c, L);
    } while (nrm < kZeroColumnTol);
    for (std::int64_t q = 0; q < L; ++q) c[q] = c[q] / nrm;
  }
  return f;
}

struct ZeroColumnFailure : std::runtime_error {
  int column;
  explicit ZeroColumnFailure(int c) : std::runtime_error("column " + std::to_string(c) + " has near-zero norm"), column(c) {}
};

// detail::rescue_zero_columns (solver.hpp:139-156)
inline void rescue_zero_columns(const Shape& sh, Vec& param, Rng* rng) {
  const std::int64_t L = sh.col_len();
  for (std::int64_t j = 0; j < sh.N; ++j) {
    double* c = &param[j * L];
    if (column_norm(c, L) >= kZeroColumnTol) continue;
    bool rescued = false;
    for (int attempt = 0; rng != nullptr && attempt < 3; ++attempt) {
      if (sh.complex_field) {
        for (std::int64_t i = 0; i < sh.d; ++i) rng->complex_normal(&c[2 * i], &c[2 * i + 1]);
      } else {
        for (std::int64_t i = 0; i < sh.d; ++i) c[i] = rng->normal();
      }
      const double nrm = column_norm(c, L);
      if (nrm >= kZeroColumnTol) {
        for (std::int64_t q = 0; q < L; ++q) c[q] = c[q] / nrm;
        rescued = true;
        break;
      }
    }
    if (!rescued) throw ZeroColumnFailure(static_cast<int>(j));
  }
}

struct StageRecord {  // solver.hpp:31-36
  double delta = 0.0, objective = 0.0, coherence = 0.0;
  int outer_iterations = 0;
  std::int64_t argmax = -1;
  int status = ST_ITERATION_LIMIT;
};

struct Counters {
  std::int64_t evals = 0;       // evaluator calls (x0 + trial + 2 per hvp + fallback)
  std::int64_t outer = 0;       // outer iterations (OuterRecord count)
  std::int64_t cg = 0;          // hvp calls
};

struct AnnealResult {
  Vec param;   // raw best-seen parameter after the last stage
  Vec frame;   // normalize_columns(param)
  double mu = 0.0;
  std::int64_t argmax = -1;
  std::vector<StageRecord> stages;
  std::vector<OuterRecord> history;  // concatenated over stages
  std::vector<int> history_stage;
  Counters counters;
};

struct SolverConfig {  // solver.hpp:21-29
  Shape shape;
  std::vector<double> delta_schedule;
  int restarts = 20;
  std::uint64_t seed = 0;
  TrustRegionConfig tr;
  double eps_target = 1e-7;
};

inline Objective make_objective(const Shape& sh, double delta, Counters* cnt) {  // solver.hpp:104-114
  return [sh, delta, cnt](const Vec& p) -> Evaluation {
    if (cnt) cnt->evals++;
    EvalResult e = eval_objective(sh, p.data(), nullptr, 0.0, delta);
    if (e.zero_col >= 0) return {std::numeric_limits<double>::infinity(), Vec(p.size(), 0.0)};
    return {e.value, std::move(e.grad)};
  };
}

// make_hvp_factory (solver.hpp:118-137).  The fallback's g0 is re-evaluated
// exactly as the reference does (the result equals the current gradient).
inline HvpFactory make_hvp_factory(const Shape& sh, double delta, Counters* cnt) {
  return [sh, delta, cnt](const Vec& x) -> HvpOperator {
    return [sh, delta, cnt, x](const Vec& dir) -> Vec {
      HvpResult r = hvp_adapter(sh, x, dir, delta, nullptr);
      if (cnt) {
        cnt->evals += r.evals;
        cnt->cg++;
      }
      if (r.path == HVP_FAILED) throw HvpFailure(r.zero_col);
      return r.hv;
    };
  };
}

// anneal (solver.hpp:164-204).  Writes into `out` stage by stage so a caller
// catching a failure still sees the completed stages; *stage_at tracks the
// stage in progress.
inline void anneal_into(const Vec& start, const SolverConfig& cfg, Rng* rescue_rng, bool keep_history,
                        AnnealResult& out, int* stage_at) {
  const Shape& sh = cfg.shape;
  std::vector<double> schedule = cfg.delta_schedule;
  if (schedule.empty()) schedule = default_delta_schedule(sh.N, cfg.eps_target);
  for (std::size_t k = 0; k + 1 < schedule.size(); ++k)
    if (!(schedule[k] > schedule[k + 1]) || schedule[k + 1] <= 0.0)
      throw std::invalid_argument("anneal: schedule must be strictly decreasing and positive");
  Vec param = start;
  for (std::size_t k = 0; k < schedule.size(); ++k) {
    if (stage_at) *stage_at = static_cast<int>(k);
    rescue_zero_columns(sh, param, rescue_rng);
    TrustRegionConfig tr = cfg.tr;
    tr.max_outer = cfg.tr.max_outer + 50 * static_cast<int>(k);
    MinimizeResult res = trust_region_minimize(make_objective(sh, schedule[k], &out.counters),
                                               make_hvp_factory(sh, schedule[k], &out.counters),
                                               std::move(param), tr, sh.lanes);
    param = std::move(res.x);
    StageRecord rec;
    rec.delta = schedule[k];
    rec.objective = res.value;
    CoherenceResult c = coherence(sh, param.data(), true);
    if (c.zero_col >= 0) throw ZeroColumnFailure(c.zero_col);
    rec.coherence = c.mu;
    rec.argmax = c.argmax;
    rec.outer_iterations = static_cast<int>(res.history.size());
    rec.status = res.status;
    out.counters.outer += rec.outer_iterations;
    out.stages.push_back(rec);
    if (keep_history) {
      for (OuterRecord h : res.history) out.history.push_back(h);
      out.history_stage.insert(out.history_stage.end(), res.history.size(), static_cast<int>(k));
    }
  }
  if (stage_at) *stage_at = -1;
  out.param = param;
  const std::int64_t L = sh.col_len();
  out.frame.resize(sh.dim());
  for (std::int64_t j = 0; j < sh.N; ++j) {
    const double a = column_norm(&param[j * L], L);
    if (a < kZeroColumnTol) throw ZeroColumnFailure(static_cast<int>(j));
    for (std::int64_t q = 0; q < L; ++q) out.frame[j * L + q] = param[j * L + q] / a;
  }
  CoherenceResult c = coherence(sh, out.frame.data(), false);
  out.mu = c.mu;
  out.argmax = c.argmax;
}

inline AnnealResult anneal(const Vec& start, const SolverConfig& cfg, Rng* rescue_rng, bool keep_history = false) {
  AnnealResult out;
  anneal_into(start, cfg, rescue_rng, keep_history, out, nullptr);
  return out;
}

struct RestartRecord {  // solver.hpp:38-45
  int restart_index = 0;
  std::uint64_t seed = 0;
  double coherence = 0.0;
  std::int64_t argmax = -1;
  bool succeeded = false;
  std::string error;
  std::vector<StageRecord> stages;
  Counters counters;
};

struct SolveResult {  // solver.hpp:47-54
  Vec best_frame;
  double best_coherence = 0.0;
  int best_restart = -1;
  std::vector<RestartRecord> per_restart;
  double wall_time_seconds = 0.0;
};

// solve (solver.hpp:210-273) over restarts [first, first+count) of the seed's
// child-seed sequence (count = cfg.restarts when first == 0).
inline SolveResult solve(const SolverConfig& cfg, int threads, std::int64_t first = 0) {
  const Shape& sh = cfg.shape;
  if (sh.d < 1 || sh.N < 1) throw std::invalid_argument("solve: need d, N >= 1");
  if (cfg.restarts < 1) throw std::invalid_argument("solve: need restarts >= 1");
  SolveResult result;
  result.per_restart.resize(cfg.restarts);
  std::vector<Vec> frames(cfg.restarts);
  auto run_restart = [&](int i) {
    RestartRecord& rec = result.per_restart[i];
    rec.restart_index = i;
    rec.seed = mix_seed(cfg.seed, static_cast<std::uint64_t>(first + i));
    try {
      Rng rng(rec.seed);
      Vec start = random_frame(sh, rng);
      AnnealResult a = anneal(start, cfg, &rng);
      rec.coherence = a.mu;
      rec.argmax = a.argmax;
      rec.stages = std::move(a.stages);
      rec.counters = a.counters;
      rec.succeeded = true;
      frames[i] = std::move(a.frame);
    } catch (const std::exception& e) {
      rec.succeeded = false;
      rec.error = e.what();
    }
  };
  const int workers = std::max(1, std::min(threads, cfg.restarts));
  if (workers == 1) {
    for (int i = 0; i < cfg.restarts; ++i) run_restart(i);
  } else {
    std::atomic<int> next{0};
    std::vector<std::thread> pool;
    for (int w = 0; w < workers; ++w)
      pool.emplace_back([&] {
        for (int i = next.fetch_add(1); i < cfg.restarts; i = next.fetch_add(1)) run_restart(i);
      });
    for (auto& t : pool) t.join();
  }
  for (int i = 0; i < cfg.restarts; ++i) {
    const RestartRecord& rec = result.per_restart[i];
    if (!rec.succeeded) continue;
    if (result.best_restart < 0 || rec.coherence < result.best_coherence) {
      result.best_restart = i;
      result.best_coherence = rec.coherence;
    }
  }
  if (result.best_restart < 0) throw std::runtime_error("solve: all restarts failed");
  result.best_frame = frames[result.best_restart];
  return result;
}

}  // namespace orc
