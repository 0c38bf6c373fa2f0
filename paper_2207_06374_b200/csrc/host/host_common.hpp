// Host-side pieces of the hot path that stay on the CPU by design:
//  * the seeded start-frame generator (rng.hpp:13-64, solver.hpp:87-98) —
//    Box-Muller needs libm log/sin/cos, so frames are drawn here and uploaded;
//  * the stage-boundary column rescue (solver.hpp:139-156), which draws from
//    the same per-trial generator (rare: the kernel flags the trial and the
//    host redraws before resuming the stage on the GPU);
//  * default_delta_schedule (solver.hpp:64-82) and welch_bound
//    (analysis.hpp:27-31).
// Compiled with -ffp-contract=off; column norms use the CAS order (an fma
// chain over the column's doubles) so they agree bit-for-bit with the device.
#pragma once
#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <vector>

namespace trstmi_host {

constexpr double kZeroColumnTol = 1e-12;

inline std::uint64_t mix_seed(std::uint64_t seed, std::uint64_t index) {
  std::uint64_t z = seed + (index + 1) * 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

class SplitMix64 {
 public:
  explicit SplitMix64(std::uint64_t seed = 0) : state_(seed) {}
  std::uint64_t next_u64() {
    std::uint64_t z = (state_ += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
  }
  double uniform() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
  double normal() {
    if (has_spare_) {
      has_spare_ = false;
      return spare_;
    }
    double u1 = uniform();
    if (u1 <= 0.0) u1 = 0x1.0p-53;
    const double u2 = uniform();
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double theta = 2.0 * 3.14159265358979323846 * u2;
    spare_ = r * std::sin(theta);
    has_spare_ = true;
    return r * std::cos(theta);
  }
  void complex_normal(double* re, double* im) {
    const double a = normal();
    const double b = normal();
    *re = a * 0.70710678118654752440;
    *im = b * 0.70710678118654752440;
  }
  void save(std::uint64_t* st) const {
    st[0] = state_;
    st[1] = has_spare_ ? 1 : 0;
    std::memcpy(&st[2], &spare_, 8);
  }
  static SplitMix64 load(const std::uint64_t* st) {
    SplitMix64 r(st[0]);
    r.has_spare_ = st[1] != 0;
    std::memcpy(&r.spare_, &st[2], 8);
    return r;
  }

 private:
  std::uint64_t state_;
  bool has_spare_ = false;
  double spare_ = 0.0;
};

inline double column_norm(const double* c, std::int64_t len) {
  double acc = 0.0;
  for (std::int64_t q = 0; q < len; ++q) acc = std::fma(c[q], c[q], acc);
  return std::sqrt(acc);
}

inline void draw_column(bool cplx, std::int64_t d, double* c, SplitMix64& rng) {
  if (cplx) {
    for (std::int64_t i = 0; i < d; ++i) rng.complex_normal(&c[2 * i], &c[2 * i + 1]);
  } else {
    for (std::int64_t i = 0; i < d; ++i) c[i] = rng.normal();
  }
}

// random_frame (solver.hpp:87-98)
inline void random_frame(bool cplx, std::int64_t d, std::int64_t N, SplitMix64& rng, double* f) {
  const std::int64_t L = (cplx ? 2 : 1) * d;
  for (std::int64_t j = 0; j < N; ++j) {
    double* c = f + j * L;
    double nrm;
    do {
      draw_column(cplx, d, c, rng);
      nrm = column_norm(c, L);
    } while (nrm < kZeroColumnTol);
    for (std::int64_t q = 0; q < L; ++q) c[q] = c[q] / nrm;
  }
}

// rescue_zero_columns (solver.hpp:139-156).  Returns -1 or the column that
// could not be rescued (ZeroColumnError).
inline int rescue_zero_columns(bool cplx, std::int64_t d, std::int64_t N, double* param, SplitMix64* rng) {
  const std::int64_t L = (cplx ? 2 : 1) * d;
  for (std::int64_t j = 0; j < N; ++j) {
    double* c = param + j * L;
    if (column_norm(c, L) >= kZeroColumnTol) continue;
    bool rescued = false;
    for (int attempt = 0; rng != nullptr && attempt < 3; ++attempt) {
      draw_column(cplx, d, c, *rng);
      const double nrm = column_norm(c, L);
      if (nrm >= kZeroColumnTol) {
        for (std::int64_t q = 0; q < L; ++q) c[q] = c[q] / nrm;
        rescued = true;
        break;
      }
    }
    if (!rescued) return static_cast<int>(j);
  }
  return -1;
}

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

inline double welch_bound(std::int64_t d, std::int64_t N) {
  if (N <= d) return 0.0;
  return std::sqrt(static_cast<double>(N - d) / (static_cast<double>(d) * static_cast<double>(N - 1)));
}

}  // namespace trstmi_host
