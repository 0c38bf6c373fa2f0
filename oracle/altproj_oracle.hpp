// TEST INFRASTRUCTURE ONLY (see oracle/Makefile): CPU restatement of the reference's alternating-projection
// baseline, /root/reference/proj/include/trstmi/baseline.hpp:68-167 (alternating_projection) and :172-199
// (solve_altproj), the checker of trstmi_altproj_batch (csrc/altproj.cu).
//
// PARITY UNPINNED against the reference itself: the baseline's arithmetic lives in Eigen's
// SelfAdjointEigenSolver (Eigen 3.3+, unpinned, absent from this image; baseline.hpp also pulls analysis.hpp with
// Eigen/QR, beyond oracle/eigen_shim), so `oracle/_ref` cannot compile it.  What pins this restatement instead:
// the reference's own expectations for the path (tests/test_baseline.cpp, ported in tests/test_altproj*.py) and an
// independent numpy.linalg.eigh restatement at 1e-8 (tests/test_altproj_cpu.py).
//
// The Hermitian eigendecomposition the reference delegates to Eigen is fixed here as a two-sided cyclic Jacobi
// method in round-robin (tournament) order — the order a GPU runs it in: the M/2 disjoint rotations of a round are
// formed from the matrix at the start of the round, applied to the columns of W and V, then to the rows of W.
// Every operation below is a single rounding in the order written (the file is compiled with -ffp-contract=off;
// the device code with -fmad=false), so the GPU reproduces these results bit for bit.
#pragma once
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <vector>

#include "cas_oracle.hpp"

namespace orc {

struct AltProjCfg {  // AltProjConfig, baseline.hpp:22-26
  int max_iters = 300;
  double mu_target = 0.0;
  double tol = 1e-10;
};

struct AltProjOut {
  double coherence = 0.0;  // best_coherence (converged: the last iterate's)
  int iterations = 0;      // StageRecord::outer_iterations: +iterations when converged, -iterations otherwise
  int jacobi_sweeps = 0;   // total over the run (diagnostic)
  std::vector<double> frame;
};

constexpr int kJacobiMaxSweeps = 60;
constexpr double kJacobiRelTol2 = 1e-30;  // stop when max |W_pq|^2 <= 1e-30 * max W_pp^2

// Hermitian W (N x N, row-major, interleaved re/im) -> eigenvalues on its diagonal, eigenvectors in the columns of V.
inline int herm_jacobi(int N, std::vector<double>& W, std::vector<double>& V) {
  const int M = (N + 1) & ~1;
  auto w = [&](int i, int j) { return &W[2 * ((size_t)i * N + j)]; };
  auto v = [&](int i, int j) { return &V[2 * ((size_t)i * N + j)]; };
  for (int i = 0; i < N; ++i)
    for (int j = 0; j < N; ++j) {
      v(i, j)[0] = i == j ? 1.0 : 0.0;
      v(i, j)[1] = 0.0;
    }
  std::vector<int> P(M / 2), Q(M / 2);
  std::vector<double> C(M / 2), SR(M / 2), SI(M / 2);
  int sweeps = 0;
  for (; sweeps < kJacobiMaxSweeps; ++sweeps) {
    double off2 = 0.0, diag2 = 0.0;
    for (int i = 0; i < N; ++i)
      for (int j = 0; j < N; ++j) {
        const double* e = w(i, j);
        const double m2 = e[0] * e[0] + e[1] * e[1];
        if (i == j)
          diag2 = std::max(diag2, m2);
        else
          off2 = std::max(off2, m2);
      }
    if (off2 <= kJacobiRelTol2 * diag2) break;
    for (int r = 0; r < M - 1; ++r) {
      for (int i = 0; i < M / 2; ++i) {
        const int a = i == 0 ? M - 1 : (r + i) % (M - 1);
        const int b = i == 0 ? r : (r + M - 1 - i) % (M - 1);
        const int p = std::min(a, b), q = std::max(a, b);
        P[i] = p;
        Q[i] = q;
        C[i] = 1.0;
        SR[i] = SI[i] = 0.0;
        if (q >= N) continue;
        const double re = w(p, q)[0], im = w(p, q)[1];
        const double bm = std::sqrt(re * re + im * im);
        if (bm == 0.0) continue;
        const double tau = (w(q, q)[0] - w(p, p)[0]) / (2.0 * bm);
        const double t = (tau < 0.0 ? -1.0 : 1.0) / (std::fabs(tau) + std::sqrt(1.0 + tau * tau));
        const double c = 1.0 / std::sqrt(1.0 + t * t);
        const double s = t * c;
        C[i] = c;
        SR[i] = s * (re / bm);
        SI[i] = s * (im / bm);
      }
      // columns of W and V: (x, y) <- (x c - y (sr - i si)^*..., ...) with J_pq = s e, J_qp = -s conj(e)
      for (int i = 0; i < M / 2; ++i) {
        const int p = P[i], q = Q[i];
        if (q >= N || (SR[i] == 0.0 && SI[i] == 0.0)) continue;
        const double c = C[i], sr = SR[i], si = SI[i];
        for (int mat = 0; mat < 2; ++mat)
          for (int row = 0; row < N; ++row) {
            double* x = mat ? v(row, p) : w(row, p);
            double* y = mat ? v(row, q) : w(row, q);
            const double xr = x[0], xi = x[1], yr = y[0], yi = y[1];
            x[0] = (xr * c - yr * sr) - yi * si;
            x[1] = (xi * c + yr * si) - yi * sr;
            y[0] = (xr * sr - xi * si) + yr * c;
            y[1] = (xr * si + xi * sr) + yi * c;
          }
      }
      // rows of W
      for (int i = 0; i < M / 2; ++i) {
        const int p = P[i], q = Q[i];
        if (q >= N || (SR[i] == 0.0 && SI[i] == 0.0)) continue;
        const double c = C[i], sr = SR[i], si = SI[i];
        for (int col = 0; col < N; ++col) {
          double* x = w(p, col);
          double* y = w(q, col);
          const double xr = x[0], xi = x[1], yr = y[0], yi = y[1];
          x[0] = (c * xr - sr * yr) + si * yi;
          x[1] = (c * xi - sr * yi) - si * yr;
          y[0] = (sr * xr + si * xi) + c * yr;
          y[1] = (sr * xi - si * xr) + c * yi;
        }
      }
      for (int i = 0; i < M / 2; ++i) {
        const int p = P[i], q = Q[i];
        if (q >= N || (SR[i] == 0.0 && SI[i] == 0.0)) continue;
        w(p, q)[0] = w(p, q)[1] = 0.0;
        w(q, p)[0] = w(q, p)[1] = 0.0;
        w(p, p)[1] = 0.0;
        w(q, q)[1] = 0.0;
      }
    }
  }
  return sweeps;
}

// alternating_projection (baseline.hpp:68-167) from a given start frame (random_frame(d, N, rng), drawn by the caller).
inline AltProjOut altproj_run(int d, int N, const AltProjCfg& cfg, const double* start) {
  Shape sh;  // complex frame; coherence() uses no CAS reduction width
  sh.complex_field = true;
  sh.d = d;
  sh.N = N;
  const int L = 2 * d;
  const double welch = N > d ? std::sqrt((double)(N - d) / ((double)d * (double)(N - 1))) : 0.0;  // analysis.hpp:27-31
  const double mu_target = cfg.mu_target > 0.0 ? cfg.mu_target : std::max(welch, 1e-12);
  std::vector<double> G(2 * (size_t)N * N), W, V(2 * (size_t)N * N), Pm(2 * (size_t)N * N);
  auto g = [&](int i, int j) { return &G[2 * ((size_t)i * N + j)]; };
  // gram_matrix(current) (frame.hpp:73-75), CAS order per entry; Hermitian by mirroring
  for (int j = 0; j < N; ++j)
    for (int k = j; k < N; ++k) {
      double re = 0.0, im = 0.0;
      for (int i = 0; i < d; ++i) {
        const double ar = start[j * L + 2 * i], ai = start[j * L + 2 * i + 1];
        const double br = start[k * L + 2 * i], bi = start[k * L + 2 * i + 1];
        re = std::fma(ar, br, re);
        re = std::fma(ai, bi, re);
        im = std::fma(ar, bi, im);
        im = std::fma(-ai, br, im);
      }
      if (j == k) im = 0.0;
      g(j, k)[0] = re;
      g(j, k)[1] = im;
      g(k, j)[0] = re;
      g(k, j)[1] = -im;
    }
  AltProjOut out;
  std::vector<double> best(start, start + (size_t)L * N), last = best, fac((size_t)L * N);
  double best_mu = coherence(sh, start, false).mu, last_mu = best_mu;
  bool converged = false;
  int iterations = 0;
  for (int it = 0; it < cfg.max_iters; ++it) {
    iterations = it + 1;
    // (a) structural projection (baseline.hpp:96-106)
    for (int j = 0; j < N; ++j) {
      g(j, j)[0] = 1.0;
      g(j, j)[1] = 0.0;
      for (int k = j + 1; k < N; ++k) {
        const double mag = cas_hypot(g(j, k)[0], g(j, k)[1]);
        if (mag > mu_target) {
          const double f = mu_target / mag;
          g(j, k)[0] *= f;
          g(j, k)[1] *= f;
          g(k, j)[0] = g(j, k)[0];
          g(k, j)[1] = -g(j, k)[1];
        }
      }
    }
    // (b) spectral projection (baseline.hpp:110-121)
    W = G;
    out.jacobi_sweeps += herm_jacobi(N, W, V);
    std::vector<int> top(d);
    {
      std::vector<int> idx(N);
      for (int i = 0; i < N; ++i) idx[i] = i;
      std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) {
        return W[2 * ((size_t)a * N + a)] > W[2 * ((size_t)b * N + b)];
      });
      for (int i = 0; i < d; ++i) top[i] = idx[i];
    }
    std::fill(Pm.begin(), Pm.end(), 0.0);
    for (int j = 0; j < N; ++j)
      for (int k = j; k < N; ++k) {
        double ar = 0.0, ai = 0.0;
        for (int i = 0; i < d; ++i) {
          const int e = top[i];
          const double lam = std::max(W[2 * ((size_t)e * N + e)], 0.0);
          const double vjr = V[2 * ((size_t)j * N + e)], vji = V[2 * ((size_t)j * N + e) + 1];
          const double vkr = V[2 * ((size_t)k * N + e)], vki = V[2 * ((size_t)k * N + e) + 1];
          const double pr = vjr * vkr + vji * vki;
          const double pi = vji * vkr - vjr * vki;
          ar = ar + lam * pr;
          ai = ai + lam * pi;
        }
        Pm[2 * ((size_t)j * N + k)] = ar;
        Pm[2 * ((size_t)j * N + k) + 1] = ai;
        Pm[2 * ((size_t)k * N + j)] = ar;
        Pm[2 * ((size_t)k * N + j) + 1] = -ai;
      }
    for (int i = 0; i < d; ++i) {
      const int e = top[i];
      const double sl = std::sqrt(std::max(W[2 * ((size_t)e * N + e)], 0.0));
      for (int j = 0; j < N; ++j) {
        fac[j * L + 2 * i] = sl * V[2 * ((size_t)j * N + e)];
        fac[j * L + 2 * i + 1] = sl * (-V[2 * ((size_t)j * N + e) + 1]);
      }
    }
    // normalize_columns + coherence (baseline.hpp:123-132); a zero column skips the update
    {
      const CoherenceResult c = coherence(sh, fac.data(), true);
      if (c.zero_col < 0) {
        last = fac;
        for (int j = 0; j < N; ++j) {  // normalize_columns (frame.hpp:60-69): CAS norm, IEEE division
          double acc = 0.0;
          for (int q = 0; q < L; ++q) acc = std::fma(fac[j * L + q], fac[j * L + q], acc);
          const double a = std::sqrt(acc);
          for (int q = 0; q < L; ++q) last[j * L + q] = fac[j * L + q] / a;
        }
        last_mu = c.mu;
        if (last_mu < best_mu) {
          best_mu = last_mu;
          best = last;
        }
      }
    }
    double change = 0.0;
    for (size_t e = 0; e < (size_t)N * N; ++e)
      change = std::max(change, cas_hypot(Pm[2 * e] - G[2 * e], Pm[2 * e + 1] - G[2 * e + 1]));
    G = Pm;
    if (change <= cfg.tol) {
      converged = true;
      break;
    }
  }
  out.coherence = converged ? last_mu : best_mu;
  out.frame = converged ? last : best;
  out.iterations = converged ? iterations : -iterations;
  return out;
}

}  // namespace orc
