// Batched anneal, small-frame path: one persistent CTA per SM slot pulls
// trial indices from an atomic counter (the restart thread pool of
// solver.hpp:239-254 moved onto the SMs) and runs the whole anneal of that
// trial — every stage's trust-region loop, every Steihaug-CG iteration, every
// finite-difference Hessian-vector product — with its state resident in
// shared memory.  No host round trip per iteration.
//
// The scalar control flow is a line-by-line restatement of
//   trust_region_minimize  trust_region.hpp:189-295
//   steihaug_cg            trust_region.hpp:81-154
//   boundary_roots         trust_region.hpp:56-69
//   make_hvp_factory       solver.hpp:118-137
//   anneal                 solver.hpp:164-204
// evaluated redundantly (and identically) by every thread of the CTA from
// CTA-reduced values, so all branches are block-uniform.
#pragma once
#include "small_gs.cuh"

namespace trstmi_dev {

struct TrCfg {  // TrustRegionConfig, resolved (trust_region.hpp:194-195)
  double delta0, delta_max, eta, shrink, grow, grad_tol, cg_force_c;
  int max_outer, max_cg;
};

struct AnnealArgs {
  Prob P;
  TrCfg tr;
  int n_stages;
  double schedule[TRSTMI_MAX_STAGES];
  int record_cap;
  int n_list;               // trials to run in this launch
  const int* list;          // nullable: trial ids (else 0..n_list-1)
  const int* start_stage;   // nullable: per-trial first stage (resume after a rescue)
  int* counter;             // work counter, zeroed before launch
  double* params;           // trials x dim (in: start, out: best-seen raw param)
  double* frames;           // nullable: trials x dim normalised final frames
  trstmi_trial_out* tout;
  trstmi_stage_out* sout;   // trials x n_stages
  trstmi_outer_out* oout;   // nullable: trials x record_cap
};

// extra doubles of the dual layout: phiS grows to a second phiC (column stride gs_col_stride(L)), a second alpha,
// one double of alignment
__host__ __device__ inline long long dual_smem_doubles(const Prob& P) {
  return (P.gs && P.dual) ? (long long)(gs_col_stride(P.L) - P.L) * P.N + P.N + 1 : 0;
}


// doubles of shared memory the anneal kernel needs for a shape
__host__ __device__ inline long long smem_doubles(const Prob& P, int S, bool cplx, int nvec) {
  const int W = S / 32;
  return (long long)P.L * P.N + P.N + pair_smem_doubles(P, cplx) + 1 + 2LL * 4 * W + 4 + (long long)nvec * P.dim + W +
         dual_smem_doubles(P);
}
__host__ __device__ inline long long anneal_smem_doubles(const Prob& P, int S, bool cplx) {
  return smem_doubles(P, S, cplx, 9);
}

template <bool CPLX>
__device__ __forceinline__ void carve(const Prob& P, int S, double* base, Smem& sm, double** vecs, int nvec) {
  const int W = S / 32;
  double* p = base;
  if (P.gs) {  // stored-Gram layout (small_gs.cuh), 16-byte aligned arrays first; pair_smem_doubles() counts it
    sm.GRI = p;
    p += ((long long)P.np * (CPLX ? 2 : 1) + 1) & ~1LL;
    sm.phiC = p;
    p += ((long long)gs_col_stride(P.L) * P.N + 1) & ~1LL;
    sm.fk = reinterpret_cast<int*>(p);
    p += (P.N + 1) / 2;
  } else {
    sm.GRI = sm.phiC = nullptr;
    sm.fk = nullptr;
  }
  if (P.gs && P.dual) p += (p - base) & 1;  // 16-byte aligned: phiS doubles as the second phiC
  sm.phiS = p;
  p += (P.gs && P.dual) ? gs_col_stride(P.L) * P.N : P.L * P.N;
  sm.alpha = p;
  p += P.N;
  sm.alpha2 = nullptr;
  if (P.gs && P.dual) {
    sm.alpha2 = p;
    p += P.N;
  }
  sm.U = p;
  p += P.gs ? P.np : P.n;
  sm.part = p;
  p += (long long)P.K * P.N * (P.L + 1);
  sm.mask = reinterpret_cast<unsigned*>(p);
  p += ((long long)P.N * mask_words(P.N) + 1) / 2;
  sm.jk = reinterpret_cast<unsigned*>(p);
  p += ((long long)P.n + 1) / 2;
  sm.red = p;
  p += 2 * 4 * W;
  sm.scal = p;
  p += 4;
  for (int v = 0; v < nvec; ++v) {
    vecs[v] = p;
    p += P.dim;
  }
  sm.ired = reinterpret_cast<int*>(p);
}

template <int S>
__device__ __forceinline__ void vcopy(double* dst, const double* src, int n) {
  for (int i = threadIdx.x; i < n; i += S) dst[i] = src[i];
}

// all-finite flag of a vector, CTA-wide (1 = all finite)
template <int S>
__device__ __forceinline__ int all_finite(const double* v, int n, const Smem& sm, int& rbuf) {
  int ok = 1;
  for (int i = threadIdx.x; i < n; i += S) ok &= isfinite(v[i]) ? 1 : 0;
  return block_min_int<S>(ok, sm.ired, rbuf);
}

template <bool CPLX, int DMAX, bool EXACT, int S, bool GS>
__global__ void __launch_bounds__(S, (S >= 512 ? 1 : 512 / S)) anneal_small_kernel(const AnnealArgs A) {
  extern __shared__ __align__(16) double smem_raw[];
  const Prob P = A.P;
  const int tid = threadIdx.x;
  const int dim = P.dim;
  Smem sm;
  double* v[9];
  carve<CPLX>(P, S, smem_raw, sm, v, 9);
  build_tables<S, CPLX, GS>(P, sm);
  double* x = v[0];   // current iterate
  double* g = v[1];   // current gradient
  double* zs = v[2];  // Steihaug step z
  double* r = v[3];   // CG residual
  double* dv = v[4];  // CG direction
  double* bd = v[5];  // B*d
  double* xt = v[6];  // trial point / FD scratch
  double* gt = v[7];  // trial gradient / g(x - h d)
  double* xb = v[8];  // best-seen iterate
  __shared__ int s_trial;
  int rbuf = 0;
  const double inf = __longlong_as_double(0x7ff0000000000000LL);

  for (;;) {
    if (tid == 0) s_trial = atomicAdd(A.counter, 1);
    __syncthreads();
    const int li = s_trial;
    __syncthreads();
    if (li >= A.n_list) break;
    const int trial = A.list ? A.list[li] : li;
#ifdef TRSTMI_PHASE_TIMERS
    const long long t_trial_ = clock64();
#endif
    const int k0 = A.start_stage ? A.start_stage[trial] : 0;
    trstmi_trial_out* TO = A.tout + trial;
    long long outer = 0, evals = 0, hvps = 0, nrec = 0;
    if (k0 > 0) {
      outer = TO->outer_iterations;
      evals = TO->evals;
      hvps = TO->hvps;
      nrec = TO->records;
    }
    int status = TRSTMI_TRIAL_OK, zero_col = -1, fail_stage = -1, stages_done = k0;
    double mu = 0.0;
    long long argmax = -1;
    double* gp = A.params + (long long)trial * dim;
    vcopy<S>(x, gp, dim);
    __syncthreads();

    for (int k = k0; k < A.n_stages; ++k) {
      // ---- stage start: rescue_zero_columns check (solver.hpp:139-156, 183)
      {
        int zc = INT_MAX;
        for (int j = tid; j < P.N; j += S) {
          double acc = 0.0;
          for (int q = 0; q < P.L; ++q) acc = fma(x[j * P.L + q], x[j * P.L + q], acc);
          if (!(sqrt(acc) >= kZeroColumnTol)) zc = min(zc, j);  // NaN norms are rescued too (solver.hpp:144)
        }
        zc = block_min_int<S>(zc, sm.ired, rbuf);
        if (zc != INT_MAX) {
          status = TRSTMI_TRIAL_NEED_RESCUE;
          zero_col = zc;
          fail_stage = k;
          break;
        }
      }
      const double delta = A.schedule[k];
      const int max_outer = A.tr.max_outer + 50 * k;  // solver.hpp:187
      // ---- x0 evaluation (trust_region.hpp:206-209)
      double Fcur;
      ++evals;
      const int zc0 = eval_any<CPLX, DMAX, EXACT, S, GS>(P, x, nullptr, 0.0, delta, sm, rbuf, g, &sm.scal[0], nullptr, nullptr);
      Fcur = sm.scal[0];
      (void)zc0;
      {
        const int fin = all_finite<S>(g, dim, sm, rbuf);
        if (!isfinite(Fcur) || !fin) {
          status = TRSTMI_TRIAL_NONFINITE_X0;
          fail_stage = k;
          break;
        }
      }
      double bestv = Fcur;
      vcopy<S>(xb, x, dim);
      double radius = A.tr.delta0;
      int mstatus = TRSTMI_ST_ITERATION_LIMIT;
      int hist = 0;
      bool failed = false;

      for (int iter = 0; iter < max_outer; ++iter) {
        double gv[2] = {dot_partial<S>(g, g, dim), dot_partial<S>(x, x, dim)};
        block_sum<S, 2>(gv, sm.red, rbuf);
        const double grad_norm = sqrt(gv[0]);
        const double xnorm = sqrt(gv[1]);
        if (grad_norm <= A.tr.grad_tol) {
          mstatus = TRSTMI_ST_GRADIENT_TOLERANCE;
          break;
        }
        const double eps_k = fmin(A.tr.cg_force_c, sqrt(grad_norm)) * grad_norm;
        // ---------------- steihaug_cg (trust_region.hpp:81-154)
        int cg_iters = 0, cg_exit = TRSTMI_CG_SMALL_RESIDUAL;
        double step_norm = 0.0, model_value = 0.0;
        for (int i = tid; i < dim; i += S) zs[i] = 0.0;
        if (grad_norm < eps_k || grad_norm == 0.0) {
          cg_exit = TRSTMI_CG_ZERO_GRADIENT;
        } else {
          for (int i = tid; i < dim; i += S) {
            r[i] = g[i];
            dv[i] = -g[i];
          }
          double rr = gv[0];  // r.squaredNorm() with r == grad: the same CAS dot
          double model = 0.0;
          bool done = false;
          for (int j = 0; j < A.tr.max_cg; ++j) {
            // ---- hvp(d): make_hvp_factory (solver.hpp:118-137)
            ++hvps;
            const double dn = sqrt(block_sum1<S>(dot_partial<S>(dv, dv, dim), sm.red, rbuf));
            if (dn == 0.0) {
              for (int i = tid; i < dim; i += S) bd[i] = 0.0;
            } else {
              const double h = kFdBaseStep * (1.0 + xnorm) / fmax(dn, 1e-300);
              __syncthreads();
              evals += 2;
              int zp = INT_MAX - 1;
              if constexpr (GS) {  // both points in one pass (bit-identical; falls through when a column vanishes)
                if (P.dual) zp = hvp_cta_gs<CPLX, DMAX, EXACT, S>(P, x, dv, h, delta, sm, rbuf, bd);
              }
              if (zp == -1) {
                // bd = (g(x + h d) - g(x - h d)) / (2h) already formed
              } else if ((zp = eval_any<CPLX, DMAX, EXACT, S, GS>(P, x, dv, h, delta, sm, rbuf, bd, nullptr, nullptr, nullptr)) < 0) {
                const int zm = eval_any<CPLX, DMAX, EXACT, S, GS>(P, x, dv, -h, delta, sm, rbuf, gt, nullptr, nullptr, nullptr);
                if (zm < 0) {
                  const double h2 = 2.0 * h;
                  for (int i = tid; i < dim; i += S) bd[i] = (bd[i] - gt[i]) / h2;
                } else {  // forward fallback: (g(x+hd) - g0)/h; the reference evaluates g0 and
                  evals += 2;  // g(x+hd) again (solver.hpp:129-130): g0 == current gradient, g(x+hd) reused
                  for (int i = tid; i < dim; i += S) bd[i] = (bd[i] - g[i]) / h;
                }
              } else {  // x+hd hit a zero column: g0, retry forward (fails again), backward
                evals += 2;
                const int zm = eval_any<CPLX, DMAX, EXACT, S, GS>(P, x, dv, -h, delta, sm, rbuf, gt, nullptr, nullptr, nullptr);
                if (zm >= 0) {
                  status = TRSTMI_TRIAL_ZERO_COLUMN;
                  zero_col = zm;
                  fail_stage = k;
                  failed = true;
                  break;
                }
                for (int i = tid; i < dim; i += S) bd[i] = (g[i] - gt[i]) / h;
              }
            }
            double dd[2] = {dot_partial<S>(dv, bd, dim), dot_partial<S>(r, dv, dim)};
            block_sum<S, 2>(dd, sm.red, rbuf);
            const double dbd = dd[0], rd = dd[1];
            if (dbd <= 0.0) {
              // boundary_roots(z, d, radius)
              double br[3] = {dot_partial<S>(dv, dv, dim), dot_partial<S>(zs, dv, dim), dot_partial<S>(zs, zs, dim)};
              block_sum<S, 3>(br, sm.red, rbuf);
              const double a = br[0], b = 2.0 * br[1], c = br[2] - radius * radius;
              double tau_lo = 0.0, tau_hi = 0.0;
              if (!(a <= 0.0)) {
                const double disc = sqrt(fmax(b * b - 4.0 * a * c, 0.0));
                const double q = -0.5 * (b + copysign(disc, b));
                double r1 = q != 0.0 ? c / q : 0.0;
                double r2 = a != 0.0 ? q / a : 0.0;
                if (r1 > r2) {
                  const double tt = r1;
                  r1 = r2;
                  r2 = tt;
                }
                tau_lo = r1;
                tau_hi = r2;
              }
              const double m_lo = model + tau_lo * rd + 0.5 * tau_lo * tau_lo * dbd;
              const double m_hi = model + tau_hi * rd + 0.5 * tau_hi * tau_hi * dbd;
              const double tau = m_lo < m_hi ? tau_lo : tau_hi;
              double zz = 0.0;
              for (int i = tid; i < dim; i += S) {
                zs[i] = zs[i] + tau * dv[i];
                zz = fma(zs[i], zs[i], zz);
              }
              step_norm = sqrt(block_sum1<S>(zz, sm.red, rbuf));
              cg_iters = j;
              cg_exit = TRSTMI_CG_NEGATIVE_CURVATURE;
              model_value = fmin(m_lo, m_hi);
              done = true;
              break;
            }
            const double alpha = rr / dbd;
            // ||z + alpha d||^2 and, speculatively, ||r + alpha B d||^2 (needed only when the step stays inside) in
            // one CTA reduction: each sum keeps its own CAS order
            double znrn[2] = {0.0, 0.0};
            for (int i = tid; i < dim; i += S) {
              const double t = zs[i] + alpha * dv[i];
              znrn[0] = fma(t, t, znrn[0]);
              const double rt = r[i] + alpha * bd[i];
              znrn[1] = fma(rt, rt, znrn[1]);
            }
            block_sum<S, 2>(znrn, sm.red, rbuf);
            if (sqrt(znrn[0]) >= radius) {
              double br[3] = {dot_partial<S>(dv, dv, dim), dot_partial<S>(zs, dv, dim), dot_partial<S>(zs, zs, dim)};
              block_sum<S, 3>(br, sm.red, rbuf);
              const double a = br[0], b = 2.0 * br[1], c = br[2] - radius * radius;
              double tau = 0.0;
              if (!(a <= 0.0)) {
                const double disc = sqrt(fmax(b * b - 4.0 * a * c, 0.0));
                const double q = -0.5 * (b + copysign(disc, b));
                double r1 = q != 0.0 ? c / q : 0.0;
                double r2 = a != 0.0 ? q / a : 0.0;
                tau = (r1 > r2) ? r1 : r2;
              }
              double zz = 0.0;
              for (int i = tid; i < dim; i += S) {
                zs[i] = zs[i] + tau * dv[i];
                zz = fma(zs[i], zs[i], zz);
              }
              step_norm = sqrt(block_sum1<S>(zz, sm.red, rbuf));
              cg_iters = j;
              cg_exit = TRSTMI_CG_BOUNDARY_HIT;
              model_value = model + tau * rd + 0.5 * tau * tau * dbd;
              done = true;
              break;
            }
            model += alpha * rd + 0.5 * alpha * alpha * dbd;
            for (int i = tid; i < dim; i += S) {
              zs[i] = zs[i] + alpha * dv[i];
              r[i] = r[i] + alpha * bd[i];
            }
            const double rr_next = znrn[1];
            cg_iters = j + 1;
            if (sqrt(rr_next) < eps_k) {
              cg_exit = TRSTMI_CG_SMALL_RESIDUAL;
              step_norm = sqrt(block_sum1<S>(dot_partial<S>(zs, zs, dim), sm.red, rbuf));
              model_value = model;
              done = true;
              break;
            }
            const double beta = rr_next / rr;
            rr = rr_next;
            for (int i = tid; i < dim; i += S) dv[i] = -r[i] + beta * dv[i];
          }
          if (failed) break;
          if (!done) {  // CG cap: converged = false (trust_region.hpp:149-153)
            cg_exit = TRSTMI_CG_SMALL_RESIDUAL;
            step_norm = sqrt(block_sum1<S>(dot_partial<S>(zs, zs, dim), sm.red, rbuf));
            model_value = model;
          }
        }
        // ---------------- outer update (trust_region.hpp:232-287)
        trstmi_outer_out rec;
        rec.stage = k;
        rec.iteration = iter;
        rec.cg_exit = cg_exit;
        rec.cg_iterations = cg_iters;
        rec.accepted = 0;
        rec.pad = 0;
        rec.value = Fcur;
        rec.grad_norm = grad_norm;
        rec.radius = radius;
        rec.rho = 0.0;
        rec.step_norm = step_norm;
        const double predicted = -model_value;
        bool underflow = false;
        if (cg_exit == TRSTMI_CG_ZERO_GRADIENT || predicted <= 0.0) {
          radius *= A.tr.shrink;
          underflow = radius < 1e-16;
        } else {
          for (int i = tid; i < dim; i += S) xt[i] = x[i] + zs[i];
          __syncthreads();
          ++evals;
          double Ft;
          eval_any<CPLX, DMAX, EXACT, S, GS>(P, xt, nullptr, 0.0, delta, sm, rbuf, gt, &sm.scal[0], nullptr, nullptr);
          Ft = sm.scal[0];
          const int gfin = all_finite<S>(gt, dim, sm, rbuf);
          const bool finite = isfinite(Ft) && gfin;
          const double rho = finite ? (Fcur - Ft) / predicted : -inf;
          rec.rho = rho;
          if (finite && Ft < bestv) {
            vcopy<S>(xb, xt, dim);
            bestv = Ft;
          }
          if (rho > A.tr.eta) {
            double* t1 = x;
            x = xt;
            xt = t1;
            double* t2 = g;
            g = gt;
            gt = t2;
            Fcur = Ft;
            rec.accepted = 1;
          }
          if (rho < 0.25) {
            radius *= A.tr.shrink;
          } else if (rho > 0.75 && step_norm >= (1.0 - 1e-10) * radius) {
            radius = fmin(A.tr.grow * radius, A.tr.delta_max);
          }
          underflow = radius < 1e-16;
        }
        if (tid == 0 && A.oout && nrec < A.record_cap) A.oout[(long long)trial * A.record_cap + nrec] = rec;
        if (A.oout && nrec < A.record_cap) ++nrec;
        ++hist;
        if (underflow) {
          mstatus = TRSTMI_ST_RADIUS_UNDERFLOW;
          break;
        }
      }
      if (failed) break;
      outer += hist;
      if (Fcur < bestv) {  // trust_region.hpp:289-293
        vcopy<S>(xb, x, dim);
        bestv = Fcur;
      }
      {  // param <- best-seen x (solver.hpp:192)
        double* t1 = x;
        x = xb;
        xb = t1;
      }
      __syncthreads();
      // ---- stage record: coherence(normalize_columns(param)) (solver.hpp:197)
      double smu;
      long long sarg;
      const int zc = coherence_cta<CPLX, DMAX, EXACT, S, GS>(P, x, true, sm, rbuf, &smu, &sarg);
      if (zc >= 0) {
        status = TRSTMI_TRIAL_ZERO_COLUMN;
        zero_col = zc;
        fail_stage = k;
        break;
      }
      if (tid == 0) {
        trstmi_stage_out so;
        so.delta = delta;
        so.objective = bestv;
        so.coherence = smu;
        so.argmax_pair = sarg;
        so.outer_iterations = hist;
        so.status = mstatus;
        A.sout[(long long)trial * A.n_stages + k] = so;
      }
      mu = smu;
      argmax = sarg;
      stages_done = k + 1;
      __syncthreads();
    }
    // ---- outputs
    __syncthreads();
    vcopy<S>(gp, x, dim);
    if (status == TRSTMI_TRIAL_OK && A.frames) {
      double* fo = A.frames + (long long)trial * dim;
      for (int i = tid; i < dim; i += S) {
        const int j = i / P.L, q = i - j * P.L;
        fo[i] = sm.phiS[q * P.N + j];
      }
    }
    if (tid == 0) {
      trstmi_trial_out o;
      o.coherence = mu;
      o.argmax_pair = argmax;
      o.status = status;
      o.stages_done = stages_done;
      o.zero_col = zero_col;
      o.fail_stage = fail_stage;
      o.outer_iterations = outer;
      o.evals = evals;
      o.hvps = hvps;
      o.records = nrec;
      *TO = o;
    }
#ifdef TRSTMI_PHASE_TIMERS
    if (tid == 0) atomicAdd(&g_phase_cycles[7], (unsigned long long)(clock64() - t_trial_));
#endif
    __syncthreads();
  }
}

}  // namespace trstmi_dev
