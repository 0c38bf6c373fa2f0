// Device-side trust-region driver of the batched large-frame engine: one CTA
// per trial in flight ("lane") advances that trial's anneal state machine —
//   anneal                 solver.hpp:164-204
//   trust_region_minimize  trust_region.hpp:189-295
//   steihaug_cg            trust_region.hpp:81-154
//   boundary_roots         trust_region.hpp:56-69
//   make_hvp_factory       solver.hpp:118-137
// — until it needs gradients (x0 / the two FD points of a Hessian-vector
// product / the trial point) or a coherence, posts those requests for the
// batched evaluation pipeline (bde.cuh) and yields.  One launch advances every
// lane; the host only launches and reads three counters per tick.  A lane
// whose trial ends pulls the next trial from an atomic counter (the
// reference's restart pool).
//
// Every scalar formula is the host driver's (large_engine.cu anneal_trial,
// itself the oracle's): the same IEEE operations (the file is compiled with
// -fmad=false), std::min / std::max semantics spelled out, and CAS dots of
// width 32768 reproduced inside one CTA: lane l sums elements l, l + 32768,
// ... by fma from +0, each 32-lane group by the xor butterfly, the 1024 group
// totals pairwise in index order — the order of large_dots +
// large_dots_reduce.
#pragma once
#include "bde.cuh"

namespace trstmi_bde {

constexpr int TR_T = 512;            // threads of a lane CTA
constexpr int TR_W = TR_T / 32;
constexpr int CAS_S = 32768;         // CAS lanes of the large path
constexpr int CAS_G = CAS_S / 32;    // 1024 lane groups

enum VecId { V_X = 0, V_G, V_ZS, V_R, V_DV, V_BD, V_XT, V_GT, V_XB, V_ZN, V_GP, V_GM, NVEC };

enum Phase {
  PH_IDLE = 0,
  PH_START,      // pull / load a trial
  PH_STAGE,      // stage start: zero-column check
  PH_STAGE_GO,   // request x0
  PH_X0,         // x0 evaluated
  PH_OUTER,      // top of an outer iteration
  PH_CG,         // top of a CG iteration
  PH_HVP,        // the two FD gradients are in
  PH_UPDATE,     // CG done: trial point or shrink
  PH_TRIAL,      // trial point evaluated
  PH_STAGE_END,  // request the stage coherence
  PH_COH,        // coherence in
  PH_FINISH,     // write the trial's outputs
  PH_PAUSED      // waiting for the host's column rescue
};

struct TrCfgD {
  double delta0, delta_max, eta, shrink, grow, grad_tol, cg_force_c;
  int max_outer, max_cg;
};

struct Lane {
  int trial, phase, stage, iter, hist, j, cg_exit, cg_iters;
  int mstatus, status, zero_col, fail_stage, stages_done, max_outer, accepted, underflow;
  int ix[NVEC];
  double delta, radius, Fcur, bestv, grad_norm, xnorm, eps_k, rr, model, h, step_norm, model_value, rho;
  double rec_radius, rec_value, mu;
  long long argmax, outer, evals, hvps, nrec;
};

struct TrArgs {
  Shape sh;
  TrCfgD tr;
  int n_stages;
  int stage_end;             // stages [start, stage_end)
  double schedule[TRSTMI_MAX_STAGES];
  int record_cap;
  int n_list;                // trials of this run
  const int* list;           // nullable: trial ids
  const int* start_stage;    // nullable: per-trial first stage
  int* next;                 // next list position (atomic)
  Lane* lanes;
  double* vecs;              // lanes x NVEC x dim
  double* params;            // trials x dim
  double* frames;            // nullable
  trstmi_trial_out* tout;
  trstmi_stage_out* sout;    // trials x n_stages
  trstmi_outer_out* oout;    // nullable: trials x record_cap
  Req* reqs;                 // 2 per lane (slots 2l, 2l+1)
  ReqOut* outs;              // 2 per lane
  int* act_obj;              // objective request ids of the next tick
  int* act_coh;              // coherence request ids
  int* counters;             // [0] objective requests, [1] coherence requests, [2] paused lanes, [3] busy lanes
  int* paused;               // paused lane ids
};

// ---- CTA-wide helpers (TR_T threads)
__device__ __forceinline__ double* vptr(const TrArgs& A, int lane, const Lane& S, int v) {
  return A.vecs + ((long long)lane * NVEC + S.ix[v]) * A.sh.dim;
}

// ND CAS dots <a_k, b_k> of length n (S = 32768 lanes).  tot: ND x 1024 smem.
template <int ND>
__device__ void cas_dots(const double* const* a, const double* const* b, long long n, double* out, double* tot) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int GU = CAS_G / TR_W;  // groups per warp
  constexpr int UN = 8;
  for (int u0 = 0; u0 < GU; u0 += UN) {
    double acc[UN][ND];
#pragma unroll
    for (int uu = 0; uu < UN; ++uu)
#pragma unroll
      for (int k = 0; k < ND; ++k) acc[uu][k] = 0.0;
    for (long long base = 0; base < n; base += CAS_S) {
#pragma unroll
      for (int uu = 0; uu < UN; ++uu) {
        const long long i = base + 32LL * (warp + TR_W * (u0 + uu)) + lane;
        if (i < n) {
#pragma unroll
          for (int k = 0; k < ND; ++k) acc[uu][k] = fma(a[k][i], b[k][i], acc[uu][k]);
        }
      }
    }
    // The eight groups' 32-lane butterflies (xor 16, 8, 4, 2, 1), transposed: at each of the first three levels a
    // lane keeps half of the groups it still holds and trades the other half with its partner, so a level costs half
    // the shuffles of the one before — 9 shuffles per dot for the eight groups instead of 40.  Every sum has the same
    // two operands as in the plain butterfly (own + partner's value of the same group), hence the same bits.  The
    // reductions of this kernel are bound by shuffle throughput (one warp-wide SHFL per clock per SM).
    static_assert(UN == 8, "transposed butterfly is written for eight groups");
#pragma unroll
    for (int k = 0; k < ND; ++k) {
      double v[UN];
#pragma unroll
      for (int uu = 0; uu < UN; ++uu) v[uu] = acc[uu][k];
#pragma unroll
      for (int half = 4, off = 16; half >= 1; half >>= 1, off >>= 1) {
        const bool hi = (lane & off) != 0;
#pragma unroll
        for (int i = 0; i < half; ++i) {
          const double send = hi ? v[i] : v[i + half];
          const double keep = hi ? v[i + half] : v[i];
          v[i] = __dadd_rn(keep, __shfl_xor_sync(FULL, send, off));
        }
      }
      v[0] = __dadd_rn(v[0], __shfl_xor_sync(FULL, v[0], 2));
      v[0] = __dadd_rn(v[0], __shfl_xor_sync(FULL, v[0], 1));
      if ((lane & 3) == 0) {
        const int uu = ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
        tot[k * CAS_G + warp + TR_W * (u0 + uu)] = v[0];
      }
    }
  }
  __syncthreads();
  // the 1024 group totals pairwise in index order: levels 1..32 inside each warp's 64 consecutive totals (one add
  // from memory, then the xor butterfly — the same pairs), the last four levels over the 16 warp values
  static_assert(CAS_G == 64 * TR_W, "one warp per 64 group totals");
  __shared__ double wtot[3 * TR_W];
  static_assert(ND <= 3, "wtot holds three dots");
#pragma unroll
  for (int k = 0; k < ND; ++k) {
    const double2 t2 = *reinterpret_cast<const double2*>(tot + k * CAS_G + 64 * warp + 2 * lane);
    double v = __dadd_rn(t2.x, t2.y);
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) v = __dadd_rn(v, __shfl_xor_sync(FULL, v, off));
    if (lane == 0) wtot[k * TR_W + warp] = v;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < ND; ++k) {
    double v = lane < TR_W ? wtot[k * TR_W + lane] : 0.0;
#pragma unroll
    for (int off = 1; off < TR_W; off <<= 1) v = __dadd_rn(v, __shfl_xor_sync(FULL, v, off));
    out[k] = __shfl_sync(FULL, v, 0);
  }
  __syncthreads();
}

__device__ __forceinline__ double cas_dot1(const double* a, const double* b, long long n, double* tot) {
  const double* aa[1] = {a};
  const double* bb[1] = {b};
  double o[1];
  cas_dots<1>(aa, bb, n, o, tot);
  return o[0];
}

// y = a + s b elementwise (mul then add)
__device__ __forceinline__ void v_axpy(double* y, const double* a, double s, const double* b, long long n) {
  for (long long i = threadIdx.x; i < n; i += TR_T) y[i] = __dadd_rn(a[i], __dmul_rn(s, b[i]));
  __syncthreads();
}
__device__ __forceinline__ void v_copy(double* y, const double* a, long long n) {
  for (long long i = threadIdx.x; i < n; i += TR_T) y[i] = a[i];
  __syncthreads();
}
__device__ __forceinline__ int v_all_finite(const double* a, long long n) {
  int bad = 0;
  for (long long i = threadIdx.x; i < n; i += TR_T) bad |= isfinite(a[i]) ? 0 : 1;
  return __syncthreads_or(bad) ? 0 : 1;
}
// first column whose CAS norm is < tol (or NaN), INT_MAX if none
__device__ __forceinline__ int first_zero_column(const double* x, int N, int L, int* sh_min) {
  if (threadIdx.x == 0) *sh_min = INT_MAX;
  __syncthreads();
  for (int j = threadIdx.x; j < N; j += TR_T) {
    const double* c = x + (long long)j * L;
    double acc = 0.0;
    for (int q = 0; q < L; ++q) acc = fma(c[q], c[q], acc);
    if (!(sqrt(acc) >= kZeroColumnTol)) atomicMin(sh_min, j);
  }
  __syncthreads();
  const int r = *sh_min;
  __syncthreads();
  return r;
}

__device__ __forceinline__ double dmin(double a, double b) { return (b < a) ? b : a; }  // std::min
__device__ __forceinline__ double dmax(double a, double b) { return (a < b) ? b : a; }  // std::max

__global__ void __launch_bounds__(TR_T, 1) bde_advance(TrArgs A) {
  __shared__ __align__(16) double tot[3 * CAS_G];
  __shared__ int sh_int[4];
  const int lane = blockIdx.x;
  const int tid = threadIdx.x;
  const long long dim = A.sh.dim;
  const int N = A.sh.N, L = A.sh.L;
  Lane S = A.lanes[lane];
  if (S.phase == PH_IDLE || S.phase == PH_PAUSED) {  // paused lanes are resumed by the host
    if (tid == 0 && S.phase == PH_PAUSED) atomicAdd(&A.counters[3], 1);
    return;
  }
  Req* rq = A.reqs + 2 * lane;
  ReqOut* ro = A.outs + 2 * lane;
  const double inf = __longlong_as_double(0x7ff0000000000000LL);
  int nobj = 0, ncoh = 0;  // requests posted this launch
  auto post = [&](int s, int kind, int vx, int vdir, double sc, int vout) {
    if (tid == 0) {
      Req r;
      r.x = vptr(A, lane, S, vx);
      r.dir = vdir >= 0 ? vptr(A, lane, S, vdir) : nullptr;
      r.sc = sc;
      r.delta = S.delta;
      r.grad = vout >= 0 ? vptr(A, lane, S, vout) : nullptr;
      r.wout = nullptr;
      r.kind = kind;
      r.squared = 1;
      r.slot = 2 * lane + s;
      r.pad = 0;
      rq[s] = r;
      ReqOut o;
      o.F = o.s = o.z = o.mu = 0.0;
      o.argmax = -1;
      o.smax = 0ull;
      o.zc = INT_MAX;
      o.pad = 0;
      ro[s] = o;
    }
    if (kind == REQ_OBJ) ++nobj;
    else ++ncoh;
  };
  bool yield = false;
  int guard = 0;
  while (!yield && ++guard < (1 << 30)) {
    switch (S.phase) {
      case PH_START: {
        int li;
        if (tid == 0) sh_int[0] = atomicAdd(A.next, 1);
        __syncthreads();
        li = sh_int[0];
        __syncthreads();
        if (li >= A.n_list) {
          S.phase = PH_IDLE;
          S.trial = -1;
          yield = true;
          break;
        }
        const int trial = A.list ? A.list[li] : li;
        S.trial = trial;
        for (int v = 0; v < NVEC; ++v) S.ix[v] = v;
        const int k0 = A.start_stage ? A.start_stage[trial] : 0;
        trstmi_trial_out* TO = A.tout + trial;
        S.outer = S.evals = S.hvps = S.nrec = 0;
        if (k0 > 0) {
          S.outer = TO->outer_iterations;
          S.evals = TO->evals;
          S.hvps = TO->hvps;
          S.nrec = TO->records;
        }
        S.status = TRSTMI_TRIAL_OK;
        S.zero_col = -1;
        S.fail_stage = -1;
        S.stages_done = k0;
        S.mu = 0.0;
        S.argmax = -1;
        S.stage = k0;
        v_copy(vptr(A, lane, S, V_X), A.params + (long long)trial * dim, dim);
        S.phase = PH_STAGE;
        break;
      }
      case PH_STAGE: {
        if (S.stage >= A.stage_end || S.stage >= A.n_stages) {
          S.phase = PH_FINISH;
          break;
        }
        // rescue_zero_columns (solver.hpp:139-156): the host redraws from the trial's generator
        const int zc = first_zero_column(vptr(A, lane, S, V_X), N, L, &sh_int[1]);
        if (zc != INT_MAX) {
          S.status = TRSTMI_TRIAL_NEED_RESCUE;
          S.zero_col = zc;
          S.fail_stage = S.stage;
          S.phase = PH_PAUSED;
          if (tid == 0) {
            const int pi = atomicAdd(&A.counters[2], 1);
            A.paused[pi] = lane;
          }
          yield = true;
          break;
        }
        S.phase = PH_STAGE_GO;
        break;
      }
      case PH_STAGE_GO: {
        S.delta = A.schedule[S.stage];
        S.max_outer = A.tr.max_outer + 50 * S.stage;  // solver.hpp:187
        ++S.evals;
        post(0, REQ_OBJ, V_X, -1, 0.0, V_G);
        S.phase = PH_X0;
        yield = true;
        break;
      }
      case PH_X0: {
        const double F = ro[0].F;
        const int fin = v_all_finite(vptr(A, lane, S, V_G), dim);
        if (!isfinite(F) || !fin) {
          S.status = TRSTMI_TRIAL_NONFINITE_X0;
          S.fail_stage = S.stage;
          S.phase = PH_FINISH;
          break;
        }
        S.Fcur = F;
        S.bestv = F;
        v_copy(vptr(A, lane, S, V_XB), vptr(A, lane, S, V_X), dim);
        S.radius = A.tr.delta0;
        S.mstatus = TRSTMI_ST_ITERATION_LIMIT;
        S.hist = 0;
        S.iter = 0;
        S.phase = PH_OUTER;
        break;
      }
      case PH_OUTER: {
        if (S.iter >= S.max_outer) {
          S.phase = PH_STAGE_END;
          break;
        }
        const double* aa[2] = {vptr(A, lane, S, V_G), vptr(A, lane, S, V_X)};
        double gv[2];
        cas_dots<2>(aa, aa, dim, gv, tot);
        S.grad_norm = sqrt(gv[0]);
        S.xnorm = sqrt(gv[1]);
        if (S.grad_norm <= A.tr.grad_tol) {
          S.mstatus = TRSTMI_ST_GRADIENT_TOLERANCE;
          S.phase = PH_STAGE_END;
          break;
        }
        S.eps_k = dmin(A.tr.cg_force_c, sqrt(S.grad_norm)) * S.grad_norm;
        S.cg_iters = 0;
        S.cg_exit = TRSTMI_CG_SMALL_RESIDUAL;
        S.step_norm = 0.0;
        S.model_value = 0.0;
        double* zs = vptr(A, lane, S, V_ZS);
        for (long long i = tid; i < dim; i += TR_T) zs[i] = 0.0;
        __syncthreads();
        if (S.grad_norm < S.eps_k || S.grad_norm == 0.0) {
          S.cg_exit = TRSTMI_CG_ZERO_GRADIENT;
          S.phase = PH_UPDATE;
          break;
        }
        const double* g = vptr(A, lane, S, V_G);
        double* r = vptr(A, lane, S, V_R);
        double* dv = vptr(A, lane, S, V_DV);
        for (long long i = tid; i < dim; i += TR_T) {
          r[i] = g[i];
          dv[i] = -g[i];
        }
        __syncthreads();
        S.rr = gv[0];
        S.model = 0.0;
        S.j = 0;
        S.phase = PH_CG;
        break;
      }
      case PH_CG: {
        if (S.j >= A.tr.max_cg) {  // CG cap: converged = false (trust_region.hpp:149-153)
          S.cg_exit = TRSTMI_CG_SMALL_RESIDUAL;
          const double* zs = vptr(A, lane, S, V_ZS);
          S.step_norm = sqrt(cas_dot1(zs, zs, dim, tot));
          S.model_value = S.model;
          S.phase = PH_UPDATE;
          break;
        }
        ++S.hvps;
        const double* dv = vptr(A, lane, S, V_DV);
        const double dn = sqrt(cas_dot1(dv, dv, dim, tot));
        if (dn == 0.0) {
          double* bd = vptr(A, lane, S, V_BD);
          for (long long i = tid; i < dim; i += TR_T) bd[i] = 0.0;
          __syncthreads();
          S.phase = PH_HVP;
          S.h = 0.0;  // marks the zero-direction product
          break;
        }
        S.h = kFdBaseStep * (1.0 + S.xnorm) / dmax(dn, 1e-300);
        S.evals += 2;
        post(0, REQ_OBJ, V_X, V_DV, S.h, V_GP);
        post(1, REQ_OBJ, V_X, V_DV, -S.h, V_GM);
        S.phase = PH_HVP;
        yield = true;
        break;
      }
      case PH_HVP: {
        if (S.h != 0.0) {
          const int zp = ro[0].zc, zm = ro[1].zc;
          double* bd = vptr(A, lane, S, V_BD);
          const double* gp = vptr(A, lane, S, V_GP);
          const double* gm = vptr(A, lane, S, V_GM);
          const double* g = vptr(A, lane, S, V_G);
          const double h = S.h;
          if (zp == INT_MAX) {
            if (zm == INT_MAX) {
              const double h2 = 2.0 * h;
              for (long long i = tid; i < dim; i += TR_T) bd[i] = __ddiv_rn(__dsub_rn(gp[i], gm[i]), h2);
            } else {  // forward fallback (solver.hpp:129-130): g0 and g(x + h d) again, reused values
              S.evals += 2;
              for (long long i = tid; i < dim; i += TR_T) bd[i] = __ddiv_rn(__dsub_rn(gp[i], g[i]), h);
            }
          } else {  // x + h d hit a zero column: g0, retry forward (fails again), backward
            S.evals += 2;
            if (zm != INT_MAX) {
              S.status = TRSTMI_TRIAL_ZERO_COLUMN;
              S.zero_col = zm;
              S.fail_stage = S.stage;
              S.phase = PH_FINISH;
              break;
            }
            for (long long i = tid; i < dim; i += TR_T) bd[i] = __ddiv_rn(__dsub_rn(g[i], gm[i]), h);
          }
          __syncthreads();
        }
        const double* dv = vptr(A, lane, S, V_DV);
        const double* bd = vptr(A, lane, S, V_BD);
        const double* r = vptr(A, lane, S, V_R);
        double* zs = vptr(A, lane, S, V_ZS);
        const double* aa[2] = {dv, r};
        const double* bb[2] = {bd, dv};
        double dd[2];
        cas_dots<2>(aa, bb, dim, dd, tot);
        const double dbd = dd[0], rd = dd[1];
        if (dbd <= 0.0) {  // negative curvature: boundary_roots, the tau of the smaller model value
          const double* a3[3] = {dv, zs, zs};
          const double* b3[3] = {dv, dv, zs};
          double br[3];
          cas_dots<3>(a3, b3, dim, br, tot);
          const double a = br[0], b = 2.0 * br[1], c = br[2] - S.radius * S.radius;
          double tau_lo = 0.0, tau_hi = 0.0;
          if (!(a <= 0.0)) {
            const double disc = sqrt(dmax(b * b - 4.0 * a * c, 0.0));
            const double qv = -0.5 * (b + copysign(disc, b));
            double r1 = qv != 0.0 ? c / qv : 0.0;
            double r2 = a != 0.0 ? qv / a : 0.0;
            if (r1 > r2) {
              const double tt = r1;
              r1 = r2;
              r2 = tt;
            }
            tau_lo = r1;
            tau_hi = r2;
          }
          const double m_lo = S.model + tau_lo * rd + 0.5 * tau_lo * tau_lo * dbd;
          const double m_hi = S.model + tau_hi * rd + 0.5 * tau_hi * tau_hi * dbd;
          const double tau = m_lo < m_hi ? tau_lo : tau_hi;
          v_axpy(zs, zs, tau, dv, dim);
          S.step_norm = sqrt(cas_dot1(zs, zs, dim, tot));
          S.cg_iters = S.j;
          S.cg_exit = TRSTMI_CG_NEGATIVE_CURVATURE;
          S.model_value = dmin(m_lo, m_hi);
          S.phase = PH_UPDATE;
          break;
        }
        const double alpha = S.rr / dbd;
        double* zn = vptr(A, lane, S, V_ZN);
        v_axpy(zn, zs, alpha, dv, dim);
        if (sqrt(cas_dot1(zn, zn, dim, tot)) >= S.radius) {  // leaves the region: positive root
          const double* a3[3] = {dv, zs, zs};
          const double* b3[3] = {dv, dv, zs};
          double br[3];
          cas_dots<3>(a3, b3, dim, br, tot);
          const double a = br[0], b = 2.0 * br[1], c = br[2] - S.radius * S.radius;
          double tau = 0.0;
          if (!(a <= 0.0)) {
            const double disc = sqrt(dmax(b * b - 4.0 * a * c, 0.0));
            const double qv = -0.5 * (b + copysign(disc, b));
            const double r1 = qv != 0.0 ? c / qv : 0.0;
            const double r2 = a != 0.0 ? qv / a : 0.0;
            tau = (r1 > r2) ? r1 : r2;
          }
          v_axpy(zs, zs, tau, dv, dim);
          S.step_norm = sqrt(cas_dot1(zs, zs, dim, tot));
          S.cg_iters = S.j;
          S.cg_exit = TRSTMI_CG_BOUNDARY_HIT;
          S.model_value = S.model + tau * rd + 0.5 * tau * tau * dbd;
          S.phase = PH_UPDATE;
          break;
        }
        S.model += alpha * rd + 0.5 * alpha * alpha * dbd;
        {  // z = z_next
          const int t = S.ix[V_ZS];
          S.ix[V_ZS] = S.ix[V_ZN];
          S.ix[V_ZN] = t;
        }
        double* rw = vptr(A, lane, S, V_R);
        v_axpy(rw, rw, alpha, bd, dim);
        const double rr_next = cas_dot1(rw, rw, dim, tot);
        S.cg_iters = S.j + 1;
        if (sqrt(rr_next) < S.eps_k) {
          S.cg_exit = TRSTMI_CG_SMALL_RESIDUAL;
          const double* z2 = vptr(A, lane, S, V_ZS);
          S.step_norm = sqrt(cas_dot1(z2, z2, dim, tot));
          S.model_value = S.model;
          S.phase = PH_UPDATE;
          break;
        }
        const double beta = rr_next / S.rr;
        S.rr = rr_next;
        double* dvw = vptr(A, lane, S, V_DV);
        for (long long i = tid; i < dim; i += TR_T) dvw[i] = __dadd_rn(-rw[i], __dmul_rn(beta, dvw[i]));
        __syncthreads();
        ++S.j;
        S.phase = PH_CG;
        break;
      }
      case PH_UPDATE: {
        S.rec_radius = S.radius;
        S.rec_value = S.Fcur;
        S.rho = 0.0;
        S.accepted = 0;
        const double predicted = -S.model_value;
        if (S.cg_exit == TRSTMI_CG_ZERO_GRADIENT || predicted <= 0.0) {
          S.radius *= A.tr.shrink;
          S.underflow = S.radius < 1e-16;
          S.phase = PH_TRIAL;  // record without a trial evaluation
          S.h = -1.0;          // marks "no trial point"
          break;
        }
        v_axpy(vptr(A, lane, S, V_XT), vptr(A, lane, S, V_X), 1.0, vptr(A, lane, S, V_ZS), dim);
        ++S.evals;
        post(0, REQ_OBJ, V_XT, -1, 0.0, V_GT);
        S.h = 1.0;
        S.phase = PH_TRIAL;
        yield = true;
        break;
      }
      case PH_TRIAL: {
        if (S.h > 0.0) {
          const double predicted = -S.model_value;
          const double Ft = ro[0].F;
          const int gfin = v_all_finite(vptr(A, lane, S, V_GT), dim);
          const bool finite = isfinite(Ft) && gfin;
          const double rho = finite ? (S.Fcur - Ft) / predicted : -inf;
          S.rho = rho;
          if (finite && Ft < S.bestv) {
            v_copy(vptr(A, lane, S, V_XB), vptr(A, lane, S, V_XT), dim);
            S.bestv = Ft;
          }
          if (rho > A.tr.eta) {
            int t = S.ix[V_X];
            S.ix[V_X] = S.ix[V_XT];
            S.ix[V_XT] = t;
            t = S.ix[V_G];
            S.ix[V_G] = S.ix[V_GT];
            S.ix[V_GT] = t;
            S.Fcur = Ft;
            S.accepted = 1;
          }
          if (rho < 0.25) {
            S.radius *= A.tr.shrink;
          } else if (rho > 0.75 && S.step_norm >= (1.0 - 1e-10) * S.radius) {
            S.radius = dmin(A.tr.grow * S.radius, A.tr.delta_max);
          }
          S.underflow = S.radius < 1e-16;
        }
        if (tid == 0 && A.oout && S.nrec < A.record_cap) {
          trstmi_outer_out rec;
          rec.stage = S.stage;
          rec.iteration = S.iter;
          rec.cg_exit = S.cg_exit;
          rec.cg_iterations = S.cg_iters;
          rec.accepted = S.accepted;
          rec.pad = 0;
          rec.value = S.rec_value;
          rec.grad_norm = S.grad_norm;
          rec.radius = S.rec_radius;
          rec.rho = S.rho;
          rec.step_norm = S.step_norm;
          A.oout[(long long)S.trial * A.record_cap + S.nrec] = rec;
        }
        if (A.oout && S.nrec < A.record_cap) ++S.nrec;
        ++S.hist;
        ++S.iter;
        if (S.underflow) {
          S.mstatus = TRSTMI_ST_RADIUS_UNDERFLOW;
          S.phase = PH_STAGE_END;
        } else {
          S.phase = PH_OUTER;
        }
        break;
      }
      case PH_STAGE_END: {
        S.outer += S.hist;
        if (S.Fcur < S.bestv) {  // trust_region.hpp:289-293
          v_copy(vptr(A, lane, S, V_XB), vptr(A, lane, S, V_X), dim);
          S.bestv = S.Fcur;
        }
        const int t = S.ix[V_X];  // param <- best-seen x (solver.hpp:192)
        S.ix[V_X] = S.ix[V_XB];
        S.ix[V_XB] = t;
        post(0, REQ_COH_NORM, V_X, -1, 0.0, -1);
        S.phase = PH_COH;
        yield = true;
        break;
      }
      case PH_COH: {
        if (ro[0].zc != INT_MAX) {
          S.status = TRSTMI_TRIAL_ZERO_COLUMN;
          S.zero_col = ro[0].zc;
          S.fail_stage = S.stage;
          S.phase = PH_FINISH;
          break;
        }
        if (tid == 0) {
          trstmi_stage_out so;
          so.delta = S.delta;
          so.objective = S.bestv;
          so.coherence = ro[0].mu;
          so.argmax_pair = ro[0].argmax;
          so.outer_iterations = S.hist;
          so.status = S.mstatus;
          A.sout[(long long)S.trial * A.n_stages + S.stage] = so;
        }
        S.mu = ro[0].mu;
        S.argmax = ro[0].argmax;
        S.stages_done = S.stage + 1;
        ++S.stage;
        S.phase = PH_STAGE;
        break;
      }
      case PH_FINISH: {
        const double* x = vptr(A, lane, S, V_X);
        v_copy(A.params + (long long)S.trial * dim, x, dim);
        if (S.status == TRSTMI_TRIAL_OK && A.frames) {  // normalize_columns(param) (solver.hpp:202)
          double* fo = A.frames + (long long)S.trial * dim;
          for (int j = tid; j < N; j += TR_T) {
            const double* c = x + (long long)j * L;
            double acc = 0.0;
            for (int q = 0; q < L; ++q) acc = fma(c[q], c[q], acc);
            const double a = sqrt(acc);
            for (int q = 0; q < L; ++q) fo[(long long)j * L + q] = __ddiv_rn(c[q], a);
          }
        }
        if (tid == 0) {
          trstmi_trial_out o;
          o.coherence = S.mu;
          o.argmax_pair = S.argmax;
          o.status = S.status;
          o.stages_done = S.stages_done;
          o.zero_col = S.zero_col;
          o.fail_stage = S.fail_stage;
          o.outer_iterations = S.outer;
          o.evals = S.evals;
          o.hvps = S.hvps;
          o.records = S.nrec;
          A.tout[S.trial] = o;
        }
        __syncthreads();
        S.phase = PH_START;
        break;
      }
      default:
        yield = true;
        break;
    }
  }
  if (tid == 0) {
    if (nobj) {
      const int b = atomicAdd(&A.counters[0], nobj);
      for (int s = 0; s < nobj; ++s) A.act_obj[b + s] = 2 * lane + s;
    }
    if (ncoh) {
      const int b = atomicAdd(&A.counters[1], ncoh);
      A.act_coh[b] = 2 * lane;
    }
    if (S.phase != PH_IDLE) atomicAdd(&A.counters[3], 1);
    A.lanes[lane] = S;
  }
}

}  // namespace trstmi_bde
