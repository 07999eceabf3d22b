// csmc.cu — auxiliary particle Gibbs on B200 (fkpg.cpp:19-280), gradient
// proposals linearized at the auxiliary observation (fkpg.cpp:154-186), plus
// the parallel-in-time conditional SMC with independent proposals.
//
// variant REFERENCE (K6): the reference's conditional SMC sweep with
//   multinomial resampling and backward index sampling (fkpg.cpp:44-152),
//   one CTA per chain, particles across threads, sequential in t.  Resampling
//   uses the reference's exact sequential cumulative sum and "first i with
//   u <= acc" rule (fkpg.cpp:29-37), so ancestor and backward indices agree
//   with the reference bit for bit given the same weights.
// variant PIT (K7, no reference: SPEC.md:16): with independent proposals the
//   particle lattice x_t^i and the parent-free weights are generated for all t
//   at once (fully parallel); the index path is then drawn exactly from the
//   lattice law P(i_{0:T}) ∝ w_0(i_0) Π p(x_t^{i_t} | x_{t-1}^{i_{t-1}}) w_t(i_t)
//   by log-sum-exp forward messages over the N×N transitions and backward
//   index sampling with the reference's stream addresses.
#include <cmath>

#include <cooperative_groups.h>

#include "common.cuh"
#include "dense.cuh"
#include "group.cuh"
#include "rng.cuh"
#include "target.cuh"

namespace auxmc_gpu {

int launch_target_factors(const DevTarget& tg, double* Ls, double* logdet, int* fst,
                          cudaStream_t s);
int launch_aux_obs(int C, int T, int d, const double* x, const double* delta, const uint64_t* it,
                   double* u, cudaStream_t s);

struct FactorRef {
  FactorLayout fl;
  const double* Ls;
  const double* logdet;
  __device__ __forceinline__ const double* L(int j) const { return Ls + (size_t)j * fl.W * fl.W; }
};

__device__ __forceinline__ double log_pot_dev(const DevTarget& tg, const FactorRef& f, int t,
                                              const double* x, double* r) {
  double lp = 0.0;
  const int d = tg.dx;
  if (tg.q > 0 && tg.emask[t]) {
    const double* H = tg.eHt(t);
    const double* cc = tg.ect(t);
    const double* y = tg.ey + (size_t)t * tg.q;
    for (int i = 0; i < tg.q; ++i) {
      double s = 0.0;
      for (int j = 0; j < d; ++j) s += H[i * d + j] * x[j];
      r[i] = y[i] - (s + cc[i]);
    }
    const int je = 1 + f.fl.nQ + (tg.ne > 1 ? t : 0);
    lp += gauss_term(tg.q, r, f.L(je), f.logdet[je]);
  }
  if (tg.gmask[t]) {
    const int jg = 1 + f.fl.nQ + f.fl.nE + (tg.ne > 1 ? t : 0);
    lp += generic_log_g(tg, t, x, f.fl.nG ? f.L(jg) : nullptr, f.fl.nG ? f.logdet[jg] : 0.0, r);
  }
  return lp;
}

__device__ __forceinline__ double log_dyn_dev(const DevTarget& tg, const FactorRef& f, int t,
                                              const double* xp, const double* x, double* r) {
  const int d = tg.dx;
  for (int i = 0; i < d; ++i) r[i] = x[i] - dyn_mean_i(tg, t, xp, i);
  const int jq = 1 + (f.fl.nQ > 1 ? t : 0);
  return gauss_term(d, r, f.L(jq), f.logdet[jq]);
}

__device__ __forceinline__ double log_prior_dev(const DevTarget& tg, const FactorRef& f,
                                                const double* x, double* r) {
  for (int i = 0; i < tg.dx; ++i) r[i] = x[i] - tg.m0[i];
  return gauss_term(tg.dx, r, f.L(0), f.logdet[0]);
}

// log N(x; mean, (δ/2) I) through the LLT path of gauss::log_pdf (gauss.cpp:51-57)
__device__ __forceinline__ double log_q_dev(int d, const double* x, const double* mean, double sq2) {
  double sq = 0.0, ld = 0.0;
  for (int i = 0; i < d; ++i) {
    const double z = (x[i] - mean[i]) / sq2;
    sq += z * z;
  }
  for (int i = 0; i < d; ++i) ld += log(sq2);
  return -0.5 * (d * kLog2Pi + sq) - ld;
}

// isotropic_log_pdf(u - x, var) (gauss.cpp:59-62)
__device__ __forceinline__ double iso_dev(int d, const double* u, const double* x, double var) {
  double sq = 0.0;
  for (int i = 0; i < d; ++i) {
    const double r = u[i] - x[i];
    sq += r * r;
  }
  return -0.5 * (d * (kLog2Pi + log(var)) + sq / var);
}

// potential of the auxiliary FK model (fkpg.cpp:212-223), gradient mode
__device__ __forceinline__ double potential_dev(const DevTarget& tg, const FactorRef& f, int t,
                                                const double* xp, const double* x, const double* u_t,
                                                const double* mq_t, double delta, double sq2,
                                                double* r) {
  const int d = tg.dx;
  double lg = log_pot_dev(tg, f, t, x, r) + iso_dev(d, u_t, x, delta / 2.0);
  const double ld = t == 0 ? log_prior_dev(tg, f, x, r) : log_dyn_dev(tg, f, t - 1, xp, x, r);
  lg += ld - log_q_dev(d, x, mq_t, sq2);
  return lg;
}

// ---------------------------------------------------------------- prep kernels
__global__ void k_pg_keys(int C, const uint64_t* root, const long long* iter, uint64_t* it) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < C) it[c] = derive(root[c], kIteration, (uint64_t)iter[c]);
}

// proposal mean u_t + (δ/2) ∇ log g_t(u_t) (fkpg.cpp:166-171), both factors
__global__ void k_pg_prop_mean(DevTarget tg, FactorRef f, int C, const double* __restrict__ u,
                               const double* __restrict__ delta, double* mq, int* bad) {
  const int T = tg.T, d = tg.dx;
  const long long n = (long long)C * (T + 1);
  double r[64], g[64];
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(q / (T + 1)), t = (int)(q % (T + 1));
    const double* ut = u + (size_t)q * d;
    const int jg = 1 + f.fl.nQ + f.fl.nE + (tg.ne > 1 ? t : 0);
    generic_grad(tg, t, ut, f.fl.nG ? f.L(jg) : nullptr, r, g);
    if (tg.q > 0 && tg.emask[t]) {  // + H^T R^{-1} (y - H x - c) (target.cpp:90-98)
      const double* H = tg.eHt(t);
      const double* cc = tg.ect(t);
      const double* y = tg.ey + (size_t)t * tg.q;
      const int je = 1 + f.fl.nQ + (tg.ne > 1 ? t : 0);
      const double* L = f.L(je);
      const int qn = tg.q;
      for (int i = 0; i < qn; ++i) {
        double s = 0.0;
        for (int j = 0; j < d; ++j) s += H[i * d + j] * ut[j];
        r[i] = (y[i] - s) - cc[i];
      }
      for (int i = 0; i < qn; ++i) {
        double s = r[i];
        for (int j = 0; j < i; ++j) s -= L[i * qn + j] * r[j];
        r[i] = s / L[i * qn + i];
      }
      for (int i = qn - 1; i >= 0; --i) {
        double s = r[i];
        for (int j = i + 1; j < qn; ++j) s -= L[j * qn + i] * r[j];
        r[i] = s / L[i * qn + i];
      }
      for (int j = 0; j < d; ++j) {
        double s = 0.0;
        for (int i = 0; i < qn; ++i) s += H[i * d + j] * r[i];
        g[j] += s;
      }
    }
    const double h = delta[c] / 2.0;
    for (int i = 0; i < d; ++i) {
      mq[(size_t)q * d + i] = ut[i] + h * g[i];
      if (!isfinite(g[i]) && bad) atomicOr(bad + c, 1);
    }
  }
}

// ---------------------------------------------------------------- block helpers
__device__ __forceinline__ double block_max(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = red[0];
    for (int i = 1; i < nw; ++i) m = fmax(m, red[i]);
    red[32] = m;
  }
  __syncthreads();
  return red[32];
}

// Sequential running sum of x[0..N) in the reference's left-to-right order.  x
// and cum are distinct shared arrays (__restrict__): with the loop unrolled by 8
// the loads of a group issue ahead of its dependent adds and stores, instead of
// one load-after-store round trip per element.
__device__ __forceinline__ void serial_cumsum(int N, const double* __restrict__ x,
                                              double* __restrict__ cum) {
  double acc = 0.0;
#pragma unroll 8
  for (int i = 0; i < N; ++i) {
    acc += x[i];
    cum[i] = acc;
  }
}

// normalize (fkpg.cpp:19-27) over logw[0..N) in shared memory -> W (shared),
// sequential sum as the reference's order; returns false if degenerate.
__device__ __forceinline__ bool block_normalize(int N, const double* logw, double* W, double* red) {
  double m = -INFINITY;
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    const double v = logw[i];
    m = (v > m || m != m) ? v : m;
  }
  // NaN handling: Eigen maxCoeff; treat NaN like the reference's non-finite max
  m = block_max(m, red);
  if (!isfinite(m)) return false;
  for (int i = threadIdx.x; i < N; i += blockDim.x) W[i] = exp(logw[i] - m);
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
#pragma unroll 8
    for (int i = 0; i < N; ++i) s += W[i];
    red[33] = s;
  }
  __syncthreads();
  const double s = red[33];
  for (int i = threadIdx.x; i < N; i += blockDim.x) W[i] = W[i] / s;
  __syncthreads();
  return true;
}

// cumulative weights in the reference's sequential order (fkpg.cpp:29-37)
__device__ __forceinline__ void block_cumsum(int N, const double* W, double* cum) {
  if (threadIdx.x == 0) serial_cumsum(N, W, cum);
  __syncthreads();
}

// first i with u <= cum[i], else N-1
__device__ __forceinline__ int draw_index(int N, const double* cum, double u) {
  int lo = 0, hi = N;  // lower_bound of u in cum (non-decreasing)
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (u <= cum[mid]) hi = mid;
    else lo = mid + 1;
  }
  return lo < N ? lo : N - 1;
}

struct PgArgs {
  int C, N;
  double* x;
  uint64_t* keys;
  const double* delta;
  const uint64_t* it;
  const double* u;
  const double* mq;
  double* part;     // [C][T+1][N][d]
  double* Wt;       // [C][T+1][N] normalized weights (or forward log-messages for PIT)
  double* traj;     // [C][T+1][d] new path
  uint64_t* tkeys;  // [C][T+1]
  int* status;
  int* bad_t;
  int* anc;         // optional [C][T+1][N]
  int* sel;         // optional [C][T+1]
  const int* grad_bad;
  int mode;         // AUXMC_PG_PRIOR / GRADIENT / ADAPTED (fkpg.hpp:58)
  const double* adf;  // ADAPTED: [C][nad][2 d^2 + 1] gain | L | logdet per proposal class
  int nad;
  const int* ad_bad;  // ADAPTED: [C] factorization failure of a proposal class
  int pm;             // AUXMC_PM_*: pseudo-marginal estimator of the potentials
};

// pm_potential (fkpg.cpp:233-250) with the device estimator family: the estimate from
// the particle's aux key, NaN / negative -> ContractError (flagged), log(est) or -inf.
__device__ __forceinline__ double pm_apply(int kind, double lg, uint64_t key, int* contract) {
  if (kind == AUXMC_PM_NONE) return lg;
  double est;
  if (kind == AUXMC_PM_TWO_POINT) {
    const double eps = uniform_at(key, 0) < 0.5 ? 0.5 : 1.5;
    est = exp(lg) * eps;
  } else if (kind == AUXMC_PM_EXACT) {
    est = exp(lg);
  } else {
    est = -0.1;
  }
  if (est != est || est < 0.0) {
    atomicOr(contract, 1);
    return -INFINITY;
  }
  return est > 0.0 ? log(est) : -INFINITY;
}

// proposal class of step t: 0 = prior at t = 0 (m0, P0), 1 + j = dynamics with Q_j
__device__ __forceinline__ int prop_class(const FactorRef& f, int t) {
  return t == 0 ? 0 : 1 + (f.fl.nQ > 1 ? t - 1 : 0);
}

// Fully adapted proposal factors (fkpg.cpp:173-185) per (chain, class): the
// conjugate combination of N(prior_mean, prior_cov) with z = x + N(0, (δ/2) I).
// gain and cov depend on (δ, class) only; the mean depends on the parent.
// One warp per item: S = pc + hI, gain = solve_spd(S, pc)^T, a = I - gain,
// cov = symm(a pc a^T + h gain gain^T), L = chol_psd(cov).
__global__ void k_pg_adapted(DevTarget tg, int C, int nad, const double* __restrict__ delta,
                             double* adf, int* bad) {
  extern __shared__ double smem[];
  const int d = tg.dx, dd = d * d;
  Grp g = warp_group();
  const int gid = threadIdx.x >> 5, gpb = blockDim.x >> 5;
  double* pc = smem + (size_t)gid * (6 * dd + 4);
  double* S = pc + dd;
  double* L = S + dd;
  double* X = L + dd;
  double* A = X + dd;
  double* Wm = A + dd;
  double* red = Wm + dd;
  int* flag = reinterpret_cast<int*>(red + 2);
  for (int j = blockIdx.x * gpb + gid; j < C * nad; j += gridDim.x * gpb) {
    const int c = j / nad, k = j % nad;
    const double* src = k == 0 ? tg.P0 : tg.Q + (size_t)(k - 1) * dd;
    const double h = delta[c] / 2.0;
    for (int i = g.lane; i < dd; i += g.size) {
      pc[i] = src[i];
      S[i] = src[i] + (i / d == i % d ? h * 1.0 : 0.0);
      X[i] = src[i];
    }
    g.sync();
    int st = g_factor_psd(g, d, S, L, Wm, flag, red);  // solve_spd (gauss.cpp:87-89)
    g_llt_solve(g, d, L, d, X);
    g.sync();
    for (int i = g.lane; i < dd; i += g.size) {
      A[i] = X[(i % d) * d + i / d];                         // gain
      Wm[i] = (i / d == i % d ? 1.0 : 0.0) - X[(i % d) * d + i / d];  // a = I - gain
    }
    g.sync();
    g_mm(g, d, d, d, Wm, pc, X);       // a pc
    g.sync();
    g_mm_nt(g, d, d, d, X, Wm, S);     // (a pc) a^T
    g.sync();
    g_mm_nt(g, d, d, d, A, A, X);      // gain gain^T
    g.sync();
    for (int i = g.lane; i < dd; i += g.size) S[i] = S[i] + h * X[i];
    g.sync();
    g_symm(g, d, S);                   // Gaussian ctor (gauss.cpp:38-42)
    g.sync();
    st |= g_chol_psd(g, d, S, L, Wm, flag, red);
    double* out = adf + (size_t)j * (2 * dd + 1);
    for (int i = g.lane; i < dd; i += g.size) {
      out[i] = A[i];
      out[dd + i] = L[i];
    }
    if (g.lane == 0) {
      double ld = 0.0;
      for (int i = 0; i < d; ++i) ld += log(L[i * d + i]);
      out[2 * dd] = ld;
      if (st) atomicOr(bad + c, 1);
    }
    g.sync();
  }
}

// mean of the prior / fully adapted proposal of step t given the parent
// (fkpg.cpp:154-185); also returns its factor and log-determinant.
__device__ __forceinline__ void parent_proposal(const DevTarget& tg, const FactorRef& f,
                                                const PgArgs& a, int c, int t, const double* parent,
                                                const double* mq_t, double* mean, const double** Lp,
                                                double* ldp) {
  const int d = tg.dx;
  for (int k = 0; k < d; ++k) mean[k] = t == 0 ? tg.m0[k] : dyn_mean_i(tg, t - 1, parent, k);
  const int cls = prop_class(f, t);
  if (a.mode == AUXMC_PG_PRIOR) {
    *Lp = f.L(cls);  // factor list: 0 = P0, 1 + j = Q_j
    *ldp = f.logdet[cls];
    return;
  }
  const double* ad = a.adf + ((size_t)c * a.nad + cls) * (2 * d * d + 1);
  double z[64];
  for (int k = 0; k < d; ++k) z[k] = mq_t[k] - mean[k];
  for (int k = 0; k < d; ++k) {
    double s = 0.0;
    for (int j = 0; j < d; ++j) s += ad[k * d + j] * z[j];
    mean[k] = mean[k] + s;
  }
  *Lp = ad + d * d;
  *ldp = ad[2 * d * d];
}

// ---------------------------------------------------------------- K6 reference cSMC
__global__ void k_csmc_reference(DevTarget tg, FactorRef f, PgArgs a) {
  extern __shared__ double sm[];
  const int N = a.N, T = tg.T, d = tg.dx;
  const int c = blockIdx.x;
  double* logw = sm;           // N
  double* W = logw + N;        // N
  double* cum = W + N;         // N
  double* red = cum + N;       // 40
  double* chosen = red + 40;   // d
  int* anc = reinterpret_cast<int*>(chosen + 64);  // N
  int* contract = anc + N;     // pseudo-marginal ContractError flag
  const double delta = a.delta[c];
  const double sq2 = sqrt(delta / 2.0);  // LLT of (δ/2) I (gauss.cpp:64-67)
  const uint64_t it = a.it[c];
  double* P = a.part + (size_t)c * (T + 1) * N * d;
  double* Wg = a.Wt + (size_t)c * (T + 1) * N;
  const double* uc = a.u + (size_t)c * (T + 1) * d;
  const double* mqc = a.mq + (size_t)c * (T + 1) * d;
  const double* ref = a.x + (size_t)c * (T + 1) * d;
  double r[64], xv[64], pmean[64];
  if (a.mode != AUXMC_PG_PRIOR && a.grad_bad && a.grad_bad[c]) {
    // non-finite proposal mean: treat as degenerate
    if (threadIdx.x == 0) { a.status[c] = AUXMC_E_DEGENERATE; a.bad_t[c] = 0; }
    return;
  }
  if (a.mode == AUXMC_PG_ADAPTED && a.ad_bad && a.ad_bad[c]) {  // solve_spd / chol failed
    if (threadIdx.x == 0) { a.status[c] = AUXMC_E_FACTOR; a.bad_t[c] = 0; }
    return;
  }
  double* tr = a.traj + (size_t)c * (T + 1) * d;
  uint64_t* tk = a.tkeys + (size_t)c * (T + 1);
  auto pm_key = [&](int t, int i) -> uint64_t {
    if (i == 0) return a.keys[(size_t)c * (T + 1) + t];
    return key_at(derive(derive(it, kStep, (uint64_t)t), kPmKey, (uint64_t)i), 0);
  };
  if (threadIdx.x == 0) *contract = 0;
  __syncthreads();
  for (int t = 0; t <= T; ++t) {
    const uint64_t st = derive(it, kStep, (uint64_t)t);
    if (t > 0) {
      block_cumsum(N, W, cum);
      const uint64_t rs = derive(st, kResample, 0);
      for (int i = threadIdx.x; i < N; i += blockDim.x)
        anc[i] = i == 0 ? 0 : draw_index(N, cum, uniform_at(rs, (uint64_t)(i - 1)));
      __syncthreads();
    }
    const uint64_t kp = derive_label(st, kParticle);
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
      const double* parent = t > 0 ? P + ((size_t)(t - 1) * N + anc[i]) * d : nullptr;
      if (a.mode != AUXMC_PG_GRADIENT) {
        // prior / fully adapted: the proposal depends on the parent (fkpg.cpp:154-185)
        const double* Lp;
        double ldp;
        parent_proposal(tg, f, a, c, t, parent, mqc + (size_t)t * d, pmean, &Lp, &ldp);
        if (i == 0) {
          for (int k = 0; k < d; ++k) xv[k] = ref[(size_t)t * d + k];
        } else {
          const uint64_t pk = derive_index(kp, (uint64_t)i);
          double xi[64];
          for (int k = 0; k < d; ++k) xi[k] = normal_at(pk, (uint64_t)k);
          for (int k = 0; k < d; ++k) {  // mean + L xi (gauss.cpp:64-67)
            double s = 0.0;
            for (int j = 0; j <= k; ++j) s += Lp[k * d + j] * xi[j];
            xv[k] = pmean[k] + s;
          }
        }
        for (int k = 0; k < d; ++k) P[((size_t)t * N + i) * d + k] = xv[k];
        // pot (fkpg.cpp:212-223)
        double lg = log_pot_dev(tg, f, t, xv, r) + iso_dev(d, uc + (size_t)t * d, xv, delta / 2.0);
        if (a.mode == AUXMC_PG_ADAPTED) {
          const double ld = t == 0 ? log_prior_dev(tg, f, xv, r) : log_dyn_dev(tg, f, t - 1, parent, xv, r);
          for (int k = 0; k < d; ++k) r[k] = xv[k] - pmean[k];
          lg += ld - gauss_term(d, r, Lp, ldp);
        }
        logw[i] = a.pm ? pm_apply(a.pm, lg, pm_key(t, i), contract) : lg;
        if (a.anc) a.anc[((size_t)c * (T + 1) + t) * N + i] = t > 0 ? anc[i] : 0;
        continue;
      }
      if (i == 0) {
        for (int k = 0; k < d; ++k) xv[k] = ref[(size_t)t * d + k];
      } else {
        const uint64_t pk = derive_index(kp, (uint64_t)i);
        for (int k = 0; k < d; ++k) xv[k] = mqc[(size_t)t * d + k] + sq2 * normal_at(pk, (uint64_t)k);
      }
      for (int k = 0; k < d; ++k) P[((size_t)t * N + i) * d + k] = xv[k];
      const double lgp = potential_dev(tg, f, t, parent, xv, uc + (size_t)t * d, mqc + (size_t)t * d,
                                       delta, sq2, r);
      logw[i] = a.pm ? pm_apply(a.pm, lgp, pm_key(t, i), contract) : lgp;
      if (a.anc) a.anc[((size_t)c * (T + 1) + t) * N + i] = t > 0 ? anc[i] : 0;
    }
    __syncthreads();
    if (*contract) {  // ContractError from the pseudo-marginal estimator (fkpg.cpp:241-243)
      if (threadIdx.x == 0) { a.status[c] = AUXMC_E_CONTRACT; a.bad_t[c] = t; }
      return;
    }
    if (!block_normalize(N, logw, W, red)) {
      if (threadIdx.x == 0) { a.status[c] = AUXMC_E_DEGENERATE; a.bad_t[c] = t; }
      return;
    }
    for (int i = threadIdx.x; i < N; i += blockDim.x) Wg[(size_t)t * N + i] = W[i];
    __syncthreads();
  }
  // terminal index (fkpg.cpp:127-133) and backward index sampling (:135-150)
  block_cumsum(N, W, cum);
  if (threadIdx.x == 0) {
    const int sel = draw_index(N, cum, uniform_at(derive(it, kTerminalIndex, 0), 0));
    for (int k = 0; k < d; ++k) {
      chosen[k] = P[((size_t)T * N + sel) * d + k];
      tr[(size_t)T * d + k] = chosen[k];
    }
    tk[T] = pm_key(T, sel);
    if (a.sel) a.sel[(size_t)c * (T + 1) + T] = sel;
  }
  __syncthreads();
  for (int t = T - 1; t >= 0; --t) {
    // m_logpdf(t+1, ., chosen) and the parent-free part of log_g(t+1, ., chosen)
    const double* mq1 = mqc + (size_t)(t + 1) * d;
    const double mlp = log_q_dev(d, chosen, mq1, sq2);
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
      const double* xi = P + ((size_t)t * N + i) * d;
      if (a.mode != AUXMC_PG_GRADIENT) {
        // log W + m_logpdf(t+1, x_t^i, chosen) + log_g(t+1, x_t^i, chosen) (fkpg.cpp:137-143)
        const double* Lp;
        double ldp;
        parent_proposal(tg, f, a, c, t + 1, xi, mq1, pmean, &Lp, &ldp);
        for (int k = 0; k < d; ++k) r[k] = chosen[k] - pmean[k];
        const double lq = gauss_term(d, r, Lp, ldp);
        double lg = log_pot_dev(tg, f, t + 1, chosen, r) +
                    iso_dev(d, uc + (size_t)(t + 1) * d, chosen, delta / 2.0);
        if (a.mode == AUXMC_PG_ADAPTED) lg += log_dyn_dev(tg, f, t, xi, chosen, r) - lq;
        if (a.pm) lg = pm_apply(a.pm, lg, tk[t + 1], contract);
        logw[i] = log(Wg[(size_t)t * N + i]) + lq + lg;
        continue;
      }
      double lg = potential_dev(tg, f, t + 1, xi, chosen, uc + (size_t)(t + 1) * d, mq1,
                                delta, sq2, r);
      if (a.pm) lg = pm_apply(a.pm, lg, tk[t + 1], contract);
      logw[i] = log(Wg[(size_t)t * N + i]) + mlp + lg;
    }
    __syncthreads();
    if (*contract) {
      if (threadIdx.x == 0) { a.status[c] = AUXMC_E_CONTRACT; a.bad_t[c] = t; }
      return;
    }
    if (!block_normalize(N, logw, W, red)) {
      if (threadIdx.x == 0) { a.status[c] = AUXMC_E_DEGENERATE; a.bad_t[c] = t; }
      return;
    }
    block_cumsum(N, W, cum);
    if (threadIdx.x == 0) {
      const int sel = draw_index(N, cum, uniform_at(derive(it, kBackwardIndex, (uint64_t)t), 0));
      for (int k = 0; k < d; ++k) {
        chosen[k] = P[((size_t)t * N + sel) * d + k];
        tr[(size_t)t * d + k] = chosen[k];
      }
      tk[t] = pm_key(t, sel);
      if (a.sel) a.sel[(size_t)c * (T + 1) + t] = sel;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- K7 PIT cSMC
// Lattice particles and parent-free log-weights for every (t, i) at once.
__global__ void k_pit_particles(DevTarget tg, FactorRef f, PgArgs a, double* lw) {
  const int N = a.N, T = tg.T, d = tg.dx;
  const long long n = (long long)a.C * (T + 1) * N;
  double r[64], xv[64];
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(q % N);
    const long long ct = q / N;
    const int t = (int)(ct % (T + 1)), c = (int)(ct / (T + 1));
    const double delta = a.delta[c], sq2 = sqrt(delta / 2.0);
    const double* mq = a.mq + ((size_t)c * (T + 1) + t) * d;
    if (i == 0) {
      for (int k = 0; k < d; ++k) xv[k] = a.x[((size_t)c * (T + 1) + t) * d + k];
    } else {
      const uint64_t pk = derive(derive(a.it[c], kStep, (uint64_t)t), kParticle, (uint64_t)i);
      for (int k = 0; k < d; ++k) xv[k] = mq[k] + sq2 * normal_at(pk, (uint64_t)k);
    }
    double* P = a.part + (size_t)q * d;
    for (int k = 0; k < d; ++k) P[k] = xv[k];
    const double* ut = a.u + ((size_t)c * (T + 1) + t) * d;
    double v = log_pot_dev(tg, f, t, xv, r) + iso_dev(d, ut, xv, delta / 2.0);
    if (t == 0) v += log_prior_dev(tg, f, xv, r);
    v -= log_q_dev(d, xv, mq, sq2);
    lw[q] = v;
  }
}

// exp(x) for x <= 0 in the LSE inner loop: x = k ln2 + r, |r| <= ln2/2, exp(r) by
// its degree-11 Taylor polynomial (truncation < 1e-15 relative), 2^k by exponent
// construction; x < -708 returns 0 (below DBL_MIN: the sum's exact online
// fallback handles total underflow).  About half the instructions of the libm
// routine, which also handles overflow, NaN and subnormal results.
__device__ __forceinline__ double exp_nonpos(double x) {
  const double kLog2e = 1.4426950408889634, kLn2Hi = 6.93147180369123816490e-01,
               kLn2Lo = 1.90821492927058770002e-10;
  const double kd = rint(x * kLog2e);
  double r = fma(-kd, kLn2Hi, x);
  r = fma(-kd, kLn2Lo, r);
  double p = 2.505210838544172e-08;  // 1/11!
  p = fma(p, r, 2.755731922398589e-07);
  p = fma(p, r, 2.7557319223985893e-06);
  p = fma(p, r, 2.48015873015873e-05);
  p = fma(p, r, 1.984126984126984e-04);
  p = fma(p, r, 1.388888888888889e-03);
  p = fma(p, r, 8.333333333333333e-03);
  p = fma(p, r, 4.1666666666666664e-02);
  p = fma(p, r, 1.6666666666666666e-01);
  p = fma(p, r, 0.5);
  p = fma(p, r, 1.0);
  p = fma(p, r, 1.0);
  const int k = (int)kd;
  const double scale = __hiloint2double((k + 1023) << 20, 0);
  return x < -708.0 ? 0.0 : p * scale;
}

// ---------------------------------------------------------------- PIT forward, cluster form
// Forward log-messages alpha_t(j) = lw_t(j) + LSE_i(alpha_{t-1}(i) + log p(x_t^j | x_{t-1}^i))
// with the whitened pair term (see k_pit_forward_backward), for small state dims.  One
// thread-block CLUSTER of CS CTAs per chain: CTA r owns the j-slice
// [r N / CS, (r+1) N / CS) of every step, and after each step the CTAs exchange their
// slices of alpha_t through distributed shared memory (one cluster barrier per step,
// slices double-buffered by step parity).  CS = 8 puts one chain on 8 SMs: the
// single-chain latency case (SURVEY.md §8(d) C4 "report 1 chain"); CS = 1 is the
// many-chain batch.  The time axis stays a recursion: an associative scan over the N x N
// log-semiring transition operators would cost O(T N^3) exp evaluations (2.7e11 at
// C4's N = 256, T = 2^14) against O(T N^2) here.
//
// The LSE over i uses one canonical partition for every cluster size, so a chain's
// messages (and hence its draws) do not depend on the batch size: 32 contiguous i-parts
// [p N / 32, (p+1) N / 32), each summed with four interleaved accumulators, combined by a
// pairwise tree; total underflow falls back to the exact online LSE over all i.
#ifndef AUXMC_PIT_EXP
#define AUXMC_PIT_EXP 0  // 9: clock64 stamps of the cluster forward pass (timing only)
#endif
constexpr int kPitParts = 32;
constexpr int kChaseBlock = 64;  // table rows staged per chase block (64 x N ints)

template <int DT>
__device__ __forceinline__ void pit_whiten(const double* LQ, const double* x, double* w) {
#pragma unroll
  for (int k = 0; k < DT; ++k) {
    double acc = x[k];
#pragma unroll
    for (int l = 0; l < k; ++l) acc -= LQ[k * DT + l] * w[l];
    w[k] = acc / LQ[k * DT + k];
  }
}

// Pre-pass: the whitened operands of every forward step, V[c][t-1][i] =
// L_q^{-1} mean(x_{t-1}^i) and X[c][t-1][j] = L_q^{-1} x_t^j (q = q(t), t = 1..T), for all
// (chain, t, i) in parallel — off the forward recursion's critical path.
template <int DT>
__global__ void k_pit_whiten(DevTarget tg, FactorRef f, PgArgs a, double* V, double* X) {
  const int N = a.N, T = tg.T;
  const long long n = (long long)a.C * T * N;
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(q % N);
    const long long ct = q / N;
    const int t = (int)(ct % T) + 1, c = (int)(ct / T);
    const double* LQ = f.L(1 + (f.fl.nQ > 1 ? t - 1 : 0));
    const double* P = a.part + (size_t)c * (T + 1) * N * DT;
    double m[DT];
#pragma unroll
    for (int k = 0; k < DT; ++k) m[k] = dyn_mean_i(tg, t - 1, P + ((size_t)(t - 1) * N + i) * DT, k);
    pit_whiten<DT>(LQ, m, V + q * DT);
    pit_whiten<DT>(LQ, P + ((size_t)t * N + i) * DT, X + q * DT);
  }
}

// The forward recursion.  Per step: am = max alpha_{t-1} (CS > 1: from the maxima the
// CTAs pushed with their slices), the pair sums of the own j-slice over the canonical
// i-partition, then each CTA pushes its alpha_t slice (and its maximum) into every CTA's
// shared memory (parity double buffers) and the cluster synchronizes once.  The next
// step's whitened operands are prefetched into registers during the pair loop.
template <int DT>
__global__ void __launch_bounds__(1024, 1)
    k_pit_forward_cluster(DevTarget tg, FactorRef f, PgArgs a, const double* lw, const double* V,
                          const double* X, int CS) {
  namespace cg = cooperative_groups;
  extern __shared__ double sm[];
  const int N = a.N, T = tg.T;
  const int rank = (int)blockIdx.x % CS;
  const int c = (int)blockIdx.x / CS;
  cg::cluster_group cluster = cg::this_cluster();
  const int j0 = (int)((long long)rank * N / CS), j1 = (int)((long long)(rank + 1) * N / CS);
  const int JL = j1 - j0, JLmax = (N + CS - 1) / CS;
  double* alpha = sm;                                // 2 x N   alpha_{t}, by parity
  double* vbuf = alpha + 2 * N;                      // 2 x N*DT
  double* xbuf = vbuf + (size_t)2 * N * DT;          // 2 x JLmax*DT
  double* ai = xbuf + (size_t)2 * JLmax * DT;        // N
  double* partial = ai + N;                          // kPitParts x JLmax
  double* smaxs = partial + kPitParts * JLmax;       // 2 x CS pushed slice maxima
  double* red = smaxs + 2 * CS;                      // 40
  const double* LW = lw + (size_t)c * (T + 1) * N;
  double* A = a.Wt + (size_t)c * (T + 1) * N;
  const double* Vc = V + (size_t)c * T * N * DT;
  const double* Xc = X + (size_t)c * T * N * DT;
  const int nV = N * DT, nX = JL * DT;
  // operands of step t into buffer t & 1 (thread-strided; one or two values per thread)
  auto load_ops = [&](int t, double* vdst, double* xdst) {
    for (int q = threadIdx.x; q < nV + nX; q += blockDim.x) {
      if (q < nV) vdst[q] = Vc[(size_t)(t - 1) * nV + q];
      else xdst[q - nV] = Xc[((size_t)(t - 1) * N + j0) * DT + (q - nV)];
    }
  };
  for (int i = threadIdx.x; i < N; i += blockDim.x) alpha[i] = LW[i];
  for (int j = j0 + (int)threadIdx.x; j < j1; j += blockDim.x) A[j] = LW[j];
  if (T >= 1) load_ops(1, vbuf + (size_t)1 * nV, xbuf + (size_t)1 * JLmax * DT);
  __syncthreads();
#if AUXMC_PIT_EXP == 9
  __shared__ long long pts[16 * 8];
  auto pst = [&](int t, int e) {
    if (blockIdx.x == 0 && threadIdx.x == 0 && t >= 1000 && t < 1016) pts[(t - 1000) * 8 + e] = clock64();
  };
#else
  auto pst = [](int, int) {};
#endif
  for (int t = 1; t <= T; ++t) {
    pst(t, 0);
    const double* aprev = alpha + (size_t)((t - 1) & 1) * N;
    double am;
    if (t > 1 && CS > 1 && JLmax <= 32) {
      am = -INFINITY;
      for (int r = 0; r < CS; ++r) am = fmax(am, smaxs[((t - 1) & 1) * CS + r]);
    } else {
      am = block_max([&] {
        double m = -INFINITY;
        for (int i = threadIdx.x; i < N; i += blockDim.x) m = fmax(m, aprev[i]);
        return m;
      }(), red);
    }
    if (!isfinite(am)) {  // every message at t-1 collapsed (fkpg.cpp:19-23 names t-1)
      if (rank == 0 && threadIdx.x == 0) {
        a.status[c] = AUXMC_E_DEGENERATE;
        a.bad_t[c] = t - 1;
      }
      break;  // uniform over the cluster: every CTA computed the same am
    }
    for (int i = threadIdx.x; i < N; i += blockDim.x) ai[i] = aprev[i] - am;
    // prefetch step t+1's operands into registers (written to the other buffer below)
    double pf[2] = {0.0, 0.0};
    if (t < T) {
      int k = 0;
      for (int q = threadIdx.x; q < nV + nX && k < 2; q += blockDim.x, ++k)
        pf[k] = q < nV ? Vc[(size_t)t * nV + q] : Xc[((size_t)t * N + j0) * DT + (q - nV)];
    }
    __syncthreads();
    pst(t, 1);
    const int jq = 1 + (f.fl.nQ > 1 ? t - 1 : 0);
    const double M = -0.5 * (DT * kLog2Pi) - f.logdet[jq];
    const double* vi = vbuf + (size_t)(t & 1) * nV;
    const double* wj = xbuf + (size_t)(t & 1) * JLmax * DT;
    for (int item = threadIdx.x; item < JL * kPitParts; item += blockDim.x) {
      const int jl = item % JL, p = item / JL;
      const int ilo = (int)((long long)p * N / kPitParts), ihi = (int)((long long)(p + 1) * N / kPitParts);
      double w[DT];
#pragma unroll
      for (int k = 0; k < DT; ++k) w[k] = wj[jl * DT + k];
      double acc4[4] = {0.0, 0.0, 0.0, 0.0};
      int i = ilo;
      for (; i + 4 <= ihi; i += 4) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          double sq = 0.0;
#pragma unroll
          for (int k = 0; k < DT; ++k) {
            const double z = w[k] - vi[(i + u) * DT + k];
            sq += z * z;
          }
          acc4[u] += exp_nonpos(ai[i + u] - 0.5 * sq);
        }
      }
      for (; i < ihi; ++i) {
        double sq = 0.0;
#pragma unroll
        for (int k = 0; k < DT; ++k) {
          const double z = w[k] - vi[i * DT + k];
          sq += z * z;
        }
        acc4[0] += exp_nonpos(ai[i] - 0.5 * sq);
      }
      partial[p * JLmax + jl] = (acc4[0] + acc4[1]) + (acc4[2] + acc4[3]);
    }
    if (t < T) {
      double* vdst = vbuf + (size_t)((t + 1) & 1) * nV;
      double* xdst = xbuf + (size_t)((t + 1) & 1) * JLmax * DT;
      int k = 0;
      for (int q = threadIdx.x; q < nV + nX && k < 2; q += blockDim.x, ++k) {
        if (q < nV) vdst[q] = pf[k];
        else xdst[q - nV] = pf[k];
      }
      for (int q = threadIdx.x + 2 * (int)blockDim.x; q < nV + nX; q += blockDim.x) {  // rest
        if (q < nV) vdst[q] = Vc[(size_t)t * nV + q];
        else xdst[q - nV] = Xc[((size_t)t * N + j0) * DT + (q - nV)];
      }
    }
    __syncthreads();
    pst(t, 2);
    double al = -INFINITY;
    for (int jl = threadIdx.x; jl < JL; jl += blockDim.x) {
      double q[kPitParts];  // canonical pairwise tree over the 32 parts
#pragma unroll
      for (int p = 0; p < kPitParts; ++p) q[p] = partial[p * JLmax + jl];
#pragma unroll
      for (int w = kPitParts / 2; w >= 1; w >>= 1)
#pragma unroll
        for (int p = 0; p < w; ++p) q[p] = q[2 * p] + q[2 * p + 1];
      double s = q[0];
      double m = 0.0;
      if (!(s > 0.0)) {  // total underflow: exact online log-sum-exp relative to M
        const double* w = wj + jl * DT;
        m = -INFINITY;
        s = 0.0;
        for (int i2 = 0; i2 < N; ++i2) {
          double sq = 0.0;
#pragma unroll
          for (int k = 0; k < DT; ++k) {
            const double z = w[k] - vi[i2 * DT + k];
            sq += z * z;
          }
          const double v = ai[i2] - 0.5 * sq;
          if (v > m) {
            s = s * exp(m - v) + 1.0;
            m = v;
          } else {
            s += exp(v - m);
          }
        }
      }
      const int j = j0 + jl;
      al = LW[(size_t)t * N + j] + (am + ((M + m) + log(s)));
      A[(size_t)t * N + j] = al;
      for (int r = 0; r < CS; ++r)  // push into every CTA's alpha_t buffer
        cluster.map_shared_rank(alpha, r)[(size_t)(t & 1) * N + j] = al;
    }
    if (CS > 1 && JLmax <= 32 && threadIdx.x < 32) {  // push this slice's maximum
      double v = (int)threadIdx.x < JL ? al : -INFINITY;
      for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
      if (threadIdx.x < CS) cluster.map_shared_rank(smaxs, threadIdx.x)[(t & 1) * CS + rank] = v;
    }
    pst(t, 3);
    if (CS > 1) cluster.sync();  // alpha_t complete everywhere; step t-1 buffers free
    else __syncthreads();
    pst(t, 4);
  }
  if (CS > 1) cluster.sync();  // no CTA leaves while peers may still write its buffers
#if AUXMC_PIT_EXP == 9
  if (blockIdx.x == 0 && threadIdx.x < 128) reinterpret_cast<long long*>(a.Wt)[threadIdx.x] = pts[threadIdx.x];
#endif
}

// Backward draws for few chains, precomputed in parallel: the uniform of every step is
// known in advance (root.derive(kBackwardIndex, t)), so for every step t and every
// possible chosen particle j at t+1 the drawn index sel(t, j) is a pure function of the
// forward messages — exactly the reference's per-step normalize + sequential cumulative
// draw (fkpg.cpp:19-37, 137-149), evaluated for all N rows of every step at once across
// the GPU (CTA per (chain, t), thread per j; three passes over i: max, sequential sum,
// sequential cumulative search).  The sequential chain is then an index chase through
// the [T][N] table (k_pit_backward_chase).  -1 marks a degenerate row.
// The backward index draws of every step at once (fkpg.cpp:112-152's backward pass,
// tabulated): for step t and each particle j at t+1, the ancestor index the uniform
// u_t selects from the normalized backward weights alpha_t(i) p(x_{t+1}^j | x_t^i).
// The transition density comes from the forward pass's whitened operands (V: means,
// X: particles, k_pit_whiten), so each weight is alpha_t(i) - |X_j - V_i|^2 / 2 (the
// Gaussian's constant cancels in the normalization); one online max/sum pass, then
// the cumulative pass to the first u <= acc.
template <int DT>
__global__ void k_pit_backward_table(DevTarget tg, PgArgs a, const double* __restrict__ V,
                                     const double* __restrict__ X, int* seltab) {
  extern __shared__ double sm[];
  const int N = a.N, T = tg.T;
  const int c = (int)(blockIdx.x / T), t = (int)(blockIdx.x % T);
  if (a.status[c] != AUXMC_OK) return;
  double* vs = sm;                          // N*DT whitened means of x_t^i
  double* At = vs + (size_t)N * DT;         // N
  const double* A = a.Wt + (size_t)c * (T + 1) * N;
  const double* Vt = V + ((size_t)c * T + t) * N * DT;   // step t+1's operands
  const double* Xt = X + ((size_t)c * T + t) * N * DT;
  for (int q = threadIdx.x; q < N * DT; q += blockDim.x) vs[q] = Vt[q];
  for (int i = threadIdx.x; i < N; i += blockDim.x) At[i] = A[(size_t)t * N + i];
  __syncthreads();
  const double u = uniform_at(derive(a.it[c], kBackwardIndex, (uint64_t)t), 0);
  for (int j = threadIdx.x; j < N; j += blockDim.x) {
    double w[DT];
#pragma unroll
    for (int k = 0; k < DT; ++k) w[k] = Xt[(size_t)j * DT + k];
    auto logb = [&](int i) {
      double sq = 0.0;
#pragma unroll
      for (int k = 0; k < DT; ++k) {
        const double z = w[k] - vs[i * DT + k];
        sq += z * z;
      }
      return At[i] - 0.5 * sq;
    };
    double m = -INFINITY, sum = 0.0;
    for (int i = 0; i < N; ++i) {
      const double v = logb(i);
      if (v > m) {
        sum = sum * exp(m - v) + 1.0;
        m = v;
      } else {
        sum += exp(v - m);
      }
    }
    int sel = -1;
    if (isfinite(m)) {
      double acc = 0.0;
      sel = N - 1;
      for (int i = 0; i < N; ++i) {
        acc += exp(logb(i) - m) / sum;
        if (u <= acc) {
          sel = i;
          break;
        }
      }
    }
    seltab[((size_t)c * T + t) * N + j] = sel;
  }
}

// The index chase: i_T from alpha_T (normalize + cumulative draw), then
// i_t = sel(t, i_{t+1}) down to t = 0, table rows staged through shared memory in
// blocks of steps.  Writes the new path, its keys and the optional selection trace.
__global__ void k_pit_backward_chase(DevTarget tg, PgArgs a, const int* seltab) {
  extern __shared__ double sm[];
  const int N = a.N, T = tg.T, d = tg.dx;
  const int c = blockIdx.x;
  if (a.status[c] != AUXMC_OK) return;
  double* alpha = sm;
  double* W = alpha + N;
  double* cum = W + N;
  double* red = cum + N;  // 40
  int* rows = reinterpret_cast<int*>(red + 40);
  int* selp = rows + (size_t)kChaseBlock * N;
  int* blk = selp + 1;  // the block's chased indices
  const double* P = a.part + (size_t)c * (T + 1) * N * d;
  const double* A = a.Wt + (size_t)c * (T + 1) * N;
  double* tr = a.traj + (size_t)c * (T + 1) * d;
  uint64_t* tk = a.tkeys + (size_t)c * (T + 1);
  const uint64_t it = a.it[c];
  auto pm_key = [&](int t, int i) -> uint64_t {
    if (i == 0) return a.keys[(size_t)c * (T + 1) + t];
    return key_at(derive(derive(it, kStep, (uint64_t)t), kPmKey, (uint64_t)i), 0);
  };
  auto take = [&](int t, int sel) {
    for (int k = 0; k < d; ++k) tr[(size_t)t * d + k] = P[((size_t)t * N + sel) * d + k];
    tk[t] = pm_key(t, sel);
    if (a.sel) a.sel[(size_t)c * (T + 1) + t] = sel;
  };
  for (int i = threadIdx.x; i < N; i += blockDim.x) alpha[i] = A[(size_t)T * N + i];
  __syncthreads();
  if (!block_normalize(N, alpha, W, red)) {
    if (threadIdx.x == 0) { a.status[c] = AUXMC_E_DEGENERATE; a.bad_t[c] = T; }
    return;
  }
  block_cumsum(N, W, cum);
  if (threadIdx.x == 0) {
    const int sel = draw_index(N, cum, uniform_at(derive(it, kTerminalIndex, 0), 0));
    *selp = sel;
    take(T, sel);
  }
  __syncthreads();
  const int* tab = seltab + (size_t)c * T * N;
  for (int hi = T; hi > 0; hi -= kChaseBlock) {  // steps [lo, hi)
    const int lo = hi > kChaseBlock ? hi - kChaseBlock : 0;
    for (int q = threadIdx.x; q < (hi - lo) * N; q += blockDim.x) rows[q] = tab[(size_t)lo * N + q];
    __syncthreads();
    if (threadIdx.x == 0) {  // the chase alone; the path writes follow in parallel
      int sel = *selp;
      for (int t = hi - 1; t >= lo; --t) {
        sel = rows[(t - lo) * N + sel];
        blk[t - lo] = sel;
        if (sel < 0) {
          a.status[c] = AUXMC_E_DEGENERATE;
          a.bad_t[c] = t;
          break;
        }
      }
      *selp = sel;
    }
    __syncthreads();
    const bool bad = *selp < 0;
    for (int t = lo + (int)threadIdx.x; t < hi; t += blockDim.x)
      if (!bad) take(t, blk[t - lo]);
    __syncthreads();
    if (bad) return;
  }
}

// Backward index sampling from the stored forward messages (rank 0 of the forward
// cluster's chain, one CTA per chain): i_T ∝ exp(alpha_T), i_t ∝ exp(alpha_t(i))
// p(x_{t+1}^{i_{t+1}} | x_t^i), with the reference's index uniforms.
__global__ void k_pit_backward(DevTarget tg, FactorRef f, PgArgs a) {
  extern __shared__ double sm[];
  const int N = a.N, T = tg.T, d = tg.dx;
  const int c = blockIdx.x;
  if (a.status[c] != AUXMC_OK) return;  // degenerate forward pass
  double* alpha = sm;
  double* W = alpha + N;
  double* cum = W + N;
  double* red = cum + N;       // 40
  double* chosen = red + 40;   // 64
  const double* P = a.part + (size_t)c * (T + 1) * N * d;
  const double* A = a.Wt + (size_t)c * (T + 1) * N;
  double r[64];
  double* tr = a.traj + (size_t)c * (T + 1) * d;
  uint64_t* tk = a.tkeys + (size_t)c * (T + 1);
  const uint64_t it = a.it[c];
  auto pm_key = [&](int t, int i) -> uint64_t {
    if (i == 0) return a.keys[(size_t)c * (T + 1) + t];
    return key_at(derive(derive(it, kStep, (uint64_t)t), kPmKey, (uint64_t)i), 0);
  };
  for (int i = threadIdx.x; i < N; i += blockDim.x) alpha[i] = A[(size_t)T * N + i];
  __syncthreads();
  if (!block_normalize(N, alpha, W, red)) {
    if (threadIdx.x == 0) { a.status[c] = AUXMC_E_DEGENERATE; a.bad_t[c] = T; }
    return;
  }
  block_cumsum(N, W, cum);
  if (threadIdx.x == 0) {
    const int sel = draw_index(N, cum, uniform_at(derive(it, kTerminalIndex, 0), 0));
    for (int k = 0; k < d; ++k) chosen[k] = tr[(size_t)T * d + k] = P[((size_t)T * N + sel) * d + k];
    tk[T] = pm_key(T, sel);
    if (a.sel) a.sel[(size_t)c * (T + 1) + T] = sel;
  }
  __syncthreads();
  for (int t = T - 1; t >= 0; --t) {
    const int jq = 1 + (f.fl.nQ > 1 ? t : 0);
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
      const double* xi = P + ((size_t)t * N + i) * d;
      for (int k = 0; k < d; ++k) r[k] = chosen[k] - dyn_mean_i(tg, t, xi, k);
      alpha[i] = A[(size_t)t * N + i] + gauss_term(d, r, f.L(jq), f.logdet[jq]);
    }
    __syncthreads();
    if (!block_normalize(N, alpha, W, red)) {
      if (threadIdx.x == 0) { a.status[c] = AUXMC_E_DEGENERATE; a.bad_t[c] = t; }
      return;
    }
    block_cumsum(N, W, cum);
    if (threadIdx.x == 0) {
      const int sel = draw_index(N, cum, uniform_at(derive(it, kBackwardIndex, (uint64_t)t), 0));
      for (int k = 0; k < d; ++k) chosen[k] = tr[(size_t)t * d + k] = P[((size_t)t * N + sel) * d + k];
      tk[t] = pm_key(t, sel);
      if (a.sel) a.sel[(size_t)c * (T + 1) + t] = sel;
    }
    __syncthreads();
  }
}

// Forward log-messages alpha_t(j) = lw_t(j) + LSE_i(alpha_{t-1}(i) + log p(x_t^j | x_{t-1}^i)),
// one CTA per chain, then backward index sampling with the reference's addresses.
__global__ void k_pit_forward_backward(DevTarget tg, FactorRef f, PgArgs a, const double* lw) {
  extern __shared__ double sm[];
  const int N = a.N, T = tg.T, d = tg.dx;
  const int c = blockIdx.x;
  double* alpha = sm;            // N
  double* W = alpha + N;         // N
  double* cum = W + N;           // N
  double* mprev = cum + N;       // N*d dynamics means of the previous particles
  double* red = mprev + (size_t)N * d;  // 40
  double* chosen = red + 40;     // d (<= 64)
  double* partial = chosen + 64; // (blockDim / N) * N partial sums
  const double* P = a.part + (size_t)c * (T + 1) * N * d;
  const double* LW = lw + (size_t)c * (T + 1) * N;
  double* A = a.Wt + (size_t)c * (T + 1) * N;
  const int jq0 = 1;
  double r[64];
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    alpha[i] = LW[i];
    A[i] = alpha[i];
  }
  __syncthreads();
  for (int t = 1; t <= T; ++t) {
    for (int q = threadIdx.x; q < N * d; q += blockDim.x) {
      const int i = q / d, k = q % d;
      mprev[q] = dyn_mean_i(tg, t - 1, P + ((size_t)(t - 1) * N + i) * d, k);
    }
    const double am = block_max([&] {
      double m = -INFINITY;
      for (int i = threadIdx.x; i < N; i += blockDim.x) m = fmax(m, alpha[i]);
      return m;
    }(), red);
    if (!isfinite(am)) {  // every message at t-1 collapsed: DegenerateWeightsError naming t-1
      if (threadIdx.x == 0) {  // (fkpg.cpp:19-23: the reference's sweep fails at that step)
        a.status[c] = AUXMC_E_DEGENERATE;
        a.bad_t[c] = t - 1;
      }
      return;
    }
    const int jq = jq0 + (f.fl.nQ > 1 ? t - 1 : 0);
    const double* LQ = f.L(jq);
    const double ldq = f.logdet[jq];
    for (int j = threadIdx.x; j < N; j += blockDim.x) {
      const double* xj = P + ((size_t)t * N + j) * d;
      double m = -INFINITY, s = 0.0;  // online log-sum-exp over i
      for (int i = 0; i < N; ++i) {
        for (int k = 0; k < d; ++k) r[k] = xj[k] - mprev[i * d + k];
        const double v = (alpha[i] - am) + gauss_term(d, r, LQ, ldq);
        if (v > m) {
          s = s * exp(m - v) + 1.0;
          m = v;
        } else {
          s += exp(v - m);
        }
      }
      W[j] = LW[(size_t)t * N + j] + (am + (m + log(s)));
    }
    __syncthreads();
    for (int j = threadIdx.x; j < N; j += blockDim.x) {
      alpha[j] = W[j];
      A[(size_t)t * N + j] = W[j];
    }
    __syncthreads();
  }
  // backward: i_T ∝ exp(alpha_T); i_t ∝ exp(alpha_t(i)) p(x_{t+1}^{i_{t+1}} | x_t^i)
  double* tr = a.traj + (size_t)c * (T + 1) * d;
  uint64_t* tk = a.tkeys + (size_t)c * (T + 1);
  const uint64_t it = a.it[c];
  auto pm_key = [&](int t, int i) -> uint64_t {
    if (i == 0) return a.keys[(size_t)c * (T + 1) + t];
    return key_at(derive(derive(it, kStep, (uint64_t)t), kPmKey, (uint64_t)i), 0);
  };
  if (!block_normalize(N, alpha, W, red)) {
    if (threadIdx.x == 0) { a.status[c] = AUXMC_E_DEGENERATE; a.bad_t[c] = T; }
    return;
  }
  block_cumsum(N, W, cum);
  if (threadIdx.x == 0) {
    const int sel = draw_index(N, cum, uniform_at(derive(it, kTerminalIndex, 0), 0));
    for (int k = 0; k < d; ++k) chosen[k] = tr[(size_t)T * d + k] = P[((size_t)T * N + sel) * d + k];
    tk[T] = pm_key(T, sel);
    if (a.sel) a.sel[(size_t)c * (T + 1) + T] = sel;
  }
  __syncthreads();
  for (int t = T - 1; t >= 0; --t) {
    const int jq = jq0 + (f.fl.nQ > 1 ? t : 0);
    for (int i = threadIdx.x; i < N; i += blockDim.x) {
      const double* xi = P + ((size_t)t * N + i) * d;
      for (int k = 0; k < d; ++k) r[k] = chosen[k] - dyn_mean_i(tg, t, xi, k);
      alpha[i] = A[(size_t)t * N + i] + gauss_term(d, r, f.L(jq), f.logdet[jq]);
    }
    __syncthreads();
    if (!block_normalize(N, alpha, W, red)) {
      if (threadIdx.x == 0) { a.status[c] = AUXMC_E_DEGENERATE; a.bad_t[c] = t; }
      return;
    }
    block_cumsum(N, W, cum);
    if (threadIdx.x == 0) {
      const int sel = draw_index(N, cum, uniform_at(derive(it, kBackwardIndex, (uint64_t)t), 0));
      for (int k = 0; k < d; ++k) chosen[k] = tr[(size_t)t * d + k] = P[((size_t)t * N + sel) * d + k];
      tk[t] = pm_key(t, sel);
      if (a.sel) a.sel[(size_t)c * (T + 1) + t] = sel;
    }
    __syncthreads();
  }
}

// adopt the new path (fkpg.cpp:269-273)
__global__ void k_pg_commit(int C, int T, int d, const double* traj, const uint64_t* tkeys,
                            const int* status, double* x, uint64_t* keys, long long* iter,
                            long long* updates, double* last_update) {
  const int c = blockIdx.x;
  __shared__ int changed;
  if (threadIdx.x == 0) changed = 0;
  __syncthreads();
  const size_t n = (size_t)(T + 1) * d;
  const bool ok = status[c] == AUXMC_OK;
  if (ok)
    for (size_t q = threadIdx.x; q < n; q += blockDim.x)
      if (__double_as_longlong(traj[c * n + q]) != __double_as_longlong(x[c * n + q])) changed = 1;
  __syncthreads();
  if (ok) {
    for (size_t q = threadIdx.x; q < n; q += blockDim.x) x[c * n + q] = traj[c * n + q];
    for (int t = threadIdx.x; t <= T; t += blockDim.x)
      keys[(size_t)c * (T + 1) + t] = tkeys[(size_t)c * (T + 1) + t];
  }
  if (threadIdx.x == 0) {
    iter[c] += 1;
    if (ok) {
      last_update[c] = changed ? 1.0 : 0.0;
      if (changed) updates[c] += 1;
    }
  }
}

__global__ void k_pg_adapt(int C, const long long* iter, const double* last_update, double target,
                           double* delta) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  const double n = (double)(iter[c] > 1 ? iter[c] : 1);
  delta[c] = exp(log(delta[c]) + pow(n, -0.6) * (last_update[c] - target));
}

#ifndef AUXMC_PIT_CS
#define AUXMC_PIT_CS 16  // CTAs per chain in the few-chain forward (16: non-portable cluster)
#endif
static int pit_cluster(int C) {
  return (AUXMC_PIT_CS > 8 && C * AUXMC_PIT_CS <= num_sms()) ? AUXMC_PIT_CS : 8;
}

template <int DT>
static int launch_pit_forward_dt(int C, int CS, int threads, size_t smem, cudaStream_t s,
                                 const DevTarget& tg, const FactorRef& f, const PgArgs& a,
                                 const double* lw, double* V, double* X) {
  const long long n = (long long)C * tg.T * a.N;
  if (n > 0)
    AUXMC_LAUNCH(k_pit_whiten<DT>, (int)std::min<long long>((n + 255) / 256, 148LL * 64), 256, 0, s,
                 tg, f, a, V, X);
  auto kern = k_pit_forward_cluster<DT>;
  AUXMC_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if (CS > 8)
    AUXMC_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C * CS);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const bool prof = g_prof_on.load(std::memory_order_relaxed);
  if (prof) prof_mark("k_pit_forward_cluster", s, true);
  AUXMC_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, tg, f, a, lw, (const double*)V, (const double*)X, CS));
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (prof) prof_mark("k_pit_forward_cluster", s, false);
  return AUXMC_OK;
}

static int launch_pit_forward(int d, int C, int CS, int threads, size_t smem, cudaStream_t s,
                              const DevTarget& tg, const FactorRef& f, const PgArgs& a,
                              const double* lw, double* V, double* X) {
  switch (d) {
#define PCASE(DT) \
  case DT: return launch_pit_forward_dt<DT>(C, CS, threads, smem, s, tg, f, a, lw, V, X);
    PCASE(1) PCASE(2) PCASE(3) PCASE(4) PCASE(5) PCASE(6) PCASE(7) PCASE(8)
#undef PCASE
  }
  return AUXMC_E_DIM;
}

static int pg_step(const DevTarget& tg, auxmc_pg_chains* ch, int mode, int variant, Arena& ws,
                   cudaStream_t s) {
  const int C = ch->C, N = ch->N, T = tg.T, d = tg.dx;
  const FactorLayout fl = factor_layout(tg);
  uint64_t* it = ws.take<uint64_t>(C);
  double* u = ws.take<double>((size_t)C * (T + 1) * d);
  double* mq = ws.take<double>((size_t)C * (T + 1) * d);
  double* part = ws.take<double>((size_t)C * (T + 1) * N * d);
  double* Wt = ws.take<double>((size_t)C * (T + 1) * N);
  double* lw = variant == AUXMC_CSMC_PIT ? ws.take<double>((size_t)C * (T + 1) * N) : nullptr;
  // few-chain PIT: cluster forward + precomputed backward draws (k_pit_backward_table)
  const bool pit_few = variant == AUXMC_CSMC_PIT && d <= 8 && N >= 64 && C * 8 <= num_sms();
  int* seltab = pit_few && T > 0 ? ws.take<int>((size_t)C * T * N) : nullptr;
  const bool pit_small = variant == AUXMC_CSMC_PIT && d <= 8;
  double* pV = pit_small ? ws.take<double>((size_t)C * T * N * d + 1) : nullptr;
  double* pX = pit_small ? ws.take<double>((size_t)C * T * N * d + 1) : nullptr;
  double* traj = ws.take<double>((size_t)C * (T + 1) * d);
  uint64_t* tkeys = ws.take<uint64_t>((size_t)C * (T + 1));
  double* Ls = ws.take<double>((size_t)fl.total() * fl.W * fl.W);
  double* logdet = ws.take<double>(fl.total());
  int* ints = ws.take<int>((size_t)C + 1);
  const int nad = 1 + fl.nQ;  // proposal classes: P0, then each Q_j
  double* adf = mode == AUXMC_PG_ADAPTED ? ws.take<double>((size_t)C * nad * (2 * d * d + 1))
                                         : nullptr;
  int* ad_bad = mode == AUXMC_PG_ADAPTED ? ws.take<int>((size_t)C) : nullptr;
  if (ws.base == nullptr) return AUXMC_OK;
  if (mode == AUXMC_PG_ADAPTED && (!adf || !ad_bad)) return AUXMC_E_WORKSPACE;
  if (!it || !u || !mq || !part || !Wt || !traj || !tkeys || !Ls || !logdet || !ints ||
      (variant == AUXMC_CSMC_PIT && !lw))
    return AUXMC_E_WORKSPACE;
  if ((pit_few && T > 0 && !seltab) || (pit_small && (!pV || !pX))) return AUXMC_E_WORKSPACE;
  AUXMC_CUDA_TRY(cudaMemsetAsync(ch->status, 0, sizeof(int) * C, s));
  AUXMC_CUDA_TRY(cudaMemsetAsync(ch->bad_t, 0xff, sizeof(int) * C, s));
  AUXMC_CUDA_TRY(cudaMemsetAsync(ints, 0, sizeof(int) * (C + 1), s));
  int rc = launch_target_factors(tg, Ls, logdet, ints + C, s);
  if (rc) return rc;
  FactorRef f{fl, Ls, logdet};
  AUXMC_LAUNCH(k_pg_keys, (C + 127) / 128, 128, 0, s, C, ch->root_keys, ch->iter, it);
  rc = launch_aux_obs(C, T, d, ch->x, ch->delta, it, u, s);
  if (rc) return rc;
  const long long nct = (long long)C * (T + 1);
  AUXMC_LAUNCH(k_pg_prop_mean, (int)std::min<long long>((nct + 127) / 128, 148LL * 32), 128, 0, s,
               tg, f, C, u, ch->delta, mq, ints);
  if (mode == AUXMC_PG_ADAPTED) {
    AUXMC_CUDA_TRY(cudaMemsetAsync(ad_bad, 0, sizeof(int) * C, s));
    const size_t per = sizeof(double) * (6 * d * d + 4);
    const int warps = (int)std::max<size_t>(1, std::min<size_t>(4, (200u << 10) / per));
    AUXMC_CUDA_TRY(cudaFuncSetAttribute(k_pg_adapted, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)(per * warps)));
    AUXMC_LAUNCH(k_pg_adapted, (C * nad + warps - 1) / warps, 32 * warps, per * warps, s, tg, C, nad,
                 ch->delta, adf, ad_bad);
  }
  PgArgs a{C, N, ch->x, ch->keys, ch->delta, it, u, mq, part, Wt, traj, tkeys, ch->status,
           ch->bad_t, ch->ancestors, ch->selected, ints, mode, adf, nad, ad_bad, ch->pm_kind};
  const int threads = N >= 256 ? 256 : ((N + 31) / 32) * 32;
  if (variant == AUXMC_CSMC_REFERENCE) {
    const size_t smem = sizeof(double) * (3 * N + 40 + 64) + sizeof(int) * (N + 1);
    AUXMC_CUDA_TRY(cudaFuncSetAttribute(k_csmc_reference,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    AUXMC_LAUNCH(k_csmc_reference, C, threads, smem, s, tg, f, a);
  } else {
    const long long np = nct * N;
    AUXMC_LAUNCH(k_pit_particles, (int)std::min<long long>((np + 255) / 256, 148LL * 64), 256, 0, s,
                 tg, f, a, lw);
    if (d <= 8) {
      // cluster-parallel forward messages: 8 SMs per chain when the batch leaves SMs idle
      const int CS = pit_few ? pit_cluster(C) : 1;
      const int JLmax = (N + CS - 1) / CS;
#ifndef AUXMC_PIT_FT16
#define AUXMC_PIT_FT16 512
#endif
      // threads per CTA: the pair items are JL x 32 parts (512 at CS = 16, N = 256)
      const int fthreads = CS >= 16 ? AUXMC_PIT_FT16 : 1024;
      const size_t fsmem = sizeof(double) * (2 * (size_t)N + 2 * (size_t)N * d + 2 * (size_t)JLmax * d +
                                             N + kPitParts * JLmax + 2 * CS + 40);
      int rc2 = launch_pit_forward(d, C, CS, fthreads, fsmem, s, tg, f, a, lw, pV, pX);
      if (rc2) return rc2;
      if (pit_few && T > 0) {
        const size_t tsmem = sizeof(double) * ((size_t)N * d + N);
        switch (d) {
#define TCASE(DT)                                                                            \
  case DT:                                                                                   \
    AUXMC_LAUNCH(k_pit_backward_table<DT>, C * T, threads, tsmem, s, tg, a, pV, pX, seltab); \
    break;
          TCASE(1) TCASE(2) TCASE(3) TCASE(4) TCASE(5) TCASE(6) TCASE(7) TCASE(8)
#undef TCASE
        }
        const size_t csmem = sizeof(double) * (3 * (size_t)N + 40) +
                             sizeof(int) * ((size_t)kChaseBlock * (N + 1) + 1);
        AUXMC_CUDA_TRY(cudaFuncSetAttribute(k_pit_backward_chase,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csmem));
        AUXMC_LAUNCH(k_pit_backward_chase, C, threads, csmem, s, tg, a, seltab);
      } else {
        const size_t bsmem = sizeof(double) * (3 * (size_t)N + 40 + 64);
        AUXMC_CUDA_TRY(cudaFuncSetAttribute(k_pit_backward, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)bsmem));
        AUXMC_LAUNCH(k_pit_backward, C, threads, bsmem, s, tg, f, a);
      }
    } else {
      const size_t smem = sizeof(double) * (3 * N + (size_t)N * d + 40 + 64 + (size_t)N);
      AUXMC_CUDA_TRY(cudaFuncSetAttribute(k_pit_forward_backward,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      AUXMC_LAUNCH((k_pit_forward_backward), C, threads, smem, s, tg, f, a, lw);
    }
  }
  AUXMC_LAUNCH(k_pg_commit, C, 256, 0, s, C, T, d, traj, tkeys, ch->status, ch->x, ch->keys,
               ch->iter, ch->updates, ch->last_update);
  return AUXMC_OK;
}

}  // namespace auxmc_gpu

using namespace auxmc_gpu;

extern "C" {

size_t auxmc_aux_pgibbs_workspace(const auxmc_target* target, int C, int N, int variant) {
  if (check_target(target) || C < 0 || N < 1) return 0;
  Arena ws{nullptr, 0, 0};
  auxmc_pg_chains ch{};
  ch.C = C;
  ch.N = N;
  pg_step(to_dev_target(*target), &ch, AUXMC_PG_ADAPTED, variant, ws, nullptr);  // largest mode
  return ws.used + 4096;
}

int auxmc_aux_pgibbs_step(const auxmc_target* target, auxmc_pg_chains* chains, int mode,
                          int variant, void* workspace, size_t workspace_bytes, void* stream) {
  if (!device_ok()) return AUXMC_E_CUDA;
  int st = check_target(target);
  if (st) return st;
  if (mode < AUXMC_PG_PRIOR || mode > AUXMC_PG_ADAPTED) return AUXMC_E_ARG;
  if (variant != AUXMC_CSMC_REFERENCE && variant != AUXMC_CSMC_PIT) return AUXMC_E_ARG;
  // the PIT lattice needs parent-free (independent) proposals: gradient mode only
  if (variant == AUXMC_CSMC_PIT && mode != AUXMC_PG_GRADIENT) return AUXMC_E_ARG;
  if (chains && (chains->pm_kind < AUXMC_PM_NONE || chains->pm_kind > AUXMC_PM_NEGATIVE ||
                 (chains->pm_kind != AUXMC_PM_NONE && variant != AUXMC_CSMC_REFERENCE)))
    return AUXMC_E_ARG;
  if (!chains || chains->C < 0 || chains->N < 1 || chains->N > 4096 || !chains->x ||
      !chains->keys || !chains->delta || !chains->iter || !chains->updates ||
      !chains->last_update || !chains->root_keys || !chains->status || !chains->bad_t)
    return AUXMC_E_ARG;
  if (chains->C == 0) return AUXMC_OK;
  if (!workspace) return AUXMC_E_WORKSPACE;
  Arena ws{(char*)workspace, workspace_bytes, 0};
  return pg_step(to_dev_target(*target), chains, mode, variant, ws, (cudaStream_t)stream);
}

int auxmc_pg_adapt_delta(auxmc_pg_chains* chains, double target_rate, void* stream) {
  if (!device_ok()) return AUXMC_E_CUDA;
  if (!chains || !chains->delta || !chains->iter || !chains->last_update) return AUXMC_E_ARG;
  if (chains->C == 0) return AUXMC_OK;
  AUXMC_LAUNCH(k_pg_adapt, (chains->C + 127) / 128, 128, 0, stream, chains->C, chains->iter,
               chains->last_update, target_rate, chains->delta);
  return AUXMC_OK;
}

}  // extern "C"
