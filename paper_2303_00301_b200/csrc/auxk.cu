// auxk.cu — auxiliary Kalman MH kernel (auxk.cpp:45-218) and the target density
// (target.cpp:47-108) for batches of chains on B200.
//
// One kernel_step for C chains is a fixed sequence of batched launches:
//   aux draws u (auxk.cpp:45-54)
//   surrogate LGSSM at x (auxk.cpp:56-118): per-chain pseudo-observations z,
//     linearized dynamics for tractable targets, per-chain R = diag(δ/2 I, R_e, I)
//   Kalman filter -> pathwise proposal (seq / prefix / dnc backend)
//   log q(x'|x) = path_logpdf(cur, x'), log γ(x'), ∇ log g(x')
//   surrogate at x', reverse filter, log q(x|x')
//   aux log-likelihoods, log α, accept with U(kMhAccept, 0) (auxk.cpp:173-193)
// Chains never branch the launch sequence: failures (factorization, non-finite
// γ or gradients, NaN log α) are per-chain status words resolved in the MH
// kernel exactly in the reference's order (auxk.cpp:151-197).  Model closures
// (target.hpp:25-38) are compiled device functors selected by target kind.
#include <cmath>

#include "common.cuh"
#include "dense.cuh"
#include "rng.cuh"
#include "target.cuh"
#include "terms.cuh"

namespace auxmc_gpu {

int launch_filter_pit(const DevModel& dm, const double* obs, int B, auxmc_filter_result* out,
                      int* status, Arena& ws, cudaStream_t stream);
int launch_filter_seq(const DevModel& dm, const double* obs, int B, auxmc_filter_result* out,
                      int* status, cudaStream_t stream);
int launch_sample_paths(const DevModel& dm, const auxmc_filter_result* fr, int fr_shared,
                        const auxmc_noise* noise, int B, int sampler, double* traj, int* status,
                        Arena& ws, cudaStream_t stream);
int launch_path_logpdf(const DevModel& dm, const double* obs, long long obs_stride,
                       const double* traj, const double* log_marginal, int lm_shared, int B,
                       double* out, int* status, cudaStream_t s);
bool filter_direct_ok(const DevTarget& tg, const DevModel& dm, bool stencil);
int launch_filter_direct(const DevTarget& tg, const DevModel& dm, bool stencil,
                         const double* xl, const double* delta, const double* z, int C,
                         auxmc_filter_result* fr, int* status, int covs, cudaStream_t s);

// auxmc_test_force_generic_filter: route the sequential aux filter through the generic
// (d+q)-dimensional filter (k_filter_cta / k_filter_seq) even when the fused
// direct-observation filter applies — the parity tests compare the two.
static int g_force_generic_filter = 0;
// auxmc_test_capture_log_marginal: device buffer [C] receiving the forward filter's
// log p(z) of every aux step (nullptr: off) — the parity tests compare filters directly.
static double* g_capture_lm = nullptr;

// dgf (nullable): per factor, 1 when it is diagonal to the bit (gauss_term's dense
// solve then reduces to its diagonal terms, gamma_term_k)
__global__ void k_target_factors(DevTarget tg, FactorLayout fl, double* Ls, double* logdet,
                                 int* status, unsigned char* dgf = nullptr) {
  extern __shared__ double smem[];
  const int W = fl.W;
  Grp g = warp_group();
  const int gid = threadIdx.x >> 5, gpb = blockDim.x >> 5;
  double* A = smem + (size_t)gid * (3 * W * W + 4);
  double* L = A + W * W;
  double* scr = L + W * W;
  double* red = scr + W * W;
  int* flag = reinterpret_cast<int*>(red + 2);
  for (int j = blockIdx.x * gpb + gid; j < fl.total(); j += gridDim.x * gpb) {
    const double* src;
    int n;
    if (j == 0) { src = tg.P0; n = tg.dx; }
    else if (j <= fl.nQ) { src = tg.Q + (size_t)(j - 1) * tg.dx * tg.dx; n = tg.dx; }
    else if (j <= fl.nQ + fl.nE) { src = tg.eR + (size_t)(j - 1 - fl.nQ) * tg.q * tg.q; n = tg.q; }
    else { src = tg.gR + (size_t)(j - 1 - fl.nQ - fl.nE) * tg.ydim * tg.ydim; n = tg.ydim; }
    for (int i = g.lane; i < n * n; i += g.size) {
      const int r = i / n, c = i % n;
      A[i] = (src[r * n + c] + src[c * n + r]) * 0.5;  // Gaussian ctor symmetrization
    }
    g.sync();
    const int st = g_factor_psd(g, n, A, L, scr, flag, red);
    double* out = Ls + (size_t)j * W * W;
    bool offz = true;
    for (int i = g.lane; i < n * n; i += g.size) {
      out[i] = L[i];
      if (i / n != i % n && L[i] != 0.0) offz = false;
    }
    offz = __all_sync(0xffffffffu, offz);
    if (dgf && g.lane == 0) dgf[j] = offz ? 1 : 0;
    if (g.lane == 0) {
      double ld = 0.0;
      for (int i = 0; i < n; ++i) ld += log(L[i * n + i]);
      logdet[j] = ld;
      if (st) atomicMax(status, st);
    }
    g.sync();
  }
}

// log γ terms (target.cpp:100-108): k = 0 prior, 1..T dynamics, T+1.. potentials
__global__ void k_gamma_terms(DevTarget tg, FactorLayout fl, int C, const double* __restrict__ traj,
                              const double* __restrict__ Ls, const double* __restrict__ logdet,
                              double* terms, const unsigned char* __restrict__ dgf) {
  const int T = tg.T, d = tg.dx;
  const int K = 2 * T + 2;
  const long long n = (long long)C * K;
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(q / K), k = (int)(q % K);
    terms[q] = gamma_term_k(tg, fl, traj + (size_t)c * (T + 1) * d, Ls, logdet, k, dgf);
  }
}

__global__ void k_gamma_sum(int T, int C, const double* terms, const int* fst, double* out,
                            int* status, const double* parts) {
  __shared__ double red[kSumThreads];
  const int c = blockIdx.x;
  const long long K = 2LL * T + 2;
  const double* tm = terms + (size_t)c * K;
  const double lg = cta_sum_fixed(K, [&](long long i) { return tm[i]; }, red,
                                  parts ? parts + (size_t)c * kSumThreads : nullptr);
  if (threadIdx.x == 0) {
    out[c] = lg;
    if (status) status[c] = *fst;
  }
}

__global__ void k_grads(DevTarget tg, FactorLayout fl, int C, const double* __restrict__ traj,
                        const double* __restrict__ Ls, double* grads, int* bad) {
  const int T = tg.T, d = tg.dx;
  const long long n = (long long)C * (T + 1);
  double r[64], g[64];
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(q / (T + 1)), t = (int)(q % (T + 1));
    const int jg = 1 + fl.nQ + fl.nE + (tg.ne > 1 ? t : 0);
    generic_grad(tg, t, traj + (size_t)q * d, fl.nG ? Ls + (size_t)jg * fl.W * fl.W : nullptr, r, g);
    bool ok = true;
    for (int i = 0; i < d; ++i) {
      grads[(size_t)q * d + i] = g[i];
      ok = ok && isfinite(g[i]);
    }
    if (!ok && bad) atomicOr(bad + c, 1);
  }
}

// ---------------------------------------------------------------- aux model
__global__ void k_iter_keys(int C, const uint64_t* root, const long long* iter, uint64_t* it) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < C) it[c] = derive(root[c], kIteration, (uint64_t)iter[c]);
}

// u_t = x_t + sqrt(δ/2) xi(kAuxObs, t) (auxk.cpp:45-54)
__global__ void k_aux_obs(int C, int T, int d, const double* __restrict__ x,
                          const double* __restrict__ delta, const uint64_t* __restrict__ it,
                          double* u) {
  const long long n = (long long)C * (T + 1) * d;
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(q % d);
    const long long ct = q / d;
    const int t = (int)(ct % (T + 1)), c = (int)(ct / (T + 1));
    const double sd = sqrt(delta[c] / 2.0);
    u[q] = x[q] + sd * normal_at(derive(it[c], kAuxObs, (uint64_t)t), (uint64_t)i);
  }
}

// Per-chain pseudo-observations and linearized dynamics (auxk.cpp:60-113)
__global__ void k_build_aux(DevTarget tg, int C, int zeroth, const double* __restrict__ xs,
                            const double* __restrict__ gs, const double* __restrict__ u,
                            const double* __restrict__ delta, double* z, double* Fa, double* ba) {
  const int T = tg.T, d = tg.dx, p = d + tg.q;
  const long long n = (long long)C * (T + 1);
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(q / (T + 1)), t = (int)(q % (T + 1));
    const double h = delta[c] / 2.0;
    double* zt = z + (size_t)q * p;
    for (int i = 0; i < d; ++i) {
      double v = u[(size_t)q * d + i];
      if (!zeroth) v += h * gs[(size_t)q * d + i];
      zt[i] = v;
    }
    for (int k = 0; k < tg.q; ++k) zt[d + k] = tg.emask[t] ? tg.ey[(size_t)t * tg.q + k] : 0.0;
    if (!tg.linear && t < T) {
      const double* xt = xs + (size_t)q * d;
      double* bb = ba + ((size_t)c * T + t) * d;
      if (Fa) {
        double* F = Fa + ((size_t)c * T + t) * d * d;
        for (int i = 0; i < d; ++i)
          for (int j = 0; j < d; ++j) F[i * d + j] = dyn_jac_ij(tg, t, xt, i, j);
        for (int i = 0; i < d; ++i) {
          double s = 0.0;
          for (int j = 0; j < d; ++j) s += F[i * d + j] * xt[j];
          bb[i] = dyn_mean_i(tg, t, xt, i) - s;
        }
      } else {  // Lorenz-96 stencil: F stays implicit; the row's nonzeros in column order
        for (int i = 0; i < d; ++i) {
          int cs[4];
          double vs[4];
          l96_row(xt, d, tg.l96_h, i, cs, vs);
          double s = 0.0;
          for (int a = 0; a < 4; ++a) s += vs[a] * xt[cs[a]];
          bb[i] = dyn_mean_i(tg, t, xt, i) - s;
        }
      }
    }
  }
}

// H = [I; H_e; 0], c = [0; c_e; 0] (shared), R = diag(δ/2 I, R_e, I) per chain
__global__ void k_build_HR(DevTarget tg, int C, int nH, const double* __restrict__ delta,
                           double* H, double* cv, double* R) {
  const int d = tg.dx, q = tg.q, p = d + q;
  const long long nR = (long long)C * nH * p * p;
  for (long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x; idx < nR;
       idx += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(idx % p), i = (int)((idx / p) % p);
    const int tt = (int)((idx / ((long long)p * p)) % nH);
    const int c = (int)(idx / ((long long)p * p * nH));
    const bool ex = q > 0 && tg.emask[tt];
    double v;
    if (i < d || j < d) v = (i == j) ? (i < d ? delta[c] / 2.0 : 1.0) : 0.0;
    else v = ex ? tg.eRt(tt)[(i - d) * q + (j - d)] : (i == j ? 1.0 : 0.0);
    R[idx] = v;
    if (c == 0) {
      if (j < d) {
        double hv;
        if (i < d) hv = (i == j) ? 1.0 : 0.0;
        else hv = ex ? tg.eHt(tt)[(i - d) * d + j] : 0.0;
        H[((size_t)tt * p + i) * d + j] = hv;
      }
      if (j == 0) cv[(size_t)tt * p + i] = (i >= d && ex) ? tg.ect(tt)[i - d] : 0.0;
    }
  }
}

__global__ void k_aux_lik_terms(int C, int T, int d, const double* __restrict__ u,
                                const double* __restrict__ x, const double* __restrict__ delta,
                                double* terms) {
  const long long n = (long long)C * (T + 1);
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(q / (T + 1));
    const double var = delta[c] / 2.0;
    double sq = 0.0;
    for (int i = 0; i < d; ++i) {
      const double r = u[(size_t)q * d + i] - x[(size_t)q * d + i];
      sq += r * r;
    }
    terms[q] = -0.5 * (d * (kLog2Pi + log(var)) + sq / var);  // gauss.cpp:59-62
  }
}

__global__ void k_row_sum(int C, int n, const double* terms, double* out, const double* parts) {
  __shared__ double red[kSumThreads];
  const int c = blockIdx.x;
  const double* tm = terms + (size_t)c * n;
  const double s = cta_sum_fixed(n, [&](long long i) { return tm[i]; }, red,
                                 parts ? parts + (size_t)c * kSumThreads : nullptr);
  if (threadIdx.x == 0) out[c] = s;
}

struct StepScalars {
  double *logq_fwd, *logq_rev, *lg_prop, *aux_prop, *aux_x;
  int *st_filt, *st_samp, *st_lqf, *st_lg, *bad, *st_filt_r, *st_lqr, *accept;
};

// auxk.cpp:130-197 decision logic, per chain
__global__ void k_mh(int C, StepScalars s, const uint64_t* it, double* log_gamma, long long* iter,
                     auxmc_kernel_stats* stats) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  auxmc_kernel_stats st = stats[c];
  iter[c] += 1;
  st.last_accept_prob = 0.0;
  st.last_log_alpha = -INFINITY;
  int acc = 0;
  if (s.st_filt[c] || s.st_samp[c] || s.st_lqf[c] || s.st_lg[c]) {
    ++st.aborted;
    ++st.rejected;
  } else if (!isfinite(s.lg_prop[c])) {
    ++st.nonfinite_gamma;
    ++st.rejected;
  } else if (s.bad[c]) {
    ++st.aborted;
    ++st.rejected;
  } else if (s.st_filt_r[c] || s.st_lqr[c]) {
    ++st.aborted;
    ++st.rejected;
  } else {
    const double la = (s.lg_prop[c] + s.aux_prop[c] + s.logq_rev[c]) -
                      (log_gamma[c] + s.aux_x[c] + s.logq_fwd[c]);
    if (isnan(la)) {
      ++st.aborted;
      ++st.rejected;
    } else {
      st.last_log_alpha = la;
      st.last_accept_prob = la >= 0.0 ? 1.0 : exp(la);
      const double uacc = uniform_at(derive(it[c], kMhAccept, 0), 0);
      if (uacc < st.last_accept_prob) {
        acc = 1;
        log_gamma[c] = s.lg_prop[c];
        ++st.accepted;
      } else {
        ++st.rejected;
      }
    }
  }
  s.accept[c] = acc;
  stats[c] = st;
}

__global__ void k_accept_copy(int C, long long row, const int* accept, const double* prop,
                              const double* gprop, double* x, double* grad) {
  const long long n = (long long)C * row;
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (long long)gridDim.x * blockDim.x) {
    if (accept[q / row]) {
      x[q] = prop[q];
      grad[q] = gprop[q];
    }
  }
}

// δ ← exp(log δ + n^{-0.6} (α̂ - target)), n = max(iter, 1) (auxk.cpp:213-218)
__global__ void k_adapt(int C, const long long* iter, const auxmc_kernel_stats* stats,
                        double target, double* delta) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  const double n = (double)(iter[c] > 1 ? iter[c] : 1);
  delta[c] = exp(log(delta[c]) + pow(n, -0.6) * (stats[c].last_accept_prob - target));
}

static int grid_for(long long n, int block = 256) {
  long long g = (n + block - 1) / block;
  if (g > 148LL * 32) g = 148LL * 32;
  return (int)(g < 1 ? 1 : g);
}

// log γ of C paths into out[C] (+ status); needs factor workspace
static int launch_log_gamma(const DevTarget& tg, int C, const double* traj, double* out,
                            int* status, Arena& ws, cudaStream_t s) {
  const FactorLayout fl = factor_layout(tg);
  double* Ls = ws.take<double>((size_t)fl.total() * fl.W * fl.W);
  double* logdet = ws.take<double>(fl.total());
  double* terms = ws.take<double>((size_t)C * (2 * tg.T + 2));
  int* fst = ws.take<int>(1);
  unsigned char* dgf = ws.take<unsigned char>(fl.total());
  if (ws.base == nullptr) return AUXMC_OK;
  if (!Ls || !logdet || !terms || !fst || !dgf) return AUXMC_E_WORKSPACE;
  AUXMC_CUDA_TRY(cudaMemsetAsync(fst, 0, sizeof(int), s));
  const int warps = factor_warps(fl.W);
  const size_t smem = sizeof(double) * (3 * fl.W * fl.W + 4) * warps;
  AUXMC_CUDA_TRY(cudaFuncSetAttribute(k_target_factors,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  AUXMC_LAUNCH(k_target_factors, (fl.total() + warps - 1) / warps, 32 * warps, smem, s, tg, fl, Ls,
               logdet, fst, dgf);
  AUXMC_LAUNCH(k_gamma_terms, grid_for((long long)C * (2 * tg.T + 2), 128), 128, 0, s, tg, fl, C,
               traj, Ls, logdet, terms, dgf);
  PFG_SUM_PARTS(C, 2LL * tg.T + 2, terms);
  AUXMC_LAUNCH(k_gamma_sum, C, kSumThreads, 0, s, tg.T, C, terms, fst, out, status, parts);
  if (parts) cudaFreeAsync(parts, s);
  return AUXMC_OK;
}

static int launch_grads(const DevTarget& tg, int C, const double* traj, double* grads, int* bad,
                        Arena& ws, cudaStream_t s) {
  const FactorLayout fl = factor_layout(tg);
  double* Ls = ws.take<double>((size_t)fl.total() * fl.W * fl.W);
  double* logdet = ws.take<double>(fl.total());
  int* fst = ws.take<int>(1);
  if (ws.base == nullptr) return AUXMC_OK;
  if (!Ls || !logdet || !fst) return AUXMC_E_WORKSPACE;
  if (fl.nG) {
    AUXMC_CUDA_TRY(cudaMemsetAsync(fst, 0, sizeof(int), s));
    const int warps = factor_warps(fl.W);
    const size_t smem = sizeof(double) * (3 * fl.W * fl.W + 4) * warps;
    AUXMC_CUDA_TRY(cudaFuncSetAttribute(k_target_factors,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    AUXMC_LAUNCH(k_target_factors, (fl.total() + warps - 1) / warps, 32 * warps, smem, s, tg, fl,
                 Ls, logdet, fst);
  }
  AUXMC_LAUNCH(k_grads, grid_for((long long)C * (tg.T + 1), 128), 128, 0, s, tg, fl, C, traj, Ls,
               grads, bad);
  return AUXMC_OK;
}

// One auxiliary Kalman step for all chains (auxk.cpp:130-198).
static int aux_step(const DevTarget& tg, auxmc_chains* ch, const auxmc_kernel_options& o,
                    Arena& ws, cudaStream_t s) {
  const int C = ch->C, T = tg.T, d = tg.dx, p = d + tg.q;
  const int nH = tg.exact_tv ? T + 1 : 1;
  const size_t nx = (size_t)C * (T + 1) * d;
  // Structure-aware path: the fused direct-observation filter (filter_direct.cu) for the
  // sequential filter; for Lorenz-96 (d > 4) also F_t as a stencil of the linearisation
  // point in every consumer (filter, backward elements, path terms), never in HBM.
  const bool stencil_ok = !tg.linear && tg.kind == AUXMC_KIND_LORENZ96 && d > 4;
  bool direct = false;
  {
    DevModel probe{};
    probe.T = T; probe.dx = d; probe.dy = p; probe.mask = nullptr;
    probe.nF = tg.linear ? tg.nF : (T > 0 ? T : 1);  // as dm below
    probe.nQ = tg.linear ? tg.nF : 1;
    direct = !o.parallel_filter && !g_force_generic_filter &&
             filter_direct_ok(tg, probe, stencil_ok);
  }
  const bool stencil = direct && stencil_ok;
  uint64_t* it = ws.take<uint64_t>(C);
  double* u = ws.take<double>(nx);
  double* prop = ws.take<double>(nx);
  double* gprop = ws.take<double>(nx);
  double* z = ws.take<double>((size_t)C * (T + 1) * p);
  double* Fa = (tg.linear || stencil) ? nullptr
                                      : ws.take<double>((size_t)C * (T > 0 ? T : 1) * d * d);
  double* ba = tg.linear ? nullptr : ws.take<double>((size_t)C * (T > 0 ? T : 1) * d);
  double* H = ws.take<double>((size_t)nH * p * d);
  double* cv = ws.take<double>((size_t)nH * p);
  double* R = ws.take<double>((size_t)C * nH * p * p);
  auxmc_filter_result fr;
  fr.pred_mean = ws.take<double>(nx);
  fr.filt_mean = ws.take<double>(nx);
  fr.pred_cov = ws.take<double>(nx * d);
  fr.filt_cov = ws.take<double>(nx * d);
  fr.log_marginal = ws.take<double>(C);
  StepScalars sc;
  sc.logq_fwd = ws.take<double>(C);
  sc.logq_rev = ws.take<double>(C);
  sc.lg_prop = ws.take<double>(C);
  sc.aux_prop = ws.take<double>(C);
  sc.aux_x = ws.take<double>(C);
  int* ints = ws.take<int>((size_t)C * 9);
  double* terms = ws.take<double>((size_t)C * (T + 1));
  auxmc_noise nz{};
  nz.kind = AUXMC_NOISE_STREAM;
  nz.keys = it;
  DevModel dm;
  dm.T = T; dm.dx = d; dm.dy = p;
  dm.m0 = tg.m0; dm.P0 = tg.P0;
  dm.F = tg.linear ? tg.F : Fa; dm.nF = tg.linear ? tg.nF : (T > 0 ? T : 1);
  dm.sF = tg.linear ? 0 : (long long)(T > 0 ? T : 1) * d * d;
  dm.b = tg.linear ? tg.b : ba; dm.nb = dm.nF;
  dm.sb = tg.linear ? 0 : (long long)(T > 0 ? T : 1) * d;
  dm.Q = tg.Q; dm.nQ = tg.linear ? tg.nF : 1; dm.sQ = 0;
  dm.H = H; dm.nH = nH; dm.sH = 0;
  dm.c = cv; dm.nc = nH; dm.sc = 0;
  dm.R = R; dm.nR = nH; dm.sR = (long long)nH * p * p;
  dm.mask = nullptr;
  dm.xl = nullptr; dm.sxl = (long long)(T + 1) * d; dm.fst = stencil ? 1 : 0; dm.fh = tg.l96_h;
  if (stencil) dm.F = nullptr;
  const int sampler = o.backend;
  int rc;
  // sub-arenas for the sampler, log γ and gradients (sizing pass included)
  if (ws.base == nullptr) {
    if (o.parallel_filter) {
      rc = launch_filter_pit(dm, z, C, &fr, nullptr, ws, s);
      if (rc) return rc;
    }
    rc = launch_sample_paths(dm, &fr, 0, &nz, C, sampler, prop, nullptr, ws, s);
    if (rc) return rc;
    rc = launch_log_gamma(tg, C, prop, sc.lg_prop, nullptr, ws, s);
    if (rc) return rc;
    return launch_grads(tg, C, prop, gprop, nullptr, ws, s);
  }
  if (!it || !u || !prop || !gprop || !z || !H || !cv || !R || !fr.filt_cov || !ints || !terms ||
      (!tg.linear && ((!stencil && !Fa) || !ba)))
    return AUXMC_E_WORKSPACE;
  sc.st_filt = ints; sc.st_samp = ints + C; sc.st_lqf = ints + 2 * C; sc.st_lg = ints + 3 * C;
  sc.bad = ints + 4 * C; sc.st_filt_r = ints + 5 * C; sc.st_lqr = ints + 6 * C;
  sc.accept = ints + 7 * C;
  AUXMC_CUDA_TRY(cudaMemsetAsync(ints, 0, sizeof(int) * C * 9, s));
  const int cb = (C + 127) / 128;
  AUXMC_LAUNCH(k_iter_keys, cb, 128, 0, s, C, ch->root_keys, ch->iter, it);
  AUXMC_LAUNCH(k_aux_obs, grid_for((long long)nx), 256, 0, s, C, T, d, ch->x, ch->delta, it, u);
  AUXMC_LAUNCH(k_build_HR, grid_for((long long)C * nH * p * p), 256, 0, s, tg, C, nH, ch->delta,
               H, cv, R);
  // forward: surrogate at x, filter, proposal, log q(x'|x)
  AUXMC_LAUNCH(k_build_aux, grid_for((long long)C * (T + 1), 128), 128, 0, s, tg, C,
               o.zeroth_order, ch->x, ch->grad_gen, u, ch->delta, z, Fa, ba);
  Arena pf_ws = ws;  // scan-filter scratch (sized in the sizing pass above)
  // covs = 0: the reverse pass needs log p(z) only (launch_path_logpdf)
  auto filter = [&](int* st, const double* xlin, int covs) {
    if (o.parallel_filter) {
      Arena sub = pf_ws;
      return launch_filter_pit(dm, z, C, &fr, st, sub, s);
    }
    if (direct) return launch_filter_direct(tg, dm, stencil, xlin, ch->delta, z, C, &fr, st, covs, s);
    return launch_filter_seq(dm, z, C, &fr, st, s);
  };
  dm.xl = ch->x;
  rc = filter(sc.st_filt, ch->x, 1);
  if (rc) return rc;
  if (g_capture_lm)
    AUXMC_CUDA_TRY(cudaMemcpyAsync(g_capture_lm, fr.log_marginal, sizeof(double) * C,
                                   cudaMemcpyDeviceToDevice, s));
  rc = launch_sample_paths(dm, &fr, 0, &nz, C, sampler, prop, sc.st_samp, ws, s);
  if (rc) return rc;
  rc = launch_path_logpdf(dm, z, (long long)(T + 1) * p, prop, fr.log_marginal, 0, C, sc.logq_fwd,
                          sc.st_lqf, s);
  if (rc) return rc;
  // log γ(x'), ∇ log g(x')
  {
    Arena sub = ws;
    rc = launch_log_gamma(tg, C, prop, sc.lg_prop, sc.st_lg, sub, s);
    if (rc) return rc;
    Arena sub2 = ws;
    rc = launch_grads(tg, C, prop, gprop, sc.bad, sub2, s);
    if (rc) return rc;
  }
  // reverse: surrogate at x', filter, log q(x|x')
  AUXMC_LAUNCH(k_build_aux, grid_for((long long)C * (T + 1), 128), 128, 0, s, tg, C,
               o.zeroth_order, prop, gprop, u, ch->delta, z, Fa, ba);
  dm.xl = prop;
  rc = filter(sc.st_filt_r, prop, 0);
  if (rc) return rc;
  rc = launch_path_logpdf(dm, z, (long long)(T + 1) * p, ch->x, fr.log_marginal, 0, C,
                          sc.logq_rev, sc.st_lqr, s);
  if (rc) return rc;
  // aux log-likelihoods Σ_t log N(u_t; ·, δ/2 I)
  AUXMC_LAUNCH(k_aux_lik_terms, grid_for((long long)C * (T + 1)), 256, 0, s, C, T, d, u, prop,
               ch->delta, terms);
  {
    PFG_SUM_PARTS(C, (long long)T + 1, terms);
    AUXMC_LAUNCH(k_row_sum, C, kSumThreads, 0, s, C, T + 1, terms, sc.aux_prop, parts);
    if (parts) cudaFreeAsync(parts, s);
  }
  AUXMC_LAUNCH(k_aux_lik_terms, grid_for((long long)C * (T + 1)), 256, 0, s, C, T, d, u, ch->x,
               ch->delta, terms);
  {
    PFG_SUM_PARTS(C, (long long)T + 1, terms);
    AUXMC_LAUNCH(k_row_sum, C, kSumThreads, 0, s, C, T + 1, terms, sc.aux_x, parts);
    if (parts) cudaFreeAsync(parts, s);
  }
  AUXMC_LAUNCH(k_mh, cb, 128, 0, s, C, sc, it, ch->log_gamma, ch->iter, ch->stats);
  AUXMC_LAUNCH(k_accept_copy, grid_for((long long)nx), 256, 0, s, C, (long long)(T + 1) * d,
               sc.accept, prop, gprop, ch->x, ch->grad_gen);
  return AUXMC_OK;
}

// factor list of the target's fixed covariances (P0, Q, R_e, generic R)
int launch_target_factors(const DevTarget& tg, double* Ls, double* logdet, int* fst,
                          cudaStream_t s) {
  const FactorLayout fl = factor_layout(tg);
  AUXMC_CUDA_TRY(cudaMemsetAsync(fst, 0, sizeof(int), s));
  const int warps = factor_warps(fl.W);
  const size_t smem = sizeof(double) * (3 * fl.W * fl.W + 4) * warps;
  AUXMC_CUDA_TRY(cudaFuncSetAttribute(k_target_factors,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  AUXMC_LAUNCH(k_target_factors, (fl.total() + warps - 1) / warps, 32 * warps, smem, s, tg, fl, Ls,
               logdet, fst);
  return AUXMC_OK;
}

int launch_aux_obs(int C, int T, int d, const double* x, const double* delta, const uint64_t* it,
                   double* u, cudaStream_t s) {
  const long long n = (long long)C * (T + 1) * d;
  AUXMC_LAUNCH(k_aux_obs, grid_for(n), 256, 0, s, C, T, d, x, delta, it, u);
  return AUXMC_OK;
}

}  // namespace auxmc_gpu

namespace auxmc_gpu {
// ---- time-sharded aux step kernels (one chain; t ranges are absolute steps)
int tshard_geometry(int T, int* LB, int* nblk, int* nsup, int* SB);
__global__ void k_factor_list(DevModel m, int nQb, int nRb, double* Ls, double* logdet,
                              unsigned char* dg, int* status);  // logpdf.cu

// aux observations (if u_out) and the surrogate LGSSM rows at the path xs on [t0, t1)
__global__ void k_ts_prep(DevTarget tg, int zeroth, const double* __restrict__ xs,
                          const double* __restrict__ gs, const double* __restrict__ delta,
                          const uint64_t* __restrict__ it, int t0, int t1, int make_u,
                          double* u, double* z, double* Fa, double* ba) {
  const int T = tg.T, d = tg.dx, p = d + tg.q;
  const double h = delta[0] / 2.0, sd = sqrt(delta[0] / 2.0);
  for (int t = t0 + blockIdx.x * blockDim.x + threadIdx.x; t < t1; t += gridDim.x * blockDim.x) {
    const double* xt = xs + (size_t)t * d;
    if (make_u) {
      const uint64_t k = derive(it[0], kAuxObs, (uint64_t)t);
      for (int i = 0; i < d; ++i) u[(size_t)t * d + i] = xt[i] + sd * normal_at(k, (uint64_t)i);
    }
    double* zt = z + (size_t)t * p;
    for (int i = 0; i < d; ++i) {
      double v = u[(size_t)t * d + i];
      if (!zeroth) v += h * gs[(size_t)t * d + i];
      zt[i] = v;
    }
    for (int k = 0; k < tg.q; ++k) zt[d + k] = tg.emask[t] ? tg.ey[(size_t)t * tg.q + k] : 0.0;
    if (!tg.linear && t < T) {
      double* F = Fa + (size_t)t * d * d;
      double* bb = ba + (size_t)t * d;
      for (int i = 0; i < d; ++i)
        for (int j = 0; j < d; ++j) F[i * d + j] = dyn_jac_ij(tg, t, xt, i, j);
      for (int i = 0; i < d; ++i) {
        double s = 0.0;
        for (int j = 0; j < d; ++j) s += F[i * d + j] * xt[j];
        bb[i] = dyn_mean_i(tg, t, xt, i) - s;
      }
    }
  }
}

// generic gradients on [t0, t1); non-finite ones on the own range [a, b) flag an abort
__global__ void k_ts_grads(DevTarget tg, FactorLayout fl, const double* __restrict__ traj,
                           const double* __restrict__ Ls, int t0, int t1, int a, int b,
                           double* grads, int* bad) {
  const int d = tg.dx;
  double r[64], g[64];
  for (int t = t0 + blockIdx.x * blockDim.x + threadIdx.x; t < t1; t += gridDim.x * blockDim.x) {
    const int jg = 1 + fl.nQ + fl.nE + (tg.ne > 1 ? t : 0);
    generic_grad(tg, t, traj + (size_t)t * d, fl.nG ? Ls + (size_t)jg * fl.W * fl.W : nullptr, r, g);
    bool ok = true;
    for (int i = 0; i < d; ++i) {
      grads[(size_t)t * d + i] = g[i];
      ok = ok && isfinite(g[i]);
    }
    if (!ok && t >= a && t < b) atomicOr(bad, 1);
  }
}

// per-t sums of a path's log-density terms: v_t = ((prior) + transition t) + observation t
__global__ void k_ts_path_v(DevModel m, const double* __restrict__ obs, const double* __restrict__ x,
                            const double* __restrict__ Ls, const double* __restrict__ logdet,
                            int a, int b, double* v) {
  const int T = m.T;
  for (int t = a + blockIdx.x * blockDim.x + threadIdx.x; t < b; t += gridDim.x * blockDim.x) {
    double s = 0.0;
    if (t == 0) s += path_term_k(m, obs, x, 0, 1, Ls, logdet, 0);
    if (t < T) s += path_term_k(m, obs, x, 0, 1, Ls, logdet, 1 + t);
    s += path_term_k(m, obs, x, 0, 1, Ls, logdet, T + 1 + t);
    v[t] = s;
  }
}
__global__ void k_ts_gamma_v(DevTarget tg, FactorLayout fl, const double* __restrict__ x,
                             const double* __restrict__ Ls, const double* __restrict__ logdet,
                             int a, int b, double* v) {
  const int T = tg.T;
  for (int t = a + blockIdx.x * blockDim.x + threadIdx.x; t < b; t += gridDim.x * blockDim.x) {
    double s = 0.0;
    if (t == 0) s += gamma_term_k(tg, fl, x, Ls, logdet, 0);
    if (t < T) s += gamma_term_k(tg, fl, x, Ls, logdet, 1 + t);
    s += gamma_term_k(tg, fl, x, Ls, logdet, T + 1 + t);
    v[t] = s;
  }
}
__global__ void k_ts_aux_v(int d, const double* __restrict__ u, const double* __restrict__ x,
                           const double* __restrict__ delta, int a, int b, double* v) {
  const double var = delta[0] / 2.0;
  for (int t = a + blockIdx.x * blockDim.x + threadIdx.x; t < b; t += gridDim.x * blockDim.x) {
    double sq = 0.0;
    for (int i = 0; i < d; ++i) {
      const double r = u[(size_t)t * d + i] - x[(size_t)t * d + i];
      sq += r * r;
    }
    v[t] = -0.5 * (d * (kLog2Pi + log(var)) + sq / var);  // gauss.cpp:59-62
  }
}
// super-block partial sums of v over the rank's super-blocks: one warp per super-block,
// lane l sums its contiguous 1/32 of the block in t order, then a fixed shuffle tree —
// an association that depends on (T, SB) only, so every split gives the same bits
__global__ void k_ts_sb_sum(const double* __restrict__ v, int T, int SB, int sup_lo, int sup_hi,
                            double* part, int col) {
  const int lane = threadIdx.x & 31;
  const int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int s = sup_lo + wid; s < sup_hi; s += nw) {
    const int lo = s * SB, hi = min((s + 1) * SB, T + 1);
    const int ch = (hi - lo + 31) / 32;
    const int a = min(lo + lane * ch, hi), b = min(a + ch, hi);
    double acc = 0.0;
    for (int t = a; t < b; ++t) acc += v[t];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
    if (lane == 0) part[(size_t)(s - sup_lo) * 5 + col] = acc;
  }
}
// the MH inputs from every rank's partials (super-block order) and the reduced flags
__global__ void k_ts_scalars(const double* __restrict__ parts, int nsup, const double* lm_fwd,
                             const double* lm_rev, const int* __restrict__ flags, StepScalars sc) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double s[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  for (int k = 0; k < nsup; ++k)
    for (int c = 0; c < 5; ++c) s[c] += parts[(size_t)k * 5 + c];
  sc.logq_fwd[0] = s[0] - lm_fwd[0];
  sc.lg_prop[0] = s[1];
  sc.logq_rev[0] = s[2] - lm_rev[0];
  sc.aux_prop[0] = s[3];
  sc.aux_x[0] = s[4];
  sc.st_filt[0] = flags[0];
  sc.st_samp[0] = flags[1];
  sc.st_lqf[0] = flags[2];
  sc.st_lg[0] = flags[3];
  sc.bad[0] = flags[4];
  sc.st_filt_r[0] = flags[5];
  sc.st_lqr[0] = flags[6];
}
__global__ void k_ts_accept(int d, int t0, int t1, const int* accept, const double* prop,
                            const double* gprop, double* x, double* grad) {
  if (!accept[0]) return;
  const long long lo = (long long)t0 * d, hi = (long long)t1 * d;
  for (long long q = lo + blockIdx.x * blockDim.x + threadIdx.x; q < hi; q += gridDim.x * blockDim.x) {
    x[q] = prop[q];
    grad[q] = gprop[q];
  }
}
}  // namespace auxmc_gpu

using namespace auxmc_gpu;

// ---------------------------------------------------------------- time-sharded aux step
// One chain (C = 1) whose scans are split over ranks (tshard.py): the caller
// runs `begin`, the sharded forward filter and prefix sampler on the auxiliary
// LGSSM it describes, all-gathers the proposal path, `middle`, the sharded reverse
// filter, then `end`.  Everything outside the scans is cheap per-t work that every
// rank repeats on the whole horizon, so every split gives the same bits.
namespace {
struct TsAux {
  uint64_t* it;
  double *u, *prop, *gprop, *z, *Fa, *ba, *H, *cv, *R, *terms;
  StepScalars sc;
  int* ints;
  DevModel dm;
};
TsAux ts_aux_take(const DevTarget& tg, Arena& ws) {
  const int T = tg.T, d = tg.dx, p = d + tg.q;
  const int nH = tg.exact_tv ? T + 1 : 1;
  const size_t nx = (size_t)(T + 1) * d;
  TsAux a;
  a.it = ws.take<uint64_t>(1);
  a.u = ws.take<double>(nx);
  a.prop = ws.take<double>(nx);
  a.gprop = ws.take<double>(nx);
  a.z = ws.take<double>((size_t)(T + 1) * p);
  a.Fa = tg.linear ? nullptr : ws.take<double>((size_t)(T > 0 ? T : 1) * d * d);
  a.ba = tg.linear ? nullptr : ws.take<double>((size_t)(T > 0 ? T : 1) * d);
  a.H = ws.take<double>((size_t)nH * p * d);
  a.cv = ws.take<double>((size_t)nH * p);
  a.R = ws.take<double>((size_t)nH * p * p);
  a.terms = ws.take<double>((size_t)(T + 1));
  double* scal = ws.take<double>(5);
  a.ints = ws.take<int>(9);
  if (scal) {
    a.sc.logq_fwd = scal; a.sc.logq_rev = scal + 1; a.sc.lg_prop = scal + 2;
    a.sc.aux_prop = scal + 3; a.sc.aux_x = scal + 4;
  }
  if (a.ints) {
    a.sc.st_filt = a.ints; a.sc.st_samp = a.ints + 1; a.sc.st_lqf = a.ints + 2;
    a.sc.st_lg = a.ints + 3; a.sc.bad = a.ints + 4; a.sc.st_filt_r = a.ints + 5;
    a.sc.st_lqr = a.ints + 6; a.sc.accept = a.ints + 7;
  }
  DevModel& dm = a.dm;
  dm.T = T; dm.dx = d; dm.dy = p;
  dm.m0 = tg.m0; dm.P0 = tg.P0;
  dm.F = tg.linear ? tg.F : a.Fa; dm.nF = tg.linear ? tg.nF : (T > 0 ? T : 1); dm.sF = 0;
  dm.b = tg.linear ? tg.b : a.ba; dm.nb = dm.nF; dm.sb = 0;
  dm.Q = tg.Q; dm.nQ = tg.linear ? tg.nF : 1; dm.sQ = 0;
  dm.H = a.H; dm.nH = nH; dm.sH = 0;
  dm.c = a.cv; dm.nc = nH; dm.sc = 0;
  dm.R = a.R; dm.nR = nH; dm.sR = 0;
  dm.mask = nullptr;
  return a;
}
}  // namespace

extern "C" {

size_t auxmc_aux_kernel_workspace(const auxmc_target* target, int C,
                                  const auxmc_kernel_options* opts) {
  if (check_target(target) || C < 0 || !opts) return 0;
  Arena ws{nullptr, 0, 0};
  auxmc_chains ch{};
  ch.C = C;
  aux_step(to_dev_target(*target), &ch, *opts, ws, nullptr);
  return ws.used + 4096;
}

int auxmc_aux_kernel_step(const auxmc_target* target, auxmc_chains* chains,
                          const auxmc_kernel_options* opts, void* workspace,
                          size_t workspace_bytes, void* stream) {
  if (!device_ok()) return AUXMC_E_CUDA;
  int st = check_target(target);
  if (st) return st;
  if (!chains || !opts || chains->C < 0 || !chains->x || !chains->delta || !chains->log_gamma ||
      !chains->grad_gen || !chains->iter || !chains->stats || !chains->root_keys)
    return AUXMC_E_ARG;
  if (opts->backend < 0 || opts->backend > 2) return AUXMC_E_ARG;
  if (chains->C == 0) return AUXMC_OK;
  if (!workspace) return AUXMC_E_WORKSPACE;
  Arena ws{(char*)workspace, workspace_bytes, 0};
  return aux_step(to_dev_target(*target), chains, *opts, ws, (cudaStream_t)stream);
}

int auxmc_init_chains(const auxmc_target* target, auxmc_chains* chains, void* workspace,
                      size_t workspace_bytes, void* stream) {
  if (!device_ok()) return AUXMC_E_CUDA;
  int st = check_target(target);
  if (st) return st;
  if (!chains || !chains->x || !chains->log_gamma || !chains->grad_gen) return AUXMC_E_ARG;
  if (chains->C == 0) return AUXMC_OK;
  const DevTarget tg = to_dev_target(*target);
  Arena sizing{nullptr, 0, 0};
  launch_log_gamma(tg, chains->C, chains->x, chains->log_gamma, nullptr, sizing, nullptr);
  launch_grads(tg, chains->C, chains->x, chains->grad_gen, nullptr, sizing, nullptr);
  if (!workspace || workspace_bytes < sizing.used) return AUXMC_E_WORKSPACE;
  Arena ws{(char*)workspace, workspace_bytes, 0};
  st = launch_log_gamma(tg, chains->C, chains->x, chains->log_gamma, nullptr, ws, (cudaStream_t)stream);
  if (st) return st;
  Arena ws2{(char*)workspace, workspace_bytes, 0};
  return launch_grads(tg, chains->C, chains->x, chains->grad_gen, nullptr, ws2, (cudaStream_t)stream);
}

int auxmc_adapt_delta(auxmc_chains* chains, double target_rate, void* stream) {
  if (!device_ok()) return AUXMC_E_CUDA;
  if (!chains || !chains->delta || !chains->iter || !chains->stats) return AUXMC_E_ARG;
  if (chains->C == 0) return AUXMC_OK;
  AUXMC_LAUNCH(k_adapt, (chains->C + 127) / 128, 128, 0, stream, chains->C, chains->iter,
               chains->stats, target_rate, chains->delta);
  return AUXMC_OK;
}

int auxmc_log_gamma(const auxmc_target* target, const double* traj, int B, double* out,
                    int* status, void* stream) {
  if (!device_ok()) return AUXMC_E_CUDA;
  int st = check_target(target);
  if (st) return st;
  if (!traj || !out || B < 0) return AUXMC_E_ARG;
  if (B == 0) return AUXMC_OK;
  const DevTarget tg = to_dev_target(*target);
  Arena sizing{nullptr, 0, 0};
  launch_log_gamma(tg, B, traj, out, status, sizing, nullptr);
  void* buf = nullptr;
  AUXMC_CUDA_TRY(cudaMallocAsync(&buf, sizing.used + 1024, (cudaStream_t)stream));
  Arena ws{(char*)buf, sizing.used + 1024, 0};
  st = launch_log_gamma(tg, B, traj, out, status, ws, (cudaStream_t)stream);
  cudaFreeAsync(buf, (cudaStream_t)stream);
  return st;
}


size_t auxmc_tshard_aux_workspace(const auxmc_target* target) {
  if (check_target(target)) return 0;
  const DevTarget tg = to_dev_target(*target);
  Arena ws{nullptr, 0, 0};
  ts_aux_take(tg, ws);
  Arena sub = ws;
  launch_log_gamma(tg, 1, nullptr, nullptr, nullptr, sub, nullptr);
  Arena sub2 = ws;
  launch_grads(tg, 1, nullptr, nullptr, nullptr, sub2, nullptr);
  return std::max(sub.used, sub2.used) + 4096;
}

static int ts_geom(const DevTarget& tg, int t_lo, int t_hi, int* SB, int* sup_lo, int* sup_hi) {
  int LB, nblk, nsup;
  tshard_geometry(tg.T, &LB, &nblk, &nsup, SB);
  if (t_lo < 0 || t_hi > tg.T + 1 || t_hi < t_lo) return AUXMC_E_ARG;
  if (t_hi == t_lo) {  // a rank that owns no super-block
    *sup_lo = *sup_hi = 0;
    return AUXMC_OK;
  }
  if (t_lo % *SB) return AUXMC_E_ARG;
  *sup_lo = t_lo / *SB;
  *sup_hi = (t_hi + *SB - 1) / *SB;
  return AUXMC_OK;
}
static inline int grid_t(int n) { return std::max(1, std::min((n + 127) / 128, 148 * 16)); }

int auxmc_tshard_aux_begin(const auxmc_target* target, auxmc_chains* ch,
                           const auxmc_kernel_options* opts, void* workspace,
                           size_t workspace_bytes, int t_lo, int t_hi, auxmc_lgssm* model_out,
                           double** z_out, double** prop_out, uint64_t** it_out, void* stream) {
  if (!device_ok()) return AUXMC_E_CUDA;
  int st = check_target(target);
  if (st) return st;
  if (!ch || ch->C != 1 || !opts || !workspace || !model_out || !z_out || !prop_out || !it_out)
    return AUXMC_E_ARG;
  const DevTarget tg = to_dev_target(*target);
  int SB, slo, shi;
  if ((st = ts_geom(tg, t_lo, t_hi, &SB, &slo, &shi))) return st;
  Arena ws{(char*)workspace, workspace_bytes, 0};
  const TsAux a = ts_aux_take(tg, ws);
  if (!a.ints || !a.R) return AUXMC_E_WORKSPACE;
  cudaStream_t s = (cudaStream_t)stream;
  const int T = tg.T, d = tg.dx, p = d + tg.q, nH = a.dm.nH;
  const bool own = t_hi > t_lo;
  const int h0 = own ? std::max(t_lo - 1, 0) : 0, h1 = own ? std::min(t_hi + 1, T + 1) : 0;
  AUXMC_CUDA_TRY(cudaMemsetAsync(a.ints, 0, sizeof(int) * 9, s));
  AUXMC_LAUNCH(k_iter_keys, 1, 32, 0, s, 1, ch->root_keys, ch->iter, a.it);
  AUXMC_LAUNCH(k_build_HR, grid_for((long long)nH * p * p), 256, 0, s, tg, 1, nH, ch->delta, a.H,
               a.cv, a.R);
  if (h1 > h0)
    AUXMC_LAUNCH(k_ts_prep, grid_t(h1 - h0), 128, 0, s, tg, opts->zeroth_order, ch->x, ch->grad_gen,
                 ch->delta, a.it, h0, h1, 1, a.u, a.z, a.Fa, a.ba);
  auxmc_lgssm& m = *model_out;
  m.T = T; m.dx = d; m.dy = p;
  m.m0 = a.dm.m0; m.P0 = a.dm.P0;
  m.F = a.dm.F; m.nF = a.dm.nF; m.b = a.dm.b; m.nb = a.dm.nb; m.Q = a.dm.Q; m.nQ = a.dm.nQ;
  m.H = a.H; m.nH = nH; m.c = a.cv; m.nc = nH; m.R = a.R; m.nR = nH; m.mask = nullptr;
  *z_out = a.z;
  *prop_out = a.prop;
  *it_out = a.it;
  return AUXMC_OK;
}

// path-logpdf terms of `traj` under the current surrogate (a.dm, pseudo-observations a.z)
static int ts_path_part(const TsAux& a, const double* traj, int t_lo, int t_hi, int SB, int slo,
                        int shi, double* part, int col, int* fst, cudaStream_t s) {
  const DevModel& dm = a.dm;
  const int W = dm.dx > dm.dy ? dm.dx : dm.dy;
  const int n_mats = 1 + dm.nQ + (dm.dy > 0 ? dm.nR : 0);
  double *Ls = nullptr, *logdet = nullptr;
  AUXMC_CUDA_TRY(cudaMallocAsync(&Ls, sizeof(double) * n_mats * W * W, s));
  AUXMC_CUDA_TRY(cudaMallocAsync(&logdet, sizeof(double) * n_mats, s));
  const int warps = factor_warps(W);
  const size_t smem = sizeof(double) * (3 * W * W + 4) * warps;
  AUXMC_CUDA_TRY(cudaFuncSetAttribute(k_factor_list, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem));
  AUXMC_LAUNCH(k_factor_list, std::min((n_mats + warps - 1) / warps, 148 * 8), 32 * warps, smem, s,
               dm, 1, 1, Ls, logdet, (unsigned char*)nullptr, fst);
  if (t_hi > t_lo) {
    AUXMC_LAUNCH(k_ts_path_v, grid_t(t_hi - t_lo), 128, 0, s, dm, a.z, traj, Ls, logdet, t_lo, t_hi,
                 a.terms);
    AUXMC_LAUNCH(k_ts_sb_sum, std::max(1, (shi - slo + 3) / 4), 128, 0, s, a.terms, dm.T, SB, slo, shi, part, col);
  }
  cudaFreeAsync(Ls, s);
  cudaFreeAsync(logdet, s);
  return AUXMC_OK;
}

int auxmc_tshard_aux_middle(const auxmc_target* target, auxmc_chains* ch,
                            const auxmc_kernel_options* opts, void* workspace,
                            size_t workspace_bytes, int t_lo, int t_hi, double* part_out,
                            int* flags_out, void* stream) {
  if (!device_ok()) return AUXMC_E_CUDA;
  int st = check_target(target);
  if (st) return st;
  if (!ch || ch->C != 1 || !opts || !workspace || !part_out || !flags_out) return AUXMC_E_ARG;
  const DevTarget tg = to_dev_target(*target);
  int SB, slo, shi;
  if ((st = ts_geom(tg, t_lo, t_hi, &SB, &slo, &shi))) return st;
  Arena ws{(char*)workspace, workspace_bytes, 0};
  const TsAux a = ts_aux_take(tg, ws);
  if (!a.ints) return AUXMC_E_WORKSPACE;
  cudaStream_t s = (cudaStream_t)stream;
  const int T = tg.T;
  const bool own = t_hi > t_lo;
  const int h0 = own ? std::max(t_lo - 1, 0) : 0, h1 = own ? std::min(t_hi + 1, T + 1) : 0;
  // log q(x'|x): the forward surrogate's path terms at the proposal
  int rc = ts_path_part(a, a.prop, t_lo, t_hi, SB, slo, shi, part_out, 0, flags_out + 2, s);
  if (rc) return rc;
  // log gamma(x') terms and the gradients at x' (target factors)
  const FactorLayout fl = factor_layout(tg);
  Arena sub = ws;
  double* Ls = sub.take<double>((size_t)fl.total() * fl.W * fl.W);
  double* logdet = sub.take<double>(fl.total());
  if (!Ls || !logdet) return AUXMC_E_WORKSPACE;
  const int warps = factor_warps(fl.W);
  const size_t smem = sizeof(double) * (3 * fl.W * fl.W + 4) * warps;
  AUXMC_CUDA_TRY(cudaFuncSetAttribute(k_target_factors, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem));
  AUXMC_LAUNCH(k_target_factors, (fl.total() + warps - 1) / warps, 32 * warps, smem, s, tg, fl, Ls,
               logdet, flags_out + 3);
  if (t_hi > t_lo) {
    AUXMC_LAUNCH(k_ts_gamma_v, grid_t(t_hi - t_lo), 128, 0, s, tg, fl, a.prop, Ls, logdet, t_lo,
                 t_hi, a.terms);
    AUXMC_LAUNCH(k_ts_sb_sum, std::max(1, (shi - slo + 3) / 4), 128, 0, s, a.terms, T, SB, slo, shi, part_out, 1);
  }
  if (h1 > h0) {
    AUXMC_LAUNCH(k_ts_grads, grid_t(h1 - h0), 128, 0, s, tg, fl, a.prop, Ls, h0, h1, t_lo, t_hi,
                 a.gprop, flags_out + 4);
    // the reverse surrogate at x' (pseudo-observations and linearized dynamics)
    AUXMC_LAUNCH(k_ts_prep, grid_t(h1 - h0), 128, 0, s, tg, opts->zeroth_order, a.prop, a.gprop,
                 ch->delta, a.it, h0, h1, 0, a.u, a.z, a.Fa, a.ba);
  }
  return AUXMC_OK;
}

int auxmc_tshard_aux_end(const auxmc_target* target, auxmc_chains* ch,
                         const auxmc_kernel_options* opts, void* workspace, size_t workspace_bytes,
                         int t_lo, int t_hi, double* part_out, int* flags_out, void* stream) {
  if (!device_ok()) return AUXMC_E_CUDA;
  int st = check_target(target);
  if (st) return st;
  if (!ch || ch->C != 1 || !opts || !workspace || !part_out || !flags_out) return AUXMC_E_ARG;
  const DevTarget tg = to_dev_target(*target);
  int SB, slo, shi;
  if ((st = ts_geom(tg, t_lo, t_hi, &SB, &slo, &shi))) return st;
  Arena ws{(char*)workspace, workspace_bytes, 0};
  const TsAux a = ts_aux_take(tg, ws);
  if (!a.ints) return AUXMC_E_WORKSPACE;
  cudaStream_t s = (cudaStream_t)stream;
  const int T = tg.T, d = tg.dx;
  // log q(x|x'): the reverse surrogate's path terms at the current path
  int rc = ts_path_part(a, ch->x, t_lo, t_hi, SB, slo, shi, part_out, 2, flags_out + 6, s);
  if (rc) return rc;
  if (t_hi > t_lo) {
    AUXMC_LAUNCH(k_ts_aux_v, grid_t(t_hi - t_lo), 128, 0, s, d, a.u, a.prop, ch->delta, t_lo, t_hi,
                 a.terms);
    AUXMC_LAUNCH(k_ts_sb_sum, std::max(1, (shi - slo + 3) / 4), 128, 0, s, a.terms, T, SB, slo, shi, part_out, 3);
    AUXMC_LAUNCH(k_ts_aux_v, grid_t(t_hi - t_lo), 128, 0, s, d, a.u, ch->x, ch->delta, t_lo, t_hi,
                 a.terms);
    AUXMC_LAUNCH(k_ts_sb_sum, std::max(1, (shi - slo + 3) / 4), 128, 0, s, a.terms, T, SB, slo, shi, part_out, 4);
  }
  return AUXMC_OK;
}

int auxmc_tshard_aux_decide(const auxmc_target* target, auxmc_chains* ch, void* workspace,
                            size_t workspace_bytes, int t_lo, int t_hi, const double* parts_all,
                            int nsup, const double* log_marginal_fwd,
                            const double* log_marginal_rev, const int* flags, void* stream) {
  if (!device_ok()) return AUXMC_E_CUDA;
  int st = check_target(target);
  if (st) return st;
  if (!ch || ch->C != 1 || !workspace || !parts_all || !log_marginal_fwd || !log_marginal_rev ||
      !flags || nsup < 1)
    return AUXMC_E_ARG;
  const DevTarget tg = to_dev_target(*target);
  int SB, slo, shi;
  if ((st = ts_geom(tg, t_lo, t_hi, &SB, &slo, &shi))) return st;
  Arena ws{(char*)workspace, workspace_bytes, 0};
  const TsAux a = ts_aux_take(tg, ws);
  if (!a.ints) return AUXMC_E_WORKSPACE;
  cudaStream_t s = (cudaStream_t)stream;
  const int T = tg.T, d = tg.dx;
  const bool own = t_hi > t_lo;
  const int h0 = own ? std::max(t_lo - 1, 0) : 0, h1 = own ? std::min(t_hi + 1, T + 1) : 0;
  AUXMC_LAUNCH(k_ts_scalars, 1, 32, 0, s, parts_all, nsup, log_marginal_fwd, log_marginal_rev, flags,
               a.sc);
  AUXMC_LAUNCH(k_mh, 1, 32, 0, s, 1, a.sc, a.it, ch->log_gamma, ch->iter, ch->stats);
  if (h1 > h0)
    AUXMC_LAUNCH(k_ts_accept, grid_t((h1 - h0) * d), 128, 0, s, d, h0, h1, a.sc.accept, a.prop, a.gprop,
                 ch->x, ch->grad_gen);
  return AUXMC_OK;
}

}  // extern "C"

extern "C" int auxmc_test_force_generic_filter(int on) {
  auxmc_gpu::g_force_generic_filter = on ? 1 : 0;
  return AUXMC_OK;
}

extern "C" int auxmc_test_capture_log_marginal(double* dev_out) {
  auxmc_gpu::g_capture_lm = dev_out;
  return AUXMC_OK;
}
