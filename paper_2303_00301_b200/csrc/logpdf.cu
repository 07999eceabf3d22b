// logpdf.cu — lgssm::path_logpdf (lgssm.cpp:179-199) for batches of paths.
//
// Every covariance the reference factors inside a log_pdf call (P0, Q_t, R_t;
// gauss.cpp:51-57) is path-independent, so each distinct matrix is factored
// once (jitter ladder included) and reused by all paths.  Per-(path, term)
// Mahalanobis terms run one per thread; each path then sums its terms in the
// reference's order (prior, transitions t = 0..T-1, observations t = 0..T).
#include "common.cuh"
#include "dense.cuh"

namespace auxmc_gpu {

// Factor matrix j of a list: P0 (j = 0), Q_i (1..nQ), R_i (nQ+1..nQ+nR).
__global__ void k_factor_list(DevModel m, double* Ls, double* logdet, int* status) {
  extern __shared__ double smem[];
  const int dx = m.dx, dy = m.dy;
  const int n_items = 1 + m.nQ + (dy > 0 ? m.nR : 0);
  const int W = dx > dy ? dx : dy;
  Grp g = warp_group();
  const int gid = threadIdx.x >> 5, gpb = blockDim.x >> 5;
  double* A = smem + (size_t)gid * (3 * W * W + 4);
  double* L = A + W * W;
  double* scr = L + W * W;
  double* red = scr + W * W;
  int* flag = reinterpret_cast<int*>(red + 2);
  for (int j = blockIdx.x * gpb + gid; j < n_items; j += gridDim.x * gpb) {
    const double* src;
    int n;
    if (j == 0) { src = m.P0; n = dx; }
    else if (j <= m.nQ) { src = m.Q + (size_t)(j - 1) * dx * dx; n = dx; }
    else { src = m.R + (size_t)(j - 1 - m.nQ) * dy * dy; n = dy; }
    for (int i = g.lane; i < n * n; i += g.size) {
      const int r = i / n, c = i % n;
      A[i] = (src[r * n + c] + src[c * n + r]) * 0.5;
    }
    g.sync();
    const int st = g_factor_psd(g, n, A, L, scr, flag, red);
    double* out = Ls + (size_t)j * W * W;
    for (int i = g.lane; i < n * n; i += g.size) out[i] = L[i];
    if (g.lane == 0) {
      double ld = 0.0;
      for (int i = 0; i < n; ++i) ld += log(L[i * n + i]);
      logdet[j] = ld;
      if (st) atomicMax(status, st);
    }
    g.sync();
  }
}

// term index k: 0 prior; 1..T transition t=k-1; T+1..2T+1 observation t=k-T-1.
__global__ void k_path_terms(DevModel m, const double* __restrict__ obs, int obs_shared,
                             const double* __restrict__ traj, int B, const double* __restrict__ Ls,
                             const double* __restrict__ logdet, double* terms) {
  const int T = m.T, dx = m.dx, dy = m.dy;
  const int W = dx > dy ? dx : dy;
  const int K = 2 * T + 2;
  const long long n = (long long)B * K;
  double r[64];
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (long long)gridDim.x * blockDim.x) {
    const int b = (int)(q / K), k = (int)(q % K);
    const double* x = traj + (size_t)b * (T + 1) * dx;
    const double* L;
    double ld;
    int nn;
    if (k == 0) {
      nn = dx;
      for (int i = 0; i < dx; ++i) r[i] = x[i] - m.m0[i];
      L = Ls;
      ld = logdet[0];
    } else if (k <= T) {
      const int t = k - 1;
      nn = dx;
      const double* F = m.Ft(t);
      const double* bb = m.bt(t);
      for (int i = 0; i < dx; ++i) {
        double s = 0.0;
        for (int j = 0; j < dx; ++j) s += F[i * dx + j] * x[(size_t)t * dx + j];
        r[i] = x[(size_t)(t + 1) * dx + i] - (s + bb[i]);
      }
      const int j = 1 + (m.nQ > 1 ? t : 0);
      L = Ls + (size_t)j * W * W;
      ld = logdet[j];
    } else {
      const int t = k - T - 1;
      if (!m.observed(t) || dy == 0) {
        terms[q] = 0.0;
        continue;
      }
      nn = dy;
      const double* H = m.Ht(t);
      const double* cc = m.ct(t);
      const double* y = obs + (size_t)(obs_shared ? 0 : b) * (T + 1) * dy + (size_t)t * dy;
      for (int i = 0; i < dy; ++i) {
        double s = 0.0;
        for (int j = 0; j < dx; ++j) s += H[i * dx + j] * x[(size_t)t * dx + j];
        r[i] = y[i] - (s + cc[i]);
      }
      const int j = 1 + m.nQ + (m.nR > 1 ? t : 0);
      L = Ls + (size_t)j * W * W;
      ld = logdet[j];
    }
    double sq = 0.0;
    for (int i = 0; i < nn; ++i) {
      double s = r[i];
      for (int j = 0; j < i; ++j) s -= L[i * nn + j] * r[j];
      r[i] = s / L[i * nn + i];
      sq += r[i] * r[i];
    }
    terms[q] = -0.5 * (nn * kLog2Pi + sq) - ld;
  }
}

__global__ void k_path_sum(int T, int B, const double* terms, const uint8_t* mask, int dy,
                           const double* log_marginal, int fr_shared, const int* fst,
                           double* out, int* status) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const int K = 2 * T + 2;
  const double* tm = terms + (size_t)b * K;
  double lp = tm[0];
  for (int t = 0; t < T; ++t) lp += tm[1 + t];
  for (int t = 0; t <= T; ++t)
    if (dy > 0 && (mask == nullptr || mask[t])) lp += tm[T + 1 + t];
  out[b] = lp - log_marginal[fr_shared ? 0 : b];
  status[b] = *fst;
}

}  // namespace auxmc_gpu

using namespace auxmc_gpu;

extern "C" int auxmc_path_logpdf(const auxmc_lgssm* model, const double* obs, int obs_shared,
                                 const double* traj, const auxmc_filter_result* fr,
                                 int fr_shared, int B, double* out, int* status, void* stream) {
  if (!device_ok()) return AUXMC_E_CUDA;
  int st = check_model(model);
  if (st) return st;
  if (!traj || !fr || !fr->log_marginal || !out || !status || B < 0 || model->dx > 64 ||
      model->dy > 64)
    return AUXMC_E_ARG;
  if (B == 0) return AUXMC_OK;
  const DevModel dm = to_dev(*model);
  const int W = dm.dx > dm.dy ? dm.dx : dm.dy;
  const int n_mats = 1 + dm.nQ + (dm.dy > 0 ? dm.nR : 0);
  const int K = 2 * dm.T + 2;
  cudaStream_t s = (cudaStream_t)stream;
  double *Ls = nullptr, *logdet = nullptr, *terms = nullptr;
  int* fst = nullptr;
  AUXMC_CUDA_TRY(cudaMallocAsync(&Ls, sizeof(double) * n_mats * W * W, s));
  AUXMC_CUDA_TRY(cudaMallocAsync(&logdet, sizeof(double) * n_mats, s));
  AUXMC_CUDA_TRY(cudaMallocAsync(&terms, sizeof(double) * (size_t)B * K, s));
  AUXMC_CUDA_TRY(cudaMallocAsync(&fst, sizeof(int), s));
  AUXMC_CUDA_TRY(cudaMemsetAsync(fst, 0, sizeof(int), s));
  const int warps = 4;
  const size_t smem = sizeof(double) * (3 * W * W + 4) * warps;
  AUXMC_CUDA_TRY(cudaFuncSetAttribute(k_factor_list, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem));
  AUXMC_LAUNCH(k_factor_list, std::min((n_mats + warps - 1) / warps, 148 * 8), 32 * warps, smem,
               s, dm, Ls, logdet, fst);
  const long long n = (long long)B * K;
  AUXMC_LAUNCH(k_path_terms, (int)std::min<long long>((n + 127) / 128, 148LL * 64), 128, 0, s, dm,
               obs, obs_shared, traj, B, Ls, logdet, terms);
  AUXMC_LAUNCH(k_path_sum, (B + 127) / 128, 128, 0, s, dm.T, B, terms, dm.mask, dm.dy,
               fr->log_marginal, fr_shared, fst, out, status);
  cudaFreeAsync(Ls, s);
  cudaFreeAsync(logdet, s);
  cudaFreeAsync(terms, s);
  cudaFreeAsync(fst, s);
  return AUXMC_OK;
}
