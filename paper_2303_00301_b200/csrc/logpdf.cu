// logpdf.cu — lgssm::path_logpdf (lgssm.cpp:179-199) for batches of paths.
//
// Every covariance the reference factors inside a log_pdf call (P0, Q_t, R_t;
// gauss.cpp:51-57) is path-independent, so each distinct matrix is factored
// once (jitter ladder included) and reused by all paths.  Per-(path, term)
// Mahalanobis terms run one per thread; each path then sums its terms in the
// reference's order (prior, transitions t = 0..T-1, observations t = 0..T).
#include "common.cuh"
#include "dense.cuh"
#include "terms.cuh"

namespace auxmc_gpu {

// Factor matrix j of a list: P0 (j = 0), then Q sets (nQb of nQ matrices),
// then R sets (nRb of nR); a set per problem when that array is batch-strided.
__global__ void k_factor_list(DevModel m, int nQb, int nRb, double* Ls, double* logdet,
                              unsigned char* dg, int* status) {
  extern __shared__ double smem[];
  const int dx = m.dx, dy = m.dy;
  const int nq = nQb * m.nQ;
  const int n_items = 1 + nq + (dy > 0 ? nRb * m.nR : 0);
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
    else if (j <= nq) {
      const int k = (j - 1) / m.nQ, i = (j - 1) % m.nQ;
      src = m.Q + (size_t)k * m.sQ + (size_t)i * dx * dx;
      n = dx;
    } else {
      const int k = (j - 1 - nq) / m.nR, i = (j - 1 - nq) % m.nR;
      src = m.R + (size_t)k * m.sR + (size_t)i * dy * dy;
      n = dy;
    }
    for (int i = g.lane; i < n * n; i += g.size) {
      const int r = i / n, c = i % n;
      A[i] = (src[r * n + c] + src[c * n + r]) * 0.5;
    }
    g.sync();
    const int st = g_factor_psd(g, n, A, L, scr, flag, red);
    double* out = Ls + (size_t)j * W * W;
    for (int i = g.lane; i < n * n; i += g.size) out[i] = L[i];
    bool off = false;  // any nonzero below the diagonal
    for (int i = g.lane; i < n * n; i += g.size) off = off || (i % n < i / n && L[i] != 0.0);
    off = __any_sync(0xffffffffu, off);
    if (g.lane == 0) {
      double ld = 0.0;
      for (int i = 0; i < n; ++i) ld += log(L[i * n + i]);
      logdet[j] = ld;
      if (dg) dg[j] = off ? 0 : 1;
      if (st) atomicMax(status, st);
    }
    g.sync();
  }
}

// per row of every H_t: the single nonzero column, -1 for a zero row, -2 otherwise
__global__ void k_row_sparsity(DevModel m, int* hsel) {
  const long long n = (long long)m.nH * m.dy;
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (long long)gridDim.x * blockDim.x) {
    const int t = (int)(q / m.dy), i = (int)(q % m.dy);
    const double* H = m.H + (size_t)t * m.dy * m.dx + (size_t)i * m.dx;
    int col = -1;
    for (int j = 0; j < m.dx; ++j)
      if (H[j] != 0.0) col = col == -1 ? j : -2;
    hsel[q] = col;
  }
}

// term index k: 0 prior; 1..T transition t=k-1; T+1..2T+1 observation t=k-T-1.
__global__ void k_path_terms(DevModel m, const double* __restrict__ obs, long long obs_stride,
                             const double* __restrict__ traj, int B, const double* __restrict__ Ls,
                             const double* __restrict__ logdet,
                             const unsigned char* __restrict__ dg,
                             const int* __restrict__ hsel, double* terms) {
  const int T = m.T;
  const int K = 2 * T + 2;
  const long long n = (long long)B * K;
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (long long)gridDim.x * blockDim.x) {
    const int b = (int)(q / K), k = (int)(q % K);
    terms[q] = path_term_k(m, obs + (size_t)b * obs_stride, traj + (size_t)b * (T + 1) * m.dx, b, B,
                           Ls, logdet, k, dg, hsel);
  }
}

// the path density's terms: T + 1 transition terms, then the observation terms of
// the observed steps
struct PathTerms {
  const double* terms;
  int T, dy;
  const uint8_t* mask;
  __device__ double operator()(int b, long long i) const {
    const double* tm = terms + (size_t)b * (2LL * T + 2);
    if (i <= T) return tm[i];
    const long long t = i - T - 1;
    return (dy > 0 && (mask == nullptr || mask[t])) ? tm[i] : 0.0;
  }
};

__global__ void k_path_sum(int T, int B, const double* terms, const uint8_t* mask, int dy,
                           const double* log_marginal, int fr_shared, const int* fst,
                           double* out, int* status, const double* parts) {
  __shared__ double red[kSumThreads];
  const int b = blockIdx.x;
  const long long K = 2LL * T + 2;
  const PathTerms pt{terms, T, dy, mask};
  const double lp = cta_sum_fixed(K, [&](long long i) { return pt(b, i); }, red,
                                  parts ? parts + (size_t)b * kSumThreads : nullptr);
  if (threadIdx.x == 0) {
    out[b] = lp - log_marginal[fr_shared ? 0 : b];
    status[b] = *fst;
  }
}

}  // namespace auxmc_gpu

namespace auxmc_gpu {

int launch_path_logpdf(const DevModel& dm, const double* obs, long long obs_stride,
                       const double* traj, const double* log_marginal, int lm_shared, int B,
                       double* out, int* status, cudaStream_t s) {
  const int W = dm.dx > dm.dy ? dm.dx : dm.dy;
  const int nQb = dm.sQ ? B : 1, nRb = dm.sR ? B : 1;
  const int n_mats = 1 + nQb * dm.nQ + (dm.dy > 0 ? nRb * dm.nR : 0);
  const int K = 2 * dm.T + 2;
  double *Ls = nullptr, *logdet = nullptr, *terms = nullptr;
  int* fst = nullptr;
  unsigned char* dg = nullptr;
  int* hsel = nullptr;
  const bool rows = dm.dy > 0 && dm.sH == 0;  // H shared by the batch
  AUXMC_CUDA_TRY(cudaMallocAsync(&dg, n_mats, s));
  if (rows) AUXMC_CUDA_TRY(cudaMallocAsync(&hsel, sizeof(int) * (size_t)dm.nH * dm.dy, s));
  AUXMC_CUDA_TRY(cudaMallocAsync(&Ls, sizeof(double) * n_mats * W * W, s));
  AUXMC_CUDA_TRY(cudaMallocAsync(&logdet, sizeof(double) * n_mats, s));
  AUXMC_CUDA_TRY(cudaMallocAsync(&terms, sizeof(double) * (size_t)B * K, s));
  AUXMC_CUDA_TRY(cudaMallocAsync(&fst, sizeof(int), s));
  AUXMC_CUDA_TRY(cudaMemsetAsync(fst, 0, sizeof(int), s));
  const int warps = factor_warps(W);
  const size_t smem = sizeof(double) * (3 * W * W + 4) * warps;
  AUXMC_CUDA_TRY(cudaFuncSetAttribute(k_factor_list, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem));
  AUXMC_LAUNCH(k_factor_list, std::min((n_mats + warps - 1) / warps, 148 * 8), 32 * warps, smem,
               s, dm, nQb, nRb, Ls, logdet, dg, fst);
  if (rows)
    AUXMC_LAUNCH(k_row_sparsity, (int)std::min<long long>(((long long)dm.nH * dm.dy + 127) / 128,
                                                         148LL * 16),
                 128, 0, s, dm, hsel);
  const long long n = (long long)B * K;
  AUXMC_LAUNCH(k_path_terms, (int)std::min<long long>((n + 127) / 128, 148LL * 64), 128, 0, s, dm,
               obs, obs_stride, traj, B, Ls, logdet, dg, hsel, terms);
  double* parts = nullptr;
  if (sum_parts_pay(B, 2LL * dm.T + 2)) {
    AUXMC_CUDA_TRY(cudaMallocAsync(&parts, sizeof(double) * B * kSumThreads, s));
    AUXMC_LAUNCH(k_sum_parts<PathTerms>, (B * kSumThreads + 7) / 8, 256, 0, s, B,
                 2LL * dm.T + 2, (PathTerms{terms, dm.T, dm.dy, dm.mask}), parts);
  }
  AUXMC_LAUNCH(k_path_sum, B, kSumThreads, 0, s, dm.T, B, terms, dm.mask, dm.dy,
               log_marginal, lm_shared, fst, out, status, parts);
  if (parts) cudaFreeAsync(parts, s);
  cudaFreeAsync(Ls, s);
  cudaFreeAsync(logdet, s);
  cudaFreeAsync(terms, s);
  cudaFreeAsync(fst, s);
  cudaFreeAsync(dg, s);
  if (hsel) cudaFreeAsync(hsel, s);
  return AUXMC_OK;
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
  return launch_path_logpdf(dm, obs, obs_shared ? 0 : (long long)(dm.T + 1) * dm.dy, traj,
                            fr->log_marginal, fr_shared, B, out, status, (cudaStream_t)stream);
}
