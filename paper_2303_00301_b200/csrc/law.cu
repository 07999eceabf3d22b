// law.cu — exact laws on the device: the RTS smoother marginals
// (lgssm::rts_smoother, lgssm.cpp:114-127) and the induced Gaussian law of an
// affine-in-noise pathwise sampler (pit::extract_affine_law, pit.cpp:303-332).
//
// extract_affine_law pushes the zero noise and every basis noise vector through
// the sampler as one batch of B = 1 + n_noise pre-drawn problems (the noise is
// address-based, so each basis vector is a one-hot entry of (kTerminalDraw, 0),
// (kBackwardNoise, t) or (kDncBridge, id)); the law is N(x(0), A A^T) with
// A_k = x(e_k) - x(0).  The reference's ProbeNoise enumerates the same
// directions in call order; A A^T does not depend on the column order.
#include "common.cuh"
#include "group.cuh"

namespace auxmc_gpu {

int launch_bwd_elements(const DevModel& dm, const double* fm, const double* fc, const double* pc,
                        int Bfr, double* elems, double* term, int* st_fr, int store_cov,
                        cudaStream_t stream, int t_lo = 0, int t_hi = -1,
                        double* recs = nullptr, int* rep = nullptr);
int launch_sample_paths(const DevModel& dm, const auxmc_filter_result* fr, int fr_shared,
                        const auxmc_noise* noise, int B, int sampler, double* traj, int* status,
                        Arena& ws, cudaStream_t stream);

namespace {

// One warp per sequence, sequential in t (lgssm.cpp:117-126):
// m_t = G_t m_{t+1} + offset_t, P_t = symm(Lambda_t + G_t P_{t+1} G_t^T).
__global__ void k_rts(int T, int d, int B, const double* __restrict__ elems,
                      const double* __restrict__ filt_mean, const double* __restrict__ filt_cov,
                      double* mean, double* cov) {
  extern __shared__ double sm[];
  const int dd = d * d;
  Grp g = warp_group();
  const int b = blockIdx.x;
  if (b >= B) return;
  double* P = sm;          // P_{t+1}
  double* X = P + dd;
  double* Y = X + dd;
  double* m = Y + dd;      // m_{t+1}
  double* mo = m + d;
  double* ms = mean + (size_t)b * (T + 1) * d;
  double* cs = cov + (size_t)b * (T + 1) * dd;
  const double* fmT = filt_mean + ((size_t)b * (T + 1) + T) * d;
  const double* fcT = filt_cov + ((size_t)b * (T + 1) + T) * dd;
  for (int i = g.lane; i < dd; i += g.size) {  // Gaussian(filt_mean[T], filt_cov[T])
    const int r = i / d, c = i % d;
    P[i] = 0.5 * (fcT[r * d + c] + fcT[c * d + r]);
    cs[(size_t)T * dd + i] = P[i];
  }
  for (int i = g.lane; i < d; i += g.size) {
    m[i] = fmT[i];
    ms[(size_t)T * d + i] = m[i];
  }
  g.sync();
  const int es = elem_stride(d);
  for (int t = T - 1; t >= 0; --t) {
    const double* e = elems + ((size_t)b * T + t) * es;
    const double* G = e;
    const double* off = e + dd;
    const double* Lam = e + dd + d;
    for (int i = g.lane; i < d; i += g.size) {
      double s = 0.0;
      for (int j = 0; j < d; ++j) s += G[i * d + j] * m[j];
      mo[i] = s + off[i];
    }
    g_mm(g, d, d, d, G, P, X);      // G P_{t+1}
    g.sync();
    g_mm_nt(g, d, d, d, X, G, Y);   // (G P) G^T
    g.sync();
    for (int i = g.lane; i < dd; i += g.size) X[i] = Lam[i] + Y[i];
    g.sync();
    for (int i = g.lane; i < dd; i += g.size) {
      const int r = i / d, c = i % d;
      P[i] = 0.5 * (X[r * d + c] + X[c * d + r]);
      cs[(size_t)t * dd + i] = P[i];
    }
    for (int i = g.lane; i < d; i += g.size) {
      m[i] = mo[i];
      ms[(size_t)t * d + i] = mo[i];
    }
    g.sync();
  }
}

// basis noise: problem 0 is all zero, problem k + 1 has a single 1 at flat
// position k of (terminal | backward | bridge).
__global__ void k_basis_noise(int B, long long nt, long long nb, long long nr, double* terminal,
                              double* backward, double* bridge) {
  const long long per = nt + nb + nr;
  const long long n = (long long)B * per;
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (long long)gridDim.x * blockDim.x) {
    const long long p = q / per, k = q % per;
    const double v = (p >= 1 && k == p - 1) ? 1.0 : 0.0;
    if (k < nt) terminal[p * nt + k] = v;
    else if (k < nt + nb) backward[p * nb + (k - nt)] = v;
    else bridge[p * nr + (k - nt - nb)] = v;
  }
}

// cov[i][j] = sum_k (x_{k+1}[i] - x_0[i]) (x_{k+1}[j] - x_0[j]), 32×32 output tiles,
// k in ascending order; then symmetrized as the Gaussian constructor does.
__global__ void k_gram(int n, int K, const double* __restrict__ traj, double* cov) {
  __shared__ double a[32][33], bsh[32][33];
  const int ti = blockIdx.y * 32, tj = blockIdx.x * 32;
  const int ly = threadIdx.y, lx = threadIdx.x;  // 32 × 8 threads, 4 rows each
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int k0 = 0; k0 < K; k0 += 32) {
    for (int r = ly; r < 32; r += 8) {
      const int k = k0 + r;
      const int i = ti + lx, j = tj + lx;
      a[r][lx] = (k < K && i < n) ? traj[(size_t)(k + 1) * n + i] - traj[i] : 0.0;
      bsh[r][lx] = (k < K && j < n) ? traj[(size_t)(k + 1) * n + j] - traj[j] : 0.0;
    }
    __syncthreads();
    for (int r = 0; r < 32; ++r) {
      const double bv = bsh[r][lx];
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[q] = fma(a[r][ly + 8 * q], bv, acc[q]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int i = ti + ly + 8 * q, j = tj + lx;
    if (i < n && j < n) cov[(size_t)i * n + j] = acc[q];
  }
}

__global__ void k_symm_full(int n, double* cov) {
  const long long nn = (long long)n * n;
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < nn;
       q += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(q / n), j = (int)(q % n);
    if (j <= i) continue;
    const double v = 0.5 * (cov[(size_t)i * n + j] + cov[(size_t)j * n + i]);
    cov[(size_t)i * n + j] = v;
    cov[(size_t)j * n + i] = v;
  }
}

__global__ void k_max_status(int B, const int* st, int* out) {
  __shared__ int m;
  if (threadIdx.x == 0) m = 0;
  __syncthreads();
  int v = 0;
  for (int i = threadIdx.x; i < B; i += blockDim.x) v = st[i] > v ? st[i] : v;
  atomicMax(&m, v);
  __syncthreads();
  if (threadIdx.x == 0) *out = m;
}

int rts(const DevModel& dm, const auxmc_filter_result* fr, int B, double* mean, double* cov,
        int* status, Arena& ws, cudaStream_t s) {
  const int T = dm.T, d = dm.dx;
  double* elems = ws.take<double>((size_t)B * (T > 0 ? T : 1) * elem_stride(d));
  double* term = ws.take<double>((size_t)B * term_stride(d));
  if (ws.base == nullptr) return AUXMC_OK;
  if (!elems || !term) return AUXMC_E_WORKSPACE;
  AUXMC_CUDA_TRY(cudaMemsetAsync(status, 0, sizeof(int) * B, s));
  int rc = launch_bwd_elements(dm, fr->filt_mean, fr->filt_cov, fr->pred_cov, B, elems, term,
                               status, 1, s);
  if (rc) return rc;
  const size_t smem = sizeof(double) * (3 * d * d + 2 * d);
  AUXMC_CUDA_TRY(cudaFuncSetAttribute(k_rts, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem));
  AUXMC_LAUNCH(k_rts, B, 32, smem, s, T, d, B, elems, fr->filt_mean, fr->filt_cov, mean, cov);
  return AUXMC_OK;
}

int affine_law(const DevModel& dm, const auxmc_filter_result* fr, int sampler, double* mean,
               double* cov, int* status, Arena& ws, cudaStream_t s) {
  const int T = dm.T, d = dm.dx;
  const long long n = (long long)(T + 1) * d;
  const long long nt = d, nb = (long long)T * d;
  const long long nbr = sampler == AUXMC_SAMPLER_DNC ? auxmc_dnc_bridge_count(T) : 0;
  const long long nr = nbr * d;
  const int B = (int)(1 + nt + nb + nr);
  double* terminal = ws.take<double>((size_t)B * nt);
  double* backward = ws.take<double>((size_t)B * (nb > 0 ? nb : 1));
  double* bridge = ws.take<double>((size_t)B * (nr > 0 ? nr : 1));
  double* traj = ws.take<double>((size_t)B * n);
  int* st = ws.take<int>((size_t)B);
  auxmc_noise nz{};
  nz.kind = AUXMC_NOISE_PREDRAWN;
  nz.terminal = terminal;
  nz.backward = backward;
  nz.bridge = nr > 0 ? bridge : nullptr;
  nz.n_bridge = nbr;
  if (ws.base == nullptr) {
    launch_sample_paths(dm, fr, 1, &nz, B, sampler, nullptr, nullptr, ws, s);
    return AUXMC_OK;
  }
  if (!terminal || !backward || !bridge || !traj || !st) return AUXMC_E_WORKSPACE;
  const long long tot = (long long)B * (nt + nb + nr);
  AUXMC_LAUNCH(k_basis_noise, (int)std::min<long long>((tot + 255) / 256, 148LL * 32), 256, 0, s,
               B, nt, nb, nr, terminal, backward, bridge);
  int rc = launch_sample_paths(dm, fr, 1, &nz, B, sampler, traj, st, ws, s);
  if (rc) return rc;
  AUXMC_CUDA_TRY(cudaMemcpyAsync(mean, traj, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
  const dim3 grid((unsigned)((n + 31) / 32), (unsigned)((n + 31) / 32));
  AUXMC_LAUNCH(k_gram, grid, dim3(32, 8), 0, s, (int)n, B - 1, traj, cov);
  AUXMC_LAUNCH(k_symm_full, (int)std::min<long long>((n * n + 255) / 256, 148LL * 32), 256, 0, s,
               (int)n, cov);
  // per-problem sampler status, reduced into status[0]
  AUXMC_LAUNCH(k_max_status, 1, 256, 0, s, B, st, status);
  return AUXMC_OK;
}

}  // namespace
}  // namespace auxmc_gpu

using namespace auxmc_gpu;

extern "C" {

size_t auxmc_rts_smoother_workspace(const auxmc_lgssm* model, int B) {
  if (check_model(model) || B < 0) return 0;
  Arena ws{nullptr, 0, 0};
  rts(to_dev(*model), nullptr, B, nullptr, nullptr, nullptr, ws, nullptr);
  return ws.used + 1024;
}

int auxmc_rts_smoother(const auxmc_lgssm* model, const auxmc_filter_result* fr, int B,
                       double* mean, double* cov, int* status, void* workspace,
                       size_t workspace_bytes, void* stream) {
  if (!device_ok()) return AUXMC_E_CUDA;
  int st = check_model(model);
  if (st) return st;
  if (!fr || !fr->filt_mean || !fr->filt_cov || !fr->pred_cov || !mean || !cov || !status ||
      B < 0 || model->dx > 64)
    return AUXMC_E_ARG;
  if (B == 0) return AUXMC_OK;
  if (!workspace) return AUXMC_E_WORKSPACE;
  Arena ws{(char*)workspace, workspace_bytes, 0};
  return rts(to_dev(*model), fr, B, mean, cov, status, ws, (cudaStream_t)stream);
}

size_t auxmc_affine_law_workspace(const auxmc_lgssm* model, int sampler) {
  if (check_model(model) || sampler < 0 || sampler > 2) return 0;
  Arena ws{nullptr, 0, 0};
  affine_law(to_dev(*model), nullptr, sampler, nullptr, nullptr, nullptr, ws, nullptr);
  return ws.used + 4096;
}

int auxmc_affine_law(const auxmc_lgssm* model, const auxmc_filter_result* fr, int sampler,
                     double* mean, double* cov, int* status, void* workspace,
                     size_t workspace_bytes, void* stream) {
  if (!device_ok()) return AUXMC_E_CUDA;
  int st = check_model(model);
  if (st) return st;
  if (!fr || !fr->filt_mean || !fr->filt_cov || !fr->pred_cov || !mean || !cov || !status ||
      sampler < 0 || sampler > 2)
    return AUXMC_E_ARG;
  if (!workspace) return AUXMC_E_WORKSPACE;
  Arena ws{(char*)workspace, workspace_bytes, 0};
  return affine_law(to_dev(*model), fr, sampler, mean, cov, status, ws, (cudaStream_t)stream);
}

}  // extern "C"
