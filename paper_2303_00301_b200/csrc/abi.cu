// abi.cu — C ABI entry points (include/auxmc_gpu.h) for filtering and pathwise
// sampling.  Argument checking mirrors the reference's require_dim contracts
// (lgssm.cpp:20-71, :78-79); per-item failures land in status arrays.
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"
#include "dense.cuh"
#include "rng.cuh"

namespace auxmc_gpu {

std::atomic<unsigned long long> g_launches{0};
std::atomic<int> g_prof_on{0};
static thread_local std::string g_last_error;

struct ProfRecord {
  std::string name;
  cudaEvent_t begin, end;
};
static std::mutex g_prof_mu;
static std::vector<ProfRecord> g_prof;
static std::vector<cudaEvent_t> g_prof_pool;

static cudaEvent_t prof_event() {
  if (!g_prof_pool.empty()) {
    cudaEvent_t e = g_prof_pool.back();
    g_prof_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

__global__ void k_seq_sum(const double* v, int n, double* out) {  // in index order
  double s = 0.0;
  for (int i = 0; i < n; ++i) s += v[i];
  *out = s;
}

void prof_mark(const char* name, cudaStream_t s, bool begin) {
  std::lock_guard<std::mutex> lock(g_prof_mu);
  if (begin) {
    ProfRecord r{name, prof_event(), prof_event()};
    cudaEventRecord(r.begin, s);
    g_prof.push_back(r);
  } else if (!g_prof.empty()) {
    cudaEventRecord(g_prof.back().end, s);
  }
}

void set_last_error(const char* where, cudaError_t e) {
  g_last_error = std::string(where) + ": " + cudaGetErrorString(e);
}

bool device_ok() {
  static int ok = -1;
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  if (ok < 0) {
    int n = 0;
    ok = 0;
    if (cudaGetDeviceCount(&n) == cudaSuccess && n > 0) {
      int dev = 0;
      cudaDeviceProp prop;
      if (cudaGetDevice(&dev) == cudaSuccess && cudaGetDeviceProperties(&prop, dev) == cudaSuccess)
        ok = prop.major == 10 ? 1 : 0;
    }
    cudaGetLastError();
  }
  return ok == 1;
}

int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

int check_model(const auxmc_lgssm* m) {
  if (m == nullptr) return AUXMC_E_ARG;
  if (m->T < 0 || m->dx < 1 || m->dy < 0) return AUXMC_E_DIM;
  auto ok = [](int got, int n) { return got == n || got == 1 || (n == 0 && got <= 1); };
  if (!ok(m->nF, m->T) || !ok(m->nb, m->T) || !ok(m->nQ, m->T)) return AUXMC_E_DIM;
  if (m->dy > 0 && (!ok(m->nH, m->T + 1) || !ok(m->nc, m->T + 1) || !ok(m->nR, m->T + 1)))
    return AUXMC_E_DIM;
  if (!m->m0 || !m->P0 || !m->F || !m->b || !m->Q) return AUXMC_E_ARG;
  if (m->dy > 0 && (!m->H || !m->c || !m->R)) return AUXMC_E_ARG;
  return AUXMC_OK;
}

// forward decls from other translation units
int launch_filter_seq(const DevModel& dm, const double* obs, int B, auxmc_filter_result* out,
                      int* status, cudaStream_t stream);
int launch_filter_pit(const DevModel& dm, const double* obs, int B, auxmc_filter_result* out,
                      int* status, Arena& ws, cudaStream_t stream);
size_t filter_pit_workspace(const DevModel& dm, int B);
int tshard_geometry(int T, int* LB, int* nblk, int* nsup, int* SB);
int tshard_filter_local(const DevModel& dm, const double* obs, int j_lo, int j_hi, Arena& ws,
                        double* sup_out, int* status, cudaStream_t s);
int tshard_filter_finish(const DevModel& dm, const double* obs, int j_lo, int j_hi, Arena& ws,
                         const double* sup_all, auxmc_filter_result* out, double* ll_out,
                         int* status, cudaStream_t s);
int tshard_elem_doubles(int dx);
int tshard_prefix_geometry(int T, int* Lb, int* P);
size_t tshard_prefix_workspace(const DevModel& dm);
int tshard_prefix_local(const DevModel& dm, const double* fm, const double* fc, const double* pc,
                        const NoiseArgs& nz, int t_lo, int t_hi, Arena& ws, double* blk_out,
                        double* xT_out, double* traj, int* status, cudaStream_t stream);
int tshard_prefix_finish(const DevModel& dm, const NoiseArgs& nz, int t_lo, int t_hi, Arena& ws,
                         const double* blk_all, const double* xT, double* traj,
                         cudaStream_t stream);
int launch_sample_paths(const DevModel& dm, const auxmc_filter_result* fr, int fr_shared,
                        const auxmc_noise* noise, int B, int sampler, double* traj, int* status,
                        Arena& ws, cudaStream_t stream);

__global__ void k_normals(const uint64_t* keys, int B, uint64_t label, uint64_t index0,
                          int n_index, int dim, double* out) {
  const long long n = (long long)B * n_index * dim;
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(q % dim);
    const long long r = q / dim;
    const int i = (int)(r % n_index);
    const int b = (int)(r / n_index);
    const uint64_t k = derive(keys[b], label, index0 + (uint64_t)i);
    out[q] = normal_at(k, (uint64_t)j);
  }
}

}  // namespace auxmc_gpu

using namespace auxmc_gpu;

extern "C" {

const char* auxmc_version(void) { return "0.1.0"; }

const char* auxmc_status_string(int s) {
  switch (s) {
    case AUXMC_OK: return "ok";
    case AUXMC_E_DIM: return "dimension error";
    case AUXMC_E_FACTOR: return "covariance not positive definite after jitter";
    case AUXMC_E_DEGENERATE: return "all particle weights degenerate";
    case AUXMC_E_CONTRACT: return "contract violation";
    case AUXMC_E_CONFIG: return "configuration error";
    case AUXMC_E_CUDA: return "CUDA error";
    case AUXMC_E_ARG: return "invalid argument";
    case AUXMC_E_WORKSPACE: return "workspace too small";
  }
  return "unknown status";
}

int auxmc_device_ok(void) { return device_ok() ? 1 : 0; }

void auxmc_profile_begin(void) {
  std::lock_guard<std::mutex> lock(g_prof_mu);
  for (auto& r : g_prof) {
    g_prof_pool.push_back(r.begin);
    g_prof_pool.push_back(r.end);
  }
  g_prof.clear();
  g_prof_on.store(1);
}

int auxmc_profile_end(const char* kernel_substr, double* total_ms, long long* count) {
  g_prof_on.store(0);
  std::lock_guard<std::mutex> lock(g_prof_mu);
  double tot = 0.0;
  long long n = 0;
  for (auto& r : g_prof) {
    if (kernel_substr && std::strstr(r.name.c_str(), kernel_substr) == nullptr) continue;
    if (cudaEventSynchronize(r.end) != cudaSuccess) return AUXMC_E_CUDA;
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, r.begin, r.end) != cudaSuccess) return AUXMC_E_CUDA;
    tot += ms;
    ++n;
  }
  if (total_ms) *total_ms = tot;
  if (count) *count = n;
  return AUXMC_OK;
}
const char* auxmc_last_error(void) { return g_last_error.c_str(); }
unsigned long long auxmc_launch_count(void) { return g_launches.load(); }

uint64_t auxmc_rng_from_seed(uint64_t seed) { return seed_key(seed); }
uint64_t auxmc_rng_derive(uint64_t key, uint64_t label, uint64_t index) {
  return derive(key, label, index);
}
double auxmc_rng_uniform(uint64_t key, uint64_t counter) { return uniform_at(key, counter); }
double auxmc_rng_normal(uint64_t key, uint64_t counter) {
  const double u1 = to_unit_open(word_at(key, 2 * counter));
  const double u2 = to_unit_open(word_at(key, 2 * counter + 1));
  return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586476925286766559 * u2);
}

int auxmc_rng_normals(const uint64_t* keys, int B, uint64_t label, uint64_t index0, int n_index,
                      int dim, double* out, void* stream) {
  if (!device_ok()) return AUXMC_E_CUDA;
  if (!keys || !out || B < 0 || n_index < 0 || dim < 0) return AUXMC_E_ARG;
  const long long n = (long long)B * n_index * dim;
  if (n == 0) return AUXMC_OK;
  const int grid = (int)std::min<long long>((n + 255) / 256, 148LL * 16);
  AUXMC_LAUNCH(k_normals, grid, 256, 0, stream, keys, B, label, index0, n_index, dim, out);
  return AUXMC_OK;
}

// One or two very long sequences: the sequential recurrence would run on one thread
// (T = 2^16 at d = 4 took 832 ms), so kalman_filter runs the reference's own
// parallel_filter algorithm (pit.cpp:117-188) for them — the same moments and
// log-likelihood up to FP rounding (tests/test_gpu_lgssm.py long-horizon case, 1e-8).
static bool seq_as_scan(const auxmc_lgssm& m, int B) {
  return B <= 2 && m.T >= 4096 && m.dx <= 32 && m.dy <= 64;
}

size_t auxmc_kalman_filter_workspace(const auxmc_lgssm* model, int B, int mode) {
  if (!model) return 0;
  if (mode == 1 || (mode == 0 && seq_as_scan(*model, B))) return filter_pit_workspace(to_dev(*model), B);
  return 0;
}

int auxmc_kalman_filter(const auxmc_lgssm* model, const double* obs, int B, int mode,
                        auxmc_filter_result* out, int* status, void* workspace,
                        size_t workspace_bytes, void* stream) {
  if (!device_ok()) return AUXMC_E_CUDA;
  int st = check_model(model);
  if (st) return st;
  if (!out || !status || (model->dy > 0 && !obs) || B < 0) return AUXMC_E_ARG;
  if (B == 0) return AUXMC_OK;
  const DevModel dm = to_dev(*model);
  if (mode == 0 && !(seq_as_scan(*model, B) && workspace &&
                     workspace_bytes >= filter_pit_workspace(dm, B)))
    return launch_filter_seq(dm, obs, B, out, status, (cudaStream_t)stream);
  if (mode == 0 || mode == 1) {
    Arena ws{(char*)workspace, workspace_bytes, 0};
    return launch_filter_pit(dm, obs, B, out, status, ws, (cudaStream_t)stream);
  }
  return AUXMC_E_ARG;
}

int auxmc_tshard_geometry(int T, int dx, int* LB, int* nblk, int* nsup, int* SB,
                          int* elem_doubles) {
  if (T < 0 || dx < 1 || !LB || !nblk || !nsup || !SB || !elem_doubles) return AUXMC_E_ARG;
  tshard_geometry(T, LB, nblk, nsup, SB);
  *elem_doubles = tshard_elem_doubles(dx);
  return AUXMC_OK;
}

size_t auxmc_tshard_filter_workspace(const auxmc_lgssm* model) {
  if (!model) return 0;
  Arena ws{nullptr, 0, 0};
  tshard_filter_local(to_dev(*model), nullptr, 0, 1, ws, nullptr, nullptr, nullptr);
  return ws.used + 1024;
}

int auxmc_tshard_filter_local(const auxmc_lgssm* model, const double* obs, int sup_lo,
                              int sup_hi, void* workspace, size_t workspace_bytes,
                              double* sup_out, int* status, void* stream) {
  if (!device_ok()) return AUXMC_E_CUDA;
  int st = check_model(model);
  if (st) return st;
  if (!sup_out || !status || (model->dy > 0 && !obs) || !workspace) return AUXMC_E_ARG;
  AUXMC_CUDA_TRY(cudaMemsetAsync(status, 0, sizeof(int), (cudaStream_t)stream));
  Arena ws{(char*)workspace, workspace_bytes, 0};
  return tshard_filter_local(to_dev(*model), obs, sup_lo, sup_hi, ws, sup_out, status,
                             (cudaStream_t)stream);
}

int auxmc_tshard_filter_finish(const auxmc_lgssm* model, const double* obs, int sup_lo,
                               int sup_hi, void* workspace, size_t workspace_bytes,
                               const double* sup_all, auxmc_filter_result* out, double* ll_out,
                               int* status, void* stream) {
  if (!device_ok()) return AUXMC_E_CUDA;
  int st = check_model(model);
  if (st) return st;
  if (!sup_all || !out || !ll_out || !status || (model->dy > 0 && !obs) || !workspace)
    return AUXMC_E_ARG;
  Arena ws{(char*)workspace, workspace_bytes, 0};
  return tshard_filter_finish(to_dev(*model), obs, sup_lo, sup_hi, ws, sup_all, out, ll_out,
                              status, (cudaStream_t)stream);
}

int auxmc_tshard_sum(const double* partials, int n, double* out, void* stream) {
  if (!device_ok()) return AUXMC_E_CUDA;
  if (!partials || !out || n < 0) return AUXMC_E_ARG;
  AUXMC_LAUNCH(k_seq_sum, 1, 1, 0, stream, partials, n, out);
  return AUXMC_OK;
}

static NoiseArgs noise_args(const auxmc_noise* noise) {
  NoiseArgs nz{};
  nz.kind = noise->kind;
  nz.keys = noise->keys;
  nz.terminal = noise->terminal;
  nz.backward = noise->backward;
  nz.bridge = noise->bridge;
  nz.n_bridge = noise->n_bridge;
  return nz;
}

int auxmc_tshard_prefix_geometry(int T, int* Lb, int* P) {
  if (T < 0 || !Lb || !P) return AUXMC_E_ARG;
  return tshard_prefix_geometry(T, Lb, P);
}

size_t auxmc_tshard_prefix_workspace(const auxmc_lgssm* model) {
  if (!model) return 0;
  return tshard_prefix_workspace(to_dev(*model));
}

int auxmc_tshard_prefix_local(const auxmc_lgssm* model, const auxmc_filter_result* fr,
                              const auxmc_noise* noise, int t_lo, int t_hi, void* workspace,
                              size_t workspace_bytes, double* blk_out, double* xT_out,
                              double* traj, int* status, void* stream) {
  if (!device_ok()) return AUXMC_E_CUDA;
  int st = check_model(model);
  if (st) return st;
  if (!fr || !noise || !blk_out || !xT_out || !traj || !status || !workspace) return AUXMC_E_ARG;
  if (noise->kind == AUXMC_NOISE_STREAM ? !noise->keys
                                        : (!noise->terminal || (model->T > 0 && !noise->backward)))
    return AUXMC_E_ARG;
  Arena ws{(char*)workspace, workspace_bytes, 0};
  return tshard_prefix_local(to_dev(*model), fr->filt_mean, fr->filt_cov, fr->pred_cov,
                             noise_args(noise), t_lo, t_hi, ws, blk_out, xT_out, traj, status,
                             (cudaStream_t)stream);
}

int auxmc_tshard_prefix_finish(const auxmc_lgssm* model, const auxmc_noise* noise, int t_lo,
                               int t_hi, void* workspace, size_t workspace_bytes,
                               const double* blk_all, const double* xT, double* traj,
                               void* stream) {
  if (!device_ok()) return AUXMC_E_CUDA;
  int st = check_model(model);
  if (st) return st;
  if (!noise || !blk_all || !xT || !traj || !workspace) return AUXMC_E_ARG;
  Arena ws{(char*)workspace, workspace_bytes, 0};
  return tshard_prefix_finish(to_dev(*model), noise_args(noise), t_lo, t_hi, ws, blk_all, xT,
                              traj, (cudaStream_t)stream);
}

int auxmc_copy_device(void* dst, const void* src, size_t bytes, void* stream) {
  if (!device_ok()) return AUXMC_E_CUDA;
  if ((!dst || !src) && bytes) return AUXMC_E_ARG;
  AUXMC_CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, (cudaStream_t)stream));
  return AUXMC_OK;
}

long long auxmc_dnc_bridge_count(int T) {
  long long cap = 1;
  while (cap < T) cap <<= 1;  // internal heap ids are < 2^ceil(log2 T)
  return cap < 2 ? 2 : cap;
}

size_t auxmc_sample_paths_workspace(const auxmc_lgssm* model, int fr_shared, int B,
                                    int sampler) {
  if (!model) return 0;
  Arena ws{nullptr, 0, 0};
  launch_sample_paths(to_dev(*model), nullptr, fr_shared, nullptr, B, sampler, nullptr, nullptr,
                      ws, nullptr);
  return ws.used + 1024;
}

int auxmc_sample_paths(const auxmc_lgssm* model, const auxmc_filter_result* fr, int fr_shared,
                       const auxmc_noise* noise, int B, int sampler, double* traj, int* status,
                       void* workspace, size_t workspace_bytes, void* stream) {
  if (!device_ok()) return AUXMC_E_CUDA;
  int st = check_model(model);
  if (st) return st;
  if (!fr || !noise || !traj || !status || B < 0) return AUXMC_E_ARG;
  if (!fr->filt_mean || !fr->filt_cov || !fr->pred_cov) return AUXMC_E_ARG;
  if (noise->kind == AUXMC_NOISE_STREAM && !noise->keys) return AUXMC_E_ARG;
  if (noise->kind == AUXMC_NOISE_PREDRAWN &&
      (!noise->terminal || (model->T > 0 && !noise->backward)))
    return AUXMC_E_ARG;
  // DnC with pre-drawn variates needs the bridge draws (one row per heap id)
  if (noise->kind == AUXMC_NOISE_PREDRAWN && sampler == AUXMC_SAMPLER_DNC && model->T > 1 &&
      (!noise->bridge || noise->n_bridge < auxmc_dnc_bridge_count(model->T)))
    return AUXMC_E_ARG;
  if (B == 0) return AUXMC_OK;
  if (!workspace) return AUXMC_E_WORKSPACE;
  Arena ws{(char*)workspace, workspace_bytes, 0};
  return launch_sample_paths(to_dev(*model), fr, fr_shared, noise, B, sampler, traj, status, ws,
                             (cudaStream_t)stream);
}

int auxmc_sample_paths_host(const auxmc_lgssm* mh, const auxmc_filter_result* frh, int fr_shared,
                            const uint64_t* keys_host, int B, int sampler, double* traj_host,
                            int* status_host) {
  if (!device_ok()) return AUXMC_E_CUDA;
  int st = check_model(mh);
  if (st) return st;
  if (!frh || !keys_host || !traj_host || !status_host || B <= 0) return AUXMC_E_ARG;
  const int T = mh->T, dx = mh->dx, dy = mh->dy;
  const int Bfr = fr_shared ? 1 : B;
  std::vector<void*> allocs;
  auto up = [&](const void* src, size_t bytes) -> void* {
    void* p = nullptr;
    if (bytes == 0 || src == nullptr) return nullptr;
    if (cudaMalloc(&p, bytes) != cudaSuccess) return nullptr;
    allocs.push_back(p);
    cudaMemcpy(p, src, bytes, cudaMemcpyHostToDevice);
    return p;
  };
  auxmc_lgssm m = *mh;
  m.m0 = (const double*)up(mh->m0, sizeof(double) * dx);
  m.P0 = (const double*)up(mh->P0, sizeof(double) * dx * dx);
  m.F = (const double*)up(mh->F, sizeof(double) * dx * dx * mh->nF);
  m.b = (const double*)up(mh->b, sizeof(double) * dx * mh->nb);
  m.Q = (const double*)up(mh->Q, sizeof(double) * dx * dx * mh->nQ);
  m.H = (const double*)up(mh->H, sizeof(double) * dy * dx * mh->nH);
  m.c = (const double*)up(mh->c, sizeof(double) * dy * mh->nc);
  m.R = (const double*)up(mh->R, sizeof(double) * dy * dy * mh->nR);
  m.mask = (const uint8_t*)up(mh->mask, mh->mask ? (size_t)(T + 1) : 0);
  auxmc_filter_result fr{};
  const size_t nm = (size_t)Bfr * (T + 1) * dx, nc = nm * dx;
  fr.filt_mean = (double*)up(frh->filt_mean, sizeof(double) * nm);
  fr.filt_cov = (double*)up(frh->filt_cov, sizeof(double) * nc);
  fr.pred_cov = (double*)up(frh->pred_cov, sizeof(double) * nc);
  auxmc_noise nz{};
  nz.kind = AUXMC_NOISE_STREAM;
  nz.keys = (const uint64_t*)up(keys_host, sizeof(uint64_t) * B);
  double* traj = nullptr;
  int* status = nullptr;
  void* ws = nullptr;
  const size_t wsb = auxmc_sample_paths_workspace(&m, fr_shared, B, sampler);
  int rc = AUXMC_OK;
  if (cudaMalloc(&traj, sizeof(double) * (size_t)B * (T + 1) * dx) != cudaSuccess ||
      cudaMalloc(&status, sizeof(int) * B) != cudaSuccess || cudaMalloc(&ws, wsb) != cudaSuccess)
    rc = AUXMC_E_CUDA;
  if (rc == AUXMC_OK)
    rc = auxmc_sample_paths(&m, &fr, fr_shared, &nz, B, sampler, traj, status, ws, wsb, nullptr);
  if (rc == AUXMC_OK) {
    cudaMemcpy(traj_host, traj, sizeof(double) * (size_t)B * (T + 1) * dx, cudaMemcpyDeviceToHost);
    cudaMemcpy(status_host, status, sizeof(int) * B, cudaMemcpyDeviceToHost);
    if (cudaGetLastError() != cudaSuccess) rc = AUXMC_E_CUDA;
  }
  cudaFree(traj);
  cudaFree(status);
  cudaFree(ws);
  for (void* p : allocs) cudaFree(p);
  return rc;
}

}  // extern "C"
