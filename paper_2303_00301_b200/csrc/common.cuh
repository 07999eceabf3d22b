// common.cuh — shared host/device plumbing of libauxmc_b200: status codes,
// launch accounting, error capture, model accessors.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdio>

#include "../../include/auxmc_gpu.h"

namespace auxmc_gpu {

extern std::atomic<unsigned long long> g_launches;
extern std::atomic<int> g_prof_on;
void set_last_error(const char* where, cudaError_t e);
// Per-launch CUDA-event bracketing while profiling is enabled (auxmc_profile_*).
void prof_mark(const char* name, cudaStream_t s, bool begin);

#define AUXMC_LAUNCH(kernel, grid, block, smem, stream, ...)                   \
  do {                                                                         \
    const bool _prof = ::auxmc_gpu::g_prof_on.load(std::memory_order_relaxed); \
    if (_prof) ::auxmc_gpu::prof_mark(#kernel, (cudaStream_t)(stream), true);  \
    kernel<<<(grid), (block), (smem), (cudaStream_t)(stream)>>>(__VA_ARGS__);  \
    ::auxmc_gpu::g_launches.fetch_add(1, std::memory_order_relaxed);           \
    cudaError_t _e = cudaGetLastError();                                       \
    if (_e != cudaSuccess) {                                                   \
      ::auxmc_gpu::set_last_error(#kernel, _e);                                \
      return AUXMC_E_CUDA;                                                     \
    }                                                                          \
    if (_prof) ::auxmc_gpu::prof_mark(#kernel, (cudaStream_t)(stream), false); \
  } while (0)

#define AUXMC_CUDA_TRY(expr)                                                   \
  do {                                                                         \
    cudaError_t _e = (expr);                                                   \
    if (_e != cudaSuccess) {                                                   \
      ::auxmc_gpu::set_last_error(#expr, _e);                                  \
      return AUXMC_E_CUDA;                                                     \
    }                                                                          \
  } while (0)

bool device_ok();
int num_sms();

inline size_t align_up(size_t n, size_t a = 256) { return (n + a - 1) / a * a; }

// Warps per CTA for warp-per-matrix factorization kernels (3 W×W tiles per warp).
inline int factor_warps(int W) {
  const size_t per = sizeof(double) * (3 * (size_t)W * W + 4);
  size_t w = (200 * 1024) / per;
  if (w > 4) w = 4;
  return w < 1 ? 1 : (int)w;
}

// Bump allocator over a caller-provided workspace.
struct Arena {
  char* base;
  size_t size, used;
  template <class T>
  T* take(size_t count) {
    size_t off = align_up(used);
    size_t bytes = sizeof(T) * count;
    if (base == nullptr) {  // sizing pass
      used = off + bytes;
      return nullptr;
    }
    if (off + bytes > size) return nullptr;
    used = off + bytes;
    return reinterpret_cast<T*>(base + off);
  }
};

// ---- lgssm model accessors (lgssm.hpp:34-40 broadcast rule) ----
// One LGSSM, or a batch of LGSSMs sharing (T, dx, dy): each array has a
// per-problem stride in doubles (0 = shared by the batch, the public API's
// case; the auxiliary kernel uses per-chain F, b, R).
struct DevModel {
  int T, dx, dy;
  const double *m0, *P0, *F, *b, *Q, *H, *c, *R;
  int nF, nb, nQ, nH, nc, nR;
  long long sF, sb, sQ, sH, sc, sR;
  const uint8_t* mask;
  // F given as a stencil instead of a dense array (fst = 1: F_t = I + h J_L96(xl_t), the
  // auxiliary model of Lorenz-96; F == nullptr): xl [B][T+1][dx] with stride sxl
  const double* xl = nullptr;
  long long sxl = 0;
  int fst = 0;
  double fh = 0.0;
  __device__ __forceinline__ const double* Ft(int t, int k = 0) const { return F + (size_t)k * sF + (size_t)(nF > 1 ? t : 0) * dx * dx; }
  __device__ __forceinline__ const double* bt(int t, int k = 0) const { return b + (size_t)k * sb + (size_t)(nb > 1 ? t : 0) * dx; }
  __device__ __forceinline__ const double* Qt(int t, int k = 0) const { return Q + (size_t)k * sQ + (size_t)(nQ > 1 ? t : 0) * dx * dx; }
  __device__ __forceinline__ const double* Ht(int t, int k = 0) const { return H + (size_t)k * sH + (size_t)(nH > 1 ? t : 0) * dy * dx; }
  __device__ __forceinline__ const double* ct(int t, int k = 0) const { return c + (size_t)k * sc + (size_t)(nc > 1 ? t : 0) * dy; }
  __device__ __forceinline__ const double* Rt(int t, int k = 0) const { return R + (size_t)k * sR + (size_t)(nR > 1 ? t : 0) * dy * dy; }
  __device__ __forceinline__ bool observed(int t) const { return mask == nullptr || mask[t] != 0; }
};

inline DevModel to_dev(const auxmc_lgssm& m) {
  DevModel d;
  d.T = m.T; d.dx = m.dx; d.dy = m.dy;
  d.m0 = m.m0; d.P0 = m.P0; d.F = m.F; d.b = m.b; d.Q = m.Q; d.H = m.H; d.c = m.c; d.R = m.R;
  d.nF = m.nF; d.nb = m.nb; d.nQ = m.nQ; d.nH = m.nH; d.nc = m.nc; d.nR = m.nR;
  d.sF = d.sb = d.sQ = d.sH = d.sc = d.sR = 0;
  d.mask = m.mask;
  d.xl = nullptr; d.sxl = 0; d.fst = 0; d.fh = 0.0;
  return d;
}

// Row i of F = I + h J_L96(x): columns ascending (dyn_jac_ij's entries, same rounding).
__device__ __forceinline__ void l96_row(const double* x, int d, double h, int i, int* cols,
                                        double* vals) {
  const int ip1 = (i + 1) % d, im1 = (i + d - 1) % d, im2 = (i + d - 2) % d;
  int c4[4] = {im2, im1, i, ip1};
  double v4[4] = {h * (0.0 - x[im1]), h * (0.0 + (x[ip1] - x[im2])), 1.0 + h * (0.0 - 1.0),
                  h * (0.0 + x[im1])};
  // sort by column (wrap-around rows)
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 3 - a; ++b)
      if (c4[b] > c4[b + 1]) {
        const int tc = c4[b]; c4[b] = c4[b + 1]; c4[b + 1] = tc;
        const double tv = v4[b]; v4[b] = v4[b + 1]; v4[b + 1] = tv;
      }
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    cols[a] = c4[a];
    vals[a] = v4[a];
  }
}

// Row i of the model's F_t for path k as (column, value) pairs; returns the count
// (dense rows: every column).  cols/vals hold up to dx entries for dense F.
__device__ __forceinline__ void stencil_row(const DevModel& m, int t, int k, int i, int* cols,
                                            double* vals) {
  l96_row(m.xl + (size_t)k * m.sxl + (size_t)t * m.dx, m.dx, m.fh, i, cols, vals);
}

// dense F_t of path k into dst (d*d), group-strided over `lane` / `size`
__device__ __forceinline__ void fill_F(const DevModel& m, int t, int k, double* dst, int lane,
                                      int size) {
  const int d = m.dx;
  if (!m.fst) {
    const double* F = m.Ft(t, k);
    for (int i = lane; i < d * d; i += size) dst[i] = F[i];
    return;
  }
  for (int i = lane; i < d; i += size) {  // row i by one lane: zero, then the stencil
    int cs[4];
    double vs[4];
    stencil_row(m, t, k, i, cs, vs);
    for (int j = 0; j < d; ++j) dst[i * d + j] = 0.0;
    for (int a = 0; a < 4; ++a) dst[i * d + cs[a]] = vs[a];
  }
}

int check_model(const auxmc_lgssm* m);

__host__ __device__ inline int elem_stride(int d) { return (2 * d * d + d + 1) & ~1; }
__host__ __device__ inline int term_stride(int d) { return (d * d + d + 1) & ~1; }

struct NoiseArgs {
  int kind;
  const uint64_t* keys;
  const double* terminal;
  const double* backward;
  const double* bridge;
  long long n_bridge;
};


// Deterministic CTA-wide sum of get(0..n): each thread sums a contiguous chunk in
// index order, then a fixed pairwise tree over the (power-of-two) thread
// partials.  Replaces the reference's left-to-right sums over the horizon
// (same terms, different association: within the FP64 parity tolerance).
// red: blockDim.x doubles of shared memory.  Returns the sum on all threads.
template <class Get>
__device__ __forceinline__ double cta_sum_fixed(long long n, Get get, double* red,
                                              const double* parts = nullptr) {
  const int nt = blockDim.x, tid = threadIdx.x;
  const long long chunk = (n + nt - 1) / nt;
  const long long lo = tid * chunk;
  const long long hi = parts ? lo : (lo + chunk < n ? lo + chunk : n);
  double s = parts ? parts[tid] : 0.0;  // parts: the chunk sums, from k_sum_parts
  long long i = lo;
  for (; i + 8 <= hi; i += 8) {  // eight loads in flight, added in index order
    double v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = get(i + k);
#pragma unroll
    for (int k = 0; k < 8; ++k) s += v[k];
  }
  for (; i < hi; ++i) s += get(i);
  red[tid] = s;
  __syncthreads();
  for (int w = nt >> 1; w > 0; w >>= 1) {
    if (tid < w) red[tid] = red[tid] + red[tid + w];
    __syncthreads();
  }
  const double r = red[0];
  __syncthreads();
  return r;
}
constexpr int kSumThreads = 256;

// cta_sum_fixed's chunk sums of a few long rows, spread over warps of many CTAs (one
// SM alone cannot stream a 2^20-term row): warp (row, c) loads chunk c 32 terms at a
// time, coalesced, and adds them in index order from 0.0 — the thread loop's sum,
// bit for bit; cta_sum_fixed(..., parts) then runs the same tree.
template <typename Get>
__global__ void __launch_bounds__(256) k_sum_parts(int rows, long long n, Get get, double* parts) {
  const long long w = (long long)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (w >= (long long)rows * kSumThreads) return;
  const int r = (int)(w / kSumThreads), c = (int)(w % kSumThreads);
  const long long chunk = (n + kSumThreads - 1) / kSumThreads;
  const long long lo = c * chunk, hi = lo + chunk < n ? lo + chunk : n;
  const int lane = threadIdx.x & 31;
  double s = 0.0;
  for (long long base = lo; base < hi; base += 32) {
    const long long i = base + lane;
    const double v = i < hi ? get(r, i) : 0.0;
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      const double vk = __shfl_sync(0xffffffffu, v, k);
      if (base + k < hi) s += vk;
    }
  }
  if (lane == 0) parts[(size_t)r * kSumThreads + c] = s;
}
// rows of a terms array
struct RowTerms {
  const double* t;
  long long stride;
  __device__ double operator()(int r, long long i) const { return t[(size_t)r * stride + i]; }
};
// the two-kernel form pays off for few, long rows
inline bool sum_parts_pay(int rows, long long n) { return rows <= 16 && n >= 65536; }
// declares `double* parts` (stream-ordered allocation, freed by the caller after the
// sum kernel) and fills it with k_sum_parts over `rows` rows of n terms, or leaves it
// null when one CTA per row is enough
#define PFG_SUM_PARTS(rows, n, terms)                                                        \
  double* parts = nullptr;                                                                   \
  if (::auxmc_gpu::sum_parts_pay((rows), (n))) {                                             \
    AUXMC_CUDA_TRY(cudaMallocAsync(&parts, sizeof(double) * (rows) * kSumThreads, s));       \
    AUXMC_LAUNCH(k_sum_parts<RowTerms>, ((rows) * kSumThreads + 7) / 8, 256, 0, s, (rows),   \
                 (long long)(n), (RowTerms{(terms), (long long)(n)}), parts);                \
  }

// k_bwd_lean's items per chunk in its reuse mode, and the chunk records
// (uniform flag, status) k_bwd_lanes reads
constexpr int kBwdChunk = 128;
inline size_t bwd_recs_doubles(int Bfr, int span) {
  return 2 * (size_t)Bfr * ((span + kBwdChunk - 1) / kBwdChunk);
}

// block length of the generic prefix sampler (prefix_gen.cu): a power of two near
// sqrt(T) / 4 — short block passes for one long chain, the serial block carry
// streamed (k_pg_carry); the scan filter's super-blocks are multiples of it
// (pfilter_gen.cu), so a time-sharded rank's range holds whole sampler blocks
inline int prefix_block_len(int T) {
  int lb = 16, lr = 16;  // ~sqrt(T) / 4; ~sqrt(T), kept up to 64 (block rows stay
  while ((long long)lb * lb * 16 < T && lb < 4096) lb <<= 1;  // well below a path's
  while ((long long)lr * lr < T && lr < 64) lr <<= 1;         // size for d < 16)
  return lb > lr ? lb : lr;
}

}  // namespace auxmc_gpu
