// prefix_gen.cu — prefix (parallel-in-time) pathwise sampler for any state
// dimension 9 <= d <= 64 (pit::prefix_sample, pit.cpp:78-106).
//
// The path obeys the affine backward recursion x_t = G_t x_{t+1} + c~_t with
// c~_t = off_t + L_t xi_t (the realized element, pit.cpp:64-76).  The horizon
// is cut into P blocks of Lb steps and scanned in three passes:
//   1. per (filter result, block): the block operator A_k = G_s G_{s+1} ... G_{e-1}
//      (DMMA products, one warp per block; shared by every chain when the filter
//      result is shared);
//   2. per (chain, block): c~_t (written into the output slot of x_t) and the
//      block offset a_k = c~_s + G_s (c~_{s+1} + G_{s+1}(...)), so that
//      x_s = A_k x_e + a_k;
//   3. per chain: the terminal draw and the serial carry over blocks, last to
//      first, giving the value x_e entering each block;
//   4. per (chain, block): x_t = G_t x_{t+1} + c~_t inside the block.
// Within a block the arithmetic is the sequential sampler's (same dot-product
// order); only the block-boundary values associate differently from the
// reference's Sklansky tree, which is within the FP64 parity tolerance.
#include <algorithm>

#include "common.cuh"
#include "dense.cuh"
#include "rng.cuh"
#include "tma.cuh"

namespace auxmc_gpu {

namespace {

constexpr int kWarpsPG = 4;

__device__ __forceinline__ void noise_vec(const NoiseArgs& nz, int c, int T, int t, int d, int lane,
                                          double* xi) {
  if (nz.kind == AUXMC_NOISE_PREDRAWN) {
    for (int i = lane; i < d; i += 32) xi[i] = nz.backward[((size_t)c * T + t) * d + i];
  } else {
    const uint64_t key = derive_index(derive_label(nz.keys[c], kBackwardNoise), (uint64_t)t);
    for (int i = lane; i < d; i += 32) xi[i] = normal_at(key, (uint64_t)i);
  }
}

// pass 1: A_k for (fr, block k); smem per warp: 2 d*d
// rep (nullable): rep[f T + t] = the element whose matrices (G, L) step t shares —
// k_bwd_lanes writes only the offsets of a uniform chunk's later steps
__device__ __forceinline__ const double* el_mat(const double* E, const int* rep, int T, int f, int t,
                                                int ES) {
  return E + (size_t)(rep ? rep[(size_t)f * T + t] : t) * ES;
}

__global__ void k_pg_block_ops(int T, int d, int Bfr, int Lb, int P, const double* __restrict__ elems,
                               double* __restrict__ ops, int k_lo, int k_hi,
                               const int* __restrict__ rep) {
  extern __shared__ double sm[];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const long long item = (long long)blockIdx.x * nw + w;
  const int span = k_hi - k_lo;  // blocks [k_lo, k_hi)
  if (item >= (long long)Bfr * span) return;
  const int f = (int)(item / span), k = k_lo + (int)(item % span);
  const int dd = d * d, ES = elem_stride(d);
  double* A = sm + (size_t)w * 2 * dd;
  double* Bm = A + dd;
  const int s = k * Lb, e = min(T, s + Lb);
  const double* E = elems + (size_t)f * T * ES;
  const Grp g = warp_group();
  // A = G_{e-1}
  {
    const double* G = el_mat(E, rep, T, f, e - 1, ES);
    for (int i = lane; i < dd; i += 32) A[i] = G[i];
  }
  __syncwarp();
  for (int t = e - 2; t >= s; --t) {  // A := G_t A
    g_dmma<false, false>(g, d, d, d, el_mat(E, rep, T, f, t, ES), d, A, d, Bm, d, false, false);
    __syncwarp();
    double* tmp = A;
    A = Bm;
    Bm = tmp;
  }
  // stored transposed: the carry's lanes read row i of A_k as a column (conflict-free)
  double* out = ops + ((size_t)f * P + k) * dd;
  for (int i = lane; i < dd; i += 32) out[(i % d) * d + i / d] = A[i];
}

// pass 2: c~_t into traj[t] and a_k; smem per warp: 2 * 64 (xi, a)
__global__ void k_pg_block_offsets(int T, int d, int B, int fr_shared, int Lb, int P,
                                   const double* __restrict__ elems, NoiseArgs nz,
                                   double* __restrict__ traj, double* __restrict__ offs, int k_lo,
                                   int k_hi, const int* __restrict__ rep) {
  __shared__ double sv[kWarpsPG][3][64];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long item = (long long)blockIdx.x * kWarpsPG + w;
  const int span = k_hi - k_lo;
  if (item >= (long long)B * span) return;
  const int c = (int)(item / span), k = k_lo + (int)(item % span);
  const int dd = d * d, ES = elem_stride(d);
  const double* E = elems + (size_t)(fr_shared ? 0 : c) * T * ES;
  double* out = traj + (size_t)c * (T + 1) * d;
  double* xi = sv[w][0];
  double* a = sv[w][1];
  double* an = sv[w][2];
  const int s = k * Lb, e = min(T, s + Lb);
  const int f = fr_shared ? 0 : c;
  for (int t = e - 1; t >= s; --t) {
    const double* el = E + (size_t)t * ES;
    const double* em = el_mat(E, rep, T, f, t, ES);
    noise_vec(nz, c, T, t, d, lane, xi);
    __syncwarp();
    for (int i = lane; i < d; i += 32) {
      double cv = 0.0;
      for (int j = 0; j < d; ++j) cv += em[dd + d + i * d + j] * xi[j];
      const double ct = el[dd + i] + cv;  // c~_t
      out[(size_t)t * d + i] = ct;
      if (t == e - 1) {
        an[i] = ct;
      } else {
        double ga = 0.0;
        for (int j = 0; j < d; ++j) ga += em[i * d + j] * a[j];
        an[i] = ga + ct;
      }
    }
    __syncwarp();
    for (int i = lane; i < d; i += 32) a[i] = an[i];
    __syncwarp();
  }
  double* o = offs + ((size_t)c * P + k) * d;
  for (int i = lane; i < d; i += 32) o[i] = a[i];
}

// pass 3: terminal draw and the serial block carry (one warp per chain, one chain
// per CTA).  The block operators (stored transposed) and offsets stream through a
// kCarryStages ring of bulk copies issued kCarryStages blocks ahead, so a step is
// the d-long dot products alone; without 16-B alignment (odd d) they are read
// from global memory directly.  Same operations in the same order either way.
constexpr int kCarryStages = 4;
__host__ __device__ inline int carry_slot(int d) { return (d * d + d + 1) & ~1; }
__host__ __device__ inline size_t carry_smem(int d) {
  return sizeof(double) * ((size_t)kCarryStages * carry_slot(d) + 128);
}
__global__ void __launch_bounds__(32)
    k_pg_carry(int T, int d, int B, int fr_shared, int P, const double* __restrict__ term,
               const double* __restrict__ ops, const double* __restrict__ offs, NoiseArgs nz,
               double* __restrict__ traj, double* __restrict__ xin,
               const double* __restrict__ xT_in) {
  extern __shared__ __align__(16) double csm[];
  __shared__ __align__(8) uint64_t bars[kCarryStages];
  const int lane = threadIdx.x;
  const int c = blockIdx.x;
  if (c >= B) return;
  const int dd = d * d, slot = carry_slot(d);
  const double* tm = term + (size_t)(fr_shared ? 0 : c) * term_stride(d);
  double* x = csm + (size_t)kCarryStages * slot;
  double* xn = x + 64;
  double* out = traj + (size_t)c * (T + 1) * d;
  const bool pre = nz.kind == AUXMC_NOISE_PREDRAWN;
  if (xT_in) {  // time-sharded: x_T drawn by the rank that owns T
    for (int i = lane; i < d; i += 32) {
      x[i] = xT_in[(size_t)c * d + i];
      out[(size_t)T * d + i] = x[i];
    }
  } else {
    for (int i = lane; i < d; i += 32)
      xn[i] = pre ? nz.terminal[(size_t)c * d + i]
                  : normal_at(derive(nz.keys[c], kTerminalDraw, 0), (uint64_t)i);
    __syncwarp();
    for (int i = lane; i < d; i += 32) {  // x_T = m_T + L_T xi (pit.cpp:85-87)
      double s = 0.0;
      for (int j = 0; j < d; ++j) s += tm[d + i * d + j] * xn[j];
      x[i] = tm[i] + s;
      out[(size_t)T * d + i] = x[i];
    }
  }
  __syncwarp();
  const double* O = ops + (size_t)(fr_shared ? 0 : c) * P * dd;
  const double* OF = offs + (size_t)c * P * d;
  const bool tma = (d % 2 == 0) && ((reinterpret_cast<uintptr_t>(O) & 15) == 0) &&
                   ((reinterpret_cast<uintptr_t>(OF) & 15) == 0);
  if (tma && lane == 0) {
    for (int st = 0; st < kCarryStages; ++st) mbar_init(&bars[st], 1);
    mbar_fence_init();
  }
  __syncwarp();
  auto issue = [&](int k, int st) {  // block k's (A_k^T | a_k) into ring slot st
    mbar_expect_tx(&bars[st], (unsigned)(dd + d) * 8u);
    bulk_g2s(csm + (size_t)st * slot, O + (size_t)k * dd, (unsigned)dd * 8u, &bars[st]);
    bulk_g2s(csm + (size_t)st * slot + dd, OF + (size_t)k * d, (unsigned)d * 8u, &bars[st]);
  };
  if (tma && lane == 0)
    for (int st = 0; st < kCarryStages && P - 1 - st >= 0; ++st) issue(P - 1 - st, st);
  for (int k = P - 1, it = 0; k >= 0; --k, ++it) {
    double* xe = xin + ((size_t)c * P + k) * d;
    for (int i = lane; i < d; i += 32) xe[i] = x[i];
    const double *At, *a;
    const int st = it % kCarryStages;
    if (tma) {
      mbar_wait(&bars[st], (unsigned)(it / kCarryStages) & 1u);
      At = csm + (size_t)st * slot;
      a = At + dd;
    } else {
      At = O + (size_t)k * dd;
      a = OF + (size_t)k * d;
    }
    if (d == 16) {  // static bounds: the 16 operand pairs load before the FMA chain
      if (lane < 16) {
        double av[16], xv[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          av[j] = At[j * 16 + lane];
          xv[j] = x[j];
        }
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < 16; ++j) s += av[j] * xv[j];
        xn[lane] = s + a[lane];
      }
    } else {
      for (int i = lane; i < d; i += 32) {
        double s = 0.0;
        for (int j = 0; j < d; ++j) s += At[j * d + i] * x[j];
        xn[i] = s + a[i];
      }
    }
    __syncwarp();
    if (tma && lane == 0 && k - kCarryStages >= 0) issue(k - kCarryStages, st);
    for (int i = lane; i < d; i += 32) x[i] = xn[i];
    __syncwarp();
  }
}

int launch_pg_carry(int T, int d, int B, int fr_shared, int P, const double* term,
                    const double* ops, const double* offs, const NoiseArgs& nz, double* traj,
                    double* xin, const double* xT_in, cudaStream_t stream) {
  AUXMC_CUDA_TRY(cudaFuncSetAttribute(k_pg_carry, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)carry_smem(d)));
  AUXMC_LAUNCH(k_pg_carry, B, 32, carry_smem(d), stream, T, d, B, fr_shared, P, term, ops, offs,
               nz, traj, xin, xT_in);
  return AUXMC_OK;
}

// pass 4: x_t = G_t x_{t+1} + c~_t inside each block
__global__ void k_pg_apply(int T, int d, int B, int fr_shared, int Lb, int P,
                           const double* __restrict__ elems, const double* __restrict__ xin,
                           double* __restrict__ traj, int k_lo, int k_hi,
                           const int* __restrict__ rep) {
  __shared__ double sv[kWarpsPG][2][64];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long item = (long long)blockIdx.x * kWarpsPG + w;
  const int span = k_hi - k_lo;
  if (item >= (long long)B * span) return;
  const int c = (int)(item / span), k = k_lo + (int)(item % span);
  const int ES = elem_stride(d);
  const double* E = elems + (size_t)(fr_shared ? 0 : c) * T * ES;
  double* out = traj + (size_t)c * (T + 1) * d;
  double* x = sv[w][0];
  double* xn = sv[w][1];
  const double* xe = xin + ((size_t)c * P + k) * d;
  for (int i = lane; i < d; i += 32) x[i] = xe[i];
  __syncwarp();
  const int s = k * Lb, e = min(T, s + Lb);
  for (int t = e - 1; t >= s; --t) {
    const double* el = el_mat(E, rep, T, fr_shared ? 0 : c, t, ES);
    for (int i = lane; i < d; i += 32) {
      double gx = 0.0;
      for (int j = 0; j < d; ++j) gx += el[i * d + j] * x[j];
      xn[i] = gx + out[(size_t)t * d + i];
    }
    __syncwarp();
    for (int i = lane; i < d; i += 32) {
      x[i] = xn[i];
      out[(size_t)t * d + i] = xn[i];
    }
    __syncwarp();
  }
}

int block_len(int T) { return prefix_block_len(T); }

}  // namespace

// elems/term from launch_bwd_elements (store_cov = 0: element holds chol(Λ)).
int launch_prefix_generic(int T, int d, int B, int fr_shared, const double* elems,
                          const double* term, const NoiseArgs& nz, double* traj, Arena& ws,
                          cudaStream_t stream, const int* rep) {
  if (d < 1 || d > 64) return AUXMC_E_DIM;
  const int Bfr = fr_shared ? 1 : B;
  const int Lb = block_len(T > 0 ? T : 1);
  const int P = T > 0 ? (T + Lb - 1) / Lb : 0;
  const int dd = d * d;
  double* ops = ws.take<double>((size_t)Bfr * (P > 0 ? P : 1) * dd);
  double* offs = ws.take<double>((size_t)B * (P > 0 ? P : 1) * d);
  double* xin = ws.take<double>((size_t)B * (P > 0 ? P : 1) * d);
  if (ws.base == nullptr) return AUXMC_OK;
  if (!ops || !offs || !xin) return AUXMC_E_WORKSPACE;
  if (T > 0) {
    const int wo = std::max(1, std::min(kWarpsPG, (int)((200 * 1024) / (16 * dd))));
    const size_t smem = sizeof(double) * 2 * dd * wo;
    AUXMC_CUDA_TRY(
        cudaFuncSetAttribute(k_pg_block_ops, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const long long nops = (long long)Bfr * P, nvec = (long long)B * P;
    AUXMC_LAUNCH(k_pg_block_ops, (int)((nops + wo - 1) / wo), 32 * wo, smem, stream, T, d, Bfr,
                 Lb, P, elems, ops, 0, P, rep);
    AUXMC_LAUNCH(k_pg_block_offsets, (int)((nvec + kWarpsPG - 1) / kWarpsPG), 32 * kWarpsPG, 0,
                 stream, T, d, B, fr_shared, Lb, P, elems, nz, traj, offs, 0, P, rep);
  }
  {
    const int rc = launch_pg_carry(T, d, B, fr_shared, P, term, ops, offs, nz, traj, xin, nullptr,
                                   stream);
    if (rc) return rc;
  }
  if (T > 0) {
    const long long nvec = (long long)B * P;
    AUXMC_LAUNCH(k_pg_apply, (int)((nvec + kWarpsPG - 1) / kWarpsPG), 32 * kWarpsPG, 0, stream, T,
                 d, B, fr_shared, Lb, P, elems, xin, traj, 0, P, rep);
  }
  return AUXMC_OK;
}

// ---------------------------------------------------------------- time-sharded prefix sampler
// One path (B = 1, pit::prefix_sample, pit.cpp:78-115) with the horizon split like
// the time-sharded filter: a rank owns the steps [t_lo, t_hi) of its super-blocks,
// whose edges fall on sampler blocks (Lb divides the super-block length).  Phase 1
// builds the rank's backward elements (the one at t_hi - 1 uses the predictive
// covariance at t_hi that the sharded filter also produced), block operators and
// offsets (+ x_T on the rank that owns T); the caller all-gathers the (A_k | a_k)
// rows of every block in order and x_T; phase 2 runs the serial block carry over all
// blocks (every rank, same bits) and expands the rank's blocks.
int launch_bwd_elements(const DevModel& dm, const double* fm, const double* fc, const double* pc,
                        int Bfr, double* elems, double* term, int* st_fr, int store_cov,
                        cudaStream_t stream, int t_lo, int t_hi, double* recs, int* rep);

namespace {
struct TsPrefixBufs {
  double *elems, *term, *ops, *offs, *xin, *recs;
  int* st;
};
TsPrefixBufs tsp_take(const DevModel& dm, Arena& ws) {
  const int T = dm.T, d = dm.dx, Lb = block_len(T > 0 ? T : 1);
  const int P = T > 0 ? (T + Lb - 1) / Lb : 1;
  TsPrefixBufs b;
  b.elems = ws.take<double>((size_t)(T > 0 ? T : 1) * elem_stride(d));
  b.term = ws.take<double>((size_t)term_stride(d));
  b.ops = ws.take<double>((size_t)P * d * d);
  b.offs = ws.take<double>((size_t)P * d);
  b.xin = ws.take<double>((size_t)P * d);
  b.st = ws.take<int>(1);
  b.recs = ws.take<double>(bwd_recs_doubles(1, T + 1));
  return b;
}

__global__ void k_tsp_pack(int d, int k_lo, int k_hi, const double* ops, const double* offs,
                           double* out) {  // rows (A_k | a_k) of blocks [k_lo, k_hi)
  const int dd = d * d, R = dd + d;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < (k_hi - k_lo) * R;
       e += gridDim.x * blockDim.x) {
    const int r = e / R, o = e % R, k = k_lo + r;
    out[e] = o < dd ? ops[(size_t)k * dd + o] : offs[(size_t)k * d + (o - dd)];
  }
}
__global__ void k_tsp_unpack(int d, int P, const double* in, double* ops, double* offs) {
  const int dd = d * d, R = dd + d;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < P * R; e += gridDim.x * blockDim.x) {
    const int k = e / R, o = e % R;
    if (o < dd) ops[(size_t)k * dd + o] = in[e];
    else offs[(size_t)k * d + (o - dd)] = in[e];
  }
}
}  // namespace

int tshard_prefix_geometry(int T, int* Lb, int* P) {
  *Lb = block_len(T > 0 ? T : 1);
  *P = T > 0 ? (T + *Lb - 1) / *Lb : 0;
  return AUXMC_OK;
}

size_t tshard_prefix_workspace(const DevModel& dm) {
  Arena ws{nullptr, 0, 0};
  tsp_take(dm, ws);
  return ws.used + 1024;
}

int tshard_prefix_local(const DevModel& dm, const double* fm, const double* fc, const double* pc,
                        const NoiseArgs& nz, int t_lo, int t_hi, Arena& ws, double* blk_out,
                        double* xT_out, double* traj, int* status, cudaStream_t stream) {
  const int T = dm.T, d = dm.dx, Lb = block_len(T > 0 ? T : 1);
  if (d < 1 || d > 64) return AUXMC_E_DIM;
  const TsPrefixBufs b = tsp_take(dm, ws);
  if (ws.base == nullptr) return AUXMC_OK;
  if (!b.elems || !b.st || !b.recs) return AUXMC_E_WORKSPACE;
  if (t_lo < 0 || t_hi > T + 1 || t_lo >= t_hi || t_lo % Lb != 0) return AUXMC_E_ARG;
  AUXMC_CUDA_TRY(cudaMemsetAsync(status, 0, sizeof(int), stream));
  // elements for steps [t_lo, min(t_hi, T)) and the terminal law when T is owned
  int rc = launch_bwd_elements(dm, fm, fc, pc, 1, b.elems, b.term, status, 0, stream, t_lo, t_hi,
                               b.recs, nullptr);
  if (rc) return rc;
  const int s_hi = std::min(t_hi, T);
  if (s_hi > t_lo) {
    const int k_lo = t_lo / Lb, k_hi = (s_hi + Lb - 1) / Lb, P = (T + Lb - 1) / Lb;
    const int wo = std::max(1, std::min(kWarpsPG, (int)((200 * 1024) / (16 * d * d))));
    const size_t smem = sizeof(double) * 2 * d * d * wo;
    AUXMC_CUDA_TRY(
        cudaFuncSetAttribute(k_pg_block_ops, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int nk = k_hi - k_lo;
    AUXMC_LAUNCH(k_pg_block_ops, (nk + wo - 1) / wo, 32 * wo, smem, stream, T, d, 1, Lb, P,
                 b.elems, b.ops, k_lo, k_hi, (const int*)nullptr);
    AUXMC_LAUNCH(k_pg_block_offsets, (nk + kWarpsPG - 1) / kWarpsPG, 32 * kWarpsPG, 0, stream, T, d,
                 1, 1, Lb, P, b.elems, nz, traj, b.offs, k_lo, k_hi, (const int*)nullptr);
    AUXMC_LAUNCH(k_tsp_pack, 64, 256, 0, stream, d, k_lo, k_hi, b.ops, b.offs, blk_out);
  }
  if (t_hi == T + 1) {  // x_T = m_T + L_T xi on the rank that owns T
    const int rc2 = launch_pg_carry(T, d, 1, 1, 0, b.term, b.ops, b.offs, nz, traj, b.xin, nullptr,
                                    stream);
    if (rc2) return rc2;
    AUXMC_CUDA_TRY(cudaMemcpyAsync(xT_out, traj + (size_t)T * d, sizeof(double) * d,
                                   cudaMemcpyDeviceToDevice, stream));
  }
  return AUXMC_OK;
}

int tshard_prefix_finish(const DevModel& dm, const NoiseArgs& nz, int t_lo, int t_hi, Arena& ws,
                         const double* blk_all, const double* xT, double* traj,
                         cudaStream_t stream) {
  const int T = dm.T, d = dm.dx, Lb = block_len(T > 0 ? T : 1);
  const TsPrefixBufs b = tsp_take(dm, ws);
  if (ws.base == nullptr) return AUXMC_OK;
  if (!b.elems || !b.st || !b.recs) return AUXMC_E_WORKSPACE;
  if (T == 0) return AUXMC_OK;
  const int P = (T + Lb - 1) / Lb;
  AUXMC_LAUNCH(k_tsp_unpack, 64, 256, 0, stream, d, P, blk_all, b.ops, b.offs);
  {
    const int rc = launch_pg_carry(T, d, 1, 1, P, b.term, b.ops, b.offs, nz, traj, b.xin, xT,
                                   stream);
    if (rc) return rc;
  }
  const int s_hi = std::min(t_hi, T);
  if (s_hi > t_lo) {
    const int k_lo = t_lo / Lb, k_hi = (s_hi + Lb - 1) / Lb;
    AUXMC_LAUNCH(k_pg_apply, (k_hi - k_lo + kWarpsPG - 1) / kWarpsPG, 32 * kWarpsPG, 0, stream, T,
                 d, 1, 1, Lb, P, b.elems, b.xin, traj, k_lo, k_hi, (const int*)nullptr);
  }
  return AUXMC_OK;
}

}  // namespace auxmc_gpu
