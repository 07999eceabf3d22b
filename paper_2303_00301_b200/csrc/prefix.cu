// prefix.cu — pit::prefix_sample (pit.cpp:78-115) for a filter result shared by
// many chains (the C2 workload: one model, C chains, long T).
//
// Realized element t is x_t = G_t x_{t+1} + c_t with c_t = off_t + L_t xi_t
// (pit.cpp:64-76); the suffix composition S_t = e_t ∘ ... ∘ e_{T-1} gives
// x_t = S_t(x_T).  The composition is evaluated as a fixed-tree
// reduce-then-scan over the time axis:
//
//   superchunk (32 sub-chunks × LS steps)   walked top-down by one CTA that
//                                           owns <= 8 chains for the whole T
//   sub-chunk (LS steps)                    one thread: reduce (phase A) and
//                                           expand (phase C) in registers
//   sub-chunk carries                       serial per chain (phase B)
//
// G_t, off_t, L_t are chain-independent: a prep kernel packs them per
// superchunk, with the sub-chunk products Gsub, into one contiguous tile that a
// single 1-D TMA bulk copy (cp.async.bulk + mbarrier) stages into shared memory,
// double-buffered; every chain of the CTA reads the tile by broadcast.  The
// per-chain data (xi in, x out) streams straight between HBM and registers.
// Per chain-timestep HBM traffic: 32 B noise read + 32 B path write (d = 4).
// The tree depends only on (T, LS), so the output is bit-deterministic.
#include "common.cuh"
#include "dense.cuh"
#include "rng.cuh"
#include "tma.cuh"

namespace auxmc_gpu {

template <int D>
int run_prefix_bulk(int T, int B, const double* elems, const double* term, Arena& ws,
                    const NoiseArgs& nz, double* traj, cudaStream_t stream);
int run_prefix_mma(int T, int B, const double* elems, const double* term, Arena& ws,
                   const NoiseArgs& nz, double* traj, cudaStream_t stream);

template <int D>
struct PfxGeom {
  static constexpr int LS = D <= 2 ? 16 : (D <= 4 ? 8 : (D <= 6 ? 4 : 2));  // steps per sub-chunk
  static constexpr int NSUB = 32;                             // sub-chunks per superchunk
  static constexpr int S = NSUB * LS;                         // steps per superchunk
  static constexpr int LP = D * (D + 1) / 2;                  // packed lower factor
  static constexpr int ES = D * D + D + LP;                   // G | off | Lp
  static constexpr int SUB = LS * ES + 1;                     // odd: bank-spread blocks
  static constexpr int EB = NSUB * SUB;
  static constexpr int TB = ((EB + NSUB * D * D) + 1) & ~1;   // tile doubles (16 B multiple)
  static constexpr int SLOTS = 8;                             // chains per CTA (max)
  static constexpr int WARPS = 8;
};

// Pack elements [T][ES_generic] into per-superchunk tiles and compute Gsub.
template <int D>
__global__ void k_prefix_pack(const double* __restrict__ elems, int T, double* tiles) {
  using P = PfxGeom<D>;
  const int n_sub = ((T + P::S - 1) / P::S) * P::NSUB;
  const int ESg = elem_stride(D);
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < n_sub; s += gridDim.x * blockDim.x) {
    const int k = s / P::NSUB, j = s % P::NSUB;
    double* tile = tiles + (size_t)k * P::TB;
    double* blk = tile + j * P::SUB;
    const int lo = k * P::S + j * P::LS;
    double Pm[D * D], Qm[D * D];
#pragma unroll
    for (int i = 0; i < D * D; ++i) Pm[i] = (i / D == i % D) ? 1.0 : 0.0;
    for (int q = P::LS - 1; q >= 0; --q) {
      const int t = lo + q;
      double* out = blk + q * P::ES;
      if (t >= T) {
        for (int i = 0; i < P::ES; ++i) out[i] = 0.0;
        continue;
      }
      const double* e = elems + (size_t)t * ESg;
#pragma unroll
      for (int i = 0; i < D * D + D; ++i) out[i] = e[i];
      int w = 0;
#pragma unroll
      for (int r = 0; r < D; ++r)
#pragma unroll
        for (int c = 0; c <= r; ++c) out[D * D + D + w++] = e[D * D + D + r * D + c];
      // Pm = G_t Pm  (walking down: Gsub = G_lo ... G_{hi-1})
#pragma unroll
      for (int a = 0; a < D; ++a)
#pragma unroll
        for (int b = 0; b < D; ++b) {
          double acc = 0.0;
#pragma unroll
          for (int q2 = 0; q2 < D; ++q2) acc += e[a * D + q2] * Pm[q2 * D + b];
          Qm[a * D + b] = acc;
        }
#pragma unroll
      for (int i = 0; i < D * D; ++i) Pm[i] = Qm[i];
    }
    blk[P::LS * P::ES] = 0.0;  // pad
    double* gs = tile + P::EB + j * D * D;
#pragma unroll
    for (int i = 0; i < D * D; ++i) gs[i] = Pm[i];
    if (j == 0 && P::TB > P::EB + P::NSUB * D * D) tile[P::TB - 1] = 0.0;
  }
}


template <int D, bool PRE>
__global__ void __launch_bounds__(PfxGeom<D>::WARPS * 32, 1)
    k_prefix_tiles(int T, int C, const double* __restrict__ tiles, const double* __restrict__ term,
                   NoiseArgs noise, double* __restrict__ traj) {
  using P = PfxGeom<D>;
  constexpr int LS = P::LS, ES = P::ES, SUB = P::SUB, S = P::S;
  extern __shared__ __align__(16) double sm[];
  double* tile[2] = {sm, sm + P::TB};
  double* csub = sm + 2 * P::TB;                 // [SLOTS][NSUB][D]
  double* xtop = csub + P::SLOTS * P::NSUB * D;  // [SLOTS][NSUB][D]
  double* carry = xtop + P::SLOTS * P::NSUB * D; // [SLOTS][D]
  uint64_t* bar = reinterpret_cast<uint64_t*>(carry + P::SLOTS * D + (D & 1));

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int slot = lane & 7;
  const int j = warp * 4 + (lane >> 3);          // sub-chunk 0..31
  const int c_begin = (int)(((long long)blockIdx.x * C) / gridDim.x);
  const int c_end = (int)(((long long)(blockIdx.x + 1) * C) / gridDim.x);
  const int c = c_begin + slot;
  const bool active = c < c_end;
  const long long row = (long long)(T + 1) * D;
  double* out = traj + (size_t)(active ? c : 0) * row;

  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // terminal draw x_T = m_T + L_T xi (pit.cpp:85-87)
  if (active && j == 0) {
    double xi[D], x[D];
    if (PRE) {
#pragma unroll
      for (int i = 0; i < D; ++i) xi[i] = noise.terminal[(size_t)c * D + i];
    } else {
      const uint64_t k = derive(noise.keys[c], kTerminalDraw, 0);
#pragma unroll
      for (int i = 0; i < D; ++i) xi[i] = normal_at(k, (uint64_t)i);
    }
    r_matvec<D>(term + D, xi, x);
#pragma unroll
    for (int i = 0; i < D; ++i) {
      x[i] = term[i] + x[i];
      carry[slot * D + i] = x[i];
      out[(size_t)T * D + i] = x[i];
    }
  }
  __syncthreads();
  if (T == 0) return;
  const int K = (T + S - 1) / S;
  const unsigned tile_bytes = P::TB * sizeof(double);
  if (threadIdx.x == 0) {
    mbar_expect_tx(&bar[(K - 1) & 1], tile_bytes);
    bulk_g2s(tile[(K - 1) & 1], tiles + (size_t)(K - 1) * P::TB, tile_bytes, &bar[(K - 1) & 1]);
  }
  unsigned phase[2] = {0u, 0u};
  uint64_t klabel = 0;
  if (!PRE && active) klabel = derive_label(noise.keys[c], kBackwardNoise);

  // noise prefetch registers (pre-drawn mode)
  double xin[LS * D];
  auto load_xi = [&](int k) {
    const int lo = k * S + j * LS;
#pragma unroll
    for (int s = 0; s < LS; ++s) {
      const int t = lo + s;
#pragma unroll
      for (int i = 0; i < D; ++i)
        xin[s * D + i] = (active && t < T) ? __ldcs(noise.backward + ((size_t)c * T + t) * D + i) : 0.0;
    }
  };
  if (PRE) load_xi(K - 1);

  for (int k = K - 1; k >= 0; --k) {
    const int buf = k & 1;
    if (threadIdx.x == 0 && k > 0) {
      const int nb = (k - 1) & 1;
      mbar_expect_tx(&bar[nb], tile_bytes);
      bulk_g2s(tile[nb], tiles + (size_t)(k - 1) * P::TB, tile_bytes, &bar[nb]);
    }
    double cs[LS * D];
    if (PRE) {
#pragma unroll
      for (int q = 0; q < LS * D; ++q) cs[q] = xin[q];
      if (k > 0) load_xi(k - 1);
    }
    mbar_wait(&bar[buf], phase[buf]);
    phase[buf] ^= 1u;
    const double* blk = tile[buf] + j * SUB;
    const int lo = k * S + j * LS;
    // Phase A: c_t = off_t + L_t xi_t, zero-carry reduction over the sub-chunk
    double y[D];
#pragma unroll
    for (int i = 0; i < D; ++i) y[i] = 0.0;
#pragma unroll
    for (int s = LS - 1; s >= 0; --s) {
      const int t = lo + s;
      if (t < T) {
        const double* e = blk + s * ES;
        double xi[D];
        if (PRE) {
#pragma unroll
          for (int i = 0; i < D; ++i) xi[i] = cs[s * D + i];
        } else {
          const uint64_t key = derive_index(klabel, (uint64_t)t);
#pragma unroll
          for (int i = 0; i < D; ++i) xi[i] = normal_at(key, (uint64_t)i);
        }
        double gy[D];
        r_matvec<D>(e, y, gy);
        int w = 0;
#pragma unroll
        for (int r = 0; r < D; ++r) {
          double acc = 0.0;
#pragma unroll
          for (int cc = 0; cc <= r; ++cc) acc += e[D * D + D + w++] * xi[cc];
          const double cv = e[D * D + r] + acc;
          cs[s * D + r] = cv;
          y[r] = gy[r] + cv;
        }
      }
    }
#pragma unroll
    for (int i = 0; i < D; ++i) csub[(slot * P::NSUB + j) * D + i] = y[i];
    __syncthreads();
    // Phase B: per-chain carry scan over the 32 sub-chunks (top-down)
    if (warp == 0 && lane < 8 && active) {
      double x[D];
#pragma unroll
      for (int i = 0; i < D; ++i) x[i] = carry[slot * D + i];
      const double* gsub = tile[buf] + P::EB;
      for (int jj = P::NSUB - 1; jj >= 0; --jj) {
#pragma unroll
        for (int i = 0; i < D; ++i) xtop[(slot * P::NSUB + jj) * D + i] = x[i];
        if (k * S + jj * LS >= T) continue;
        double gx[D];
        r_matvec<D>(gsub + jj * D * D, x, gx);
#pragma unroll
        for (int i = 0; i < D; ++i) x[i] = gx[i] + csub[(slot * P::NSUB + jj) * D + i];
      }
#pragma unroll
      for (int i = 0; i < D; ++i) carry[slot * D + i] = x[i];
    }
    __syncthreads();
    // Phase C: expand x_t = G_t x_{t+1} + c_t from the sub-chunk's top
    if (active) {
      double x[D];
#pragma unroll
      for (int i = 0; i < D; ++i) x[i] = xtop[(slot * P::NSUB + j) * D + i];
#pragma unroll
      for (int s = LS - 1; s >= 0; --s) {
        const int t = lo + s;
        if (t < T) {
          double gx[D];
          r_matvec<D>(blk + s * ES, x, gx);
#pragma unroll
          for (int i = 0; i < D; ++i) {
            x[i] = gx[i] + cs[s * D + i];
            __stcs(out + (size_t)t * D + i, x[i]);
          }
        }
      }
    }
    __syncthreads();  // tile[buf] free for the copy issued next iteration
  }
}

template <int D>
constexpr size_t prefix_tiles_smem() {
  using P = PfxGeom<D>;
  return sizeof(double) * (2 * P::TB + 2 * P::SLOTS * P::NSUB * D + P::SLOTS * D + 2) + 16;
}

template <int D>
int run_prefix_tiles(int T, int B, const double* elems, const double* term, Arena& ws,
                     const NoiseArgs& nz, double* traj, cudaStream_t stream) {
  using P = PfxGeom<D>;
  const int K = T > 0 ? (T + P::S - 1) / P::S : 1;
  double* tiles = ws.take<double>((size_t)K * P::TB);
  if (ws.base == nullptr) return AUXMC_OK;
  if (!tiles) return AUXMC_E_WORKSPACE;
  if (T > 0) {
    const int n_sub = K * P::NSUB;
    AUXMC_LAUNCH(k_prefix_pack<D>, std::min((n_sub + 127) / 128, 148 * 16), 128, 0, stream, elems,
                 T, tiles);
  }
  constexpr size_t smem = prefix_tiles_smem<D>();
  const int grid = std::max((B + P::SLOTS - 1) / P::SLOTS, std::min(B, num_sms()));
  if (nz.kind == AUXMC_NOISE_PREDRAWN) {
    auto kern = k_prefix_tiles<D, true>;
    AUXMC_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    AUXMC_LAUNCH(kern, grid, P::WARPS * 32, smem, stream, T, B, tiles, term, nz, traj);
  } else {
    auto kern = k_prefix_tiles<D, false>;
    AUXMC_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    AUXMC_LAUNCH(kern, grid, P::WARPS * 32, smem, stream, T, B, tiles, term, nz, traj);
  }
  return AUXMC_OK;
}

int launch_prefix_shared(int d, int T, int B, const double* elems, const double* term, Arena& ws,
                         const NoiseArgs& nz, double* traj, cudaStream_t stream) {
  switch (d) {
    case 1: return run_prefix_tiles<1>(T, B, elems, term, ws, nz, traj, stream);
    case 2: return run_prefix_bulk<2>(T, B, elems, term, ws, nz, traj, stream);
    case 3: return run_prefix_tiles<3>(T, B, elems, term, ws, nz, traj, stream);
    case 4: return run_prefix_mma(T, B, elems, term, ws, nz, traj, stream);  // C2 (DMMA)
    case 5: return run_prefix_tiles<5>(T, B, elems, term, ws, nz, traj, stream);
    case 6: return run_prefix_tiles<6>(T, B, elems, term, ws, nz, traj, stream);
    case 7: return run_prefix_tiles<7>(T, B, elems, term, ws, nz, traj, stream);
    case 8: return run_prefix_tiles<8>(T, B, elems, term, ws, nz, traj, stream);
  }
  return AUXMC_E_DIM;
}

}  // namespace auxmc_gpu
