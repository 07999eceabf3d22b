// prefix_mma.cu — the C2 headline kernel on the FP64 tensor cores: shared-element
// prefix sampler (pit::prefix_sample, pit.cpp:78-115) for d = 4, 8 chains per CTA.
//
// Realized element t: x_t = G_t x_{t+1} + c_t, c_t = off_t + L_t xi_t (pit.cpp:64-76).
// G_t, off_t, L_t are shared by every chain of the sweep (one Kalman filter result),
// so for the CTA's 8 chains a step is a dense contraction X_t^T (8 chains x 4) =
// X_{t+1}^T G_t^T + C_t^T, and mma.sync.m8n8k4.f64 (DMMA) computes it with
// A = X^T (lane l = chain l/4, dim l%4).  The 8 accumulator columns hold two steps:
// column 2j = dim j of step t (B = G_t^T), column 2j+1 = dim j of step t-1
// (B = (G_{t-1} G_t)^T, C = the pair offset p_{t-1} = G_{t-1} c_t + c_{t-1}), so
// each DMMA advances a step PAIR and its second register is exactly the next A
// fragment (no shuffles).  Per step pair (hi = t, lo = t-1), for 8 chains:
//   r1 = Xi_hi^T [L_hi | G_lo L_hi]^T + [off_hi | G_lo off_hi + off_lo] -> c_hi, G_lo c_hi + off_lo
//   r2 = Xi_lo^T [L_lo | L_lo]^T + [0 | r1's second column]                -> p_lo
//   y  = y^T [G_hi | G_lo G_hi]^T + [c_hi | p_lo]               -> y_hi, y_lo
// B fragments are stored in lane order (one 256-B contiguous shared load), so the
// round-1 kernel's limiter — 16-B broadcast loads of G_t per lane, bound by shared
// wavefronts (profiles/r2_c2/) — is gone.
//
// Fixed association tree (depends on T only):
//   warp group  16 consecutive steps = 8 pairs, one warp: zero-carry reduction
//               (phase A), re-expansion from the group's top state (phase C)
//   superchunk  8 warp groups (S = 128 steps); the carry warp walks the 8 group
//               aggregates with the group spans Gw (phase B), one DMMA per group
//   sweep       superchunks top-down, carry x at the superchunk top
// Warps: 8 compute, 1 carry, 1 producer (every TMA load).  Iteration k overlaps phase
// B(k) with phase A(k-1), then expands superchunk k (phase C); (c_hi, p_lo) stay in
// registers between the phases.  Paths leave from registers (each store instruction
// writes 8 full 32-B sectors: 4 dims of 8 chains).  HBM per chain-timestep: 32 B
// noise read + 32 B path write (pre-drawn), 32 B (device RNG).  Bit-deterministic.
#include "common.cuh"
#include "dense.cuh"
#include "rng.cuh"
#include "tma.cuh"

#ifndef AUXMC_PM_EXP
#define AUXMC_PM_EXP 0  // 9: clock64 phase stamps (tools/c2_stamps.py), results invalid
#endif

namespace auxmc_gpu {

struct MmaGeom {
  static constexpr int D = 4, W = 8, GS = 16, NP = GS / 2, ROWS = 8;
  static constexpr int S = W * GS;               // 128 steps per superchunk
  // per step pair: fragGG (32) | fragL1 (32) | L_lo (16) | {off_hi, G_lo off_hi + off_lo} (8)
  static constexpr int PR = 88;
  static constexpr int ES = PR;                  // record stride (per pair)
  static constexpr int EB = (S / 2) * PR;
  static constexpr int TB = EB + W * 16;         // + warp-group spans Gw
  static constexpr int ROW = S * D + 4;          // noise row: 32-B skew per chain
  static constexpr int IOB = ROWS * ROW;
  static constexpr int TSTG = 3, NSTG = 2;
  static constexpr size_t SMEM =
      sizeof(double) * (TSTG * TB + NSTG * IOB + 2 * W * 32 + W * 32 + 32) +
      (TSTG + NSTG) * sizeof(uint64_t);
};
static_assert(MmaGeom::SMEM <= 227 * 1024, "one CTA per SM");
static_assert(MmaGeom::TB % 2 == 0 && MmaGeom::ROW % 2 == 0, "16-B aligned stages");

__device__ __forceinline__ void dmma2(double a, double b, double c0, double c1, double& d0,
                                      double& d1) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};"
      : "=d"(d0), "=d"(d1)
      : "d"(a), "d"(b), "d"(c0), "d"(c1));
}
__device__ __forceinline__ double dmma_d0(double a, double b, double c0) {
  double d0, d1;  // d1 = the odd (zero) column, unused
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};"
               : "=d"(d0), "=d"(d1)
               : "d"(a), "d"(b), "d"(c0), "d"(0.0));
  (void)d1;
  return d0;
}

__device__ __forceinline__ void mm4(const double* A, const double* B, double* C) {
  for (int a = 0; a < 4; ++a)
    for (int b = 0; b < 4; ++b) {
      double acc = 0.0;
      for (int c = 0; c < 4; ++c) acc += A[a * 4 + c] * B[c * 4 + b];
      C[a * 4 + b] = acc;
    }
}
// B fragment of [M_even | M_odd] (4 x 8, columns interleaved) in lane order:
// lane l holds M_{(l/4) % 2}[l / 8][l % 4]
__device__ __forceinline__ void frag2(const double* Me, const double* Mo, double* out) {
  for (int l = 0; l < 32; ++l) out[l] = (((l >> 2) & 1) ? Mo : Me)[4 * (l >> 3) + (l & 3)];
}

// The step-pair records, one thread per pair (dead steps t >= T: G = I, off = 0, L = 0, so
// they pass the state through).
__global__ void k_mma_pack(const double* __restrict__ elems, int T, double* tiles) {
  using G = MmaGeom;
  const int n = ((T + G::S - 1) / G::S) * (G::S / 2);
  const int ESg = elem_stride(G::D);
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x) {
    const int k = q / (G::S / 2), pr = q % (G::S / 2);  // pair pr = w * NP + j of superchunk k
    double* rec = tiles + (size_t)k * G::TB + (size_t)pr * G::PR;
    double Gs[2][16], Ls[2][16], off[2][4], GG[16], GL[16];
    for (int h = 0; h < 2; ++h) {  // h = 0: lo step, h = 1: hi step
      const int t = k * G::S + 2 * pr + h;
      if (t >= T) {
        for (int i = 0; i < 16; ++i) Gs[h][i] = (i / 4 == i % 4) ? 1.0 : 0.0;
        for (int i = 0; i < 16; ++i) Ls[h][i] = 0.0;
        for (int i = 0; i < 4; ++i) off[h][i] = 0.0;
        continue;
      }
      const double* e = elems + (size_t)t * ESg;
      for (int i = 0; i < 16; ++i) Gs[h][i] = e[i];
      for (int i = 0; i < 4; ++i) off[h][i] = e[16 + i];
      for (int r = 0; r < 4; ++r)
        for (int c = 0; c < 4; ++c) Ls[h][r * 4 + c] = c <= r ? e[20 + r * 4 + c] : 0.0;
    }
    mm4(Gs[0], Gs[1], GG);
    mm4(Gs[0], Ls[1], GL);
    frag2(Gs[1], GG, rec);
    frag2(Ls[1], GL, rec + 32);
    for (int i = 0; i < 16; ++i) rec[64 + i] = Ls[0][i];
    for (int d = 0; d < 4; ++d) {
      double acc = 0.0;
      for (int c = 0; c < 4; ++c) acc += Gs[0][d * 4 + c] * off[1][c];
      rec[80 + 2 * d] = off[1][d];
      rec[80 + 2 * d + 1] = acc + off[0][d];
    }
  }
}

// Gw = G_lo ... G_{lo+15} per (superchunk, warp group): GG_j (read back from the odd
// fragment lanes) composed top-down, GG_7 first.
__global__ void k_mma_spans(int T, double* tiles) {
  using G = MmaGeom;
  const int n = ((T + G::S - 1) / G::S) * G::W;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < n; q += gridDim.x * blockDim.x) {
    const int k = q / G::W, w = q % G::W;
    double* tile = tiles + (size_t)k * G::TB;
    double P[16], Q[16], GG[16];
    for (int i = 0; i < 16; ++i) P[i] = (i / 4 == i % 4) ? 1.0 : 0.0;
    for (int j = G::NP - 1; j >= 0; --j) {
      const double* fr = tile + (size_t)(w * G::NP + j) * G::PR;
      for (int l = 0; l < 32; ++l)
        if ((l >> 2) & 1) GG[4 * (l >> 3) + (l & 3)] = fr[l];
      mm4(GG, P, Q);
      for (int i = 0; i < 16; ++i) P[i] = Q[i];
    }
    double* gw = tile + G::EB + w * 16;
    for (int i = 0; i < 16; ++i) gw[i] = P[i];
  }
}

template <bool PRE>
__global__ void __launch_bounds__((MmaGeom::W + 2) * 32, 1)
    k_prefix_mma(int T, int C, const double* __restrict__ tiles, const double* __restrict__ term,
                 NoiseArgs noise, double* __restrict__ traj) {
  using G = MmaGeom;
  constexpr int D = G::D, GS = G::GS, S = G::S, W = G::W, ES = G::ES;
  extern __shared__ __align__(16) double sm[];
  auto tile = [&](int k) { return sm + (k % G::TSTG) * G::TB; };
  auto xin = [&](int k) { return sm + G::TSTG * G::TB + (k % G::NSTG) * G::IOB; };
  double* agg0 = sm + G::TSTG * G::TB + G::NSTG * G::IOB;
  auto cagg = [&](int k) { return agg0 + (k & 1) * W * 32; };  // [W][lane]
  double* xwtop = agg0 + 2 * W * 32;                             // [W][lane]
  double* carry = xwtop + W * 32;                                // [lane]
  uint64_t* barT = reinterpret_cast<uint64_t*>(carry + 32);
  uint64_t* barN = barT + G::TSTG;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool cw = warp == W, pw = warp == W + 1;
  const int chain = lane >> 2, dim = lane & 3;
  // B fragment of a 4x4 matrix M placed in the even columns: lane holds M[chain/2][dim]
  // for even chain (= column), zero for odd
  const bool bcol = (chain & 1) == 0;
  const int boff = 4 * (lane >> 3) + dim;
  const int c_begin = (int)(((long long)blockIdx.x * C) / gridDim.x);
  const int c_end = (int)(((long long)(blockIdx.x + 1) * C) / gridDim.x);
  const int nc = c_end - c_begin;
  const bool live = chain < nc;
  const long long row = (long long)(T + 1) * D;
  double* out_row = traj + (size_t)(c_begin + (live ? chain : 0)) * row + dim;

  if (tid == 0) {
    for (int b = 0; b < G::TSTG; ++b) mbar_init(&barT[b], 1);
    for (int b = 0; b < G::NSTG; ++b) mbar_init(&barN[b], 1);
    mbar_fence_init();
  }
  if (cw) {  // x_T = m_T + L_T xi (pit.cpp:85-87), lane = (chain, dim)
    double x = 0.0;
    if (live) {
      const int c = c_begin + chain;
      double xi[D];
      if (PRE) {
#pragma unroll
        for (int i = 0; i < D; ++i) xi[i] = noise.terminal[(size_t)c * D + i];
      } else {
        const uint64_t key = derive(noise.keys[c], kTerminalDraw, 0);
#pragma unroll
        for (int i = 0; i < D; ++i) xi[i] = normal_at(key, (uint64_t)i);
      }
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < D; ++j) acc += term[D + dim * D + j] * xi[j];
      x = term[dim] + acc;
      out_row[(size_t)T * D] = x;
    }
    carry[lane] = x;
  }
  __syncthreads();
  if (T == 0) return;
  const int K = (T + S - 1) / S;
  auto issue_tile = [&](int k) {
    const unsigned tb = G::TB * sizeof(double);
    uint64_t* bar = &barT[k % G::TSTG];
    mbar_expect_tx(bar, tb);
    bulk_g2s(tile(k), tiles + (size_t)k * G::TB, tb, bar);
  };
  auto issue_noise = [&](int k) {
    const int t0 = k * S, len = min(S, T - t0);
    const unsigned xb = (unsigned)(len * D * sizeof(double));
    uint64_t* bar = &barN[k % G::NSTG];
    mbar_expect_tx(bar, xb * nc);
    for (int ch = 0; ch < nc; ++ch)
      bulk_g2s(xin(k) + ch * G::ROW, noise.backward + ((size_t)(c_begin + ch) * T + t0) * D, xb,
               bar);
  };
  if (pw && lane == 0) {
    issue_tile(K - 1);
    if (PRE) issue_noise(K - 1);
    if (K >= 2) {
      issue_tile(K - 2);
      if (PRE) issue_noise(K - 2);
    }
  }
  unsigned tph = 0u, nph = 0u;
  auto wait_tile = [&](int k) {
    const int b = k % G::TSTG;
    mbar_wait(&barT[b], (tph >> b) & 1u);
    tph ^= 1u << b;
  };
  auto wait_noise = [&](int k) {
    const int b = k % G::NSTG;
    mbar_wait(&barN[b], (nph >> b) & 1u);
    nph ^= 1u << b;
  };
  uint64_t klabel = 0;
  if (!PRE && !cw && !pw && live) klabel = derive_label(noise.keys[c_begin + chain], kBackwardNoise);

  // Phase A, superchunk k, warp group `warp`: per step pair the offsets (c_hi, p_lo)
  // (two DMMAs, independent across pairs: gathered first), then the zero-carry
  // reduction over the 8 pairs (one dependent DMMA per pair); the group aggregate goes
  // to cagg(k), (c_hi, p_lo) stay in registers for phase C.
  auto phase_a = [&](int k, double* ch, double* pl) {
    wait_tile(k);
    if (PRE) wait_noise(k);
    const double* tl = tile(k) + warp * G::NP * G::PR;
    const double* X = xin(k) + chain * G::ROW + warp * GS * D + dim;
    const int lo = k * S + warp * GS;
    auto xi_at = [&](int s) {
      const int t = lo + s;
      double v = 0.0;
      if (live && t < T) v = PRE ? X[s * D] : normal_at(derive_index(klabel, (uint64_t)t), (uint64_t)dim);
      return v;
    };
#pragma unroll
    for (int j = 0; j < G::NP; ++j) {
      const double* r = tl + j * G::PR;
      const double2 oc = *reinterpret_cast<const double2*>(r + 80 + 2 * dim);
      double c_hi, gc;
      dmma2(xi_at(2 * j + 1), r[32 + lane], oc.x, oc.y, c_hi, gc);
      double c_lo, p_lo;  // c_lo (= L_lo xi_lo) unused
      dmma2(xi_at(2 * j), r[64 + 4 * (lane >> 3) + dim], 0.0, gc, c_lo, p_lo);
      ch[j] = c_hi;
      pl[j] = p_lo;
    }
    double bf[G::NP];
#pragma unroll
    for (int j = 0; j < G::NP; ++j) bf[j] = tl[j * G::PR + lane];
    double y = pl[G::NP - 1];  // zero carry: the top pair gives (c_hi, p_lo) itself
#pragma unroll
    for (int j = G::NP - 2; j >= 0; --j) {
      double y_hi;
      dmma2(y, bf[j], ch[j], pl[j], y_hi, y);
    }
    cagg(k)[warp * 32 + lane] = y;
  };

  double chA[G::NP], plA[G::NP], chB[G::NP], plB[G::NP];
  if (!cw && !pw) phase_a(K - 1, chA, plA);
  __syncthreads();

#if AUXMC_PM_EXP == 9  // clock64 stamps of 16 steady-state superchunks (tools/c2_stamps.py)
  __shared__ long long ts[16 * 8];
  auto stamp = [&](int k, int e) {
    const int it = K - 1 - k - 100;
    if (blockIdx.x == 0 && lane == 0 && it >= 0 && it < 16) ts[it * 8 + e] = clock64();
  };
#endif
  for (int k = K - 1; k >= 0; --k) {
    const int t0 = k * S;
#if AUXMC_PM_EXP == 9
    if (cw) {
      stamp(k, 0);
      stamp(k, 1);
    } else if (warp == 0) {
      stamp(k, 4);
    }
#endif
    if (pw) {
      if (lane == 0 && k >= 2) {  // stages of tile k+1 / noise k were consumed last iteration
        issue_tile(k - 2);
        if (PRE) issue_noise(k - 2);
      }
    } else if (cw) {
      // Phase B: x_top of each warp group from the incoming carry, top-down
      wait_tile(k);
#if AUXMC_PM_EXP == 9
      stamp(k, 2);
#endif
      const double* gw = tile(k) + G::EB;
      const double* ca = cagg(k);
      double gwf[W], cav[W];  // operands first: the stores below may not alias them
#pragma unroll
      for (int w = 0; w < W; ++w) {
        gwf[w] = bcol ? gw[w * 16 + boff] : 0.0;
        cav[w] = ca[w * 32 + lane];
      }
      double x = carry[lane];
#pragma unroll
      for (int w = W - 1; w >= 0; --w) {
        xwtop[w * 32 + lane] = x;
        x = dmma_d0(x, gwf[w], cav[w]);
      }
      carry[lane] = x;
#if AUXMC_PM_EXP == 9
      stamp(k, 3);
#endif
    } else if (k >= 1) {
      phase_a(k - 1, chB, plB);
#if AUXMC_PM_EXP == 9
      if (warp == 0) stamp(k, 5);
#endif
    }
    __syncthreads();
#if AUXMC_PM_EXP == 9
    if (!cw && !pw && warp == 0) stamp(k, 6);
#endif
    if (!cw && !pw) {  // Phase C: both steps of a pair per DMMA from the group's top state
      const double* tl = tile(k) + warp * G::NP * G::PR;
      const int lo = t0 + warp * GS;
      double bf[G::NP];  // operands first: the path stores may not alias shared memory
#pragma unroll
      for (int j = 0; j < G::NP; ++j) bf[j] = tl[j * G::PR + lane];
      double x = xwtop[warp * 32 + lane];
#pragma unroll
      for (int j = G::NP - 1; j >= 0; --j) {
        const int t = lo + 2 * j;
        double x_hi;
        dmma2(x, bf[j], chA[j], plA[j], x_hi, x);
        if (live && t + 1 < T) out_row[(size_t)(t + 1) * D] = x_hi;
        if (live && t < T) out_row[(size_t)t * D] = x;
      }
#pragma unroll
      for (int j = 0; j < G::NP; ++j) {
        chA[j] = chB[j];
        plA[j] = plB[j];
      }
#if AUXMC_PM_EXP == 9
      if (warp == 0) stamp(k, 7);
#endif
    }
    __syncthreads();
  }
#if AUXMC_PM_EXP == 9
  __syncthreads();
  if (blockIdx.x == 0 && tid < 128) reinterpret_cast<long long*>(traj)[tid] = ts[tid];
#endif
}

int run_prefix_mma(int T, int B, const double* elems, const double* term, Arena& ws,
                   const NoiseArgs& nz, double* traj, cudaStream_t stream) {
  using G = MmaGeom;
  const int K = T > 0 ? (T + G::S - 1) / G::S : 1;
  double* tiles = ws.take<double>((size_t)K * G::TB);
  if (ws.base == nullptr) return AUXMC_OK;
  if (!tiles) return AUXMC_E_WORKSPACE;
  if (nz.kind == AUXMC_NOISE_PREDRAWN && (reinterpret_cast<uintptr_t>(nz.backward) & 15))
    return AUXMC_E_ARG;  // cp.async.bulk stages noise rows: 16-B aligned source required
  if (T > 0) {
    const int np = K * (G::S / 2), ng = K * G::W;
    AUXMC_LAUNCH(k_mma_pack, std::min((np + 127) / 128, 148 * 32), 128, 0, stream, elems, T, tiles);
    AUXMC_LAUNCH(k_mma_spans, std::min((ng + 127) / 128, 148 * 16), 128, 0, stream, T, tiles);
  }
  const int grid = std::max((B + G::ROWS - 1) / G::ROWS, std::min(B, num_sms()));
  if (nz.kind == AUXMC_NOISE_PREDRAWN) {
    AUXMC_CUDA_TRY(cudaFuncSetAttribute(k_prefix_mma<true>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::SMEM));
    AUXMC_LAUNCH((k_prefix_mma<true>), grid, (G::W + 2) * 32, G::SMEM, stream, T, B, tiles, term,
                 nz, traj);
  } else {
    AUXMC_CUDA_TRY(cudaFuncSetAttribute(k_prefix_mma<false>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::SMEM));
    AUXMC_LAUNCH((k_prefix_mma<false>), grid, (G::W + 2) * 32, G::SMEM, stream, T, B, tiles, term,
                 nz, traj);
  }
  return AUXMC_OK;
}

}  // namespace auxmc_gpu
