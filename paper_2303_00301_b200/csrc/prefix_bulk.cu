// prefix_bulk.cu — bulk-copy (1-D TMA) variant of the shared-element prefix
// sampler (pit::prefix_sample, pit.cpp:78-115) for even state dimension.
//
// Same fixed reduce-then-scan tree family as prefix.cu, with all chain I/O done
// by the TMA engine: per superchunk, one bulk copy stages the packed elements
// and scan tables, one bulk copy per chain stages that chain's noise rows, and
// one bulk store per chain writes its path rows from shared memory.  No thread
// issues a global load or store in the steady state, so HBM sees full sectors
// in both directions.
//
// Thread map (8 warps): lane = slot + 8 q, slot = chain of the CTA (<= 8),
// sub-chunk j = 4 warp + q.  Sub-chunk carries are scanned in two levels:
// Kogge-Stone over the 4 sub-chunks of a warp (shuffles, chain-independent
// G-span tables), then a serial pass over the 8 warp aggregates per chain.
#include "common.cuh"
#include "dense.cuh"
#include "rng.cuh"
#include "tma.cuh"

// Kernel experiments (tools/exp_build.sh only; the product build leaves it 0):
// 1 = no tile / noise / path traffic (arithmetic and barriers alone).
#ifndef AUXMC_PB_EXP
#define AUXMC_PB_EXP 0
#endif

namespace auxmc_gpu {

template <int D>
struct BulkGeom {
  static constexpr int LS = 16 / D;        // steps per sub-chunk (D = 2, 4)
  static constexpr int NSUB = 32, WARPS = 8, SLOTS = 8;  // compute warps; lane slots
  static constexpr int ROWS = 7;           // chains per CTA (148 CTAs cover 1036 chains)
  static constexpr int S = NSUB * LS;      // steps per superchunk
  static constexpr int LP = D * (D + 1) / 2;
  static constexpr int ES = D * D + D + LP;
  // D = 4: sub-chunk blocks 16-B aligned (LDS.128) and 976 B apart, which puts
  // a warp's 4 sub-chunks on disjoint bank quads; odd D: an odd stride.
  static constexpr bool VEC = (ES % 2 == 0);
  static constexpr int SUB = VEC ? LS * ES + 2 : LS * ES + ((LS * ES) % 2 == 0 ? 1 : 0);
  static constexpr int EB = NSUB * SUB;
  static constexpr int TAB = 3 * NSUB * D * D;  // Gsub | Gpair | Gin
  static constexpr int TB = (EB + TAB + 1) & ~1;
  static constexpr int ROW = S * D + 2;    // io row stride: slot stride = 4 banks
  static constexpr int IOB = ROWS * ROW;
  static constexpr int TSTG = 3, NSTG = 2; // element-tile stages, noise stages
  static constexpr int CS = D + 2;         // per-(warp, slot) carry stride: conflict-free LDS.128
  static constexpr int CB = SLOTS * WARPS * CS;
  static constexpr size_t SMEM = sizeof(double) * (TSTG * TB + NSTG * IOB + IOB + 3 * CB +
                                                   SLOTS * D) +
                                 (TSTG + NSTG) * sizeof(uint64_t);
};
static_assert(BulkGeom<4>::SMEM <= 227 * 1024, "one CTA per SM");
static_assert(BulkGeom<2>::SMEM <= 227 * 1024, "one CTA per SM");

template <int D>
__device__ __forceinline__ void mat_mul(const double* A, const double* B, double* C) {
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int b = 0; b < D; ++b) {
      double acc = 0.0;
#pragma unroll
      for (int q = 0; q < D; ++q) acc += A[a * D + q] * B[q * D + b];
      C[a * D + b] = acc;
    }
}

// elements + Gsub per (superchunk, sub-chunk)
template <int D>
__global__ void k_bulk_pack1(const double* __restrict__ elems, int T, double* tiles) {
  using G = BulkGeom<D>;
  const int n_sub = ((T + G::S - 1) / G::S) * G::NSUB;
  const int ESg = elem_stride(D);
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < n_sub; s += gridDim.x * blockDim.x) {
    const int k = s / G::NSUB, j = s % G::NSUB;
    double* tile = tiles + (size_t)k * G::TB;
    double* blk = tile + j * G::SUB;
    const int lo = k * G::S + j * G::LS;
    double P[D * D], Q[D * D];
#pragma unroll
    for (int i = 0; i < D * D; ++i) P[i] = (i / D == i % D) ? 1.0 : 0.0;
    for (int q = G::LS - 1; q >= 0; --q) {
      const int t = lo + q;
      double* out = blk + q * G::ES;
      if (t >= T) {
        for (int i = 0; i < G::ES; ++i) out[i] = 0.0;
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
      mat_mul<D>(e, P, Q);
#pragma unroll
      for (int i = 0; i < D * D; ++i) P[i] = Q[i];
    }
    for (int i = G::LS * G::ES; i < G::SUB; ++i) blk[i] = 0.0;
    double* gs = tile + G::EB + j * D * D;
#pragma unroll
    for (int i = 0; i < D * D; ++i) gs[i] = P[i];
    if (j == 0 && G::TB > G::EB + G::TAB) tile[G::TB - 1] = 0.0;
  }
}

// Gpair_j = Gsub_j Gsub_{j+1} (j % 4 <= 2); Gin_j = Gsub_j ... Gsub_{4(j/4)+3}
template <int D>
__global__ void k_bulk_pack2(int T, double* tiles) {
  using G = BulkGeom<D>;
  const int n_sub = ((T + G::S - 1) / G::S) * G::NSUB;
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < n_sub; s += gridDim.x * blockDim.x) {
    const int k = s / G::NSUB, j = s % G::NSUB;
    double* tile = tiles + (size_t)k * G::TB;
    const double* gsub = tile + G::EB;
    double* gpair = tile + G::EB + G::NSUB * D * D;
    double* gin = gpair + G::NSUB * D * D;
    const int gend = 4 * (j / 4) + 3;
    double P[D * D], Q[D * D];
#pragma unroll
    for (int i = 0; i < D * D; ++i) P[i] = gsub[gend * D * D + i];
    for (int jj = gend - 1; jj >= j; --jj) {
      mat_mul<D>(gsub + jj * D * D, P, Q);
#pragma unroll
      for (int i = 0; i < D * D; ++i) P[i] = Q[i];
    }
#pragma unroll
    for (int i = 0; i < D * D; ++i) gin[j * D * D + i] = P[i];
    if (j < gend) {
      mat_mul<D>(gsub + j * D * D, gsub + (j + 1) * D * D, Q);
#pragma unroll
      for (int i = 0; i < D * D; ++i) gpair[j * D * D + i] = Q[i];
    } else {
#pragma unroll
      for (int i = 0; i < D * D; ++i) gpair[j * D * D + i] = 0.0;
    }
  }
}

// n (even) doubles from a 16-B aligned shared-memory address as LDS.128
template <int N>
__device__ __forceinline__ void lds_vec(const double* p, double* v) {
#pragma unroll
  for (int i = 0; i < N; i += 2) {
    const double2 t = *reinterpret_cast<const double2*>(p + i);
    v[i] = t.x;
    v[i + 1] = t.y;
  }
}

template <int D>
__device__ __forceinline__ void shfl_down_vec(const double* v, double* out, int delta) {
#pragma unroll
  for (int i = 0; i < D; ++i) out[i] = __shfl_down_sync(0xffffffffu, v[i], delta);
}

// Software-pipelined sweep.  Eight compute warps own (chain slot, sub-chunk)
// pairs; a ninth "carry" warp runs the serial pass over warp aggregates and
// drives the TMA engine.  Iteration k overlaps the carry pass of superchunk k
// with the reduction (phase A) of superchunk k-1, then expands superchunk k
// (phase C): two CTA barriers per superchunk.  Element tiles are triple
// buffered (tiles k and k-1 are live while k-2 streams in), noise rows double
// buffered, path rows single buffered (drained during the next phase A).
template <int D, bool PRE>
__global__ void __launch_bounds__((BulkGeom<D>::WARPS + 2) * 32, 1)
    k_prefix_bulk(int T, int C, const double* __restrict__ tiles, const double* __restrict__ term,
                  NoiseArgs noise, double* __restrict__ traj) {
  using G = BulkGeom<D>;
  constexpr int LS = G::LS, ES = G::ES, S = G::S, NS = G::NSUB, W = G::WARPS, CS = G::CS;
  extern __shared__ __align__(16) double sm[];
  auto tile = [&](int k) { return sm + (k % G::TSTG) * G::TB; };
  auto xin = [&](int k) { return sm + G::TSTG * G::TB + (k % G::NSTG) * G::IOB; };
  double* xo = sm + G::TSTG * G::TB + G::NSTG * G::IOB;
  auto cagg = [&](int k) { return xo + G::IOB + (k & 1) * G::CB; };  // [W][SLOTS][CS]
  double* xwtop = xo + G::IOB + 2 * G::CB;                             // [W][SLOTS][CS]
  double* carry = xwtop + G::CB;                                       // [SLOTS][D]
  uint64_t* barT = reinterpret_cast<uint64_t*>(carry + G::SLOTS * D);
  uint64_t* barN = barT + G::TSTG;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool cw = warp == W;      // carry warp (phase B)
  const bool pw = warp == W + 1;  // producer warp: every TMA load and store
  const int slot = lane & 7, q = lane >> 3, j = warp * 4 + q;
  const int c_begin = (int)(((long long)blockIdx.x * C) / gridDim.x);
  const int c_end = (int)(((long long)(blockIdx.x + 1) * C) / gridDim.x);
  const int nc = c_end - c_begin;
  const int c = c_begin + slot;
  const bool active = slot < nc;
  const long long row = (long long)(T + 1) * D;

  if (tid == 0) {
    for (int b = 0; b < G::TSTG; ++b) mbar_init(&barT[b], 1);
    for (int b = 0; b < G::NSTG; ++b) mbar_init(&barN[b], 1);
    mbar_fence_init();
  }
  if (cw && lane < 8 && active) {  // x_T = m_T + L_T xi (pit.cpp:85-87)
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
      traj[(size_t)c * row + (size_t)T * D + i] = x[i];
    }
  }
  __syncthreads();
  if (T == 0) return;
  const int K = (T + S - 1) / S;
  auto issue_tile = [&](int k) {
    if (AUXMC_PB_EXP == 1) return;
    const unsigned tb = G::TB * sizeof(double);
    uint64_t* bar = &barT[k % G::TSTG];
    mbar_expect_tx(bar, tb);
    bulk_g2s(tile(k), tiles + (size_t)k * G::TB, tb, bar);
  };
  auto issue_noise = [&](int k) {
    if (AUXMC_PB_EXP == 1) return;
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
  unsigned tph = 0u, nph = 0u;  // per-stage mbarrier parities seen by this thread
  auto wait_tile = [&](int k) {
    if (AUXMC_PB_EXP == 1) return;
    const int b = k % G::TSTG;
    mbar_wait(&barT[b], (tph >> b) & 1u);
    tph ^= 1u << b;
  };
  auto wait_noise = [&](int k) {
    if (AUXMC_PB_EXP == 1) return;
    const int b = k % G::NSTG;
    mbar_wait(&barN[b], (nph >> b) & 1u);
    nph ^= 1u << b;
  };
  uint64_t klabel = 0;
  if (!PRE && !cw && !pw && active) klabel = derive_label(noise.keys[c], kBackwardNoise);

  // Phase A for superchunk k: realize c_t = off_t + L_t xi_t, reduce each
  // sub-chunk (zero carry), Kogge-Stone over the warp's 4 sub-chunks; the warp
  // aggregates go to cagg(k).
  auto phase_a = [&](int k, double* cs, double* y) {
    wait_tile(k);
    if (PRE) wait_noise(k);
    const double* tl = tile(k);
    const int t0 = k * S, t1 = min(t0 + S, T);
    const int lo = t0 + j * LS;
    const bool full = (t1 - t0) == S;
    const double* E = tl + j * G::SUB;
    const double* gsub = tl + G::EB;
    const double* gpair = gsub + NS * D * D;
    const double* X = xin(k) + slot * G::ROW + j * LS * D;
#pragma unroll
    for (int i = 0; i < D; ++i) y[i] = 0.0;
    if (full && G::VEC) {
      // full superchunk: the LS offsets c_t are independent — realize them all
      // first, then run the dependent chain y = G_t y + c_t (same arithmetic)
#pragma unroll
      for (int s = LS - 1; s >= 0; --s) {
        const int t = lo + s;
        double xi[D];
        if (PRE) {
          lds_vec<D>(X + s * D, xi);
        } else {
          const uint64_t key = derive_index(klabel, (uint64_t)t);
#pragma unroll
          for (int i = 0; i < D; ++i) xi[i] = normal_at(key, (uint64_t)i);
        }
        double lv[D + G::LP];  // off | L packed
        lds_vec<D + G::LP>(E + s * ES + D * D, lv);
        int w = 0;
#pragma unroll
        for (int r = 0; r < D; ++r) {
          double acc = 0.0;
#pragma unroll
          for (int cc = 0; cc <= r; ++cc) acc += lv[D + w++] * xi[cc];
          cs[s * D + r] = lv[r] + acc;
        }
      }
#pragma unroll
      for (int s = LS - 1; s >= 0; --s) {
        double gm[D * D], gy[D];
        lds_vec<D * D>(E + s * ES, gm);
        r_matvec<D>(gm, y, gy);
#pragma unroll
        for (int r = 0; r < D; ++r) y[r] = gy[r] + cs[s * D + r];
      }
    } else {
#pragma unroll
    for (int s = LS - 1; s >= 0; --s) {
      const int t = lo + s;
      if (full || t < t1) {  // inactive slots compute on scratch rows; only live rows are stored
        const double* e = E + s * ES;
        double xi[D];
        if (PRE) {
#pragma unroll
          for (int i = 0; i < D; i += 2) {
            const double2 v = *reinterpret_cast<const double2*>(X + s * D + i);
            xi[i] = v.x;
            xi[i + 1] = v.y;
          }
        } else {
          const uint64_t key = derive_index(klabel, (uint64_t)t);
#pragma unroll
          for (int i = 0; i < D; ++i) xi[i] = normal_at(key, (uint64_t)i);
        }
        double ev[G::VEC ? ES : 1];
        const double* er = e;
        if constexpr (G::VEC) {
          lds_vec<ES>(e, ev);
          er = ev;
        }
        double gy[D];
        r_matvec<D>(er, y, gy);
        int w = 0;
#pragma unroll
        for (int r = 0; r < D; ++r) {
          double acc = 0.0;
#pragma unroll
          for (int cc = 0; cc <= r; ++cc) acc += er[D * D + D + w++] * xi[cc];
          const double cv = er[D * D + r] + acc;
          cs[s * D + r] = cv;
          y[r] = gy[r] + cv;
        }
      } else {
#pragma unroll
        for (int r = 0; r < D; ++r) cs[s * D + r] = 0.0;
      }
    }
    }
    double yn[D], gy[D];  // suffix Kogge-Stone: y -> c over [j, group end)
    shfl_down_vec<D>(y, yn, 8);
    if (q < 3) {
      r_matvec<D>(gsub + j * D * D, yn, gy);
#pragma unroll
      for (int i = 0; i < D; ++i) y[i] = gy[i] + y[i];
    }
    shfl_down_vec<D>(y, yn, 16);
    if (q < 2) {
      r_matvec<D>(gpair + j * D * D, yn, gy);
#pragma unroll
      for (int i = 0; i < D; ++i) y[i] = gy[i] + y[i];
    }
    if (q == 0) {
#pragma unroll
      for (int i = 0; i < D; ++i) cagg(k)[(warp * G::SLOTS + slot) * CS + i] = y[i];
    }
  };

  double csA[LS * D], yA[D], csB[LS * D], yB[D];
  if (!cw && !pw) phase_a(K - 1, csA, yA);
  __syncthreads();

  for (int k = K - 1; k >= 0; --k) {
    const int t0 = k * S, t1 = min(t0 + S, T);
    if (pw) {
      // loads of superchunk k-2 into the stages of tile k+1 / noise k (consumed), then
      // the path store of superchunk k+1 must have left xo before phase C(k) rewrites
      // it: the wait overlaps phases A / B instead of delaying them
      if (lane == 0) {
        if (k >= 2) {
          issue_tile(k - 2);
          if (PRE) issue_noise(k - 2);
        }
        bulk_wait_read<0>();
      }
      __syncwarp();
    } else if (cw) {
      // Phase B (carry): serial pass over the 8 warp aggregates, top-down
      wait_tile(k);
      if (lane < 8 && active) {
        const double* gin = tile(k) + G::EB + 2 * NS * D * D;
        const double* ca = cagg(k);
        double x[D];
#pragma unroll
        for (int i = 0; i < D; ++i) x[i] = carry[slot * D + i];
        // warps whose sub-chunks start at or past t1 (partial last superchunk) pass x through
        const int wlive = min(W, (t1 - t0 + 4 * LS - 1) / (4 * LS));
        for (int w = W - 1; w >= wlive; --w) {
#pragma unroll
          for (int i = 0; i < D; ++i) xwtop[(w * G::SLOTS + slot) * CS + i] = x[i];
        }
#pragma unroll
        for (int w = W - 1; w >= 0; --w) {
          if (w < wlive) {
#pragma unroll
            for (int i = 0; i < D; ++i) xwtop[(w * G::SLOTS + slot) * CS + i] = x[i];
            double gm[D * D], gx[D];
            if constexpr (G::VEC) {
              lds_vec<D * D>(gin + 4 * w * D * D, gm);
            } else {
#pragma unroll
              for (int i = 0; i < D * D; ++i) gm[i] = gin[4 * w * D * D + i];
            }
            r_matvec<D>(gm, x, gx);
#pragma unroll
            for (int i = 0; i < D; ++i) x[i] = gx[i] + ca[(w * G::SLOTS + slot) * CS + i];
          }
        }
#pragma unroll
        for (int i = 0; i < D; ++i) carry[slot * D + i] = x[i];
      }
    } else if (k >= 1) {
      phase_a(k - 1, csB, yB);
    }
    __syncthreads();
    if (!cw && !pw) {  // Phase C: x at the top of each sub-chunk, then x_t = G_t x_{t+1} + c_t
      const double* tl = tile(k);
      const double* E = tl + j * G::SUB;
      const double* gin = tl + G::EB + 2 * NS * D * D;
      const int lo = t0 + j * LS;
      const bool full = (t1 - t0) == S;
      double xt[D], xb[D], xn[D], x[D];
#pragma unroll
      for (int i = 0; i < D; ++i) xt[i] = xwtop[(warp * G::SLOTS + slot) * CS + i];
      r_matvec<D>(gin + j * D * D, xt, xb);
#pragma unroll
      for (int i = 0; i < D; ++i) xb[i] = xb[i] + yA[i];
      shfl_down_vec<D>(xb, xn, 8);
#pragma unroll
      for (int i = 0; i < D; ++i) x[i] = q < 3 ? xn[i] : xt[i];
      double* XO = xo + slot * G::ROW + j * LS * D;
      const bool live = slot < G::ROWS;
      if (full && G::VEC) {
        double xs[LS * D];
#pragma unroll
        for (int s = LS - 1; s >= 0; --s) {
          double gm[D * D], gx[D];
          lds_vec<D * D>(E + s * ES, gm);
          r_matvec<D>(gm, x, gx);
#pragma unroll
          for (int i = 0; i < D; ++i) x[i] = gx[i] + csA[s * D + i];
#pragma unroll
          for (int i = 0; i < D; ++i) xs[s * D + i] = x[i];
        }
        if (live) {
#pragma unroll
          for (int i = 0; i < LS * D; i += 2)
            *reinterpret_cast<double2*>(XO + i) = make_double2(xs[i], xs[i + 1]);
        }
      } else
#pragma unroll
      for (int s = LS - 1; s >= 0; --s) {
        const int t = lo + s;
        if (full || t < t1) {
          double gx[D];
          if constexpr (G::VEC) {
            double gm[D * D];
            lds_vec<D * D>(E + s * ES, gm);
            r_matvec<D>(gm, x, gx);
          } else {
            r_matvec<D>(E + s * ES, x, gx);
          }
#pragma unroll
          for (int i = 0; i < D; ++i) x[i] = gx[i] + csA[s * D + i];
          if (live) {
#pragma unroll
            for (int i = 0; i < D; i += 2)
              *reinterpret_cast<double2*>(XO + s * D + i) = make_double2(x[i], x[i + 1]);
          }
        }
      }
      fence_proxy_async();
#pragma unroll
      for (int i = 0; i < LS * D; ++i) csA[i] = csB[i];
#pragma unroll
      for (int i = 0; i < D; ++i) yA[i] = yB[i];
    }
    __syncthreads();
    if (pw && lane == 0 && AUXMC_PB_EXP != 1) {
      const unsigned xb = (unsigned)((t1 - t0) * D * sizeof(double));
      for (int ch = 0; ch < nc; ++ch)
        bulk_s2g(traj + (size_t)(c_begin + ch) * row + (size_t)t0 * D, xo + ch * G::ROW, xb);
      bulk_commit();
    }
  }
  if (pw && lane == 0) bulk_wait<0>();
}

template <int D>
int run_prefix_bulk(int T, int B, const double* elems, const double* term, Arena& ws,
                    const NoiseArgs& nz, double* traj, cudaStream_t stream) {
  using G = BulkGeom<D>;
  const int K = T > 0 ? (T + G::S - 1) / G::S : 1;
  double* tiles = ws.take<double>((size_t)K * G::TB);
  if (ws.base == nullptr) return AUXMC_OK;
  if (!tiles) return AUXMC_E_WORKSPACE;
  if (nz.kind == AUXMC_NOISE_PREDRAWN && (reinterpret_cast<uintptr_t>(nz.backward) & 15))
    return AUXMC_E_ARG;  // cp.async.bulk stages noise rows: 16-B aligned source required
  if (T > 0) {
    const int n_sub = K * G::NSUB;
    const int grid = std::min((n_sub + 127) / 128, 148 * 16);
    AUXMC_LAUNCH(k_bulk_pack1<D>, grid, 128, 0, stream, elems, T, tiles);
    AUXMC_LAUNCH(k_bulk_pack2<D>, grid, 128, 0, stream, T, tiles);
  }
  const int grid = std::max((B + G::ROWS - 1) / G::ROWS, std::min(B, num_sms()));
  if (nz.kind == AUXMC_NOISE_PREDRAWN) {
    AUXMC_CUDA_TRY(cudaFuncSetAttribute(k_prefix_bulk<D, true>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::SMEM));
    AUXMC_LAUNCH((k_prefix_bulk<D, true>), grid, (G::WARPS + 2) * 32, G::SMEM, stream, T, B, tiles,
                 term, nz, traj);
  } else {
    AUXMC_CUDA_TRY(cudaFuncSetAttribute(k_prefix_bulk<D, false>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::SMEM));
    AUXMC_LAUNCH((k_prefix_bulk<D, false>), grid, (G::WARPS + 2) * 32, G::SMEM, stream, T, B,
                 tiles, term, nz, traj);
  }
  return AUXMC_OK;
}

template int run_prefix_bulk<2>(int, int, const double*, const double*, Arena&, const NoiseArgs&,
                                double*, cudaStream_t);


}  // namespace auxmc_gpu
