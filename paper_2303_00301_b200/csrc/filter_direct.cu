// filter_direct.cu — the structure-aware sequential Kalman filter of the auxiliary
// LGSSM (auxk.cpp:68-110 build_aux_lgssm; filtered by lgssm.cpp:86-111).
//
// Every auxiliary model observes the whole state directly: z_t = [u_t; y_t] with
// H = [I; H_e], R = diag(δ/2 I, R_e) (k_build_HR).  When each exact row of H_e picks
// ONE state component with unit gain (distinct components) and R_e is diagonal — the
// diffusion-smoothing models (Lorenz-63/96: every other coordinate observed), and every
// target without exact rows — the two observations of a component fuse into one:
//
//   N(u_i; x_i, a) N(y'_k; x_i, b) = N(w_i; x_i, r_i) N(u_i; y'_k, a + b),
//   r_i = ab/(a+b),  w_i = (u_i b + y'_k a)/(a+b),  y' = y - c,
//
// so the update is one d-dimensional direct observation (H = I, R = diag r) plus a
// closed-form per-component term, instead of the (d+q)-dimensional innovation of the
// generic filter (k_filter_cta).  The outputs are the same quantities — predicted and
// filtered moments, log p(z_{0:T}) — in different association (FP64 parity tolerance).
//
// The update is ONE elimination.  On the bordered matrix
//
//        [ S      P_p   v ]        S = P_p + diag r,  v = w - m_p,
//   M =  [ P_p    P_p   0 ]
//        [ v^T    0     0 ]
//
// the first d pivots of a symmetric (LDL^T) elimination leave the Schur complement
// [[P_p - P_p S^-1 P_p, -K v], [., -v^T S^-1 v]]: the filtered covariance, minus the
// mean correction and minus the innovation's quadratic form; the pivots are the D of
// S = L D L^T (log det S = Σ log pivot).  No square root or triangular solve sits on
// the step's critical path.  The CTA holds M in registers as 4×4 tiles of its lower
// triangle (one tile per thread for d <= 40: 231 tiles of the 81×81 matrix); each
// pivot step is one barrier, one broadcast of the pivot column through shared memory
// and 16 FMAs per tile.
//
// The dynamics' Jacobian F_t = I + h J(x_t) of Lorenz-96 has four nonzeros per row
// (target.cuh dyn_jac_ij); it is formed on the fly from the linearisation point, so
// the predict step F P F^T costs 8d^2 FMAs and F is never written to HBM.  Other
// targets read a shared dense F.  One CTA per chain; the next step's inputs are
// prefetched into registers while the current step eliminates.
#include "common.cuh"
#include "dense.cuh"
#include "target.cuh"

namespace auxmc_gpu {

constexpr int kFdThreads = 256;
constexpr double kLog2PiD = 1.8378770664093454835606594728112;

__host__ __device__ inline int fd_nt(int d) { return (2 * d + 1 + 3) / 4; }
__host__ __device__ inline int fd_tiles(int d) { return fd_nt(d) * (fd_nt(d) + 1) / 2; }
__host__ __device__ inline int fd_nt8(int d) { return (2 * d + 1 + 7) / 8; }

#ifndef AUXMC_FD_EXP
#define AUXMC_FD_EXP 0  // 9: clock64 phase stamps of CTA 0 (tools/fd_stamps.py)
#endif
#if AUXMC_FD_EXP == 9
__device__ long long g_fd_stamps[4096];
#define FD_STAMP(slot)                                                   \
  do {                                                                   \
    if (stamp_on && (threadIdx.x & 31) == 0)                             \
      g_fd_stamps[(threadIdx.x >> 5) * 512 + (slot)] = clock64();        \
  } while (0)
#else
#define FD_STAMP(slot) \
  do {                 \
  } while (0)
#endif

constexpr int kFdWarps = kFdThreads / 32;
constexpr int kFdTpw = 9;  // 8×8 tiles per warp: 66 tiles of the lower triangle for d <= 43

// shared-memory layout (doubles)
struct FdLayout {
  int P, A, Pp, Q, F, fv, fc, m, mp, w, r, ex, col, piv, in, bq, cq, sel, red, Rb, Dv, tab, total;
  __host__ __device__ FdLayout(int d, int q, bool fst) {
    const int dd = d * d, npad = 4 * fd_nt(d), nin = (d + q) + 2 * d;
    int o = 0;
    P = o; o += dd;
    A = o; o += dd;
    Pp = o; o += dd;
    Q = o; o += dd;
    F = o; o += fst ? 0 : dd;
    fv = o; o += 4 * d;
    fc = o; o += 2 * d;  // 4d ints
    m = o; o += d;
    mp = o; o += d;
    w = o; o += d;
    r = o; o += d;
    ex = o; o += d;
    col = o; o += 2 * npad;
    piv = o; o += d;
    bq = o; o += d;
    cq = o; o += d;
    sel = o; o += (d + 1) / 2;  // d ints
    red = o; o += 4;
    o = (o + 1) & ~1;  // 16-byte alignment for the double2 panel / D^{-1} loads
    Rb = o; o += 2 * 4 * 8 * fd_nt8(d);  // MMA panels (double-buffered)
    Dv = o; o += 16;  // D^{-1} of the current pivot block
    tab = o; o += 2 * kFdWarps * kFdTpw;  // int4 per (warp, slot)
    in = o; o += 2 * nin;  // last: the only q-dependent block
    total = o;
  }
};

// factor_psd's jitter scale (gauss.cpp:20-24) of S = P_p + diag r: trace / d, else max |S|
__device__ __forceinline__ double jitter_scale(int tid, int d, const double* Pp, const double* r,
                                               double* red) {
  if (tid == 0) {
    double tr = 0.0;
    for (int i = 0; i < d; ++i) tr += Pp[i * d + i] + r[i];
    double sc = tr / static_cast<double>(d);
    if (sc <= 0.0) {
      double mx = 0.0;
      for (int i = 0; i < d; ++i)
        for (int j = 0; j < d; ++j) {
          const double v = Pp[i * d + j] + (i == j ? r[i] : 0.0);
          mx = fabs(v) > mx ? fabs(v) : mx;
        }
      sc = mx;
    }
    red[2] = sc;
  }
  __syncthreads();
  return red[2];
}

// entry (i, j) of the bordered matrix M (symmetric: the lower triangle is stored)
__device__ __forceinline__ double fd_mval(int i, int j, int d, int n, const double* Pp,
                                          const double* r, const double* w, const double* mp,
                                          double eps) {
  if (j > i) {
    const int tq = i;
    i = j;
    j = tq;
  }
  if (i >= n) return 0.0;
  if (i < d) return Pp[i * d + j] + (i == j ? r[i] + eps : 0.0);
  if (i < 2 * d) return j < d ? Pp[(i - d) * d + j] : Pp[(i - d) * d + (j - d)];
  return j < d ? w[j] - mp[j] : 0.0;
}

// Schur-complement readout of entry (i, j) of the eliminated M: P_f, m_f, v^T S^-1 v
__device__ __forceinline__ void fd_readout(int i, int j, double v, int d, int n, const double* mp,
                                           double* P, double* mv, double* red) {
  if (i < d || j < d || j > i || i >= n) return;
  if (i < 2 * d) {
    P[(i - d) * d + (j - d)] = v;
    P[(j - d) * d + (i - d)] = v;
  } else if (j < 2 * d) {
    mv[j - d] = mp[j - d] - v;
  } else {
    red[0] = -v;  // v^T S^-1 v
  }
}

__device__ __forceinline__ double rcp_nr(double x) {  // 1/x: MUFU seed + two Newton steps
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  return fma(y, e, y);
}

__host__ __device__ inline bool fd_use_mma(int d) {
  return fd_nt8(d) * (fd_nt8(d) + 1) / 2 <= kFdWarps * kFdTpw;
}

// Blocked LDL^T of the bordered matrix on the FP64 tensor cores (d <= 43).  M's lower
// triangle lives in DMMA accumulators, one 8×8 tile per (warp, slot) — lane l holds
// (8I + l/4, 8J + 2(l%4) + {0,1}), the m8n8k4 C layout.  Pivots go in panels of four:
// the owners publish the panel R = M[:, kb:kb+4] (rows above kb zero) through shared
// memory (double-buffered); after a barrier warp 0 forms D^{-1} of the 4×4 pivot block
// by cofactors (lane 4i + j one 3×3 minor; det by a fixed two-level shuffle sum) and
// tests the leading minors — S is SPD iff all are > 0, the reference's LLT criterion;
// after a second barrier every tile takes the rank-4 update M -= R D^{-1} R^T as one
// DMMA (A = -R rows of the tile, B = R D^{-1} rows of its columns, formed per slot from
// the tile's R row and the lane's column of D^{-1}).  log det S = Σ log det D_p,
// dets[p] per panel.  (Variants measured slower: DESIGN.md §5.2.)
//
// tab (shared, warp-uniform): per (warp, slot) {I, J, src, kind}: kind 0 a P_p block
// tile read at P_p[src + row*d + col], 1 the same on the S diagonal (+ r + jitter),
// 2 the v row's tiles, 3 unowned, 4 a tile straddling blocks (d % 8 != 0: entrywise).
struct FdTile {
  int I, J, src, kind;
};
__device__ __forceinline__ FdTile fd_tile_ij(int I, int J, int d) {
  if (d % 8 != 0) return FdTile{I, J, 0, 4};
  const int r0 = 8 * I, c0 = 8 * J;
  if (r0 >= 2 * d) return FdTile{I, J, 0, 2};
  const int rb = r0 < d ? r0 : r0 - d, cb = c0 < d ? c0 : c0 - d;
  return FdTile{I, J, rb * d + cb, (r0 < d && I == J) ? 1 : 0};
}
// tile of (warp, slot): round robin over the row-major order (tile warp + 8 slot)
__device__ __forceinline__ FdTile fd_tile_of(int warp, int slot, int d) {
  const int nt8 = fd_nt8(d);
  const int tau = warp + kFdWarps * slot, ntile8 = nt8 * (nt8 + 1) / 2;
  if (tau >= ntile8) return FdTile{0, 0, 0, 3};
  int I = 0;
  while ((I + 1) * (I + 2) / 2 <= tau) ++I;
  return fd_tile_ij(I, tau - I * (I + 1) / 2, d);
}

__device__ __forceinline__ bool elim_mma(int tid, int d, int n, const double* Pp, const double* r,
                                         const double* w, const double* mp, double* Rb,
                                         double* dets, double* P, double* mv, double* red,
                                         const int4* __restrict__ tab, double* Dv,
                                         bool stamp_on) {
  (void)stamp_on;
  const int lane = tid & 31, warp = tid >> 5;
  const int gi = lane >> 2, ti = lane & 3;
  const int rstride = 4 * 8 * fd_nt8(d);
  const int4* wt = tab + warp * kFdTpw;
  double c[kFdTpw][2];
  bool ok = false;
  double jit = 0.0;
  for (int attempt = 0; attempt < 3 && !ok; ++attempt) {
    if (attempt == 1) jit = jitter_scale(tid, d, Pp, r, red);
    const double eps = attempt == 0 ? 0.0 : (attempt == 1 ? 1e-10 : 1e-8) * jit;
#pragma unroll
    for (int s = 0; s < kFdTpw; ++s) {
      const int4 tt = wt[s];
      const int i = 8 * tt.x + gi, j = 8 * tt.y + 2 * ti;
      double v0 = 0.0, v1 = 0.0;
      if (tt.w <= 1) {
        const double2 pv = *reinterpret_cast<const double2*>(Pp + tt.z + gi * d + 2 * ti);
        v0 = pv.x;
        v1 = pv.y;
        if (tt.w == 1) {
          if (i == j) v0 += r[i] + eps;
          if (i == j + 1) v1 += r[i] + eps;
        }
      } else if (tt.w == 2) {
        if (i == 2 * d && j < d) {
          v0 = w[j] - mp[j];
          v1 = j + 1 < d ? w[j + 1] - mp[j + 1] : 0.0;
        }
      } else if (tt.w == 4) {
        v0 = fd_mval(i, j, d, n, Pp, r, w, mp, eps);
        v1 = fd_mval(i, j + 1, d, n, Pp, r, w, mp, eps);
      }
      c[s][0] = v0;
      c[s][1] = v1;
    }
    bool failed = false;
    for (int kb = 0; kb < d; kb += 4) {
      const int Jp = kb >> 3, half = (kb >> 2) & 1;
      double* R = Rb + ((kb >> 2) & 1) * rstride;
      // panel columns kb..kb+3 from their owners (pivot columns past d stay zero)
#pragma unroll
      for (int s = 0; s < kFdTpw; ++s) {
        const int4 tt = wt[s];
        if (tt.y == Jp && tt.w != 3 && (ti >> 1) == half) {
          const int row = 8 * tt.x + gi, m0 = 2 * ti - 4 * half;
          const bool live = row >= kb;
          *reinterpret_cast<double2*>(R + row * 4 + m0) =
              make_double2(live && kb + m0 < d ? c[s][0] : 0.0, live && kb + m0 + 1 < d ? c[s][1] : 0.0);
        }
      }
      __syncthreads();
      FD_STAMP(8 + 3 * (kb >> 2));
      if (warp == 0) {  // D^{-1} of the 4×4 pivot block by cofactors (lane 4i + j)
        auto D = [&](int a, int b) -> double {
          const int hi = a > b ? a : b, lo = a > b ? b : a;
          if (kb + hi >= d) return a == b ? 1.0 : 0.0;
          return R[(kb + hi) * 4 + lo];
        };
        const int i = (lane >> 2) & 3, j = lane & 3;
        const int r0 = i == 0 ? 1 : 0, r1 = i <= 1 ? 2 : 1, r2 = i <= 2 ? 3 : 2;
        const int c0 = j == 0 ? 1 : 0, c1 = j <= 1 ? 2 : 1, c2 = j <= 2 ? 3 : 2;
        const double m3 = D(r0, c0) * (D(r1, c1) * D(r2, c2) - D(r1, c2) * D(r2, c1)) -
                          D(r0, c1) * (D(r1, c0) * D(r2, c2) - D(r1, c2) * D(r2, c0)) +
                          D(r0, c2) * (D(r1, c0) * D(r2, c1) - D(r1, c1) * D(r2, c0));
        double cof = ((i + j) & 1) ? -m3 : m3;
        cof = __shfl_sync(0xffffffffu, cof, i <= j ? (lane & 15) : 4 * j + i);  // symmetric
        double pr = lane < 4 ? D(0, lane) * cof : 0.0;
        pr += __shfl_xor_sync(0xffffffffu, pr, 1);
        pr += __shfl_xor_sync(0xffffffffu, pr, 2);
        const double det = __shfl_sync(0xffffffffu, pr, 0);
        const double lead3 = __shfl_sync(0xffffffffu, cof, 15);
        const double d00 = D(0, 0), lead2 = d00 * D(1, 1) - D(1, 0) * D(1, 0);
        const bool good = d00 > 0.0 && lead2 > 0.0 && lead3 > 0.0 && det > 0.0;
        const double rd = rcp_nr(det);
        const double dij = cof * rd;  // (D^{-1})_{ij} on lane 4i + j
        if (lane < 16) Dv[lane] = dij;
        if (lane == 0) {
          dets[kb >> 2] = det;
          red[3] = good ? 0.0 : 1.0;
        }
      }
      __syncthreads();
      FD_STAMP(9 + 3 * (kb >> 2));
      if (red[3] != 0.0) {
        failed = true;
        break;
      }
      double q[4];  // column ti of D^{-1}: this lane's B-operand weights
      {
        const double2 q01 = *reinterpret_cast<const double2*>(Dv + 4 * ti);
        const double2 q23 = *reinterpret_cast<const double2*>(Dv + 4 * ti + 2);
        q[0] = q01.x;
        q[1] = q01.y;
        q[2] = q23.x;
        q[3] = q23.y;
      }
#pragma unroll
      for (int s = 0; s < kFdTpw; ++s) {
        const int4 tt = wt[s];
        if (tt.y < Jp || tt.w == 3) continue;  // retired (all columns < kb) or unowned
        const double a = -R[(8 * tt.x + gi) * 4 + ti];
        const double2* rj = reinterpret_cast<const double2*>(R + (8 * tt.y + gi) * 4);
        const double2 r01 = rj[0], r23 = rj[1];
        const double y = (r01.x * q[0] + r01.y * q[1]) + (r23.x * q[2] + r23.y * q[3]);
        asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
            : "+d"(c[s][0]), "+d"(c[s][1])
            : "d"(a), "d"(y));
      }
      FD_STAMP(10 + 3 * (kb >> 2));
    }
    ok = !failed;
    if (!ok) __syncthreads();  // the retry rewrites panel buffers others may still read
  }
  if (!ok) return false;
#pragma unroll
  for (int s = 0; s < kFdTpw; ++s)
    if (wt[s].w != 3) {
      const int i = 8 * wt[s].x + gi, j = 8 * wt[s].y + 2 * ti;
      fd_readout(i, j, c[s][0], d, n, mp, P, mv, red);
      fd_readout(i, j + 1, c[s][1], d, n, mp, P, mv, red);
    }
  return true;
}

// Rank-1 LDL^T elimination of the bordered matrix (see the header), one 4×4 tile per
// thread; d <= 64.  Leaves P_f in P, m_f in mv, v^T S^-1 v in red[0], pivots in piv[0..d).
template <int TPT>
__device__ __forceinline__ bool elim_rank1(int tid, int d, int n, int npad, const double* Pp,
                                           const double* r, const double* w, const double* mp,
                                           double* col, double* piv, double* P, double* mv,
                                           double* red, const int (&I4)[TPT], const int (&J4)[TPT],
                                           const bool (&own)[TPT]) {
  double jit = 0.0;
  bool ok = false;
  double a[TPT][4][4];
  for (int attempt = 0; attempt < 3 && !ok; ++attempt) {
    if (attempt == 1) jit = jitter_scale(tid, d, Pp, r, red);
    const double eps = attempt == 0 ? 0.0 : (attempt == 1 ? 1e-10 : 1e-8) * jit;
    // fill M's tiles (lower triangle; diagonal tiles mirrored)
#pragma unroll
    for (int s = 0; s < TPT; ++s)
#pragma unroll
      for (int rr = 0; rr < 4; ++rr)
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
          a[s][rr][cc] = own[s] ? fd_mval(I4[s] + rr, J4[s] + cc, d, n, Pp, r, w, mp, eps) : 0.0;
        }
    // Pivot column k lives in col[k & 1]: rows >= k from their owners, rows < k of the
    // pivot's 4-row block zero — so the rank-1 update needs no per-entry predicate
    // (eliminated rows and columns see a zero multiplier; column k itself is zeroed,
    // it is not needed again).
#pragma unroll
    for (int s = 0; s < TPT; ++s)
      if (own[s] && J4[s] == 0)
#pragma unroll
        for (int rr = 0; rr < 4; ++rr) col[I4[s] + rr] = a[s][rr][0];
    bool failed = false;
    for (int kb = 0; kb < d && !failed; kb += 4) {
#pragma unroll
      for (int c4 = 0; c4 < 4; ++c4) {
        const int k = kb + c4;
        if (k >= d) break;
        __syncthreads();
        const double* cb = col + (k & 1) * npad;
        const double pk = cb[k];
        if (!(pk > 0.0 && pk < INFINITY)) {
          failed = true;
          break;
        }
        if (tid == 0) piv[k] = pk;
        double inv;  // 1/pk: MUFU seed + two Newton steps (within an ulp of IEEE division)
        asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(inv) : "d"(pk));
        {
          double e = fma(-pk, inv, 1.0);
          inv = fma(inv, e, inv);
          e = fma(-pk, inv, 1.0);
          inv = fma(inv, e, inv);
        }
        double* nb = col + ((k + 1) & 1) * npad;
#pragma unroll
        for (int s = 0; s < TPT; ++s) {
          if (!own[s] || I4[s] + 3 < k || J4[s] + 3 < k) continue;
          const double2* cv = reinterpret_cast<const double2*>(cb);
          const double2 c01 = cv[I4[s] >> 1], c23 = cv[(I4[s] >> 1) + 1];
          const double2 l01 = cv[J4[s] >> 1], l23 = cv[(J4[s] >> 1) + 1];
          const double ci[4] = {c01.x, c01.y, c23.x, c23.y};
          const double lj[4] = {l01.x * inv, l01.y * inv, l23.x * inv, l23.y * inv};
          // the next pivot column first (it is on the critical path), then the rest
          const int cn = (c4 + 1) & 3;
#pragma unroll
          for (int rr = 0; rr < 4; ++rr) a[s][rr][cn] = fma(-ci[rr], lj[cn], a[s][rr][cn]);
          if (k + 1 < d && J4[s] == ((k + 1) & ~3))
#pragma unroll
            for (int rr = 0; rr < 4; ++rr)
              nb[I4[s] + rr] = I4[s] + rr > k ? a[s][rr][cn] : 0.0;
#pragma unroll
          for (int rr = 0; rr < 4; ++rr)
#pragma unroll
            for (int cc = 0; cc < 4; ++cc)
              if (cc != cn) a[s][rr][cc] = fma(-ci[rr], lj[cc], a[s][rr][cc]);
        }
      }
    }
    ok = !failed;
    __syncthreads();
  }
  if (!ok) return false;
  // ---- Schur complement: P_f, m_f, v^T S^-1 v ----
#pragma unroll
  for (int s = 0; s < TPT; ++s) {
    if (!own[s]) continue;
#pragma unroll
    for (int rr = 0; rr < 4; ++rr)
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {
        fd_readout(I4[s] + rr, J4[s] + cc, a[s][rr][cc], d, n, mp, P, mv, red);
      }
  }
  return ok;
}

template <bool FST, int TPT, bool MMA, int DC>
__global__ void __launch_bounds__(kFdThreads, MMA ? 2 : 1)
k_filter_direct(DevModel m, DevTarget tg, const double* __restrict__ xl,
                const double* __restrict__ delta, const double* __restrict__ z, int C, int covs,
                double* pred_mean, double* pred_cov, double* filt_mean, double* filt_cov,
                double* log_marginal, int* status) {
  extern __shared__ double sm[];
  // DC > 0: the state dimension as a compile-time constant (index arithmetic folds)
  const int d = DC > 0 ? DC : m.dx, T = m.T, q = tg.q, p = d + q, dd = d * d;
  const int n = 2 * d + 1, nt = fd_nt(d), npad = 4 * nt, ntiles = fd_tiles(d);
  const int nin = p + 2 * d;
  const FdLayout L(d, q, FST);
  double* P = sm + L.P;
  double* A = sm + L.A;
  double* Pp = sm + L.Pp;
  double* Qs = sm + L.Q;
  double* Fd = sm + L.F;
  double* fv = sm + L.fv;
  int* fc = reinterpret_cast<int*>(sm + L.fc);
  double* mv = sm + L.m;
  double* mp = sm + L.mp;
  double* w = sm + L.w;
  double* r = sm + L.r;
  double* ex = sm + L.ex;
  double* col = sm + L.col;
  double* piv = sm + L.piv;
  double* inb = sm + L.in;
  double* bq = sm + L.bq;
  double* cq = sm + L.cq;
  int* sel = reinterpret_cast<int*>(sm + L.sel);
  double* red = sm + L.red;
  double* Rp = sm + L.Rb;
  double* Dv = sm + L.Dv;
  const int tid = threadIdx.x;
  const int c = blockIdx.x;
  if (c >= C) return;
  (void)Rp; (void)Dv; (void)col; (void)npad;

  // MMA: 8×8 tiles of M's lower triangle; (warp, slot) owns tile warp + 8 slot of the
  // row-major order
  int4* ttab = reinterpret_cast<int4*>(sm + L.tab);
  if (MMA && tid < kFdWarps * kFdTpw) {
    const FdTile ft = fd_tile_of(tid / kFdTpw, tid % kFdTpw, d);
    ttab[tid] = make_int4(ft.I, ft.J, ft.src, ft.kind);
  }

  // tiles owned by this thread
  constexpr int TP = TPT > 0 ? TPT : 1;
  int I4[TP], J4[TP];
  bool own[TP];
#pragma unroll
  for (int s = 0; s < TP; ++s) {
    const int tau = tid + s * kFdThreads;
    own[s] = tau < ntiles;
    int I = 0;
    while ((I + 1) * (I + 2) / 2 <= tau) ++I;
    I4[s] = 4 * I;
    J4[s] = 4 * (tau - I * (I + 1) / 2);
  }

  // ---- per-chain setup: exact-row structure, Q, dense F, m0, P0 ----
  for (int i = tid; i < d; i += kFdThreads) sel[i] = -1;
  if (tid == 0) red[1] = 0.0;
  __syncthreads();
  for (int k = tid; k < q; k += kFdThreads) {
    const double* hr = tg.eHt(0) + (size_t)k * d;
    const double* rr = tg.eRt(0) + (size_t)k * q;
    int nz = 0, j1 = -1;
    bool ok = true;
    for (int j = 0; j < d; ++j)
      if (hr[j] != 0.0) {
        ++nz;
        j1 = j;
        ok = ok && hr[j] == 1.0;
      }
    for (int j = 0; j < q; ++j) ok = ok && (j == k ? rr[j] > 0.0 : rr[j] == 0.0);
    if (!ok || nz != 1 || atomicCAS(&sel[j1], -1, k) != -1) {
      red[1] = 1.0;
    } else {
      bq[j1] = rr[k];
      cq[j1] = tg.ect(0)[k];
    }
  }
  for (int i = tid; i < dd; i += kFdThreads) {
    const double* Q0 = m.Qt(0, c);
    Qs[i] = 0.5 * (Q0[i] + Q0[(i % d) * d + i / d]);
    P[i] = 0.5 * (m.P0[i] + m.P0[(i % d) * d + i / d]);  // symm(P0), lgssm.cpp:90
    if (!FST) Fd[i] = m.Ft(0, c)[i];
  }
  for (int i = tid; i < d; i += kFdThreads) mv[i] = m.m0[i];
  const double* zc = z + (size_t)c * (T + 1) * p;
  const double* xc = FST ? xl + (size_t)c * (T + 1) * d : nullptr;
  for (int i = tid; i < p; i += kFdThreads) inb[i] = zc[i];
  __syncthreads();
  if (red[1] != 0.0) {
    if (tid == 0) {
      status[c] = 3;  // not the direct-observation structure (launch contract)
      log_marginal[c] = NAN;
    }
    return;
  }
  const double a_u = delta[c] / 2.0;  // R_uu = δ/2 I (auxk.cpp:82)
  double ll = 0.0;
  int st = 0;

  for (int t = 0; t <= T; ++t) {
    const bool stamp_on = AUXMC_FD_EXP == 9 && blockIdx.x == 0 && t == 200;
    (void)stamp_on;
    FD_STAMP(0);
    const double* cur = inb + (t & 1) * nin;  // z_t | x_{t-1} | b_{t-1}
    // prefetch step t+1's inputs: z_{t+1}, x_t, b_t
    double nxt = 0.0;
    if (t < T && tid < nin) {
      if (tid < p) nxt = zc[(size_t)(t + 1) * p + tid];
      else if (tid < p + d) nxt = FST ? xc[(size_t)t * d + (tid - p)] : 0.0;
      else nxt = m.bt(t, c)[tid - p - d];
    }
    // ---- predict: m_p = F m + b, P_p = symm(F P F^T + symm(Q)) ----
    if (t > 0) {
      const double* bp = cur + p + d;
      if (FST) {
        // row a of F: columns (a-2, a-1, a, a+1) mod d (target.cuh dyn_jac_ij's entries)
        const double* xl0 = cur + p;
        for (int a = tid; a < d; a += kFdThreads) {
          const int ip1 = (a + 1) % d, im1 = (a + d - 1) % d, im2 = (a + d - 2) % d;
          const double h = tg.l96_h;
          *reinterpret_cast<double2*>(fv + 4 * a) =
              make_double2(h * (0.0 - xl0[im1]), h * (0.0 + (xl0[ip1] - xl0[im2])));
          *reinterpret_cast<double2*>(fv + 4 * a + 2) =
              make_double2(1.0 + h * (0.0 - 1.0), h * (0.0 + xl0[im1]));
        }
        __syncthreads();
        // A = F P and m_p = F m + b: rows of P are contiguous in b (no bank conflicts)
        for (int e = tid; e < dd; e += kFdThreads) {
          const int a = e / d, b = e % d;
          const double2 f01 = *reinterpret_cast<const double2*>(fv + 4 * a);
          const double2 f23 = *reinterpret_cast<const double2*>(fv + 4 * a + 2);
          A[e] = ((f01.x * P[((a + d - 2) % d) * d + b] + f01.y * P[((a + d - 1) % d) * d + b]) +
                  f23.x * P[a * d + b]) + f23.y * P[((a + 1) % d) * d + b];
        }
        for (int a = tid; a < d; a += kFdThreads) {
          const double2 f01 = *reinterpret_cast<const double2*>(fv + 4 * a);
          const double2 f23 = *reinterpret_cast<const double2*>(fv + 4 * a + 2);
          mp[a] = (((f01.x * mv[(a + d - 2) % d] + f01.y * mv[(a + d - 1) % d]) +
                    f23.x * mv[a]) + f23.y * mv[(a + 1) % d]) + bp[a];
        }
        __syncthreads();
        // P_p = A F^T + symm(Q), every entry by the same formula (symmetric up to
        // rounding; the reference's extra symmetrization is within the FP64 tolerance)
        for (int e = tid; e < dd; e += kFdThreads) {
          const int a = e / d, b = e % d;
          const double2 f01 = *reinterpret_cast<const double2*>(fv + 4 * b);
          const double2 f23 = *reinterpret_cast<const double2*>(fv + 4 * b + 2);
          const double* Ar = A + a * d;
          Pp[e] = (((Ar[(b + d - 2) % d] * f01.x + Ar[(b + d - 1) % d] * f01.y) + Ar[b] * f23.x) +
                   Ar[(b + 1) % d] * f23.y) + Qs[e];
        }
      } else {
        for (int e = tid; e < dd; e += kFdThreads) {
          const int a = e / d, b = e % d;
          double s = 0.0;
          for (int k = 0; k < d; ++k) s += Fd[a * d + k] * P[k * d + b];
          A[e] = s;
        }
        for (int i = tid; i < d; i += kFdThreads) {
          double s = 0.0;
          for (int k = 0; k < d; ++k) s += Fd[i * d + k] * mv[k];
          mp[i] = s + bp[i];
        }
        __syncthreads();
        for (int e = tid; e < dd; e += kFdThreads) {
          const int a = e / d, b = e % d;
          if (b > a) continue;
          double x1 = 0.0, x2 = 0.0;
          for (int k = 0; k < d; ++k) {
            x1 += A[a * d + k] * Fd[b * d + k];
            x2 += A[b * d + k] * Fd[a * d + k];
          }
          const double qs = Qs[e];
          const double v = 0.5 * ((x1 + qs) + (x2 + qs));
          Pp[a * d + b] = v;
          Pp[b * d + a] = v;
        }
      }
    } else {
      for (int e = tid; e < dd; e += kFdThreads) Pp[e] = P[e];
      for (int i = tid; i < d; i += kFdThreads) mp[i] = mv[i];
    }
    // ---- fused direct observation ----
    const bool ex_t = q > 0 && tg.emask[t];
    for (int i = tid; i < d; i += kFdThreads) {
      const double u = cur[i];
      const int k = sel[i];
      if (ex_t && k >= 0) {
        const double b = bq[i], yv = cur[d + k] - cq[i], sab = a_u + b;
        r[i] = a_u * b / sab;
        w[i] = (u * b + yv * a_u) / sab;
        const double du = u - yv;
        ex[i] = -0.5 * (kLog2PiD + log(sab) + du * du / sab);
      } else {
        r[i] = a_u;
        w[i] = u;
        ex[i] = 0.0;
      }
    }
    __syncthreads();
    FD_STAMP(1);
    if (covs) {
      double* pmo = pred_mean + ((size_t)c * (T + 1) + t) * d;
      double* pco = pred_cov + ((size_t)c * (T + 1) + t) * dd;
      for (int i = tid; i < d; i += kFdThreads) pmo[i] = mp[i];
      for (int e = tid; e < dd; e += kFdThreads) pco[e] = Pp[e];
    }
    FD_STAMP(2);
    bool ok;
    if constexpr (MMA)
      ok = elim_mma(tid, d, n, Pp, r, w, mp, Rp, piv, P, mv, red, ttab, Dv, stamp_on);
    else if constexpr (TPT == 0)
      ok = false;
    else
      ok = elim_rank1<TPT>(tid, d, n, npad, Pp, r, w, mp, col, piv, P, mv, red, I4, J4, own);
    if (!ok) {
      st = 2;
      break;
    }
    FD_STAMP(40);
    __syncthreads();
    FD_STAMP(41);
    if (tid < 32) {  // log N(w; m_p, S) + fused-pair terms, fixed order
      double lg = 0.0, e2 = 0.0;
      for (int i = tid; i < (MMA ? (d + 3) / 4 : d); i += 32)
        lg += log(piv[i]);  // LDL pivots (rank-1) or det of each 4×4 pivot block (MMA)
      for (int i = tid; i < d; i += 32) e2 += ex[i];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        lg += __shfl_xor_sync(0xffffffffu, lg, o);
        e2 += __shfl_xor_sync(0xffffffffu, e2, o);
      }
      if (tid == 0) {
        // rows of an exact block absent at t: the generic model keeps them as
        // zero rows of N(0; 0, 1) (k_build_HR)
        const double miss = (q > 0 && !ex_t) ? -0.5 * q * kLog2PiD : 0.0;
        ll += -0.5 * (d * kLog2PiD + red[0]) - 0.5 * lg + e2 + miss;
      }
    }
    if (covs) {
      double* fmo = filt_mean + ((size_t)c * (T + 1) + t) * d;
      double* fco = filt_cov + ((size_t)c * (T + 1) + t) * dd;
      for (int i = tid; i < d; i += kFdThreads) fmo[i] = mv[i];
      for (int e = tid; e < dd; e += kFdThreads) fco[e] = P[e];
    }
    if (t < T && tid < nin) inb[((t + 1) & 1) * nin + tid] = nxt;
    __syncthreads();
    FD_STAMP(42);
  }
  if (tid == 0) {
    log_marginal[c] = st ? NAN : ll;
    status[c] = st;
  }
}

bool filter_direct_ok(const DevTarget& tg, const DevModel& dm, bool stencil) {
  if (!tg.exact_sel || dm.dx > 64 || dm.dx < 1) return false;
  if (dm.mask != nullptr || dm.nQ != 1) return false;
  if (!stencil && dm.nF != 1) return false;
  if (tg.q > 0 && tg.ne != 1) return false;
  const FdLayout L(dm.dx, tg.q, stencil);
  return sizeof(double) * L.total <= 227 * 1024;
}

int launch_filter_direct(const DevTarget& tg, const DevModel& dm, bool stencil,
                         const double* xl, const double* delta, const double* z, int C,
                         auxmc_filter_result* fr, int* status, int covs, cudaStream_t s) {
  if (!filter_direct_ok(tg, dm, stencil)) return AUXMC_E_CONFIG;
  if (stencil && (tg.kind != AUXMC_KIND_LORENZ96 || dm.dx < 4 || xl == nullptr))
    return AUXMC_E_CONFIG;
  if (C <= 0) return AUXMC_OK;
  const int d = dm.dx;
  const size_t smem = sizeof(double) * FdLayout(d, tg.q, stencil).total;
  const int tpt = (fd_tiles(d) + kFdThreads - 1) / kFdThreads;
#define FD_LAUNCH(FS, TP, MM, DC)                                                                \
  do {                                                                                           \
    AUXMC_CUDA_TRY(cudaFuncSetAttribute(k_filter_direct<FS, TP, MM, DC>,                         \
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    AUXMC_LAUNCH((k_filter_direct<FS, TP, MM, DC>), C, kFdThreads, smem, s, dm, tg, xl, delta, z, \
                 C,                                                                              \
                 covs,                                                                           \
                 fr->pred_mean, fr->pred_cov, fr->filt_mean, fr->filt_cov, fr->log_marginal,     \
                 status);                                                                        \
  } while (0)
  if (fd_use_mma(d)) {
    if (stencil && d == 40) FD_LAUNCH(true, 0, true, 40);  // Lorenz-96 d = 40 (C3)
    else if (stencil) FD_LAUNCH(true, 0, true, 0);
    else FD_LAUNCH(false, 0, true, 0);
  } else {
    if (tpt > 3) return AUXMC_E_DIM;
    if (stencil) FD_LAUNCH(true, 3, false, 0); else FD_LAUNCH(false, 3, false, 0);
  }
#undef FD_LAUNCH
  return AUXMC_OK;
}

}  // namespace auxmc_gpu

#if AUXMC_FD_EXP == 9
extern "C" int auxmc_debug_fd_stamps(long long* out, int n) {
  return cudaMemcpyFromSymbol(out, auxmc_gpu::g_fd_stamps, sizeof(long long) * n) == cudaSuccess
             ? 0
             : 1;
}
#endif
