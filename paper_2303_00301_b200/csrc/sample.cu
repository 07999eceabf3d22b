// sample.cu — pathwise posterior samplers on B200.
//
//  * k_bwd_elements: one-step backward conditionals (lgssm.cpp:129-149) as
//    affine elements (G_t, offset_t, L_t = chol_psd(Λ_t)) plus the terminal law
//    (m_T, chol_psd(P_T)) (lgssm.cpp:151-154, pit.cpp:85-87).  Group-cooperative.
//  * k_prefix: pit::prefix_sample (pit.cpp:78-115).  The suffix composition of
//    realized elements is evaluated as a fixed-tree reduce-then-scan: one CTA
//    owns a few chains over the whole horizon and walks it top-down in
//    superchunks staged through shared memory (cp.async double buffering);
//    inside a superchunk each thread reduces a sub-chunk, the sub-chunk
//    aggregates are scanned with the superchunk's carry, and each thread
//    expands its sub-chunk.  The association tree depends only on (T, LS, S), so
//    the output is bit-deterministic; noise is consumed by address (kBackwardNoise, t),
//    never by evaluation order (rng.hpp:128-137).
//  * k_seq: lgssm::backward_sample (lgssm.cpp:151-177), thread per path.
#include "common.cuh"
#include "dense.cuh"
#include "rng.cuh"
#include "tma.cuh"

namespace auxmc_gpu {


__device__ int g_flip_backward_gain = 0;  // testhooks::flip_backward_gain (testhooks.hpp:11)
// k_bwd_lean's steady-state reuse (auxmc_test_pfg_fixed_point switches it with the
// scan filter's fixed point); host-side
int g_bwd_reuse = 1;

// ---------------------------------------------------------------- elements
// smem per group: bwd_buffers(f_smem) d*d matrices + 4 d doubles + 2 ints.  Five
// d*d buffers rotate through the step (liveness below); the sixth holds F when
// f_smem, else F is read from global memory (L1-resident: the same d*d block is
// read by every product).  The operation sequence is the same either way, so the
// elements are bit-identical to the eight-buffer layout; fewer buffers put three
// d = 40 items on an SM instead of two.
__host__ __device__ constexpr int bwd_buffers(bool f_smem) { return f_smem ? 6 : 5; }
__device__ __forceinline__ int backward_step_group(const Grp& g, const DevModel& m, int t,
                                                   const double* fm, const double* fc,
                                                   const double* pc, double* sm, int* flag,
                                                   double* out /* G | off | L (or Λ) */, int k,
                                                   int store_cov, bool f_smem) {
  const int d = m.dx, dd = d * d;
  double* B0 = sm;         // P; then G Q G^T; then factor scratch
  double* B1 = B0 + dd;    // S (predicted covariance); then G
  double* B2 = B1 + dd;    // cross; factor scratch (jitter matrix / inverted blocks); then Λ
  double* B3 = B2 + dd;    // L (factor of S); then A = I - G F; then Q
  double* B4 = B3 + dd;    // solve rhs/result; then products; then chol(Λ)
  double* v = B4 + (f_smem ? 2 : 1) * dd;
  double* red = v + 2 * d;
  const double* F = m.fst ? nullptr : m.Ft(t, k);
  if (f_smem) {  // staged (stencil models: formed here, never read from HBM)
    fill_F(m, t, k, B4 + dd, g.lane, g.size);
    F = B4 + dd;
  }
  double* P = B0;
  double* S = B1;
  double* X = B2;
  double* L = B3;
  double* W = B4;
  g_copy(g, dd, fc + (size_t)t * dd, P);
  g_copy(g, dd, pc + (size_t)(t + 1) * dd, S);
  g.sync();
  g_mm_nt(g, d, d, d, P, F, X);  // cross = P F^T
  g.sync();
  double* G = B1;  // S is dead once the gain is solved
  int st = 0;
  if (g_all_zero(g, dd, X, flag)) {
    g_zero(g, dd, G);
    g.sync();
  } else {
    // rhs = cross^T (into W), W := S^{-1} cross^T, G = W^T
    for (int i = g.lane; i < dd; i += g.size) W[i] = X[(i % d) * d + i / d];
    g.sync();
    st = g_factor_psd(g, d, S, L, X, flag, red);  // X (cross) is consumed
    if (st) return st;
    g_llt_solve(g, d, L, d, W, X);
    for (int i = g.lane; i < dd; i += g.size) G[i] = W[(i % d) * d + i / d];
    g.sync();
  }
  if (g_flip_backward_gain) {
    for (int i = g.lane; i < dd; i += g.size) G[i] = -G[i];
    g.sync();
  }
  // offset = m_t - G (F m_t + b_t)
  const double* mt = fm + (size_t)t * d;
  const double* bt = m.bt(t, k);
  for (int i = g.lane; i < d; i += g.size) {
    double s = 0.0;
    for (int j = 0; j < d; ++j) s += F[i * d + j] * mt[j];
    v[i] = s + bt[i];
  }
  g.sync();
  for (int i = g.lane; i < d; i += g.size) {
    double s = 0.0;
    for (int j = 0; j < d; ++j) s += G[i * d + j] * v[j];
    v[d + i] = mt[i] - s;
  }
  // A = I - G F
  double* A = B3;
  g_mm(g, d, d, d, G, F, A);
  g.sync();
  for (int i = g.lane; i < dd; i += g.size) A[i] = (i / d == i % d ? 1.0 : 0.0) - A[i];
  g.sync();
  // Λ = symm(A P A^T + G Q G^T)
  g_mm(g, d, d, d, A, P, W);
  g.sync();
  g_mm_nt(g, d, d, d, W, A, X);  // X = A P A^T
  g.sync();
  double* Q = B3;
  g_copy(g, dd, m.Qt(t, k), Q);
  g.sync();
  g_mm(g, d, d, d, G, Q, W);
  g.sync();
  g_mm_nt(g, d, d, d, W, G, P);  // P = G Q G^T
  g.sync();
  for (int i = g.lane; i < dd; i += g.size) X[i] += P[i];
  g.sync();
  g_symm(g, d, X);
  g.sync();
  double* Lam = B4;
  if (!store_cov) {
    st = g_chol_psd(g, d, X, Lam, P, flag, red);  // P (G Q G^T) is consumed
    if (st) return st;
  }
  for (int i = g.lane; i < dd; i += g.size) {
    out[i] = G[i];
    out[dd + d + i] = store_cov ? X[i] : Lam[i];
  }
  for (int i = g.lane; i < d; i += g.size) out[dd + i] = v[d + i];
  g.sync();
  return 0;
}

// items: (b, t) for t in [0, T]; t == T is the terminal law.
template <bool BLOCK>
__global__ void k_bwd_elements(DevModel m, const double* __restrict__ filt_mean,
                               const double* __restrict__ filt_cov,
                               const double* __restrict__ pred_cov, int Bfr, double* elems,
                               double* term, int* status, int store_cov, int t_lo, int t_hi) {
  extern __shared__ double smem[];
  const int d = m.dx, dd = d * d;
  const int T = m.T;
  const bool f_smem = !BLOCK || m.fst;
  const int per = bwd_buffers(f_smem) * dd + 4 * d + 4;
  Grp g = BLOCK ? block_group() : warp_group();
  const int gid = BLOCK ? 0 : (threadIdx.x >> 5);
  const int groups_per_block = BLOCK ? 1 : (blockDim.x >> 5);
  double* sm = smem + (size_t)gid * per;
  int* flag = reinterpret_cast<int*>(sm + per - 2);
  const int span = t_hi - t_lo;  // items (b, t) for t in [t_lo, t_hi)
  const long long n_items = (long long)Bfr * span;
  for (long long item = (long long)blockIdx.x * groups_per_block + gid; item < n_items;
       item += (long long)gridDim.x * groups_per_block) {
    const int b = (int)(item / span);
    const int t = t_lo + (int)(item % span);
    const double* fm = filt_mean + (size_t)b * (T + 1) * d;
    const double* fc = filt_cov + (size_t)b * (T + 1) * dd;
    const double* pc = pred_cov + (size_t)b * (T + 1) * dd;
    int st;
    if (t == T) {
      double* out = term + (size_t)b * term_stride(d);
      double* P = sm;
      double* L = P + dd;
      double* scr = L + dd;
      double* red = scr + dd;
      g_copy(g, dd, fc + (size_t)T * dd, P);
      g.sync();
      st = g_chol_psd(g, d, P, L, scr, flag, red);
      for (int i = g.lane; i < d; i += g.size) out[i] = fm[(size_t)T * d + i];
      for (int i = g.lane; i < dd; i += g.size) out[d + i] = L[i];
    } else {
      st = backward_step_group(g, m, t, fm, fc, pc, sm, flag,
                               elems + ((size_t)b * T + t) * elem_stride(d), b, store_cov, f_smem);
    }
    if (st && g.lane == 0) atomicMax(status + b, st);
    g.sync();
  }
}

// Lean backward elements for CTA-sized d (d > 16): the same conditional law
// (lgssm.cpp:129-149) in the Schur form
//   C = F P,  S = L L^T,  W = L^{-1} C,  Λ = P - W^T W,  G^T = L^{-T} W,
//   off = m - G (F m + b),  L_Λ = chol_psd(Λ)
// (Λ = P - P F^T S^{-1} F P, algebraically the reference's Joseph form; FP64
// association differs, within the parity tolerance).  Three d×d buffers: the factor
// of S is built in place from HBM and rebuilt from HBM for the jitter ladder, the
// cross block is solved in place twice, Λ overwrites P.  Products, factors and solves
// are the blocked DMMA routines of group.cuh; a stencil F (m.fst) forms C with four
// FMAs per entry.  About 1/4 of the FLOPs and 3/5 of the shared memory of
// backward_step_group, so five items run per SM.
constexpr int kBwdLeanThreads = 128;
#ifndef AUXMC_BWD_EXP
#define AUXMC_BWD_EXP 0  // 9: clock64 phase stamps of the first item of CTA 0 (tools/bwd_stamps.py)
#endif
#if AUXMC_BWD_EXP == 9
__device__ long long g_bwd_stamps[64];
#define BWD_STAMP(k)                                                       \
  do {                                                                     \
    if (stamp && threadIdx.x == 0) g_bwd_stamps[(k)] = clock64();          \
  } while (0)
#else
#define BWD_STAMP(k) \
  do {               \
  } while (0)
#endif
#ifndef BWD_LEAN_MIN_D
#define BWD_LEAN_MIN_D 16  // smallest d on the CTA Schur-form kernel (below: warp groups)
#endif
#ifndef BWD_LEAN_MINB
#define BWD_LEAN_MINB 4  // CTAs per SM the register budget is cut for (smem allows 5 at d = 40)
#endif
__host__ __device__ inline int bwd_lean_doubles(int d) {
  return 3 * d * d + dinv_doubles(d) + 8 * d + 4;
}

__global__ void __launch_bounds__(kBwdLeanThreads, BWD_LEAN_MINB)
k_bwd_lean(DevModel m, const double* __restrict__ filt_mean, const double* __restrict__ filt_cov,
           const double* __restrict__ pred_cov, int Bfr, double* elems, double* term,
           int* status, int store_cov, int t_lo, int t_hi, int reuse, double* recs, int* rep) {
  extern __shared__ double smem[];
  const int d = m.dx, dd = d * d, T = m.T;
  const bool flip = g_flip_backward_gain != 0;
  const Grp g = block_group();
  double* Lb = smem;                    // chol(S), then chol(Λ)
  double* W = Lb + dd;                  // C = F P -> L^{-1} C -> G^T
  double* P = W + dd;                   // P -> Λ
  double* dinv = P + dd;                // inverted 8×8 diagonal blocks
  double* v = dinv + dinv_doubles(d);   // F m + b
  double* fvb = v + 2 * d;              // stencil values [d][4]
  int* fcb = reinterpret_cast<int*>(fvb + 4 * d);  // stencil columns [d][4]
  double* red = fvb + 6 * d;
  int* flag = reinterpret_cast<int*>(red + 2);
  __shared__ __align__(8) uint64_t bar[1];
  unsigned phase = 0;
  // bulk copies need 16-B aligned sources and sizes
  const bool tma = (dd % 2 == 0) && ((reinterpret_cast<uintptr_t>(filt_cov) & 15) == 0) &&
                   ((reinterpret_cast<uintptr_t>(pred_cov) & 15) == 0);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_fence_init();
  }
  __syncthreads();
  const int span = t_hi - t_lo;
  const long long n_items = (long long)Bfr * span;
  // reuse (dense F shared by every step, no stencil): each CTA takes chunks of
  // kBwdChunk consecutive items, and an item whose P_t and P_{t+1|t} have the bits of
  // the previous item's keeps that item's G, Λ and factor (the time-invariant
  // filter's steady state: only the offset moves).  recs (d <= 16): when every
  // later item of a chunk repeats its first item's inputs, the chunk is recorded
  // and left to k_bwd_lanes.  Otherwise the items are strided over the grid.
  const int nchk = reuse ? (span + kBwdChunk - 1) / kBwdChunk : 0;
  const long long n_units = reuse ? (long long)Bfr * nchk : n_items;
  bool have = false;  // smem holds W, P (Λ), Lb of item (b, t - 1)
  int st_keep = 0, b_prev = -1, t_prev = -1;
  for (long long unit = blockIdx.x; unit < n_units; unit += gridDim.x) {
  long long i0 = unit, i1 = unit + 1;
  if (reuse) {
    const long long bu = unit / nchk, cu = unit % nchk;
    i0 = bu * span + cu * kBwdChunk;
    i1 = bu * span + min((long long)span, (cu + 1) * kBwdChunk);
  }
  for (long long item = i0; item < i1; ++item) {
    const int b = (int)(item / span);
    const int t = t_lo + (int)(item % span);
    if (recs && item == i0 + 1) {
      const int t_last = t_lo + (int)((i1 - 1) % span);
      bool all = have && b == b_prev && t == t_prev + 1 && t_last < T;
      if (all) {
        const double* f0 = filt_cov + ((size_t)b * (T + 1) + t - 1) * dd;
        const double* p0 = pred_cov + ((size_t)b * (T + 1) + t) * dd;
        const int nrest = t_last - t + 1;
        const bool mine = rows_match_part(f0 + dd, f0, nrest, dd, g.lane, g.size) &&
                          rows_match_part(p0 + dd, p0, nrest, dd, g.lane, g.size);
        all = __syncthreads_and(mine) != 0;
      }
      if (g.lane == 0) {
        recs[2 * unit] = all ? 1.0 : 0.0;
        recs[2 * unit + 1] = (double)st_keep;
      }
      if (all) break;
    }
    const double* fm = filt_mean + (size_t)b * (T + 1) * d;
    const double* fc = filt_cov + (size_t)b * (T + 1) * dd;
    const double* pc = pred_cov + (size_t)b * (T + 1) * dd;
    int st = 0;
    bool hit = false;
    if (have && b == b_prev && t == t_prev + 1 && t < T) {
      if (g.lane == 0) *flag = 1;
      g.sync();
      const long long* x0 = reinterpret_cast<const long long*>(fc + (size_t)t * dd);
      const long long* x1 = reinterpret_cast<const long long*>(pc + (size_t)(t + 1) * dd);
      for (int i = g.lane; i < dd; i += g.size)
        if (x0[i] != x0[i - dd] || x1[i] != x1[i - dd]) *flag = 0;
      g.sync();
      hit = *flag != 0;
      g.sync();
    }
    have = false;
    b_prev = b;
    t_prev = t;
    if (t == T) {  // terminal law (pit.cpp:85-87)
      double* out = term + (size_t)b * term_stride(d);
      g_copy(g, dd, fc + (size_t)T * dd, P);
      g.sync();
      st = g_chol_psd(g, d, P, Lb, dinv, flag, red);
      for (int i = g.lane; i < d; i += g.size) out[i] = fm[(size_t)T * d + i];
      for (int i = g.lane; i < dd; i += g.size) out[d + i] = Lb[i];
      if (st && g.lane == 0) atomicMax(status + b, st);
      g.sync();
      continue;
    }
    double* out = elems + ((size_t)b * T + t) * elem_stride(d);
    if (rep && g.lane == 0) rep[(size_t)b * T + t] = t;  // this element holds its own matrices
    const double* S = pc + (size_t)(t + 1) * dd;
    const bool stamp = AUXMC_BWD_EXP == 9 && blockIdx.x == 0 && item == 0;
    (void)stamp;
    BWD_STAMP(0);
    if (!hit) {
    // P_t and S = P_{t+1|t} by two TMA bulk copies (one HBM round trip, not a load/store
    // loop per element); S's upper triangle is zeroed once it lands
    if (tma) {
      if (g.lane == 0) {
        mbar_expect_tx(bar, 2u * (unsigned)dd * 8u);
        bulk_g2s(P, fc + (size_t)t * dd, (unsigned)dd * 8u, bar);
        bulk_g2s(Lb, S, (unsigned)dd * 8u, bar);
      }
    } else {
      g_copy(g, dd, fc + (size_t)t * dd, P);
      g_copy(g, dd, S, Lb);
    }
    if (m.fst)
      for (int i = g.lane; i < d; i += g.size) stencil_row(m, t, b, i, fcb + 4 * i, fvb + 4 * i);
    if (tma) {
      mbar_wait(bar, phase);
      phase ^= 1u;
    } else {
      g.sync();
    }
    for (int i = g.ty(); i < d; i += g.ny())
      for (int j = g.tx(); j < d; j += 16)
        if (j > i) Lb[i * d + j] = 0.0;
    g.sync();
    // C = F P
    if (m.fst) {
      for (int e = g.lane; e < dd; e += g.size) {
        const int a = e / d, c = e % d;
        double x = 0.0;
#pragma unroll
        for (int k = 0; k < 4; ++k) x += fvb[4 * a + k] * P[fcb[4 * a + k] * d + c];
        W[e] = x;
      }
    } else {
      g_dmma<false, false>(g, d, d, d, m.Ft(t, b), d, P, d, W, d, false, false);
    }
    g.sync();
    BWD_STAMP(1);
    if (!g_all_zero(g, dd, W, flag)) {
      BWD_STAMP(2);
      bool ok = g_llt_blocked(g, d, Lb, flag, dinv);
      BWD_STAMP(3);
      if (!ok) {  // factor_psd ladder (gauss.cpp:26-35) on S, rebuilt from HBM
        if (g.lane == 0) {
          double tr = 0.0;
          for (int i = 0; i < d; ++i) tr += S[i * d + i];
          double sc = tr / static_cast<double>(d);
          if (sc <= 0.0) {
            double mx = 0.0;
            for (int i = 0; i < dd; ++i) mx = fabs(S[i]) > mx ? fabs(S[i]) : mx;
            sc = mx;
          }
          *red = sc;
        }
        g.sync();
        const double sc = *red;
        for (int e = 0; e < 2 && !ok; ++e) {
          const double eps = e == 0 ? 1e-10 : 1e-8;
          for (int i = g.ty(); i < d; i += g.ny())
            for (int j = g.tx(); j < d; j += 16)
              Lb[i * d + j] = j <= i ? S[i * d + j] + (i == j ? (eps * sc) * 1.0 : 0.0) : 0.0;
          g.sync();
          ok = g_llt_blocked(g, d, Lb, flag, dinv);
        }
      }
      if (!ok) {
        if (g.lane == 0) atomicMax(status + b, 2);
        g.sync();
        continue;  // have stays false
      }
      g_trsm_lower_blocked(g, d, Lb, dinv, d, W, d);                    // W = L^{-1} C
      BWD_STAMP(4);
      g_dmma<true, false>(g, d, d, d, W, d, W, d, P, d, true, true);   // Λ (lower) = P - W^T W
      g.sync();
      BWD_STAMP(5);
      g_trsm_lower_t_blocked(g, d, Lb, dinv, d, W, d);                  // W = S^{-1} C = G^T
      BWD_STAMP(6);
      for (int i = g.ty(); i < d; i += g.ny())
        for (int j = g.tx(); j < d; j += 16)
          if (j > i) P[i * d + j] = P[j * d + i];
      g.sync();
    }
    }  // !hit
    BWD_STAMP(7);
    // offset = m_t - G (F m_t + b_t)
    const double* mt = fm + (size_t)t * d;
    const double* bt = m.bt(t, b);
    for (int i = g.lane; i < d; i += g.size) {
      double x = 0.0;
      if (m.fst) {
#pragma unroll
        for (int k = 0; k < 4; ++k) x += fvb[4 * i + k] * mt[fcb[4 * i + k]];
      } else {
        const double* F = m.Ft(t, b);
        for (int k = 0; k < d; ++k) x += F[i * d + k] * mt[k];
      }
      v[i] = x + bt[i];
    }
    g.sync();
    // flip (testhooks::flip_backward_gain): the gain enters negated; W itself is kept
    for (int i = g.lane; i < d; i += g.size) {
      double x = 0.0;
      for (int k = 0; k < d; ++k) x += (flip ? -W[k * d + i] : W[k * d + i]) * v[k];
      out[dd + i] = mt[i] - x;
    }
    for (int e = g.lane; e < dd; e += g.size) {
      const double w = W[(e % d) * d + e / d];
      out[e] = flip ? -w : w;
    }
    if (store_cov) {
      for (int e = g.lane; e < dd; e += g.size) out[dd + d + e] = P[e];
    } else {
      BWD_STAMP(8);
      if (!hit) st_keep = g_chol_psd(g, d, P, Lb, dinv, flag, red);
      st = st_keep;
      BWD_STAMP(9);
      for (int e = g.lane; e < dd; e += g.size) out[dd + d + e] = Lb[e];
    }
    if (st && g.lane == 0) atomicMax(status + b, st);
    g.sync();
    have = reuse != 0;
    BWD_STAMP(10);
  }
  }
}

// The items (c0, c1) of every chunk k_bwd_lean recorded uniform (each repeats item
// c0's P_t and P_{t+1|t}): their G and factor are item c0's, copied row by row, and
// lane j forms item c0 + 1 + j's offset m_t - G (F m_t + b_t) by k_bwd_lean's
// operations in its order (G read from item c0's element: the bits k_bwd_lean
// wrote, gain flip included).  Dense shared F, d <= 16.
constexpr int kBwdLaneWarps = 8;
__global__ void __launch_bounds__(kBwdLaneWarps * 32)
    k_bwd_lanes(DevModel m, const double* __restrict__ filt_mean, int Bfr, double* elems,
                int* status, int t_lo, int t_hi, const double* __restrict__ recs, int* rep) {
  constexpr int MX = 16;
  const int d = m.dx, dd = d * d, T = m.T, es = elem_stride(d);
  const int lane = threadIdx.x & 31;
  const int span = t_hi - t_lo;
  const int nchk = (span + kBwdChunk - 1) / kBwdChunk;
  const long long n_units = (long long)Bfr * nchk;
  for (long long unit = (long long)blockIdx.x * kBwdLaneWarps + (threadIdx.x >> 5); unit < n_units;
       unit += (long long)gridDim.x * kBwdLaneWarps) {
    if (recs[2 * unit] == 0.0) continue;
    const int b = (int)(unit / nchk), cu = (int)(unit % nchk);
    const int c0 = t_lo + cu * kBwdChunk, c1 = t_lo + min(span, (cu + 1) * kBwdChunk);
    const int st = (int)recs[2 * unit + 1];
    if (st && lane == 0) atomicMax(status + b, st);
    const double* src = elems + ((size_t)b * T + c0) * es;
    if (rep) {  // the sampler reads these steps' matrices from item c0's element
      for (int u = c0 + 1 + lane; u < c1; u += 32) rep[(size_t)b * T + u] = c0;
    } else {
      for (int u = c0 + 1; u < c1; ++u) {
        double* o = elems + ((size_t)b * T + u) * es;
        for (int e = lane; e < dd; e += 32) {
          o[e] = src[e];
          o[dd + d + e] = src[dd + d + e];
        }
      }
    }
    const double* F = m.Ft(0, b);
    for (int t = c0 + 1 + lane; t < c1; t += 32) {
      const double* mt = filt_mean + ((size_t)b * (T + 1) + t) * d;
      const double* bt = m.bt(t, b);
      double mv[MX], v[MX];
#pragma unroll
      for (int k = 0; k < MX; ++k) mv[k] = k < d ? mt[k] : 0.0;
#pragma unroll
      for (int i = 0; i < MX; ++i) {
        if (i < d) {
          double x = 0.0;
#pragma unroll
          for (int k = 0; k < MX; ++k)
            if (k < d) x += F[i * d + k] * mv[k];
          v[i] = x + bt[i];
        }
      }
      double* o = elems + ((size_t)b * T + t) * es;
#pragma unroll
      for (int i = 0; i < MX; ++i) {
        if (i < d) {
          double x = 0.0;
#pragma unroll
          for (int k = 0; k < MX; ++k)
            if (k < d) x += src[i * d + k] * v[k];
          o[dd + i] = mv[i] - x;
        }
      }
    }
  }
}

// Register path of k_bwd_elements for small d: one thread per (b, t).
template <int D>
__global__ void k_bwd_elements_reg(DevModel m, const double* __restrict__ filt_mean,
                                   const double* __restrict__ filt_cov,
                                   const double* __restrict__ pred_cov, int Bfr, double* elems,
                                   double* term, int* status, int store_cov, int t_lo, int t_hi) {
  constexpr int DD = D * D;
  const int T = m.T;
  const int span = t_hi - t_lo;
  const long long n_items = (long long)Bfr * span;
  for (long long item = (long long)blockIdx.x * blockDim.x + threadIdx.x; item < n_items;
       item += (long long)gridDim.x * blockDim.x) {
    const int b = (int)(item / span), t = t_lo + (int)(item % span);
    const double* fm = filt_mean + (size_t)b * (T + 1) * D;
    const double* fc = filt_cov + (size_t)b * (T + 1) * DD;
    double P[DD], L[DD];
#pragma unroll
    for (int i = 0; i < DD; ++i) P[i] = fc[(size_t)t * DD + i];
    int st = 0;
    if (t == T) {  // terminal law (pit.cpp:85-87)
      st = r_chol_psd<D>(P, L);
      double* out = term + (size_t)b * term_stride(D);
#pragma unroll
      for (int i = 0; i < D; ++i) out[i] = fm[(size_t)T * D + i];
#pragma unroll
      for (int i = 0; i < DD; ++i) out[D + i] = L[i];
    } else {  // backward_step (lgssm.cpp:129-149)
      const double* Fp = m.Ft(t, b);
      double F[DD], G[DD], X[DD], A[DD], W[DD];
#pragma unroll
      for (int i = 0; i < DD; ++i) F[i] = Fp[i];
      bool zero = true;
#pragma unroll
      for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) {  // X = cross^T = (P F^T)^T, X[j][i] = cross[i][j]
          double s = 0.0;
#pragma unroll
          for (int k = 0; k < D; ++k) s += P[i * D + k] * F[j * D + k];
          X[j * D + i] = s;
          zero = zero && (s == 0.0);
        }
      if (zero) {
#pragma unroll
        for (int i = 0; i < DD; ++i) G[i] = 0.0;
      } else {
        double S[DD];
        const double* Sp = pred_cov + ((size_t)b * (T + 1) + t + 1) * DD;
#pragma unroll
        for (int i = 0; i < DD; ++i) S[i] = Sp[i];
        st = r_factor_psd<D>(S, L);
        r_llt_solve<D, D>(L, X);
#pragma unroll
        for (int i = 0; i < D; ++i)
#pragma unroll
          for (int j = 0; j < D; ++j) G[i * D + j] = X[j * D + i];
      }
      if (g_flip_backward_gain) {
#pragma unroll
        for (int i = 0; i < DD; ++i) G[i] = -G[i];
      }
      const double* mt = fm + (size_t)t * D;
      const double* bt = m.bt(t, b);
      double v[D], off[D];
#pragma unroll
      for (int i = 0; i < D; ++i) {
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < D; ++j) s += F[i * D + j] * mt[j];
        v[i] = s + bt[i];
      }
#pragma unroll
      for (int i = 0; i < D; ++i) {
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < D; ++j) s += G[i * D + j] * v[j];
        off[i] = mt[i] - s;
      }
#pragma unroll
      for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) {  // A = I - G F
          double s = 0.0;
#pragma unroll
          for (int k = 0; k < D; ++k) s += G[i * D + k] * F[k * D + j];
          A[i * D + j] = (i == j ? 1.0 : 0.0) - s;
        }
      // Λ = symm(A P A^T + G Q G^T)
#pragma unroll
      for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) {
          double s = 0.0;
#pragma unroll
          for (int k = 0; k < D; ++k) s += A[i * D + k] * P[k * D + j];
          W[i * D + j] = s;
        }
      double Lam[DD];
#pragma unroll
      for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) {
          double s = 0.0;
#pragma unroll
          for (int k = 0; k < D; ++k) s += W[i * D + k] * A[j * D + k];
          Lam[i * D + j] = s;
        }
      const double* Qp = m.Qt(t, b);
#pragma unroll
      for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) {
          double s = 0.0;
#pragma unroll
          for (int k = 0; k < D; ++k) s += G[i * D + k] * Qp[k * D + j];
          W[i * D + j] = s;
        }
#pragma unroll
      for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) {
          double s = 0.0;
#pragma unroll
          for (int k = 0; k < D; ++k) s += W[i * D + k] * G[j * D + k];
          Lam[i * D + j] += s;
        }
#pragma unroll
      for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = i + 1; j < D; ++j) {
          const double s = 0.5 * (Lam[i * D + j] + Lam[j * D + i]);
          Lam[i * D + j] = s;
          Lam[j * D + i] = s;
        }
      if (!store_cov && !st) st = r_chol_psd<D>(Lam, L);
      double* out = elems + ((size_t)b * T + t) * elem_stride(D);
#pragma unroll
      for (int i = 0; i < DD; ++i) {
        out[i] = G[i];
        out[DD + D + i] = store_cov ? Lam[i] : L[i];
      }
#pragma unroll
      for (int i = 0; i < D; ++i) out[DD + i] = off[i];
    }
    if (st) atomicMax(status + b, st);
  }
}

// ---------------------------------------------------------------- noise

template <int D>
__device__ __forceinline__ void stream_normals(uint64_t key, double* xi) {
#pragma unroll
  for (int i = 0; i < D; ++i) xi[i] = normal_at(key, (uint64_t)i);
}

// The stream variates of B paths, drawn in parallel ahead of a latency-bound
// sampler (same keys and indices as the samplers' own draws, so the paths are
// bit-identical): thread per (path, t), t = T the terminal draw.
template <int D>
__global__ void k_draw_stream(int T, int B, const uint64_t* __restrict__ keys, double* term,
                              double* back) {
  const long long n = (long long)B * (T + 1);
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(q / (T + 1)), t = (int)(q % (T + 1));
    double xi[D];
    if (t == T) {
      stream_normals<D>(derive(keys[c], kTerminalDraw, 0), xi);
#pragma unroll
      for (int i = 0; i < D; ++i) term[(size_t)c * D + i] = xi[i];
    } else {
      stream_normals<D>(derive_index(derive_label(keys[c], kBackwardNoise), (uint64_t)t), xi);
#pragma unroll
      for (int i = 0; i < D; ++i) back[((size_t)c * T + t) * D + i] = xi[i];
    }
  }
}

// ---------------------------------------------------------------- sequential / per-path elements
// Thread per path; elements either shared (es = 0) or per path.
template <int D, bool PRE>
__global__ void k_seq_sample(int T, int C, const double* __restrict__ elems, long long estride,
                             const double* __restrict__ term, long long tstride, NoiseArgs noise,
                             double* __restrict__ traj) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  constexpr int ES = (2 * D * D + D + 1) & ~1;
  const double* E = elems + (size_t)c * estride;
  const double* tm = term + (size_t)c * tstride;
  const long long row = (long long)(T + 1) * D;
  double x[D], xi[D];
  if (PRE) {
#pragma unroll
    for (int i = 0; i < D; ++i) xi[i] = noise.terminal[(size_t)c * D + i];
  } else {
    stream_normals<D>(derive(noise.keys[c], kTerminalDraw, 0), xi);
  }
  r_matvec<D>(tm + D, xi, x);
#pragma unroll
  for (int i = 0; i < D; ++i) {
    x[i] = tm[i] + x[i];
    traj[(size_t)c * row + (size_t)T * D + i] = x[i];
  }
  const uint64_t kl = PRE ? 0 : derive_label(noise.keys[c], kBackwardNoise);
  for (int t = T - 1; t >= 0; --t) {
    const double* e = E + (size_t)t * ES;
    if (PRE) {
#pragma unroll
      for (int i = 0; i < D; ++i) xi[i] = noise.backward[((size_t)c * T + t) * D + i];
    } else {
      stream_normals<D>(derive_index(kl, (uint64_t)t), xi);
    }
    double cv[D], gx[D];
    r_matvec<D>(e + D * D + D, xi, cv);
    r_matvec<D>(e, x, gx);
#pragma unroll
    for (int i = 0; i < D; ++i) {
      x[i] = gx[i] + (e[D * D + i] + cv[i]);
      traj[(size_t)c * row + (size_t)t * D + i] = x[i];
    }
  }
}

// Any state dimension (d <= 64): warp per path, lanes over rows.
__global__ void k_seq_sample_warp(int T, int d, int C, const double* __restrict__ elems,
                                  long long estride, const double* __restrict__ term,
                                  long long tstride, NoiseArgs noise, double* __restrict__ traj) {
  __shared__ double sx[4][2][64];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x * 4 + w;
  if (c >= C) return;
  const int ES = elem_stride(d), dd = d * d;
  const double* E = elems + (size_t)c * estride;
  const double* tm = term + (size_t)c * tstride;
  const long long row = (long long)(T + 1) * d;
  double* out = traj + (size_t)c * row;
  double* xi = sx[w][0];
  double* x = sx[w][1];
  const bool pre = noise.kind == AUXMC_NOISE_PREDRAWN;
  for (int i = lane; i < d; i += 32)
    xi[i] = pre ? noise.terminal[(size_t)c * d + i]
                : normal_at(derive(noise.keys[c], kTerminalDraw, 0), (uint64_t)i);
  __syncwarp();
  for (int i = lane; i < d; i += 32) {
    double s = 0.0;
    for (int j = 0; j < d; ++j) s += tm[d + i * d + j] * xi[j];
    x[i] = tm[i] + s;
    out[(size_t)T * d + i] = x[i];
  }
  const uint64_t kl = pre ? 0 : derive_label(noise.keys[c], kBackwardNoise);
  double xn[2];
  for (int t = T - 1; t >= 0; --t) {
    const double* e = E + (size_t)t * ES;
    __syncwarp();
    const uint64_t key = pre ? 0 : derive_index(kl, (uint64_t)t);
    for (int i = lane; i < d; i += 32)
      xi[i] = pre ? noise.backward[((size_t)c * T + t) * d + i] : normal_at(key, (uint64_t)i);
    __syncwarp();
    int r = 0;
    for (int i = lane; i < d; i += 32, ++r) {
      double cv = 0.0, gx = 0.0;
      for (int j = 0; j < d; ++j) cv += e[dd + d + i * d + j] * xi[j];
      for (int j = 0; j < d; ++j) gx += e[i * d + j] * x[j];
      xn[r] = gx + (e[dd + i] + cv);
    }
    __syncwarp();
    r = 0;
    for (int i = lane; i < d; i += 32, ++r) {
      x[i] = xn[r];
      out[(size_t)t * d + i] = xn[r];
    }
  }
}

// Any state dimension (8 < d <= 64), one CTA per path: the backward recursion
// x_t = G_t x_{t+1} + off_t + L_t ξ_t (lgssm.cpp:151-177) streams its elements — one
// contiguous 8·elem_stride(d) block per step, 26 KB at d = 40 — through an NS-stage
// shared-memory ring filled by 1-D TMA bulk copies issued NS steps ahead, so the HBM
// stream never waits on the recursion.  Row i is one warp's dot products (lanes over
// columns, fixed xor-tree sums); ξ_t and L_t ξ_t do not depend on the path and are
// formed before x_{t+1} is needed, so only G_t x_{t+1} is on the serial chain.
constexpr int kSeqCtaThreads = 256;
__host__ __device__ inline int seq_cta_stages(int d) {
  const long long es = (long long)elem_stride(d) * 8;
  return 3 * es <= 112 * 1024 ? 3 : 2;
}
__host__ __device__ inline size_t seq_cta_smem(int d) {
  return (size_t)seq_cta_stages(d) * elem_stride(d) * 8 + sizeof(double) * 4 * 64 + 64;
}

__device__ __forceinline__ double warp_sum_xor(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void __launch_bounds__(kSeqCtaThreads)
k_seq_sample_cta(int T, int d, int C, const double* __restrict__ elems, long long estride,
                 const double* __restrict__ term, long long tstride, NoiseArgs noise,
                 double* __restrict__ traj) {
  extern __shared__ __align__(128) double smem[];
  const int c = blockIdx.x;
  if (c >= C) return;
  const int NS = seq_cta_stages(d), ES = elem_stride(d), dd = d * d;
  double* stage = smem;
  double* xb = stage + (size_t)NS * ES;  // [2][64] path rows
  double* xi = xb + 128;                 // ξ_t
  double* lx = xi + 64;                  // off_t + L_t ξ_t
  uint64_t* bar = reinterpret_cast<uint64_t*>(lx + 64);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double* E = elems + (size_t)c * estride;
  const double* tm = term + (size_t)c * tstride;
  double* out = traj + (size_t)c * (T + 1) * d;
  const bool pre = noise.kind == AUXMC_NOISE_PREDRAWN;
  const unsigned bytes = (unsigned)ES * 8u;
  if (tid == 0) {
    for (int s = 0; s < NS; ++s) mbar_init(bar + s, 1);
    mbar_fence_init();
    for (int s = 0; s < NS && T - 1 - s >= 0; ++s) {
      mbar_expect_tx(bar + s, bytes);
      bulk_g2s(stage + (size_t)s * ES, E + (size_t)(T - 1 - s) * ES, bytes, bar + s);
    }
  }
  // terminal draw x_T = m_T + chol(P_T) ξ (pit.cpp:85-87)
  for (int i = tid; i < d; i += kSeqCtaThreads)
    xi[i] = pre ? noise.terminal[(size_t)c * d + i]
                : normal_at(derive(noise.keys[c], kTerminalDraw, 0), (uint64_t)i);
  __syncthreads();
  for (int i = tid; i < d; i += kSeqCtaThreads) {
    double s = 0.0;
    for (int j = 0; j < d; ++j) s += tm[d + i * d + j] * xi[j];
    const double v = tm[i] + s;
    xb[i] = v;
    out[(size_t)T * d + i] = v;
  }
  const uint64_t kl = pre ? 0 : derive_label(noise.keys[c], kBackwardNoise);
  auto draw = [&](int t) {  // ξ_t into xi
    const uint64_t key = pre ? 0 : derive_index(kl, (uint64_t)t);
    for (int i = tid; i < d; i += kSeqCtaThreads)
      xi[i] = pre ? noise.backward[((size_t)c * T + t) * d + i] : normal_at(key, (uint64_t)i);
  };
  if (T > 0) draw(T - 1);
  __syncthreads();
  for (int k = 0; k < T; ++k) {
    const int t = T - 1 - k, s = k % NS;
    const double* e = stage + (size_t)s * ES;
    mbar_wait(bar + s, (unsigned)((k / NS) & 1));
    // off_t + L_t ξ_t (independent of the path)
    for (int i = warp; i < d; i += kSeqCtaThreads / 32) {
      const double* Lr = e + dd + d + (size_t)i * d;
      double v = lane < d ? Lr[lane] * xi[lane] : 0.0;
      if (lane + 32 < d) v += Lr[lane + 32] * xi[lane + 32];
      v = warp_sum_xor(v);
      if (lane == 0) lx[i] = e[dd + i] + v;
    }
    __syncthreads();
    // x_t = G_t x_{t+1} + (off_t + L_t ξ_t)
    const double* xp = xb + (k & 1) * 64;
    double* xn = xb + ((k + 1) & 1) * 64;
    for (int i = warp; i < d; i += kSeqCtaThreads / 32) {
      const double* Gr = e + (size_t)i * d;
      double v = lane < d ? Gr[lane] * xp[lane] : 0.0;
      if (lane + 32 < d) v += Gr[lane + 32] * xp[lane + 32];
      v = warp_sum_xor(v);
      if (lane == 0) {
        const double x = v + lx[i];
        xn[i] = x;
        out[(size_t)t * d + i] = x;
      }
    }
    if (t > 0) draw(t - 1);
    __syncthreads();
    if (tid == 0 && t - NS >= 0) {  // refill this stage NS steps ahead
      mbar_expect_tx(bar + s, bytes);
      bulk_g2s(stage + (size_t)s * ES, E + (size_t)(t - NS) * ES, bytes, bar + s);
    }
  }
}

// Per-path-element prefix sampler (aux-kernel backend): thread per (path,
// sub-chunk) with in-thread sub-chunk products; sub-chunk carries scanned by
// one thread per path.  Same fixed tree as k_prefix_shared.
template <int D, int NS, int LS, bool PRE>
__global__ void __launch_bounds__(NS)
    k_prefix_private(int T, const double* __restrict__ elems, const double* __restrict__ term,
                     NoiseArgs noise, double* __restrict__ traj) {
  constexpr int S = NS * LS;
  constexpr int ES = (2 * D * D + D + 1) & ~1;
  __shared__ double csub[NS * D], gsub[NS * D * D], xtop[NS * D], carry[D];
  const int c = blockIdx.x, j = threadIdx.x;
  const double* E = elems + (size_t)c * T * ES;
  const double* tm = term + (size_t)c * ((D * D + D + 1) & ~1);
  const long long row = (long long)(T + 1) * D;
  double* out = traj + (size_t)c * row;
  if (j == 0) {
    double xi[D], x[D];
    if (PRE) {
#pragma unroll
      for (int i = 0; i < D; ++i) xi[i] = noise.terminal[(size_t)c * D + i];
    } else {
      stream_normals<D>(derive(noise.keys[c], kTerminalDraw, 0), xi);
    }
    r_matvec<D>(tm + D, xi, x);
#pragma unroll
    for (int i = 0; i < D; ++i) {
      x[i] = tm[i] + x[i];
      carry[i] = x[i];
      out[(size_t)T * D + i] = x[i];
    }
  }
  if (T == 0) return;
  const uint64_t kl = PRE ? 0 : derive_label(noise.keys[c], kBackwardNoise);
  const int K = (T + S - 1) / S;
  for (int k = K - 1; k >= 0; --k) {
    __syncthreads();
    const int t0 = k * S, t1 = min(t0 + S, T);
    const int lo = t0 + j * LS, hi = min(lo + LS, t1);
    double y[D], P[D * D];
#pragma unroll
    for (int i = 0; i < D; ++i) y[i] = 0.0;
#pragma unroll
    for (int i = 0; i < D * D; ++i) P[i] = (i / D == i % D) ? 1.0 : 0.0;
#pragma unroll(D <= 4 ? LS : 1)
    for (int u = LS - 1; u >= 0; --u) {  // t = hi-1 .. lo, unrolled so the loads issue early
      const int t = lo + u;
      if (t >= hi) continue;
      const double* e = E + (size_t)t * ES;
      double xi[D], cv[D], gy[D], Q[D * D];
      if (PRE) {
#pragma unroll
        for (int i = 0; i < D; ++i) xi[i] = noise.backward[((size_t)c * T + t) * D + i];
      } else {
        stream_normals<D>(derive_index(kl, (uint64_t)t), xi);
      }
      r_matvec<D>(e + D * D + D, xi, cv);
      r_matvec<D>(e, y, gy);
#pragma unroll
      for (int i = 0; i < D; ++i) {
        cv[i] = e[D * D + i] + cv[i];
        out[(size_t)t * D + i] = cv[i];  // park c_t in the output row
        y[i] = gy[i] + cv[i];
      }
#pragma unroll
      for (int a = 0; a < D; ++a)
#pragma unroll
        for (int b = 0; b < D; ++b) {
          double acc = 0.0;
#pragma unroll
          for (int q = 0; q < D; ++q) acc += e[a * D + q] * P[q * D + b];
          Q[a * D + b] = acc;
        }
#pragma unroll
      for (int i = 0; i < D * D; ++i) P[i] = Q[i];
    }
#pragma unroll
    for (int i = 0; i < D; ++i) csub[j * D + i] = y[i];
#pragma unroll
    for (int i = 0; i < D * D; ++i) gsub[j * D * D + i] = P[i];
    __syncthreads();
    if (j == 0) {
      double x[D];
#pragma unroll
      for (int i = 0; i < D; ++i) x[i] = carry[i];
      for (int jj = NS - 1; jj >= 0; --jj) {
#pragma unroll
        for (int i = 0; i < D; ++i) xtop[jj * D + i] = x[i];
        if (t0 + jj * LS >= t1) continue;
        double gx[D];
        r_matvec<D>(gsub + jj * D * D, x, gx);
#pragma unroll
        for (int i = 0; i < D; ++i) x[i] = gx[i] + csub[jj * D + i];
      }
#pragma unroll
      for (int i = 0; i < D; ++i) carry[i] = x[i];
    }
    __syncthreads();
    double x[D];
#pragma unroll
    for (int i = 0; i < D; ++i) x[i] = xtop[j * D + i];
#pragma unroll(D <= 4 ? LS : 1)
    for (int u = LS - 1; u >= 0; --u) {
      const int t = lo + u;
      if (t >= hi) continue;
      const double* e = E + (size_t)t * ES;
      double gx[D];
      r_matvec<D>(e, x, gx);
#pragma unroll
      for (int i = 0; i < D; ++i) {
        x[i] = gx[i] + out[(size_t)t * D + i];
        out[(size_t)t * D + i] = x[i];
      }
    }
  }
}

}  // namespace auxmc_gpu

namespace auxmc_gpu {

__global__ void k_fanout_status(const int* st_fr, int fr_shared, int B, int* status) {
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < B; b += gridDim.x * blockDim.x)
    status[b] = st_fr[fr_shared ? 0 : b];
}

int launch_prefix_shared(int d, int T, int B, const double* elems, const double* term, Arena& ws,
                         const NoiseArgs& nz, double* traj, cudaStream_t stream);
int launch_dnc(const DevModel& dm, int Bfr, int fr_shared, const double* elems,
               const double* term, const NoiseArgs& nz, int B, double* traj, Arena& ws,
               int* st_fr, cudaStream_t stream);
int launch_prefix_generic(int T, int d, int B, int fr_shared, const double* elems,
                          const double* term, const NoiseArgs& nz, double* traj, Arena& ws,
                          cudaStream_t stream, const int* rep);

namespace {

constexpr int kNSp = 32, kLSp = 8;             // per-path prefix tiling
constexpr int kNSs = 64, kLSs = 16;            // few paths (B <= 2 per SM): one 1024-step superchunk

template <int D>
int run_sampler(int sampler, int T, int B, int fr_shared, const double* elems,
                const double* term, Arena& ws, const NoiseArgs& nz, double* traj,
                cudaStream_t stream) {
  const bool pre = nz.kind == AUXMC_NOISE_PREDRAWN;
  if (sampler == AUXMC_SAMPLER_PREFIX && fr_shared)
    return launch_prefix_shared(D, T, B, elems, term, ws, nz, traj, stream);
  const bool few = B <= 2 * 148 && D <= 4;
  double *nterm = nullptr, *nback = nullptr;
  if (sampler == AUXMC_SAMPLER_PREFIX && few && !pre) {
    nterm = ws.take<double>((size_t)B * D);
    nback = ws.take<double>((size_t)B * (T > 0 ? T : 1) * D);
  }
  if (ws.base == nullptr) return AUXMC_OK;
  const long long es = fr_shared ? 0 : (long long)T * elem_stride(D);
  const long long ts = fr_shared ? 0 : term_stride(D);
  if (sampler == AUXMC_SAMPLER_PREFIX) {
    if (few) {
      NoiseArgs pz = nz;
      if (nterm && nback) {  // few long serial chains: draw the variates in parallel first
        const long long n = (long long)B * (T + 1);
        AUXMC_LAUNCH(k_draw_stream<D>, (int)std::min<long long>((n + 127) / 128, 148LL * 16),
                     128, 0, stream, T, B, nz.keys, nterm, nback);
        pz.kind = AUXMC_NOISE_PREDRAWN;
        pz.terminal = nterm;
        pz.backward = nback;
      } else if (!pre) {
        return AUXMC_E_WORKSPACE;
      }
      AUXMC_LAUNCH((k_prefix_private<D, kNSs, kLSs, true>), B, kNSs, 0, stream, T, elems, term, pz,
                   traj);
    } else if (pre) {
      AUXMC_LAUNCH((k_prefix_private<D, kNSp, kLSp, true>), B, kNSp, 0, stream, T, elems, term, nz, traj);
    } else {
      AUXMC_LAUNCH((k_prefix_private<D, kNSp, kLSp, false>), B, kNSp, 0, stream, T, elems, term, nz, traj);
    }
    return AUXMC_OK;
  }
  const int grid = (B + 127) / 128;
  if (pre)
    AUXMC_LAUNCH((k_seq_sample<D, true>), grid, 128, 0, stream, T, B, elems, es, term, ts, nz, traj);
  else
    AUXMC_LAUNCH((k_seq_sample<D, false>), grid, 128, 0, stream, T, B, elems, es, term, ts, nz, traj);
  return AUXMC_OK;
}

}  // namespace

// items (b, t) for t in [t_lo, t_hi) (default: the whole horizon [0, T]; t = T is the
// terminal law)
int launch_bwd_elements(const DevModel& dm, const double* fm, const double* fc, const double* pc,
                        int Bfr, double* elems, double* term, int* st_fr, int store_cov,
                        cudaStream_t stream, int t_lo = 0, int t_hi = -1,
                        double* recs = nullptr, int* rep = nullptr) {
  const int d = dm.dx;
  const int per_blk = bwd_buffers(dm.fst != 0) * d * d + 4 * d + 4;  // CTA items: F from global
  const int per = bwd_buffers(true) * d * d + 4 * d + 4;       // warp items: F staged
  if (t_hi < 0) t_hi = dm.T + 1;
  if (t_hi <= t_lo) return AUXMC_OK;
  const long long n_items = (long long)Bfr * (t_hi - t_lo);
  if (d <= 4) {
    if (dm.fst) return AUXMC_E_CONFIG;  // the register path reads a dense F
    const int grid = (int)std::min<long long>((n_items + 127) / 128, 148LL * 16);
    switch (d) {
#define CASE(D)                                                                                  \
  case D:                                                                                        \
    AUXMC_LAUNCH(k_bwd_elements_reg<D>, grid, 128, 0, stream, dm, fm, fc, pc, Bfr, elems, term, \
                 st_fr, store_cov, t_lo, t_hi);                                                  \
    break;
      CASE(1) CASE(2) CASE(3) CASE(4)
#undef CASE
    }
  } else if (d >= BWD_LEAN_MIN_D) {
    const size_t smem = sizeof(double) * bwd_lean_doubles(d);
    AUXMC_CUDA_TRY(cudaFuncSetAttribute(k_bwd_lean, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)smem));
    const int grid = (int)std::min<long long>(n_items, 148LL * 64);
    const int reuse = g_bwd_reuse && !dm.fst && dm.nF <= 1;
    double* recs_on = (reuse && d <= 16) ? recs : nullptr;  // k_bwd_lanes: d <= 16
    int* rep_on = rep;  // every item k_bwd_lean takes points at itself
    AUXMC_LAUNCH(k_bwd_lean, grid, kBwdLeanThreads, smem, stream, dm, fm, fc, pc, Bfr, elems, term,
                 st_fr, store_cov, t_lo, t_hi, reuse, recs_on, rep_on);
    if (recs_on) {
      const long long nu = (long long)Bfr * ((t_hi - t_lo + kBwdChunk - 1) / kBwdChunk);
      AUXMC_LAUNCH(k_bwd_lanes,
                   (int)std::min<long long>((nu + kBwdLaneWarps - 1) / kBwdLaneWarps, 148LL * 32),
                   32 * kBwdLaneWarps, 0, stream, dm, fm, Bfr, elems, st_fr, t_lo, t_hi, recs_on,
                   rep_on);
    }
    (void)per_blk;
  } else {
    const int warps = 4;
    const size_t smem = sizeof(double) * per * warps;
    AUXMC_CUDA_TRY(cudaFuncSetAttribute(k_bwd_elements<false>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int grid = (int)std::min<long long>((n_items + warps - 1) / warps, 148LL * 64);
    AUXMC_LAUNCH(k_bwd_elements<false>, grid, 32 * warps, smem, stream, dm, fm, fc, pc, Bfr, elems,
                 term, st_fr, store_cov, t_lo, t_hi);
  }
  return AUXMC_OK;
}

int launch_sample_paths(const DevModel& dm, const auxmc_filter_result* fr, int fr_shared,
                        const auxmc_noise* noise, int B, int sampler, double* traj, int* status,
                        Arena& ws, cudaStream_t stream) {
  const int d = dm.dx, T = dm.T;
  const int Bfr = fr_shared ? 1 : B;
  if (sampler < 0 || sampler > 2) return AUXMC_E_ARG;
  double* elems = ws.take<double>((size_t)Bfr * (T > 0 ? T : 1) * elem_stride(d));
  double* term = ws.take<double>((size_t)Bfr * term_stride(d));
  int* st_fr = ws.take<int>((size_t)Bfr);
  double* recs = ws.take<double>(bwd_recs_doubles(Bfr, T + 1));
  // the generic prefix sampler reads each step's matrices through rep (filled by the
  // CTA Schur-form elements, d >= BWD_LEAN_MIN_D), so uniform chunks skip the copies
  const bool use_rep = sampler == AUXMC_SAMPLER_PREFIX && d > 8 && d >= BWD_LEAN_MIN_D && d <= 64;
  int* rep = use_rep ? ws.take<int>((size_t)Bfr * (T > 0 ? T : 1)) : nullptr;
  NoiseArgs nz{};
  if (noise) {
    nz.kind = noise->kind;
    nz.keys = noise->keys;
    nz.terminal = noise->terminal;
    nz.backward = noise->backward;
    nz.bridge = noise->bridge;
    nz.n_bridge = noise->n_bridge;
  }
  if (ws.base != nullptr) {
    if (!elems || !term || !st_fr || !recs || (use_rep && !rep)) return AUXMC_E_WORKSPACE;
    AUXMC_CUDA_TRY(cudaMemsetAsync(st_fr, 0, sizeof(int) * Bfr, stream));
    int rc = launch_bwd_elements(dm, fr->filt_mean, fr->filt_cov, fr->pred_cov, Bfr, elems, term,
                                 st_fr, sampler == AUXMC_SAMPLER_DNC ? 1 : 0, stream, 0, -1, recs,
                                 rep);
    if (rc) return rc;
  }
  int rc = AUXMC_OK;
  if (sampler == AUXMC_SAMPLER_DNC) {
    rc = launch_dnc(dm, Bfr, fr_shared, elems, term, nz, B, traj, ws, st_fr, stream);
  } else {
    switch (d) {
#define CASE(D) \
  case D: rc = run_sampler<D>(sampler, T, B, fr_shared, elems, term, ws, nz, traj, stream); break;
      CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8)
#undef CASE
      default:
        if (d > 64) {
          rc = AUXMC_E_DIM;
        } else if (sampler == AUXMC_SAMPLER_PREFIX) {
          rc = launch_prefix_generic(T, d, B, fr_shared, elems, term, nz, traj, ws, stream, rep);
        } else if (ws.base != nullptr) {
          const long long es = fr_shared ? 0 : (long long)T * elem_stride(d);
          const long long ts = fr_shared ? 0 : term_stride(d);
          if (d > 8) {
            const size_t smem = seq_cta_smem(d);
            AUXMC_CUDA_TRY(cudaFuncSetAttribute(k_seq_sample_cta,
                                                cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                (int)smem));
            AUXMC_LAUNCH(k_seq_sample_cta, B, kSeqCtaThreads, smem, stream, T, d, B, elems, es,
                         term, ts, nz, traj);
          } else {
            AUXMC_LAUNCH(k_seq_sample_warp, (B + 3) / 4, 128, 0, stream, T, d, B, elems, es, term,
                         ts, nz, traj);
          }
        }
    }
  }
  if (rc || ws.base == nullptr) return rc;
  AUXMC_LAUNCH(k_fanout_status, (B + 255) / 256, 256, 0, stream, st_fr, fr_shared, B, status);
  return AUXMC_OK;
}

}  // namespace auxmc_gpu

extern "C" int auxmc_test_flip_backward_gain(int on) {
  // testhooks::flip_backward_gain (testhooks.hpp:11): deliberately wrong gains so
  // the law checks must fail (runner.cpp:301-312)
  if (!auxmc_gpu::device_ok()) return AUXMC_E_CUDA;
  const int v = on ? 1 : 0;
  return cudaMemcpyToSymbol(auxmc_gpu::g_flip_backward_gain, &v, sizeof v) == cudaSuccess
             ? AUXMC_OK
             : AUXMC_E_CUDA;
}

#if AUXMC_BWD_EXP == 9
extern "C" int auxmc_debug_bwd_stamps(long long* out, int n) {
  return cudaMemcpyFromSymbol(out, auxmc_gpu::g_bwd_stamps, sizeof(long long) * n) == cudaSuccess
             ? 0
             : 1;
}
#endif
