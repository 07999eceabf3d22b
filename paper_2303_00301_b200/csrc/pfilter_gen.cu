// pfilter_gen.cu — pit::parallel_filter (pit.cpp:117-188) for state dims
// 7 <= dx <= 32 (or observation rows > 8): the same blocked scan as pfilter.cu
// (S1 block reductions, S2 serial carries, S3 inclusive application, then the
// recovery pass), with every element build / combine / recovery done by a
// cooperative group on shared memory — a warp when dx, dy <= 16, a 128-thread
// CTA otherwise (DMMA products and blocked factorizations from group.cuh).
// Results follow the register kernels' operation order where the group
// routines do (scalar products, row-sequential LU solves); DMMA products and
// blocked Cholesky associate differently, within the FP64 parity tolerance.
#include <algorithm>

#include "common.cuh"
#include "dense.cuh"

namespace auxmc_gpu {

namespace {

__host__ __device__ inline int fe_size_g(int d) { return 3 * d * d + 2 * d; }

// ---------------------------------------------------------------- partial-pivot LU
// Row-pivoted LU in place (Eigen PartialPivLU: the first row of largest |.|
// in the column is the pivot, zero pivots skip the elimination).  perm in
// shared memory; idx: 1 int of scratch.
__device__ void g_lu_factor(const Grp& g, int d, double* M, int* perm, int* idx) {
  for (int i = g.lane; i < d; i += g.size) perm[i] = i;
  g.sync();
  for (int k = 0; k < d; ++k) {
    if (g.lane < 32) {  // pivot search in warp 0: first max of |M[i][k]|, i >= k
      double best = -1.0;
      int bi = d;
      for (int i = k + g.lane; i < d; i += 32) {
        const double v = fabs(M[i * d + k]);
        if (v > best) {
          best = v;
          bi = i;
        }
      }
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) {
          best = ob;
          bi = oi;
        }
      }
      if (g.lane == 0) *idx = bi < d ? bi : k;  // all-NaN column: keep row k
    }
    g.sync();
    const int p = *idx;
    if (p != k) {
      for (int j = g.lane; j < d; j += g.size) {
        const double t = M[k * d + j];
        M[k * d + j] = M[p * d + j];
        M[p * d + j] = t;
      }
      if (g.lane == 0) {
        const int t = perm[k];
        perm[k] = perm[p];
        perm[p] = t;
      }
    }
    g.sync();
    const double piv = M[k * d + k];
    if (piv != 0.0) {
      for (int i = k + 1 + g.lane; i < d; i += g.size) M[i * d + k] = M[i * d + k] / piv;
      g.sync();
      for (int i = k + 1 + g.ty(); i < d; i += g.ny()) {
        const double f = M[i * d + k];
        for (int j = k + 1 + g.tx(); j < d; j += 16) M[i * d + j] -= f * M[k * d + j];
      }
    }
    g.sync();
  }
}

// X (d×r) = M^{-1} B (B row-major d×r, may not alias X); lanes over columns
__device__ void g_lu_solve(const Grp& g, int d, const double* LU, const int* perm, int r,
                           const double* B, double* X) {
  for (int c = g.lane; c < r; c += g.size) {
    for (int i = 0; i < d; ++i) {
      double s = B[perm[i] * r + c];
      for (int j = 0; j < i; ++j) s -= LU[i * d + j] * X[j * r + c];
      X[i * r + c] = s;
    }
    for (int i = d - 1; i >= 0; --i) {
      double s = X[i * r + c];
      for (int j = i + 1; j < d; ++j) s -= LU[i * d + j] * X[j * r + c];
      X[i * r + c] = s / LU[i * d + i];
    }
  }
}

// One warp, d <= 16: Minv = M^{-1} by Gauss-Jordan with partial pivoting on the
// augmented [M | I], lane j holding column j in registers (2d <= 32 lanes).  The
// pivot rule is PartialPivLU's (first row of largest |.| at or below the
// diagonal); rows are swapped and eliminated inside every lane's column, the
// pivot column is broadcast by shuffles — no shared-memory round trips.
// DN > 0: the dimension is the compile-time DN (every bound static); DN = 0: d <= 16
// at run time.  Same operations in the same order either way.
template <int DN>
__device__ __forceinline__ void w_inverse_gj_t(int lane, int d_rt, const double* M,
                                               double* Minv) {
  constexpr int MX = DN ? DN : 16;
  const int d = DN ? DN : d_rt;
  double col[MX];
  const int j = lane;
#pragma unroll
  for (int i = 0; i < MX; ++i)
    col[i] = (i < d && j < 2 * d) ? (j < d ? M[i * d + j] : (i == j - d ? 1.0 : 0.0)) : 0.0;
#pragma unroll
  for (int k = 0; k < MX; ++k) {  // fully unrolled: every index but the pivot row is static
    if (k >= d) break;
    // pivot search by the lane owning column k (rows k..d-1): pairwise tree over
    // the candidates, a later row wins only when strictly larger — the first
    // row of largest |.|, as a sequential scan finds it
    double av[MX];
    int ai[MX];
#pragma unroll
    for (int i = 0; i < MX; ++i) {
      av[i] = (i >= k && i < d) ? fabs(col[i]) : -1.0;
      ai[i] = i;
    }
#pragma unroll
    for (int w = 1; w < MX; w *= 2)
#pragma unroll
      for (int i = 0; i + w < MX; i += 2 * w)
        if (av[i + w] > av[i]) {
          av[i] = av[i + w];
          ai[i] = ai[i + w];
        }
    int p = __shfl_sync(0xffffffffu, ai[0] < k ? k : ai[0], k);  // NaN column: row k
    // swap rows k and p (p >= k) in every column
    const double vk = col[k];
    double vp = vk;
#pragma unroll
    for (int i = k + 1; i < MX; ++i) vp = i == p ? col[i] : vp;
#pragma unroll
    for (int i = k + 1; i < MX; ++i) col[i] = i == p ? vk : col[i];
    col[k] = vp;
    // eliminate with the pivot column (broadcast from lane k)
    const double piv = __shfl_sync(0xffffffffu, vp, k);
    const double xk = vp / piv;  // this column's entry of the normalized pivot row
#pragma unroll
    for (int i = 0; i < MX; ++i) {
      const double m = __shfl_sync(0xffffffffu, col[i], k);  // pivot column entry, row i
      if (i < d) col[i] = i == k ? xk : fma(-m, xk, col[i]);
    }
  }
  if (j >= d && j < 2 * d) {
#pragma unroll
    for (int i = 0; i < MX; ++i)
      if (i < d) Minv[i * d + (j - d)] = col[i];
  }
  __syncwarp();
}

// o = combine(u, v) (pit.cpp:36-51); scratch: 3 dd + 2 d doubles, 2 d + 1 ints.  The
// LU / inverse work matrices M1, Minv live in o's C and J blocks, which are only
// written at the very end (o never aliases u or v).
struct CombScratch {
  double *S, *T1, *T2, *t, *w;
  int *p1, *p2, *idx;
};

// With C and J symmetric (every element and every combine output is
// symmetrized), M2 = I + vJ uC is exactly M1^T for M1 = I + uC vJ (same
// products, same summation order), so one LU gives both solves: Minv = M1^{-1}
// (LU with partial pivoting, solved against I) and M2^{-1} = Minv^T; the
// remaining algebra is dense products.
template <int DC>
__device__ __forceinline__ void g_combine_t(const Grp& g, int d_rt, const double* u,
                                            const double* v, double* o, const CombScratch& s,
                                            double* save_minv) {
  const int d = DC ? DC : d_rt;
  const int dd = d * d;
  const double *uA = u, *ub = u + dd, *uC = u + dd + d, *ueta = u + 2 * dd + d,
               *uJ = u + 2 * dd + 2 * d;
  const double *vA = v, *vb = v + dd, *vC = v + dd + d, *veta = v + 2 * dd + d,
               *vJ = v + 2 * dd + 2 * d;
  double *oA = o, *ob = o + dd, *oC = o + dd + d, *oeta = o + 2 * dd + d, *oJ = o + 2 * dd + 2 * d;
  double* const M1 = oC;
  double* Minv = oJ;
  g_mm(g, d, d, d, uC, vJ, M1);
  g_eye(g, d, s.T2);
  g.sync();
  for (int i = g.lane; i < d; i += g.size) M1[i * d + i] += 1.0;
  g.sync();
  if (!g.block && d <= 16) {
    w_inverse_gj_t<DC>(g.lane, d, M1, Minv);  // M1^{-1}, registers and shuffles
  } else {
    g_lu_factor(g, d, M1, s.p1, s.idx);
    g_lu_solve(g, d, M1, s.p1, d, s.T2, Minv);  // M1^{-1}
  }
  // t = uC veta + ub ; t2 = veta - vJ ub
  for (int i = g.lane; i < d; i += g.size) {
    double acc = 0.0, acc2 = 0.0;
    for (int k = 0; k < d; ++k) {
      acc += uC[i * d + k] * veta[k];
      acc2 += vJ[i * d + k] * ub[k];
    }
    s.t[i] = acc + ub[i];
    s.w[i] = veta[i] - acc2;
  }
  g.sync();
  if (save_minv) g_copy(g, dd, Minv, save_minv);  // k_pfg_reduce_proto
  // A = vA (Minv uA) ; S = Minv uC ; T2 = Minv^T vJ
  g_mm(g, d, d, d, Minv, uA, s.S);
  g_mm(g, d, d, d, Minv, uC, s.T1);
  g_mm_tn(g, d, d, d, Minv, vJ, s.T2);
  // b = vA (Minv t) + vb ; eta = uA^T (Minv^T t2) + ueta  (vectors kept in M1's rows)
  double* mt = M1;
  double* mt2 = M1 + d;
  for (int i = g.lane; i < d; i += g.size) {
    double acc = 0.0, acc2 = 0.0;
    for (int k = 0; k < d; ++k) {
      acc += Minv[i * d + k] * s.t[k];
      acc2 += Minv[k * d + i] * s.w[k];
    }
    mt[i] = acc;
    mt2[i] = acc2;
  }
  g.sync();
  g_mm(g, d, d, d, vA, s.S, oA);
  for (int i = g.lane; i < d; i += g.size) {
    double acc = 0.0, acc2 = 0.0;
    for (int k = 0; k < d; ++k) {
      acc += vA[i * d + k] * mt[k];
      acc2 += uA[k * d + i] * mt2[k];
    }
    ob[i] = acc + vb[i];
    oeta[i] = acc2 + ueta[i];
  }
  // C = symm(vA (Minv uC) vA^T + vC) ; J = symm(uA^T (Minv^T vJ) uA + uJ)
  g_mm(g, d, d, d, vA, s.T1, Minv);  // Minv consumed
  g.sync();
  g_mm_tn(g, d, d, d, uA, s.T2, s.S);
  g_mm_nt(g, d, d, d, Minv, vA, s.T1, vC);
  g.sync();
  g_mm(g, d, d, d, s.S, uA, s.T2, uJ);
  g.sync();
  for (int i = g.ty(); i < d; i += g.ny())
    for (int j = g.tx(); j < d; j += 16) {
      oC[i * d + j] = 0.5 * (s.T1[i * d + j] + s.T1[j * d + i]);
      oJ[i * d + j] = 0.5 * (s.T2[i * d + j] + s.T2[j * d + i]);
    }
  g.sync();
}

// d = 16 (the C5 state dimension) gets a fully static instance: the Gauss-Jordan
// inverse dominated the generic combine's instruction count (runtime bounds).
__device__ __noinline__ void g_combine(const Grp& g, int d, const double* u, const double* v,
                                       double* o, const CombScratch& s,
                                       double* save_minv = nullptr) {
  if (d == 16) g_combine_t<16>(g, d, u, v, o, s, save_minv);
  else g_combine_t<0>(g, d, u, v, o, s, save_minv);
}

// (u then v) when u is a prefix from t = 0, whose A is exactly zero (the first
// element sets A := 0, pit.cpp:151, and A_out = v.A solve(u.A) keeps it zero):
// b and C depend on (u.b, u.C, v) alone and are formed by exactly the operations
// g_combine_t uses for them; with u.A = 0 the full combine's other outputs reduce
// to A = 0, eta = 0 + u.eta, J = symm(0 + u.J), written directly.  The output is
// bit-identical to g_combine_t's, at 4 instead of 9 d^3 products.
// vm: where v's matrices (A, C, J) are read — v itself, or an element with the same
// matrices (the shared element of a time-invariant model, whose per-step copies the
// element fill then need not write)
template <int DC>
__device__ __forceinline__ void g_combine_bc_t(const Grp& g, int d_rt, const double* u,
                                               const double* v, const double* vm, double* o,
                                               const CombScratch& s, bool keep_minv) {
  const int d = DC ? DC : d_rt;
  const int dd = d * d;
  const double *ub = u + dd, *uC = u + dd + d, *ueta = u + 2 * dd + d, *uJ = u + 2 * dd + 2 * d;
  const double *vA = vm, *vb = v + dd, *vC = vm + dd + d, *veta = v + 2 * dd + d,
               *vJ = vm + 2 * dd + 2 * d;
  double *oA = o, *ob = o + dd, *oC = o + dd + d, *oeta = o + 2 * dd + d, *oJ = o + 2 * dd + 2 * d;
  double* const M1 = oC;
  double* Minv = oJ;
  g_mm(g, d, d, d, uC, vJ, M1);
  g_eye(g, d, s.T2);
  g.sync();
  for (int i = g.lane; i < d; i += g.size) M1[i * d + i] += 1.0;
  g.sync();
  if (!g.block && d <= 16) {
    w_inverse_gj_t<DC>(g.lane, d, M1, Minv);
  } else {
    g_lu_factor(g, d, M1, s.p1, s.idx);
    g_lu_solve(g, d, M1, s.p1, d, s.T2, Minv);
  }
  for (int i = g.lane; i < d; i += g.size) {
    double acc = 0.0;
    for (int k = 0; k < d; ++k) acc += uC[i * d + k] * veta[k];
    s.t[i] = acc + ub[i];
  }
  g.sync();
  if (keep_minv)  // Minv^T into s.S, free in this form (g_bc_vec_t reads it by columns)
    for (int e = g.lane; e < dd; e += g.size) s.S[e] = Minv[(e % d) * d + e / d];
  g_mm(g, d, d, d, Minv, uC, s.T1);
  double* mt = M1;
  for (int i = g.lane; i < d; i += g.size) {
    double acc = 0.0;
    for (int k = 0; k < d; ++k) acc += Minv[i * d + k] * s.t[k];
    mt[i] = acc;
  }
  g.sync();
  for (int i = g.lane; i < d; i += g.size) {
    double acc = 0.0;
    for (int k = 0; k < d; ++k) acc += vA[i * d + k] * mt[k];
    ob[i] = acc + vb[i];
    oeta[i] = 0.0 + ueta[i];
  }
  g_mm(g, d, d, d, vA, s.T1, Minv);  // Minv consumed
  g.sync();
  g_mm_nt(g, d, d, d, Minv, vA, s.T1, vC);
  g.sync();
  for (int i = g.ty(); i < d; i += g.ny())
    for (int j = g.tx(); j < d; j += 16) {
      oC[i * d + j] = 0.5 * (s.T1[i * d + j] + s.T1[j * d + i]);
      oA[i * d + j] = 0.0;
    }
  g.sync();  // oJ held Minv until the last product
  for (int i = g.ty(); i < d; i += g.ny())
    for (int j = g.tx(); j < d; j += 16)
      oJ[i * d + j] = 0.5 * ((0.0 + uJ[i * d + j]) + (0.0 + uJ[j * d + i]));
  g.sync();
}

__device__ __noinline__ void g_combine_bc(const Grp& g, int d, const double* u, const double* v,
                                          double* o, const CombScratch& s,
                                          bool keep_minv = false, const double* vm = nullptr) {
  if (!vm) vm = v;
  if (d == 16) g_combine_bc_t<16>(g, d, u, v, vm, o, s, keep_minv);
  else g_combine_bc_t<0>(g, d, u, v, vm, o, s, keep_minv);
}

// ---------------------------------------------------------------- covariance fixed point
// A chain of prefix combines u <- (u then v) whose v all carry the same matrices
// (A, C, J) — the steps t >= 1 of a time-invariant model, or the aggregates of its
// full blocks — maps u.C through the same function at every step: the Riccati
// recursion of the filtered covariance.  Once one combine returns u.C unchanged
// (same bits), every later combine of the chain receives the same C and the same
// v matrices, so it forms the same inverse and returns the same C, A = 0 and J:
// only (b, eta) still move.  g_bc_vec_t advances them in place with the inverse
// the last full combine kept (keep_minv: its transpose in s.S) and v's A (its
// transpose in s.T1, written when the fixed point is found), by the vector
// operations of g_combine_bc_t in their order — the bits of the full combine,
// without its d^3 products.  Every operand is read by columns (u.C by symmetry:
// a combine output's C is symmetric to the bit), so the lanes' shared-memory
// reads are conflict-free.  (A rounding 2-cycle never triggers the test and keeps
// the full combines; the result is identical either way.)
template <int DC>
__device__ __forceinline__ void g_bc_vec_t(const Grp& g, int d_rt, double* u, const double* vb,
                                           const double* veta, const CombScratch& s) {
  const int d = DC ? DC : d_rt;
  const int dd = d * d;
  double *ub = u + dd, *ueta = u + 2 * dd + d;
  const double* uC = u + dd + d;  // symmetric: uC[k][i] = uC[i][k]
  const double* vAt = s.T1;       // v's A, transposed
  const double* MinvT = s.S;
  for (int i = g.lane; i < d; i += g.size) {
    double acc = 0.0;
    for (int k = 0; k < d; ++k) acc += uC[k * d + i] * veta[k];
    s.t[i] = acc + ub[i];
  }
  g.sync();
  for (int i = g.lane; i < d; i += g.size) {
    double acc = 0.0;
    for (int k = 0; k < d; ++k) acc += MinvT[k * d + i] * s.t[k];
    s.w[i] = acc;
  }
  g.sync();
  for (int i = g.lane; i < d; i += g.size) {
    double acc = 0.0;
    for (int k = 0; k < d; ++k) acc += vAt[k * d + i] * s.w[k];
    ub[i] = acc + vb[i];
    ueta[i] = 0.0 + ueta[i];
  }
  g.sync();
}

// v's vectors (b, eta) at vb, veta: in the element, or staged by the caller
__device__ __noinline__ void g_bc_vec2(const Grp& g, int d, double* u, const double* vb,
                                       const double* veta, const CombScratch& s) {
  if (d == 16) g_bc_vec_t<16>(g, d, u, vb, veta, s);
  else g_bc_vec_t<0>(g, d, u, vb, veta, s);
}
__device__ __forceinline__ void g_bc_vec(const Grp& g, int d, double* u, const double* v,
                                         const CombScratch& s) {
  g_bc_vec2(g, d, u, v + d * d, v + 2 * d * d + d, s);
}

// vector-only steps taken (auxmc_test_fixed_point_steps)
__device__ unsigned long long g_fp_steps = 0;

// one step u <- (u then v) of a prefix chain; `same`: v's matrices are the
// chain's shared ones (read from vsh when given).  fixed: the chain sits at a
// covariance fixed point (its A transposed into s.T1, the kept inverse's transpose
// in s.S: g_bc_vec_t); o is the full combine's output buffer.
__device__ __forceinline__ void bc_chain_step(const Grp& g, int d, double* u, const double* v,
                                              bool same, double* o, const CombScratch& s,
                                              bool& fixed, int& nvec,
                                              const double* vsh = nullptr) {
  const int dd = d * d;
  if (fixed && same) {
    g_bc_vec(g, d, u, v, s);
    ++nvec;
    return;
  }
  const double* vm = same && vsh ? vsh : v;
  g_combine_bc(g, d, u, v, o, s, same, vm);
  fixed = same && g_all_same(g, dd, o + dd + d, u + dd + d, s.idx);
  if (fixed)
    for (int e = g.lane; e < dd; e += g.size) s.T1[e] = vm[(e % d) * d + e / d];
  g_copy(g, fe_size_g(d), o, u);
  g.sync();
}

__host__ __device__ inline int comb_doubles(int d) { return 3 * d * d + 2 * d; }
__host__ __device__ inline int comb_ints(int d) { return 2 * d + 2; }

__device__ CombScratch comb_scratch(int d, double* base, int* ibase) {
  CombScratch s;
  const int dd = d * d;
  s.S = base;
  s.T1 = s.S + dd;
  s.T2 = s.T1 + dd;
  s.t = s.T2 + dd;
  s.w = s.t + d;
  s.p1 = ibase;
  s.p2 = ibase + d;
  s.idx = ibase + 2 * d;
  return s;
}

struct GrpCfg {
  bool block;
  int groups;  // per CTA
  int threads;
};

__host__ __device__ inline GrpCfg grp_cfg(int dx, int dy) {
  if (dx <= 16 && dy <= 16) return GrpCfg{false, 4, 128};
  return GrpCfg{true, 1, 128};
}

// gain^T and hs factors of the time-invariant step (k_pfg_elem_fill)
__host__ __device__ inline int proto_doubles(int d, int dy) { return 2 * dy * d; }

// ---------------------------------------------------------------- element build
// per (b, t); smem per group: f, q, a, t1, t2 (dd), hq, X1, X2, gr (dy*dx), s, L, scr (dy^2),
// innov, hv, bd (vectors)
__host__ __device__ inline int elem_smem(int d, int dy) {
  const int W = d > dy ? d : dy;
  return 5 * d * d + 4 * dy * d + 4 * dy * dy + 3 * W + 8;
}

template <bool BLOCK>
__global__ void k_pfg_elements(DevModel m, const double* __restrict__ obs, int B, double* el,
                               int* status, int t_lo, int t_hi, double* proto = nullptr) {
  extern __shared__ double smem[];
  const int T = m.T, d = m.dx, dy = m.dy, dd = d * d, ES = fe_size_g(d);
  const int W = d > dy ? d : dy;
  const Grp g = BLOCK ? block_group() : warp_group();
  const int gid = BLOCK ? 0 : (threadIdx.x >> 5), gpb = BLOCK ? 1 : (blockDim.x >> 5);
  double* sm = smem + (size_t)gid * elem_smem(d, dy);
  double *f = sm, *qm = f + dd, *a = qm + dd, *t1 = a + dd, *t2 = t1 + dd;
  double *hq = t2 + dd, *X1 = hq + dy * d, *X2 = X1 + dy * d, *gr = X2 + dy * d;
  double *s = gr + dy * d, *L = s + dy * dy, *scr = L + dy * dy, *fs = scr + dy * dy;
  double *innov = fs + dy * dy, *hv = innov + W, *bd = hv + W;
  double* red = bd + W;
  int* flag = reinterpret_cast<int*>(red + 2);
  const int span = t_hi - t_lo;  // time range [t_lo, t_hi) of this launch
  const long long n = (long long)B * span;
  for (long long qq = (long long)blockIdx.x * gpb + gid; qq < n; qq += (long long)gridDim.x * gpb) {
    const int b = (int)(qq / span), t = t_lo + (int)(qq % span);
    const long long q = (long long)b * (T + 1) + t;
    double* e = el + (size_t)q * ES;
    double *eA = e, *eb = e + dd, *eC = e + dd + d, *eeta = e + 2 * dd + d, *eJ = e + 2 * dd + 2 * d;
    const double* Qs = t == 0 ? m.P0 : m.Qt(t - 1, b);
    for (int i = g.ty(); i < d; i += g.ny())
      for (int j = g.tx(); j < d; j += 16) {
        f[i * d + j] = t == 0 ? (i == j ? 1.0 : 0.0) : m.Ft(t - 1, b)[i * d + j];
        qm[i * d + j] = 0.5 * (Qs[i * d + j] + Qs[j * d + i]);  // Model ctor symmetrization
      }
    for (int i = g.lane; i < d; i += g.size) bd[i] = t == 0 ? m.m0[i] : m.bt(t - 1, b)[i];
    g.sync();
    int st = 0;
    if (dy > 0 && m.observed(t)) {
      const double* h = m.Ht(t, b);
      const double* c = m.ct(t, b);
      const double* R = m.Rt(t, b);
      const double* y = obs + (size_t)q * dy;
      for (int i = g.lane; i < dy; i += g.size) {
        double acc = 0.0;
        for (int j = 0; j < d; ++j) acc += h[i * d + j] * bd[j];
        innov[i] = (y[i] - acc) - c[i];
      }
      g_mm(g, dy, d, d, h, qm, hq);
      for (int i = g.ty(); i < dy; i += g.ny())
        for (int j = g.tx(); j < dy; j += 16) scr[i * dy + j] = 0.5 * (R[i * dy + j] + R[j * dy + i]);
      g.sync();
      g_mm_nt(g, dy, d, dy, hq, h, s, scr);
      g.sync();
      g_symm(g, dy, s);
      g.sync();
      st = g_factor_psd(g, dy, s, L, fs, flag, red);  // fs: jitter matrix / inverted blocks
      if (st == 0) {
        g_copy(g, dy * d, hq, X1);
        g_copy(g, dy * d, h, X2);
        g.sync();
        g_llt_solve(g, dy, L, d, X1, fs);  // gain = X1^T
        g_llt_solve(g, dy, L, d, X2, fs);  // hs = X2^T
        // a = I - gain h ; A = a f
        g_mm_tn(g, d, dy, d, X1, h, a);
        g.sync();
        for (int i = g.ty(); i < d; i += g.ny())
          for (int j = g.tx(); j < d; j += 16) a[i * d + j] = (i == j ? 1.0 : 0.0) - a[i * d + j];
        g.sync();
        g_mm(g, d, d, d, a, f, eA);
        for (int i = g.lane; i < d; i += g.size) {
          double acc = 0.0;
          for (int k = 0; k < dy; ++k) acc += X1[k * d + i] * innov[k];
          eb[i] = bd[i] + acc;
        }
        // C = symm(a q a^T + gain Rs gain^T)
        g_mm(g, d, d, d, a, qm, t1);
        g_mm_tn(g, d, dy, dy, X1, scr, gr);
        g.sync();
        g_mm_nt(g, d, d, d, t1, a, t2);
        g.sync();
        g_mm(g, d, dy, d, gr, X1, t1, t2);
        g.sync();
        for (int i = g.ty(); i < d; i += g.ny())
          for (int j = g.tx(); j < d; j += 16) eC[i * d + j] = 0.5 * (t1[i * d + j] + t1[j * d + i]);
        // eta = f^T (hs innov) ; J = symm(((f^T hs) h) f)
        for (int i = g.lane; i < d; i += g.size) {
          double acc = 0.0;
          for (int k = 0; k < dy; ++k) acc += X2[k * d + i] * innov[k];
          hv[i] = acc;
        }
        g.sync();
        for (int i = g.lane; i < d; i += g.size) {
          double acc = 0.0;
          for (int k = 0; k < d; ++k) acc += f[k * d + i] * hv[k];
          eeta[i] = acc;
        }
        g_mm(g, dy, d, d, X2, f, gr);  // (f^T hs)^T = X2 f  (dy×d)
        g.sync();
        g_mm_tn(g, d, dy, d, gr, h, t1);  // (f^T hs) h
        g.sync();
        g_mm(g, d, d, d, t1, f, t2);
        g.sync();
        for (int i = g.ty(); i < d; i += g.ny())
          for (int j = g.tx(); j < d; j += 16) eJ[i * d + j] = 0.5 * (t2[i * d + j] + t2[j * d + i]);
        if (proto && t == 1) {  // gain^T and hs of the time-invariant step (k_pfg_elem_fill)
          g_copy(g, dy * d, X1, proto + (size_t)b * proto_doubles(d, dy));
          g_copy(g, dy * d, X2, proto + (size_t)b * proto_doubles(d, dy) + dy * d);
        }
      }
    } else {
      for (int i = g.lane; i < dd; i += g.size) {
        eA[i] = f[i];
        eC[i] = qm[i];
        eJ[i] = 0.0;
      }
      for (int i = g.lane; i < d; i += g.size) {
        eb[i] = bd[i];
        eeta[i] = 0.0;
      }
    }
    g.sync();
    if (t == 0)
      for (int i = g.lane; i < dd; i += g.size) eA[i] = 0.0;
    if (st && g.lane == 0 && status) atomicMax(status + b, st);
    g.sync();
  }
}

// ---------------------------------------------------------------- time-invariant elements
// When F, b, Q, H, c, R are shared by every step (strides 0, no mask; e.g. the
// auxiliary LGSSM of a linear-dynamics target), the elements of t >= 1 differ
// only in (b, eta): A, C, J and the gain / hs factors are those of t = 1.  One
// group builds t = 1 in full (k_pfg_elements, proto != nullptr keeps X1, X2);
// k_pfg_elem_fill then forms every other step's vectors with the same loops in
// the same order as the full build and copies the matrices — identical bits.
inline bool pfg_time_invariant(const DevModel& m) {
  return m.T >= 2 && m.dy > 0 && m.mask == nullptr && m.dx <= 16 && m.dy <= 16 && m.nF <= 1 &&
         m.nb <= 1 && m.nQ <= 1 && m.nH <= 1 && m.nc <= 1 && m.nR <= 1;
}

// Every step t >= 1 builds its element matrices (A, C, J) from the same F, Q, H, R
// by the same operations (b, c and the data only reach the vectors): the
// covariance fixed point of the prefix chains applies (bc_chain_step).
inline bool pfg_shared_mats(const DevModel& m) {
  return m.T >= 2 && m.mask == nullptr && m.nF <= 1 && m.nQ <= 1 && m.nH <= 1 && m.nR <= 1;
}
// auxmc_test_pfg_fixed_point(0): every prefix step a full combine (the parity
// tests compare both forms bit for bit)
int g_pfg_fixed_on = 1;
// the prefix chains over the elements read the matrices of every step t >= 1 from
// el[1] (the fill path's shared element), so the fill writes only the vectors
inline bool shared_el_reads(const DevModel& m, bool block) {
  return g_pfg_fixed_on && !block && pfg_time_invariant(m);
}
struct SameRanges {
  int el_lo, el_hi;    // element indices t with the shared matrices
  int agg_lo, agg_hi;  // block aggregates (full blocks past the first)
  int sup_lo, sup_hi;  // super-block aggregates (made of such blocks only)
};
inline SameRanges same_ranges(const DevModel& m, int LB, int LB2) {
  SameRanges r{0, 0, 0, 0, 0, 0};
  if (!g_pfg_fixed_on || !pfg_shared_mats(m)) return r;
  const int nfull = (m.T + 1) / LB;
  r.el_lo = 1;
  r.el_hi = m.T + 1;
  r.agg_lo = 1;
  r.agg_hi = nfull;
  r.sup_lo = 1;
  r.sup_hi = LB2 > 0 ? nfull / LB2 : 0;
  return r;
}

constexpr int kFillWarps = 8;
// warp w of a CTA: 32 consecutive steps of sequence b, lane = step
__global__ void __launch_bounds__(kFillWarps * 32)
    k_pfg_elem_fill(DevModel m, const double* __restrict__ obs, int B, double* el,
                    const double* __restrict__ proto, int t_lo, int t_hi, int write_mats) {
  __shared__ double s_mat[3 * 256], s_x1[256], s_x2[256], s_h[256], s_f[256], s_c[16], s_bd[16];
  const int T = m.T, d = m.dx, dy = m.dy, dd = d * d, ES = fe_size_g(d);
  const int span = t_hi - t_lo;
  const int per_b = (span + 32 * kFillWarps - 1) / (32 * kFillWarps);
  const int b = blockIdx.x / per_b, chunk = blockIdx.x % per_b;
  if (b >= B) return;
  const double* e1 = el + ((size_t)b * (T + 1) + 1) * ES;
  const double* pr = proto + (size_t)b * proto_doubles(d, dy);
  for (int i = threadIdx.x; i < dd; i += blockDim.x) {
    s_mat[i] = e1[i];                    // A
    s_mat[dd + i] = e1[dd + d + i];      // C
    s_mat[2 * dd + i] = e1[2 * dd + 2 * d + i];  // J
    s_f[i] = m.Ft(0, b)[i];
  }
  for (int i = threadIdx.x; i < dy * d; i += blockDim.x) {
    s_x1[i] = pr[i];
    s_x2[i] = pr[dy * d + i];
    s_h[i] = m.Ht(0, b)[i];
  }
  for (int i = threadIdx.x; i < dy; i += blockDim.x) s_c[i] = m.ct(0, b)[i];
  for (int i = threadIdx.x; i < d; i += blockDim.x) s_bd[i] = m.bt(0, b)[i];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t0 = t_lo + (chunk * kFillWarps + warp) * 32;
  if (t0 >= t_hi) return;
  const int t = t0 + lane;
  if (t < t_hi) {
    double* e = el + ((size_t)b * (T + 1) + t) * ES;
    const double* y = obs + ((size_t)b * (T + 1) + t) * dy;
    double innov[16], hv[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (i < dy) {
        double acc = 0.0;
        for (int j = 0; j < d; ++j) acc += s_h[i * d + j] * s_bd[j];
        innov[i] = (y[i] - acc) - s_c[i];
      }
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (i < d) {
        double acc = 0.0, acc2 = 0.0;
#pragma unroll
        for (int k = 0; k < 16; ++k)
          if (k < dy) {
            acc += s_x1[k * d + i] * innov[k];
            acc2 += s_x2[k * d + i] * innov[k];
          }
        e[dd + i] = s_bd[i] + acc;  // b
        hv[i] = acc2;
      }
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (i < d) {
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < 16; ++k)
          if (k < d) acc += s_f[k * d + i] * hv[k];
        e[2 * dd + d + i] = acc;  // eta
      }
    }
  }
  // A, C, J of the warp's 32 steps, coalesced — unless every reader takes them from
  // the shared element el[1] (write_mats = 0: the prefix chains' vsh)
  if (!write_mats) return;
  const int nt = min(32, t_hi - t0);
  for (int u = 0; u < nt; ++u) {
    double* e = el + ((size_t)b * (T + 1) + t0 + u) * ES;
    for (int i = lane; i < dd; i += 32) {
      e[i] = s_mat[i];
      e[dd + d + i] = s_mat[dd + i];
      e[2 * dd + 2 * d + i] = s_mat[2 * dd + i];
    }
  }
}

// ---------------------------------------------------------------- S1 / S2 / S3
// per group: nes element buffers (2 for S1/S2, 3 for S3) + combine scratch
__host__ __device__ inline int scan_smem(int d, int nes) {
  return nes * fe_size_g(d) + comb_doubles(d) + comb_ints(d);
}

template <bool BLOCK>
__global__ void k_pfg_reduce(int T, int d, int B, int LB, const double* __restrict__ el, double* agg,
                             int k_lo, int k_hi) {
  extern __shared__ double smem[];
  const int ES = fe_size_g(d);
  const Grp g = BLOCK ? block_group() : warp_group();
  const int gid = BLOCK ? 0 : (threadIdx.x >> 5), gpb = BLOCK ? 1 : (blockDim.x >> 5);
  double* sm = smem + (size_t)gid * scan_smem(d, 2);
  double *acc = sm, *o = acc + ES;
  const CombScratch cs = comb_scratch(d, o + ES, reinterpret_cast<int*>(o + ES + comb_doubles(d)));
  const int nblk = (T + 1 + LB - 1) / LB;
  const int span = k_hi - k_lo;  // block range [k_lo, k_hi) of this launch
  const long long n = (long long)B * span;
  for (long long qq = (long long)blockIdx.x * gpb + gid; qq < n; qq += (long long)gridDim.x * gpb) {
    const int b = (int)(qq / span), k = k_lo + (int)(qq % span);
    const long long q = (long long)b * nblk + k;
    const int lo = k * LB, hi = min(lo + LB, T + 1);
    const double* base = el + (size_t)b * (T + 1) * ES;
    g_copy(g, ES, base + (size_t)lo * ES, acc);
    g.sync();
    for (int t = lo + 1; t < hi; ++t) {
      g_combine(g, d, acc, base + (size_t)t * ES, o, cs);
      g_copy(g, ES, o, acc);
      g.sync();
    }
    g_copy(g, ES, acc, agg + (size_t)q * ES);
    g.sync();
  }
}

// S1 for a time-invariant model (pfg_time_invariant): every block but the first
// combines elements whose matrix parts are those of t = 1, so the running
// aggregate's matrices after p combines, and the inverse each combine forms, are
// the same in every block.  k_pfg_reduce_proto runs that matrix sequence once
// (on el[1] alone) and keeps, per position p, [A_p | C_p | J_p | Minv_{p+1} | its
// transpose] (the transpose lets the fill read every operand column-wise);
// k_pfg_reduce_fill then carries each block's (b, eta) through the combine's
// vector formulas, in g_combine's loop order — identical bits to k_pfg_reduce.
__host__ __device__ inline int rproto_doubles(int d, int LB) { return 5 * d * d * LB; }

template <bool BLOCK>
__global__ void k_pfg_reduce_proto(int T, int d, int B, int LB, const double* __restrict__ el,
                                   double* mats) {
  extern __shared__ double smem[];
  const int ES = fe_size_g(d), dd = d * d;
  const Grp g = BLOCK ? block_group() : warp_group();
  const int gid = BLOCK ? 0 : (threadIdx.x >> 5), gpb = BLOCK ? 1 : (blockDim.x >> 5);
  double* sm = smem + (size_t)gid * scan_smem(d, 3);
  double *acc = sm, *o = acc + ES, *e1 = o + ES;  // e1: the shared element, staged
  const CombScratch cs = comb_scratch(d, e1 + ES, reinterpret_cast<int*>(e1 + ES + comb_doubles(d)));
  for (int b = blockIdx.x * gpb + gid; b < B; b += gridDim.x * gpb) {
    const double* e1g = el + ((size_t)b * (T + 1) + 1) * ES;
    double* M = mats + (size_t)b * rproto_doubles(d, LB);
    g_copy(g, ES, e1g, acc);
    g_copy(g, ES, e1g, e1);
    g.sync();
    for (int p = 0; p < LB; ++p) {
      double* Mp = M + (size_t)p * 5 * dd;
      g_copy(g, dd, acc, Mp);
      g_copy(g, dd, acc + dd + d, Mp + dd);
      g_copy(g, dd, acc + 2 * dd + 2 * d, Mp + 2 * dd);
      g.sync();
      if (p + 1 < LB) {
        g_combine(g, d, acc, e1, o, cs, Mp + 3 * dd);
        for (int e = g.lane; e < dd; e += g.size) Mp[4 * dd + e] = Mp[3 * dd + (e % d) * d + e / d];
        g_copy(g, ES, o, acc);
        g.sync();
      }
    }
  }
}

// g_combine_t (warp groups, d <= 16) spread over four warps of a CTA: every product
// and vector loop is the same warp-level routine on the same operands as in the
// one-warp combine (identical bits); the independent ones run side by side, so the
// chain of dependent products is four long instead of nine.  X: one extra d×d buffer
// (uA^T T2 while S is still being read).  Minv (and its transpose) saved for the fill.
template <int DC>
__device__ __forceinline__ void combine4_t(int d_rt, const double* u, const double* v, double* o,
                                           const CombScratch& s, double* X, double* save_minv,
                                           double* save_minv_t) {
  const int d = DC ? DC : d_rt;
  const int dd = d * d;
  const Grp g = warp_group();
  const int warp = threadIdx.x >> 5;
  const double *uA = u, *ub = u + dd, *uC = u + dd + d, *ueta = u + 2 * dd + d,
               *uJ = u + 2 * dd + 2 * d;
  const double *vA = v, *vb = v + dd, *vC = v + dd + d, *veta = v + 2 * dd + d,
               *vJ = v + 2 * dd + 2 * d;
  double *oA = o, *ob = o + dd, *oC = o + dd + d, *oeta = o + 2 * dd + d, *oJ = o + 2 * dd + 2 * d;
  double* const M1 = oC;
  double* Minv = oJ;
  double* mt = M1;
  double* mt2 = M1 + d;
  // A: Minv = (I + uC vJ)^{-1} (warp 0) | t, w (warp 1)
  if (warp == 0) {
    g_mm(g, d, d, d, uC, vJ, M1);
    g.sync();
    for (int i = g.lane; i < d; i += g.size) M1[i * d + i] += 1.0;
    g.sync();
    w_inverse_gj_t<DC>(g.lane, d, M1, Minv);
  } else if (warp == 1) {
    for (int i = g.lane; i < d; i += g.size) {
      double acc = 0.0, acc2 = 0.0;
      for (int k = 0; k < d; ++k) {
        acc += uC[i * d + k] * veta[k];
        acc2 += vJ[i * d + k] * ub[k];
      }
      s.t[i] = acc + ub[i];
      s.w[i] = veta[i] - acc2;
    }
  }
  __syncthreads();
  // B: S = Minv uA | T1 = Minv uC | T2 = Minv^T vJ | mt, mt2 and the saved inverse
  if (warp == 0) {
    g_mm(g, d, d, d, Minv, uA, s.S);
  } else if (warp == 1) {
    g_mm(g, d, d, d, Minv, uC, s.T1);
  } else if (warp == 2) {
    g_mm_tn(g, d, d, d, Minv, vJ, s.T2);
  } else {
    for (int i = g.lane; i < d; i += g.size) {
      double acc = 0.0, acc2 = 0.0;
      for (int k = 0; k < d; ++k) {
        acc += Minv[i * d + k] * s.t[k];
        acc2 += Minv[k * d + i] * s.w[k];
      }
      mt[i] = acc;
      mt2[i] = acc2;
    }
    if (save_minv)
      for (int e = g.lane; e < dd; e += 32) {
        save_minv[e] = Minv[e];
        save_minv_t[e] = Minv[(e % d) * d + e / d];
      }
  }
  __syncthreads();
  // C: A = vA S | Minv' = vA T1 | X = uA^T T2 | b, eta
  if (warp == 0) {
    g_mm(g, d, d, d, vA, s.S, oA);
  } else if (warp == 1) {
    g_mm(g, d, d, d, vA, s.T1, Minv);
  } else if (warp == 2) {
    g_mm_tn(g, d, d, d, uA, s.T2, X);
  } else {
    for (int i = g.lane; i < d; i += g.size) {
      double acc = 0.0, acc2 = 0.0;
      for (int k = 0; k < d; ++k) {
        acc += vA[i * d + k] * mt[k];
        acc2 += uA[k * d + i] * mt2[k];
      }
      ob[i] = acc + vb[i];
      oeta[i] = acc2 + ueta[i];
    }
  }
  __syncthreads();
  // D: T1 = Minv' vA^T + vC | T2 = X uA + uJ
  if (warp == 0) g_mm_nt(g, d, d, d, Minv, vA, s.T1, vC);
  else if (warp == 1) g_mm(g, d, d, d, X, uA, s.T2, uJ);
  __syncthreads();
  for (int e = threadIdx.x; e < dd; e += blockDim.x) {
    const int i = e / d, j = e % d;
    oC[e] = 0.5 * (s.T1[i * d + j] + s.T1[j * d + i]);
    oJ[e] = 0.5 * (s.T2[i * d + j] + s.T2[j * d + i]);
  }
  __syncthreads();
}

__device__ __noinline__ void combine4(int d, const double* u, const double* v, double* o,
                                      const CombScratch& s, double* X, double* save_minv,
                                      double* save_minv_t) {
  if (d == 16) combine4_t<16>(d, u, v, o, s, X, save_minv, save_minv_t);
  else combine4_t<0>(d, u, v, o, s, X, save_minv, save_minv_t);
}

// k_pfg_reduce for warp-group models on four warps (combine4), a CTA per item: the
// super-block reduction of the two-level scan, whose LB2-long chains of full
// combines are its serial depth
__global__ void __launch_bounds__(128)
    k_pfg_reduce4(int T, int d, int B, int LB, const double* __restrict__ el, double* agg,
                  int k_lo, int k_hi) {
  extern __shared__ double smem[];
  const int ES = fe_size_g(d);
  double *acc = smem, *o = acc + ES, *vs = o + ES;
  const CombScratch cs = comb_scratch(d, vs + ES, reinterpret_cast<int*>(vs + ES + comb_doubles(d)));
  double* X = vs + ES + comb_doubles(d) + comb_ints(d);
  const int nblk = (T + 1 + LB - 1) / LB;
  const int span = k_hi - k_lo;
  const long long n = (long long)B * span;
  for (long long qq = blockIdx.x; qq < n; qq += gridDim.x) {
    const int b = (int)(qq / span), k = k_lo + (int)(qq % span);
    const long long q = (long long)b * nblk + k;
    const int lo = k * LB, hi = min(lo + LB, T + 1);
    const double* base = el + (size_t)b * (T + 1) * ES;
    for (int e = threadIdx.x; e < ES; e += blockDim.x) acc[e] = base[(size_t)lo * ES + e];
    __syncthreads();
    for (int t = lo + 1; t < hi; ++t) {
      for (int e = threadIdx.x; e < ES; e += blockDim.x) vs[e] = base[(size_t)t * ES + e];
      __syncthreads();
      combine4(d, acc, vs, o, cs, X, nullptr, nullptr);
      for (int e = threadIdx.x; e < ES; e += blockDim.x) acc[e] = o[e];
      __syncthreads();
    }
    for (int e = threadIdx.x; e < ES; e += blockDim.x) agg[(size_t)q * ES + e] = acc[e];
    __syncthreads();
  }
}

// k_pfg_reduce_proto for warp-group models on four warps (combine4): a CTA per
// sequence, the same matrices bit for bit
constexpr int kProto4Threads = 128;
__host__ __device__ inline int proto4_smem(int d) {
  return 3 * fe_size_g(d) + comb_doubles(d) + comb_ints(d) + d * d;
}
__global__ void __launch_bounds__(kProto4Threads)
    k_pfg_reduce_proto4(int T, int d, int B, int LB, const double* __restrict__ el,
                        double* mats) {
  extern __shared__ double smem[];
  const int ES = fe_size_g(d), dd = d * d;
  double *acc = smem, *o = acc + ES, *e1 = o + ES;
  const CombScratch cs = comb_scratch(d, e1 + ES, reinterpret_cast<int*>(e1 + ES + comb_doubles(d)));
  double* X = e1 + ES + comb_doubles(d) + comb_ints(d);
  for (int b = blockIdx.x; b < B; b += gridDim.x) {
    const double* e1g = el + ((size_t)b * (T + 1) + 1) * ES;
    double* M = mats + (size_t)b * rproto_doubles(d, LB);
    for (int e = threadIdx.x; e < ES; e += blockDim.x) {
      acc[e] = e1g[e];
      e1[e] = e1g[e];
    }
    __syncthreads();
    for (int p = 0; p < LB; ++p) {
      double* Mp = M + (size_t)p * 5 * dd;
      for (int e = threadIdx.x; e < dd; e += blockDim.x) {
        Mp[e] = acc[e];
        Mp[dd + e] = acc[dd + d + e];
        Mp[2 * dd + e] = acc[2 * dd + 2 * d + e];
      }
      __syncthreads();
      if (p + 1 < LB) {
        combine4(d, acc, e1, o, cs, X, Mp + 3 * dd, Mp + 4 * dd);
        for (int e = threadIdx.x; e < ES; e += blockDim.x) acc[e] = o[e];
        __syncthreads();
      }
    }
  }
}

// warp per (sequence, block), blocks [max(k_lo, 1), k_hi): lane i of the low half
// carries b_i, lane i of the high half eta_i; each length-d sum is one lane's, over
// the other half's entries gathered by shuffles, in g_combine's order — identical bits
constexpr int kFillWarpsR = 8;
__global__ void __launch_bounds__(kFillWarpsR * 32)
    k_pfg_reduce_fill(int T, int d, int B, int LB, const double* __restrict__ el,
                      const double* __restrict__ mats, double* agg, int k_lo, int k_hi) {
  __shared__ double s_vt[kFillWarpsR][2][256];  // per warp: vA^T, vJ^T of its sequence
  const int ES = fe_size_g(d), dd = d * d;
  const int nblk = (T + 1 + LB - 1) / LB;
  const int k0 = max(k_lo, 1), span = k_hi - k0;
  const long long n = (long long)B * span;
  const int lane = threadIdx.x & 31, hi = lane >> 4, i = lane & 15;
  const int src = lane & 16;  // this half's first lane
  const bool row = i < d;
  for (long long qq = (long long)blockIdx.x * kFillWarpsR + (threadIdx.x >> 5); qq < n;
       qq += (long long)gridDim.x * kFillWarpsR) {
    const int b = (int)(qq / span), k = k0 + (int)(qq % span);
    const int lo = k * LB, hb = min(lo + LB, T + 1);
    const double* base = el + (size_t)b * (T + 1) * ES;
    const double* M = mats + (size_t)b * rproto_doubles(d, LB);
    const double* e1 = base + ES;  // v matrices (shared by every t >= 1)
    const double* e = base + (size_t)lo * ES;
    // the constant operands transposed in shared memory: the lane's row of vJ (high
    // half) / vA (low half) is read as a column, conflict-free
    double* vt = s_vt[threadIdx.x >> 5][0];
    for (int e2 = lane; e2 < dd; e2 += 32) {
      const int r2 = e2 / d, c2 = e2 % d;
      vt[c2 * d + r2] = e1[e2];
      vt[256 + c2 * d + r2] = e1[2 * dd + 2 * d + e2];
    }
    __syncwarp();
    const double* vr = vt + (hi ? 256 : 0);
    // x: b_i (low half) / eta_i (high half)
    double x = row ? (hi ? e[2 * dd + d + i] : e[dd + i]) : 0.0;
    for (int t = lo + 1; t < hb; ++t) {
      const int p = t - lo - 1;  // u = aggregate after p combines
      const double* Mp = M + (size_t)p * 5 * dd;
      // column-wise reads (coalesced across the half): uC is symmetric (bits), uA^T's
      // column i is uA[:, i]; Minv's row i is column i of its stored transpose.  All of
      // the step's operands are loaded up front (one memory latency per step).
      const double* Pa = Mp + (hi ? 0 : dd);           // high: uA[q][i]; low: uC[q][i] = uC[i][q]
      const double* Pm = Mp + (hi ? 3 * dd : 4 * dd);  // high: Minv[q][i]; low: Minv^T[q][i]
      const double* ev = base + (size_t)t * ES;
      double pa[16], pm[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        pa[q] = (row && q < d) ? Pa[q * d + i] : 0.0;
        pm[q] = (row && q < d) ? Pm[q * d + i] : 0.0;
      }
      const double veta_i = row ? ev[2 * dd + d + i] : 0.0;
      const double vb_i = (row && !hi) ? ev[dd + i] : 0.0;
      // low: tt_i = uC[i,:] veta + ub_i ; high: w_i = veta_i - vJ[i,:] ub
      double acc = 0.0;
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        if (q < d) {
          const double ubq = __shfl_sync(0xffffffffu, x, q);
          const double veq = __shfl_sync(0xffffffffu, veta_i, q);
          if (row) acc += (hi ? vr[q * d + i] : pa[q]) * (hi ? ubq : veq);
        }
      }
      const double z = row ? (hi ? veta_i - acc : acc + x) : 0.0;
      // low: mt_i = Minv[i,:] tt ; high: mt2_i = Minv[:,i] . w
      acc = 0.0;
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        if (q < d) {
          const double zq = __shfl_sync(0xffffffffu, z, src + q);
          if (row) acc += pm[q] * zq;
        }
      }
      const double mz = acc;
      // low: ub_i = vA[i,:] mt + vb_i ; high: ueta_i = uA[:,i] . mt2 + ueta_i
      acc = 0.0;
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        if (q < d) {
          const double mq = __shfl_sync(0xffffffffu, mz, src + q);
          if (row) acc += (hi ? pa[q] : vr[q * d + i]) * mq;
        }
      }
      if (row) x = hi ? acc + x : acc + vb_i;
    }
    const double* Mf = M + (size_t)(hb - lo - 1) * 5 * dd;
    double* out = agg + ((size_t)b * nblk + k) * ES;
    for (int e2 = lane; e2 < dd; e2 += 32) {
      out[e2] = Mf[e2];
      out[dd + d + e2] = Mf[dd + e2];
      out[2 * dd + 2 * d + e2] = Mf[2 * dd + e2];
    }
    if (row) out[hi ? 2 * dd + d + i : dd + i] = x;
    __syncwarp();  // s_vt is rewritten for the warp's next block
  }
}

// Block 0 of a model with shared step matrices: its first element (t = 0) has
// A = 0, so the block is a prefix chain (bc_chain_step, the carries' form and
// fixed point) — the aggregate g_combine's chain would give, at 4 d^3 products
// per step or none once the covariance is fixed.
template <bool BLOCK>
__global__ void k_pfg_reduce0_bc(int T, int d, int B, int LB, const double* __restrict__ el,
                                 double* agg, int same_lo, int same_hi, int shared_el) {
  extern __shared__ double smem[];
  const int ES = fe_size_g(d);
  const Grp g = BLOCK ? block_group() : warp_group();
  const int gid = BLOCK ? 0 : (threadIdx.x >> 5), gpb = BLOCK ? 1 : (blockDim.x >> 5);
  double* sm = smem + (size_t)gid * scan_smem(d, 2);
  double *acc = sm, *o = acc + ES;
  const CombScratch cs = comb_scratch(d, o + ES, reinterpret_cast<int*>(o + ES + comb_doubles(d)));
  const int nblk = (T + 1 + LB - 1) / LB;
  const int hb = min(LB, T + 1);
  for (int b = blockIdx.x * gpb + gid; b < B; b += gridDim.x * gpb) {
    const double* base = el + (size_t)b * (T + 1) * ES;
    g_copy(g, ES, base, acc);
    g.sync();
    bool fixed = false;
    int nvec = 0;
    const double* vsh = shared_el ? base + (size_t)same_lo * ES : nullptr;
    for (int t = 1; t < hb; ++t)
      bc_chain_step(g, d, acc, base + (size_t)t * ES, t >= same_lo && t < same_hi, o, cs, fixed,
                    nvec, vsh);
    g_copy(g, ES, acc, agg + (size_t)b * nblk * ES);
    if (g.lane == 0 && nvec) atomicAdd(&g_fp_steps, (unsigned long long)nvec);
    g.sync();
  }
}

template <bool BLOCK>
__global__ void k_pfg_carry(int T, int d, int B, int LB, const double* __restrict__ agg, double* carry,
                            int same_lo, int same_hi) {
  extern __shared__ double smem[];
  const int ES = fe_size_g(d);
  const Grp g = BLOCK ? block_group() : warp_group();
  const int gid = BLOCK ? 0 : (threadIdx.x >> 5), gpb = BLOCK ? 1 : (blockDim.x >> 5);
  double* sm = smem + (size_t)gid * scan_smem(d, 2);
  double *acc = sm, *o = acc + ES;
  const CombScratch cs = comb_scratch(d, o + ES, reinterpret_cast<int*>(o + ES + comb_doubles(d)));
  const int nblk = (T + 1 + LB - 1) / LB;
  for (int b = blockIdx.x * gpb + gid; b < B; b += gridDim.x * gpb) {
    const double* ab = agg + (size_t)b * nblk * ES;
    g_copy(g, ES, ab, acc);
    g.sync();
    bool fixed = false;
    int nvec = 0;
    for (int k = 1; k < nblk; ++k) {
      g_copy(g, ES, acc, carry + ((size_t)b * nblk + k) * ES);
      g.sync();
      bc_chain_step(g, d, acc, ab + (size_t)k * ES, k >= same_lo && k < same_hi, o, cs, fixed,
                    nvec);  // prefixes
    }
    if (g.lane == 0 && nvec) atomicAdd(&g_fp_steps, (unsigned long long)nvec);
  }
}

// S2 for many blocks, second level: carries of the level-1 aggregates from the
// exclusive carries of super-blocks of LB2 aggregates (carry2, from k_pfg_carry
// over the super-block aggregates).
template <bool BLOCK>
__global__ void k_pfg_carry_seg(int nblk, int d, int B, int LB2, const double* __restrict__ agg,
                                const double* __restrict__ carry2, double* carry, int j_lo,
                                int j_hi, int same_lo, int same_hi) {
  extern __shared__ double smem[];
  const int ES = fe_size_g(d);
  const Grp g = BLOCK ? block_group() : warp_group();
  const int gid = BLOCK ? 0 : (threadIdx.x >> 5), gpb = BLOCK ? 1 : (blockDim.x >> 5);
  double* sm = smem + (size_t)gid * scan_smem(d, 2);
  double *acc = sm, *o = acc + ES;
  const CombScratch cs = comb_scratch(d, o + ES, reinterpret_cast<int*>(o + ES + comb_doubles(d)));
  const int nsup = (nblk + LB2 - 1) / LB2;
  const int span = j_hi - j_lo;  // super-block range [j_lo, j_hi) of this launch
  const long long n = (long long)B * span;
  for (long long qq = (long long)blockIdx.x * gpb + gid; qq < n; qq += (long long)gridDim.x * gpb) {
    const int b = (int)(qq / span), j = j_lo + (int)(qq % span);
    const long long q = (long long)b * nsup + j;
    const int lo = j * LB2, hi = min(lo + LB2, nblk);
    const double* A = agg + (size_t)b * nblk * ES;
    double* Cy = carry + (size_t)b * nblk * ES;
    int k = lo;
    if (j == 0) {
      g_copy(g, ES, A + (size_t)lo * ES, acc);
      k = lo + 1;
    } else {
      g_copy(g, ES, carry2 + (size_t)q * ES, acc);
    }
    g.sync();
    bool fixed = false;
    int nvec = 0;
    for (; k < hi; ++k) {
      g_copy(g, ES, acc, Cy + (size_t)k * ES);
      g.sync();
      if (k + 1 < hi)
        bc_chain_step(g, d, acc, A + (size_t)k * ES, k >= same_lo && k < same_hi, o, cs, fixed,
                      nvec);  // prefixes
    }
    if (g.lane == 0 && nvec) atomicAdd(&g_fp_steps, (unsigned long long)nvec);
  }
}

// per applied block: [flag, next step, b (d), C, Minv^T, vA^T (d*d each)] — a block
// that reached the covariance fixed point hands its remaining steps to
// k_pfg_apply_lanes
__host__ __device__ inline int apply_rec_doubles(int d) { return 2 + d + 3 * d * d; }

template <bool BLOCK>
__global__ void k_pfg_apply(int T, int d, int B, int LB, const double* __restrict__ el,
                            const double* __restrict__ carry, double* filt_mean, double* filt_cov,
                            int k_lo, int k_hi, int same_lo, int same_hi, int shared_el,
                            double* recs) {
  extern __shared__ double smem[];
  const int ES = fe_size_g(d), dd = d * d;
  const Grp g = BLOCK ? block_group() : warp_group();
  const int gid = BLOCK ? 0 : (threadIdx.x >> 5), gpb = BLOCK ? 1 : (blockDim.x >> 5);
  double* sm = smem + (size_t)gid * scan_smem(d, 2);
  // the block's carry is read only by the first combine, whose output is acc: it
  // shares the combine output buffer o (two element buffers per group, not three)
  double *acc = sm, *o = acc + ES, *cy = o;
  const CombScratch cs = comb_scratch(d, o + ES, reinterpret_cast<int*>(o + ES + comb_doubles(d)));
  const int nblk = (T + 1 + LB - 1) / LB;
  const int span = k_hi - k_lo;
  const long long n = (long long)B * span;
  for (long long qq = (long long)blockIdx.x * gpb + gid; qq < n; qq += (long long)gridDim.x * gpb) {
    const int b = (int)(qq / span), k = k_lo + (int)(qq % span);
    const long long q = (long long)b * nblk + k;
    const int lo = k * LB, hi = min(lo + LB, T + 1);
    const double* base = el + (size_t)b * (T + 1) * ES;
    const double* vsh = shared_el ? base + (size_t)same_lo * ES : nullptr;
    bool fixed = false;
    int nvec = 0;
    if (recs && g.lane == 0) recs[(size_t)qq * apply_rec_doubles(d)] = 0.0;
    if (k == 0) {
      g_copy(g, ES, base + (size_t)lo * ES, acc);
      g.sync();
    } else {
      g_copy(g, ES, carry + (size_t)q * ES, cy);
      g.sync();
      const bool same = lo >= same_lo && lo < same_hi;
      const double* vm = same && vsh ? vsh : base + (size_t)lo * ES;
      g_combine_bc(g, d, cy, base + (size_t)lo * ES, acc, cs, same, vm);  // carries are prefixes
      fixed = same && g_all_same(g, dd, acc + dd + d, cy + dd + d, cs.idx);
      if (fixed) {
        for (int e = g.lane; e < dd; e += g.size) cs.T1[e] = vm[(e % d) * d + e / d];
        g.sync();
      }
    }
    // at the fixed point the next step's (b, eta) are loaded one step ahead into
    // registers (lane i < d: its entries) and staged in cs.T2 (free in this form)
    double pvb = 0.0, pve = 0.0;
    bool pre = false;
    for (int t = lo;; ++t) {
      for (int i = g.lane; i < d; i += g.size)
        filt_mean[((size_t)b * (T + 1) + t) * d + i] = acc[dd + i];
      for (int i = g.lane; i < dd; i += g.size)
        filt_cov[((size_t)b * (T + 1) + t) * dd + i] = acc[dd + d + i];
      if (t + 1 >= hi) break;
      g.sync();
      const bool same1 = t + 1 >= same_lo && t + 1 < same_hi;
      if (recs && fixed && same1 && hi - 1 < same_hi) {
        // every remaining step is a vector step: record the state and stop here
        double* rc = recs + (size_t)qq * apply_rec_doubles(d);
        for (int i = g.lane; i < d; i += g.size) rc[2 + i] = acc[dd + i];
        for (int e = g.lane; e < dd; e += g.size) {
          rc[2 + d + e] = acc[dd + d + e];
          rc[2 + d + dd + e] = cs.S[e];
          rc[2 + d + 2 * dd + e] = cs.T1[e];
        }
        if (g.lane == 0) {
          rc[0] = 1.0;
          rc[1] = (double)(t + 1);
        }
        break;
      }
      if (fixed && same1) {
        const double* v1 = base + (size_t)(t + 1) * ES;
        if (!pre && g.lane < d) {
          pvb = v1[dd + g.lane];
          pve = v1[2 * dd + d + g.lane];
        }
        if (g.lane < d) {
          cs.T2[g.lane] = pvb;
          cs.T2[d + g.lane] = pve;
        }
        pre = t + 2 < hi && t + 2 >= same_lo && t + 2 < same_hi;
        if (pre && g.lane < d) {
          const double* v2 = v1 + ES;
          pvb = v2[dd + g.lane];
          pve = v2[2 * dd + d + g.lane];
        }
        g.sync();
        if (d == 16) g_bc_vec_t<16>(g, d, acc, cs.T2, cs.T2 + d, cs);  // inlined: no call frame
        else g_bc_vec2(g, d, acc, cs.T2, cs.T2 + d, cs);
        ++nvec;
      } else {
        bc_chain_step(g, d, acc, base + (size_t)(t + 1) * ES, same1, o, cs, fixed, nvec, vsh);
        pre = false;
      }
    }
    if (g.lane == 0 && nvec) atomicAdd(&g_fp_steps, (unsigned long long)nvec);
    g.sync();
  }
}

// ---------------------------------------------------------------- recovery
__host__ __device__ inline int rec_smem(int d, int dy) {
  const int W = d > dy ? d : dy;
  return 4 * d * d + dy * d + 3 * dy * dy + 2 * W + 8;
}
// steps per group in the recovery: consecutive steps, so a group can keep the
// predictive covariance and the innovation factor of the previous step
#ifndef AUXMC_REC_CHUNK
#define AUXMC_REC_CHUNK 128
#endif
constexpr int kRecChunk = AUXMC_REC_CHUNK;

// warp groups per CTA, per kernel: as many as its per-group shared-memory
// footprint and its register count allow (<= 16; 12 -> 16 took the C5 iteration
// 200 -> 196 ms, 20/24 no further) — the combine chains are latency-bound, so
// occupancy matters
struct KCfg {
  int gp, threads;
  size_t smem;
};
template <typename K>
KCfg kcfg(K kernel, int d, int dy, int per_doubles) {
  const GrpCfg c = grp_cfg(d, dy);
  const size_t per = sizeof(double) * (size_t)per_doubles;
  if (c.block) return KCfg{1, c.threads, per};
  cudaFuncAttributes fa{};
  int regs = 128, max_warps = 32;
  if (cudaFuncGetAttributes(&fa, kernel) == cudaSuccess && fa.numRegs > 0) {
    regs = fa.numRegs;
    max_warps = fa.maxThreadsPerBlock / 32;  // the driver's per-block resource bound
  }
  const int by_regs = std::min(max_warps, 65536 / (32 * ((regs + 7) / 8 * 8)));
  const int gp = (int)std::max<size_t>(
      1, std::min<size_t>({(size_t)16, (size_t)by_regs, (220 * 1024) / per}));
  return KCfg{gp, 32 * gp, per * gp};
}
inline int kgrid(const KCfg& c, long long k) {
  return (int)std::max(1LL, std::min((k + c.gp - 1) / c.gp, 148LL * 16));
}
template <typename K>
int set_smem(K kernel, const KCfg& c) {
  if (c.smem > 227 * 1024) return AUXMC_E_DIM;
  AUXMC_CUDA_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)c.smem));
  return AUXMC_OK;
}
#define PFG_TRY(x)          \
  do {                      \
    const int rc_ = (x);    \
    if (rc_) return rc_;    \
  } while (0)

// the super-block reduction: combine4 CTAs for warp-group models (the one-warp
// combine's bits), the group kernel otherwise
template <bool BLOCK>
int launch_sup_reduce(int T, int d, int B, int LB, const double* agg, double* agg2, int k_lo,
                      int k_hi, const KCfg& c2, cudaStream_t s) {
  if (!BLOCK) {
    const size_t sm = sizeof(double) * proto4_smem(d);
    AUXMC_CUDA_TRY(cudaFuncSetAttribute(k_pfg_reduce4,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    const long long n = (long long)B * (k_hi - k_lo);
    AUXMC_LAUNCH(k_pfg_reduce4, (int)std::min<long long>(n, 148LL * 16), 128, sm, s, T, d, B, LB,
                 agg, agg2, k_lo, k_hi);
  } else {
    AUXMC_LAUNCH(k_pfg_reduce<BLOCK>, kgrid(c2, (long long)B * (k_hi - k_lo)), c2.threads,
                 c2.smem, s, T, d, B, LB, agg, agg2, k_lo, k_hi);
  }
  return AUXMC_OK;
}

// the block-matrix sequence: four warps per sequence for warp-group models (the
// one-warp combine's bits), the group kernel otherwise
template <bool BLOCK>
int launch_proto(int T, int d, int B, int LB, const double* el, double* mats, const KCfg& cp,
                 cudaStream_t s) {
  if (!BLOCK) {
    const size_t sm = sizeof(double) * proto4_smem(d);
    AUXMC_CUDA_TRY(cudaFuncSetAttribute(k_pfg_reduce_proto4,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    AUXMC_LAUNCH(k_pfg_reduce_proto4, B, kProto4Threads, sm, s, T, d, B, LB, el, mats);
  } else {
    AUXMC_LAUNCH(k_pfg_reduce_proto<BLOCK>, kgrid(cp, B), cp.threads, cp.smem, s, T, d, B, LB, el,
                 mats);
  }
  return AUXMC_OK;
}

// The block-matrix sequence (k_pfg_reduce_proto, one warp, LB serial combines)
// needs only the shared element el[1]: it is forked onto a side stream once that
// element is built and runs beside the element fill and block 0's chain; the block
// fill waits for it.
struct ProtoJob {
  int LB;
  double* mats;
  KCfg cp;
  bool forked;
};
struct SideStream {
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
inline int side_stream(SideStream** out) {
  static SideStream sd;
  if (!sd.s) {
    AUXMC_CUDA_TRY(cudaStreamCreateWithFlags(&sd.s, cudaStreamNonBlocking));
    AUXMC_CUDA_TRY(cudaEventCreateWithFlags(&sd.fork, cudaEventDisableTiming));
    AUXMC_CUDA_TRY(cudaEventCreateWithFlags(&sd.join, cudaEventDisableTiming));
  }
  *out = &sd;
  return AUXMC_OK;
}

// elements of [t_lo, t_hi): the fill path when the model is time-invariant
// (t = 1 always built in full for its factors), the full build otherwise
template <bool BLOCK>
int launch_elements(const DevModel& dm, const double* obs, int B, double* el, double* proto,
                    int* status, int t_lo, int t_hi, const KCfg& ce, cudaStream_t s,
                    ProtoJob* pj = nullptr) {
  if (t_hi <= t_lo) return AUXMC_OK;
  if (!proto || !pfg_time_invariant(dm) || BLOCK) {
    AUXMC_LAUNCH(k_pfg_elements<BLOCK>, kgrid(ce, (long long)B * (t_hi - t_lo)), ce.threads,
                 ce.smem, s, dm, obs, B, el, status, t_lo, t_hi, (double*)nullptr);
    return AUXMC_OK;
  }
  const int f_lo = t_lo == 0 ? 0 : 1;  // full build of t = 1 (and t = 0 when owned)
  AUXMC_LAUNCH(k_pfg_elements<BLOCK>, kgrid(ce, (long long)B * (2 - f_lo)), ce.threads, ce.smem,
               s, dm, obs, B, el, status, f_lo, 2, proto);
  if (pj && pj->mats && pj->LB >= 2) {
    SideStream* sd = nullptr;
    PFG_TRY(side_stream(&sd));
    AUXMC_CUDA_TRY(cudaEventRecord(sd->fork, s));
    AUXMC_CUDA_TRY(cudaStreamWaitEvent(sd->s, sd->fork, 0));
    PFG_TRY(launch_proto<BLOCK>(dm.T, dm.dx, B, pj->LB, el, pj->mats, pj->cp, sd->s));
    AUXMC_CUDA_TRY(cudaEventRecord(sd->join, sd->s));
    pj->forked = true;
  }
  const int g_lo = std::max(t_lo, 2);
  if (t_hi > g_lo) {
    const int per_b = (t_hi - g_lo + 32 * kFillWarps - 1) / (32 * kFillWarps);
    AUXMC_LAUNCH(k_pfg_elem_fill, B * per_b, 32 * kFillWarps, 0, s, dm, obs, B, el, proto, g_lo,
                 t_hi, shared_el_reads(dm, BLOCK) ? 0 : 1);
  }
  return AUXMC_OK;
}

// S1 over blocks [k_lo, k_hi): the proto + fill path for time-invariant models
template <bool BLOCK>
int launch_reduce(const DevModel& dm, int B, int LB, const double* el, double* mats, double* agg,
                  int k_lo, int k_hi, const KCfg& c2, const KCfg& cp, cudaStream_t s,
                  int same_lo = 0, int same_hi = 0, const ProtoJob* pj = nullptr) {
  const int T = dm.T, d = dm.dx;
  if (k_hi <= k_lo) return AUXMC_OK;
  if (!mats || BLOCK || !pfg_time_invariant(dm) || LB < 2) {
    AUXMC_LAUNCH(k_pfg_reduce<BLOCK>, kgrid(c2, (long long)B * (k_hi - k_lo)), c2.threads,
                 c2.smem, s, T, d, B, LB, el, agg, k_lo, k_hi);
    return AUXMC_OK;
  }
  const bool forked = pj && pj->forked;
  if (!forked) PFG_TRY(launch_proto<BLOCK>(T, d, B, LB, el, mats, cp, s));
  if (k_lo == 0) {
    if (same_hi > same_lo) {
      const KCfg c0 = kcfg(k_pfg_reduce0_bc<BLOCK>, d, dm.dy, scan_smem(d, 2));
      PFG_TRY(set_smem(k_pfg_reduce0_bc<BLOCK>, c0));
      AUXMC_LAUNCH(k_pfg_reduce0_bc<BLOCK>, kgrid(c0, B), c0.threads, c0.smem, s, T, d, B, LB, el,
                   agg, same_lo, same_hi, shared_el_reads(dm, BLOCK) ? 1 : 0);
    } else {
      AUXMC_LAUNCH(k_pfg_reduce<BLOCK>, kgrid(c2, B), c2.threads, c2.smem, s, T, d, B, LB, el, agg,
                   0, 1);
    }
  }
  if (forked) {
    SideStream* sd = nullptr;
    PFG_TRY(side_stream(&sd));
    AUXMC_CUDA_TRY(cudaStreamWaitEvent(s, sd->join, 0));
  }
  const int k0 = std::max(k_lo, 1);
  if (k_hi > k0) {
    const long long n = (long long)B * (k_hi - k0);
    AUXMC_LAUNCH(k_pfg_reduce_fill,
                 (int)std::min<long long>((n + kFillWarpsR - 1) / kFillWarpsR, 148LL * 32),
                 32 * kFillWarpsR, 0, s, T, d, B, LB, el, mats, agg, k_lo, k_hi);
  }
  return AUXMC_OK;
}

// The remaining steps of every block k_pfg_apply recorded at the fixed point: a warp
// per block advances b by g_bc_vec_t's three products in its order (same bits) from
// shared-memory copies of the record, and writes the block's filtered moments — a
// light kernel at full occupancy instead of the combine kernel's.  d <= 16.
constexpr int kApplyLaneWarps = 8;
__global__ void __launch_bounds__(kApplyLaneWarps * 32)
    k_pfg_apply_lanes(int T, int d, int B, int LB, const double* __restrict__ el,
                      const double* __restrict__ recs, double* filt_mean, double* filt_cov,
                      int k_lo, int k_hi) {
  extern __shared__ double asm_[];
  const int ES = fe_size_g(d), dd = d * d;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double* sm = asm_ + (size_t)w * (3 * dd + 4 * 16);
  double *uC = sm, *MinvT = uC + dd, *vAt = MinvT + dd, *ub = vAt + dd, *tt = ub + 16,
         *ww = tt + 16;
  const int span = k_hi - k_lo;
  const long long n = (long long)B * span;
  for (long long qq = (long long)blockIdx.x * kApplyLaneWarps + w; qq < n;
       qq += (long long)gridDim.x * kApplyLaneWarps) {
    const double* rc = recs + (size_t)qq * apply_rec_doubles(d);
    if (rc[0] == 0.0) continue;
    const int b = (int)(qq / span), k = k_lo + (int)(qq % span);
    const int lo = k * LB, hi = min(lo + LB, T + 1);
    const int t0 = (int)rc[1];
    if (lane == 0) atomicAdd(&g_fp_steps, (unsigned long long)(hi - t0));
    for (int i = lane; i < d; i += 32) ub[i] = rc[2 + i];
    for (int e = lane; e < dd; e += 32) {
      uC[e] = rc[2 + d + e];
      MinvT[e] = rc[2 + d + dd + e];
      vAt[e] = rc[2 + d + 2 * dd + e];
    }
    __syncwarp();
    const double* base = el + (size_t)b * (T + 1) * ES;
    for (int t = t0; t < hi; ++t) {
      const double* v = base + (size_t)t * ES;
      const double *vb = v + dd, *veta = v + 2 * dd + d;
      if (lane < d) {
        double acc = 0.0;
        for (int kk = 0; kk < d; ++kk) acc += uC[kk * d + lane] * veta[kk];
        tt[lane] = acc + ub[lane];
      }
      __syncwarp();
      if (lane < d) {
        double acc = 0.0;
        for (int kk = 0; kk < d; ++kk) acc += MinvT[kk * d + lane] * tt[kk];
        ww[lane] = acc;
      }
      __syncwarp();
      if (lane < d) {
        double acc = 0.0;
        for (int kk = 0; kk < d; ++kk) acc += vAt[kk * d + lane] * ww[kk];
        ub[lane] = acc + vb[lane];
        filt_mean[((size_t)b * (T + 1) + t) * d + lane] = ub[lane];
      }
      double* fc = filt_cov + ((size_t)b * (T + 1) + t) * dd;
      for (int e = lane; e < dd; e += 32) fc[e] = uC[e];
      __syncwarp();
    }
  }
}

int launch_apply_lanes(int T, int d, int B, int LB, const double* el, const double* recs,
                       auxmc_filter_result* out, int k_lo, int k_hi, cudaStream_t s) {
  const size_t sm = sizeof(double) * (size_t)kApplyLaneWarps * (3 * d * d + 64);
  AUXMC_CUDA_TRY(cudaFuncSetAttribute(k_pfg_apply_lanes,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  const long long n = (long long)B * (k_hi - k_lo);
  AUXMC_LAUNCH(k_pfg_apply_lanes,
               (int)std::min<long long>((n + kApplyLaneWarps - 1) / kApplyLaneWarps, 148LL * 16),
               32 * kApplyLaneWarps, sm, s, T, d, B, LB, el, recs, out->filt_mean, out->filt_cov,
               k_lo, k_hi);
  return AUXMC_OK;
}

// per recovery chunk (kRecChunk steps): [uniform flag, status, log det, L (dy^2)]
__host__ __device__ inline int rec_rec_doubles(int dy) { return 3 + dy * dy; }

// The steps (c0, c1) of every chunk k_pfg_recover marked uniform — each previous
// filtered covariance has the bits of step c0's, so every step has step c0's
// predictive covariance (pc row c0) and innovation factor (the chunk record):
// one lane per step forms its predictive mean and innovation term by the per-step
// code's operations in its order (the warp log-density's forward substitution and
// square sum element by element; the log-diagonal sum is the record's) — the same
// bits, as independent lanes of a light kernel instead of the step-serial chain of
// the warp group.  d, dy <= 16.
constexpr int kRecLaneWarps = 8;
__global__ void __launch_bounds__(kRecLaneWarps * 32)
    k_pfg_recover_lanes(DevModel m, const double* __restrict__ obs, int B,
                        const double* __restrict__ fm, double* pm, double* pc, double* terms,
                        int* status, int t_lo, int t_hi, const double* __restrict__ recs) {
  constexpr int MX = 16;
  const int T = m.T, d = m.dx, dy = m.dy, dd = d * d;
  const int lane = threadIdx.x & 31;
  const int span = t_hi - t_lo;
  const int nch = (span + kRecChunk - 1) / kRecChunk;
  const long long n = (long long)B * nch;
  for (long long qq = (long long)blockIdx.x * kRecLaneWarps + (threadIdx.x >> 5); qq < n;
       qq += (long long)gridDim.x * kRecLaneWarps) {
    const double* rc = recs + (size_t)qq * rec_rec_doubles(dy);
    if (rc[0] == 0.0) continue;  // not uniform: k_pfg_recover took every step
    const int b = (int)(qq / nch), c0 = t_lo + (int)(qq % nch) * kRecChunk;
    const int c1 = min(c0 + kRecChunk, t_hi);
    const int st = (int)rc[1];
    const double ld = rc[2];
    const double* L = rc + 3;
    const double* P = pc + ((size_t)b * (T + 1) + c0) * dd;
    for (int u = c0 + 1; u < c1; ++u) {
      double* row = pc + ((size_t)b * (T + 1) + u) * dd;
      for (int e = lane; e < dd; e += 32) row[e] = P[e];
    }
    for (int t = c0 + 1 + lane; t < c1; t += 32) {
      const long long q = (long long)b * (T + 1) + t;
      const double* F = m.Ft(t - 1, b);
      const double* bb = m.bt(t - 1, b);
      const double* x = fm + (size_t)(q - 1) * d;
      double xv[MX], mv[MX];
#pragma unroll
      for (int k = 0; k < MX; ++k) xv[k] = k < d ? x[k] : 0.0;
#pragma unroll
      for (int i = 0; i < MX; ++i) {
        if (i < d) {
          double acc = 0.0;
#pragma unroll
          for (int k = 0; k < MX; ++k)
            if (k < d) acc += F[i * d + k] * xv[k];
          mv[i] = acc + bb[i];
          pm[(size_t)q * d + i] = mv[i];
        }
      }
      double term = 0.0;
      if (dy > 0 && m.observed(t)) {
        if (st) {
          atomicMax(status + b, st);
        } else {
          const double* h = m.Ht(t, b);
          const double* c = m.ct(t, b);
          const double* y = obs + (size_t)q * dy;
          const int nn = dy;
          double w[MX];
#pragma unroll
          for (int i = 0; i < MX; ++i) {
            if (i < nn) {
              double acc = 0.0;
#pragma unroll
              for (int k = 0; k < MX; ++k)
                if (k < d) acc += h[i * d + k] * mv[k];
              w[i] = y[i] - (acc + c[i]);  // x - mean, mean = H m + c
            }
          }
          w[0] = w[0] / L[0];
#pragma unroll
          for (int i = 0; i < MX; ++i) {
            if (i < nn) {
#pragma unroll
              for (int j = i + 1; j < MX; ++j) {
                if (j < nn) {
                  if (j == i + 1) w[j] = (w[j] - L[j * nn + i] * w[i]) / L[j * nn + j];
                  else w[j] -= L[j * nn + i] * w[i];
                }
              }
            }
          }
          double sq = 0.0;
#pragma unroll
          for (int i = 0; i < MX; ++i)
            if (i < nn) sq += w[i] * w[i];
          term = -0.5 * (nn * kLog2Pi + sq) - ld;
        }
      }
      terms[q] = term;
    }
  }
}

template <bool BLOCK>
__global__ void k_pfg_recover(DevModel m, const double* __restrict__ obs, int B,
                              const double* __restrict__ fm, const double* __restrict__ fc,
                              double* pm, double* pc, double* terms, int* status, int t_lo,
                              int t_hi, int sb, const double* bnd, int reuse, double* recs) {
  extern __shared__ double smem[];
  const int T = m.T, d = m.dx, dy = m.dy, dd = d * d;
  const int W = d > dy ? d : dy;
  const Grp g = BLOCK ? block_group() : warp_group();
  const int gid = BLOCK ? 0 : (threadIdx.x >> 5), gpb = BLOCK ? 1 : (blockDim.x >> 5);
  double* sm = smem + (size_t)gid * rec_smem(d, dy);
  double *P = sm, *t1 = P + dd, *qs = t1 + dd, *hp = qs + dd, *s = hp + dy * d, *L = s + dy * dy,
         *scr = L + dy * dy;
  double *mp = scr + dy * dy, *r = mp + W, *red = r + W;
  int* flag = reinterpret_cast<int*>(red + 2);
  double* Cprev = red + 4;  // the filtered covariance P, L and scr were formed from
  const int span = t_hi - t_lo;
  const int nch = (span + kRecChunk - 1) / kRecChunk;
  const long long n = (long long)B * nch;
  for (long long qq = (long long)blockIdx.x * gpb + gid; qq < n; qq += (long long)gridDim.x * gpb) {
    const int b = (int)(qq / nch), c0 = t_lo + (int)(qq % nch) * kRecChunk;
    const int c1 = min(c0 + kRecChunk, t_hi);
    // reuse (shared F, Q, H, R; pfg_shared_mats): a step whose previous filtered
    // covariance has the bits of the one P, L were formed from has the same
    // predictive covariance and innovation factor — the time-invariant filter's
    // steady state, where only the means move
    bool have = false;
    int st_keep = 0;
    for (int t = c0; t < c1; ++t) {
    const long long q = (long long)b * (T + 1) + t;
    bool hit = false;
    if constexpr (!BLOCK) {
      // every later step of the chunk repeats step c0's covariance: leave them to
      // k_pfg_recover_lanes with the chunk's record
      if (t == c0 + 1 && recs) {
        double* rc = recs + (size_t)qq * rec_rec_doubles(dy);
        bool all = have && !(sb > 0 && c0 / sb != (c1 - 1) / sb);
        if (all) {
          all = __all_sync(0xffffffffu, rows_match_part(fc + (size_t)(q - 1) * dd, Cprev, c1 - t,
                                                        dd, g.lane, 32));
        }
        if (g.lane == 0) {
          rc[0] = all ? 1.0 : 0.0;
          rc[1] = (double)st_keep;
          double ld = 0.0;  // the warp log-density's sum of the logs of L's diagonal
          if (all && st_keep == 0 && dy > 0)
            for (int i = 0; i < dy; ++i) ld += log(L[i * dy + i]);
          rc[2] = ld;
        }
        if (all) {
          for (int e = g.lane; e < dy * dy; e += 32) rc[3 + e] = L[e];
          __syncwarp();
          break;
        }
        __syncwarp();
      }
    }
    if (t == 0) {
      have = false;
      for (int i = g.lane; i < d; i += g.size) mp[i] = m.m0[i];
      for (int i = g.ty(); i < d; i += g.ny())
        for (int j = g.tx(); j < d; j += 16) P[i * d + j] = 0.5 * (m.P0[i * d + j] + m.P0[j * d + i]);
      g.sync();
    } else {
      const double* F = m.Ft(t - 1, b);
      const double* bb = m.bt(t - 1, b);
      const double* Q = m.Qt(t - 1, b);
      // time-sharded filter: at a super-block start the previous filtered moments
      // are the super-block carry's (b, C), so every rank split sees the same bits
      const bool at_sb = sb > 0 && t % sb == 0;
      const double* x = at_sb ? bnd + (size_t)(t / sb) * (d + dd) : fm + (size_t)(q - 1) * d;
      const double* C = at_sb ? x + d : fc + (size_t)(q - 1) * dd;
      for (int i = g.lane; i < d; i += g.size) {
        double acc = 0.0;
        for (int k = 0; k < d; ++k) acc += F[i * d + k] * x[k];
        mp[i] = acc + bb[i];
      }
      hit = reuse && have && g_all_same(g, dd, C, Cprev, flag);
      if (!hit) {
        g_mm(g, d, d, d, F, C, t1);
        for (int i = g.ty(); i < d; i += g.ny())
          for (int j = g.tx(); j < d; j += 16) qs[i * d + j] = 0.5 * (Q[i * d + j] + Q[j * d + i]);
        if (reuse) g_copy(g, dd, C, Cprev);
        g.sync();
        g_mm_nt(g, d, d, d, t1, F, P, qs);
        g.sync();
        g_symm(g, d, P);
        g.sync();
        have = reuse != 0;
      }
    }
    for (int i = g.lane; i < d; i += g.size) pm[(size_t)q * d + i] = mp[i];
    for (int i = g.lane; i < dd; i += g.size) pc[(size_t)q * dd + i] = P[i];
    double term = 0.0;
    if (dy > 0 && m.observed(t)) {
      const double* h = m.Ht(t, b);
      const double* c = m.ct(t, b);
      const double* R = m.Rt(t, b);
      const double* y = obs + (size_t)q * dy;
      for (int i = g.lane; i < dy; i += g.size) {
        double acc = 0.0;
        for (int k = 0; k < d; ++k) acc += h[i * d + k] * mp[k];
        r[i] = acc + c[i];  // mean H m + c
      }
      int st = st_keep;
      if (!hit) {
        g_mm(g, dy, d, d, h, P, hp);
        g.sync();
        g_mm_nt(g, dy, d, dy, hp, h, s, R);
        g.sync();
        g_symm(g, dy, s);
        g.sync();
        st = st_keep = g_factor_psd(g, dy, s, L, scr, flag, red);
      } else {
        g.sync();
      }
      if (st) {
        if (g.lane == 0 && status) atomicMax(status + b, st);
      } else {
        term = g_log_pdf_factored(g, dy, y, r, L, hp /* work */, red, scr);
      }
    }
    if (g.lane == 0) terms[q] = term;
    g.sync();
    }
  }
}

__global__ void k_pfg_sum(int T, int B, const double* terms, double* out, const double* parts) {
  __shared__ double red[kSumThreads];
  const int b = blockIdx.x;
  const double* tm = terms + (size_t)b * (T + 1);
  const double s = cta_sum_fixed((long long)T + 1, [&](long long i) { return tm[i]; }, red,
                                 parts ? parts + (size_t)b * kSumThreads : nullptr);
  if (threadIdx.x == 0) out[b] = s;
}

// block length ~ (T+1)^(1/3): S1 and S3 run LB sequential combines, S2 runs two
// levels of ~LB when there are many blocks.
// super-blocks of LB / 4 blocks (the super-level reduction's full combines are the
// serial depth the carries' fixed point cannot shorten), at least one prefix-sampler
// block long (both powers of two: the super-block is a multiple of it)
int pf_sup_g(int T, int LB) {
  return std::max({2, LB / 4, prefix_block_len(T > 0 ? T : 1) / LB});
}
int pf_block_g(int T) {
  int lb = 4;
  while ((long long)lb * lb * lb < T + 1) lb <<= 1;
  return lb;
}
constexpr int kPfTwoLevel = 64;  // blocks above which S2 is itself blocked

template <bool BLOCK>
int run_pfg(const DevModel& dm, const double* obs, int B, auxmc_filter_result* out, int* status,
            Arena& ws, cudaStream_t s) {
  const int T = dm.T, d = dm.dx, dy = dm.dy, LB = pf_block_g(T);
  const int ES = fe_size_g(d);
  const int nblk = (T + 1 + LB - 1) / LB;
  double* el = ws.take<double>((size_t)B * (T + 1) * ES);
  double* agg = ws.take<double>((size_t)B * nblk * ES);
  double* carry = ws.take<double>((size_t)B * nblk * ES);
  double* terms = ws.take<double>((size_t)B * (T + 1));
  double* proto = ws.take<double>((size_t)B * proto_doubles(d, dy));
  double* mats = ws.take<double>((size_t)B * rproto_doubles(d, LB));
  double* recs = ws.take<double>((size_t)B * ((T + kRecChunk) / kRecChunk) * rec_rec_doubles(dy));
  double* arecs = ws.take<double>((size_t)B * nblk * apply_rec_doubles(d));
  const bool two = nblk > kPfTwoLevel;
  const int LB2 = pf_sup_g(T, LB), nsup = (nblk + LB2 - 1) / LB2;
  double* agg2 = two ? ws.take<double>((size_t)B * nsup * ES) : nullptr;
  double* carry2 = two ? ws.take<double>((size_t)B * nsup * ES) : nullptr;
  if (ws.base == nullptr) return AUXMC_OK;
  if (!el || !agg || !carry || !terms || !proto || !mats || !recs || !arecs ||
      (two && (!agg2 || !carry2)))
    return AUXMC_E_WORKSPACE;
  const KCfg ce = kcfg(k_pfg_elements<BLOCK>, d, dy, elem_smem(d, dy));
  const KCfg c2 = kcfg(k_pfg_reduce<BLOCK>, d, dy, scan_smem(d, 2));
  const KCfg cp = kcfg(k_pfg_reduce_proto<BLOCK>, d, dy, scan_smem(d, 3));
  const KCfg cc = kcfg(k_pfg_carry<BLOCK>, d, dy, scan_smem(d, 2));
  const KCfg cg = kcfg(k_pfg_carry_seg<BLOCK>, d, dy, scan_smem(d, 2));
  const KCfg c3 = kcfg(k_pfg_apply<BLOCK>, d, dy, scan_smem(d, 2));
  const KCfg cr = kcfg(k_pfg_recover<BLOCK>, d, dy, rec_smem(d, dy));
  PFG_TRY(set_smem(k_pfg_elements<BLOCK>, ce));
  PFG_TRY(set_smem(k_pfg_reduce<BLOCK>, c2));
  PFG_TRY(set_smem(k_pfg_reduce_proto<BLOCK>, cp));
  PFG_TRY(set_smem(k_pfg_carry<BLOCK>, cc));
  PFG_TRY(set_smem(k_pfg_carry_seg<BLOCK>, cg));
  PFG_TRY(set_smem(k_pfg_apply<BLOCK>, c3));
  PFG_TRY(set_smem(k_pfg_recover<BLOCK>, cr));
  if (status) AUXMC_CUDA_TRY(cudaMemsetAsync(status, 0, sizeof(int) * B, s));
  const long long nb = (long long)B * nblk;
  const SameRanges sr = same_ranges(dm, LB, LB2);
  ProtoJob pj{LB, mats, cp, false};
  PFG_TRY(launch_elements<BLOCK>(dm, obs, B, el, proto, status, 0, T + 1, ce, s, &pj));
  PFG_TRY(launch_reduce<BLOCK>(dm, B, LB, el, mats, agg, 0, nblk, c2, cp, s, sr.el_lo, sr.el_hi,
                               &pj));
  if (two) {
    const long long ns = (long long)B * nsup;
    PFG_TRY(launch_sup_reduce<BLOCK>(nblk - 1, d, B, LB2, agg, agg2, 0, nsup, c2, s));
    AUXMC_LAUNCH(k_pfg_carry<BLOCK>, kgrid(cc, B), cc.threads, cc.smem, s, nsup - 1, d, B, 1, agg2,
                 carry2, sr.sup_lo, sr.sup_hi);
    AUXMC_LAUNCH(k_pfg_carry_seg<BLOCK>, kgrid(cg, ns), cg.threads, cg.smem, s, nblk, d, B, LB2,
                 agg, carry2, carry, 0, nsup, sr.agg_lo, sr.agg_hi);
  } else {
    AUXMC_LAUNCH(k_pfg_carry<BLOCK>, kgrid(cc, B), cc.threads, cc.smem, s, T, d, B, LB, agg, carry,
                 sr.agg_lo, sr.agg_hi);
  }
  double* arecs_on = (!BLOCK && sr.el_hi > 0) ? arecs : nullptr;
  AUXMC_LAUNCH(k_pfg_apply<BLOCK>, kgrid(c3, nb), c3.threads, c3.smem, s, T, d, B, LB, el, carry,
               out->filt_mean, out->filt_cov, 0, nblk, sr.el_lo, sr.el_hi,
               shared_el_reads(dm, BLOCK) ? 1 : 0, arecs_on);
  if (arecs_on) PFG_TRY(launch_apply_lanes(T, d, B, LB, el, arecs_on, out, 0, nblk, s));
  const long long nrc = (long long)B * ((T + kRecChunk) / kRecChunk);
  double* recs_on = (!BLOCK && sr.el_hi > 0) ? recs : nullptr;
  AUXMC_LAUNCH(k_pfg_recover<BLOCK>, kgrid(cr, nrc), cr.threads, cr.smem, s, dm, obs, B,
               out->filt_mean, out->filt_cov, out->pred_mean, out->pred_cov, terms, status, 0, T + 1,
               0, (const double*)nullptr, sr.el_hi > 0 ? 1 : 0, recs_on);
  if (recs_on)
    AUXMC_LAUNCH(k_pfg_recover_lanes,
                 (int)std::min<long long>((nrc + kRecLaneWarps - 1) / kRecLaneWarps, 148LL * 32),
                 32 * kRecLaneWarps, 0, s, dm, obs, B, out->filt_mean, out->pred_mean,
                 out->pred_cov, terms, status, 0, T + 1, recs_on);
  double* parts = nullptr;
  if (sum_parts_pay(B, (long long)T + 1)) {
    AUXMC_CUDA_TRY(cudaMallocAsync(&parts, sizeof(double) * B * kSumThreads, s));
    AUXMC_LAUNCH(k_sum_parts<RowTerms>, (B * kSumThreads + 7) / 8, 256, 0, s, B, (long long)T + 1,
                 RowTerms{terms, (long long)T + 1}, parts);
  }
  AUXMC_LAUNCH(k_pfg_sum, B, kSumThreads, 0, s, T, B, terms, out->log_marginal, parts);
  if (parts) cudaFreeAsync(parts, s);
  return AUXMC_OK;
}

// ---------------------------------------------------------------- time-sharded scan filter
// One sequence, horizon split over ranks by runs of super-blocks (SB = LB * LB2
// steps).  The whole block tree — blocks, super-blocks, the serial carry over
// super-block aggregates, the per-super-block log-likelihood partial sums —
// depends only on T, so every rank count reproduces the single-rank result bit
// for bit.  Exchange between the two phases: an all-gather of the super-block
// aggregates (ES doubles each).
struct TsGeom {
  int LB, nblk, LB2, nsup, SB;
};
TsGeom ts_geom(int T) {
  TsGeom g;
  g.LB = pf_block_g(T);
  g.nblk = (T + 1 + g.LB - 1) / g.LB;
  g.LB2 = pf_sup_g(T, g.LB);
  g.nsup = (g.nblk + g.LB2 - 1) / g.LB2;
  g.SB = g.LB * g.LB2;
  return g;
}

struct TsBufs {
  double *el, *agg, *carry, *terms, *agg2, *carry2, *bnd, *proto, *mats, *recs, *arecs;
};
TsBufs ts_take(const DevModel& dm, Arena& ws) {
  const TsGeom G = ts_geom(dm.T);
  const int ES = fe_size_g(dm.dx), T = dm.T;
  TsBufs b;
  b.el = ws.take<double>((size_t)(T + 1) * ES);
  b.agg = ws.take<double>((size_t)G.nblk * ES);
  b.carry = ws.take<double>((size_t)G.nblk * ES);
  b.terms = ws.take<double>((size_t)(T + 2));
  b.agg2 = ws.take<double>((size_t)G.nsup * ES);
  b.carry2 = ws.take<double>((size_t)G.nsup * ES);
  b.bnd = ws.take<double>((size_t)G.nsup * (dm.dx + dm.dx * dm.dx));
  b.proto = ws.take<double>((size_t)proto_doubles(dm.dx, dm.dy));
  b.mats = ws.take<double>((size_t)rproto_doubles(dm.dx, G.LB));
  b.recs = ws.take<double>((size_t)((T + kRecChunk) / kRecChunk + 1) * rec_rec_doubles(dm.dy));
  b.arecs = ws.take<double>((size_t)G.nblk * apply_rec_doubles(dm.dx));
  return b;
}

// filtered moments just before each owned super-block start j*SB (j > 0): (b, C)
// of the composed prefix that ends there, i.e. the carry of the super-block's
// first block
// (the carry of a super-block's first block is the super-block carry itself, so
// it is taken from carry2, which every rank holds)
__global__ void k_ts_boundary(int d, int j_lo, int j_hi, const double* carry2, double* bnd) {
  const int dd = d * d, ES = fe_size_g(d);
  for (int j = max(j_lo, 1) + blockIdx.x; j < j_hi; j += gridDim.x) {
    const double* ck = carry2 + (size_t)j * ES;
    for (int i = threadIdx.x; i < d + dd; i += blockDim.x)
      bnd[(size_t)j * (d + dd) + i] = ck[dd + i];  // (b | C) are contiguous in the element
  }
}

// sequential log-likelihood partial sum of each super-block in [j_lo, j_hi)
__global__ void k_ts_partials(int T, int SB, int j_lo, int j_hi, const double* terms, double* out) {
  const int j = j_lo + blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= j_hi) return;
  double s = 0.0;
  const int hi = min((j + 1) * SB, T + 1);
  for (int t = j * SB; t < hi; ++t) s += terms[t];
  out[j - j_lo] = s;
}

template <bool BLOCK>
int ts_filter_local(const DevModel& dm, const double* obs, int j_lo, int j_hi, Arena& ws,
                    double* sup_out, int* status, cudaStream_t s) {
  const int T = dm.T, d = dm.dx, dy = dm.dy, ES = fe_size_g(d);
  const TsGeom G = ts_geom(T);
  const TsBufs b = ts_take(dm, ws);
  if (ws.base == nullptr) return AUXMC_OK;
  if (!b.el || !b.carry2 || !b.proto || !b.mats) return AUXMC_E_WORKSPACE;
  if (j_lo < 0 || j_hi > G.nsup || j_lo >= j_hi) return AUXMC_E_ARG;
  const KCfg ce = kcfg(k_pfg_elements<BLOCK>, d, dy, elem_smem(d, dy));
  const KCfg c2 = kcfg(k_pfg_reduce<BLOCK>, d, dy, scan_smem(d, 2));
  const KCfg cp = kcfg(k_pfg_reduce_proto<BLOCK>, d, dy, scan_smem(d, 3));
  PFG_TRY(set_smem(k_pfg_elements<BLOCK>, ce));
  PFG_TRY(set_smem(k_pfg_reduce<BLOCK>, c2));
  PFG_TRY(set_smem(k_pfg_reduce_proto<BLOCK>, cp));
  const int t_lo = j_lo * G.SB, t_hi = std::min(j_hi * G.SB, T + 1);
  const int k_lo = j_lo * G.LB2, k_hi = std::min(j_hi * G.LB2, G.nblk);
  ProtoJob pj{G.LB, b.mats, cp, false};
  PFG_TRY(launch_elements<BLOCK>(dm, obs, 1, b.el, b.proto, status, t_lo, t_hi, ce, s, &pj));
  const SameRanges sr = same_ranges(dm, G.LB, G.LB2);
  PFG_TRY(launch_reduce<BLOCK>(dm, 1, G.LB, b.el, b.mats, b.agg, k_lo, k_hi, c2, cp, s, sr.el_lo,
                               sr.el_hi, &pj));
  PFG_TRY(launch_sup_reduce<BLOCK>(G.nblk - 1, d, 1, G.LB2, b.agg, b.agg2, j_lo, j_hi, c2, s));
  AUXMC_CUDA_TRY(cudaMemcpyAsync(sup_out, b.agg2 + (size_t)j_lo * ES,
                                 sizeof(double) * (size_t)(j_hi - j_lo) * ES,
                                 cudaMemcpyDeviceToDevice, s));
  return AUXMC_OK;
}

template <bool BLOCK>
int ts_filter_finish(const DevModel& dm, const double* obs, int j_lo, int j_hi, Arena& ws,
                     const double* sup_all, auxmc_filter_result* out, double* ll_out, int* status,
                     cudaStream_t s) {
  const int T = dm.T, d = dm.dx, dy = dm.dy, ES = fe_size_g(d);
  const TsGeom G = ts_geom(T);
  const TsBufs b = ts_take(dm, ws);
  if (ws.base == nullptr) return AUXMC_OK;
  if (!b.el || !b.carry2 || !b.proto || !b.mats) return AUXMC_E_WORKSPACE;
  if (j_lo < 0 || j_hi > G.nsup || j_lo >= j_hi) return AUXMC_E_ARG;
  const KCfg cc = kcfg(k_pfg_carry<BLOCK>, d, dy, scan_smem(d, 2));
  const KCfg cg = kcfg(k_pfg_carry_seg<BLOCK>, d, dy, scan_smem(d, 2));
  const KCfg c3 = kcfg(k_pfg_apply<BLOCK>, d, dy, scan_smem(d, 2));
  const KCfg cr = kcfg(k_pfg_recover<BLOCK>, d, dy, rec_smem(d, dy));
  PFG_TRY(set_smem(k_pfg_carry<BLOCK>, cc));
  PFG_TRY(set_smem(k_pfg_carry_seg<BLOCK>, cg));
  PFG_TRY(set_smem(k_pfg_apply<BLOCK>, c3));
  PFG_TRY(set_smem(k_pfg_recover<BLOCK>, cr));
  const int t_lo = j_lo * G.SB, t_hi = std::min(j_hi * G.SB, T + 1);
  const int k_lo = j_lo * G.LB2, k_hi = std::min(j_hi * G.LB2, G.nblk);
  AUXMC_CUDA_TRY(cudaMemcpyAsync(b.agg2, sup_all, sizeof(double) * (size_t)G.nsup * ES,
                                 cudaMemcpyDeviceToDevice, s));
  // every rank runs the same serial carry over all super-block aggregates
  const SameRanges sr = same_ranges(dm, G.LB, G.LB2);
  AUXMC_LAUNCH(k_pfg_carry<BLOCK>, 1, cc.threads, cc.smem, s, G.nsup - 1, d, 1, 1, b.agg2,
               b.carry2, sr.sup_lo, sr.sup_hi);
  AUXMC_LAUNCH(k_pfg_carry_seg<BLOCK>, kgrid(cg, j_hi - j_lo), cg.threads, cg.smem, s, G.nblk, d,
               1, G.LB2, b.agg, b.carry2, b.carry, j_lo, j_hi, sr.agg_lo, sr.agg_hi);
  double* arecs_on = (!BLOCK && sr.el_hi > 0) ? b.arecs : nullptr;
  AUXMC_LAUNCH(k_pfg_apply<BLOCK>, kgrid(c3, k_hi - k_lo), c3.threads, c3.smem, s, T, d, 1, G.LB,
               b.el, b.carry, out->filt_mean, out->filt_cov, k_lo, k_hi, sr.el_lo, sr.el_hi,
               shared_el_reads(dm, BLOCK) ? 1 : 0, arecs_on);
  if (arecs_on) PFG_TRY(launch_apply_lanes(T, d, 1, G.LB, b.el, arecs_on, out, k_lo, k_hi, s));
  const int jb_hi = std::min(j_hi + 1, G.nsup);  // owned super-blocks and the next one's start
  AUXMC_LAUNCH(k_ts_boundary, std::max(1, jb_hi - j_lo), 128, 0, s, d, j_lo, jb_hi, b.carry2,
               b.bnd);
  // + the predictive moments at t_hi (the next range's first step, from the
  // carry of super-block j_hi: identical bits on both ranks) for the sampler
  const int r_hi = std::min(t_hi + 1, T + 1);
  const long long nrc = (r_hi - t_lo + kRecChunk - 1) / kRecChunk;
  double* recs_on = (!BLOCK && sr.el_hi > 0) ? b.recs : nullptr;
  AUXMC_LAUNCH(k_pfg_recover<BLOCK>, kgrid(cr, nrc), cr.threads, cr.smem, s, dm, obs, 1,
               out->filt_mean, out->filt_cov, out->pred_mean, out->pred_cov, b.terms, status, t_lo,
               r_hi, G.SB, b.bnd, sr.el_hi > 0 ? 1 : 0, recs_on);
  if (recs_on)
    AUXMC_LAUNCH(k_pfg_recover_lanes,
                 (int)std::min<long long>((nrc + kRecLaneWarps - 1) / kRecLaneWarps, 148LL * 32),
                 32 * kRecLaneWarps, 0, s, dm, obs, 1, out->filt_mean, out->pred_mean,
                 out->pred_cov, b.terms, status, t_lo, r_hi, recs_on);
  AUXMC_LAUNCH(k_ts_partials, (j_hi - j_lo + 127) / 128, 128, 0, s, T, G.SB, j_lo, j_hi, b.terms,
               ll_out);
  return AUXMC_OK;
}

}  // namespace

int tshard_geometry(int T, int* LB, int* nblk, int* nsup, int* SB) {
  const TsGeom G = ts_geom(T);
  *LB = G.LB;
  *nblk = G.nblk;
  *nsup = G.nsup;
  *SB = G.SB;
  return AUXMC_OK;
}
int tshard_filter_local(const DevModel& dm, const double* obs, int j_lo, int j_hi, Arena& ws,
                        double* sup_out, int* status, cudaStream_t s) {
  if (dm.dx > 32 || dm.dy > 64) return AUXMC_E_DIM;
  return grp_cfg(dm.dx, dm.dy).block ? ts_filter_local<true>(dm, obs, j_lo, j_hi, ws, sup_out, status, s)
                                     : ts_filter_local<false>(dm, obs, j_lo, j_hi, ws, sup_out, status, s);
}
int tshard_filter_finish(const DevModel& dm, const double* obs, int j_lo, int j_hi, Arena& ws,
                         const double* sup_all, auxmc_filter_result* out, double* ll_out,
                         int* status, cudaStream_t s) {
  if (dm.dx > 32 || dm.dy > 64) return AUXMC_E_DIM;
  return grp_cfg(dm.dx, dm.dy).block
             ? ts_filter_finish<true>(dm, obs, j_lo, j_hi, ws, sup_all, out, ll_out, status, s)
             : ts_filter_finish<false>(dm, obs, j_lo, j_hi, ws, sup_all, out, ll_out, status, s);
}
int tshard_elem_doubles(int dx) { return fe_size_g(dx); }

void pfg_set_fixed_point(int on) { g_pfg_fixed_on = on ? 1 : 0; }
unsigned long long pfg_fixed_point_steps(int reset) {
  unsigned long long v = 0;
  cudaMemcpyFromSymbol(&v, g_fp_steps, sizeof(v));
  if (reset) {
    const unsigned long long z = 0;
    cudaMemcpyToSymbol(g_fp_steps, &z, sizeof(z));
  }
  return v;
}

int dispatch_pf_generic(const DevModel& dm, const double* obs, int B, auxmc_filter_result* out,
                        int* status, Arena& ws, cudaStream_t s) {
  if (dm.dx > 32 || dm.dy > 64) return AUXMC_E_DIM;
  return grp_cfg(dm.dx, dm.dy).block ? run_pfg<true>(dm, obs, B, out, status, ws, s)
                                     : run_pfg<false>(dm, obs, B, out, status, ws, s);
}

}  // namespace auxmc_gpu

namespace auxmc_gpu {
extern int g_bwd_reuse;
}

extern "C" int auxmc_test_pfg_fixed_point(int on) {
  auxmc_gpu::pfg_set_fixed_point(on);
  auxmc_gpu::g_bwd_reuse = on ? 1 : 0;
  return AUXMC_OK;
}

extern "C" long long auxmc_test_pfg_fixed_point_steps(int reset) {
  if (!auxmc_gpu::device_ok()) return -1;
  return (long long)auxmc_gpu::pfg_fixed_point_steps(reset);
}
