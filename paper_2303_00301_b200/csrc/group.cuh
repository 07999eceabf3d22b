// group.cuh — group-cooperative dense FP64 routines on shared-memory matrices
// (included by dense.cuh).  A group is one warp or one CTA (size a multiple of
// 16); lanes are laid out as a 16-wide grid (tx = lane & 15, ty = lane >> 4) so
// 2-D loops carry no integer division and a warp touches 16 consecutive
// columns (conflict-free) of at most two rows (broadcast).  Every output element
// is owned by one lane and accumulated in ascending index order, so results are
// deterministic and independent of the group size.
#pragma once

namespace auxmc_gpu {

struct Grp {
  int lane, size;
  bool block;
  int bar;  // CTA groups: 0 = whole CTA (__syncthreads), > 0 = named barrier of `size` threads
  __device__ __forceinline__ void sync() const {
    if (!block) __syncwarp();
    else if (bar == 0) __syncthreads();
    else asm volatile("bar.sync %0, %1;" ::"r"(bar), "r"(size) : "memory");
  }
  __device__ __forceinline__ int tx() const { return lane & 15; }
  __device__ __forceinline__ int ty() const { return lane >> 4; }
  __device__ __forceinline__ int ny() const { return size >> 4; }
};

__device__ __forceinline__ Grp warp_group() { return Grp{int(threadIdx.x & 31), 32, false, 0}; }
__device__ __forceinline__ Grp block_group() {
  return Grp{int(threadIdx.x), int(blockDim.x), true, 0};
}
// warps [first, first + count) of the CTA as a group synchronized by named barrier `bar`
__device__ __forceinline__ Grp warps_group(int first, int count, int bar) {
  return Grp{int(threadIdx.x) - 32 * first, 32 * count, true, bar};
}

// ---------------------------------------------------------------- copies
__device__ __forceinline__ void g_copy(const Grp& g, int n, const double* __restrict__ src,
                                       double* __restrict__ dst) {
  for (int i = g.lane; i < n; i += g.size) dst[i] = src[i];
}
__device__ __forceinline__ void g_zero(const Grp& g, int n, double* dst) {
  for (int i = g.lane; i < n; i += g.size) dst[i] = 0.0;
}
__device__ __forceinline__ void g_eye(const Grp& g, int n, double* dst) {
  for (int i = g.ty(); i < n; i += g.ny())
    for (int j = g.tx(); j < n; j += 16) dst[i * n + j] = (i == j) ? 1.0 : 0.0;
}

// ---------------------------------------------------------------- FP64 tensor-core products
// For CTA groups on d >= 16 matrices the element algebra is a real dense
// contraction: 8×8 output tiles are accumulated with mma.sync m8n8k4 f64
// (DMMA, one instruction per 256 FMAs instead of 32) — fragments gathered from
// shared memory with bounds guards, so no padding is needed.
// TA/TB: operand transposed in memory (A^T B, A B^T forms).
template <bool TA, bool TB>
__device__ __forceinline__ void g_dmma(const Grp& g, int m, int k, int n, const double* A, int lda,
                                       const double* B, int ldb, double* C, int ldc, bool sub,
                                       bool lower, const double* Dadd = nullptr);
template <bool TA, bool TB>
__device__ __forceinline__ void g_mm_dmma(const Grp& g, int m, int k, int n, const double* A,
                                          const double* B, double* C, const double* D) {
  g_dmma<TA, TB>(g, m, k, n, A, TA ? m : k, B, TB ? k : n, C, n, false, false, D);
}

// CTA groups and single warps (mma.sync is warp-wide) on operands of at least
// 16×16: below that the scalar loops have less latency than DMMA tiles.
__device__ __forceinline__ bool use_dmma(const Grp& g, int m, int k, int n) {
  return (g.block || g.size == 32) && m >= 16 && n >= 16 && k >= 8;
}

// ---------------------------------------------------------------- products
// Each lane owns outputs (i, j), (i + ny, j): two independent FMA chains.
// C (m×n) = A (m×k) B (k×n) [+ D]
__device__ __forceinline__ void g_mm(const Grp& g, int m, int k, int n, const double* A,
                                     const double* B, double* C, const double* D = nullptr) {
  if (use_dmma(g, m, k, n)) {
    g_mm_dmma<false, false>(g, m, k, n, A, B, C, D);
    return;
  }
  const int ny = g.ny();
  for (int i = g.ty(); i < m; i += 2 * ny) {
    const int i2 = i + ny;
    const bool two = i2 < m;
    for (int j = g.tx(); j < n; j += 16) {
      double s = 0.0, s2 = 0.0;
      for (int l = 0; l < k; ++l) {
        const double b = B[l * n + j];
        s += A[i * k + l] * b;
        if (two) s2 += A[i2 * k + l] * b;
      }
      C[i * n + j] = D ? s + D[i * n + j] : s;
      if (two) C[i2 * n + j] = D ? s2 + D[i2 * n + j] : s2;
    }
  }
}
// C (m×n) = A (m×k) B^T, B (n×k) [+ D]
__device__ __forceinline__ void g_mm_nt(const Grp& g, int m, int k, int n, const double* A,
                                        const double* B, double* C, const double* D = nullptr) {
  if (use_dmma(g, m, k, n)) {
    g_mm_dmma<false, true>(g, m, k, n, A, B, C, D);
    return;
  }
  const int ny = g.ny();
  for (int i = g.ty(); i < m; i += 2 * ny) {
    const int i2 = i + ny;
    const bool two = i2 < m;
    for (int j = g.tx(); j < n; j += 16) {
      double s = 0.0, s2 = 0.0;
      for (int l = 0; l < k; ++l) {
        const double b = B[j * k + l];
        s += A[i * k + l] * b;
        if (two) s2 += A[i2 * k + l] * b;
      }
      C[i * n + j] = D ? s + D[i * n + j] : s;
      if (two) C[i2 * n + j] = D ? s2 + D[i2 * n + j] : s2;
    }
  }
}
// C (m×n) = A^T B, A (k×m), B (k×n) [+ D]
__device__ __forceinline__ void g_mm_tn(const Grp& g, int m, int k, int n, const double* A,
                                        const double* B, double* C, const double* D = nullptr) {
  if (use_dmma(g, m, k, n)) {
    g_mm_dmma<true, false>(g, m, k, n, A, B, C, D);
    return;
  }
  const int ny = g.ny();
  for (int i = g.ty(); i < m; i += 2 * ny) {
    const int i2 = i + ny;
    const bool two = i2 < m;
    for (int j = g.tx(); j < n; j += 16) {
      double s = 0.0, s2 = 0.0;
      for (int l = 0; l < k; ++l) {
        const double b = B[l * n + j];
        s += A[l * m + i] * b;
        if (two) s2 += A[l * m + i2] * b;
      }
      C[i * n + j] = D ? s + D[i * n + j] : s;
      if (two) C[i2 * n + j] = D ? s2 + D[i2 * n + j] : s2;
    }
  }
}
// y (m) = A (m×n) x [+ add]
__device__ __forceinline__ void g_mv(const Grp& g, int m, int n, const double* A, const double* x,
                                     double* y, const double* add = nullptr) {
  for (int i = g.lane; i < m; i += g.size) {
    double s = 0.0;
    for (int j = 0; j < n; ++j) s += A[i * n + j] * x[j];
    y[i] = add ? s + add[i] : s;
  }
}
// y (n) = A^T x, A (m×n)
__device__ __forceinline__ void g_mtv(const Grp& g, int m, int n, const double* A,
                                      const double* x, double* y) {
  for (int j = g.lane; j < n; j += g.size) {
    double s = 0.0;
    for (int i = 0; i < m; ++i) s += A[i * n + j] * x[i];
    y[j] = s;
  }
}
// Quad dot products: lanes 4i..4i+3 of a group own row i and sum interleaved
// terms (j ≡ q mod 4), combined as (s0+s1)+(s2+s3) by xor shuffles — four short
// FMA chains instead of one long one, fixed order.  The row loop is uniform
// over the group so every shuffle is full-warp.
__device__ __forceinline__ double quad_sum(double s) {
  s += __shfl_xor_sync(0xffffffffu, s, 1);
  s += __shfl_xor_sync(0xffffffffu, s, 2);
  return s;
}
// y[i] = Σ_j A(i,j) x[j] (+ add[i]) ; A(i,j) = TA ? A[j*lda+i] : A[i*lda+j]
template <bool TA>
__device__ __forceinline__ void g_mv4(const Grp& g, int m, int n, const double* A, int lda,
                                      const double* x, double* y, const double* add = nullptr) {
  const int q = g.lane & 3, rows = g.size >> 2;
  for (int i0 = 0; i0 < m; i0 += rows) {
    const int i = i0 + (g.lane >> 2);
    double s = 0.0;
    if (i < m)
      for (int j = q; j < n; j += 4) s += (TA ? A[j * lda + i] : A[i * lda + j]) * x[j];
    s = quad_sum(s);
    if (i < m && q == 0) y[i] = add ? s + add[i] : s;
  }
}

// in-place symm(A) = (A + A^T)/2 ; caller syncs before (A complete) and after
__device__ __forceinline__ void g_symm(const Grp& g, int n, double* A) {
  for (int i = g.ty(); i < n; i += g.ny())
    for (int j = i + 1 + g.tx(); j < n; j += 16) {
      const double v = 0.5 * (A[i * n + j] + A[j * n + i]);
      A[i * n + j] = v;
      A[j * n + i] = v;
    }
}
// A := symm(A + B)  (both complete)
__device__ __forceinline__ void g_add_symm(const Grp& g, int n, double* A, const double* B) {
  for (int i = g.ty(); i < n; i += g.ny())
    for (int j = i + g.tx(); j < n; j += 16) {
      const double a = A[i * n + j] + B[i * n + j];
      const double b = A[j * n + i] + B[j * n + i];
      const double v = 0.5 * (a + b);
      A[i * n + j] = v;
      A[j * n + i] = v;
    }
}

// group-wide boolean "all entries exactly zero"; flag in shared memory
__device__ __forceinline__ bool g_all_zero(const Grp& g, int n, const double* A, int* flag) {
  if (g.lane == 0) *flag = 1;
  g.sync();
  for (int i = g.lane; i < n; i += g.size)
    if (A[i] != 0.0) *flag = 0;
  g.sync();
  const bool r = *flag != 0;
  g.sync();
  return r;
}

// group-wide boolean "A and B hold the same bits" (n doubles); flag in shared memory
__device__ __forceinline__ bool g_all_same(const Grp& g, int n, const double* A, const double* B,
                                           int* flag) {
  if (g.lane == 0) *flag = 1;
  g.sync();
  for (int i = g.lane; i < n; i += g.size)
    if (__double_as_longlong(A[i]) != __double_as_longlong(B[i])) *flag = 0;
  g.sync();
  const bool r = *flag != 0;
  g.sync();
  return r;
}

// this thread's share of "every row r < nrows of rows (row length n) has the bits of
// ref": threads tid, tid + nth, ... of each row, eight rows' loads in flight per
// round (a streaming compare: the rows are read once, at memory bandwidth)
__device__ __forceinline__ bool rows_match_part(const double* __restrict__ rows,
                                                const double* __restrict__ ref, int nrows, int n,
                                                int tid, int nth) {
  const long long* a = reinterpret_cast<const long long*>(rows);
  const long long* z = reinterpret_cast<const long long*>(ref);
  bool ok = true;
  for (int e = tid; e < n; e += nth) {
    const long long z0 = z[e];
    int r = 0;
    for (; r + 8 <= nrows; r += 8) {
      long long v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = a[(size_t)(r + k) * n + e];
#pragma unroll
      for (int k = 0; k < 8; ++k) ok &= v[k] == z0;
    }
    for (; r < nrows; ++r) ok &= a[(size_t)r * n + e] == z0;
  }
  return ok;
}

// ---------------------------------------------------------------- blocked (CTA, n >= 16)
// Blocked factor/solves with 8-wide panels.  The diagonal 8×8 blocks are
// factored and inverted by one warp; every other step (panel solve, trailing
// SYRK, triangular solves) is an 8×8-tile DMMA product, so the serial depth is
// O(n/8) group syncs and the O(n^3) work runs on the FP64 tensor cores.  The
// inverted diagonal blocks (dinv: ceil(n/8) row-major 8×8 blocks, 64*ceil(n/8)
// doubles) are kept for the triangular solves that follow a factorization.
constexpr int kNB = 8;

__host__ __device__ constexpr int dinv_doubles(int n) { return 64 * ((n + 7) / 8); }

// C (m×n, ldc) = op(A) op(B) [+ Dadd]  or  C -= op(A) op(B)  (sub);
// A(i,l) = TA ? A[l*lda+i] : A[i*lda+l], B(l,j) = TB ? B[j*ldb+l] : B[l*ldb+j];
// lower: only j <= i is written (tiles above the diagonal skipped).  For sub
// the accumulator starts at C and the A fragment is negated (one fused chain
// C - Σ a b).  Each warp owns a pair of horizontally adjacent 8×8 tiles (two
// independent DMMA chains sharing the A fragment).  A tile loads its whole
// k-range before it stores, so C may alias the rows of A when n <= 8, or the
// columns of B when m <= 8.
template <bool TA, bool TB>
__device__ __forceinline__ void g_dmma(const Grp& g, int m, int k, int n, const double* A, int lda,
                                       const double* B, int ldb, double* C, int ldc, bool sub,
                                       bool lower, const double* Dadd) {
  const int warp = g.lane >> 5, lane = g.lane & 31, nw = g.size >> 5;
  const int gi = lane >> 2, ti = lane & 3;
  const int mt = (m + 7) >> 3, nt = (n + 7) >> 3, kt = (k + 3) >> 2;
  const int np = (nt + 1) >> 1;
  const float rnp = 1.0f / (float)np;
  for (int w = warp; w < mt * np; w += nw) {
    const int It = (int)(((float)w + 0.5f) * rnp);  // exact for these small ranges
    const int Jt = (w - It * np) * 2;
    if (lower && Jt > It) continue;
    const bool two = Jt + 1 < nt && !(lower && Jt + 1 > It);
    const int r = It * 8 + gi;
    const int c0c = Jt * 8 + 2 * ti, c1c = c0c + 8;
    double c00 = 0.0, c01 = 0.0, c10 = 0.0, c11 = 0.0;
    if (sub && r < m) {
      if (c0c < n) c00 = C[r * ldc + c0c];
      if (c0c + 1 < n) c01 = C[r * ldc + c0c + 1];
      if (two && c1c < n) c10 = C[r * ldc + c1c];
      if (two && c1c + 1 < n) c11 = C[r * ldc + c1c + 1];
    }
    const int b0 = Jt * 8 + gi, b1 = b0 + 8;
    const double sg = sub ? -1.0 : 1.0;
    // interior tiles (the common case): unguarded fragment loads, pointer walks
    const bool inner = (k & 3) == 0 && It * 8 + 8 <= m && Jt * 8 + (two ? 16 : 8) <= n;
    if (inner) {
      const double* pa = TA ? A + ti * lda + r : A + r * lda + ti;
      const double* p0 = TB ? B + b0 * ldb + ti : B + ti * ldb + b0;
      const double* p1 = TB ? B + b1 * ldb + ti : B + ti * ldb + b1;
      const int sa = TA ? 4 * lda : 4, sb = TB ? 4 : 4 * ldb;
#pragma unroll 2
      for (int K = 0; K < kt; ++K) {
        const double a = sg * pa[0];
        const double x0 = p0[0];
        asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
            : "+d"(c00), "+d"(c01)
            : "d"(a), "d"(x0));
        if (two) {
          const double x1 = p1[0];
          asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
              : "+d"(c10), "+d"(c11)
              : "d"(a), "d"(x1));
        }
        pa += sa;
        p0 += sb;
        p1 += sb;
      }
    } else if ((k & 3) == 0) {
      // edge tiles with a whole k range: the interior pointer walks, with the
      // out-of-range rows / columns predicated to zero (the guarded loop's values)
      const bool ra = r < m, rb0 = b0 < n, rb1 = two && b1 < n;
      const double* pa = TA ? A + ti * lda + r : A + r * lda + ti;
      const double* p0 = TB ? B + b0 * ldb + ti : B + ti * ldb + b0;
      const double* p1 = TB ? B + b1 * ldb + ti : B + ti * ldb + b1;
      const int sa = TA ? 4 * lda : 4, sb = TB ? 4 : 4 * ldb;
#pragma unroll 2
      for (int K = 0; K < kt; ++K) {
        double a = ra ? pa[0] : 0.0;
        const double x0 = rb0 ? p0[0] : 0.0;
        a = sg * a;
        asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
            : "+d"(c00), "+d"(c01)
            : "d"(a), "d"(x0));
        if (two) {
          const double x1 = rb1 ? p1[0] : 0.0;
          asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
              : "+d"(c10), "+d"(c11)
              : "d"(a), "d"(x1));
        }
        pa += sa;
        p0 += sb;
        p1 += sb;
      }
    } else {
      for (int K = 0; K < kt; ++K) {
        const int kk = K * 4 + ti;
        double a = 0.0, x0 = 0.0, x1 = 0.0;
        if (r < m && kk < k) a = TA ? A[kk * lda + r] : A[r * lda + kk];
        if (kk < k) {
          if (b0 < n) x0 = TB ? B[b0 * ldb + kk] : B[kk * ldb + b0];
          if (two && b1 < n) x1 = TB ? B[b1 * ldb + kk] : B[kk * ldb + b1];
        }
        a = sg * a;
        asm volatile(
            "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
            : "+d"(c00), "+d"(c01)
            : "d"(a), "d"(x0));
        if (two)
          asm volatile(
              "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
              : "+d"(c10), "+d"(c11)
              : "d"(a), "d"(x1));
      }
    }
    if (r < m) {
      if (c0c < n && (!lower || c0c <= r))
        C[r * ldc + c0c] = Dadd ? c00 + Dadd[r * ldc + c0c] : c00;
      if (c0c + 1 < n && (!lower || c0c + 1 <= r))
        C[r * ldc + c0c + 1] = Dadd ? c01 + Dadd[r * ldc + c0c + 1] : c01;
      if (two && c1c < n && (!lower || c1c <= r))
        C[r * ldc + c1c] = Dadd ? c10 + Dadd[r * ldc + c1c] : c10;
      if (two && c1c + 1 < n && (!lower || c1c + 1 <= r))
        C[r * ldc + c1c + 1] = Dadd ? c11 + Dadd[r * ldc + c1c + 1] : c11;
    }
  }
}

// One warp: factor the nb×nb diagonal block D (row stride n, lower triangle holds
// the updated A) in place and write its inverse to Di (8×8, zero padded).
// Rows live in registers of lanes 0..7 (column broadcasts by shuffle), so the
// serial chain per column is one rsqrt and two shuffles; columns are scaled by
// the reciprocal pivot.  Returns false (warp-uniformly) on a
// pivot <= 0 (NaN passes, as in Eigen).
__device__ __forceinline__ bool w_factor_diag(int lane, int n, int nb, double* D, double* Di) {
  const int i = lane & 7;
  double a[kNB], inv[kNB];
#pragma unroll
  for (int k = 0; k < kNB; ++k) {
    a[k] = (i < nb && k <= i) ? D[i * n + k] : (k == i ? 1.0 : 0.0);
    inv[k] = 0.0;
  }
  bool ok = true;
#pragma unroll
  for (int j = 0; j < kNB; ++j) {
    if (j < nb) {
      // the column's unscaled entries travel while the pivot's rsqrt runs; the
      // receiving lane forms l_kj = a_kj * r itself (the same product lane k forms)
      const double d = __shfl_sync(0xffffffffu, a[j], j);
      double akj[kNB];
#pragma unroll
      for (int k = j + 1; k < kNB; ++k) akj[k] = __shfl_sync(0xffffffffu, a[j], k);
      if (d <= 0.0) {
        ok = false;
        break;
      }
      const double r = rsqrt(d);  // 1/sqrt(d) to ~1 ulp; the pivot is d * r
      const double piv = d * r;
      inv[j] = r;
      if (i > j) a[j] = a[j] * r;
      else if (i == j) a[j] = piv;
#pragma unroll
      for (int k = j + 1; k < kNB; ++k) {
        const double lkj = akj[k] * r;
        if (k <= i && i > j) a[k] -= a[j] * lkj;
      }
    }
  }
  if (!ok) return false;
  // rows of L by shuffle (lane r holds row r) before any store: the forward
  // substitution below runs from registers, no shared-memory round trip
  double Lr[kNB][kNB];
#pragma unroll
  for (int r = 1; r < kNB; ++r)
#pragma unroll
    for (int l = 0; l < r; ++l) Lr[r][l] = __shfl_sync(0xffffffffu, a[l], r);
  if (lane < nb) {
#pragma unroll
    for (int k = 0; k < kNB; ++k)
      if (k <= i) D[i * n + k] = a[k];
  }
  if (lane < kNB) {  // column `lane` of D^{-1} by forward substitution
    const int j = lane;
    double x[kNB];
#pragma unroll
    for (int r = 0; r < kNB; ++r) {
      double v = 0.0;
      if (j < nb && r < nb && r >= j) {
        if (r == j) {
          v = inv[r];
        } else {
          double s = 0.0;
#pragma unroll
          for (int l = 0; l < r; ++l)
            if (l >= j) s += Lr[r][l] * x[l];
          v = -s * inv[r];
        }
      }
      x[r] = v;
      Di[r * kNB + j] = v;
    }
  }
  __syncwarp();
  return true;
}

// Right-looking blocked LLT of L (lower triangle already holds A, upper zero).
__device__ __forceinline__ bool g_llt_blocked(const Grp& g, int n, double* L, int* flag,
                                              double* dinv) {
  if (g.lane == 0) *flag = 1;
  for (int kb = 0; kb < n; kb += kNB) {
    const int nb = n - kb < kNB ? n - kb : kNB;
    double* Di = dinv + (kb / kNB) * kNB * kNB;
    if (g.lane < 32) {
      const bool ok = w_factor_diag(g.lane, n, nb, L + kb * n + kb, Di);
      if (!ok && g.lane == 0) *flag = 0;
    }
    g.sync();
    if (*flag == 0) {
      g.sync();
      return false;
    }
    const int rest = n - kb - nb;
    if (rest <= 0) break;
    double* P = L + (kb + nb) * n + kb;
    g_dmma<false, true>(g, rest, nb, nb, P, n, Di, kNB, P, n, false, false);  // P D^{-T}
    g.sync();
    g_dmma<false, true>(g, rest, nb, rest, P, n, P, n, P + nb, n, true, true);  // L22 -= P P^T
    g.sync();
  }
  return true;
}

// In-place L Y = B (B n×r, row stride ldb) with the inverted diagonal blocks.
__device__ __forceinline__ void g_trsm_lower_blocked(const Grp& g, int n, const double* L,
                                                     const double* dinv, int r, double* B,
                                                     int ldb) {
  for (int kb = 0; kb < n; kb += kNB) {
    const int nb = n - kb < kNB ? n - kb : kNB;
    double* Bk = B + kb * ldb;
    g_dmma<false, false>(g, nb, nb, r, dinv + (kb / kNB) * kNB * kNB, kNB, Bk, ldb, Bk, ldb, false,
                         false);
    g.sync();
    const int rest = n - kb - nb;
    if (rest <= 0) break;
    g_dmma<false, false>(g, rest, nb, r, L + (kb + nb) * n + kb, n, Bk, ldb, Bk + nb * ldb, ldb,
                         true, false);
    g.sync();
  }
}

// In-place L^T X = Y.
__device__ __forceinline__ void g_trsm_lower_t_blocked(const Grp& g, int n, const double* L,
                                                       const double* dinv, int r, double* B,
                                                       int ldb) {
  const int nblk = (n + kNB - 1) / kNB;
  for (int bi = nblk - 1; bi >= 0; --bi) {
    const int kb = bi * kNB;
    const int nb = n - kb < kNB ? n - kb : kNB;
    double* Bk = B + kb * ldb;
    g_dmma<true, false>(g, nb, nb, r, dinv + bi * kNB * kNB, kNB, Bk, ldb, Bk, ldb, false, false);
    g.sync();
    if (kb == 0) break;
    g_dmma<true, false>(g, kb, nb, r, L + kb * n, n, Bk, ldb, B, ldb, true, false);
    g.sync();
  }
}

// One warp: in-place L z = r (vector) with the inverted diagonal blocks.
__device__ __forceinline__ void w_lower_solve_vec(int lane, int n, const double* L,
                                                  const double* dinv, double* r) {
  for (int kb = 0; kb < n; kb += kNB) {
    const int nb = n - kb < kNB ? n - kb : kNB;
    const double* Di = dinv + (kb / kNB) * kNB * kNB;
    double z = 0.0;
    if (lane < nb)
      for (int l = 0; l <= lane; ++l) z += Di[lane * kNB + l] * r[kb + l];
    __syncwarp();
    if (lane < nb) r[kb + lane] = z;
    __syncwarp();
    for (int i = kb + nb + lane; i < n; i += 32) {
      double s = r[i];
      for (int l = 0; l < nb; ++l) s -= L[i * n + kb + l] * r[kb + l];
      r[i] = s;
    }
    __syncwarp();
  }
}

// fixed-order warp sum (lane-strided partials, then an xor tree): deterministic
__device__ __forceinline__ double w_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

constexpr double kLog2PiB = 1.8378770664093454835606594728112;

// One warp: log N(x; mean, L L^T) with the inverted diagonal blocks; work: n doubles.
__device__ __forceinline__ double w_log_pdf_factored(int lane, int n, const double* x,
                                                     const double* mean, const double* L,
                                                     const double* dinv, double* work) {
  for (int i = lane; i < n; i += 32) work[i] = x[i] - mean[i];
  __syncwarp();
  w_lower_solve_vec(lane, n, L, dinv, work);
  double sq = 0.0, ld = 0.0;
  for (int i = lane; i < n; i += 32) {
    sq += work[i] * work[i];
    ld += log(L[i * n + i]);
  }
  sq = w_sum(sq);
  ld = w_sum(ld);
  return -0.5 * (n * kLog2PiB + sq) - ld;
}

__device__ __forceinline__ bool use_blocked(const Grp& g, int n) { return g.block && n >= 16; }

// ---------------------------------------------------------------- Cholesky
// LLT of the lower triangle of A (n×n) into L; Eigen semantics: fail iff a
// pivot x <= 0 (NaN passes).  Right-looking: the trailing update of column k is
// spread over the group, so the serial depth is O(n) syncs.
// One warp, n <= NM: lane i holds row i of the factor in registers; column k's
// pivot and the L_jk of the trailing update travel by shuffles.  Every lane
// performs exactly the divisions and fused updates of g_llt's shared-memory
// loop below in the same order, so the factor is bit-identical — without the
// two warp barriers and shared round trips per column.  A may alias L.
template <int NM>
__device__ __forceinline__ bool w_llt_reg(int lane, int n, const double* A, double* L) {
  double a[NM];
#pragma unroll
  for (int j = 0; j < NM; ++j) a[j] = (lane < n && j < n && j <= lane) ? A[lane * n + j] : 0.0;
  __syncwarp();
  bool ok = true;
#pragma unroll
  for (int k = 0; k < NM; ++k) {
    if (k >= n) break;
    const double x = __shfl_sync(0xffffffffu, a[k], k);
    if (x <= 0.0) {  // uniform: every lane holds the same pivot
      ok = false;
      break;
    }
    const double piv = sqrt(x);
    if (lane > k && lane < n) a[k] = a[k] / piv;
#pragma unroll
    for (int j = k + 1; j < NM; ++j) {
      if (j >= n) break;
      const double ljk = __shfl_sync(0xffffffffu, a[k], j);
      if (lane >= j && lane < n) a[j] -= a[k] * ljk;
    }
    if (lane == k) a[k] = piv;
  }
  if (ok && lane < n) {
#pragma unroll
    for (int j = 0; j < NM; ++j)
      if (j < n) L[lane * n + j] = j <= lane ? a[j] : 0.0;
  }
  __syncwarp();
  return ok;
}

__device__ __forceinline__ bool g_llt(const Grp& g, int n, const double* A, double* L,
                                      int* flag) {
  if (!g.block && n <= 16) return w_llt_reg<16>(g.lane, n, A, L);
  for (int i = g.ty(); i < n; i += g.ny())
    for (int j = g.tx(); j < n; j += 16) L[i * n + j] = j <= i ? A[i * n + j] : 0.0;
  (void)flag;
  g.sync();
  for (int k = 0; k < n; ++k) {
    // every lane reads the same (final) pivot, so the failure test is uniform
    const double x = L[k * n + k];
    if (x <= 0.0) {
      g.sync();
      return false;
    }
    const double piv = sqrt(x);
    for (int i = k + 1 + g.lane; i < n; i += g.size) L[i * n + k] = L[i * n + k] / piv;
    g.sync();
    if (g.lane == 0) L[k * n + k] = piv;  // not read by the trailing update
    for (int i = k + 1 + g.ty(); i < n; i += g.ny()) {
      const double lik = L[i * n + k];
      for (int j = k + 1 + g.tx(); j <= i; j += 16) L[i * n + j] -= lik * L[j * n + k];
    }
    g.sync();
  }
  return true;
}

// factor_psd (gauss.cpp:26-35): LLT, then + eps*s*I for eps in {1e-10, 1e-8}.
// scratch: n*n doubles.  Returns 0 ok, 2 (AUXMC_E_FACTOR) on failure.
// Blocked (CTA, n >= 16): the jittered matrix is built in L directly and
// scratch (>= dinv_doubles(n)) receives the inverted diagonal blocks, which
// g_llt_solve / g_log_pdf_factored take as `dinv`.
__device__ __forceinline__ int g_factor_psd(const Grp& g, int n, const double* A, double* L,
                                            double* scratch, int* flag, double* red) {
  const bool blk = use_blocked(g, n);
  if (blk) {
    for (int i = g.ty(); i < n; i += g.ny())
      for (int j = g.tx(); j < n; j += 16) L[i * n + j] = j <= i ? A[i * n + j] : 0.0;
    g.sync();
    if (g_llt_blocked(g, n, L, flag, scratch)) return 0;
  } else if (g_llt(g, n, A, L, flag)) {
    return 0;
  }
  if (g.lane == 0) {  // jitter scale (gauss.cpp:20-24)
    double tr = 0.0;
    for (int i = 0; i < n; ++i) tr += A[i * n + i];
    double s = tr / static_cast<double>(n);
    if (s <= 0.0) {
      double m = 0.0;
      for (int i = 0; i < n * n; ++i) m = fabs(A[i]) > m ? fabs(A[i]) : m;
      s = m;
    }
    *red = s;
  }
  g.sync();
  const double s = *red;
  const double eps[2] = {1e-10, 1e-8};
  for (int e = 0; e < 2; ++e) {
    if (blk) {
      for (int i = g.ty(); i < n; i += g.ny())
        for (int j = g.tx(); j < n; j += 16)
          L[i * n + j] = j <= i ? A[i * n + j] + (i == j ? (eps[e] * s) * 1.0 : 0.0) : 0.0;
      g.sync();
      if (g_llt_blocked(g, n, L, flag, scratch)) return 0;
      continue;
    }
    for (int i = g.ty(); i < n; i += g.ny())
      for (int j = g.tx(); j < n; j += 16)
        scratch[i * n + j] = A[i * n + j] + (i == j ? (eps[e] * s) * 1.0 : 0.0);
    g.sync();
    if (g_llt(g, n, scratch, L, flag)) return 0;
  }
  return 2;
}

// chol_psd (gauss.cpp:45-49): exactly-zero matrix factors to zero.
__device__ __forceinline__ int g_chol_psd(const Grp& g, int n, const double* A, double* L,
                                          double* scratch, int* flag, double* red) {
  if (g_all_zero(g, n * n, A, flag)) {
    for (int i = g.lane; i < n * n; i += g.size) L[i] = 0.0;
    g.sync();
    return 0;
  }
  return g_factor_psd(g, n, A, L, scratch, flag, red);
}

// In-place solve L L^T X = B for X (B n×r), L lower.  One group sync per row.
// Row i of the running right-hand side holds the solved x_i once step i starts:
// the lane that applies the last update to row i+1 also divides it by L_{i+1,i+1},
// so each x is divided exactly once (x_i = (b_i - Σ_j L_ij x_j) / L_ii in
// ascending j, the reference's order) and there is one group sync per row.
// dinv: the inverted diagonal blocks from a blocked g_factor_psd (CTA, n >= 16).
__device__ __forceinline__ void g_llt_solve(const Grp& g, int n, const double* L, int r,
                                            double* B, const double* dinv = nullptr) {
  if (dinv && use_blocked(g, n)) {
    g_trsm_lower_blocked(g, n, L, dinv, r, B, r);
    g_trsm_lower_t_blocked(g, n, L, dinv, r, B, r);
    return;
  }
  if (!g.block && r <= 32) {
    // one warp: lane c owns column c (conflict-free rows, broadcast L reads) and
    // runs both substitutions without synchronization; same operation order as
    // the row-synchronous form below (ascending / descending update sequences)
    const int c = g.lane;
    if (c < r) {
      for (int i = 0; i < n; ++i) {
        double v = B[i * r + c];
        for (int j = 0; j < i; ++j) v -= L[i * n + j] * B[j * r + c];
        B[i * r + c] = v / L[i * n + i];
      }
      for (int i = n - 1; i >= 0; --i) {
        double v = B[i * r + c];
        for (int j = n - 1; j > i; --j) v -= L[j * n + i] * B[j * r + c];
        B[i * r + c] = v / L[i * n + i];
      }
    }
    __syncwarp();
    return;
  }
  const int ny = g.ny();
  for (int c = g.lane; c < r; c += g.size) B[c] = B[c] / L[0];
  g.sync();
  for (int i = 0; i < n; ++i) {  // forward: L Y = B
    for (int j = i + 1 + g.ty(); j < n; j += ny) {
      const double lji = L[j * n + i];
      if (j == i + 1) {  // last update of row j: finish it
        const double ljj = L[j * n + j];
        for (int c = g.tx(); c < r; c += 16) B[j * r + c] = (B[j * r + c] - lji * B[i * r + c]) / ljj;
      } else {
        for (int c = g.tx(); c < r; c += 16) B[j * r + c] -= lji * B[i * r + c];
      }
    }
    g.sync();
  }
  for (int c = g.lane; c < r; c += g.size)
    B[(n - 1) * r + c] = B[(n - 1) * r + c] / L[(n - 1) * n + (n - 1)];
  g.sync();
  for (int i = n - 1; i >= 0; --i) {  // backward: L^T X = Y
    for (int j = g.ty(); j < i; j += ny) {
      const double lij = L[i * n + j];
      if (j == i - 1) {
        const double ljj = L[j * n + j];
        for (int c = g.tx(); c < r; c += 16) B[j * r + c] = (B[j * r + c] - lij * B[i * r + c]) / ljj;
      } else {
        for (int c = g.tx(); c < r; c += 16) B[j * r + c] -= lij * B[i * r + c];
      }
    }
    g.sync();
  }
}

// In-place forward substitution L z = r (vector), same scheme.
__device__ __forceinline__ void g_lower_solve_vec(const Grp& g, int n, const double* L, double* r) {
  if (g.lane == 0) r[0] = r[0] / L[0];
  g.sync();
  for (int i = 0; i < n; ++i) {
    for (int j = i + 1 + g.lane; j < n; j += g.size) {
      if (j == i + 1) r[j] = (r[j] - L[j * n + i] * r[i]) / L[j * n + j];
      else r[j] -= L[j * n + i] * r[i];
    }
    g.sync();
  }
}

// group sum of v[0..n) into *out (lane 0 sequential for determinism)
__device__ __forceinline__ double g_sum_seq(const Grp& g, int n, const double* v, double* out) {
  if (g.lane == 0) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += v[i];
    *out = s;
  }
  g.sync();
  const double r = *out;
  g.sync();
  return r;
}

constexpr double kLog2Pi = 1.8378770664093454835606594728112;

// log N(x; mean, cov) (gauss.cpp:51-57) given the LLT factor L of symm(cov).
// work: n doubles.  Returns value on all lanes.
__device__ __forceinline__ double g_log_pdf_factored(const Grp& g, int n, const double* x,
                                                     const double* mean, const double* L,
                                                     double* work, double* red,
                                                     const double* dinv = nullptr) {
  if (dinv && use_blocked(g, n)) {
    if (g.lane < 32) {
      const double v = w_log_pdf_factored(g.lane, n, x, mean, L, dinv, work);
      if (g.lane == 0) *red = v;
    }
    g.sync();
    const double v = *red;
    g.sync();
    return v;
  }
  if (!g.block && n <= 32) {
    // one warp: lane j owns r_j; forward substitution by shuffles with the same
    // operations as g_lower_solve_vec, and the n logs of the diagonal in
    // parallel, summed in index order (gauss.cpp:51-57) on every lane
    const int j = g.lane;
    double r = j < n ? x[j] - mean[j] : 0.0;
    if (j == 0) r = r / L[0];
    for (int i = 0; i < n; ++i) {
      const double ri = __shfl_sync(0xffffffffu, r, i);
      if (j == i + 1) r = (r - L[j * n + i] * ri) / L[j * n + j];
      else if (j > i + 1 && j < n) r -= L[j * n + i] * ri;
    }
    const double lg = j < n ? log(L[j * n + j]) : 0.0;
    if (j < n) work[j] = r;
    double sq = 0.0, ld = 0.0;
    for (int i = 0; i < n; ++i) {
      const double wi = __shfl_sync(0xffffffffu, r, i);
      sq += wi * wi;
    }
    for (int i = 0; i < n; ++i) ld += __shfl_sync(0xffffffffu, lg, i);
    __syncwarp();
    return -0.5 * (n * kLog2Pi + sq) - ld;
  }
  for (int i = g.lane; i < n; i += g.size) work[i] = x[i] - mean[i];
  g.sync();
  g_lower_solve_vec(g, n, L, work);
  if (g.lane == 0) {
    double sq = 0.0, ld = 0.0;
    for (int i = 0; i < n; ++i) sq += work[i] * work[i];
    for (int i = 0; i < n; ++i) ld += log(L[i * n + i]);
    *red = -0.5 * (n * kLog2Pi + sq) - ld;
  }
  g.sync();
  const double v = *red;
  g.sync();
  return v;
}

}  // namespace auxmc_gpu
