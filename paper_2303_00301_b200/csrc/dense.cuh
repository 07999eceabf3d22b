// dense.cuh — small dense FP64 linear algebra for batched state-space work.
//
// Two layers:
//  * Grp-cooperative routines on shared-memory matrices with runtime sizes: a
//    group is either one warp (small d: one (chain, t) item per warp) or a whole
//    CTA (d >= 17: one item per CTA).  Every output element is owned by one lane
//    and accumulated in ascending index order, so results are deterministic and
//    independent of the group size.
//  * Register templates on a compile-time dimension D for the thread-per-item
//    hot loops (pathwise samplers).
//
// Semantics follow the reference's Eigen usage: LLT fails iff a pivot x <= 0
// (NaN pivots pass, gauss.cpp:13-17), the jitter ladder of factor_psd
// (gauss.cpp:20-35), the exact-zero fast path of chol_psd (gauss.cpp:45-49),
// symm(X) = (X + X^T)/2 (lgssm.cpp:14).
#pragma once
#include <cstdint>

namespace auxmc_gpu {

struct Grp {
  int lane, size;
  bool block;
  __device__ __forceinline__ void sync() const {
    if (block) __syncthreads();
    else __syncwarp();
  }
};

__device__ __forceinline__ Grp warp_group() { return Grp{int(threadIdx.x & 31), 32, false}; }
__device__ __forceinline__ Grp block_group() { return Grp{int(threadIdx.x), int(blockDim.x), true}; }

// ---------------------------------------------------------------- copies
__device__ __forceinline__ void g_copy(const Grp& g, int n, const double* __restrict__ src,
                                       double* __restrict__ dst) {
  for (int i = g.lane; i < n; i += g.size) dst[i] = src[i];
}
__device__ __forceinline__ void g_zero(const Grp& g, int n, double* dst) {
  for (int i = g.lane; i < n; i += g.size) dst[i] = 0.0;
}
__device__ __forceinline__ void g_eye(const Grp& g, int n, double* dst) {
  for (int i = g.lane; i < n * n; i += g.size) dst[i] = (i / n == i % n) ? 1.0 : 0.0;
}

// ---------------------------------------------------------------- products
// C (m×n) = A (m×k) B (k×n) [+ D]
__device__ __forceinline__ void g_mm(const Grp& g, int m, int k, int n, const double* A,
                                     const double* B, double* C, const double* D = nullptr) {
  for (int idx = g.lane; idx < m * n; idx += g.size) {
    const int i = idx / n, j = idx % n;
    double s = 0.0;
    for (int l = 0; l < k; ++l) s += A[i * k + l] * B[l * n + j];
    C[idx] = D ? s + D[idx] : s;
  }
}
// C (m×n) = A (m×k) B^T, B (n×k) [+ D]
__device__ __forceinline__ void g_mm_nt(const Grp& g, int m, int k, int n, const double* A,
                                        const double* B, double* C, const double* D = nullptr) {
  for (int idx = g.lane; idx < m * n; idx += g.size) {
    const int i = idx / n, j = idx % n;
    double s = 0.0;
    for (int l = 0; l < k; ++l) s += A[i * k + l] * B[j * k + l];
    C[idx] = D ? s + D[idx] : s;
  }
}
// C (m×n) = A^T B, A (k×m), B (k×n) [+ D]
__device__ __forceinline__ void g_mm_tn(const Grp& g, int m, int k, int n, const double* A,
                                        const double* B, double* C, const double* D = nullptr) {
  for (int idx = g.lane; idx < m * n; idx += g.size) {
    const int i = idx / n, j = idx % n;
    double s = 0.0;
    for (int l = 0; l < k; ++l) s += A[l * m + i] * B[l * n + j];
    C[idx] = D ? s + D[idx] : s;
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
// in-place symm(A) = (A + A^T)/2 ; caller syncs before (A complete) and after
__device__ __forceinline__ void g_symm(const Grp& g, int n, double* A) {
  for (int idx = g.lane; idx < n * n; idx += g.size) {
    const int i = idx / n, j = idx % n;
    if (j > i) {
      const double v = 0.5 * (A[i * n + j] + A[j * n + i]);
      A[i * n + j] = v;
      A[j * n + i] = v;
    }
  }
}
// A := symm(A + B)  (both complete); safe in place for the upper/lower pairs
__device__ __forceinline__ void g_add_symm(const Grp& g, int n, double* A, const double* B) {
  for (int idx = g.lane; idx < n * n; idx += g.size) {
    const int i = idx / n, j = idx % n;
    if (j >= i) {
      const double a = A[i * n + j] + B[i * n + j];
      const double b = A[j * n + i] + B[j * n + i];
      const double v = 0.5 * (a + b);
      A[i * n + j] = v;
      A[j * n + i] = v;
    }
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

// ---------------------------------------------------------------- Cholesky
// Unblocked LLT of the lower triangle of A (n×n) into L; Eigen semantics: fail
// iff a pivot x <= 0.  Returns true on success (uniform across the group).
__device__ __forceinline__ bool g_llt(const Grp& g, int n, const double* A, double* L,
                                      int* flag) {
  for (int i = g.lane; i < n * n; i += g.size) L[i] = 0.0;
  if (g.lane == 0) *flag = 1;
  g.sync();
  for (int k = 0; k < n; ++k) {
    if (g.lane == 0) {
      double x = A[k * n + k];
      for (int j = 0; j < k; ++j) x -= L[k * n + j] * L[k * n + j];
      if (x <= 0.0) *flag = 0;
      else L[k * n + k] = sqrt(x);
    }
    g.sync();
    if (*flag == 0) {
      g.sync();
      return false;
    }
    const double piv = L[k * n + k];
    for (int i = k + 1 + g.lane; i < n; i += g.size) {
      double s = A[i * n + k];
      for (int j = 0; j < k; ++j) s -= L[i * n + j] * L[k * n + j];
      L[i * n + k] = s / piv;
    }
    g.sync();
  }
  return true;
}

// factor_psd (gauss.cpp:26-35): LLT, then + eps*s*I for eps in {1e-10, 1e-8}.
// scratch: n*n doubles.  Returns 0 ok, 2 (AUXMC_E_FACTOR) on failure.
__device__ __forceinline__ int g_factor_psd(const Grp& g, int n, const double* A, double* L,
                                            double* scratch, int* flag, double* red) {
  if (g_llt(g, n, A, L, flag)) return 0;
  // jitter scale (gauss.cpp:20-24)
  if (g.lane == 0) {
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
    for (int i = g.lane; i < n * n; i += g.size)
      scratch[i] = A[i] + ((i / n == i % n) ? (eps[e] * s) * 1.0 : 0.0);
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
__device__ __forceinline__ void g_llt_solve(const Grp& g, int n, const double* L, int r,
                                            double* B) {
  // forward: L Y = B
  for (int i = 0; i < n; ++i) {
    const double lii = L[i * n + i];
    const int rows = n - i - 1;
    for (int idx = g.lane; idx < rows * r; idx += g.size) {
      const int j = i + 1 + idx / r, c = idx % r;
      B[j * r + c] -= L[j * n + i] * (B[i * r + c] / lii);
    }
    g.sync();
  }
  for (int idx = g.lane; idx < n * r; idx += g.size) B[idx] = B[idx] / L[(idx / r) * n + idx / r];
  g.sync();
  // backward: L^T X = Y
  for (int i = n - 1; i >= 0; --i) {
    const double lii = L[i * n + i];
    for (int idx = g.lane; idx < i * r; idx += g.size) {
      const int j = idx / r, c = idx % r;
      B[j * r + c] -= L[i * n + j] * (B[i * r + c] / lii);
    }
    g.sync();
  }
  for (int idx = g.lane; idx < n * r; idx += g.size) B[idx] = B[idx] / L[(idx / r) * n + idx / r];
  g.sync();
}

// In-place forward substitution L z = r (vector), then returns via r.
__device__ __forceinline__ void g_lower_solve_vec(const Grp& g, int n, const double* L, double* r) {
  for (int i = 0; i < n; ++i) {
    const double lii = L[i * n + i];
    for (int j = i + 1 + g.lane; j < n; j += g.size) r[j] -= L[j * n + i] * (r[i] / lii);
    g.sync();
  }
  for (int i = g.lane; i < n; i += g.size) r[i] = r[i] / L[i * n + i];
  g.sync();
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
                                                     double* work, double* red) {
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

// ================================================================ register layer
template <int D>
struct Vec {
  double v[D];
};

template <int D>
__device__ __forceinline__ void r_matvec(const double* __restrict__ A, const double* x, double* y) {
#pragma unroll
  for (int i = 0; i < D; ++i) {
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < D; ++j) s += A[i * D + j] * x[j];
    y[i] = s;
  }
}

// ---- register LLT / solves for fixed small D (thread-per-item) ----
template <int D>
__device__ __forceinline__ bool r_llt(const double* A, double* L) {
#pragma unroll
  for (int i = 0; i < D * D; ++i) L[i] = 0.0;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    double x = A[k * D + k];
#pragma unroll
    for (int j = 0; j < k; ++j) x -= L[k * D + j] * L[k * D + j];
    if (!(x > 0.0) && !(x != x)) return false;  // fail iff x <= 0 (NaN passes)
    x = sqrt(x);
    L[k * D + k] = x;
#pragma unroll
    for (int i = k + 1; i < D; ++i) {
      double s = A[i * D + k];
#pragma unroll
      for (int j = 0; j < k; ++j) s -= L[i * D + j] * L[k * D + j];
      L[i * D + k] = s / x;
    }
  }
  return true;
}

template <int D>
__device__ __forceinline__ int r_factor_psd(const double* A, double* L) {
  if (r_llt<D>(A, L)) return 0;
  double tr = 0.0;
#pragma unroll
  for (int i = 0; i < D; ++i) tr += A[i * D + i];
  double s = tr / static_cast<double>(D);
  if (s <= 0.0) {
    double m = 0.0;
#pragma unroll
    for (int i = 0; i < D * D; ++i) m = fabs(A[i]) > m ? fabs(A[i]) : m;
    s = m;
  }
  double J[D * D];
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const double eps = e == 0 ? 1e-10 : 1e-8;
#pragma unroll
    for (int i = 0; i < D * D; ++i) J[i] = A[i] + ((i / D == i % D) ? (eps * s) * 1.0 : 0.0);
    if (r_llt<D>(J, L)) return 0;
  }
  return 2;
}

template <int D>
__device__ __forceinline__ bool r_all_zero(const double* A) {
  bool z = true;
#pragma unroll
  for (int i = 0; i < D * D; ++i) z = z && (A[i] == 0.0);
  return z;
}

template <int D>
__device__ __forceinline__ int r_chol_psd(const double* A, double* L) {
  if (r_all_zero<D>(A)) {
#pragma unroll
    for (int i = 0; i < D * D; ++i) L[i] = 0.0;
    return 0;
  }
  return r_factor_psd<D>(A, L);
}

// X (D×R) := (L L^T)^{-1} B in place
template <int D, int R>
__device__ __forceinline__ void r_llt_solve(const double* L, double* B) {
#pragma unroll
  for (int c = 0; c < R; ++c) {
#pragma unroll
    for (int i = 0; i < D; ++i) {
      double s = B[i * R + c];
#pragma unroll
      for (int j = 0; j < i; ++j) s -= L[i * D + j] * B[j * R + c];
      B[i * R + c] = s / L[i * D + i];
    }
#pragma unroll
    for (int i = D - 1; i >= 0; --i) {
      double s = B[i * R + c];
#pragma unroll
      for (int j = i + 1; j < D; ++j) s -= L[j * D + i] * B[j * R + c];
      B[i * R + c] = s / L[i * D + i];
    }
  }
}

}  // namespace auxmc_gpu
