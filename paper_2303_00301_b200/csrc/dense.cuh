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

#include "group.cuh"

namespace auxmc_gpu {

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
