// pfilter.cu — pit::parallel_filter (pit.cpp:117-188) on B200.
//
// Filtering elements (A, b, C, eta, J) per step (pit.cpp:126-152) are combined
// with the associative operator of pit.cpp:36-51 by a fixed-tree blocked scan:
//   S1  per (sequence, block of LB steps): sequential reduction -> aggregate
//   S2  per sequence: exclusive scan of the block aggregates -> block carries
//   S3  per (sequence, block): carry ∘ e_0 ∘ e_1 ... -> inclusive elements
// then the recovery pass (pit.cpp:167-186) rebuilds predictive moments from the
// filtered ones and sums the log-likelihood terms in time order.  About 2T
// combines instead of Sklansky's (T/2) log T, with span T/LB + 2 LB; the tree
// depends only on (T, LB), so results are run-to-run deterministic.
// Thread-level register algebra for d <= 8, observation rows <= 8.
#include "common.cuh"
#include "dense.cuh"

namespace auxmc_gpu {

constexpr int kMaxDY = 8;

template <int D>
struct FElem {
  double A[D * D], b[D], C[D * D], eta[D], J[D * D];
};

template <int D>
__device__ __forceinline__ void fe_load(const double* p, FElem<D>& e) {
#pragma unroll
  for (int i = 0; i < D * D; ++i) e.A[i] = p[i];
#pragma unroll
  for (int i = 0; i < D; ++i) e.b[i] = p[D * D + i];
#pragma unroll
  for (int i = 0; i < D * D; ++i) e.C[i] = p[D * D + D + i];
#pragma unroll
  for (int i = 0; i < D; ++i) e.eta[i] = p[2 * D * D + D + i];
#pragma unroll
  for (int i = 0; i < D * D; ++i) e.J[i] = p[2 * D * D + 2 * D + i];
}
template <int D>
__device__ __forceinline__ void fe_store(double* p, const FElem<D>& e) {
#pragma unroll
  for (int i = 0; i < D * D; ++i) p[i] = e.A[i];
#pragma unroll
  for (int i = 0; i < D; ++i) p[D * D + i] = e.b[i];
#pragma unroll
  for (int i = 0; i < D * D; ++i) p[D * D + D + i] = e.C[i];
#pragma unroll
  for (int i = 0; i < D; ++i) p[2 * D * D + D + i] = e.eta[i];
#pragma unroll
  for (int i = 0; i < D * D; ++i) p[2 * D * D + 2 * D + i] = e.J[i];
}
template <int D>
constexpr int fe_size() { return 3 * D * D + 2 * D; }

// Row-pivoted LU in place (Eigen PartialPivLU semantics, pit.cpp:41-42)
template <int D>
__device__ __forceinline__ void lu_factor(double* M, int* perm) {
#pragma unroll
  for (int i = 0; i < D; ++i) perm[i] = i;
#pragma unroll
  for (int k = 0; k < D; ++k) {
    int p = k;
    double best = fabs(M[k * D + k]);
#pragma unroll
    for (int i = k + 1; i < D; ++i)
      if (fabs(M[i * D + k]) > best) {
        best = fabs(M[i * D + k]);
        p = i;
      }
    if (p != k) {
#pragma unroll
      for (int j = 0; j < D; ++j) {
        const double t = M[k * D + j];
        M[k * D + j] = M[p * D + j];
        M[p * D + j] = t;
      }
      const int t = perm[k];
      perm[k] = perm[p];
      perm[p] = t;
    }
    const double piv = M[k * D + k];
    if (piv != 0.0) {
#pragma unroll
      for (int i = k + 1; i < D; ++i) {
        const double f = M[i * D + k] / piv;
        M[i * D + k] = f;
#pragma unroll
        for (int j = k + 1; j < D; ++j) M[i * D + j] -= f * M[k * D + j];
      }
    }
  }
}
// X (D×R) = M^{-1} B
template <int D, int R>
__device__ __forceinline__ void lu_solve(const double* LU, const int* perm, const double* B,
                                         double* X) {
#pragma unroll
  for (int c = 0; c < R; ++c) {
#pragma unroll
    for (int i = 0; i < D; ++i) {
      double s = B[perm[i] * R + c];
#pragma unroll
      for (int j = 0; j < i; ++j) s -= LU[i * D + j] * X[j * R + c];
      X[i * R + c] = s;
    }
#pragma unroll
    for (int i = D - 1; i >= 0; --i) {
      double s = X[i * R + c];
#pragma unroll
      for (int j = i + 1; j < D; ++j) s -= LU[i * D + j] * X[j * R + c];
      X[i * R + c] = s / LU[i * D + i];
    }
  }
}

template <int D>
__device__ __forceinline__ void mm(const double* A, const double* B, double* C) {
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) {
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < D; ++k) s += A[i * D + k] * B[k * D + j];
      C[i * D + j] = s;
    }
}

// combine(u, v): u covers the earlier block (pit.cpp:36-51)
template <int D>
__device__ __forceinline__ void fe_combine(const FElem<D>& u, const FElem<D>& v, FElem<D>& o) {
  double M1[D * D], M2[D * D], S[D * D], T1[D * D], T2[D * D];
  int p1[D], p2[D];
  mm<D>(u.C, v.J, M1);
  mm<D>(v.J, u.C, M2);
#pragma unroll
  for (int i = 0; i < D; ++i) {
    M1[i * D + i] += 1.0;
    M2[i * D + i] += 1.0;
  }
  lu_factor<D>(M1, p1);
  lu_factor<D>(M2, p2);
  // A = vA lu.solve(uA)
  lu_solve<D, D>(M1, p1, u.A, S);
  mm<D>(v.A, S, o.A);
  // b = vA lu.solve(ub + uC veta) + vb
  double t[D], w[D];
#pragma unroll
  for (int i = 0; i < D; ++i) {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) s += u.C[i * D + k] * v.eta[k];
    t[i] = s + u.b[i];
  }
  lu_solve<D, 1>(M1, p1, t, w);
#pragma unroll
  for (int i = 0; i < D; ++i) {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) s += v.A[i * D + k] * w[k];
    o.b[i] = s + v.b[i];
  }
  // C = symm(vA lu.solve(uC) vA^T + vC)
  lu_solve<D, D>(M1, p1, u.C, S);
  mm<D>(v.A, S, T1);
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) {
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < D; ++k) s += T1[i * D + k] * v.A[j * D + k];
      T2[i * D + j] = s + v.C[i * D + j];
    }
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) o.C[i * D + j] = 0.5 * (T2[i * D + j] + T2[j * D + i]);
  // eta = uA^T lu_t.solve(veta - vJ ub) + ueta
#pragma unroll
  for (int i = 0; i < D; ++i) {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) s += v.J[i * D + k] * u.b[k];
    t[i] = v.eta[i] - s;
  }
  lu_solve<D, 1>(M2, p2, t, w);
#pragma unroll
  for (int i = 0; i < D; ++i) {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) s += u.A[k * D + i] * w[k];
    o.eta[i] = s + u.eta[i];
  }
  // J = symm(uA^T lu_t.solve(vJ) uA + uJ)
  lu_solve<D, D>(M2, p2, v.J, S);
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) {
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < D; ++k) s += u.A[k * D + i] * S[k * D + j];
      T1[i * D + j] = s;
    }
  mm<D>(T1, u.A, T2);
#pragma unroll
  for (int i = 0; i < D * D; ++i) T2[i] += u.J[i];
#pragma unroll
  for (int i = 0; i < D; ++i)
#pragma unroll
    for (int j = 0; j < D; ++j) o.J[i * D + j] = 0.5 * (T2[i * D + j] + T2[j * D + i]);
}

// ---- element build (pit.cpp:126-152), thread per (b, t)
// DY > 0: the observation count is the compile-time DY (static loop bounds, every
// array in registers); DY = 0: any dy <= kMaxDY (arrays in local memory).
template <int D, int DY>
__global__ void k_pf_elements(DevModel m, const double* __restrict__ obs, int B, double* el,
                              int* status) {
  constexpr int MY = DY > 0 ? DY : kMaxDY;
  const int T = m.T, dy = DY > 0 ? DY : m.dy;
  const long long n = (long long)B * (T + 1);
  constexpr int ES = fe_size<D>();
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (long long)gridDim.x * blockDim.x) {
    const int b = (int)(q / (T + 1)), t = (int)(q % (T + 1));
    double f[D * D], bd[D], qm[D * D];
#pragma unroll
    for (int i = 0; i < D * D; ++i) {
      f[i] = t == 0 ? ((i / D == i % D) ? 1.0 : 0.0) : m.Ft(t - 1, b)[i];
      const int r = i / D, c = i % D;
      const double* Qs = t == 0 ? m.P0 : m.Qt(t - 1, b);
      qm[i] = 0.5 * (Qs[r * D + c] + Qs[c * D + r]);  // Model ctor symmetrization
    }
#pragma unroll
    for (int i = 0; i < D; ++i) bd[i] = t == 0 ? m.m0[i] : m.bt(t - 1, b)[i];
    FElem<D> e;
    int st = 0;
    if (dy > 0 && m.observed(t)) {
      const double* h = m.Ht(t, b);
      const double* c = m.ct(t, b);
      const double* R = m.Rt(t, b);
      const double* y = obs + ((size_t)b * (T + 1) + t) * dy;
      double innov[MY], s[MY * MY], L[MY * MY], hq[MY * D],
          X1[MY * D], X2[MY * D];
      for (int i = 0; i < dy; ++i) {
        double acc = 0.0;
        for (int j = 0; j < D; ++j) acc += h[i * D + j] * bd[j];
        innov[i] = (y[i] - acc) - c[i];
      }
      for (int i = 0; i < dy; ++i)
        for (int j = 0; j < D; ++j) {
          double acc = 0.0;
          for (int k = 0; k < D; ++k) acc += h[i * D + k] * qm[k * D + j];
          hq[i * D + j] = acc;
        }
      for (int i = 0; i < dy; ++i)
        for (int j = 0; j < dy; ++j) {
          double acc = 0.0;
          for (int k = 0; k < D; ++k) acc += hq[i * D + k] * h[j * D + k];
          s[i * dy + j] = acc + 0.5 * (R[i * dy + j] + R[j * dy + i]);
        }
      for (int i = 0; i < dy; ++i)
        for (int j = i + 1; j < dy; ++j) {
          const double v = 0.5 * (s[i * dy + j] + s[j * dy + i]);
          s[i * dy + j] = v;
          s[j * dy + i] = v;
        }
      // factor_psd(s) (gauss.cpp:26-35), then X1 = s^-1 hq, X2 = s^-1 h
      auto llt = [&](const double* a) -> bool {
        for (int i = 0; i < dy * dy; ++i) L[i] = 0.0;
        for (int k = 0; k < dy; ++k) {
          double x = a[k * dy + k];
          for (int j = 0; j < k; ++j) x -= L[k * dy + j] * L[k * dy + j];
          if (x <= 0.0) return false;
          x = sqrt(x);
          L[k * dy + k] = x;
          for (int i = k + 1; i < dy; ++i) {
            double acc = a[i * dy + k];
            for (int j = 0; j < k; ++j) acc -= L[i * dy + j] * L[k * dy + j];
            L[i * dy + k] = acc / x;
          }
        }
        return true;
      };
      if (!llt(s)) {
        double tr = 0.0;
        for (int i = 0; i < dy; ++i) tr += s[i * dy + i];
        double sc = tr / dy;
        if (sc <= 0.0) {
          sc = 0.0;
          for (int i = 0; i < dy * dy; ++i) sc = fabs(s[i]) > sc ? fabs(s[i]) : sc;
        }
        bool ok = false;
        double sj[MY * MY];
        for (int e2 = 0; e2 < 2 && !ok; ++e2) {
          const double eps = e2 == 0 ? 1e-10 : 1e-8;
          for (int i = 0; i < dy * dy; ++i) sj[i] = s[i] + ((i / dy == i % dy) ? (eps * sc) * 1.0 : 0.0);
          ok = llt(sj);
        }
        if (!ok) st = AUXMC_E_FACTOR;
      }
      auto solve = [&](double* X) {  // X (dy×D) := (L L^T)^{-1} X
        for (int col = 0; col < D; ++col) {
          for (int i = 0; i < dy; ++i) {
            double acc = X[i * D + col];
            for (int j = 0; j < i; ++j) acc -= L[i * dy + j] * X[j * D + col];
            X[i * D + col] = acc / L[i * dy + i];
          }
          for (int i = dy - 1; i >= 0; --i) {
            double acc = X[i * D + col];
            for (int j = i + 1; j < dy; ++j) acc -= L[j * dy + i] * X[j * D + col];
            X[i * D + col] = acc / L[i * dy + i];
          }
        }
      };
      for (int i = 0; i < dy * D; ++i) {
        X1[i] = hq[i];
        X2[i] = h[i];
      }
      solve(X1);  // gain = X1^T
      solve(X2);  // hs = X2^T
      double a[D * D];
#pragma unroll
      for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) {
          double acc = 0.0;
          for (int k = 0; k < dy; ++k) acc += X1[k * D + i] * h[k * D + j];
          a[i * D + j] = (i == j ? 1.0 : 0.0) - acc;
        }
      mm<D>(a, f, e.A);
#pragma unroll
      for (int i = 0; i < D; ++i) {
        double acc = 0.0;
        for (int k = 0; k < dy; ++k) acc += X1[k * D + i] * innov[k];
        e.b[i] = bd[i] + acc;
      }
      double t1[D * D], t2[D * D];
      mm<D>(a, qm, t1);
#pragma unroll
      for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) {
          double acc = 0.0;
#pragma unroll
          for (int k = 0; k < D; ++k) acc += t1[i * D + k] * a[j * D + k];
          t2[i * D + j] = acc;
        }
      // + gain R gain^T
      double gr[D * MY];
      for (int i = 0; i < D; ++i)
        for (int j = 0; j < dy; ++j) {
          double acc = 0.0;
          for (int k = 0; k < dy; ++k) acc += X1[k * D + i] * (0.5 * (R[k * dy + j] + R[j * dy + k]));
          gr[i * MY + j] = acc;
        }
#pragma unroll
      for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) {
          double acc = 0.0;
          for (int k = 0; k < dy; ++k) acc += gr[i * MY + k] * X1[k * D + j];
          t2[i * D + j] += acc;
        }
#pragma unroll
      for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) e.C[i * D + j] = 0.5 * (t2[i * D + j] + t2[j * D + i]);
      // eta = f^T (hs innov); J = symm(((f^T hs) h) f)
      double hv[D];
#pragma unroll
      for (int i = 0; i < D; ++i) {
        double acc = 0.0;
        for (int k = 0; k < dy; ++k) acc += X2[k * D + i] * innov[k];
        hv[i] = acc;
      }
#pragma unroll
      for (int i = 0; i < D; ++i) {
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < D; ++k) acc += f[k * D + i] * hv[k];
        e.eta[i] = acc;
      }
      double fh[D * MY];
      for (int i = 0; i < D; ++i)
        for (int j = 0; j < dy; ++j) {
          double acc = 0.0;
          for (int k = 0; k < D; ++k) acc += f[k * D + i] * X2[j * D + k];
          fh[i * MY + j] = acc;
        }
#pragma unroll
      for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) {
          double acc = 0.0;
          for (int k = 0; k < dy; ++k) acc += fh[i * MY + k] * h[k * D + j];
          t1[i * D + j] = acc;
        }
      mm<D>(t1, f, t2);
#pragma unroll
      for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) e.J[i * D + j] = 0.5 * (t2[i * D + j] + t2[j * D + i]);
    } else {
#pragma unroll
      for (int i = 0; i < D * D; ++i) {
        e.A[i] = f[i];
        e.C[i] = qm[i];
        e.J[i] = 0.0;
      }
#pragma unroll
      for (int i = 0; i < D; ++i) {
        e.b[i] = bd[i];
        e.eta[i] = 0.0;
      }
    }
    if (t == 0) {
#pragma unroll
      for (int i = 0; i < D * D; ++i) e.A[i] = 0.0;
    }
    fe_store<D>(el + (size_t)q * ES, e);
    if (st) atomicMax(status + b, st);
  }
}

// S1: aggregate of each block
template <int D>
__global__ void k_pf_reduce(int T, int B, int LB, const double* __restrict__ el, double* agg) {
  constexpr int ES = fe_size<D>();
  const int nblk = (T + 1 + LB - 1) / LB;
  const long long n = (long long)B * nblk;
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (long long)gridDim.x * blockDim.x) {
    const int b = (int)(q / nblk), k = (int)(q % nblk);
    const int lo = k * LB, hi = min(lo + LB, T + 1);
    const double* base = el + (size_t)b * (T + 1) * ES;
    FElem<D> acc, e, o;
    fe_load<D>(base + (size_t)lo * ES, acc);
    for (int t = lo + 1; t < hi; ++t) {
      fe_load<D>(base + (size_t)t * ES, e);
      fe_combine<D>(acc, e, o);
      acc = o;
    }
    fe_store<D>(agg + (size_t)q * ES, acc);
  }
}

// S2: exclusive carries over blocks (carry_0 unused)
template <int D>
__global__ void k_pf_carry(int T, int B, int LB, const double* __restrict__ agg, double* carry) {
  constexpr int ES = fe_size<D>();
  const int nblk = (T + 1 + LB - 1) / LB;
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  FElem<D> acc, e, o;
  fe_load<D>(agg + (size_t)b * nblk * ES, acc);
  for (int k = 1; k < nblk; ++k) {
    fe_store<D>(carry + ((size_t)b * nblk + k) * ES, acc);
    fe_load<D>(agg + ((size_t)b * nblk + k) * ES, e);
    fe_combine<D>(acc, e, o);
    acc = o;
  }
}

// S3: inclusive elements; write filtered moments directly (filt = (b, C))
template <int D>
__global__ void k_pf_apply(int T, int B, int LB, const double* __restrict__ el,
                           const double* __restrict__ carry, double* filt_mean, double* filt_cov) {
  constexpr int ES = fe_size<D>();
  const int nblk = (T + 1 + LB - 1) / LB;
  const long long n = (long long)B * nblk;
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (long long)gridDim.x * blockDim.x) {
    const int b = (int)(q / nblk), k = (int)(q % nblk);
    const int lo = k * LB, hi = min(lo + LB, T + 1);
    const double* base = el + (size_t)b * (T + 1) * ES;
    FElem<D> acc, e, o;
    if (k == 0) {
      fe_load<D>(base + (size_t)lo * ES, acc);
    } else {
      fe_load<D>(carry + (size_t)q * ES, acc);
      fe_load<D>(base + (size_t)lo * ES, e);
      fe_combine<D>(acc, e, o);
      acc = o;
    }
    for (int t = lo;; ++t) {
#pragma unroll
      for (int i = 0; i < D; ++i) filt_mean[((size_t)b * (T + 1) + t) * D + i] = acc.b[i];
#pragma unroll
      for (int i = 0; i < D * D; ++i) filt_cov[((size_t)b * (T + 1) + t) * D * D + i] = acc.C[i];
      if (t + 1 >= hi) break;
      fe_load<D>(base + (size_t)(t + 1) * ES, e);
      fe_combine<D>(acc, e, o);
      acc = o;
    }
  }
}

// Small horizons: the whole scan of one sequence in one CTA, with the
// reference's own Sklansky fan (scan.hpp:22-41: at stride s, element j with
// bit s set absorbs the prefix ending at (j & ~(s-1)) - 1), elements resident
// in shared memory; ⌈log2 n⌉ barriers instead of the three launches and ~3
// sqrt(n) sequential combines of the blocked scan.
template <int D>
__global__ void __launch_bounds__(D == 1 ? 1024 : 256) k_pf_sklansky(int T, int B, const double* __restrict__ el,
                                                      double* filt_mean, double* filt_cov) {
  extern __shared__ double sm[];
  constexpr int ES = fe_size<D>();
  const int n = T + 1, b = blockIdx.x;
  const double* base = el + (size_t)b * n * ES;
  for (int i = threadIdx.x; i < n * ES; i += blockDim.x) sm[i] = base[i];
  __syncthreads();
  for (int stride = 1; stride < n; stride <<= 1) {
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
      if (!(j & stride)) continue;
      const int pivot = (j & ~(stride - 1)) - 1;
      FElem<D> u, v, o;
      fe_load<D>(sm + (size_t)pivot * ES, u);
      fe_load<D>(sm + (size_t)j * ES, v);
      fe_combine<D>(u, v, o);  // a level writes only bit-set slots and reads only pivots
      fe_store<D>(sm + (size_t)j * ES, o);
    }
    __syncthreads();
  }
  for (int t = threadIdx.x; t < n; t += blockDim.x) {
#pragma unroll
    for (int i = 0; i < D; ++i) filt_mean[((size_t)b * n + t) * D + i] = sm[(size_t)t * ES + D * D + i];
#pragma unroll
    for (int i = 0; i < D * D; ++i)
      filt_cov[((size_t)b * n + t) * D * D + i] = sm[(size_t)t * ES + D * D + D + i];
  }
}

template <int D>
constexpr int sklansky_max_n() {
  return (200 * 1024) / (int)(sizeof(double) * fe_size<D>());
}

// recovery (pit.cpp:167-186): predictive moments from filt[t-1]; log-likelihood terms
template <int D, int DY>
__global__ void k_pf_recover(DevModel m, const double* __restrict__ obs, int B,
                             const double* __restrict__ fm, const double* __restrict__ fc,
                             double* pm, double* pc, double* terms, int* status) {
  constexpr int MY = DY > 0 ? DY : kMaxDY;
  const int T = m.T, dy = DY > 0 ? DY : m.dy;
  const long long n = (long long)B * (T + 1);
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (long long)gridDim.x * blockDim.x) {
    const int b = (int)(q / (T + 1)), t = (int)(q % (T + 1));
    double mp[D], P[D * D];
    if (t == 0) {
#pragma unroll
      for (int i = 0; i < D; ++i) mp[i] = m.m0[i];
#pragma unroll
      for (int i = 0; i < D * D; ++i) {
        const int r = i / D, c = i % D;
        P[i] = 0.5 * (m.P0[r * D + c] + m.P0[c * D + r]);
      }
    } else {
      const double* F = m.Ft(t - 1, b);
      const double* bb = m.bt(t - 1, b);
      const double* Q = m.Qt(t - 1, b);
      const double* x = fm + (size_t)(q - 1) * D;
      const double* C = fc + (size_t)(q - 1) * D * D;
#pragma unroll
      for (int i = 0; i < D; ++i) {
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < D; ++k) acc += F[i * D + k] * x[k];
        mp[i] = acc + bb[i];
      }
      double t1[D * D];
#pragma unroll
      for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) {
          double acc = 0.0;
#pragma unroll
          for (int k = 0; k < D; ++k) acc += F[i * D + k] * C[k * D + j];
          t1[i * D + j] = acc;
        }
#pragma unroll
      for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) {
          double acc = 0.0;
#pragma unroll
          for (int k = 0; k < D; ++k) acc += t1[i * D + k] * F[j * D + k];
          P[i * D + j] = acc + 0.5 * (Q[i * D + j] + Q[j * D + i]);
        }
#pragma unroll
      for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = i + 1; j < D; ++j) {
          const double v = 0.5 * (P[i * D + j] + P[j * D + i]);
          P[i * D + j] = v;
          P[j * D + i] = v;
        }
    }
#pragma unroll
    for (int i = 0; i < D; ++i) pm[(size_t)q * D + i] = mp[i];
#pragma unroll
    for (int i = 0; i < D * D; ++i) pc[(size_t)q * D * D + i] = P[i];
    double term = 0.0;
    if (dy > 0 && m.observed(t)) {
      const double* h = m.Ht(t, b);
      const double* c = m.ct(t, b);
      const double* R = m.Rt(t, b);
      const double* y = obs + (size_t)q * dy;
      double s[MY * MY], L[MY * MY], r[MY], hp[MY * D];
      for (int i = 0; i < dy; ++i) {
        double acc = 0.0;
        for (int k = 0; k < D; ++k) acc += h[i * D + k] * mp[k];
        r[i] = y[i] - (acc + c[i]);
        for (int j = 0; j < D; ++j) {
          double a2 = 0.0;
          for (int k = 0; k < D; ++k) a2 += h[i * D + k] * P[k * D + j];
          hp[i * D + j] = a2;
        }
      }
      for (int i = 0; i < dy; ++i)
        for (int j = 0; j < dy; ++j) {
          double acc = 0.0;
          for (int k = 0; k < D; ++k) acc += hp[i * D + k] * h[j * D + k];
          s[i * dy + j] = acc + R[i * dy + j];
        }
      for (int i = 0; i < dy; ++i)
        for (int j = i; j < dy; ++j) {
          const double v = 0.5 * (s[i * dy + j] + s[j * dy + i]);
          s[i * dy + j] = v;
          s[j * dy + i] = v;
        }
      // log_pdf(y; Hm + c, S) with factor_psd (gauss.cpp:51-57)
      bool ok = true;
      for (int pass = 0; pass < 3; ++pass) {
        double sc = 0.0;
        if (pass > 0) {
          double tr = 0.0;
          for (int i = 0; i < dy; ++i) tr += s[i * dy + i];
          sc = tr / dy;
          if (sc <= 0.0)
            for (int i = 0; i < dy * dy; ++i) sc = fabs(s[i]) > sc ? fabs(s[i]) : sc;
          sc *= pass == 1 ? 1e-10 : 1e-8;
        }
        ok = true;
        for (int i = 0; i < dy * dy; ++i) L[i] = 0.0;
        for (int k = 0; k < dy && ok; ++k) {
          double x = s[k * dy + k] + (pass ? sc * 1.0 : 0.0);
          for (int j = 0; j < k; ++j) x -= L[k * dy + j] * L[k * dy + j];
          if (x <= 0.0) { ok = false; break; }
          x = sqrt(x);
          L[k * dy + k] = x;
          for (int i = k + 1; i < dy; ++i) {
            double acc = s[i * dy + k];
            for (int j = 0; j < k; ++j) acc -= L[i * dy + j] * L[k * dy + j];
            L[i * dy + k] = acc / x;
          }
        }
        if (ok) break;
      }
      if (!ok) atomicMax(status + b, AUXMC_E_FACTOR);
      double sq = 0.0, ld = 0.0;
      for (int i = 0; i < dy; ++i) {
        double acc = r[i];
        for (int j = 0; j < i; ++j) acc -= L[i * dy + j] * r[j];
        r[i] = acc / L[i * dy + i];
        sq += r[i] * r[i];
      }
      for (int i = 0; i < dy; ++i) ld += log(L[i * dy + i]);
      term = -0.5 * (dy * kLog2Pi + sq) - ld;
    }
    terms[q] = term;
  }
}

__global__ void k_pf_sum(int T, int B, const double* terms, double* out) {
  __shared__ double red[kSumThreads];
  const int b = blockIdx.x;
  const double* tm = terms + (size_t)b * (T + 1);
  const double s = cta_sum_fixed((long long)T + 1, [&](long long i) { return tm[i]; }, red);
  if (threadIdx.x == 0) out[b] = s;
}

static int pf_block(int T) {
  int lb = 1;
  while ((long long)lb * lb < T + 1) lb <<= 1;  // ~sqrt(T+1): balances S1/S3 and S2 spans
  return lb < 4 ? 4 : lb;
}

template <int D>
static int run_pf(const DevModel& dm, const double* obs, int B, auxmc_filter_result* out,
                  int* status, Arena& ws, cudaStream_t s) {
  constexpr int ES = fe_size<D>();
  const int T = dm.T, LB = pf_block(T);
  const int nblk = (T + 1 + LB - 1) / LB;
  double* el = ws.take<double>((size_t)B * (T + 1) * ES);
  double* agg = ws.take<double>((size_t)B * nblk * ES);
  double* carry = ws.take<double>((size_t)B * nblk * ES);
  double* terms = ws.take<double>((size_t)B * (T + 1));
  if (ws.base == nullptr) return AUXMC_OK;
  if (!el || !agg || !carry || !terms) return AUXMC_E_WORKSPACE;
  AUXMC_CUDA_TRY(cudaMemsetAsync(status, 0, sizeof(int) * B, s));
  const long long n = (long long)B * (T + 1);
  const long long nb = (long long)B * nblk;
  auto grid = [](long long k) { return (int)std::max(1LL, std::min((k + 127) / 128, 148LL * 16)); };
  switch (dm.dy) {  // small observation counts: register-resident element builds
#define PF_EL(DYV)                                                                         \
  case DYV:                                                                                \
    AUXMC_LAUNCH((k_pf_elements<D, DYV>), grid(n), 128, 0, s, dm, obs, B, el, status);  \
    break;
    PF_EL(1) PF_EL(2) PF_EL(3) PF_EL(4)
#undef PF_EL
    default:
      AUXMC_LAUNCH((k_pf_elements<D, 0>), grid(n), 128, 0, s, dm, obs, B, el, status);
  }
  if (T + 1 <= sklansky_max_n<D>() && B <= 2 * 148) {
    // few short sequences: one CTA each, Sklansky in shared memory
    const size_t smem = sizeof(double) * (size_t)(T + 1) * ES;
    AUXMC_CUDA_TRY(cudaFuncSetAttribute(k_pf_sklansky<D>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int threads = std::min(D == 1 ? 1024 : 256, std::max(32, ((T + 1 + 31) / 32) * 32));
    AUXMC_LAUNCH(k_pf_sklansky<D>, B, threads, smem, s, T, B, el, out->filt_mean, out->filt_cov);
  } else {
    AUXMC_LAUNCH(k_pf_reduce<D>, grid(nb), 128, 0, s, T, B, LB, el, agg);
    AUXMC_LAUNCH(k_pf_carry<D>, (B + 127) / 128, 128, 0, s, T, B, LB, agg, carry);
    AUXMC_LAUNCH(k_pf_apply<D>, grid(nb), 128, 0, s, T, B, LB, el, carry, out->filt_mean,
                 out->filt_cov);
  }
  switch (dm.dy) {
#define PF_RC(DYV)                                                                          \
  case DYV:                                                                                 \
    AUXMC_LAUNCH((k_pf_recover<D, DYV>), grid(n), 128, 0, s, dm, obs, B, out->filt_mean,   \
                 out->filt_cov, out->pred_mean, out->pred_cov, terms, status);              \
    break;
    PF_RC(1) PF_RC(2) PF_RC(3) PF_RC(4)
#undef PF_RC
    default:
      AUXMC_LAUNCH((k_pf_recover<D, 0>), grid(n), 128, 0, s, dm, obs, B, out->filt_mean,
                   out->filt_cov, out->pred_mean, out->pred_cov, terms, status);
  }
  AUXMC_LAUNCH(k_pf_sum, B, kSumThreads, 0, s, T, B, terms, out->log_marginal);
  return AUXMC_OK;
}

int dispatch_pf_generic(const DevModel& dm, const double* obs, int B, auxmc_filter_result* out,
                        int* status, Arena& ws, cudaStream_t s);

static int dispatch_pf(const DevModel& dm, const double* obs, int B, auxmc_filter_result* out,
                       int* status, Arena& ws, cudaStream_t s) {
  if (dm.dy > kMaxDY || dm.dx > 6) return dispatch_pf_generic(dm, obs, B, out, status, ws, s);
  switch (dm.dx) {
    case 1: return run_pf<1>(dm, obs, B, out, status, ws, s);
    case 2: return run_pf<2>(dm, obs, B, out, status, ws, s);
    case 3: return run_pf<3>(dm, obs, B, out, status, ws, s);
    case 4: return run_pf<4>(dm, obs, B, out, status, ws, s);
    case 5: return run_pf<5>(dm, obs, B, out, status, ws, s);
    case 6: return run_pf<6>(dm, obs, B, out, status, ws, s);
  }
  return AUXMC_E_DIM;
}

size_t filter_pit_workspace(const DevModel& dm, int B) {
  Arena ws{nullptr, 0, 0};
  dispatch_pf(dm, nullptr, B, nullptr, nullptr, ws, nullptr);
  return ws.used + 1024;
}

int launch_filter_pit(const DevModel& dm, const double* obs, int B, auxmc_filter_result* out,
                      int* status, Arena& ws, cudaStream_t stream) {
  return dispatch_pf(dm, obs, B, out, status, ws, stream);
}

}  // namespace auxmc_gpu
