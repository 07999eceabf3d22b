// target.cuh — device view of auxmc_target (target.hpp:34-93) and the model
// functors shared by the auxiliary Kalman and particle Gibbs kernels.
#pragma once
#include "common.cuh"
#include "dense.cuh"

namespace auxmc_gpu {

struct DevTarget {
  int kind, T, dx, ydim, linear;
  const double *m0, *P0, *F, *b, *Q;
  int nF, q, ne, exact_tv;
  const double *eH, *ec, *eR, *ey;
  const uint8_t* emask;
  const double* data;
  const uint8_t* gmask;
  const double *gH, *gc, *gR;
  double lz_sigma, lz_rho, lz_beta, lz_h, l96_F, l96_h;
  int exact_sel;
  __device__ __forceinline__ const double* Ft(int t) const { return F + (size_t)(nF > 1 ? t : 0) * dx * dx; }
  __device__ __forceinline__ const double* bt(int t) const { return b + (size_t)(nF > 1 ? t : 0) * dx; }
  __device__ __forceinline__ const double* Qt(int t) const { return Q + (size_t)(nF > 1 ? t : 0) * dx * dx; }
  __device__ __forceinline__ const double* eHt(int t) const { return eH + (size_t)(ne > 1 ? t : 0) * q * dx; }
  __device__ __forceinline__ const double* ect(int t) const { return ec + (size_t)(ne > 1 ? t : 0) * q; }
  __device__ __forceinline__ const double* eRt(int t) const { return eR + (size_t)(ne > 1 ? t : 0) * q * q; }
  __device__ __forceinline__ const double* gHt(int t) const { return gH + (size_t)(ne > 1 ? t : 0) * ydim * dx; }
  __device__ __forceinline__ const double* gct(int t) const { return gc + (size_t)(ne > 1 ? t : 0) * ydim; }
  __device__ __forceinline__ const double* gRt(int t) const { return gR + (size_t)(ne > 1 ? t : 0) * ydim * ydim; }
};

static DevTarget to_dev_target(const auxmc_target& t) {
  DevTarget d;
  d.kind = t.kind; d.T = t.T; d.dx = t.dx; d.ydim = t.ydim; d.linear = t.linear;
  d.m0 = t.m0; d.P0 = t.P0; d.F = t.F; d.b = t.b; d.Q = t.Q; d.nF = t.nF;
  d.q = t.q; d.ne = t.ne; d.exact_tv = t.exact_tv;
  d.eH = t.eH; d.ec = t.ec; d.eR = t.eR; d.ey = t.ey; d.emask = t.emask;
  d.data = t.data; d.gmask = t.gmask; d.gH = t.gH; d.gc = t.gc; d.gR = t.gR;
  d.lz_sigma = t.lz_sigma; d.lz_rho = t.lz_rho; d.lz_beta = t.lz_beta; d.lz_h = t.lz_h;
  d.l96_F = t.l96_F; d.l96_h = t.l96_h;
  d.exact_sel = t.exact_sel;
  return d;
}

static int check_target(const auxmc_target* t) {
  if (!t) return AUXMC_E_ARG;
  if (t->T < 0 || t->dx < 1 || t->dx > 64 || t->q < 0 || t->dx + t->q > 64 || t->ydim < 0 ||
      t->ydim > 64)
    return AUXMC_E_DIM;
  if (!t->m0 || !t->P0 || !t->Q || !t->emask || !t->gmask) return AUXMC_E_ARG;
  if (t->linear && (!t->F || !t->b)) return AUXMC_E_ARG;
  if (t->q > 0 && (!t->eH || !t->ec || !t->eR || !t->ey)) return AUXMC_E_ARG;
  if (t->kind == AUXMC_KIND_GAUSS_GENERIC && (!t->gH || !t->gc || !t->gR || !t->data))
    return AUXMC_E_ARG;
  if ((t->kind == AUXMC_KIND_STOCHVOL || t->kind == AUXMC_KIND_SPATIO) && !t->data)
    return AUXMC_E_ARG;
  if (!t->linear && t->kind != AUXMC_KIND_LORENZ63 && t->kind != AUXMC_KIND_LORENZ96)
    return AUXMC_E_CONFIG;
  return AUXMC_OK;
}

// ---------------------------------------------------------------- functors
// E[x_{t+1} | x_t = x]_i (target.cpp:47-49; models.cpp:283-297; Lorenz-96)
__device__ __forceinline__ double dyn_mean_i(const DevTarget& tg, int t, const double* x, int i) {
  const int d = tg.dx;
  if (tg.linear) {
    const double* F = tg.Ft(t);
    double s = 0.0;
    for (int j = 0; j < d; ++j) s += F[i * d + j] * x[j];
    return s + tg.bt(t)[i];
  }
  if (tg.kind == AUXMC_KIND_LORENZ63) {
    const double f = i == 0 ? tg.lz_sigma * (x[1] - x[0])
                     : i == 1 ? x[0] * (tg.lz_rho - x[2]) - x[1]
                              : x[0] * x[1] - tg.lz_beta * x[2];
    return x[i] + tg.lz_h * f;
  }
  const double f = (x[(i + 1) % d] - x[(i + d - 2) % d]) * x[(i + d - 1) % d] - x[i] + tg.l96_F;
  return x[i] + tg.l96_h * f;
}

// ∂ mean_i / ∂ x_j (target.cpp:51-53)
__device__ __forceinline__ double dyn_jac_ij(const DevTarget& tg, int t, const double* x, int i, int j) {
  const int d = tg.dx;
  if (tg.linear) return tg.Ft(t)[i * d + j];
  double J;
  if (tg.kind == AUXMC_KIND_LORENZ63) {
    const double Jm[9] = {-tg.lz_sigma, tg.lz_sigma, 0.0, tg.lz_rho - x[2], -1.0, -x[0],
                          x[1],         x[0],        -tg.lz_beta};
    J = Jm[i * 3 + j];
    return (i == j ? 1.0 : 0.0) + tg.lz_h * J;
  }
  const int ip1 = (i + 1) % d, im1 = (i + d - 1) % d, im2 = (i + d - 2) % d;
  J = 0.0;
  if (j == ip1) J += x[im1];
  if (j == im2) J -= x[im1];
  if (j == im1) J += x[ip1] - x[im2];
  if (j == i) J -= 1.0;
  return (i == j ? 1.0 : 0.0) + tg.l96_h * J;
}

// Mahalanobis term with a precomputed lower factor: -0.5 (n log 2π + |L^-1 r|^2) - logdet
__device__ __forceinline__ double gauss_term(int n, double* r, const double* L, double logdet) {
  double sq = 0.0;
  for (int i = 0; i < n; ++i) {
    double s = r[i];
    for (int j = 0; j < i; ++j) s -= L[i * n + j] * r[j];
    r[i] = s / L[i * n + i];
    sq += r[i] * r[i];
  }
  return -0.5 * (n * kLog2Pi + sq) - logdet;
}

// generic factor log g_t(x) (models.cpp:261-317; testutil.hpp:112-140)
__device__ __forceinline__ double generic_log_g(const DevTarget& tg, int t, const double* x, const double* Lg,
                                double ldg, double* r) {
  const int d = tg.dx;
  const double* y = tg.data + (size_t)t * tg.ydim;
  switch (tg.kind) {
    case AUXMC_KIND_STOCHVOL: {
      double sx = 0.0, sy = 0.0;
      for (int i = 0; i < d; ++i) sx += x[i];
      for (int i = 0; i < d; ++i) sy += (y[i] * y[i]) * exp(-x[i]);
      return -0.5 * (log(2.0 * 3.14159265358979323846) * d + sx + sy);
    }
    case AUXMC_KIND_SPATIO: {
      double s = 0.0;
      for (int j = 0; j < d; ++j) s += y[j] * x[j] - exp(x[j]) - lgamma(y[j] + 1.0);
      return s;
    }
    case AUXMC_KIND_GRID1D:
      return -x[0] * x[0] * x[0] * x[0];
    case AUXMC_KIND_GAUSS_GENERIC: {
      const int n = tg.ydim;
      const double* H = tg.gHt(t);
      const double* c = tg.gct(t);
      for (int i = 0; i < n; ++i) {
        double s = 0.0;
        for (int j = 0; j < d; ++j) s += H[i * d + j] * x[j];
        r[i] = ((y[i] - c[i]) - s) - 0.0;
      }
      return gauss_term(n, r, Lg, ldg);
    }
    case AUXMC_KIND_TEST_ABORT:
      return -0.5 * x[0] * x[0];
    case AUXMC_KIND_TEST_SUPPORT:
      return x[0] > 0.4 ? -INFINITY : 0.0;
    case AUXMC_KIND_TEST_COLLAPSE:
      return t == 2 ? -INFINITY : 0.0;
  }
  return 0.0;
}

__device__ __forceinline__ void generic_grad(const DevTarget& tg, int t, const double* x, const double* Lg,
                             double* r, double* g) {
  const int d = tg.dx;
  if (!tg.gmask[t]) {
    for (int i = 0; i < d; ++i) g[i] = 0.0;
    return;
  }
  const double* y = tg.data + (size_t)t * tg.ydim;
  switch (tg.kind) {
    case AUXMC_KIND_STOCHVOL:
      for (int i = 0; i < d; ++i) g[i] = 0.5 * ((y[i] * y[i]) * exp(-x[i]) - 1.0);
      return;
    case AUXMC_KIND_SPATIO:
      for (int i = 0; i < d; ++i) g[i] = y[i] - exp(x[i]);
      return;
    case AUXMC_KIND_GRID1D:
      g[0] = -4.0 * x[0] * x[0] * x[0];
      return;
    case AUXMC_KIND_TEST_ABORT:
      g[0] = fabs(x[0]) > 0.5 ? __longlong_as_double(0x7ff8000000000000ll) : -x[0];
      return;
    case AUXMC_KIND_GAUSS_GENERIC: {
      const int n = tg.ydim;
      const double* H = tg.gHt(t);
      const double* c = tg.gct(t);
      for (int i = 0; i < n; ++i) {
        double s = 0.0;
        for (int j = 0; j < d; ++j) s += H[i * d + j] * x[j];
        r[i] = (y[i] - c[i]) - s;
      }
      for (int i = 0; i < n; ++i) {  // L L^T z = r
        double s = r[i];
        for (int j = 0; j < i; ++j) s -= Lg[i * n + j] * r[j];
        r[i] = s / Lg[i * n + i];
      }
      for (int i = n - 1; i >= 0; --i) {
        double s = r[i];
        for (int j = i + 1; j < n; ++j) s -= Lg[j * n + i] * r[j];
        r[i] = s / Lg[i * n + i];
      }
      for (int j = 0; j < d; ++j) {
        double s = 0.0;
        for (int i = 0; i < n; ++i) s += H[i * d + j] * r[i];
        g[j] = s;
      }
      return;
    }
  }
  for (int i = 0; i < d; ++i) g[i] = 0.0;
}

// ---------------------------------------------------------------- target factors
// items: P0 | Q_i (nF) | eR_i (ne, if q > 0) | gR_i (ne, if generic Gaussian)
struct FactorLayout {
  int nQ, nE, nG, W;
  __host__ __device__ int total() const { return 1 + nQ + nE + nG; }
};

static FactorLayout factor_layout(const DevTarget& tg) {
  FactorLayout f;
  f.nQ = tg.linear ? tg.nF : 1;
  f.nE = tg.q > 0 ? tg.ne : 0;
  f.nG = tg.kind == AUXMC_KIND_GAUSS_GENERIC ? tg.ne : 0;
  int W = tg.dx;
  if (tg.q > W) W = tg.q;
  if (f.nG && tg.ydim > W) W = tg.ydim;
  f.W = W;
  return f;
}


}  // namespace auxmc_gpu
