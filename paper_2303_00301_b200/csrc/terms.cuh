// terms.cuh — per-term bodies of the path log-densities, shared by the full-horizon
// kernels (one thread per (path, term), fixed-order sums: logpdf.cu, auxk.cu) and the
// time-sharded aux step (per-t sums over super-blocks, auxk.cu tshard section).
//
// Term index k of a path of T steps: 0 prior, 1..T transitions t = k-1, T+1..2T+1
// observations t = k-T-1 (lgssm.cpp:179-199, target.cpp:100-108).
#pragma once
#include "common.cuh"
#include "dense.cuh"
#include "target.cuh"

namespace auxmc_gpu {

// lgssm::path_logpdf term k of path b (x = its [T+1][dx] rows, obs_b its [T+1][dy] rows).
// Masked or absent observations contribute 0 (lgssm.cpp:193-196).  dg (optional): 1 per
// factor whose L is diagonal — the residual is then scaled entry by entry with no local
// residual array (the same operations: the off-diagonal updates are exact zeros).
__device__ __forceinline__ double path_term_k(const DevModel& m, const double* __restrict__ obs_b,
                                              const double* __restrict__ x, int b, int B,
                                              const double* __restrict__ Ls,
                                              const double* __restrict__ logdet, int k,
                                              const unsigned char* __restrict__ dg = nullptr,
                                              const int* __restrict__ hsel = nullptr) {
  const int T = m.T, dx = m.dx, dy = m.dy;
  const int W = dx > dy ? dx : dy;
  int nn, j, t = 0, kind;
  if (k == 0) {
    kind = 0;
    nn = dx;
    j = 0;
  } else if (k <= T) {
    kind = 1;
    t = k - 1;
    nn = dx;
    j = 1 + (m.sQ ? b * m.nQ : 0) + (m.nQ > 1 ? t : 0);
  } else {
    kind = 2;
    t = k - T - 1;
    if (!m.observed(t) || dy == 0) return 0.0;
    nn = dy;
    const int nq = (m.sQ ? B : 1) * m.nQ;
    j = 1 + nq + (m.sR ? b * m.nR : 0) + (m.nR > 1 ? t : 0);
  }
  const double* L = Ls + (size_t)j * W * W;
  const double ld = logdet[j];
  const double* bb = kind == 1 ? m.bt(t, b) : nullptr;
  const double* H = kind == 2 ? m.Ht(t, b) : nullptr;
  const double* cc = kind == 2 ? m.ct(t, b) : nullptr;
  const double* y = kind == 2 ? obs_b + (size_t)t * dy : nullptr;
  auto res = [&](int i) -> double {  // residual entry i
    if (kind == 0) return x[i] - m.m0[i];
    double s = 0.0;
    if (kind == 1) {
      if (m.fst) {  // stencil F (l96_row): the dense row's nonzeros in column order
        int cs[4];
        double vs[4];
        stencil_row(m, t, b, i, cs, vs);
        for (int a = 0; a < 4; ++a) s += vs[a] * x[(size_t)t * dx + cs[a]];
      } else {
        const double* F = m.Ft(t, b);
        for (int jj = 0; jj < dx; ++jj) s += F[i * dx + jj] * x[(size_t)t * dx + jj];
      }
      return x[(size_t)(t + 1) * dx + i] - (s + bb[i]);
    }
    // hsel: per H row, the one nonzero column (-1: none; -2: dense) — the dense sum's
    // value exactly (its other products are zeros)
    const int hs = hsel ? hsel[(size_t)(m.nH > 1 ? t : 0) * dy + i] : -2;
    if (hs >= 0) s = H[i * dx + hs] * x[(size_t)t * dx + hs];
    else if (hs == -2)
      for (int jj = 0; jj < dx; ++jj) s += H[i * dx + jj] * x[(size_t)t * dx + jj];
    return y[i] - (s + cc[i]);
  };
  double sq = 0.0;
  if (kind == 1 && !m.fst && dx == 16) {
    // dense transition at d = 16: the row x_t loaded once into registers, the same
    // products and solve in the same order (static bounds)
    const double* F = m.Ft(t, b);
    double xv[16], r[16];
#pragma unroll
    for (int jj = 0; jj < 16; ++jj) xv[jj] = x[(size_t)t * 16 + jj];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      double s = 0.0;
#pragma unroll
      for (int jj = 0; jj < 16; ++jj) s += F[i * 16 + jj] * xv[jj];
      r[i] = x[(size_t)(t + 1) * 16 + i] - (s + bb[i]);
    }
    if (dg && dg[j]) {
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const double v = r[i] / L[i * 16 + i];
        sq += v * v;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        double s = r[i];
#pragma unroll
        for (int jj = 0; jj < i; ++jj) s -= L[i * 16 + jj] * r[jj];
        r[i] = s / L[i * 16 + i];
        sq += r[i] * r[i];
      }
    }
    return -0.5 * (nn * kLog2Pi + sq) - ld;
  }
  if (dg && dg[j]) {
    for (int i = 0; i < nn; ++i) {
      const double v = res(i) / L[i * nn + i];
      sq += v * v;
    }
  } else {
    double r[64];
    for (int i = 0; i < nn; ++i) r[i] = res(i);
    for (int i = 0; i < nn; ++i) {
      double s = r[i];
      for (int jj = 0; jj < i; ++jj) s -= L[i * nn + jj] * r[jj];
      r[i] = s / L[i * nn + i];
      sq += r[i] * r[i];
    }
  }
  return -0.5 * (nn * kLog2Pi + sq) - ld;
}

// target.log_gamma term k of the path x (target.cpp:100-108), with the target's factors.
__device__ __forceinline__ double gamma_term_k(const DevTarget& tg, const FactorLayout& fl,
                                               const double* __restrict__ x,
                                               const double* __restrict__ Ls,
                                               const double* __restrict__ logdet, int k,
                                               const unsigned char* __restrict__ dgf = nullptr) {
  const int T = tg.T, d = tg.dx, W = fl.W;
  // a factor diagonal to the bit: gauss_term's dense solve subtracts only exact zeros
  // (each s - 0 r_j is s, r_j finite), so its value is the diagonal terms' own
  auto gterm = [&](int n, double* r, int jf) -> double {
    const double* L = Ls + (size_t)jf * W * W;
    if (dgf && dgf[jf]) {
      double sq = 0.0;
      for (int i = 0; i < n; ++i) {
        r[i] = r[i] / L[i * n + i];
        sq += r[i] * r[i];
      }
      return -0.5 * (n * kLog2Pi + sq) - logdet[jf];
    }
    return gauss_term(n, r, L, logdet[jf]);
  };
  double r[64];
  if (k == 0) {
    for (int i = 0; i < d; ++i) r[i] = x[i] - tg.m0[i];
    return gterm(d, r, 0);
  }
  if (k <= T) {
    const int t = k - 1;
    const int jq = 1 + (fl.nQ > 1 ? t : 0);
    if (tg.linear && d == 16) {
      // d = 16 linear dynamics: dyn_mean_i and gauss_term's operations in their order,
      // with the state row in registers and static bounds
      const double* F = tg.Ft(t);
      const double* bt = tg.bt(t);
      const double* L = Ls + (size_t)jq * W * W;
      double xv[16], rr[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) xv[j] = x[(size_t)t * 16 + j];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < 16; ++j) s += F[i * 16 + j] * xv[j];
        rr[i] = x[(size_t)(t + 1) * 16 + i] - (s + bt[i]);
      }
      double sq = 0.0;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        double s = rr[i];
#pragma unroll
        for (int j = 0; j < i; ++j) s -= L[i * 16 + j] * rr[j];
        rr[i] = s / L[i * 16 + i];
        sq += rr[i] * rr[i];
      }
      return -0.5 * (16 * kLog2Pi + sq) - logdet[jq];
    }
    for (int i = 0; i < d; ++i) r[i] = x[(size_t)(t + 1) * d + i] - dyn_mean_i(tg, t, x + (size_t)t * d, i);
    return gterm(d, r, jq);
  }
  const int t = k - T - 1;
  const double* xt = x + (size_t)t * d;
  double lp = 0.0;
  if (tg.q > 0 && tg.emask[t]) {
    const double* H = tg.eHt(t);
    const double* cc = tg.ect(t);
    const double* y = tg.ey + (size_t)t * tg.q;
    for (int i = 0; i < tg.q; ++i) {
      double s = 0.0;
      for (int j = 0; j < d; ++j) s += H[i * d + j] * xt[j];
      r[i] = y[i] - (s + cc[i]);
    }
    const int je = 1 + fl.nQ + (tg.ne > 1 ? t : 0);
    lp += gterm(tg.q, r, je);
  }
  if (tg.gmask[t]) {
    const int jg = 1 + fl.nQ + fl.nE + (tg.ne > 1 ? t : 0);
    lp += generic_log_g(tg, t, xt, fl.nG ? Ls + (size_t)jg * W * W : nullptr,
                        fl.nG ? logdet[jg] : 0.0, r);
  }
  return lp;
}

}  // namespace auxmc_gpu
