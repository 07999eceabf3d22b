// filter.cu — batched Kalman filtering on B200.
//
//  * k_filter_seq: lgssm::kalman_filter (lgssm.cpp:73-112), covariance form with
//    Joseph update, one sequence per group (warp for small dims, CTA for large).
//    The innovation factor is computed once and reused for the log-likelihood
//    term: the reference factors the identical symmetrized S twice
//    (lgssm.cpp:101 and :105-106), which yields the same bits.
#include "common.cuh"
#include "dense.cuh"

namespace auxmc_gpu {

__host__ __device__ inline int filter_smem_doubles(int dx, int dy) {
  const int W = dx > dy ? dx : dy;
  return 4 * dx + 3 * W + 4 * dx * dx + 3 * dy * dx + 3 * dy * dy + 8;
}

// Per step the model blocks F, Q, H, R are staged into shared memory with
// coalesced loads (the symmetrizations then run on shared memory), so every
// product reads shared operands only.
template <bool BLOCK>
__global__ void k_filter_seq(DevModel m, const double* __restrict__ obs, int B,
                             double* pred_mean, double* pred_cov, double* filt_mean,
                             double* filt_cov, double* log_marginal, int* status) {
  extern __shared__ double smem[];
  const int dx = m.dx, dy = m.dy, T = m.T;
  const int W = dx > dy ? dx : dy;
  const int per = filter_smem_doubles(dx, dy);
  Grp g = BLOCK ? block_group() : warp_group();
  const int gid = BLOCK ? 0 : (threadIdx.x >> 5);
  const int gpb = BLOCK ? 1 : (blockDim.x >> 5);
  double* sm = smem + (size_t)gid * per;
  double* mm = sm;
  double* mp = mm + dx;
  double* v = mp + dx;
  double* innov = v + W;
  double* v2 = innov + W;
  double* p = v2 + W;
  double* tmp = p + dx * dx;   // tmp, a, work contiguous: also the factor scratch
  double* a = tmp + dx * dx;   // F during the prediction
  double* work = a + dx * dx;  // Qs during the prediction
  double* Hs = work + dx * dx;
  double* hp = Hs + dy * dx;
  double* X = hp + dy * dx;
  double* S = X + dy * dx;
  double* L = S + dy * dy;     // raw R while staging
  double* scr = L + dy * dy;   // Rs
  double* red = scr + dy * dy;
  // factor scratch: dy*dy doubles (warp groups: jitter matrix) or the inverted
  // diagonal blocks (CTA groups, dy >= 16); tmp..work when it fits, else Rs
  const bool fits = dy * dy <= 3 * dx * dx && dinv_doubles(dy) <= dx * dx;
  double* fscr = fits ? tmp : scr;
  int* flag = reinterpret_cast<int*>(red + 2);
  const int ddx = dx * dx;
  for (int b = blockIdx.x * gpb + gid; b < B; b += gridDim.x * gpb) {
    const double* y_all = obs + (size_t)b * (T + 1) * dy;
    double* pm_out = pred_mean + (size_t)b * (T + 1) * dx;
    double* pc_out = pred_cov + (size_t)b * (T + 1) * ddx;
    double* fm_out = filt_mean + (size_t)b * (T + 1) * dx;
    double* fc_out = filt_cov + (size_t)b * (T + 1) * ddx;
    double ll = 0.0;
    int st = 0;
    for (int i = g.lane; i < dx; i += g.size) mm[i] = m.m0[i];
    g_copy(g, ddx, m.P0, p);
    g.sync();
    g_symm(g, dx, p);
    g.sync();
    for (int t = 0; t <= T; ++t) {
      if (t > 0) {
        g_copy(g, ddx, m.Ft(t - 1, b), a);
        g_copy(g, ddx, m.Qt(t - 1, b), work);
        g.sync();
        const double* bb = m.bt(t - 1, b);
        for (int i = g.lane; i < dx; i += g.size) {
          double s = 0.0;
          for (int j = 0; j < dx; ++j) s += a[i * dx + j] * mm[j];
          v[i] = s + bb[i];
        }
        g_symm(g, dx, work);
        g_mm(g, dx, dx, dx, a, p, tmp);
        g.sync();
        for (int i = g.lane; i < dx; i += g.size) mm[i] = v[i];
        g_mm_nt(g, dx, dx, dx, tmp, a, p, work);
        g.sync();
        g_symm(g, dx, p);
        g.sync();
      }
      for (int i = g.lane; i < dx; i += g.size) {
        pm_out[(size_t)t * dx + i] = mm[i];
        mp[i] = mm[i];
      }
      for (int i = g.lane; i < ddx; i += g.size) pc_out[(size_t)t * ddx + i] = p[i];
      if (m.observed(t)) {
        const double* c = m.ct(t, b);
        const double* y = y_all + (size_t)t * dy;
        g_copy(g, dy * dx, m.Ht(t, b), Hs);
        g_copy(g, dy * dy, m.Rt(t, b), L);
        g.sync();
        for (int i = g.lane; i < dy; i += g.size) {
          double s = 0.0;
          for (int j = 0; j < dx; ++j) s += Hs[i * dx + j] * mm[j];
          innov[i] = (y[i] - s) - c[i];
          v2[i] = s + c[i];  // H m_pred + c
        }
        g_mm(g, dy, dx, dx, Hs, p, hp);  // H P
        for (int i = g.ty(); i < dy; i += g.ny())  // Rs = symm(R)
          for (int j = g.tx(); j < dy; j += 16)
            scr[i * dy + j] = 0.5 * (L[i * dy + j] + L[j * dy + i]);
        g.sync();
        g_mm_nt(g, dy, dx, dy, hp, Hs, S, scr);
        g.sync();
        g_symm(g, dy, S);
        g.sync();
        st = g_factor_psd(g, dy, S, L, fscr, flag, red);
        if (st) break;
        const bool blk = use_blocked(g, dy) && g.size > 32;
        const double* dinv = blk ? fscr : nullptr;  // inverted diagonal blocks of L
        g_copy(g, dy * dx, hp, X);
        g.sync();
        g_llt_solve(g, dy, L, dx, X, dinv);  // X = S^{-1} H P ; gain = X^T
        if (blk) {
          // warp 0: log-likelihood term (serial triangular solve); the other
          // warps meanwhile update the mean and form a = I - X^T H.
          if (g.lane < 32) {
            ll += w_log_pdf_factored(g.lane, dy, y, v2, L, dinv, v);
          } else {
            const Grp gw = warps_group(1, g.size / 32 - 1, 1);
            for (int j = gw.lane; j < dx; j += gw.size) {
              double s = 0.0;
              for (int i = 0; i < dy; ++i) s += X[i * dx + j] * innov[i];
              mm[j] += s;
            }
            g_mm_tn(gw, dx, dy, dx, X, Hs, a);
            gw.sync();
            for (int i = gw.ty(); i < dx; i += gw.ny())
              for (int j = gw.tx(); j < dx; j += 16)
                a[i * dx + j] = (i == j ? 1.0 : 0.0) - a[i * dx + j];
          }
          g.sync();
        } else {
          // m += X^T innov
          for (int j = g.lane; j < dx; j += g.size) {
            double s = 0.0;
            for (int i = 0; i < dy; ++i) s += X[i * dx + j] * innov[i];
            mm[j] += s;
          }
          // a = I - X^T H
          g_mm_tn(g, dx, dy, dx, X, Hs, a);
          g.sync();
          for (int i = g.ty(); i < dx; i += g.ny())
            for (int j = g.tx(); j < dx; j += 16) a[i * dx + j] = (i == j ? 1.0 : 0.0) - a[i * dx + j];
          g.sync();
        }
        if (fscr == scr) {  // factor scratch overlapped Rs: restage it
          g_copy(g, dy * dy, m.Rt(t, b), S);
          g.sync();
          for (int i = g.ty(); i < dy; i += g.ny())
            for (int j = g.tx(); j < dy; j += 16)
              scr[i * dy + j] = 0.5 * (S[i * dy + j] + S[j * dy + i]);
          g.sync();
        }
        g_mm(g, dx, dx, dx, a, p, tmp);       // a p
        g_mm_tn(g, dx, dy, dy, X, scr, hp);   // X^T R  (dx×dy), reuses hp
        g.sync();
        g_mm_nt(g, dx, dx, dx, tmp, a, work); // a p a^T
        g_mm(g, dx, dy, dx, hp, X, p);        // X^T R X
        g.sync();
        for (int i = g.lane; i < ddx; i += g.size) p[i] = work[i] + p[i];
        g.sync();
        g_symm(g, dx, p);
        g.sync();
        if (!blk) ll += g_log_pdf_factored(g, dy, y, v2, L, innov, red);
      }
      for (int i = g.lane; i < dx; i += g.size) fm_out[(size_t)t * dx + i] = mm[i];
      for (int i = g.lane; i < ddx; i += g.size) fc_out[(size_t)t * ddx + i] = p[i];
      g.sync();
    }
    if (g.lane == 0) {
      log_marginal[b] = ll;
      status[b] = st;
    }
    g.sync();
  }
}

// ---------------------------------------------------------------------------
// k_filter_cta: the CTA-group filter for large dims (dx > 16 or dy > 16), laid
// out to fit two CTAs per SM (one sequence each), so one sequence's serial
// phases (diagonal-block factorizations, triangular-solve steps) overlap the
// other's tensor-core products.  The innovation covariance is factored in
// place; its symmetrized R is restaged from global memory where needed.  The
// jitter ladder of factor_psd (gauss.cpp:26-35) rebuilds S and retries with
// + eps*s*I, as the reference does.
struct CtaFilterLayout {
  int dx, dy, W;
  int o_mm, o_v, o_innov, o_v2, o_p, o_tmp, o_a, o_Hs, o_X, o_SL, o_work, o_dinv, o_red, total;
  __host__ __device__ CtaFilterLayout(int dx_, int dy_) : dx(dx_), dy(dy_) {
    W = dx > dy ? dx : dy;
    const int ddx = dx * dx, ddy = dy * dy;
    int o = 0;
    o_mm = o; o += (dx + 1) & ~1;
    o_v = o; o += (W + 1) & ~1;
    o_innov = o; o += (W + 1) & ~1;
    o_v2 = o; o += (W + 1) & ~1;
    o_p = o; o += ddx;
    o_tmp = o; o += ddx;
    o_a = o; o += ddx;
    o_Hs = o; o += dy * dx;
    o_X = o; o += dy * dx;
    o_SL = o; o += ddy;
    // Qs / (a p a^T) need dx*dx: the S/L region when large enough
    if (ddy >= ddx) { o_work = o_SL; } else { o_work = o; o += ddx; }
    // inverted diagonal blocks of L live in tmp when they fit
    if (dinv_doubles(dy) <= ddx) { o_dinv = o_tmp; } else { o_dinv = o; o += dinv_doubles(dy); }
    o_red = o; o += 4;
    total = o;
  }
};

__global__ void __launch_bounds__(256, 2)
k_filter_cta(DevModel m, const double* __restrict__ obs, int B, double* pred_mean,
             double* pred_cov, double* filt_mean, double* filt_cov, double* log_marginal,
             int* status) {
  extern __shared__ double smem[];
  const int dx = m.dx, dy = m.dy, T = m.T;
  const CtaFilterLayout lo(dx, dy);
  const Grp g = block_group();
  double* mm = smem + lo.o_mm;
  double* v = smem + lo.o_v;
  double* innov = smem + lo.o_innov;
  double* v2 = smem + lo.o_v2;
  double* p = smem + lo.o_p;
  double* tmp = smem + lo.o_tmp;
  double* a = smem + lo.o_a;
  double* Hs = smem + lo.o_Hs;
  double* X = smem + lo.o_X;
  double* SL = smem + lo.o_SL;
  double* work = smem + lo.o_work;
  double* dinv = smem + lo.o_dinv;
  double* red = smem + lo.o_red;
  int* flag = reinterpret_cast<int*>(red + 2);
  const int ddx = dx * dx;
  const bool blk = dy >= 16;
  for (int b = blockIdx.x; b < B; b += gridDim.x) {
    const double* y_all = obs + (size_t)b * (T + 1) * dy;
    double* pm_out = pred_mean + (size_t)b * (T + 1) * dx;
    double* pc_out = pred_cov + (size_t)b * (T + 1) * ddx;
    double* fm_out = filt_mean + (size_t)b * (T + 1) * dx;
    double* fc_out = filt_cov + (size_t)b * (T + 1) * ddx;
    double ll = 0.0;
    int st = 0;
    for (int i = g.lane; i < dx; i += g.size) mm[i] = m.m0[i];
    g_copy(g, ddx, m.P0, p);
    g.sync();
    g_symm(g, dx, p);
    g.sync();
    for (int t = 0; t <= T; ++t) {
      if (t > 0) {  // predict: m = F m + b, P = symm(F P F^T + symm(Q))
        g_copy(g, ddx, m.Ft(t - 1, b), a);
        g_copy(g, ddx, m.Qt(t - 1, b), work);
        g.sync();
        g_mv4<false>(g, dx, dx, a, dx, mm, v, m.bt(t - 1, b));
        g_symm(g, dx, work);
        g_mm(g, dx, dx, dx, a, p, tmp);
        g.sync();
        for (int i = g.lane; i < dx; i += g.size) mm[i] = v[i];
        g_mm_nt(g, dx, dx, dx, tmp, a, p, work);
        g.sync();
        g_symm(g, dx, p);
        g.sync();
      }
      for (int i = g.lane; i < dx; i += g.size) pm_out[(size_t)t * dx + i] = mm[i];
      for (int i = g.lane; i < ddx; i += g.size) pc_out[(size_t)t * ddx + i] = p[i];
      if (m.observed(t)) {
        const double* c = m.ct(t, b);
        const double* y = y_all + (size_t)t * dy;
        const double* R = m.Rt(t, b);
        g_copy(g, dy * dx, m.Ht(t, b), Hs);
        g.sync();
        {  // innovation v = (y - H m) - c and the log-pdf mean H m + c
          const int q = g.lane & 3, rows = g.size >> 2;
          for (int i0 = 0; i0 < dy; i0 += rows) {
            const int i = i0 + (g.lane >> 2);
            double s = 0.0;
            if (i < dy)
              for (int j = q; j < dx; j += 4) s += Hs[i * dx + j] * mm[j];
            s = quad_sum(s);
            if (i < dy && q == 0) {
              innov[i] = (y[i] - s) - c[i];
              v2[i] = s + c[i];
            }
          }
        }
        g_mm(g, dy, dx, dx, Hs, p, X);  // H P (solved in place below)
        double jit = 0.0;
        bool ok = false;
        for (int attempt = 0; attempt < 3 && !ok; ++attempt) {
          // S = symm(H P H^T + symm(R)) [+ eps*s*I]
          g_copy(g, dy * dy, R, SL);
          g.sync();
          g_symm(g, dy, SL);
          g.sync();
          g_mm_nt(g, dy, dx, dy, X, Hs, SL, SL);
          g.sync();
          g_symm(g, dy, SL);
          g.sync();
          if (attempt > 0) {
            if (attempt == 1) {  // jitter scale (gauss.cpp:20-24) from the rebuilt S
              if (g.lane == 0) {
                double tr = 0.0;
                for (int i = 0; i < dy; ++i) tr += SL[i * dy + i];
                double sc = tr / static_cast<double>(dy);
                if (sc <= 0.0) {
                  double mx = 0.0;
                  for (int i = 0; i < dy * dy; ++i) mx = fabs(SL[i]) > mx ? fabs(SL[i]) : mx;
                  sc = mx;
                }
                *red = sc;
              }
              g.sync();
              jit = *red;
              g.sync();
            }
            const double eps = attempt == 1 ? 1e-10 : 1e-8;
            for (int i = g.lane; i < dy; i += g.size) SL[i * dy + i] = SL[i * dy + i] + (eps * jit) * 1.0;
            g.sync();
          }
          // lower triangle in place, upper zeroed
          for (int i = g.ty(); i < dy; i += g.ny())
            for (int j = i + 1 + g.tx(); j < dy; j += 16) SL[i * dy + j] = 0.0;
          g.sync();
          ok = blk ? g_llt_blocked(g, dy, SL, flag, dinv) : g_llt(g, dy, SL, SL, flag);
        }
        if (!ok) {
          st = 2;
          break;
        }
        g_llt_solve(g, dy, SL, dx, X, blk ? dinv : nullptr);  // X = S^{-1} H P ; gain = X^T
        if (blk) {
          // warp 0: log-likelihood term; the other warps: mean update and a = I - X^T H
          if (g.lane < 32) {
            ll += w_log_pdf_factored(g.lane, dy, y, v2, SL, dinv, v);
          } else {
            const Grp gw = warps_group(1, g.size / 32 - 1, 1);
            g_mv4<true>(gw, dx, dy, X, dx, innov, mm, mm);
            g_mm_tn(gw, dx, dy, dx, X, Hs, a);
            gw.sync();
            for (int i = gw.ty(); i < dx; i += gw.ny())
              for (int j = gw.tx(); j < dx; j += 16)
                a[i * dx + j] = (i == j ? 1.0 : 0.0) - a[i * dx + j];
          }
          g.sync();
        } else {
          ll += g_log_pdf_factored(g, dy, y, v2, SL, v, red);
          g_mv4<true>(g, dx, dy, X, dx, innov, mm, mm);
          g_mm_tn(g, dx, dy, dx, X, Hs, a);
          g.sync();
          for (int i = g.ty(); i < dx; i += g.ny())
            for (int j = g.tx(); j < dx; j += 16) a[i * dx + j] = (i == j ? 1.0 : 0.0) - a[i * dx + j];
          g.sync();
        }
        // Joseph form P = symm(a P a^T + X^T Rs X); Rs restaged into SL
        g_copy(g, dy * dy, R, SL);
        g_mm(g, dx, dx, dx, a, p, tmp);  // a P
        g.sync();
        g_symm(g, dy, SL);
        g.sync();
        g_mm_tn(g, dx, dy, dy, X, SL, Hs);  // X^T Rs (dx×dy) into the H slot
        g.sync();
        g_mm_nt(g, dx, dx, dx, tmp, a, work);  // a P a^T (work may alias SL: Rs consumed)
        g_mm(g, dx, dy, dx, Hs, X, p);         // X^T Rs X
        g.sync();
        for (int i = g.lane; i < ddx; i += g.size) p[i] = work[i] + p[i];
        g.sync();
        g_symm(g, dx, p);
        g.sync();
      }
      for (int i = g.lane; i < dx; i += g.size) fm_out[(size_t)t * dx + i] = mm[i];
      for (int i = g.lane; i < ddx; i += g.size) fc_out[(size_t)t * ddx + i] = p[i];
      g.sync();
    }
    if (g.lane == 0) {
      log_marginal[b] = ll;
      status[b] = st;
    }
    g.sync();
  }
}

// Register path for small dims: one thread per sequence, state and covariance
// in registers (D <= 6, observation rows <= DY).  Same operation order as the
// group kernel (lgssm.cpp:73-112).
template <int D, int DY>
__global__ void k_filter_reg(DevModel m, const double* __restrict__ obs, int B, double* pred_mean,
                             double* pred_cov, double* filt_mean, double* filt_cov,
                             double* log_marginal, int* status) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const int T = m.T, dy = m.dy;
  constexpr int DD = D * D;
  double mm[D], p[DD];
#pragma unroll
  for (int i = 0; i < D; ++i) mm[i] = m.m0[i];
#pragma unroll
  for (int i = 0; i < DD; ++i) p[i] = 0.5 * (m.P0[(i / D) * D + i % D] + m.P0[(i % D) * D + i / D]);
  double ll = 0.0;
  int st = 0;
  const double* y_all = obs + (size_t)b * (T + 1) * dy;
  for (int t = 0; t <= T && !st; ++t) {
    if (t > 0) {
      const double* F = m.Ft(t - 1, b);
      const double* bb = m.bt(t - 1, b);
      const double* Q = m.Qt(t - 1, b);
      double Fr[DD], v[D], tmp[DD];
#pragma unroll
      for (int i = 0; i < DD; ++i) Fr[i] = F[i];
#pragma unroll
      for (int i = 0; i < D; ++i) {
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < D; ++j) s += Fr[i * D + j] * mm[j];
        v[i] = s + bb[i];
      }
#pragma unroll
      for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) {
          double s = 0.0;
#pragma unroll
          for (int k = 0; k < D; ++k) s += Fr[i * D + k] * p[k * D + j];
          tmp[i * D + j] = s;
        }
#pragma unroll
      for (int i = 0; i < D; ++i) {
        mm[i] = v[i];
#pragma unroll
        for (int j = 0; j < D; ++j) {
          double s = 0.0;
#pragma unroll
          for (int k = 0; k < D; ++k) s += tmp[i * D + k] * Fr[j * D + k];
          p[i * D + j] = s + 0.5 * (Q[i * D + j] + Q[j * D + i]);
        }
      }
#pragma unroll
      for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = i + 1; j < D; ++j) {
          const double s = 0.5 * (p[i * D + j] + p[j * D + i]);
          p[i * D + j] = s;
          p[j * D + i] = s;
        }
    }
    double* pmo = pred_mean + ((size_t)b * (T + 1) + t) * D;
    double* pco = pred_cov + ((size_t)b * (T + 1) + t) * DD;
#pragma unroll
    for (int i = 0; i < D; ++i) pmo[i] = mm[i];
#pragma unroll
    for (int i = 0; i < DD; ++i) pco[i] = p[i];
    if (dy > 0 && m.observed(t)) {
      const double* H = m.Ht(t, b);
      const double* c = m.ct(t, b);
      const double* R = m.Rt(t, b);
      const double* y = y_all + (size_t)t * dy;
      double innov[DY], v2[DY], hp[DY * D], S[DY * DY], L[DY * DY], X[DY * D];
      for (int i = 0; i < dy; ++i) {
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < D; ++j) s += H[i * D + j] * mm[j];
        innov[i] = (y[i] - s) - c[i];
        v2[i] = s + c[i];
#pragma unroll
        for (int j = 0; j < D; ++j) {
          double a = 0.0;
#pragma unroll
          for (int k = 0; k < D; ++k) a += H[i * D + k] * p[k * D + j];
          hp[i * D + j] = a;
        }
      }
      for (int i = 0; i < dy; ++i)
        for (int j = 0; j < dy; ++j) {
          double s = 0.0;
#pragma unroll
          for (int k = 0; k < D; ++k) s += hp[i * D + k] * H[j * D + k];
          S[i * dy + j] = s + 0.5 * (R[i * dy + j] + R[j * dy + i]);
        }
      for (int i = 0; i < dy; ++i)
        for (int j = i + 1; j < dy; ++j) {
          const double s = 0.5 * (S[i * dy + j] + S[j * dy + i]);
          S[i * dy + j] = s;
          S[j * dy + i] = s;
        }
      // factor_psd(S) (gauss.cpp:26-35)
      bool ok = false;
      for (int pass = 0; pass < 3 && !ok; ++pass) {
        double jit = 0.0;
        if (pass > 0) {
          double tr = 0.0;
          for (int i = 0; i < dy; ++i) tr += S[i * dy + i];
          double sc = tr / dy;
          if (sc <= 0.0) {
            sc = 0.0;
            for (int i = 0; i < dy * dy; ++i) sc = fabs(S[i]) > sc ? fabs(S[i]) : sc;
          }
          jit = (pass == 1 ? 1e-10 : 1e-8) * sc;
        }
        ok = true;
        for (int k = 0; k < dy && ok; ++k) {
          double x = S[k * dy + k] + (pass ? jit * 1.0 : 0.0);
          for (int j = 0; j < k; ++j) x -= L[k * dy + j] * L[k * dy + j];
          if (x <= 0.0) {
            ok = false;
            break;
          }
          x = sqrt(x);
          L[k * dy + k] = x;
          for (int i = k + 1; i < dy; ++i) {
            double s = S[i * dy + k];
            for (int j = 0; j < k; ++j) s -= L[i * dy + j] * L[k * dy + j];
            L[i * dy + k] = s / x;
          }
          for (int j = k + 1; j < dy; ++j) L[k * dy + j] = 0.0;
        }
      }
      if (!ok) {
        st = AUXMC_E_FACTOR;
        break;
      }
      // X = S^{-1} H P (dy×D)
      for (int col = 0; col < D; ++col) {
        for (int i = 0; i < dy; ++i) {
          double s = hp[i * D + col];
          for (int j = 0; j < i; ++j) s -= L[i * dy + j] * X[j * D + col];
          X[i * D + col] = s / L[i * dy + i];
        }
        for (int i = dy - 1; i >= 0; --i) {
          double s = X[i * D + col];
          for (int j = i + 1; j < dy; ++j) s -= L[j * dy + i] * X[j * D + col];
          X[i * D + col] = s / L[i * dy + i];
        }
      }
      double a[DD], tmp[DD], gr[D * DY];
#pragma unroll
      for (int j = 0; j < D; ++j) {
        double s = 0.0;
        for (int i = 0; i < dy; ++i) s += X[i * D + j] * innov[i];
        mm[j] += s;
      }
#pragma unroll
      for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) {
          double s = 0.0;
          for (int k = 0; k < dy; ++k) s += X[k * D + i] * H[k * D + j];
          a[i * D + j] = (i == j ? 1.0 : 0.0) - s;
        }
#pragma unroll
      for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) {
          double s = 0.0;
#pragma unroll
          for (int k = 0; k < D; ++k) s += a[i * D + k] * p[k * D + j];
          tmp[i * D + j] = s;
        }
      for (int i = 0; i < D; ++i)
        for (int j = 0; j < dy; ++j) {
          double s = 0.0;
          for (int k = 0; k < dy; ++k) s += X[k * D + i] * (0.5 * (R[k * dy + j] + R[j * dy + k]));
          gr[i * DY + j] = s;
        }
#pragma unroll
      for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) {
          double s = 0.0, s2 = 0.0;
#pragma unroll
          for (int k = 0; k < D; ++k) s += tmp[i * D + k] * a[j * D + k];
          for (int k = 0; k < dy; ++k) s2 += gr[i * DY + k] * X[k * D + j];
          p[i * D + j] = s + s2;
        }
#pragma unroll
      for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = i + 1; j < D; ++j) {
          const double s = 0.5 * (p[i * D + j] + p[j * D + i]);
          p[i * D + j] = s;
          p[j * D + i] = s;
        }
      // log N(y; H m_pred + c, S) with the same factor
      double sq = 0.0, ld = 0.0, z[DY];
      for (int i = 0; i < dy; ++i) {
        double s = y[i] - v2[i];
        for (int j = 0; j < i; ++j) s -= L[i * dy + j] * z[j];
        z[i] = s / L[i * dy + i];
        sq += z[i] * z[i];
      }
      for (int i = 0; i < dy; ++i) ld += log(L[i * dy + i]);
      ll += -0.5 * (dy * kLog2Pi + sq) - ld;
    }
    double* fmo = filt_mean + ((size_t)b * (T + 1) + t) * D;
    double* fco = filt_cov + ((size_t)b * (T + 1) + t) * DD;
#pragma unroll
    for (int i = 0; i < D; ++i) fmo[i] = mm[i];
#pragma unroll
    for (int i = 0; i < DD; ++i) fco[i] = p[i];
  }
  log_marginal[b] = ll;
  status[b] = st;
}

int launch_filter_seq(const DevModel& dm, const double* obs, int B, auxmc_filter_result* out,
                      int* status, cudaStream_t stream) {
  if (dm.dy <= 8 && dm.dx <= 6) {
    const int grid = (B + 63) / 64;
#define FCASE(D)                                                                              \
  case D:                                                                                     \
    AUXMC_LAUNCH((k_filter_reg<D, 8>), grid, 64, 0, stream, dm, obs, B, out->pred_mean,       \
                 out->pred_cov, out->filt_mean, out->filt_cov, out->log_marginal, status);    \
    return AUXMC_OK;
    switch (dm.dx) { FCASE(1) FCASE(2) FCASE(3) FCASE(4) FCASE(5) FCASE(6) }
#undef FCASE
  }
  const int per = filter_smem_doubles(dm.dx, dm.dy);
  const bool block = (dm.dx > 16 || dm.dy > 16);
  if (block) {
    const size_t smem = sizeof(double) * CtaFilterLayout(dm.dx, dm.dy).total;
    if (smem > 227 * 1024) return AUXMC_E_DIM;
    AUXMC_CUDA_TRY(cudaFuncSetAttribute(k_filter_cta, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)smem));
    AUXMC_LAUNCH(k_filter_cta, B, 256, smem, stream, dm, obs, B, out->pred_mean, out->pred_cov,
                 out->filt_mean, out->filt_cov, out->log_marginal, status);
  } else {
    const int warps = 4;
    const size_t smem = sizeof(double) * per * warps;
    AUXMC_CUDA_TRY(cudaFuncSetAttribute(k_filter_seq<false>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int grid = (B + warps - 1) / warps;
    AUXMC_LAUNCH(k_filter_seq<false>, grid, 32 * warps, smem, stream, dm, obs, B, out->pred_mean,
                 out->pred_cov, out->filt_mean, out->filt_cov, out->log_marginal, status);
  }
  return AUXMC_OK;
}

}  // namespace auxmc_gpu

