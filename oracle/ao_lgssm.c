/* ao_lgssm.c — sequential Kalman filter, backward sampler, path density,
 * RTS smoother and dense oracle; restates proj/src/lgssm.cpp.
 * TEST INFRASTRUCTURE (parity oracle); see auxmc_oracle.h. */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "auxmc_oracle.h"
#include "ao_internal.h"

/* lgssm.cpp:20-71: owned copy with symmetrized P0, Q, R */
int ao_lgssm_normalize(const ao_lgssm* in, ao_lgssm* out) {
  *out = *in;
  const int dx = in->dx, dy = in->dy;
  if (in->T < 0) return AO_E_DIM;
  double* P0 = (double*)malloc(sizeof(double) * dx * dx);
  memcpy(P0, in->P0, sizeof(double) * dx * dx);
  ao_symm(dx, P0);
  double* Q = (double*)malloc(sizeof(double) * dx * dx * in->nQ);
  memcpy(Q, in->Q, sizeof(double) * dx * dx * in->nQ);
  for (int i = 0; i < in->nQ; ++i) ao_symm(dx, Q + (size_t)i * dx * dx);
  double* R = (double*)malloc(sizeof(double) * dy * dy * (in->nR > 0 ? in->nR : 1));
  if (in->nR > 0) memcpy(R, in->R, sizeof(double) * dy * dy * in->nR);
  for (int i = 0; i < in->nR; ++i) ao_symm(dy, R + (size_t)i * dy * dy);
  out->P0 = P0;
  out->Q = Q;
  out->R = R;
  return AO_OK;
}

void ao_lgssm_free(ao_lgssm* m) {
  free((void*)m->P0);
  free((void*)m->Q);
  free((void*)m->R);
  m->P0 = m->Q = m->R = NULL;
}

/* lgssm.cpp:73-112 */
int ao_kalman_filter(const ao_lgssm* m, const double* obs, ao_filter* fr) {
  const int T = m->T, dx = m->dx, dy = m->dy;
  const int W = dx > dy ? dx : dy;
  double* buf = (double*)malloc(sizeof(double) * (8 * W * W + 8 * W));
  double* mm = buf;
  double* p = mm + W;
  double* tmp = p + W * W;
  double* s = tmp + W * W;
  double* hp = s + W * W;
  double* x = hp + W * W;      /* S^{-1} H P, dy×dx */
  double* a = x + W * W;
  double* work = a + W * W;
  double* innov = work + W * W;
  double* v = innov + W;
  int status = AO_OK;
  fr->log_marginal = 0.0;
  memcpy(mm, m->m0, sizeof(double) * dx);
  memcpy(p, m->P0, sizeof(double) * dx * dx);
  for (int t = 0; t <= T && status == AO_OK; ++t) {
    if (t > 0) {
      const double* F = AO_F(m, t - 1);
      ao_matvec(dx, dx, F, mm, v);
      const double* b = AO_B(m, t - 1);
      for (int i = 0; i < dx; ++i) mm[i] = v[i] + b[i];
      ao_sandwich(dx, dx, F, p, tmp, work);
      const double* Q = AO_Q(m, t - 1);
      for (int i = 0; i < dx * dx; ++i) p[i] = tmp[i] + Q[i];
      ao_symm(dx, p);
    }
    memcpy(fr->pred_mean + (size_t)t * dx, mm, sizeof(double) * dx);
    memcpy(fr->pred_cov + (size_t)t * dx * dx, p, sizeof(double) * dx * dx);
    if (AO_OBSERVED(m, t)) {
      const double* H = AO_H(m, t);
      const double* c = AO_C(m, t);
      const double* R = AO_R(m, t);
      const double* y = obs + (size_t)t * dy;
      ao_matvec(dy, dx, H, mm, v);
      for (int i = 0; i < dy; ++i) innov[i] = (y[i] - v[i]) - c[i];
      ao_sandwich(dy, dx, H, p, s, work);
      for (int i = 0; i < dy * dy; ++i) s[i] += R[i];
      ao_symm(dy, s);
      ao_matmul(dy, dx, dx, H, p, hp);
      status = ao_solve_spd(dy, s, dx, hp, x); /* x = S^{-1} H P, gain = x^T */
      if (status != AO_OK) break;
      /* m += gain innov, gain = x^T (dx×dy) */
      ao_matvec_t(dy, dx, x, innov, v);
      for (int i = 0; i < dx; ++i) mm[i] += v[i];
      /* a = I - gain H */
      ao_matmul_at(dx, dy, dx, x, H, a);
      for (int i = 0; i < dx * dx; ++i) a[i] = -a[i];
      for (int i = 0; i < dx; ++i) a[i * dx + i] += 1.0;
      ao_sandwich(dx, dx, a, p, tmp, work);
      /* gain R gain^T = x^T R x */
      double* gr = hp; /* reuse: x^T R (dx×dy) */
      ao_matmul_at(dx, dy, dy, x, R, gr);
      ao_matmul(dx, dy, dx, gr, x, work);
      for (int i = 0; i < dx * dx; ++i) p[i] = tmp[i] + work[i];
      ao_symm(dx, p);
      /* log N(y; H m_pred + c, S) */
      ao_matvec(dy, dx, H, fr->pred_mean + (size_t)t * dx, v);
      for (int i = 0; i < dy; ++i) v[i] += c[i];
      fr->log_marginal += ao_log_pdf(dy, y, v, s, &status);
    }
    memcpy(fr->filt_mean + (size_t)t * dx, mm, sizeof(double) * dx);
    memcpy(fr->filt_cov + (size_t)t * dx * dx, p, sizeof(double) * dx * dx);
  }
  free(buf);
  return status;
}

/* lgssm.cpp:129-149 */
int ao_backward_step(const ao_lgssm* m, const ao_filter* fr, int t, double* gain,
                     double* offset, double* cov) {
  const int dx = m->dx;
  const double* F = AO_F(m, t);
  const double* P = fr->filt_cov + (size_t)t * dx * dx;
  const double* S = fr->pred_cov + (size_t)(t + 1) * dx * dx;
  double* buf = (double*)malloc(sizeof(double) * (4 * dx * dx + 2 * dx));
  double* cross = buf;         /* P F^T */
  double* crossT = cross + dx * dx;
  double* a = crossT + dx * dx;
  double* work = a + dx * dx;
  double* v = work + dx * dx;
  double* w = v + dx;
  int status = AO_OK;
  ao_matmul_bt(dx, dx, dx, P, F, cross);
  if (ao_all_zero(dx * dx, cross)) {
    memset(gain, 0, sizeof(double) * dx * dx);
  } else {
    ao_transpose(dx, dx, cross, crossT);
    status = ao_solve_spd(dx, S, dx, crossT, a); /* a = S^{-1} cross^T; gain = a^T */
    if (status != AO_OK) {
      free(buf);
      return status;
    }
    ao_transpose(dx, dx, a, gain);
  }
  /* offset = m_t - gain (F m_t + b_t) */
  const double* mt = fr->filt_mean + (size_t)t * dx;
  ao_matvec(dx, dx, F, mt, v);
  const double* b = AO_B(m, t);
  for (int i = 0; i < dx; ++i) v[i] += b[i];
  ao_matvec(dx, dx, gain, v, w);
  for (int i = 0; i < dx; ++i) offset[i] = mt[i] - w[i];
  /* Joseph: a = I - G F; cov = symm(a P a^T + G Q G^T) */
  ao_matmul(dx, dx, dx, gain, F, a);
  for (int i = 0; i < dx * dx; ++i) a[i] = -a[i];
  for (int i = 0; i < dx; ++i) a[i * dx + i] += 1.0;
  ao_sandwich(dx, dx, a, P, cov, work);
  ao_sandwich(dx, dx, gain, AO_Q(m, t), a, work);
  for (int i = 0; i < dx * dx; ++i) cov[i] += a[i];
  ao_symm(dx, cov);
  free(buf);
  return AO_OK;
}

/* lgssm.cpp:151-172 */
int ao_backward_sample(const ao_lgssm* m, const ao_filter* fr, ao_noise* noise, double* traj) {
  const int T = m->T, dx = m->dx;
  double* buf = (double*)malloc(sizeof(double) * (4 * dx * dx + 4 * dx));
  double* l = buf;
  double* g = l + dx * dx;
  double* cov = g + dx * dx;
  double* off = cov + dx * dx;
  double* xi = off + dx;
  double* v = xi + dx;
  int st = ao_chol_psd(dx, fr->filt_cov + (size_t)T * dx * dx, l);
  if (st != AO_OK) goto done;
  ao_noise_normal(noise, AO_L_TERMINAL_DRAW, 0, dx, xi);
  ao_matvec(dx, dx, l, xi, v);
  for (int i = 0; i < dx; ++i) traj[(size_t)T * dx + i] = fr->filt_mean[(size_t)T * dx + i] + v[i];
  for (int t = T - 1; t >= 0; --t) {
    st = ao_backward_step(m, fr, t, g, off, cov);
    if (st != AO_OK) goto done;
    st = ao_chol_psd(dx, cov, l);
    if (st != AO_OK) goto done;
    ao_noise_normal(noise, AO_L_BACKWARD_NOISE, (uint64_t)t, dx, xi);
    ao_matvec(dx, dx, l, xi, v);
    for (int i = 0; i < dx; ++i) off[i] += v[i];  /* shifted = offset + L xi */
    ao_matvec(dx, dx, g, traj + (size_t)(t + 1) * dx, v);
    for (int i = 0; i < dx; ++i) traj[(size_t)t * dx + i] = v[i] + off[i];
  }
done:
  free(buf);
  return st;
}

/* lgssm.cpp:114-127 */
int ao_rts_smoother(const ao_lgssm* m, const ao_filter* fr, double* mean, double* cov) {
  const int T = m->T, dx = m->dx;
  double* buf = (double*)malloc(sizeof(double) * (5 * dx * dx + 2 * dx));
  double* g = buf;
  double* bc = g + dx * dx;
  double* work = bc + dx * dx;
  double* tmp = work + dx * dx;
  double* off = tmp + dx * dx;
  double* v = off + dx;
  int st = AO_OK;
  memcpy(mean + (size_t)T * dx, fr->filt_mean + (size_t)T * dx, sizeof(double) * dx);
  memcpy(cov + (size_t)T * dx * dx, fr->filt_cov + (size_t)T * dx * dx, sizeof(double) * dx * dx);
  ao_symm(dx, cov + (size_t)T * dx * dx);
  for (int t = T - 1; t >= 0 && st == AO_OK; --t) {
    st = ao_backward_step(m, fr, t, g, off, bc);
    ao_matvec(dx, dx, g, mean + (size_t)(t + 1) * dx, v);
    for (int i = 0; i < dx; ++i) mean[(size_t)t * dx + i] = v[i] + off[i];
    ao_sandwich(dx, dx, g, cov + (size_t)(t + 1) * dx * dx, tmp, work);
    double* c = cov + (size_t)t * dx * dx;
    for (int i = 0; i < dx * dx; ++i) c[i] = bc[i] + tmp[i];
    ao_symm(dx, c);
  }
  free(buf);
  return st;
}

/* lgssm.cpp:179-199 */
double ao_path_logpdf(const ao_lgssm* m, const double* obs, const double* traj,
                      const ao_filter* fr, int* status) {
  const int T = m->T, dx = m->dx, dy = m->dy;
  const int W = dx > dy ? dx : dy;
  double* v = (double*)malloc(sizeof(double) * W);
  int st = AO_OK;
  double lp = ao_log_pdf(dx, traj, m->m0, m->P0, &st);
  for (int t = 0; t < T; ++t) {
    ao_matvec(dx, dx, AO_F(m, t), traj + (size_t)t * dx, v);
    const double* b = AO_B(m, t);
    for (int i = 0; i < dx; ++i) v[i] += b[i];
    lp += ao_log_pdf(dx, traj + (size_t)(t + 1) * dx, v, AO_Q(m, t), &st);
  }
  for (int t = 0; t <= T; ++t) {
    if (!AO_OBSERVED(m, t)) continue;
    ao_matvec(dy, dx, AO_H(m, t), traj + (size_t)t * dx, v);
    const double* c = AO_C(m, t);
    for (int i = 0; i < dy; ++i) v[i] += c[i];
    lp += ao_log_pdf(dy, obs + (size_t)t * dy, v, AO_R(m, t), &st);
  }
  free(v);
  if (status) *status = st;
  return lp - fr->log_marginal;
}

/* lgssm.cpp:201-261 — Gaussian conditioning over the stacked path (test oracle). */
int ao_dense_oracle(const ao_lgssm* m, const double* obs, int cap, double* post_mean,
                    double* post_cov, double* log_evidence) {
  const int T = m->T, dx = m->dx, dy = m->dy;
  const int n = (T + 1) * dx;
  if (n > cap) return AO_E_DIM;
  double* mean = (double*)calloc(n, sizeof(double));
  double* cov = (double*)calloc((size_t)n * n, sizeof(double));
  double* blk = (double*)malloc(sizeof(double) * dx * dx);
  double* blk2 = (double*)malloc(sizeof(double) * dx * dx);
  memcpy(mean, m->m0, sizeof(double) * dx);
  for (int i = 0; i < dx; ++i)
    for (int j = 0; j < dx; ++j) cov[i * n + j] = m->P0[i * dx + j];
  for (int t = 0; t < T; ++t) {
    const double* F = AO_F(m, t);
    ao_matvec(dx, dx, F, mean + t * dx, mean + (t + 1) * dx);
    const double* b = AO_B(m, t);
    for (int i = 0; i < dx; ++i) mean[(t + 1) * dx + i] += b[i];
    for (int s = 0; s <= t; ++s) {
      for (int i = 0; i < dx; ++i)
        for (int j = 0; j < dx; ++j) blk2[i * dx + j] = cov[(t * dx + i) * n + s * dx + j];
      ao_matmul(dx, dx, dx, F, blk2, blk);
      for (int i = 0; i < dx; ++i)
        for (int j = 0; j < dx; ++j) {
          cov[((t + 1) * dx + i) * n + s * dx + j] = blk[i * dx + j];
          cov[(s * dx + j) * n + (t + 1) * dx + i] = blk[i * dx + j];
        }
    }
    for (int i = 0; i < dx; ++i)
      for (int j = 0; j < dx; ++j) blk2[i * dx + j] = cov[(t * dx + i) * n + t * dx + j];
    double* work = (double*)malloc(sizeof(double) * dx * dx);
    ao_sandwich(dx, dx, F, blk2, blk, work);
    free(work);
    const double* Q = AO_Q(m, t);
    for (int i = 0; i < dx; ++i)
      for (int j = 0; j < dx; ++j)
        cov[((t + 1) * dx + i) * n + (t + 1) * dx + j] = blk[i * dx + j] + Q[i * dx + j];
  }
  ao_symm(n, cov);
  int nobs = 0;
  for (int t = 0; t <= T; ++t) nobs += AO_OBSERVED(m, t);
  int st = AO_OK;
  if (nobs == 0 || dy == 0) {
    memcpy(post_mean, mean, sizeof(double) * n);
    memcpy(post_cov, cov, sizeof(double) * n * n);
    *log_evidence = 0.0;
  } else {
    const int ny = nobs * dy;
    double* h = (double*)calloc((size_t)ny * n, sizeof(double));
    double* c = (double*)calloc(ny, sizeof(double));
    double* y = (double*)calloc(ny, sizeof(double));
    double* r = (double*)calloc((size_t)ny * ny, sizeof(double));
    int k = 0;
    for (int t = 0; t <= T; ++t) {
      if (!AO_OBSERVED(m, t)) continue;
      const double* H = AO_H(m, t);
      const double* cc = AO_C(m, t);
      const double* R = AO_R(m, t);
      for (int i = 0; i < dy; ++i) {
        for (int j = 0; j < dx; ++j) h[(k * dy + i) * n + t * dx + j] = H[i * dx + j];
        c[k * dy + i] = cc[i];
        y[k * dy + i] = obs[(size_t)t * dy + i];
        for (int j = 0; j < dy; ++j) r[(k * dy + i) * ny + k * dy + j] = R[i * dy + j];
      }
      ++k;
    }
    double* my = (double*)malloc(sizeof(double) * ny);
    ao_matvec(ny, n, h, mean, my);
    for (int i = 0; i < ny; ++i) my[i] += c[i];
    double* cxy = (double*)malloc(sizeof(double) * n * ny); /* cov h^T */
    ao_matmul_bt(n, n, ny, cov, h, cxy);
    double* cyy = (double*)malloc(sizeof(double) * ny * ny);
    ao_matmul(ny, n, ny, h, cxy, cyy);
    for (int i = 0; i < ny * ny; ++i) cyy[i] += r[i];
    ao_symm(ny, cyy);
    /* condition (gauss.cpp:69-87): gain = cxy cyy^{-1} */
    double* cyxT = (double*)malloc(sizeof(double) * ny * n);
    ao_transpose(n, ny, cxy, cyxT);
    double* sol = (double*)malloc(sizeof(double) * ny * n); /* cyy^{-1} cxy^T */
    st = ao_solve_spd(ny, cyy, n, cyxT, sol);
    double* resid = (double*)malloc(sizeof(double) * ny);
    for (int i = 0; i < ny; ++i) resid[i] = y[i] - my[i];
    for (int i = 0; i < n; ++i) {
      double s = 0.0;
      for (int j = 0; j < ny; ++j) s += sol[j * n + i] * resid[j];
      post_mean[i] = mean[i] + s;
    }
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        double s = 0.0;
        for (int l = 0; l < ny; ++l) s += sol[l * n + i] * cxy[j * ny + l];
        post_cov[i * n + j] = cov[i * n + j] - s;
      }
    ao_symm(n, post_cov);
    *log_evidence = ao_log_pdf(ny, y, my, cyy, &st);
    free(h); free(c); free(y); free(r); free(my); free(cxy); free(cyy); free(cyxT);
    free(sol); free(resid);
  }
  free(mean); free(cov); free(blk); free(blk2);
  return st;
}
