/* ao_models.c — bench models and the GenSSMTarget density; restates
 * proj/src/bench/models.cpp and proj/src/target.cpp.  Lorenz-96 (absent from the
 * reference) follows the Lorenz-63 template models.cpp:70-85, :280-297.
 * TEST INFRASTRUCTURE (parity oracle); see auxmc_oracle.h. */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "auxmc_oracle.h"
#include "ao_internal.h"


/* models.hpp:16-54 defaults (+ Lorenz-96 block) */
void ao_spec_default(ao_spec* s) {
  memset(s, 0, sizeof *s);
  s->kind = AO_KIND_LGSSM;
  s->T = 50;
  s->dx = 2;
  s->dy = 1;
  s->grid = 3;
  s->data_seed = 1;
  s->sv_mu = -1.0; s->sv_phi = 0.9; s->sv_sig2 = 0.1; s->sv_rho = 0.25;
  s->lz_sigma = 10.0; s->lz_rho = 28.0; s->lz_beta = 8.0 / 3.0; s->lz_h = 0.01;
  s->lz_gamma = 2.0; s->lz_obs_var = 1.0;
  s->st_phi = 0.8; s->st_kappa2 = 1.0; s->st_tau2 = 0.3;
  s->g1_phi = 0.8; s->g1_q = 0.09; s->g1_m0 = 0.5; s->g1_p0 = 0.25;
  s->l96_F = 8.0; s->l96_h = 0.01; s->l96_gamma = 1.0; s->l96_obs_var = 1.0;
}

/* models.cpp:144-160 */
int ao_latent_dim(const ao_spec* s) {
  switch (s->kind) {
    case AO_KIND_LGSSM: case AO_KIND_STOCHVOL: case AO_KIND_LORENZ96: return s->dx;
    case AO_KIND_LORENZ63: return 3;
    case AO_KIND_SPATIO: return s->grid * s->grid;
    case AO_KIND_GRID1D: return 1;
  }
  return -1;
}
int ao_obs_dim(const ao_spec* s) {
  switch (s->kind) {
    case AO_KIND_LGSSM: return s->dy;
    case AO_KIND_STOCHVOL: return s->dx;
    case AO_KIND_LORENZ63: return 1;
    case AO_KIND_SPATIO: return s->grid * s->grid;
    case AO_KIND_GRID1D: return 0;
    case AO_KIND_LORENZ96: return (s->dx + 1) / 2;
  }
  return -1;
}

/* models.cpp:39-43 */
static void random_spd(ao_stream* s, int d, double ridge, double* out) {
  double* g = (double*)malloc(sizeof(double) * d * d);
  for (int i = 0; i < d; ++i) ao_normal_vec(s, d, g + i * d);
  ao_matmul_bt(d, d, d, g, g, out);
  for (int i = 0; i < d * d; ++i) out[i] = out[i] / d;
  for (int i = 0; i < d; ++i) out[i * d + i] += ridge;
  free(g);
}

/* models.cpp:51-68 */
int ao_synth_mats(const ao_spec* s, double* m0, double* b, double* P0, double* F, double* Q,
                  double* H, double* R) {
  ao_stream ms = ao_derive(ao_from_seed(s->data_seed), AO_L_PARAM, 0);
  const int dx = s->dx, dy = s->dy;
  for (int i = 0; i < dx; ++i) {
    ao_normal_vec(&ms, dx, F + i * dx);
    for (int j = 0; j < dx; ++j) F[i * dx + j] = F[i * dx + j] / sqrt((double)dx);
  }
  double radius = ao_spectral_radius(dx, F);
  double scale = 0.7 / (radius > 1e-12 ? radius : 1e-12);
  for (int i = 0; i < dx * dx; ++i) F[i] *= scale;
  ao_normal_vec(&ms, dx, b);
  for (int i = 0; i < dx; ++i) b[i] = 0.1 * b[i];
  random_spd(&ms, dx, 0.1, Q);
  ao_normal_vec(&ms, dx, m0);
  random_spd(&ms, dx, 0.1, P0);
  for (int i = 0; i < dy; ++i) ao_normal_vec(&ms, dx, H + i * dx);
  random_spd(&ms, dy, 0.1, R);
  return AO_OK;
}

/* models.cpp:70-78 */
static void lorenz63_drift(const ao_spec* s, const double* v, double* f) {
  f[0] = s->lz_sigma * (v[1] - v[0]);
  f[1] = v[0] * (s->lz_rho - v[2]) - v[1];
  f[2] = v[0] * v[1] - s->lz_beta * v[2];
}
static void lorenz63_jac(const ao_spec* s, const double* v, double* j) {
  j[0] = -s->lz_sigma; j[1] = s->lz_sigma; j[2] = 0.0;
  j[3] = s->lz_rho - v[2]; j[4] = -1.0; j[5] = -v[0];
  j[6] = v[1]; j[7] = v[0]; j[8] = -s->lz_beta;
}

/* Lorenz-96 (new): f_i = (x_{i+1} - x_{i-2}) x_{i-1} - x_i + F, cyclic */
static void lorenz96_drift(const ao_spec* s, int d, const double* x, double* f) {
  for (int i = 0; i < d; ++i) {
    const double xp1 = x[(i + 1) % d], xm1 = x[(i + d - 1) % d], xm2 = x[(i + d - 2) % d];
    f[i] = (xp1 - xm2) * xm1 - x[i] + s->l96_F;
  }
}
static void lorenz96_jac(int d, const double* x, double* j) {
  memset(j, 0, sizeof(double) * d * d);
  for (int i = 0; i < d; ++i) {
    const int ip1 = (i + 1) % d, im1 = (i + d - 1) % d, im2 = (i + d - 2) % d;
    j[i * d + ip1] += x[im1];
    j[i * d + im2] -= x[im1];
    j[i * d + im1] += x[ip1] - x[im2];
    j[i * d + i] -= 1.0;
  }
}

/* models.cpp:88-103 */
static void lattice_laplacian(int k, double* lap) {
  const int n = k * k;
  memset(lap, 0, sizeof(double) * n * n);
#define LINK(a, b)            \
  do {                        \
    lap[(a) * n + (a)] += 1.0; \
    lap[(b) * n + (b)] += 1.0; \
    lap[(a) * n + (b)] -= 1.0; \
    lap[(b) * n + (a)] -= 1.0; \
  } while (0)
  for (int r = 0; r < k; ++r)
    for (int c = 0; c < k; ++c) {
      if (c + 1 < k) LINK(r * k + c, r * k + c + 1);
      if (r + 1 < k) LINK(r * k + c, (r + 1) * k + c);
    }
#undef LINK
}

/* models.cpp:105-111 */
static void spatio_innovation_cov(const ao_spec* s, double* cov) {
  const int n = s->grid * s->grid;
  double* prec = (double*)malloc(sizeof(double) * n * n);
  double* eye = (double*)malloc(sizeof(double) * n * n);
  double* l = (double*)malloc(sizeof(double) * n * n);
  lattice_laplacian(s->grid, prec);
  for (int i = 0; i < n; ++i) prec[i * n + i] += s->st_kappa2 * 1.0;
  ao_eye(n, eye);
  ao_llt(n, prec, l);
  ao_llt_solve(n, l, n, eye, cov);
  for (int i = 0; i < n * n; ++i) cov[i] = s->st_tau2 * cov[i];
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j) {
      double v = (cov[i * n + j] + cov[j * n + i]) / 2.0;
      cov[i * n + j] = cov[j * n + i] = v;
    }
  free(prec);
  free(eye);
  free(l);
}

/* models.cpp:113-119 */
static void stochvol_q(const ao_spec* s, double* q) {
  const int d = s->dx;
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < d; ++j)
      q[i * d + j] = s->sv_sig2 * ((1.0 - s->sv_rho) * (i == j ? 1.0 : 0.0) + s->sv_rho * 1.0);
}

/* models.cpp:123-128 */
static void ar1_p0(double phi, const double* q, int d, double* p0) {
  if (fabs(phi) < 1.0)
    for (int i = 0; i < d * d; ++i) p0[i] = q[i] / (1.0 - phi * phi);
  else
    memcpy(p0, q, sizeof(double) * d * d);
}

/* models.cpp:130-140 */
static long poisson_draw(double lambda, ao_stream* s) {
  const double u = ao_next_uniform(s);
  double p = exp(-lambda), cdf = p;
  long k = 0;
  while (u > cdf && k < 100000) {
    ++k;
    p *= lambda / k;
    cdf += p;
  }
  return k;
}

static void dyn_mean_kind(const ao_spec* s, int kind, int d, const double* x, double* out,
                          const double* F, const double* b) {
  if (kind == AO_KIND_LORENZ63) {
    double f[3];
    lorenz63_drift(s, x, f);
    for (int i = 0; i < 3; ++i) out[i] = x[i] + s->lz_h * f[i];
  } else if (kind == AO_KIND_LORENZ96) {
    double* f = (double*)malloc(sizeof(double) * d);
    lorenz96_drift(s, d, x, f);
    for (int i = 0; i < d; ++i) out[i] = x[i] + s->l96_h * f[i];
    free(f);
  } else {
    ao_matvec(d, d, F, x, out);
    for (int i = 0; i < d; ++i) out[i] += b[i];
  }
}

/* models.cpp:162-238 */
int ao_simulate(const ao_spec* s, double* latent, double* data) {
  const int dx = ao_latent_dim(s), dy = ao_obs_dim(s), T = s->T;
  if (dx < 1 || dy < 0 || T < 0) return AO_E_CONFIG;
  ao_stream root = ao_from_seed(s->data_seed);
  double* m0 = (double*)calloc(dx, sizeof(double));
  double* p0l = (double*)calloc(dx * dx, sizeof(double));
  double* ql = (double*)calloc(dx * dx, sizeof(double));
  double* F = (double*)calloc(dx * dx, sizeof(double));
  double* b = (double*)calloc(dx, sizeof(double));
  double* tmp = (double*)calloc(dx * dx, sizeof(double));
  double* tmp2 = (double*)calloc(dx * dx, sizeof(double));
  double *sH = NULL, *sRl = NULL;
  if (s->kind == AO_KIND_LGSSM) {
    sH = (double*)calloc(dy * dx, sizeof(double));
    double* sR = (double*)calloc(dy * dy, sizeof(double));
    sRl = (double*)calloc(dy * dy, sizeof(double));
    ao_synth_mats(s, m0, b, tmp, F, tmp2, sH, sR);
    ao_chol_psd(dx, tmp, p0l);
    ao_chol_psd(dx, tmp2, ql);
    ao_chol_psd(dy, sR, sRl);
    free(sR);
  } else if (s->kind == AO_KIND_STOCHVOL) {
    for (int i = 0; i < dx; ++i) m0[i] = s->sv_mu;
    stochvol_q(s, tmp);
    ar1_p0(s->sv_phi, tmp, dx, tmp2);
    ao_chol_psd(dx, tmp2, p0l);
    ao_chol_psd(dx, tmp, ql);
    for (int i = 0; i < dx; ++i) {
      F[i * dx + i] = s->sv_phi;
      b[i] = 0.0;
    }
  } else if (s->kind == AO_KIND_LORENZ63) {
    m0[0] = 1.0; m0[1] = 1.0; m0[2] = 25.0;
    ao_eye(3, p0l);
    for (int i = 0; i < 3; ++i) ql[i * 3 + i] = sqrt(s->lz_h) * s->lz_gamma;
  } else if (s->kind == AO_KIND_LORENZ96) {
    for (int i = 0; i < dx; ++i) m0[i] = s->l96_F;
    m0[0] += 0.01;
    ao_eye(dx, p0l);
    for (int i = 0; i < dx; ++i) ql[i * dx + i] = sqrt(s->l96_h) * s->l96_gamma;
  } else if (s->kind == AO_KIND_SPATIO) {
    spatio_innovation_cov(s, tmp);
    ar1_p0(s->st_phi, tmp, dx, tmp2);
    ao_chol_psd(dx, tmp2, p0l);
    ao_chol_psd(dx, tmp, ql);
    for (int i = 0; i < dx; ++i) F[i * dx + i] = s->st_phi;
  } else if (s->kind == AO_KIND_GRID1D) {
    m0[0] = s->g1_m0;
    p0l[0] = sqrt(s->g1_p0);
    ql[0] = sqrt(s->g1_q);
    F[0] = s->g1_phi;
  } else {
    return AO_E_CONFIG;
  }
  double* xi = (double*)malloc(sizeof(double) * (dx > dy ? dx : dy + 1));
  double* v = (double*)malloc(sizeof(double) * (dx > dy ? dx : dy + 1));
  double* x = (double*)malloc(sizeof(double) * dx);
  for (int t = 0; t <= T; ++t) {
    ao_stream st = ao_derive(root, AO_L_SIMULATE, (uint64_t)t);
    ao_normal_vec(&st, dx, xi);
    if (t == 0) {
      ao_matvec(dx, dx, p0l, xi, v);
      for (int i = 0; i < dx; ++i) x[i] = m0[i] + v[i];
    } else {
      double* mean = (double*)malloc(sizeof(double) * dx);
      if (s->kind == AO_KIND_STOCHVOL) {
        const double* xp = latent + (size_t)(t - 1) * dx;
        for (int i = 0; i < dx; ++i) mean[i] = s->sv_mu + s->sv_phi * (xp[i] - s->sv_mu);
      } else if (s->kind == AO_KIND_SPATIO || s->kind == AO_KIND_GRID1D) {
        const double phi = s->kind == AO_KIND_SPATIO ? s->st_phi : s->g1_phi;
        const double* xp = latent + (size_t)(t - 1) * dx;
        for (int i = 0; i < dx; ++i) mean[i] = phi * xp[i];
      } else {
        dyn_mean_kind(s, s->kind, dx, latent + (size_t)(t - 1) * dx, mean, F, b);
      }
      ao_matvec(dx, dx, ql, xi, v);
      for (int i = 0; i < dx; ++i) x[i] = mean[i] + v[i];
      free(mean);
    }
    memcpy(latent + (size_t)t * dx, x, sizeof(double) * dx);
    double* y = data + (size_t)t * dy;
    if (s->kind == AO_KIND_LGSSM) {
      double* e = (double*)malloc(sizeof(double) * dy);
      double* hx = (double*)malloc(sizeof(double) * dy);
      ao_matvec(dy, dx, sH, x, hx);
      ao_normal_vec(&st, dy, e);
      ao_matvec(dy, dy, sRl, e, v);
      for (int i = 0; i < dy; ++i) y[i] = hx[i] + v[i];
      free(e);
      free(hx);
    } else if (s->kind == AO_KIND_STOCHVOL) {
      for (int j = 0; j < dy; ++j) y[j] = exp(x[j] / 2.0) * ao_next_normal(&st);
    } else if (s->kind == AO_KIND_LORENZ63) {
      y[0] = x[0] + sqrt(s->lz_obs_var) * ao_next_normal(&st);
    } else if (s->kind == AO_KIND_LORENZ96) {
      for (int k = 0; k < dy; ++k) y[k] = x[2 * k] + sqrt(s->l96_obs_var) * ao_next_normal(&st);
    } else if (s->kind == AO_KIND_SPATIO) {
      for (int j = 0; j < dy; ++j) y[j] = (double)poisson_draw(exp(x[j]), &st);
    }
  }
  free(xi); free(v); free(x);
  free(m0); free(p0l); free(ql); free(F); free(b); free(tmp); free(tmp2);
  free(sH); free(sRl);
  return AO_OK;
}

/* ---------------- targets (target.cpp) ---------------- */
void ao_target_free(ao_target* t) {
  free(t->m0); free(t->P0); free(t->F); free(t->b); free(t->Q);
  free(t->eH); free(t->ec); free(t->eR); free(t->ey); free(t->emask);
  free(t->data); free(t->gmask);
  memset(t, 0, sizeof *t);
}

static double* dup(const double* p, size_t n) {
  double* o = (double*)malloc(sizeof(double) * (n ? n : 1));
  if (n) memcpy(o, p, sizeof(double) * n);
  return o;
}

/* models.cpp:240-336 */
int ao_make_target(const ao_spec* s, const double* data, ao_target* out) {
  memset(out, 0, sizeof *out);
  const int dx = ao_latent_dim(s), dy = ao_obs_dim(s), T = s->T;
  if (dx < 1) return AO_E_CONFIG;
  out->kind = s->kind;
  out->T = T;
  out->dx = dx;
  out->ydim = dy;
  out->spec = *s;
  out->data = dup(data, (size_t)(T + 1) * dy);
  out->emask = (uint8_t*)calloc(T + 1, 1);
  out->gmask = (uint8_t*)calloc(T + 1, 1);
  out->m0 = (double*)calloc(dx, sizeof(double));
  out->P0 = (double*)calloc(dx * dx, sizeof(double));
  out->nF = 1;
  out->F = (double*)calloc(dx * dx, sizeof(double));
  out->b = (double*)calloc(dx, sizeof(double));
  out->Q = (double*)calloc(dx * dx, sizeof(double));
  out->linear = 1;
  if (s->kind == AO_KIND_LGSSM) {
    double* H = (double*)malloc(sizeof(double) * dy * dx);
    double* R = (double*)malloc(sizeof(double) * dy * dy);
    ao_synth_mats(s, out->m0, out->b, out->P0, out->F, out->Q, H, R);
    out->q = dy;
    out->ne = 1;
    out->eH = H;
    out->ec = (double*)calloc(dy, sizeof(double));
    out->eR = R;
    out->ey = dup(data, (size_t)(T + 1) * dy);
    memset(out->emask, 1, T + 1);
  } else if (s->kind == AO_KIND_STOCHVOL) {
    stochvol_q(s, out->Q);
    for (int i = 0; i < dx; ++i) {
      out->m0[i] = s->sv_mu;
      out->F[i * dx + i] = s->sv_phi;
      out->b[i] = (1.0 - s->sv_phi) * s->sv_mu;
    }
    ar1_p0(s->sv_phi, out->Q, dx, out->P0);
    memset(out->gmask, 1, T + 1);
  } else if (s->kind == AO_KIND_LORENZ63 || s->kind == AO_KIND_LORENZ96) {
    out->linear = 0;
    const int q = dy;
    out->q = q;
    out->ne = 1;
    out->eH = (double*)calloc(q * dx, sizeof(double));
    for (int k = 0; k < q; ++k) out->eH[k * dx + 2 * k] = 1.0; /* L63: q = 1, H = [1 0 0] */
    out->ec = (double*)calloc(q, sizeof(double));
    out->eR = (double*)calloc(q * q, sizeof(double));
    const double ov = s->kind == AO_KIND_LORENZ63 ? s->lz_obs_var : s->l96_obs_var;
    for (int k = 0; k < q; ++k) out->eR[k * q + k] = ov * 1.0;
    out->ey = dup(data, (size_t)(T + 1) * q);
    memset(out->emask, 1, T + 1);
    if (s->kind == AO_KIND_LORENZ63) {
      out->m0[0] = 1.0; out->m0[1] = 1.0; out->m0[2] = 25.0;
      for (int i = 0; i < 3; ++i) out->Q[i * 3 + i] = s->lz_h * s->lz_gamma * s->lz_gamma;
    } else {
      for (int i = 0; i < dx; ++i) out->m0[i] = s->l96_F;
      out->m0[0] += 0.01;
      for (int i = 0; i < dx; ++i) out->Q[i * dx + i] = s->l96_h * s->l96_gamma * s->l96_gamma;
    }
    ao_eye(dx, out->P0);
  } else if (s->kind == AO_KIND_SPATIO) {
    spatio_innovation_cov(s, out->Q);
    for (int i = 0; i < dx; ++i) out->F[i * dx + i] = s->st_phi;
    ar1_p0(s->st_phi, out->Q, dx, out->P0);
    memset(out->gmask, 1, T + 1);
  } else if (s->kind == AO_KIND_GRID1D) {
    out->m0[0] = s->g1_m0;
    out->P0[0] = s->g1_p0 * 1.0;
    out->F[0] = s->g1_phi * 1.0;
    out->Q[0] = s->g1_q * 1.0;
    memset(out->gmask, 1, T + 1);
  } else {
    ao_target_free(out);
    return AO_E_CONFIG;
  }
  return AO_OK;
}

/* tests/testutil.hpp:88-140 */
int ao_target_from_lgssm(const ao_lgssm* m, const double* obs, int generic, ao_target* out) {
  memset(out, 0, sizeof *out);
  const int T = m->T, dx = m->dx, dy = m->dy;
  ao_spec_default(&out->spec);
  out->kind = generic ? AO_KIND_GAUSS_GENERIC : AO_KIND_LGSSM;
  out->T = T;
  out->dx = dx;
  out->ydim = dy;
  out->linear = 1;
  out->m0 = dup(m->m0, dx);
  out->P0 = dup(m->P0, dx * dx);
  const int nd = (m->nF > 1 || m->nb > 1 || m->nQ > 1) ? (T > 0 ? T : 1) : 1;
  out->nF = nd;
  out->F = (double*)malloc(sizeof(double) * dx * dx * nd);
  out->b = (double*)malloc(sizeof(double) * dx * nd);
  out->Q = (double*)malloc(sizeof(double) * dx * dx * nd);
  for (int t = 0; t < nd; ++t) {
    memcpy(out->F + (size_t)t * dx * dx, AO_F(m, t), sizeof(double) * dx * dx);
    memcpy(out->b + (size_t)t * dx, AO_B(m, t), sizeof(double) * dx);
    memcpy(out->Q + (size_t)t * dx * dx, AO_Q(m, t), sizeof(double) * dx * dx);
  }
  const int ne = (m->nH > 1 || m->nc > 1 || m->nR > 1) ? T + 1 : 1;
  out->ne = ne;
  out->eH = (double*)malloc(sizeof(double) * dy * dx * ne);
  out->ec = (double*)malloc(sizeof(double) * dy * ne);
  out->eR = (double*)malloc(sizeof(double) * dy * dy * ne);
  for (int t = 0; t < ne; ++t) {
    memcpy(out->eH + (size_t)t * dy * dx, AO_H(m, t), sizeof(double) * dy * dx);
    memcpy(out->ec + (size_t)t * dy, AO_C(m, t), sizeof(double) * dy);
    memcpy(out->eR + (size_t)t * dy * dy, AO_R(m, t), sizeof(double) * dy * dy);
  }
  out->ey = dup(obs, (size_t)(T + 1) * dy);
  out->data = dup(obs, (size_t)(T + 1) * dy);
  out->emask = (uint8_t*)calloc(T + 1, 1);
  out->gmask = (uint8_t*)calloc(T + 1, 1);
  for (int t = 0; t <= T; ++t) {
    if (!AO_OBSERVED(m, t)) continue;
    if (generic) out->gmask[t] = 1; else out->emask[t] = 1;
  }
  out->q = generic ? 0 : dy;
  if (generic) {
    /* keep the Gaussian blocks for the generic closures; no exact rows */
    out->q = 0;
  }
  /* generic Gaussian rows are stored in eH/ec/eR with row count ydim */
  return AO_OK;
}

#define TG_F(tg, t) ((tg)->F + (size_t)((tg)->nF > 1 ? (t) : 0) * (tg)->dx * (tg)->dx)
#define TG_B(tg, t) ((tg)->b + (size_t)((tg)->nF > 1 ? (t) : 0) * (tg)->dx)
#define TG_Q(tg, t) ((tg)->Q + (size_t)((tg)->nF > 1 ? (t) : 0) * (tg)->dx * (tg)->dx)
#define E_ROWS(tg) ((tg)->kind == AO_KIND_GAUSS_GENERIC ? (tg)->ydim : (tg)->q)
#define TG_EH(tg, t) ((tg)->eH + (size_t)((tg)->ne > 1 ? (t) : 0) * E_ROWS(tg) * (tg)->dx)
#define TG_EC(tg, t) ((tg)->ec + (size_t)((tg)->ne > 1 ? (t) : 0) * E_ROWS(tg))
#define TG_ER(tg, t) ((tg)->eR + (size_t)((tg)->ne > 1 ? (t) : 0) * E_ROWS(tg) * E_ROWS(tg))

/* target.cpp:47-57 */
void ao_dyn_mean(const ao_target* tg, int t, const double* x, double* out) {
  dyn_mean_kind(&tg->spec, tg->linear ? -1 : tg->kind, tg->dx, x, out, TG_F(tg, t), TG_B(tg, t));
}
void ao_dyn_jac(const ao_target* tg, int t, const double* x, double* out) {
  const int d = tg->dx;
  if (tg->linear) {
    memcpy(out, TG_F(tg, t), sizeof(double) * d * d);
  } else if (tg->kind == AO_KIND_LORENZ63) {
    double j[9];
    lorenz63_jac(&tg->spec, x, j);
    for (int i = 0; i < 9; ++i) out[i] = (i % 4 == 0 ? 1.0 : 0.0) + tg->spec.lz_h * j[i];
  } else {
    lorenz96_jac(d, x, out);
    for (int i = 0; i < d * d; ++i) out[i] = ((i % (d + 1)) == 0 ? 1.0 : 0.0) + tg->spec.l96_h * out[i];
  }
}
void ao_dyn_cov(const ao_target* tg, int t, const double* x, double* out) {
  (void)x;
  memcpy(out, TG_Q(tg, t), sizeof(double) * tg->dx * tg->dx);
}

/* generic log-potential and gradient per kind (models.cpp:261-317, testutil.hpp:112-140) */
static double generic_log_g(const ao_target* tg, int t, const double* x, int* status) {
  const int d = tg->dx;
  const double* y = tg->data + (size_t)t * tg->ydim;
  if (tg->kind == AO_KIND_STOCHVOL) {
    double sx = 0.0, sy = 0.0;
    for (int i = 0; i < d; ++i) sx += x[i];
    for (int i = 0; i < d; ++i) sy += (y[i] * y[i]) * exp(-x[i]);
    return -0.5 * (log(2.0 * M_PI) * d + sx + sy);
  }
  if (tg->kind == AO_KIND_SPATIO) {
    double s = 0.0;
    for (int j = 0; j < d; ++j) s += y[j] * x[j] - exp(x[j]) - lgamma(y[j] + 1.0);
    return s;
  }
  if (tg->kind == AO_KIND_GRID1D) return -x[0] * x[0] * x[0] * x[0];
  if (tg->kind == AO_KIND_GAUSS_GENERIC) {
    const int q = tg->ydim;
    double* r = (double*)malloc(sizeof(double) * 2 * q);
    double* z = r + q;
    const double* H = TG_EH(tg, t);
    const double* c = TG_EC(tg, t);
    ao_matvec(q, d, H, x, z);
    for (int i = 0; i < q; ++i) r[i] = (y[i] - c[i]) - z[i];
    for (int i = 0; i < q; ++i) z[i] = 0.0;
    double v = ao_log_pdf(q, r, z, TG_ER(tg, t), status);
    free(r);
    return v;
  }
  return 0.0;
}

void ao_grad_pot_generic(const ao_target* tg, int t, const double* x, double* g) {
  const int d = tg->dx;
  if (!tg->gmask[t]) {
    for (int i = 0; i < d; ++i) g[i] = 0.0;
    return;
  }
  const double* y = tg->data + (size_t)t * tg->ydim;
  if (tg->kind == AO_KIND_STOCHVOL) {
    for (int i = 0; i < d; ++i) g[i] = 0.5 * ((y[i] * y[i]) * exp(-x[i]) - 1.0);
  } else if (tg->kind == AO_KIND_SPATIO) {
    for (int i = 0; i < d; ++i) g[i] = y[i] - exp(x[i]);
  } else if (tg->kind == AO_KIND_GRID1D) {
    g[0] = -4.0 * x[0] * x[0] * x[0];
  } else if (tg->kind == AO_KIND_GAUSS_GENERIC) {
    const int q = tg->ydim;
    double* r = (double*)malloc(sizeof(double) * 2 * q);
    double* z = r + q;
    const double* H = TG_EH(tg, t);
    const double* c = TG_EC(tg, t);
    ao_matvec(q, d, H, x, z);
    for (int i = 0; i < q; ++i) r[i] = (y[i] - c[i]) - z[i];
    ao_solve_spd(q, TG_ER(tg, t), 1, r, z);
    ao_matvec_t(q, d, H, z, g);
    free(r);
  } else {
    for (int i = 0; i < d; ++i) g[i] = 0.0;
  }
}

/* target.cpp:75-83 */
double ao_log_pot(const ao_target* tg, int t, const double* x, int* status) {
  double lp = 0.0;
  const int d = tg->dx;
  if (tg->emask[t] && tg->q > 0) {
    const int q = tg->q;
    double* mu = (double*)malloc(sizeof(double) * q);
    ao_matvec(q, d, TG_EH(tg, t), x, mu);
    const double* c = TG_EC(tg, t);
    for (int i = 0; i < q; ++i) mu[i] += c[i];
    lp += ao_log_pdf(q, tg->ey + (size_t)t * q, mu, TG_ER(tg, t), status);
    free(mu);
  }
  if (tg->gmask[t]) lp += generic_log_g(tg, t, x, status);
  return lp;
}

/* target.cpp:90-98 */
void ao_grad_pot(const ao_target* tg, int t, const double* x, double* g, int* status) {
  const int d = tg->dx;
  ao_grad_pot_generic(tg, t, x, g);
  if (tg->emask[t] && tg->q > 0) {
    const int q = tg->q;
    double* r = (double*)malloc(sizeof(double) * (2 * q + d));
    double* z = r + q;
    double* w = z + q;
    ao_matvec(q, d, TG_EH(tg, t), x, z);
    const double* c = TG_EC(tg, t);
    const double* y = tg->ey + (size_t)t * q;
    for (int i = 0; i < q; ++i) r[i] = (y[i] - z[i]) - c[i];
    int st = ao_solve_spd(q, TG_ER(tg, t), 1, r, z);
    if (status && st != AO_OK) *status = st;
    ao_matvec_t(q, d, TG_EH(tg, t), z, w);
    for (int i = 0; i < d; ++i) g[i] += w[i];
    free(r);
  }
}

/* target.cpp:100-108 */
double ao_log_gamma(const ao_target* tg, const double* traj, int* status) {
  const int T = tg->T, d = tg->dx;
  double* mean = (double*)malloc(sizeof(double) * (d + d * d));
  double* cov = mean + d;
  int st = AO_OK;
  double lg = ao_log_pdf(d, traj, tg->m0, tg->P0, &st);
  for (int t = 0; t < T; ++t) {
    ao_dyn_mean(tg, t, traj + (size_t)t * d, mean);
    ao_dyn_cov(tg, t, traj + (size_t)t * d, cov);
    lg += ao_log_pdf(d, traj + (size_t)(t + 1) * d, mean, cov, &st);
  }
  for (int t = 0; t <= T; ++t) lg += ao_log_pot(tg, t, traj + (size_t)t * d, &st);
  free(mean);
  if (status) *status = st;
  return lg;
}
