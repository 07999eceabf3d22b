/* ao_auxk.c — auxiliary Kalman MH kernel; restates proj/src/auxk.cpp.
 * TEST INFRASTRUCTURE (parity oracle); see auxmc_oracle.h. */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "auxmc_oracle.h"
#include "ao_internal.h"

/* auxk.cpp:45-54 */
void ao_sample_aux_obs(const double* x, int T, int dx, double delta, ao_stream it, double* u) {
  const double sd = sqrt(delta / 2.0);
  double* xi = (double*)malloc(sizeof(double) * dx);
  for (int t = 0; t <= T; ++t) {
    ao_stream s = ao_derive(it, AO_L_AUX_OBS, (uint64_t)t);
    ao_normal_vec(&s, dx, xi);
    for (int j = 0; j < dx; ++j) u[(size_t)t * dx + j] = x[(size_t)t * dx + j] + sd * xi[j];
  }
  free(xi);
}

/* auxk.cpp:14-20 */
static void generic_grads(const ao_target* tg, const double* x, double* g) {
  for (int t = 0; t <= tg->T; ++t)
    ao_grad_pot_generic(tg, t, x + (size_t)t * tg->dx, g + (size_t)t * tg->dx);
}

/* auxk.cpp:23-29: sum_t log N(u_t; x_t, delta/2 I) */
static double aux_loglik(const double* u, const double* x, int T, int dx, double delta) {
  double lp = 0.0;
  double* r = (double*)malloc(sizeof(double) * dx);
  for (int t = 0; t <= T; ++t) {
    for (int j = 0; j < dx; ++j) r[j] = u[(size_t)t * dx + j] - x[(size_t)t * dx + j];
    lp += ao_isotropic_log_pdf(dx, r, delta / 2.0);
  }
  free(r);
  return lp;
}

/* auxk.cpp:56-118 */
int ao_build_aux_lgssm(const ao_target* tg, const double* x, const double* u, double delta,
                       int zeroth_order, const double* grads, ao_lgssm* out, double** obs_out) {
  const int T = tg->T, dx = tg->dx;
  const int extra = tg->q;
  const int dy = dx + extra;
  memset(out, 0, sizeof *out);
  out->T = T;
  out->dx = dx;
  out->dy = dy;
  double* m0 = (double*)malloc(sizeof(double) * dx);
  double* P0 = (double*)malloc(sizeof(double) * dx * dx);
  memcpy(m0, tg->m0, sizeof(double) * dx);
  memcpy(P0, tg->P0, sizeof(double) * dx * dx);
  ao_symm(dx, P0);
  const int nd = T > 0 ? T : 1;
  double* F = (double*)calloc((size_t)nd * dx * dx, sizeof(double));
  double* b = (double*)calloc((size_t)nd * dx, sizeof(double));
  double* Q = (double*)calloc((size_t)nd * dx * dx, sizeof(double));
  double* fx = (double*)malloc(sizeof(double) * dx);
  for (int t = 0; t < T; ++t) {
    double* Ft = F + (size_t)t * dx * dx;
    double* bt = b + (size_t)t * dx;
    double* Qt = Q + (size_t)t * dx * dx;
    const double* xt = x + (size_t)t * dx;
    if (tg->linear) {
      ao_dyn_jac(tg, t, xt, Ft);
      memcpy(bt, tg->b + (size_t)(tg->nF > 1 ? t : 0) * dx, sizeof(double) * dx);
      ao_dyn_cov(tg, t, xt, Qt);
    } else {
      ao_dyn_jac(tg, t, xt, Ft);
      ao_dyn_mean(tg, t, xt, bt);
      ao_matvec(dx, dx, Ft, xt, fx);
      for (int i = 0; i < dx; ++i) bt[i] -= fx[i];
      ao_dyn_cov(tg, t, xt, Qt);
    }
    ao_symm(dx, Qt);
  }
  free(fx);
  double* H = (double*)calloc((size_t)(T + 1) * dy * dx, sizeof(double));
  double* c = (double*)calloc((size_t)(T + 1) * dy, sizeof(double));
  double* R = (double*)calloc((size_t)(T + 1) * dy * dy, sizeof(double));
  double* obs = (double*)calloc((size_t)(T + 1) * dy, sizeof(double));
  double* g = (double*)malloc(sizeof(double) * dx);
  for (int t = 0; t <= T; ++t) {
    double* Ht = H + (size_t)t * dy * dx;
    double* Rt = R + (size_t)t * dy * dy;
    for (int i = 0; i < dx; ++i) Ht[i * dx + i] = 1.0;
    for (int i = 0; i < dy; ++i) Rt[i * dy + i] = 1.0;
    for (int i = 0; i < dx; ++i) Rt[i * dy + i] = delta / 2.0;
    double* z = obs + (size_t)t * dy;
    for (int i = 0; i < dx; ++i) z[i] = u[(size_t)t * dx + i];
    if (!zeroth_order) {
      if (grads)
        memcpy(g, grads + (size_t)t * dx, sizeof(double) * dx);
      else
        ao_grad_pot_generic(tg, t, x + (size_t)t * dx, g);
      for (int i = 0; i < dx; ++i) z[i] += (delta / 2.0) * g[i];
    }
    if (tg->emask[t] && extra > 0) {
      const int q = extra;
      const size_t eo = (size_t)(tg->ne > 1 ? t : 0);
      const double* eH = tg->eH + eo * q * dx;
      const double* ec = tg->ec + eo * q;
      const double* eR = tg->eR + eo * q * q;
      for (int i = 0; i < q; ++i) {
        for (int j = 0; j < dx; ++j) Ht[(dx + i) * dx + j] = eH[i * dx + j];
        c[(size_t)t * dy + dx + i] = ec[i];
        for (int j = 0; j < q; ++j) Rt[(dx + i) * dy + dx + j] = eR[i * q + j];
        z[dx + i] = tg->ey[(size_t)t * q + i];
      }
    }
    ao_symm(dy, Rt);
  }
  free(g);
  out->m0 = m0;
  out->P0 = P0;
  out->F = F; out->nF = nd;
  out->b = b; out->nb = nd;
  out->Q = Q; out->nQ = nd;
  out->H = H; out->nH = T + 1;
  out->c = c; out->nc = T + 1;
  out->R = R; out->nR = T + 1;
  out->mask = NULL;
  *obs_out = obs;
  return AO_OK;
}

static void free_aux(ao_lgssm* m, double* obs) {
  free((void*)m->m0); free((void*)m->P0); free((void*)m->F); free((void*)m->b);
  free((void*)m->Q); free((void*)m->H); free((void*)m->c); free((void*)m->R);
  free(obs);
}

static int alloc_filter(ao_filter* fr, int T, int dx) {
  fr->pred_mean = (double*)malloc(sizeof(double) * (size_t)(T + 1) * dx);
  fr->filt_mean = (double*)malloc(sizeof(double) * (size_t)(T + 1) * dx);
  fr->pred_cov = (double*)malloc(sizeof(double) * (size_t)(T + 1) * dx * dx);
  fr->filt_cov = (double*)malloc(sizeof(double) * (size_t)(T + 1) * dx * dx);
  fr->log_marginal = 0.0;
  return AO_OK;
}
static void free_filter(ao_filter* fr) {
  free(fr->pred_mean); free(fr->filt_mean); free(fr->pred_cov); free(fr->filt_cov);
}

/* auxk.cpp:120-128 */
int ao_init_chain(const ao_target* tg, const double* x0, double delta, ao_chain* st) {
  const size_t n = (size_t)(tg->T + 1) * tg->dx;
  memset(st, 0, sizeof *st);
  st->x = (double*)malloc(sizeof(double) * n);
  memcpy(st->x, x0, sizeof(double) * n);
  st->grad_gen = (double*)malloc(sizeof(double) * n);
  st->delta = delta;
  int s = AO_OK;
  st->log_gamma = ao_log_gamma(tg, st->x, &s);
  generic_grads(tg, st->x, st->grad_gen);
  return s;
}
void ao_chain_free(ao_chain* st) {
  free(st->x);
  free(st->grad_gen);
  st->x = st->grad_gen = NULL;
}

static int run_filter(const ao_lgssm* m, const double* obs, ao_filter* fr, int parallel) {
  return parallel ? ao_parallel_filter(m, obs, fr, NULL, NULL) : ao_kalman_filter(m, obs, fr);
}

static int draw_path(const ao_lgssm* m, const ao_filter* fr, ao_stream it, int backend,
                     double* out) {
  ao_noise noise;
  memset(&noise, 0, sizeof noise);
  noise.kind = 0;
  noise.base = it;
  if (backend == AO_BACKEND_SEQ) return ao_backward_sample(m, fr, &noise, out);
  if (backend == AO_BACKEND_PREFIX) return ao_prefix_sample(m, fr, &noise, out, NULL, NULL);
  return ao_dnc_sample(m, fr, &noise, out);
}

static int all_finite(const double* v, size_t n) {
  for (size_t i = 0; i < n; ++i)
    if (!isfinite(v[i])) return 0;
  return 1;
}

/* auxk.cpp:130-198 */
int ao_kernel_step(const ao_target* tg, ao_chain* st, ao_stream rng, int backend,
                   int parallel_filter, int zeroth_order) {
  const int T = tg->T, dx = tg->dx;
  const size_t n = (size_t)(T + 1) * dx;
  const ao_stream it = ao_derive(rng, AO_L_ITERATION, (uint64_t)st->iter);
  ++st->iter;
  st->stats.last_accept_prob = 0.0;
  st->stats.last_log_alpha = -INFINITY;
  double* u = (double*)malloc(sizeof(double) * n);
  double* prop = (double*)malloc(sizeof(double) * n);
  double* grads_prop = (double*)malloc(sizeof(double) * n);
  ao_sample_aux_obs(st->x, T, dx, st->delta, it, u);
  ao_lgssm cur, rev;
  double *cobs = NULL, *robs = NULL;
  ao_filter fr, frr;
  alloc_filter(&fr, T, dx);
  alloc_filter(&frr, T, dx);
  int s = AO_OK;
  int have_rev = 0;
  ao_build_aux_lgssm(tg, st->x, u, st->delta, zeroth_order, st->grad_gen, &cur, &cobs);
  s = run_filter(&cur, cobs, &fr, parallel_filter);
  if (s == AO_OK) s = draw_path(&cur, &fr, it, backend, prop);
  double logq_fwd = 0.0;
  if (s == AO_OK) logq_fwd = ao_path_logpdf(&cur, cobs, prop, &fr, &s);
  if (s != AO_OK) goto factor_fail;
  {
    const double lg_prop = ao_log_gamma(tg, prop, &s);
    if (s != AO_OK) goto factor_fail;
    if (!isfinite(lg_prop)) {
      ++st->stats.nonfinite_gamma;
      ++st->stats.rejected;
      goto done;
    }
    generic_grads(tg, prop, grads_prop);
    if (!all_finite(grads_prop, n)) {
      ++st->stats.aborted;
      ++st->stats.rejected;
      goto done;
    }
    ao_build_aux_lgssm(tg, prop, u, st->delta, zeroth_order, grads_prop, &rev, &robs);
    have_rev = 1;
    s = run_filter(&rev, robs, &frr, parallel_filter);
    double logq_rev = 0.0;
    if (s == AO_OK) logq_rev = ao_path_logpdf(&rev, robs, st->x, &frr, &s);
    if (s != AO_OK) goto factor_fail;
    const double log_alpha = (lg_prop + aux_loglik(u, prop, T, dx, st->delta) + logq_rev) -
                             (st->log_gamma + aux_loglik(u, st->x, T, dx, st->delta) + logq_fwd);
    if (isnan(log_alpha)) {
      ++st->stats.aborted;
      ++st->stats.rejected;
      goto done;
    }
    st->stats.last_log_alpha = log_alpha;
    st->stats.last_accept_prob = log_alpha >= 0.0 ? 1.0 : exp(log_alpha);
    ao_stream acc = ao_derive(it, AO_L_MH_ACCEPT, 0);
    if (ao_next_uniform(&acc) < st->stats.last_accept_prob) {
      memcpy(st->x, prop, sizeof(double) * n);
      st->log_gamma = lg_prop;
      memcpy(st->grad_gen, grads_prop, sizeof(double) * n);
      ++st->stats.accepted;
    } else {
      ++st->stats.rejected;
    }
    goto done;
  }
factor_fail:
  ++st->stats.aborted;
  ++st->stats.rejected;
done:
  free_aux(&cur, cobs);
  if (have_rev) free_aux(&rev, robs);
  free_filter(&fr);
  free_filter(&frr);
  free(u);
  free(prop);
  free(grads_prop);
  return AO_OK;
}

/* auxk.cpp:200-211 */
double ao_mh_log_ratio(const ao_target* tg, const double* x, const double* xp, const double* u,
                       double delta, int zeroth_order, int* status) {
  const int T = tg->T, dx = tg->dx;
  ao_lgssm cur, rev;
  double *cobs, *robs;
  ao_filter fr, frr;
  alloc_filter(&fr, T, dx);
  alloc_filter(&frr, T, dx);
  int s = AO_OK;
  ao_build_aux_lgssm(tg, x, u, delta, zeroth_order, NULL, &cur, &cobs);
  ao_build_aux_lgssm(tg, xp, u, delta, zeroth_order, NULL, &rev, &robs);
  s = ao_kalman_filter(&cur, cobs, &fr);
  if (s == AO_OK) s = ao_kalman_filter(&rev, robs, &frr);
  double r = NAN;
  if (s == AO_OK) {
    const double a = ao_log_gamma(tg, xp, &s) + aux_loglik(u, xp, T, dx, delta) +
                     ao_path_logpdf(&rev, robs, x, &frr, &s);
    const double b = ao_log_gamma(tg, x, &s) + aux_loglik(u, x, T, dx, delta) +
                     ao_path_logpdf(&cur, cobs, xp, &fr, &s);
    r = a - b;
  }
  free_aux(&cur, cobs);
  free_aux(&rev, robs);
  free_filter(&fr);
  free_filter(&frr);
  if (status) *status = s;
  return r;
}

/* auxk.cpp:213-218 */
void ao_adapt_delta(ao_chain* st, double target_rate) {
  const double n = (double)(st->iter > 1 ? st->iter : 1);
  const double step = pow(n, -0.6);
  st->delta = exp(log(st->delta) + step * (st->stats.last_accept_prob - target_rate));
}

/* runner.cpp:61-85 gamma_move: random-walk MH on log gamma (the diffusion
 * coefficient, Q = h gamma^2 I) with a standard normal prior on log gamma.  The drift
 * does not depend on gamma, so the residual sum of squares is computed once (:65-70).
 * The reference hard-codes d = 3 (Lorenz-63, "-1.5 * T"); the same density with
 * 0.5 * d covers Lorenz-96 (0.5 * 3 == 1.5 exactly, so d = 3 is bit-identical).
 * s = root.derive(kParam, iter) (:160-161); normal at counter 0, uniform at 1.
 * Returns 1 and updates *gamma when the move is accepted. */
int ao_gamma_move(const ao_target* tg, const double* x, double* gamma, double step,
                  ao_stream s) {
  const int T = tg->T, d = tg->dx;
  double* mean = (double*)malloc(sizeof(double) * d);
  double sse = 0.0;
  for (int t = 0; t < T; ++t) {
    ao_dyn_mean(tg, t, x + (size_t)t * d, mean);
    double sq = 0.0;
    for (int i = 0; i < d; ++i) {
      const double r = x[(size_t)(t + 1) * d + i] - mean[i];
      sq += r * r;
    }
    sse += sq;
  }
  free(mean);
  const double h = tg->kind == AO_KIND_LORENZ63 ? tg->spec.lz_h : tg->spec.l96_h;
  const double hd = 0.5 * d;
  const double g0 = *gamma;
#define AO_GLL(g) (-hd * T * log(2.0 * M_PI * h * (g) * (g)) - sse / (2.0 * h * (g) * (g)))
  const double lg = log(g0);
  const double lg_prop = lg + step * ao_next_normal(&s);
  const double g_prop = exp(lg_prop);
  const double log_r = AO_GLL(g_prop) - 0.5 * lg_prop * lg_prop - (AO_GLL(g0) - 0.5 * lg * lg);
#undef AO_GLL
  if (log(ao_next_uniform(&s)) < log_r) {
    *gamma = g_prop;
    return 1;
  }
  return 0;
}
