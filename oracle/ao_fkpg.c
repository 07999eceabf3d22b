/* ao_fkpg.c — conditional SMC with backward index sampling and the auxiliary
 * particle Gibbs sweep; restates proj/src/fkpg.cpp (prior / gradient / fully
 * adapted proposals linearized at the auxiliary observation).  Also a
 * forward-backward oracle for the parallel-in-time cSMC lattice law.
 * TEST INFRASTRUCTURE (parity oracle); see auxmc_oracle.h. */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "auxmc_oracle.h"
#include "ao_internal.h"

/* fkpg.cpp:19-27 */
static int normalize(const double* logw, int n, double* W, double* log_mean) {
  double m = logw[0];
  for (int i = 1; i < n; ++i) m = logw[i] > m ? logw[i] : m;
  if (!isfinite(m)) return AO_E_DEGENERATE;
  double s = 0.0;
  for (int i = 0; i < n; ++i) {
    W[i] = exp(logw[i] - m);
    s += W[i];
  }
  for (int i = 0; i < n; ++i) W[i] = W[i] / s;
  if (log_mean) *log_mean = m + log(s) - log((double)n);
  return AO_OK;
}

/* fkpg.cpp:29-37 */
static int multinomial_draw(const double* w, int n, double u) {
  double acc = 0.0;
  for (int i = 0; i < n; ++i) {
    acc += w[i];
    if (u <= acc) return i;
  }
  return n - 1;
}

typedef struct {
  const ao_target* tg;
  const double* u;
  double delta;
  int mode;
} aux_fk;

/* fkpg.cpp:154-186, linearize = kAuxObs */
static int proposal(const aux_fk* fk, int t, const double* xprev, double* mean, double* cov) {
  const ao_target* tg = fk->tg;
  const int d = tg->dx;
  const double* ut = fk->u + (size_t)t * d;
  const double h = fk->delta / 2.0;
  double* pm = (double*)malloc(sizeof(double) * (3 * d * d + 3 * d));
  double* pc = pm + d;
  double* g = pc + d * d;
  double* s = g + d;
  double* gain = s + d * d;
  double* z = gain + d * d;
  int st = AO_OK;
  if (t == 0) {
    memcpy(pm, tg->m0, sizeof(double) * d);
    memcpy(pc, tg->P0, sizeof(double) * d * d);
  } else if (fk->mode != AO_PG_GRADIENT) {
    ao_dyn_mean(tg, t - 1, xprev, pm);
    ao_dyn_cov(tg, t - 1, xprev, pc);
  }
  if (fk->mode == AO_PG_PRIOR) {
    memcpy(mean, pm, sizeof(double) * d);
    memcpy(cov, pc, sizeof(double) * d * d);
  } else if (fk->mode == AO_PG_GRADIENT) {
    ao_grad_pot(tg, t, ut, g, &st);
    for (int i = 0; i < d; ++i) mean[i] = ut[i] + h * g[i];
    for (int i = 0; i < d * d; ++i) cov[i] = 0.0;
    for (int i = 0; i < d; ++i) cov[i * d + i] = h * 1.0;
  } else {
    ao_grad_pot(tg, t, ut, g, &st);
    for (int i = 0; i < d; ++i) z[i] = ut[i] + h * g[i];
    for (int i = 0; i < d * d; ++i) s[i] = pc[i];
    for (int i = 0; i < d; ++i) s[i * d + i] += h * 1.0;
    double* sol = (double*)malloc(sizeof(double) * 3 * d * d);
    double* a = sol + d * d;
    double* w = a + d * d;
    st = ao_solve_spd(d, s, d, pc, sol);
    ao_transpose(d, d, sol, gain);
    for (int i = 0; i < d * d; ++i) a[i] = -gain[i];
    for (int i = 0; i < d; ++i) a[i * d + i] += 1.0;
    ao_sandwich(d, d, a, pc, cov, w);
    ao_matmul_bt(d, d, d, gain, gain, w);
    for (int i = 0; i < d * d; ++i) cov[i] += h * w[i];
    for (int i = 0; i < d; ++i) z[i] -= pm[i];
    ao_matvec(d, d, gain, z, mean);
    for (int i = 0; i < d; ++i) mean[i] = pm[i] + mean[i];
    free(sol);
  }
  ao_symm(d, cov);
  free(pm);
  return st;
}

/* fkpg.cpp:212-223 pot(t, xp, x) */
static double potential(const aux_fk* fk, int t, const double* xp, const double* x, int* st) {
  const ao_target* tg = fk->tg;
  const int d = tg->dx;
  double* r = (double*)malloc(sizeof(double) * (2 * d + d * d));
  double* mean = r + d;
  double* cov = mean + d;
  for (int i = 0; i < d; ++i) r[i] = fk->u[(size_t)t * d + i] - x[i];
  double lg = ao_log_pot(tg, t, x, st) + ao_isotropic_log_pdf(d, r, fk->delta / 2.0);
  if (fk->mode != AO_PG_PRIOR) {
    double ld;
    if (t == 0) {
      ld = ao_log_pdf(d, x, tg->m0, tg->P0, st);
    } else {
      ao_dyn_mean(tg, t - 1, xp, mean);
      ao_dyn_cov(tg, t - 1, xp, cov);
      ld = ao_log_pdf(d, x, mean, cov, st);
    }
    *st |= proposal(fk, t, xp, mean, cov);
    lg += ld - ao_log_pdf(d, x, mean, cov, st);
  }
  free(r);
  return lg;
}

static double m_logpdf(const aux_fk* fk, int t, const double* xp, const double* x, int* st) {
  const int d = fk->tg->dx;
  double* mean = (double*)malloc(sizeof(double) * (d + d * d));
  double* cov = mean + d;
  *st |= proposal(fk, t, xp, mean, cov);
  double v = ao_log_pdf(d, x, mean, cov, st);
  free(mean);
  return v;
}

static int sample_proposal(const aux_fk* fk, int t, const double* xp, ao_stream* rng, double* x) {
  const int d = fk->tg->dx;
  double* mean = (double*)malloc(sizeof(double) * (2 * d + 2 * d * d));
  double* cov = mean + d;
  double* l = cov + d * d;
  double* xi = l + d * d;
  int st = proposal(fk, t, xp, mean, cov);
  if (st == AO_OK) st = ao_chol_psd(d, cov, l);
  ao_normal_vec(rng, d, xi);
  ao_matvec(d, d, l, xi, x);
  for (int i = 0; i < d; ++i) x[i] = mean[i] + x[i];
  free(mean);
  return st;
}

int ao_init_pg(const ao_target* tg, const double* x0, double delta, ao_pg* st) {
  const size_t n = (size_t)(tg->T + 1) * tg->dx;
  memset(st, 0, sizeof *st);
  st->x = (double*)malloc(sizeof(double) * n);
  memcpy(st->x, x0, sizeof(double) * n);
  st->keys = (uint64_t*)calloc(tg->T + 1, sizeof(uint64_t));
  st->delta = delta;
  return AO_OK;
}
void ao_pg_free(ao_pg* st) {
  free(st->x);
  free(st->keys);
  st->x = NULL;
  st->keys = NULL;
}

/* fkpg.cpp:44-152 (sweep + csmc_step) and :260-274 (aux_pgibbs_step) */
int ao_aux_pgibbs_step(const ao_target* tg, ao_pg* pg, int N, ao_stream rng, int mode,
                       int* anc_out, int* sel_out, int* bad_t) {
  const int T = tg->T, d = tg->dx;
  const size_t n = (size_t)(T + 1) * d;
  const ao_stream it = ao_derive(rng, AO_L_ITERATION, (uint64_t)pg->iter);
  ++pg->iter;
  double* u = (double*)malloc(sizeof(double) * n);
  ao_sample_aux_obs(pg->x, T, d, pg->delta, it, u);
  aux_fk fk = {tg, u, pg->delta, mode};

  double* part = (double*)malloc(sizeof(double) * (size_t)(T + 1) * N * d);
  double* W = (double*)malloc(sizeof(double) * (size_t)(T + 1) * N);
  double* logw = (double*)malloc(sizeof(double) * N);
  int* anc = (int*)calloc((size_t)(T + 1) * N, sizeof(int));
  uint64_t* keys = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(T + 1) * N);
  double* traj = (double*)malloc(sizeof(double) * n);
  uint64_t* tkeys = (uint64_t*)malloc(sizeof(uint64_t) * (T + 1));
  int st = AO_OK;
  for (int t = 0; t <= T && st == AO_OK; ++t) {
    ao_stream sst = ao_derive(it, AO_L_STEP, (uint64_t)t);
    if (t > 0) {
      ao_stream rs = ao_derive(sst, AO_L_RESAMPLE, 0);
      for (int i = 1; i < N; ++i)
        anc[(size_t)t * N + i] = multinomial_draw(W + (size_t)(t - 1) * N, N, ao_next_uniform(&rs));
    }
    for (int i = 0; i < N; ++i) {
      ao_stream ks = ao_derive(sst, AO_L_PM_KEY, (uint64_t)i);
      uint64_t key = ao_next_key(&ks);
      double* x = part + ((size_t)t * N + i) * d;
      const double* parent =
          t > 0 ? part + ((size_t)(t - 1) * N + anc[(size_t)t * N + i]) * d : NULL;
      if (i == 0) {
        memcpy(x, pg->x + (size_t)t * d, sizeof(double) * d);
        key = pg->keys[t];
      } else {
        ao_stream pi = ao_derive(sst, AO_L_PARTICLE, (uint64_t)i);
        st |= sample_proposal(&fk, t, parent, &pi, x);
      }
      keys[(size_t)t * N + i] = key;
      logw[i] = potential(&fk, t, parent, x, &st);
    }
    if (st != AO_OK) break;
    if (normalize(logw, N, W + (size_t)t * N, NULL) != AO_OK) {
      st = AO_E_DEGENERATE;
      if (bad_t) *bad_t = t;
    }
  }
  if (st == AO_OK) {
    ao_stream ti = ao_derive(it, AO_L_TERMINAL_INDEX, 0);
    int sel = multinomial_draw(W + (size_t)T * N, N, ao_next_uniform(&ti));
    if (sel_out) sel_out[T] = sel;
    memcpy(traj + (size_t)T * d, part + ((size_t)T * N + sel) * d, sizeof(double) * d);
    tkeys[T] = keys[(size_t)T * N + sel];
    double* logb = (double*)malloc(sizeof(double) * N);
    double* bw = (double*)malloc(sizeof(double) * N);
    for (int t = T - 1; t >= 0 && st == AO_OK; --t) {
      const double* chosen = traj + (size_t)(t + 1) * d;
      for (int i = 0; i < N; ++i) {
        const double* xi = part + ((size_t)t * N + i) * d;
        logb[i] = log(W[(size_t)t * N + i]) + m_logpdf(&fk, t + 1, xi, chosen, &st) +
                  potential(&fk, t + 1, xi, chosen, &st);
      }
      if (normalize(logb, N, bw, NULL) != AO_OK) {
        st = AO_E_DEGENERATE;
        if (bad_t) *bad_t = t;
        break;
      }
      ao_stream bs = ao_derive(it, AO_L_BACKWARD_INDEX, (uint64_t)t);
      sel = multinomial_draw(bw, N, ao_next_uniform(&bs));
      if (sel_out) sel_out[t] = sel;
      memcpy(traj + (size_t)t * d, part + ((size_t)t * N + sel) * d, sizeof(double) * d);
      tkeys[t] = keys[(size_t)t * N + sel];
    }
    free(logb);
    free(bw);
  }
  if (st == AO_OK) {
    int changed = memcmp(traj, pg->x, sizeof(double) * n) != 0;
    memcpy(pg->x, traj, sizeof(double) * n);
    memcpy(pg->keys, tkeys, sizeof(uint64_t) * (T + 1));
    pg->last_update = changed ? 1.0 : 0.0;
    if (changed) ++pg->updates;
  }
  if (anc_out) memcpy(anc_out, anc, sizeof(int) * (size_t)(T + 1) * N);
  free(u); free(part); free(W); free(logw); free(anc); free(keys); free(traj); free(tkeys);
  return st;
}

/* fkpg.cpp:276-280 */
void ao_pg_adapt_delta(ao_pg* st, double target_rate) {
  const double n = (double)(st->iter > 1 ? st->iter : 1);
  st->delta = exp(log(st->delta) + pow(n, -0.6) * (st->last_update - target_rate));
}

/* One parallel-in-time auxiliary particle Gibbs sweep with independent
 * (gradient, kAuxObs) proposals — the checker for the GPU PIT variant.
 * Particles use the reference's addresses (fkpg.cpp:77-84); the index path is
 * drawn from the lattice law by forward log-messages and backward sampling
 * with the reference's terminal/backward index uniforms (fkpg.cpp:127-150). */
int ao_pit_pgibbs_step(const ao_target* tg, ao_pg* pg, int N, ao_stream rng, int* sel_out,
                       int* bad_t) {
  const int T = tg->T, d = tg->dx;
  const size_t n = (size_t)(T + 1) * d;
  const ao_stream it = ao_derive(rng, AO_L_ITERATION, (uint64_t)pg->iter);
  ++pg->iter;
  double* u = (double*)malloc(sizeof(double) * n);
  ao_sample_aux_obs(pg->x, T, d, pg->delta, it, u);
  aux_fk fk = {tg, u, pg->delta, AO_PG_GRADIENT};
  double* part = (double*)malloc(sizeof(double) * (size_t)(T + 1) * N * d);
  double* lw = (double*)malloc(sizeof(double) * (size_t)(T + 1) * N);
  double* alpha = (double*)malloc(sizeof(double) * (size_t)(T + 1) * N);
  double* tmp = (double*)malloc(sizeof(double) * N);
  double* W = (double*)malloc(sizeof(double) * N);
  double* traj = (double*)malloc(sizeof(double) * n);
  uint64_t* tkeys = (uint64_t*)malloc(sizeof(uint64_t) * (T + 1));
  double* mean = (double*)malloc(sizeof(double) * (2 * d + d * d + 64));
  double* cov = mean + d;
  double* r = cov + d * d;
  int st = AO_OK;
  for (int t = 0; t <= T; ++t) {
    ao_stream sst = ao_derive(it, AO_L_STEP, (uint64_t)t);
    proposal(&fk, t, NULL, mean, cov);
    for (int i = 0; i < N; ++i) {
      double* x = part + ((size_t)t * N + i) * d;
      if (i == 0) {
        memcpy(x, pg->x + (size_t)t * d, sizeof(double) * d);
      } else {
        ao_stream pi = ao_derive(sst, AO_L_PARTICLE, (uint64_t)i);
        st |= sample_proposal(&fk, t, NULL, &pi, x);
      }
      for (int k = 0; k < d; ++k) r[k] = u[(size_t)t * d + k] - x[k];
      double v = ao_log_pot(tg, t, x, &st) + ao_isotropic_log_pdf(d, r, pg->delta / 2.0);
      if (t == 0) v += ao_log_pdf(d, x, tg->m0, tg->P0, &st);
      v -= ao_log_pdf(d, x, mean, cov, &st);
      lw[(size_t)t * N + i] = v;
    }
  }
  double* dm = (double*)malloc(sizeof(double) * (size_t)N * d);
  double* dc = (double*)malloc(sizeof(double) * d * d);
  for (int i = 0; i < N; ++i) alpha[i] = lw[i];
  for (int t = 1; t <= T && st == AO_OK; ++t) {
    for (int i = 0; i < N; ++i)
      ao_dyn_mean(tg, t - 1, part + ((size_t)(t - 1) * N + i) * d, dm + (size_t)i * d);
    ao_dyn_cov(tg, t - 1, NULL, dc);
    for (int j = 0; j < N; ++j) {
      const double* xj = part + ((size_t)t * N + j) * d;
      double m = -INFINITY;
      for (int i = 0; i < N; ++i) {
        tmp[i] = alpha[(size_t)(t - 1) * N + i] + ao_log_pdf(d, xj, dm + (size_t)i * d, dc, &st);
        m = tmp[i] > m ? tmp[i] : m;
      }
      double s = 0.0;
      for (int i = 0; i < N; ++i) s += exp(tmp[i] - m);
      alpha[(size_t)t * N + j] = lw[(size_t)t * N + j] + (m + log(s));
    }
  }
  int sel = 0;
  if (st == AO_OK && normalize(alpha + (size_t)T * N, N, W, NULL) != AO_OK) {
    st = AO_E_DEGENERATE;
    if (bad_t) *bad_t = T;
  }
  if (st == AO_OK) {
    ao_stream ti = ao_derive(it, AO_L_TERMINAL_INDEX, 0);
    sel = multinomial_draw(W, N, ao_next_uniform(&ti));
    if (sel_out) sel_out[T] = sel;
    memcpy(traj + (size_t)T * d, part + ((size_t)T * N + sel) * d, sizeof(double) * d);
    for (int t = T - 1; t >= 0 && st == AO_OK; --t) {
      const double* chosen = traj + (size_t)(t + 1) * d;
      ao_dyn_cov(tg, t, NULL, dc);
      for (int i = 0; i < N; ++i) {
        ao_dyn_mean(tg, t, part + ((size_t)t * N + i) * d, dm);
        tmp[i] = alpha[(size_t)t * N + i] + ao_log_pdf(d, chosen, dm, dc, &st);
      }
      if (normalize(tmp, N, W, NULL) != AO_OK) {
        st = AO_E_DEGENERATE;
        if (bad_t) *bad_t = t;
        break;
      }
      ao_stream bs = ao_derive(it, AO_L_BACKWARD_INDEX, (uint64_t)t);
      sel = multinomial_draw(W, N, ao_next_uniform(&bs));
      if (sel_out) sel_out[t] = sel;
      memcpy(traj + (size_t)t * d, part + ((size_t)t * N + sel) * d, sizeof(double) * d);
    }
  }
  if (st == AO_OK) {
    for (int t = 0; t <= T; ++t) {
      const int s_t = sel_out ? sel_out[t] : 0;
      if (s_t == 0) {
        tkeys[t] = pg->keys[t];
      } else {
        ao_stream ks = ao_derive(ao_derive(it, AO_L_STEP, (uint64_t)t), AO_L_PM_KEY, (uint64_t)s_t);
        tkeys[t] = ao_next_key(&ks);
      }
    }
    int changed = memcmp(traj, pg->x, sizeof(double) * n) != 0;
    memcpy(pg->x, traj, sizeof(double) * n);
    memcpy(pg->keys, tkeys, sizeof(uint64_t) * (T + 1));
    pg->last_update = changed ? 1.0 : 0.0;
    if (changed) ++pg->updates;
  }
  free(u); free(part); free(lw); free(alpha); free(tmp); free(W); free(traj); free(tkeys);
  free(mean); free(dm); free(dc);
  return st;
}

/* Parallel-in-time cSMC lattice law (no reference: SPEC.md:16).  With
 * independent proposals q_t (gradient mode at the aux obs), the conditional law
 * of the index path given all particles is
 *   P(i_{0:T}) ∝ w_0(i_0) prod_{t>=1} p(x_t^{i_t} | x_{t-1}^{i_{t-1}}) w_t(i_t),
 *   w_t(i) = g_t(x) N(u_t; x, δ/2) / q_t(x) (times p(x_0)/q_0 at t = 0).
 * Forward-backward marginals of i_t (exact, O(T N^2)); path_probs receives the
 * per-time marginals [T+1][N]. */
int ao_pit_csmc_marginals(const ao_target* tg, const double* u, double delta,
                          const double* particles, int N, double* marg) {
  const int T = tg->T, d = tg->dx;
  aux_fk fk = {tg, u, delta, AO_PG_GRADIENT};
  double* lw = (double*)malloc(sizeof(double) * (size_t)(T + 1) * N);
  double* la = (double*)malloc(sizeof(double) * (size_t)(T + 1) * N);
  double* lb = (double*)malloc(sizeof(double) * (size_t)(T + 1) * N);
  double* mean = (double*)malloc(sizeof(double) * (d + d * d));
  double* cov = mean + d;
  int st = AO_OK;
  for (int t = 0; t <= T; ++t)
    for (int i = 0; i < N; ++i) {
      const double* x = particles + ((size_t)t * N + i) * d;
      /* potential without the transition term: log_pot + aux + (t==0: prior) - log q */
      double r[64];
      for (int k = 0; k < d; ++k) r[k] = u[(size_t)t * d + k] - x[k];
      double v = ao_log_pot(tg, t, x, &st) + ao_isotropic_log_pdf(d, r, delta / 2.0);
      if (t == 0) v += ao_log_pdf(d, x, tg->m0, tg->P0, &st);
      proposal(&fk, t, NULL, mean, cov);
      v -= ao_log_pdf(d, x, mean, cov, &st);
      lw[(size_t)t * N + i] = v;
    }
  /* forward log messages */
  for (int i = 0; i < N; ++i) la[i] = lw[i];
  double* tmp = (double*)malloc(sizeof(double) * N);
  for (int t = 1; t <= T; ++t)
    for (int j = 0; j < N; ++j) {
      const double* xj = particles + ((size_t)t * N + j) * d;
      double m = -INFINITY;
      for (int i = 0; i < N; ++i) {
        const double* xi = particles + ((size_t)(t - 1) * N + i) * d;
        ao_dyn_mean(tg, t - 1, xi, mean);
        ao_dyn_cov(tg, t - 1, xi, cov);
        tmp[i] = la[(size_t)(t - 1) * N + i] + ao_log_pdf(d, xj, mean, cov, &st);
        m = tmp[i] > m ? tmp[i] : m;
      }
      double s = 0.0;
      for (int i = 0; i < N; ++i) s += exp(tmp[i] - m);
      la[(size_t)t * N + j] = m + log(s) + lw[(size_t)t * N + j];
    }
  /* backward log messages */
  for (int i = 0; i < N; ++i) lb[(size_t)T * N + i] = 0.0;
  for (int t = T - 1; t >= 0; --t)
    for (int i = 0; i < N; ++i) {
      const double* xi = particles + ((size_t)t * N + i) * d;
      ao_dyn_mean(tg, t, xi, mean);
      ao_dyn_cov(tg, t, xi, cov);
      double m = -INFINITY;
      for (int j = 0; j < N; ++j) {
        const double* xj = particles + ((size_t)(t + 1) * N + j) * d;
        tmp[j] = ao_log_pdf(d, xj, mean, cov, &st) + lw[(size_t)(t + 1) * N + j] +
                 lb[(size_t)(t + 1) * N + j];
        m = tmp[j] > m ? tmp[j] : m;
      }
      double s = 0.0;
      for (int j = 0; j < N; ++j) s += exp(tmp[j] - m);
      lb[(size_t)t * N + i] = m + log(s);
    }
  for (int t = 0; t <= T; ++t) {
    double m = -INFINITY;
    for (int i = 0; i < N; ++i) {
      tmp[i] = la[(size_t)t * N + i] + lb[(size_t)t * N + i];
      m = tmp[i] > m ? tmp[i] : m;
    }
    double s = 0.0;
    for (int i = 0; i < N; ++i) s += exp(tmp[i] - m);
    for (int i = 0; i < N; ++i) marg[(size_t)t * N + i] = exp(tmp[i] - m) / s;
  }
  free(tmp); free(lw); free(la); free(lb); free(mean);
  return st;
}
