/*
 * auxmc_oracle.h — CPU restatement of the auxmc 0.1.0 hot path (arXiv 2303.00301).
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the parity checker for the B200
 * product in paper_2303_00301_b200/.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it.  The product
 * path never links or calls it.
 *
 * Every function cites the reference file:line it restates (paths relative to
 * /root/reference/proj).  Matrices are dense, row-major, double.  Where the
 * reference throws, these functions return a status code (AO_OK, AO_E_*).
 *
 * Parity pinning: the restatement is checked against the known-answer tests
 * the reference's own suites hold (tests/test_gauss.cpp, test_lgssm.cpp,
 * test_pit.cpp, test_target_auxk.cpp, test_fkpg.cpp, test_rng.cpp) — see
 * tests/test_oracle_kat.py — and against golden vectors produced by the
 * reference itself when it is compiled here (oracle/_ref).
 */
#ifndef AUXMC_ORACLE_H
#define AUXMC_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  AO_OK = 0,
  AO_E_DIM = 1,
  AO_E_FACTOR = 2,
  AO_E_DEGENERATE = 3,
  AO_E_CONTRACT = 4,
  AO_E_CONFIG = 5,
  AO_E_NOMEM = 6
};

/* Stream labels, rng.hpp:14-30 */
enum {
  AO_L_BACKWARD_NOISE = 1, AO_L_TERMINAL_DRAW = 2, AO_L_AUX_OBS = 3,
  AO_L_DNC_BRIDGE = 4, AO_L_MH_ACCEPT = 5, AO_L_ITERATION = 6, AO_L_CHAIN = 7,
  AO_L_STEP = 8, AO_L_PARTICLE = 9, AO_L_RESAMPLE = 10, AO_L_TERMINAL_INDEX = 11,
  AO_L_BACKWARD_INDEX = 12, AO_L_PM_KEY = 13, AO_L_SIMULATE = 14, AO_L_PARAM = 15
};

/* ---------------- counter RNG (rng.hpp:35-118) ---------------- */
typedef struct { uint64_t key; uint64_t counter; } ao_stream;

uint64_t ao_mix64(uint64_t z);
uint64_t ao_word_at(uint64_t key, uint64_t i);
double ao_to_unit_open(uint64_t w);
ao_stream ao_from_seed(uint64_t seed);
ao_stream ao_from_key(uint64_t key);
ao_stream ao_derive(ao_stream s, uint64_t label, uint64_t index);
double ao_next_uniform(ao_stream* s);
double ao_next_normal(ao_stream* s);
uint64_t ao_next_key(ao_stream* s);
void ao_normal_vec(ao_stream* s, int d, double* out);

/* Noise sources (rng.hpp:123-161). kind 0: StreamNoise over `base`.
 * kind 1: pre-drawn arrays addressed by (label, index).  kind 2: ProbeNoise. */
typedef struct {
  int kind;
  ao_stream base;
  int dx;
  const double* terminal;  /* [dx]            (kTerminalDraw, 0) */
  const double* backward;  /* [n_backward][dx] (kBackwardNoise, t) */
  long n_backward;
  const double* bridge;    /* [n_bridge][dx]   (kDncBridge, id) */
  long n_bridge;
  int active, cursor;      /* probe */
} ao_noise;
void ao_noise_normal(ao_noise* n, uint64_t label, uint64_t index, int dim, double* out);

/* ---------------- Gaussian primitives (gauss.cpp:13-91) ---------------- */
int ao_llt(int n, const double* a, double* l);            /* 1 on success (Eigen LLT::info) */
int ao_factor_psd(int n, const double* a, double* l);     /* jitter ladder */
int ao_chol_psd(int n, const double* a, double* l);       /* zero fast path */
void ao_llt_solve(int n, const double* l, int nrhs, const double* b, double* x);
int ao_solve_spd(int n, const double* s, int nrhs, const double* b, double* x);
double ao_log_pdf(int n, const double* x, const double* mean, const double* cov, int* status);
double ao_isotropic_log_pdf(int n, const double* resid, double var);
int ao_lu_solve(int n, const double* a, int nrhs, const double* b, double* x); /* PartialPivLU */
double ao_spectral_radius(int n, const double* a);        /* |eig|max (models.cpp:58) */

/* ---------------- LGSSM (lgssm.hpp:19-91, lgssm.cpp) ---------------- */
typedef struct {
  int T, dx, dy;
  const double *m0, *P0;
  const double *F, *b, *Q;   /* counts nF, nb, nQ in {1, T} */
  const double *H, *c, *R;   /* counts nH, nc, nR in {1, T+1} */
  int nF, nb, nQ, nH, nc, nR;
  const uint8_t* mask;       /* NULL or [T+1] */
} ao_lgssm;

typedef struct {
  double *pred_mean, *pred_cov, *filt_mean, *filt_cov; /* [T+1][dx], [T+1][dx][dx] */
  double log_marginal;
} ao_filter;

/* Symmetrizes P0/Q/R into owned copies as the Model constructor does (lgssm.cpp:20-71).
 * Caller frees with ao_lgssm_free. */
int ao_lgssm_normalize(const ao_lgssm* in, ao_lgssm* out);
void ao_lgssm_free(ao_lgssm* m);

int ao_kalman_filter(const ao_lgssm* m, const double* obs, ao_filter* fr);
int ao_backward_step(const ao_lgssm* m, const ao_filter* fr, int t, double* gain,
                     double* offset, double* cov);
int ao_backward_sample(const ao_lgssm* m, const ao_filter* fr, ao_noise* noise, double* traj);
int ao_rts_smoother(const ao_lgssm* m, const ao_filter* fr, double* mean, double* cov);
double ao_path_logpdf(const ao_lgssm* m, const double* obs, const double* traj,
                      const ao_filter* fr, int* status);
/* Dense Gaussian conditioning oracle (lgssm.cpp:201-261); posterior over stacked
 * x_{0:T} (n=(T+1)dx, n <= cap). */
int ao_dense_oracle(const ao_lgssm* m, const double* obs, int cap, double* post_mean,
                    double* post_cov, double* log_evidence);

/* ---------------- PIT (pit.cpp) ---------------- */
int ao_prefix_sample(const ao_lgssm* m, const ao_filter* fr, ao_noise* noise, double* traj,
                     int* critical_path, long* applications);
int ao_parallel_filter(const ao_lgssm* m, const double* obs, ao_filter* fr,
                       int* critical_path, long* applications);
int ao_dnc_sample(const ao_lgssm* m, const ao_filter* fr, ao_noise* noise, double* traj);
/* scan element combine on raw arrays (pit.cpp:36-51): A,b,C,eta,J for u and v */
void ao_filter_combine(int d, const double* uA, const double* ub, const double* uC,
                       const double* ueta, const double* uJ, const double* vA,
                       const double* vb, const double* vC, const double* veta,
                       const double* vJ, double* oA, double* ob, double* oC,
                       double* oeta, double* oJ);
/* Exact law of an affine sampler (pit.cpp:303-332): which 0 seq, 1 prefix, 2 dnc.
 * mean [(T+1)dx], cov [(T+1)dx]^2 */
int ao_extract_affine_law(int which, const ao_lgssm* m, const ao_filter* fr,
                          double* mean, double* cov);

/* ---------------- targets and bench models (target.cpp, models.cpp) -------- */
enum {
  AO_KIND_LGSSM = 0,      /* lgssm-synthetic (or any linear target with exact potentials) */
  AO_KIND_STOCHVOL = 1,
  AO_KIND_LORENZ63 = 2,   /* diffusion-smoothing */
  AO_KIND_SPATIO = 3,
  AO_KIND_GRID1D = 4,
  AO_KIND_LORENZ96 = 5,   /* new: d-dim Lorenz-96 diffusion, even coordinates observed */
  AO_KIND_GAUSS_GENERIC = 6 /* linear target with Gaussian potentials in generic form
                               (tests/testutil.hpp:112-140) */
};

typedef struct {
  int kind;
  int T, dx, dy, grid;
  uint64_t data_seed;
  double sv_mu, sv_phi, sv_sig2, sv_rho;
  double lz_sigma, lz_rho, lz_beta, lz_h, lz_gamma, lz_obs_var;
  double st_phi, st_kappa2, st_tau2;
  double g1_phi, g1_q, g1_m0, g1_p0;
  double l96_F, l96_h, l96_gamma, l96_obs_var;
} ao_spec;

void ao_spec_default(ao_spec* s);
int ao_latent_dim(const ao_spec* s);
int ao_obs_dim(const ao_spec* s);

/* Target over x_{0:T} (target.hpp:34-93) with owned arrays. */
typedef struct {
  int kind, T, dx, ydim;      /* ydim = data columns */
  int linear;
  double *m0, *P0;            /* dx, dx*dx */
  double *F, *b, *Q;          /* linear: counts nF (1 or T) */
  int nF;
  /* exact Gaussian potentials: q rows, per-t (count ne = 1 or T+1), mask */
  int q, ne;
  double *eH, *ec, *eR;       /* [ne][q][dx], [ne][q], [ne][q][q] */
  double *ey;                 /* [T+1][q] */
  uint8_t* emask;             /* [T+1] : potential t has an exact block */
  /* generic potential data */
  double* data;               /* [T+1][ydim] */
  uint8_t* gmask;             /* [T+1] : potential t has a generic factor */
  ao_spec spec;
} ao_target;

void ao_target_free(ao_target* t);
/* models.cpp:51-68 synth_mats */
int ao_synth_mats(const ao_spec* s, double* m0, double* b, double* P0, double* F, double* Q,
                  double* H, double* R);
/* models.cpp:162-238 */
int ao_simulate(const ao_spec* s, double* latent, double* data);
/* models.cpp:240-336 */
int ao_make_target(const ao_spec* s, const double* data, ao_target* out);
/* testutil.hpp:88-140: target from an explicit LGSSM + obs; generic=1 gives the
 * generic-potential form */
int ao_target_from_lgssm(const ao_lgssm* m, const double* obs, int generic, ao_target* out);

void ao_dyn_mean(const ao_target* tg, int t, const double* x, double* out);
void ao_dyn_jac(const ao_target* tg, int t, const double* x, double* out);
void ao_dyn_cov(const ao_target* tg, int t, const double* x, double* out);
double ao_log_pot(const ao_target* tg, int t, const double* x, int* status);
void ao_grad_pot_generic(const ao_target* tg, int t, const double* x, double* g);
void ao_grad_pot(const ao_target* tg, int t, const double* x, double* g, int* status);
double ao_log_gamma(const ao_target* tg, const double* traj, int* status);

/* ---------------- auxiliary Kalman kernel (auxk.cpp) ---------------- */
typedef struct {
  long accepted, rejected, aborted, nonfinite_gamma;
  double last_log_alpha, last_accept_prob;
} ao_kstats;

enum { AO_BACKEND_SEQ = 0, AO_BACKEND_PREFIX = 1, AO_BACKEND_DNC = 2 };

typedef struct {
  double* x;        /* [T+1][dx] */
  double delta;
  double log_gamma;
  double* grad_gen; /* [T+1][dx] */
  long iter;
  ao_kstats stats;
} ao_chain;

/* aux model construction: builds an owned ao_lgssm + obs [T+1][p] */
int ao_build_aux_lgssm(const ao_target* tg, const double* x, const double* u, double delta,
                       int zeroth_order, const double* grads, ao_lgssm* out, double** obs);
void ao_sample_aux_obs(const double* x, int T, int dx, double delta, ao_stream it, double* u);
int ao_init_chain(const ao_target* tg, const double* x0, double delta, ao_chain* st);
void ao_chain_free(ao_chain* st);
int ao_kernel_step(const ao_target* tg, ao_chain* st, ao_stream rng, int backend,
                   int parallel_filter, int zeroth_order);
double ao_mh_log_ratio(const ao_target* tg, const double* x, const double* xp,
                       const double* u, double delta, int zeroth_order, int* status);
void ao_adapt_delta(ao_chain* st, double target_rate);
/* runner.cpp:61-85 diffusion-coefficient RW-MH move; returns 1 if accepted */
int ao_gamma_move(const ao_target* tg, const double* x, double* gamma, double step,
                  ao_stream s);

/* ---------------- particle Gibbs (fkpg.cpp), gradient mode ---------------- */
typedef struct {
  double* x; uint64_t* keys; double delta; long iter; long updates; double last_update;
} ao_pg;
enum { AO_PG_PRIOR = 0, AO_PG_GRADIENT = 1, AO_PG_ADAPTED = 2 };
int ao_init_pg(const ao_target* tg, const double* x0, double delta, ao_pg* st);
void ao_pg_free(ao_pg* st);
/* One auxiliary particle Gibbs sweep (fkpg.cpp:260-274) in the given proposal mode
 * (linearized at the aux obs).  If trace is non-NULL it receives ancestors
 * [T+1][N] (int) and the selected indices [T+1] for parity checks.  On a
 * degenerate step returns AO_E_DEGENERATE and *bad_t = t. */
int ao_aux_pgibbs_step(const ao_target* tg, ao_pg* st, int N, ao_stream rng, int mode,
                       int* ancestors, int* selected, int* bad_t);
void ao_pg_adapt_delta(ao_pg* st, double target_rate);
/* Parallel-in-time auxiliary particle Gibbs sweep (independent gradient
 * proposals, lattice forward-backward over indices); sel_out [T+1] required. */
int ao_pit_pgibbs_step(const ao_target* tg, ao_pg* st, int N, ao_stream rng, int* sel_out,
                       int* bad_t);

/* ---------------- parallel-in-time cSMC with independent proposals -----------
 * No reference implementation exists.  Law-level oracle: brute
 * force path enumeration over the N^(T+1) particle lattice for tiny problems. */
int ao_pit_csmc_marginals(const ao_target* tg, const double* u, double delta,
                          const double* particles /*[T+1][N][dx]*/, int N,
                          double* path_probs /* N^(T+1) */);

#ifdef __cplusplus
}
#endif
#endif
