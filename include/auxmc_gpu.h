/*
 * auxmc_gpu.h — C ABI of the B200-native hot path of auxmc 0.1.0 (arXiv 2303.00301).
 *
 * The reference (/root/reference/proj) is a C++20 + Eigen library with no FFI
 * layer.  Its seams are free functions; each entry point below
 * replaces one of them in batched form (C chains / B independent problems) and
 * cites the reference interface it stands for.  INTEGRATION.md shows the
 * binding a maintainer would add on the reference side.
 *
 * Conventions
 *  - Plain pointers and sizes only; no C++ or torch types.
 *  - Array arguments are DEVICE pointers unless the name ends in `_host`.
 *  - Row-major dense matrices of double.  Batched arrays are batch-major:
 *    trajectories [B][T+1][dx], filter moments [B][T+1][dx] and [B][T+1][dx][dx].
 *  - Every call is asynchronous on the given stream (cudaStream_t passed as
 *    void*; NULL = legacy default stream) unless documented otherwise.
 *  - Return value: AUXMC_OK or an AUXMC_E_* code.  Exceptions of the reference
 *    (common.hpp:17-43) become codes; per-chain failures inside a batched call
 *    are reported through per-item status arrays, never by aborting the batch.
 *  - There is no CPU fallback: on a machine without a usable sm_100 device every
 *    compute entry point returns AUXMC_E_CUDA.
 */
#ifndef AUXMC_GPU_H
#define AUXMC_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (common.hpp:17-43) ---- */
#define AUXMC_OK 0
#define AUXMC_E_DIM 1          /* DimensionError */
#define AUXMC_E_FACTOR 2       /* FactorizationError */
#define AUXMC_E_DEGENERATE 3   /* DegenerateWeightsError */
#define AUXMC_E_CONTRACT 4     /* ContractError */
#define AUXMC_E_CONFIG 5       /* ConfigError */
#define AUXMC_E_CUDA 6         /* no device / launch failure */
#define AUXMC_E_ARG 7          /* invalid argument (null pointer, bad size) */
#define AUXMC_E_WORKSPACE 8    /* workspace too small */

/* ---- stream labels (rng.hpp:14-30) ---- */
#define AUXMC_L_BACKWARD_NOISE 1
#define AUXMC_L_TERMINAL_DRAW 2
#define AUXMC_L_AUX_OBS 3
#define AUXMC_L_DNC_BRIDGE 4
#define AUXMC_L_MH_ACCEPT 5
#define AUXMC_L_ITERATION 6
#define AUXMC_L_CHAIN 7
#define AUXMC_L_STEP 8
#define AUXMC_L_PARTICLE 9
#define AUXMC_L_RESAMPLE 10
#define AUXMC_L_TERMINAL_INDEX 11
#define AUXMC_L_BACKWARD_INDEX 12
#define AUXMC_L_PM_KEY 13
#define AUXMC_L_SIMULATE 14
#define AUXMC_L_PARAM 15

const char* auxmc_version(void);             /* version.hpp kVersion "0.1.0" */
const char* auxmc_status_string(int status);
/* 1 if a CUDA device with compute capability 10.x is usable, else 0. */
int auxmc_device_ok(void);
/* Last CUDA error text recorded by the library (thread-local). */
const char* auxmc_last_error(void);
/* Number of kernel launches issued by this library since load (all threads). */
unsigned long long auxmc_launch_count(void);
/* Bracket every subsequent launch with CUDA events on its stream (measurement
 * support for bench.py: per-kernel device time inside a timed region). */
void auxmc_profile_begin(void);
/* Stop bracketing; sum the durations of launches whose kernel name contains
 * kernel_substr (NULL = all). Synchronizes on the recorded events. */
int auxmc_profile_end(const char* kernel_substr, double* total_ms, long long* count);

/* ---- counter RNG, host side, bit-exact with rng.hpp:35-118 ---- */
uint64_t auxmc_rng_from_seed(uint64_t seed);                               /* RngStream::from_seed */
uint64_t auxmc_rng_derive(uint64_t key, uint64_t label, uint64_t index);   /* RngStream::derive */
double auxmc_rng_uniform(uint64_t key, uint64_t counter);                  /* next_uniform at counter */
double auxmc_rng_normal(uint64_t key, uint64_t counter);                   /* next_normal at counter */

/* Device batch generation, for tests and pre-drawn noise:
 * out[b][i][j] = normal_vec of keys[b].derive(label, index0 + i), component j.
 * (StreamNoise::normal, rng.hpp:128-137) */
int auxmc_rng_normals(const uint64_t* keys, int B, uint64_t label, uint64_t index0, int n_index,
                      int dim, double* out, void* stream);

/* ---- linear-Gaussian state-space model (lgssm.hpp:19-49) ----
 * Time-varying arrays carry a count: 1 (broadcast, lgssm.hpp:34-40) or T (F,b,Q) /
 * T+1 (H,c,R).  The library symmetrizes P0, Q, R on use exactly as the Model
 * constructor does (lgssm.cpp:20-71). */
typedef struct {
  int T, dx, dy;
  const double* m0; const double* P0;
  const double* F; int nF;
  const double* b; int nb;
  const double* Q; int nQ;
  const double* H; int nH;
  const double* c; int nc;
  const double* R; int nR;
  const uint8_t* mask;   /* NULL = every step observed, else [T+1] */
} auxmc_lgssm;

/* FilterResult (lgssm.hpp:51-55), batch-major */
typedef struct {
  double* pred_mean;   /* [B][T+1][dx] */
  double* pred_cov;    /* [B][T+1][dx][dx] */
  double* filt_mean;   /* [B][T+1][dx] */
  double* filt_cov;    /* [B][T+1][dx][dx] */
  double* log_marginal;/* [B] */
} auxmc_filter_result;

/* Kalman filtering of B observation sequences obs [B][T+1][dy] under one model.
 * mode 0: sequential covariance filter (lgssm::kalman_filter, lgssm.cpp:73-112)
 * mode 1: parallel-in-time scan filter (pit::parallel_filter, pit.cpp:117-188)
 * status[B] receives per-sequence codes. */
int auxmc_kalman_filter(const auxmc_lgssm* model, const double* obs, int B, int mode,
                        auxmc_filter_result* out, int* status, void* workspace,
                        size_t workspace_bytes, void* stream);
size_t auxmc_kalman_filter_workspace(const auxmc_lgssm* model, int B, int mode);

/* ---- time-sharded scan filter (pit::parallel_filter, pit.cpp:117-188, over G ranks)
 * One observation sequence; the horizon's block tree (blocks of LB steps,
 * super-blocks of SB = LB*LB steps, nsup of them) depends only on T.  A rank owns
 * the super-blocks [sup_lo, sup_hi) (contiguous, any split) and runs:
 *   1. auxmc_tshard_filter_local: elements, block and super-block aggregates of its
 *      range; writes its (sup_hi - sup_lo) aggregates, elem_doubles each, to sup_out;
 *   2. the caller all-gathers every rank's aggregates, in super-block order, into
 *      sup_all (nsup * elem_doubles) — the only exchange;
 *   3. auxmc_tshard_filter_finish: carries, filtered and predictive moments for
 *      t in [sup_lo*SB, min(sup_hi*SB, T+1)) (plus the predictive moments at the
 *      range end) written into full-length result arrays, and the log-likelihood
 *      partial sum of each owned super-block into ll_out;
 *   4. log_marginal = auxmc_tshard_sum over all ranks' partials in order.
 * Every split (G = 1, 2, 4, 8, ...) gives bit-identical results. */
int auxmc_tshard_geometry(int T, int dx, int* LB, int* nblk, int* nsup, int* SB,
                          int* elem_doubles);
size_t auxmc_tshard_filter_workspace(const auxmc_lgssm* model);
int auxmc_tshard_filter_local(const auxmc_lgssm* model, const double* obs, int sup_lo,
                              int sup_hi, void* workspace, size_t workspace_bytes,
                              double* sup_out, int* status, void* stream);
int auxmc_tshard_filter_finish(const auxmc_lgssm* model, const double* obs, int sup_lo,
                               int sup_hi, void* workspace, size_t workspace_bytes,
                               const double* sup_all, auxmc_filter_result* out, double* ll_out,
                               int* status, void* stream);
int auxmc_tshard_sum(const double* partials, int n, double* out, void* stream);


/* ---- noise sources (rng.hpp:123-137) ----
 * kind 0 (stream): per-problem stream keys; draws at keys[b].derive(label, index).
 * kind 1 (pre-drawn): arrays addressed by (label, index); the NoiseSource
 *   analogue used for strict parity and for affine-law probing. */
#define AUXMC_NOISE_STREAM 0
#define AUXMC_NOISE_PREDRAWN 1
typedef struct {
  int kind;
  const uint64_t* keys;       /* [B] */
  const double* terminal;     /* [B][dx]            (kTerminalDraw, 0) */
  const double* backward;     /* [B][T][dx]         (kBackwardNoise, t) */
  const double* bridge;       /* [B][n_bridge][dx]  (kDncBridge, node id) */
  long long n_bridge;
} auxmc_noise;

/* Number of bridge ids a pre-drawn DnC noise array must cover for horizon T
 * (heap ids of the BFS segment tree, pit.cpp:214-234). */
long long auxmc_dnc_bridge_count(int T);

/* ---- time-sharded prefix sampler (pit::prefix_sample, pit.cpp:78-115, one path)
 * On the same time ranges as the sharded filter ([t_lo, t_hi) of the rank's
 * super-blocks; sampler blocks of Lb steps, P of them, never straddle a range):
 *   1. auxmc_tshard_prefix_local: backward elements of the range (the sharded
 *      filter result supplies the predictive covariance at t_hi), the rows
 *      (A_k | a_k), d*d + d doubles, of its blocks into blk_out, and — on the rank
 *      with t_hi == T+1 — the terminal draw x_T into xT_out;
 *   2. the caller all-gathers the rows of all P blocks in order and x_T;
 *   3. auxmc_tshard_prefix_finish: the serial block carry (all ranks, same bits)
 *      and the path for the range.  Noise: stream keys or pre-drawn, B = 1. */
int auxmc_tshard_prefix_geometry(int T, int* Lb, int* P);
size_t auxmc_tshard_prefix_workspace(const auxmc_lgssm* model);
int auxmc_tshard_prefix_local(const auxmc_lgssm* model, const auxmc_filter_result* fr,
                              const auxmc_noise* noise, int t_lo, int t_hi, void* workspace,
                              size_t workspace_bytes, double* blk_out, double* xT_out,
                              double* traj, int* status, void* stream);
int auxmc_tshard_prefix_finish(const auxmc_lgssm* model, const auxmc_noise* noise, int t_lo,
                               int t_hi, void* workspace, size_t workspace_bytes,
                               const double* blk_all, const double* xT, double* traj,
                               void* stream);

/* Pathwise posterior draws of B paths traj [B][T+1][dx] from filter results.
 * fr_shared = 1: one filter result (B_fr = 1) shared by all paths (the C2
 * workload: one model, many chains); 0: one per path.
 *   sampler 0: lgssm::backward_sample (lgssm.cpp:151-177)
 *   sampler 1: pit::prefix_sample     (pit.cpp:78-115)
 *   sampler 2: pit::dnc_sample        (pit.cpp:192-301)
 * status[B] receives per-path codes. */
#define AUXMC_SAMPLER_SEQ 0
#define AUXMC_SAMPLER_PREFIX 1
#define AUXMC_SAMPLER_DNC 2
int auxmc_sample_paths(const auxmc_lgssm* model, const auxmc_filter_result* fr, int fr_shared,
                       const auxmc_noise* noise, int B, int sampler, double* traj, int* status,
                       void* workspace, size_t workspace_bytes, void* stream);
size_t auxmc_sample_paths_workspace(const auxmc_lgssm* model, int fr_shared, int B, int sampler);

/* lgssm::rts_smoother (lgssm.cpp:114-127) for B filter results (batch-major):
 * smoothed marginals mean [B][T+1][dx], cov [B][T+1][dx][dx]; status[B]. */
int auxmc_rts_smoother(const auxmc_lgssm* model, const auxmc_filter_result* fr, int B,
                       double* mean, double* cov, int* status, void* workspace,
                       size_t workspace_bytes, void* stream);
size_t auxmc_rts_smoother_workspace(const auxmc_lgssm* model, int B);

/* pit::extract_affine_law (pit.cpp:303-332) for sampler 0/1/2 on one filter
 * result: the exact Gaussian law N(mean, cov) of the sampled path over the flat
 * index t*dx + j, from the zero noise and every basis noise vector pushed through
 * the sampler as one pre-drawn batch.  mean [n], cov [n][n], n = (T+1)*dx;
 * status[0] = the worst sampler status.  Memory grows as n^2 (a test-scale tool,
 * like the reference's). */
int auxmc_affine_law(const auxmc_lgssm* model, const auxmc_filter_result* fr, int sampler,
                     double* mean, double* cov, int* status, void* workspace,
                     size_t workspace_bytes, void* stream);
size_t auxmc_affine_law_workspace(const auxmc_lgssm* model, int sampler);

/* testhooks::flip_backward_gain (testhooks.hpp:11): negate every backward gain
 * (a deliberate bug the law checks must catch, runner.cpp:301-312). */
int auxmc_test_flip_backward_gain(int on);
/* Test hook: 1 routes the auxiliary step's sequential filter through the generic
 * (d+q)-dimensional filter even where the fused direct-observation filter applies
 * (auxmc_target::exact_sel); the parity tests compare the two.  Host-side switch. */
int auxmc_test_force_generic_filter(int on);
/* Test hook: device buffer [C] that receives the forward filter's log p(z) of each
 * auxiliary step (NULL: off).  Host-side switch. */
int auxmc_test_capture_log_marginal(double* dev_out);
/* Test hook: 0 makes every step of the scan filter's prefix chains a full combine
 * and every backward element a full build; 1 (default) lets a chain whose element
 * matrices repeat (time-invariant model) continue with vector-only steps once the
 * filtered covariance reaches a fixed point, and lets the recovery and the
 * backward elements (dense shared F) keep the matrices of a step whose covariance
 * inputs repeat the previous step's bits (same results either way; pfilter_gen.cu,
 * sample.cu).  Host-side switch. */
int auxmc_test_pfg_fixed_point(int on);
/* Test hook: vector-only scan-filter steps taken since the last reset (reset != 0
 * zeroes the device counter afterwards); -1 without a device. */
long long auxmc_test_pfg_fixed_point_steps(int reset);

/* Host-buffer convenience entry for the reference-facing facade: copies the
 * model, filter result and noise keys to the device, draws B paths and copies
 * them back into traj_host [B][T+1][dx] (pinned or pageable).  All host pointers. */
int auxmc_sample_paths_host(const auxmc_lgssm* model_host, const auxmc_filter_result* fr_host,
                            int fr_shared, const uint64_t* keys_host, int B, int sampler,
                            double* traj_host, int* status_host);

/* lgssm::path_logpdf (lgssm.cpp:179-199) for B paths traj [B][T+1][dx] against
 * observations obs [B or 1][T+1][dy] and filter results (fr_shared as above). */
int auxmc_path_logpdf(const auxmc_lgssm* model, const double* obs, int obs_shared,
                      const double* traj, const auxmc_filter_result* fr, int fr_shared, int B,
                      double* out, int* status, void* stream);

/* ---- targets (target.hpp:34-93) and bench models (models.hpp:16-54) ----
 * Model closures become compiled device functors selected by `kind`. */
#define AUXMC_KIND_LGSSM 0          /* linear dynamics, exact Gaussian potentials */
#define AUXMC_KIND_STOCHVOL 1       /* models.cpp:113-128, :261-278 */
#define AUXMC_KIND_LORENZ63 2       /* diffusion-smoothing, models.cpp:70-85, :280-297 */
#define AUXMC_KIND_SPATIO 3         /* models.cpp:88-111, :299-317 */
#define AUXMC_KIND_GRID1D 4         /* models.cpp:319-333 */
#define AUXMC_KIND_LORENZ96 5       /* new: Lorenz-96 diffusion, even coordinates observed */
#define AUXMC_KIND_GAUSS_GENERIC 6  /* linear, Gaussian potentials in generic form */
/* Test-only generic potentials reaching the reference's failure semantics on the device
 * (1-d linear dynamics m0 = 0, P0 = 0.04, F = 0.5, b = 0, Q = 0.04):                    */
#define AUXMC_KIND_TEST_ABORT 7     /* log g = -x^2/2, grad NaN for |x| > 0.5   (test_target_auxk.cpp:374-392) */
#define AUXMC_KIND_TEST_SUPPORT 8   /* log g = -inf for x > 0.4, grad 0         (test_target_auxk.cpp:394-414) */
#define AUXMC_KIND_TEST_COLLAPSE 9  /* log g_t = -inf at t = 2, else 0          (test_fkpg.cpp:447-465) */

typedef struct {
  int kind;
  int T, dx;
  int ydim;                 /* data columns */
  int linear;               /* 1: F,b,Q below; 0: tractable (kind-specific functors) */
  const double* m0; const double* P0;
  const double* F; const double* b; const double* Q; int nF;   /* count 1 or T */
  /* exact Gaussian potential rows q = max_exact_rows (target.cpp:65-70) */
  int q; int ne;            /* ne = 1 or T+1 */
  int exact_tv;             /* 1 if the exact blocks differ across t (ne > 1, or emask mixed) */
  const double* eH; const double* ec; const double* eR;   /* [ne][q][dx], [ne][q], [ne][q][q] */
  const double* ey;         /* [T+1][q] */
  const uint8_t* emask;     /* [T+1] 1 where an exact block exists */
  const double* data;       /* [T+1][ydim] generic-potential data */
  const uint8_t* gmask;     /* [T+1] 1 where a generic factor exists */
  /* GAUSS_GENERIC blocks: [ne][ydim][dx], [ne][ydim], [ne][ydim][ydim] */
  const double* gH; const double* gc; const double* gR;
  /* kind parameters (ModelSpec fields) */
  double lz_sigma, lz_rho, lz_beta, lz_h;
  double l96_F, l96_h;
  /* 1: every exact row has one nonzero, a 1, in a distinct state column, R_e is diagonal
   * positive and ne = 1 (the diffusion-smoothing models; any target with q = 0).  The
   * auxiliary step then filters with the fused direct-observation filter (filter_direct.cu)
   * and, for Lorenz-96, never materializes the dynamics Jacobian.  The kernel re-checks
   * the structure and marks the chain's filter status 3 if it does not hold; 0 is always
   * valid (generic filter). */
  int exact_sel;
} auxmc_target;

/* ---- auxiliary Kalman MH kernel (auxk.hpp:15-79) ---- */
#define AUXMC_BACKEND_SEQ 0
#define AUXMC_BACKEND_PREFIX 1
#define AUXMC_BACKEND_DNC 2
typedef struct {
  int backend;          /* KernelOptions::backend */
  int parallel_filter;  /* KernelOptions::parallel_filter */
  int zeroth_order;     /* KernelOptions::zeroth_order */
} auxmc_kernel_options;

/* KernelStats (auxk.hpp:41-48), one per chain, device memory */
typedef struct {
  long long accepted, rejected, aborted, nonfinite_gamma;
  double last_log_alpha, last_accept_prob;
} auxmc_kernel_stats;

/* Batched chain state (AuxChainState, auxk.hpp:50-57), device arrays over C chains. */
typedef struct {
  int C;
  double* x;            /* [C][T+1][dx] */
  double* delta;        /* [C] */
  double* log_gamma;    /* [C] */
  double* grad_gen;     /* [C][T+1][dx] */
  long long* iter;      /* [C] */
  auxmc_kernel_stats* stats;  /* [C] */
  const uint64_t* root_keys;  /* [C] chain roots (from_seed(seed).derive(kChain, c)) */
} auxmc_chains;

/* auxk::init_chain (auxk.cpp:120-128) for every chain: log_gamma and grad_gen from x. */
int auxmc_init_chains(const auxmc_target* target, auxmc_chains* chains, void* workspace,
                      size_t workspace_bytes, void* stream);
/* auxk::kernel_step (auxk.cpp:130-198) for every chain. */
int auxmc_aux_kernel_step(const auxmc_target* target, auxmc_chains* chains,
                          const auxmc_kernel_options* opts, void* workspace,
                          size_t workspace_bytes, void* stream);
size_t auxmc_aux_kernel_workspace(const auxmc_target* target, int C,
                                  const auxmc_kernel_options* opts);
/* auxk::adapt_delta (auxk.cpp:213-218) for every chain. */
int auxmc_adapt_delta(auxmc_chains* chains, double target_rate, void* stream);
/* gamma_move (bench/runner.cpp:61-85): random-walk MH on log γ, the diffusion
 * coefficient of a Lorenz target (Q = h γ² I; Lorenz-63 as in the reference, Lorenz-96
 * with the same density at d = dx), N(0, 1) prior on log γ.  x [C][T+1][dx] device
 * paths; per chain the stream root_keys[c].derive(kParam = 15, iter) (runner.cpp:160-161);
 * gamma [C] updated in place on acceptance, moved [C] = 1 if accepted.  The caller
 * rebuilds the chain's target with the new γ, as runner.cpp:162-167 does.
 * AUXMC_E_CONFIG for a non-Lorenz target. */
int auxmc_gamma_move(const auxmc_target* target, int C, const double* x,
                     const uint64_t* root_keys, long long iter, double step, double* gamma,
                     int* moved, void* stream);

/* ---- time-sharded auxiliary Kalman step (one chain, kernel_step, auxk.cpp:130-198,
 * with the prefix backend and the scan filter split over ranks; tshard.py drives it).
 * Rank r owns the time range [t_lo, t_hi) of whole filter super-blocks (t_hi = T+1 on
 * the last rank) and keeps the chain's path valid on [t_lo-1, t_hi] (halo rows):
 *   begin:  iteration key, aux observations and the surrogate LGSSM at x on the halo'd
 *           range (model_out; pseudo-observations at *z_out);
 *   caller: sharded filter of (model, z), sharded prefix draw with the key at *it_out
 *           into *prop_out on [t_lo, t_hi), then the halo rows x'_{t_lo-1}, x'_{t_hi}
 *           from the neighbours (d doubles each);
 *   middle: per-t terms of log q(x'|x) and log gamma(x') on [t_lo, t_hi) summed per
 *           super-block into part_out[:, 0:2], gradients at x', surrogate at x';
 *   caller: sharded reverse filter;
 *   end:    per-t terms of log q(x|x') and both aux likelihoods -> part_out[:, 2:5];
 *   caller: all-gather of every rank's super-block partials and flags (a few KB);
 *   decide: the sums in super-block order, the MH decision (every rank identical), the
 *           accepted path on the halo'd range.
 * part_out: [owned super-blocks][5]; flags_out: int[8] of this rank (filter / sampler /
 * path-logpdf / log-gamma factor failures, non-finite gradients), max-reduced by the
 * caller into decide's flags.  Every split gives the same bits: every sum is per
 * super-block in t order, then over super-blocks in order. */
size_t auxmc_tshard_aux_workspace(const auxmc_target* target);
int auxmc_tshard_aux_begin(const auxmc_target* target, auxmc_chains* chains,
                           const auxmc_kernel_options* opts, void* workspace,
                           size_t workspace_bytes, int t_lo, int t_hi, auxmc_lgssm* model_out,
                           double** z_out, double** prop_out, uint64_t** it_out, void* stream);
int auxmc_tshard_aux_middle(const auxmc_target* target, auxmc_chains* chains,
                            const auxmc_kernel_options* opts, void* workspace,
                            size_t workspace_bytes, int t_lo, int t_hi, double* part_out,
                            int* flags_out, void* stream);
int auxmc_tshard_aux_end(const auxmc_target* target, auxmc_chains* chains,
                         const auxmc_kernel_options* opts, void* workspace, size_t workspace_bytes,
                         int t_lo, int t_hi, double* part_out, int* flags_out, void* stream);
int auxmc_tshard_aux_decide(const auxmc_target* target, auxmc_chains* chains, void* workspace,
                            size_t workspace_bytes, int t_lo, int t_hi, const double* parts_all,
                            int nsup, const double* log_marginal_fwd,
                            const double* log_marginal_rev, const int* flags, void* stream);
int auxmc_copy_device(void* dst, const void* src, size_t bytes, void* stream);
/* target.log_gamma (target.cpp:100-108) of B paths. */
int auxmc_log_gamma(const auxmc_target* target, const double* traj, int B, double* out,
                    int* status, void* stream);

/* ---- auxiliary particle Gibbs (fkpg.hpp:61-109) ---- */
#define AUXMC_PG_PRIOR 0
#define AUXMC_PG_GRADIENT 1
#define AUXMC_PG_ADAPTED 2
#define AUXMC_CSMC_REFERENCE 0   /* sequential cSMC with multinomial resampling (fkpg.cpp:44-152) */
#define AUXMC_CSMC_PIT 1         /* parallel-in-time cSMC, independent proposals (new) */
typedef struct {
  int C, N;
  double* x;            /* [C][T+1][dx] reference trajectories */
  uint64_t* keys;       /* [C][T+1] reference aux keys */
  double* delta;        /* [C] */
  long long* iter;      /* [C] */
  long long* updates;   /* [C] */
  double* last_update;  /* [C] */
  const uint64_t* root_keys;  /* [C] */
  int* status;          /* [C] AUXMC_OK or AUXMC_E_DEGENERATE */
  int* bad_t;           /* [C] step named by DegenerateWeightsError */
  int* ancestors;       /* optional [C][T+1][N] trace of ancestor indices (NULL = off) */
  int* selected;        /* optional [C][T+1] trace of selected indices (NULL = off) */
  int pm_kind;          /* pseudo-marginal potentials (fkpg.cpp:233-250 pm_potential), AUXMC_PM_* */
} auxmc_pg_chains;
/* Pseudo-marginal wrappers of the auxiliary FK potentials (reference cSMC only).  The
 * reference wraps any user estimator (t, x_prev, x, key) -> est >= 0; on the device the
 * estimator is one of a fixed family evaluated from the particle's aux key
 * (st.derive(kPmKey, i).next_key(), fkpg.cpp:72), log g' = est > 0 ? log(est) : -inf, and
 * NaN or est < 0 is the reference's ContractError (AUXMC_E_CONTRACT, bad_t = t):       */
#define AUXMC_PM_NONE 0       /* the plain potentials */
#define AUXMC_PM_TWO_POINT 1  /* est = exp(log g) * (U(key) < 0.5 ? 0.5 : 1.5), unbiased
                                 (acceptance.cpp:249-290, test_fkpg.cpp:402-434) */
#define AUXMC_PM_EXACT 2      /* est = exp(log g): zero variance (test_fkpg.cpp:365-381) */
#define AUXMC_PM_NEGATIVE 3   /* est = -0.1: contract violation (test_fkpg.cpp:436-445) */

int auxmc_aux_pgibbs_step(const auxmc_target* target, auxmc_pg_chains* chains, int mode,
                          int variant, void* workspace, size_t workspace_bytes, void* stream);
size_t auxmc_aux_pgibbs_workspace(const auxmc_target* target, int C, int N, int variant);
int auxmc_pg_adapt_delta(auxmc_pg_chains* chains, double target_rate, void* stream);

/* ---- host-side bench models (models.cpp:51-68, :162-238, :240-336) ----
 * Spec mirrors ModelSpec (models.hpp:16-54) plus the Lorenz-96 block. */
typedef struct {
  int kind;
  int T, dx, dy, grid;
  uint64_t data_seed;
  double sv_mu, sv_phi, sv_sig2, sv_rho;
  double lz_sigma, lz_rho, lz_beta, lz_h, lz_gamma, lz_obs_var;
  double st_phi, st_kappa2, st_tau2;
  double g1_phi, g1_q, g1_m0, g1_p0;
  double l96_F, l96_h, l96_gamma, l96_obs_var;
} auxmc_model_spec;

void auxmc_spec_default(auxmc_model_spec* spec);
int auxmc_latent_dim(const auxmc_model_spec* spec);
int auxmc_obs_dim(const auxmc_model_spec* spec);
/* bench::simulate — host buffers latent_host [T+1][dx], data_host [T+1][ydim]. */
int auxmc_simulate(const auxmc_model_spec* spec, double* latent_host, double* data_host);
/* bench::synth_mats for lgssm-synthetic, host buffers (row-major). */
int auxmc_synth_mats(const auxmc_model_spec* spec, double* m0, double* b, double* P0, double* F,
                     double* Q, double* H, double* R);
/* Host-side parameter arrays of make_target for kinds STOCHVOL / SPATIO / GRID1D /
 * LORENZ63 / LORENZ96 (m0 [dx], P0 [dx][dx], Q [dx][dx]; F,b for linear kinds). */
int auxmc_target_params(const auxmc_model_spec* spec, double* m0, double* P0, double* F,
                        double* b, double* Q);

#ifdef __cplusplus
}
#endif
#endif /* AUXMC_GPU_H */
