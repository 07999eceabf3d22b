// ref_bridge.cpp — TEST INFRASTRUCTURE: a flat extern "C" surface over the REFERENCE's
// own C++ API (compiled unmodified into oracle/_ref/libauxmc_ref.so by oracle/ref.mk),
// so Python parity tests and bench.py's CPU legs can execute the reference itself.
// Nothing here re-implements an algorithm: every entry point calls the reference
// function named in its comment.  The one addition is the Lorenz-96 target (C3), which
// the reference lacks: it is built with the reference's own GenSSMTarget::tractable
// (target.cpp:29-45) from closures modelled on models.cpp:280-297.
//
// Arrays are row-major float64 (C order), as in oracle/auxmc_oracle.h.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <limits>
#include <memory>
#include <string>
#include <vector>

#include "auxmc/auxk.hpp"
#include "auxmc/bench/config.hpp"
#include "auxmc/bench/grid_hmm.hpp"
#include "auxmc/bench/models.hpp"
#include "auxmc/bench/runner.hpp"
#include "auxmc/fkpg.hpp"
#include "auxmc/lgssm.hpp"
#include "auxmc/pit.hpp"
#include "auxmc/rng.hpp"
#include "auxmc/target.hpp"
#include "auxmc/testhooks.hpp"
#include "testutil.hpp"  // the reference's own test targets (proj/tests/testutil.hpp:86-140)

using namespace auxmc;

namespace {

// Same layout as oracle/auxmc_oracle.h ao_spec, so pyoracle.Spec passes through.
struct rb_spec {
  int kind;
  int T, dx, dy, grid;
  std::uint64_t data_seed;
  double sv_mu, sv_phi, sv_sig2, sv_rho;
  double lz_sigma, lz_rho, lz_beta, lz_h, lz_gamma, lz_obs_var;
  double st_phi, st_kappa2, st_tau2;
  double g1_phi, g1_q, g1_m0, g1_p0;
  double l96_F, l96_h, l96_gamma, l96_obs_var;
};

enum { K_LGSSM = 0, K_STOCHVOL = 1, K_L63 = 2, K_SPATIO = 3, K_GRID1D = 4, K_L96 = 5 };
enum { RB_OK = 0, RB_E_DIM = 1, RB_E_FACTOR = 2, RB_E_DEGENERATE = 3, RB_E_CONTRACT = 4,
       RB_E_CONFIG = 5, RB_E_OTHER = 9 };

const char* kind_name(int k) {
  switch (k) {
    case K_LGSSM: return "lgssm-synthetic";
    case K_STOCHVOL: return "stochvol";
    case K_L63: return "diffusion-smoothing";
    case K_SPATIO: return "spatio-temporal";
    case K_GRID1D: return "grid-1d-test";
    default: return "";
  }
}

bench::ModelSpec to_spec(const rb_spec& s) {
  bench::ModelSpec m;
  m.kind = kind_name(s.kind);
  m.T = s.T;
  m.dx = s.dx;
  m.dy = s.dy;
  m.grid = s.grid;
  m.data_seed = s.data_seed;
  m.sv_mu = s.sv_mu, m.sv_phi = s.sv_phi, m.sv_sig2 = s.sv_sig2, m.sv_rho = s.sv_rho;
  m.lz_sigma = s.lz_sigma, m.lz_rho = s.lz_rho, m.lz_beta = s.lz_beta;
  m.lz_h = s.lz_h, m.lz_gamma = s.lz_gamma, m.lz_obs_var = s.lz_obs_var;
  m.st_phi = s.st_phi, m.st_kappa2 = s.st_kappa2, m.st_tau2 = s.st_tau2;
  m.g1_phi = s.g1_phi, m.g1_q = s.g1_q, m.g1_m0 = s.g1_m0, m.g1_p0 = s.g1_p0;
  return m;
}

Mat mat_in(const double* p, int r, int c) {
  Mat m(r, c);
  for (int i = 0; i < r; ++i)
    for (int j = 0; j < c; ++j) m(i, j) = p[i * c + j];
  return m;
}
Vec vec_in(const double* p, int n) {
  Vec v(n);
  for (int i = 0; i < n; ++i) v[i] = p[i];
  return v;
}
void mat_out(const Mat& m, double* p) {
  for (long i = 0; i < m.rows(); ++i)
    for (long j = 0; j < m.cols(); ++j) p[i * m.cols() + j] = m(i, j);
}
void vec_out(const Vec& v, double* p) {
  for (long i = 0; i < v.size(); ++i) p[i] = v[i];
}

template <class F>
int guarded(F f) {
  try {
    f();
    return RB_OK;
  } catch (const FactorizationError&) {
    return RB_E_FACTOR;
  } catch (const DimensionError&) {
    return RB_E_DIM;
  } catch (const DegenerateWeightsError&) {
    return RB_E_DEGENERATE;
  } catch (const ContractError&) {
    return RB_E_CONTRACT;
  } catch (const ConfigError&) {
    return RB_E_CONFIG;
  } catch (const std::exception&) {
    return RB_E_OTHER;
  }
}

// Lorenz-96 (d = dx, cyclic): f_i = (x_{i+1} - x_{i-2}) x_{i-1} - x_i + F; Euler step h,
// Q = h gamma^2 I, exact observations of the even coordinates with variance obs_var,
// m0 = F 1 + 0.01 e_0, P0 = I (pattern of models.cpp:280-297).
auxk::GenSSMTarget l96_target(const rb_spec& s, const Mat& data) {
  const int d = s.dx, T = s.T, q = (d + 1) / 2;
  const double F = s.l96_F, h = s.l96_h;
  auto drift = [d, F](const Vec& x) {
    Vec f(d);
    for (int i = 0; i < d; ++i)
      f[i] = (x[(i + 1) % d] - x[(i + d - 2) % d]) * x[(i + d - 1) % d] - x[i] + F;
    return f;
  };
  auto jac = [d](const Vec& x) {
    Mat j = Mat::Zero(d, d);
    for (int i = 0; i < d; ++i) {
      const int ip1 = (i + 1) % d, im1 = (i + d - 1) % d, im2 = (i + d - 2) % d;
      j(i, ip1) += x[im1];
      j(i, im2) -= x[im1];
      j(i, im1) += x[ip1] - x[im2];
      j(i, i) -= 1.0;
    }
    return j;
  };
  Mat H = Mat::Zero(q, d);
  for (int k = 0; k < q; ++k) H(k, 2 * k) = 1.0;
  std::vector<auxk::Potential> pots(T + 1);
  for (int t = 0; t <= T; ++t)
    pots[t].exact = auxk::ExactGaussPotential{H, Vec::Zero(q), Mat(s.l96_obs_var * Mat::Identity(q, q)),
                                              Vec(data.row(t).transpose())};
  const Mat Q = h * s.l96_gamma * s.l96_gamma * Mat::Identity(d, d);
  Vec m0 = Vec::Constant(d, F);
  m0[0] += 0.01;
  return auxk::GenSSMTarget::tractable(
      T, d, m0, Mat::Identity(d, d),
      [drift, h](int, const Vec& x) { return Vec(x + h * drift(x)); },
      [jac, h, d](int, const Vec& x) { return Mat(Mat::Identity(d, d) + h * jac(x)); },
      [Q](int, const Vec&) { return Q; }, std::move(pots));
}

struct PredrawnNoise final : NoiseSource {
  // Addresses as the reference's samplers request them: (kTerminalDraw, 0),
  // (kBackwardNoise, t), (kDncBridge, node id).
  const double *terminal, *backward, *bridge;
  long n_backward, n_bridge;
  Vec normal(std::uint64_t label, std::uint64_t index, int dim) override {
    const double* src = nullptr;
    if (label == stream::kTerminalDraw) src = terminal;
    else if (label == stream::kBackwardNoise && static_cast<long>(index) < n_backward)
      src = backward + index * dim;
    else if (label == stream::kDncBridge && static_cast<long>(index) < n_bridge)
      src = bridge + index * dim;
    Vec v = Vec::Zero(dim);
    if (src)
      for (int i = 0; i < dim; ++i) v[i] = src[i];
    return v;
  }
};

}  // namespace

extern "C" {

// ---------------------------------------------------------------- RNG (rng.hpp:35-118)
std::uint64_t rb_from_seed(std::uint64_t seed) { return RngStream::from_seed(seed).key(); }
std::uint64_t rb_derive(std::uint64_t key, std::uint64_t label, std::uint64_t index) {
  return RngStream::from_key(key).derive(label, index).key();
}
// Draws n values from the stream with this key, counters 0..n-1:
// kind 0 next_normal, 1 next_uniform, 2 next_key (as doubles' bit patterns in out_u64).
void rb_draw(std::uint64_t key, int kind, int n, double* out, std::uint64_t* out_u64) {
  RngStream s = RngStream::from_key(key);
  for (int i = 0; i < n; ++i) {
    if (kind == 0) out[i] = s.next_normal();
    else if (kind == 1) out[i] = s.next_uniform();
    else out_u64[i] = s.next_key();
  }
}

// ---------------------------------------------------------------- models (models.cpp)
int rb_simulate(const rb_spec* s, double* latent, double* data) {
  return guarded([&] {
    bench::SimResult r = bench::simulate(to_spec(*s));
    mat_out(r.latent, latent);
    if (r.data.size()) mat_out(r.data, data);
  });
}

void* rb_target_new(const rb_spec* s, const double* data, int ydim, int* status) {
  auxk::GenSSMTarget* out = nullptr;
  *status = guarded([&] {
    const Mat d = mat_in(data, s->T + 1, ydim);
    out = new auxk::GenSSMTarget(s->kind == K_L96 ? l96_target(*s, d)
                                                  : bench::make_target(to_spec(*s), d));
  });
  return out;
}
void rb_target_free(void* t) { delete static_cast<auxk::GenSSMTarget*>(t); }

double rb_log_gamma(const void* tg, const double* x, int* status) {
  const auto& t = *static_cast<const auxk::GenSSMTarget*>(tg);
  double v = NAN;
  *status = guarded([&] { v = t.log_gamma(mat_in(x, t.horizon() + 1, t.dx())); });
  return v;
}
int rb_grad_pot(const void* tg, int t, const double* x, int generic_only, double* out) {
  const auto& g = *static_cast<const auxk::GenSSMTarget*>(tg);
  return guarded([&] {
    const Vec xv = vec_in(x, g.dx());
    vec_out(generic_only ? g.grad_pot_generic(t, xv) : g.grad_pot(t, xv), out);
  });
}
double rb_log_pot(const void* tg, int t, const double* x) {
  const auto& g = *static_cast<const auxk::GenSSMTarget*>(tg);
  return g.log_pot(t, vec_in(x, g.dx()));
}

// Test-only targets: the reference's own failure-path test targets, closures verbatim in
// meaning (kind 7: test_target_auxk.cpp:374-392, 8: :394-414, 9: a collapse at t = 2 as in
// test_fkpg.cpp:447-465, on the same 1-d linear dynamics).
void* rb_target_test(int kind, int T) {
  std::vector<auxk::Potential> pots(T + 1);
  for (int t = 0; t <= T; ++t) {
    auto& p = pots[t];
    if (kind == 7) {
      p.log_g = [](const Vec& x) { return -0.5 * x[0] * x[0]; };
      p.grad_log_g = [](const Vec& x) {
        return Vec(Vec::Constant(1, std::abs(x[0]) > 0.5 ? std::nan("") : -x[0]));
      };
    } else if (kind == 8) {
      p.log_g = [](const Vec& x) { return x[0] > 0.4 ? -std::numeric_limits<double>::infinity() : 0.0; };
      p.grad_log_g = [](const Vec&) { return Vec(Vec::Zero(1)); };
    } else {
      p.log_g = [t](const Vec&) { return t == 2 ? -std::numeric_limits<double>::infinity() : 0.0; };
      p.grad_log_g = [](const Vec&) { return Vec(Vec::Zero(1)); };
    }
  }
  return new auxk::GenSSMTarget(auxk::GenSSMTarget::linear(
      T, Vec::Zero(1), Mat::Constant(1, 1, 0.04), {Mat::Constant(1, 1, 0.5)}, {Vec::Zero(1)},
      {Mat::Constant(1, 1, 0.04)}, std::move(pots)));
}

// The LGSSM posterior as a target: exact Gaussian potentials (testutil.hpp:88-108) or the
// same factors as generic log-potentials (:112-140).
void* rb_target_lgssm(const void* model, const double* obs, int generic) {
  const auto& m = *static_cast<const lgssm::Model*>(model);
  const Mat o = mat_in(obs, m.horizon() + 1, m.dy());
  return new auxk::GenSSMTarget(generic ? testutil::lgssm_target_generic(m, o)
                                        : testutil::lgssm_target_exact(m, o));
}

// ---------------------------------------------------------------- LGSSM (lgssm.cpp)
void* rb_lgssm_synthetic(const rb_spec* s, int* status) {
  lgssm::Model* m = nullptr;
  *status = guarded([&] { m = new lgssm::Model(bench::synthetic_lgssm(to_spec(*s))); });
  return m;
}
// Arrays with counts in {1, T} (dynamics) and {1, T+1} (observations); mask may be NULL.
void* rb_lgssm_new(int T, int dx, int dy, const double* m0, const double* P0, const double* F, int nF,
                   const double* b, int nb, const double* Q, int nQ, const double* H, int nH,
                   const double* c, int nc, const double* R, int nR, const std::uint8_t* mask,
                   int* status) {
  lgssm::Model* m = nullptr;
  *status = guarded([&] {
    std::vector<Mat> vF, vQ, vH, vR;
    std::vector<Vec> vb, vc;
    for (int k = 0; k < nF; ++k) vF.push_back(mat_in(F + k * dx * dx, dx, dx));
    for (int k = 0; k < nb; ++k) vb.push_back(vec_in(b + k * dx, dx));
    for (int k = 0; k < nQ; ++k) vQ.push_back(mat_in(Q + k * dx * dx, dx, dx));
    for (int k = 0; k < nH; ++k) vH.push_back(mat_in(H + k * dy * dx, dy, dx));
    for (int k = 0; k < nc; ++k) vc.push_back(vec_in(c + k * dy, dy));
    for (int k = 0; k < nR; ++k) vR.push_back(mat_in(R + k * dy * dy, dy, dy));
    std::vector<std::uint8_t> vm;
    if (mask) vm.assign(mask, mask + T + 1);
    m = new lgssm::Model(T, vec_in(m0, dx), mat_in(P0, dx, dx), vF, vb, vQ, vH, vc, vR, vm);
  });
  return m;
}
void rb_lgssm_free(void* m) { delete static_cast<lgssm::Model*>(m); }

// kalman_filter (lgssm.cpp:73-112) or parallel_filter (pit.cpp:117-188).
void* rb_filter(const void* model, const double* obs, int parallel, int workers, int* status) {
  const auto& m = *static_cast<const lgssm::Model*>(model);
  lgssm::FilterResult* fr = nullptr;
  *status = guarded([&] {
    const Mat o = mat_in(obs, m.horizon() + 1, m.dy());
    fr = new lgssm::FilterResult(parallel ? pit::parallel_filter(m, o, workers)
                                          : lgssm::kalman_filter(m, o));
  });
  return fr;
}
void rb_filter_get(const void* f, double* pred_mean, double* pred_cov, double* filt_mean,
                   double* filt_cov, double* log_marginal) {
  const auto& fr = *static_cast<const lgssm::FilterResult*>(f);
  const long n = static_cast<long>(fr.filt_mean.size());
  const int d = n ? static_cast<int>(fr.filt_mean[0].size()) : 0;
  for (long t = 0; t < n; ++t) {
    if (pred_mean) vec_out(fr.pred_mean[t], pred_mean + t * d);
    if (filt_mean) vec_out(fr.filt_mean[t], filt_mean + t * d);
    if (pred_cov) mat_out(fr.pred_cov[t], pred_cov + t * d * d);
    if (filt_cov) mat_out(fr.filt_cov[t], filt_cov + t * d * d);
  }
  *log_marginal = fr.log_marginal;
}
void rb_filter_free(void* f) { delete static_cast<lgssm::FilterResult*>(f); }

// which: 0 backward_sample (lgssm.cpp:151-177), 1 prefix_sample (pit.cpp:78-115),
// 2 dnc_sample (pit.cpp:192-301).  terminal == NULL: StreamNoise over the stream with
// this key (rng.hpp:128-137); else pre-drawn variates at the samplers' addresses.
int rb_sample(const void* model, const void* f, int which, std::uint64_t key, const double* terminal,
              const double* backward, const double* bridge, long n_bridge, int workers, double* out) {
  const auto& m = *static_cast<const lgssm::Model*>(model);
  const auto& fr = *static_cast<const lgssm::FilterResult*>(f);
  return guarded([&] {
    StreamNoise sn(RngStream::from_key(key));
    PredrawnNoise pn;
    pn.terminal = terminal, pn.backward = backward, pn.bridge = bridge;
    pn.n_backward = m.horizon(), pn.n_bridge = n_bridge;
    NoiseSource& noise = terminal ? static_cast<NoiseSource&>(pn) : static_cast<NoiseSource&>(sn);
    Trajectory x = which == 0   ? lgssm::backward_sample(m, fr, noise)
                   : which == 1 ? pit::prefix_sample(m, fr, noise, workers)
                                : pit::dnc_sample(m, fr, noise, workers);
    mat_out(x, out);
  });
}

double rb_path_logpdf(const void* model, const double* obs, const double* traj, const void* f,
                      int* status) {
  const auto& m = *static_cast<const lgssm::Model*>(model);
  const auto& fr = *static_cast<const lgssm::FilterResult*>(f);
  double v = NAN;
  *status = guarded([&] {
    v = lgssm::path_logpdf(m, mat_in(obs, m.horizon() + 1, m.dy()),
                           mat_in(traj, m.horizon() + 1, m.dx()), fr);
  });
  return v;
}

void rb_set_flip_backward_gain(int on) { testhooks::flip_backward_gain.store(on != 0); }

// ---------------------------------------------------------------- aux Kalman (auxk.cpp)
void* rb_aux_chain_new(const void* tg, const double* x0, double delta, int* status) {
  const auto& t = *static_cast<const auxk::GenSSMTarget*>(tg);
  auxk::AuxChainState* st = nullptr;
  *status = guarded([&] {
    st = new auxk::AuxChainState(auxk::init_chain(t, mat_in(x0, t.horizon() + 1, t.dx()), delta));
  });
  return st;
}
void rb_aux_chain_free(void* s) { delete static_cast<auxk::AuxChainState*>(s); }

// kernel_step (auxk.cpp:130-198) with the chain root stream of this key.
int rb_aux_step(const void* tg, void* s, std::uint64_t root_key, int backend, int parallel_filter,
                int zeroth_order, int workers) {
  const auto& t = *static_cast<const auxk::GenSSMTarget*>(tg);
  auto& st = *static_cast<auxk::AuxChainState*>(s);
  auxk::KernelOptions o;
  o.backend = static_cast<auxk::Backend>(backend);
  o.parallel_filter = parallel_filter != 0;
  o.zeroth_order = zeroth_order != 0;
  o.workers = workers;
  return guarded([&] { auxk::kernel_step(t, st, RngStream::from_key(root_key), o); });
}
void rb_aux_adapt(void* s, double rate) { auxk::adapt_delta(*static_cast<auxk::AuxChainState*>(s), rate); }
// stats: accepted, rejected, aborted, nonfinite_gamma, iter
void rb_aux_get(const void* s, double* x, double* scal, long* stats) {
  const auto& st = *static_cast<const auxk::AuxChainState*>(s);
  if (x) mat_out(st.x, x);
  scal[0] = st.delta;
  scal[1] = st.log_gamma;
  scal[2] = st.stats.last_log_alpha;
  scal[3] = st.stats.last_accept_prob;
  stats[0] = st.stats.accepted;
  stats[1] = st.stats.rejected;
  stats[2] = st.stats.aborted;
  stats[3] = st.stats.nonfinite_gamma;
  stats[4] = st.iter;
}
int rb_sample_aux_obs(const double* x, int T, int dx, double delta, std::uint64_t it_key, double* u) {
  return guarded([&] { mat_out(auxk::sample_aux_obs(mat_in(x, T + 1, dx), delta, RngStream::from_key(it_key)), u); });
}
double rb_mh_log_ratio(const void* tg, const double* x, const double* xp, const double* u, double delta,
                       int zeroth_order, int* status) {
  const auto& t = *static_cast<const auxk::GenSSMTarget*>(tg);
  double v = NAN;
  *status = guarded([&] {
    const int T = t.horizon(), d = t.dx();
    v = auxk::mh_log_ratio(t, mat_in(x, T + 1, d), mat_in(xp, T + 1, d), mat_in(u, T + 1, d), delta,
                           zeroth_order != 0);
  });
  return v;
}

// ---------------------------------------------------------------- particle Gibbs (fkpg.cpp)
void* rb_pg_new(const double* x0, int T, int dx, double delta) {
  return new fkpg::PGState(fkpg::init_pg(mat_in(x0, T + 1, dx), delta));
}
void rb_pg_free(void* s) { delete static_cast<fkpg::PGState*>(s); }
// aux_pgibbs_step (fkpg.cpp:252-271); mode: 0 prior, 1 gradient, 2 fully adapted.
// On DegenerateWeightsError, *bad_t is parsed from the message ("t=<k>").
int rb_pg_step(const void* tg, void* s, int N, std::uint64_t root_key, int mode, int* bad_t) {
  const auto& t = *static_cast<const auxk::GenSSMTarget*>(tg);
  auto& st = *static_cast<fkpg::PGState*>(s);
  fkpg::PgOptions o;
  o.mode = static_cast<fkpg::ProposalMode>(mode);
  *bad_t = -1;
  try {
    fkpg::aux_pgibbs_step(t, st, N, RngStream::from_key(root_key), o);
    return RB_OK;
  } catch (const DegenerateWeightsError& e) {
    const char* p = std::strstr(e.what(), "t=");
    if (p) *bad_t = std::atoi(p + 2);
    return RB_E_DEGENERATE;
  } catch (const FactorizationError&) {
    return RB_E_FACTOR;
  } catch (const std::exception&) {
    return RB_E_OTHER;
  }
}
// aux_pgibbs_step with PgOptions::fk_transform = pm_potential(fk, estimator) and the
// estimators of the reference's own tests (auxmc_gpu.h AUXMC_PM_*): 1 two-point noise
// (acceptance.cpp:256-268), 2 exact (test_fkpg.cpp:370-373), 3 negative (:441-442).
int rb_pg_step_pm(const void* tg, void* s, int N, std::uint64_t root_key, int mode, int pm, int* bad_t) {
  const auto& t = *static_cast<const auxk::GenSSMTarget*>(tg);
  auto& st = *static_cast<fkpg::PGState*>(s);
  fkpg::PgOptions o;
  o.mode = static_cast<fkpg::ProposalMode>(mode);
  o.fk_transform = [pm](const fkpg::FeynmanKacModel& fk) {
    fkpg::FeynmanKacModel orig = fk;
    return fkpg::pm_potential(fk, [orig, pm](int t, const Vec& prev, const Vec& cur, std::uint64_t key) {
      if (pm == 3) return -0.1;
      const double lg = t == 0 ? orig.log_g0(cur, 0) : orig.log_g(t, prev, cur, 0);
      if (pm == 2) return std::exp(lg);
      RngStream ks = RngStream::from_key(key);
      const double eps = ks.next_uniform() < 0.5 ? 0.5 : 1.5;
      return std::exp(lg) * eps;
    });
  };
  *bad_t = -1;
  try {
    fkpg::aux_pgibbs_step(t, st, N, RngStream::from_key(root_key), o);
    return RB_OK;
  } catch (const ContractError&) {
    return RB_E_CONTRACT;
  } catch (const DegenerateWeightsError& e) {
    const char* p = std::strstr(e.what(), "t=");
    if (p) *bad_t = std::atoi(p + 2);
    return RB_E_DEGENERATE;
  } catch (const std::exception&) {
    return RB_E_OTHER;
  }
}

void rb_pg_adapt(void* s, double rate) { fkpg::adapt_delta(*static_cast<fkpg::PGState*>(s), rate); }
// scal: delta, last_update; ints: iter, updates
void rb_pg_get(const void* s, double* x, std::uint64_t* keys, double* scal, long* ints) {
  const auto& st = *static_cast<const fkpg::PGState*>(s);
  if (x) mat_out(st.x, x);
  if (keys)
    for (std::size_t i = 0; i < st.keys.size(); ++i) keys[i] = st.keys[i];
  scal[0] = st.delta;
  scal[1] = st.last_update;
  ints[0] = st.iter;
  ints[1] = st.updates;
}

// csmc_step on the auxiliary Feynman-Kac model (fkpg.cpp:112-152 over build_aux_fk
// :188-231), exposing the ancestors and the selected indices for index-level parity.
int rb_csmc_trace(const void* tg, const double* ref, const std::uint64_t* ref_keys, const double* u,
                  double delta, int N, std::uint64_t it_key, int mode, int* ancestors, double* traj,
                  int* bad_t) {
  const auto& t = *static_cast<const auxk::GenSSMTarget*>(tg);
  const int T = t.horizon(), d = t.dx();
  fkpg::PgOptions o;
  o.mode = static_cast<fkpg::ProposalMode>(mode);
  *bad_t = -1;
  try {
    const fkpg::FeynmanKacModel fk = fkpg::build_aux_fk(t, mat_in(u, T + 1, d), delta, o);
    std::vector<std::uint64_t> rk(ref_keys, ref_keys + T + 1);
    fkpg::CsmcResult r = fkpg::csmc_step(fk, mat_in(ref, T + 1, d), rk, N, RngStream::from_key(it_key));
    if (ancestors)
      for (int s = 0; s <= T; ++s)
        for (int i = 0; i < N; ++i) ancestors[s * N + i] = r.system.ancestors[s][i];
    mat_out(r.traj, traj);
    return RB_OK;
  } catch (const DegenerateWeightsError& e) {
    const char* p = std::strstr(e.what(), "t=");
    if (p) *bad_t = std::atoi(p + 2);
    return RB_E_DEGENERATE;
  } catch (const std::exception&) {
    return RB_E_OTHER;
  }
}

// ---------------------------------------------------------------- run driver (runner.cpp)
// bench::run on a JSON run config (config.cpp:92-135); writes trace.csv / summary.json
// into the config's output_dir.  Returns the accept (or update) rate via *rate.
int rb_run_json(const char* json_text, double* rate) {
  return guarded([&] {
    const bench::RunConfig cfg = bench::parse_run_config(nlohmann::json::parse(json_text));
    const bench::RunResult r = bench::run(cfg);
    *rate = r.summary.rate;
  });
}

}  // extern "C"
