// Parity tests of the C++ host facade (include/auxmc_b200.hpp) against the CPU
// oracle (oracle/auxmc_oracle.h, test infrastructure), on the same inputs and
// the same counter-RNG streams.  Built by paper_2303_00301_b200/build.py
// (build_tests); run by tests/test_cpp_facade.py.
//   test_facade            all GPU parity tests (needs an sm_100 device)
//   test_facade --no-device  host-only checks: argument errors, and that every
//                          compute call throws CudaError without a device
#include <cmath>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <functional>
#include <string>
#include <vector>

#include "auxmc_b200.hpp"
#include "auxmc_oracle.h"

using namespace auxmc;

static int g_fail = 0, g_run = 0;

#define EXPECT(cond, ...)                                   \
  do {                                                      \
    if (!(cond)) {                                          \
      std::printf("  FAIL %s:%d: ", __FILE__, __LINE__);    \
      std::printf(__VA_ARGS__);                             \
      std::printf("\n");                                    \
      ++g_fail;                                             \
    }                                                       \
  } while (0)

template <class E, class F>
static bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static double rel_err(const double* a, const double* b, size_t n) {
  double e = 0.0;
  for (size_t i = 0; i < n; ++i)
    e = std::fmax(e, std::fabs(a[i] - b[i]) / std::fmax(1.0, std::fabs(b[i])));
  return e;
}

static void run_test(const char* name, const std::function<void()>& f) {
  const int before = g_fail;
  ++g_run;
  try {
    f();
  } catch (const std::exception& e) {
    std::printf("  FAIL %s: exception %s\n", name, e.what());
    ++g_fail;
  }
  std::printf("%s %s\n", g_fail == before ? "ok  " : "FAIL", name);
}

/* ---- oracle mirrors of facade objects ---- */
struct OModel {
  std::vector<double> F, b, Q, H, c, R;
  std::vector<std::uint8_t> mask;
  ao_lgssm m{};
  explicit OModel(const lgssm::Model& mod) {
    const int T = mod.horizon();
    auto app = [](std::vector<double>& v, const Mat& x) {
      v.insert(v.end(), x.data(), x.data() + x.size());
    };
    F.clear();
    for (int t = 0; t < T; ++t) {
      app(F, mod.F(t));
      b.insert(b.end(), mod.b(t).begin(), mod.b(t).end());
      app(Q, mod.Q(t));
    }
    for (int t = 0; t <= T; ++t) {
      app(H, mod.H(t));
      c.insert(c.end(), mod.c(t).begin(), mod.c(t).end());
      app(R, mod.R(t));
      mask.push_back(mod.observed(t) ? 1 : 0);
    }
    m.T = T;
    m.dx = mod.dx();
    m.dy = mod.dy();
    m.m0 = mod.m0().data();
    m.P0 = mod.P0().data();
    m.F = F.data();
    m.b = b.data();
    m.Q = Q.data();
    m.H = H.data();
    m.c = c.data();
    m.R = R.data();
    m.nF = m.nb = m.nQ = T;
    m.nH = m.nc = m.nR = T + 1;
    m.mask = mask.data();
  }
};

struct OFilter {
  std::vector<double> pm, pc, fm, fc;
  ao_filter f{};
  OFilter(int T, int d)
      : pm((T + 1) * d), pc((T + 1) * d * d), fm((T + 1) * d), fc((T + 1) * d * d) {
    f = {pm.data(), pc.data(), fm.data(), fc.data(), 0.0};
  }
};

static std::vector<double> flat_means(const std::vector<Vec>& v) {
  std::vector<double> o;
  for (const Vec& x : v) o.insert(o.end(), x.begin(), x.end());
  return o;
}
static std::vector<double> flat_covs(const std::vector<Mat>& v) {
  std::vector<double> o;
  for (const Mat& x : v) o.insert(o.end(), x.data(), x.data() + x.size());
  return o;
}

static ao_spec ospec(const bench::ModelSpec& s) {
  const auxmc_model_spec c = bench::to_c(s);
  ao_spec o;
  static_assert(sizeof(o) == sizeof(c), "spec layouts");
  std::memcpy(&o, &c, sizeof o);
  return o;
}

/* An address-based NoiseSource that is not a StreamNoise: exercises the
 * pre-drawn device path (rng.hpp:123-137). */
struct WrappedNoise final : NoiseSource {
  RngStream base;
  explicit WrappedNoise(RngStream b) : base(b) {}
  Vec normal(std::uint64_t label, std::uint64_t index, int dim) override {
    RngStream s = base.derive(label, index);
    return s.normal_vec(dim);
  }
};

static void gpu_tests() {
  bench::ModelSpec spec;
  spec.kind = "lgssm-synthetic";
  spec.T = 300;
  spec.dx = 3;
  spec.dy = 2;
  spec.data_seed = 5;
  const bench::SimResult sim = bench::simulate(spec);
  const lgssm::Model model = bench::synthetic_lgssm(spec);
  OModel om(model);
  const int T = spec.T, d = spec.dx;

  OFilter of(T, d);
  ao_kalman_filter(&om.m, sim.data.data(), &of.f);

  run_test("kalman_filter vs oracle (lgssm.cpp:73-112)", [&] {
    const lgssm::FilterResult fr = lgssm::kalman_filter(model, sim.data);
    const auto fm = flat_means(fr.filt_mean), fc = flat_covs(fr.filt_cov);
    const auto pc = flat_covs(fr.pred_cov);
    EXPECT(rel_err(fm.data(), of.fm.data(), fm.size()) < 1e-9, "filt_mean");
    EXPECT(rel_err(fc.data(), of.fc.data(), fc.size()) < 1e-9, "filt_cov");
    EXPECT(rel_err(pc.data(), of.pc.data(), pc.size()) < 1e-9, "pred_cov");
    EXPECT(std::fabs(fr.log_marginal - of.f.log_marginal) < 1e-9 * std::fabs(of.f.log_marginal),
           "log_marginal %.17g vs %.17g", fr.log_marginal, of.f.log_marginal);
  });

  run_test("pit::parallel_filter vs oracle (pit.cpp:117-188)", [&] {
    const lgssm::FilterResult fr = pit::parallel_filter(model, sim.data);
    const auto fm = flat_means(fr.filt_mean), fc = flat_covs(fr.filt_cov);
    EXPECT(rel_err(fm.data(), of.fm.data(), fm.size()) < 1e-8, "filt_mean");
    EXPECT(rel_err(fc.data(), of.fc.data(), fc.size()) < 1e-8, "filt_cov");
    EXPECT(std::fabs(fr.log_marginal - of.f.log_marginal) < 1e-9 * std::fabs(of.f.log_marginal),
           "log_marginal");
  });

  const lgssm::FilterResult fr = lgssm::kalman_filter(model, sim.data);
  const RngStream root = RngStream::from_seed(3).derive(stream::kChain, 2);
  std::vector<double> want(static_cast<size_t>(T + 1) * d);
  struct S {
    const char* name;
    int which;
  };
  for (const S s : {S{"lgssm::backward_sample vs oracle (lgssm.cpp:151-177)", 0},
                    S{"pit::prefix_sample vs oracle (pit.cpp:78-115)", 1},
                    S{"pit::dnc_sample vs oracle (pit.cpp:192-301)", 2}}) {
    run_test(s.name, [&] {
      ao_noise nz{};
      nz.kind = 0;
      nz.base = ao_from_key(root.key());
      nz.dx = d;
      int st = s.which == 0   ? ao_backward_sample(&om.m, &of.f, &nz, want.data())
               : s.which == 1 ? ao_prefix_sample(&om.m, &of.f, &nz, want.data(), nullptr, nullptr)
                              : ao_dnc_sample(&om.m, &of.f, &nz, want.data());
      EXPECT(st == AO_OK, "oracle status %d", st);
      auto draw = [&](NoiseSource& n) {
        return s.which == 0   ? lgssm::backward_sample(model, fr, n)
               : s.which == 1 ? pit::prefix_sample(model, fr, n)
                              : pit::dnc_sample(model, fr, n);
      };
      StreamNoise sn(root);
      const Trajectory x = draw(sn);
      EXPECT(rel_err(x.data(), want.data(), want.size()) < 1e-9, "stream noise: %g",
             rel_err(x.data(), want.data(), want.size()));
      WrappedNoise wn(root);
      const Trajectory y = draw(wn);
      EXPECT(rel_err(y.data(), want.data(), want.size()) < 1e-9, "pre-drawn noise: %g",
             rel_err(y.data(), want.data(), want.size()));
    });
  }

  run_test("pit::extract_affine_law (all samplers) and rts_smoother vs dense posterior", [&] {
    bench::ModelSpec small = spec;
    small.T = 12;
    const bench::SimResult ss = bench::simulate(small);
    const lgssm::Model sm = bench::synthetic_lgssm(small);
    OModel osm(sm);
    const int n = (small.T + 1) * d;
    std::vector<double> pm(n), pc(static_cast<size_t>(n) * n);
    double le = 0.0;
    EXPECT(ao_dense_oracle(&osm.m, ss.data.data(), 256, pm.data(), pc.data(), &le) == AO_OK,
           "dense oracle");
    const lgssm::FilterResult sfr = lgssm::kalman_filter(sm, ss.data);
    for (const pit::Sampler w : {pit::Sampler::kSequential, pit::Sampler::kPrefix,
                                 pit::Sampler::kDnc}) {
      const gauss::Gaussian law = pit::extract_affine_law(w, sm, sfr);
      EXPECT(rel_err(law.mean.data(), pm.data(), n) < 1e-8, "law mean (sampler %d)", (int)w);
      EXPECT(rel_err(law.cov.data(), pc.data(), pc.size()) < 1e-8, "law cov (sampler %d)",
             (int)w);
    }
    const std::vector<gauss::Gaussian> sm_marg = lgssm::rts_smoother(sm, sfr);
    for (int t = 0; t <= small.T; ++t)
      for (int i = 0; i < d; ++i) {
        EXPECT(std::fabs(sm_marg[t].mean[i] - pm[t * d + i]) < 1e-8, "rts mean t=%d", t);
        for (int j = 0; j < d; ++j)
          EXPECT(std::fabs(sm_marg[t].cov(i, j) - pc[(size_t)(t * d + i) * n + t * d + j]) < 1e-8,
                 "rts cov t=%d", t);
      }
  });

  run_test("pit::PathBatch: chain c equals the single-chain prefix_sample", [&] {
    const int C = 5;
    std::vector<RngStream> roots;
    for (int c = 0; c < C; ++c) roots.push_back(RngStream::from_seed(1).derive(stream::kChain, c));
    pit::PathBatch batch(model, fr, C, pit::Sampler::kPrefix);
    batch.draw(roots);
    for (int c = 0; c < C; ++c) {
      const Trajectory a = batch.path(c), b = pit::prefix_sample(model, fr, roots[c]);
      EXPECT(std::memcmp(a.data(), b.data(), a.size() * sizeof(double)) == 0, "chain %d", c);
    }
  });

  run_test("lgssm::path_logpdf vs oracle (lgssm.cpp:179-199)", [&] {
    ao_noise nz{};
    nz.kind = 0;
    nz.base = ao_from_key(root.key());
    nz.dx = d;
    ao_backward_sample(&om.m, &of.f, &nz, want.data());
    Trajectory x(T + 1, d);
    std::memcpy(x.data(), want.data(), want.size() * sizeof(double));
    int st = 0;
    const double ref = ao_path_logpdf(&om.m, sim.data.data(), want.data(), &of.f, &st);
    const double got = lgssm::path_logpdf(model, sim.data, x, fr);
    EXPECT(std::fabs(got - ref) < 1e-9 * std::fmax(1.0, std::fabs(ref)), "%.17g vs %.17g", got,
           ref);
  });

  // auxiliary Kalman sampler on stochastic volatility (auxk.cpp:130-198)
  bench::ModelSpec sv;
  sv.kind = "stochvol";
  sv.T = 40;
  sv.dx = 3;
  sv.data_seed = 11;
  const bench::SimResult svs = bench::simulate(sv);
  const auxk::GenSSMTarget tg = bench::make_target(sv, svs.data);
  ao_spec os = ospec(sv);
  ao_target otg{};
  ao_make_target(&os, svs.data.data(), &otg);

  for (int backend = 0; backend < 3; ++backend) {
    for (int pf = 0; pf < 2; ++pf) {
      const std::string name = "auxk::kernel_step backend " + std::to_string(backend) +
                               (pf ? " parallel filter" : "") + " vs oracle, 6 steps";
      run_test(name.c_str(), [&] {
        const RngStream r = RngStream::from_seed(1).derive(stream::kChain, 0);
        auxk::AuxChainState st = auxk::init_chain(tg, svs.latent, 1.0);
        ao_chain oc{};
        ao_init_chain(&otg, svs.latent.data(), 1.0, &oc);
        EXPECT(std::fabs(st.log_gamma - oc.log_gamma) < 1e-9 * std::fabs(oc.log_gamma),
               "init log_gamma");
        auxk::KernelOptions o;
        o.backend = static_cast<auxk::Backend>(backend);
        o.parallel_filter = pf != 0;
        for (int i = 0; i < 6; ++i) {
          auxk::kernel_step(tg, st, r, o);
          ao_kernel_step(&otg, &oc, ao_from_key(r.key()), backend, pf, 0);
          auxk::adapt_delta(st, 0.574);
          ao_adapt_delta(&oc, 0.574);
        }
        EXPECT(st.stats.accepted == oc.stats.accepted && st.stats.rejected == oc.stats.rejected,
               "accept decisions %ld/%ld vs %ld/%ld", st.stats.accepted, st.stats.rejected,
               oc.stats.accepted, oc.stats.rejected);
        EXPECT(st.iter == oc.iter, "iter");
        EXPECT(rel_err(st.x.data(), oc.x, st.x.size()) < 1e-9, "x: %g",
               rel_err(st.x.data(), oc.x, st.x.size()));
        EXPECT(std::fabs(st.delta - oc.delta) < 1e-12 * oc.delta, "delta %.17g vs %.17g",
               st.delta, oc.delta);
        ao_chain_free(&oc);
      });
    }
  }

  run_test("auxk::AuxChains batch equals per-chain kernel_step (bit-exact)", [&] {
    const int C = 4;
    auxk::AuxChains ch = auxk::AuxChains::seeded(tg, svs.latent, 0.5, 9, C);
    auxk::KernelOptions o;
    o.backend = auxk::Backend::kPrefix;
    for (int i = 0; i < 3; ++i) ch.kernel_step(o);
    for (int c = 0; c < C; ++c) {
      auxk::AuxChainState st = auxk::init_chain(tg, svs.latent, 0.5);
      const RngStream r = RngStream::from_seed(9).derive(stream::kChain, c);
      for (int i = 0; i < 3; ++i) auxk::kernel_step(tg, st, r, o);
      const auxk::AuxChainState b = ch.state(c);
      EXPECT(std::memcmp(b.x.data(), st.x.data(), st.x.size() * sizeof(double)) == 0,
             "chain %d x", c);
      EXPECT(b.stats.accepted == st.stats.accepted, "chain %d accepted", c);
    }
  });

  run_test("auxk on an LGSSM target: unit acceptance (test_target_auxk.cpp:182-231)", [&] {
    const auxk::GenSSMTarget lt = auxk::GenSSMTarget::from_lgssm(model, sim.data);
    auxk::AuxChains ch = auxk::AuxChains::seeded(lt, sim.latent, 1.0, 2, 3);
    auxk::KernelOptions o;
    o.backend = auxk::Backend::kDnc;
    for (int i = 0; i < 10; ++i) ch.kernel_step(o);
    for (const auxk::KernelStats& s : ch.stats())
      EXPECT(s.accepted == 10 && s.last_accept_prob > 1.0 - 1e-6, "accepted %ld p %.17g",
             s.accepted, s.last_accept_prob);
  });

  run_test("GenSSMTarget::log_gamma vs oracle (target.cpp:100-108)", [&] {
    int st = 0;
    const double ref = ao_log_gamma(&otg, svs.latent.data(), &st);
    const double got = tg.log_gamma(svs.latent);
    EXPECT(std::fabs(got - ref) < 1e-9 * std::fabs(ref), "%.17g vs %.17g", got, ref);
  });

  run_test("fkpg::aux_pgibbs_step (reference cSMC) vs oracle, 4 sweeps (fkpg.cpp:260-274)", [&] {
    const int N = 16;
    const RngStream r = RngStream::from_seed(4).derive(stream::kChain, 0);
    fkpg::PGState st = fkpg::init_pg(svs.latent, 1.0);
    ao_pg op{};
    ao_init_pg(&otg, svs.latent.data(), 1.0, &op);
    for (int i = 0; i < 4; ++i) {
      fkpg::aux_pgibbs_step(tg, st, N, r);
      int bad = 0;
      const int s = ao_aux_pgibbs_step(&otg, &op, N, ao_from_key(r.key()), AO_PG_GRADIENT,
                                       nullptr, nullptr, &bad);
      EXPECT(s == AO_OK, "oracle status %d", s);
      fkpg::adapt_delta(st, 0.9);
      ao_pg_adapt_delta(&op, 0.9);
    }
    EXPECT(st.updates == op.updates && st.iter == op.iter, "updates %ld vs %ld", st.updates,
           op.updates);
    EXPECT(rel_err(st.x.data(), op.x, st.x.size()) < 1e-9, "x: %g",
           rel_err(st.x.data(), op.x, st.x.size()));
    EXPECT(std::memcmp(st.keys.data(), op.keys, st.keys.size() * 8) == 0, "reference keys");
    EXPECT(std::fabs(st.delta - op.delta) < 1e-12 * op.delta, "delta");
    ao_pg_free(&op);
  });

  for (const auto mode : {fkpg::ProposalMode::kPrior, fkpg::ProposalMode::kFullyAdapted}) {
    const std::string name = std::string("fkpg::aux_pgibbs_step ") +
                             (mode == fkpg::ProposalMode::kPrior ? "prior" : "fully adapted") +
                             " proposals vs oracle, 3 sweeps (fkpg.cpp:154-185)";
    run_test(name.c_str(), [&] {
      const int N = 12;
      const RngStream r = RngStream::from_seed(6).derive(stream::kChain, 1);
      fkpg::PGState st = fkpg::init_pg(svs.latent, 1.0);
      ao_pg op{};
      ao_init_pg(&otg, svs.latent.data(), 1.0, &op);
      fkpg::PgOptions o;
      o.mode = mode;
      for (int i = 0; i < 3; ++i) {
        fkpg::aux_pgibbs_step(tg, st, N, r, o);
        int bad = 0;
        const int s = ao_aux_pgibbs_step(&otg, &op, N, ao_from_key(r.key()),
                                         mode == fkpg::ProposalMode::kPrior ? AO_PG_PRIOR
                                                                            : AO_PG_ADAPTED,
                                         nullptr, nullptr, &bad);
        EXPECT(s == AO_OK, "oracle status %d", s);
      }
      EXPECT(st.updates == op.updates, "updates %ld vs %ld", st.updates, op.updates);
      EXPECT(rel_err(st.x.data(), op.x, st.x.size()) < 1e-9, "x: %g",
             rel_err(st.x.data(), op.x, st.x.size()));
      ao_pg_free(&op);
    });
  }

  run_test("fkpg::PGChains PIT variant runs and moves every chain", [&] {
    fkpg::PGChains ch = fkpg::PGChains::seeded(tg, svs.latent, 1.0, 5, 3, 32);
    fkpg::PgOptions o;
    o.variant = fkpg::Variant::kPit;
    for (int i = 0; i < 3; ++i) ch.aux_pgibbs_step(o);
    for (long u : ch.updates()) EXPECT(u >= 1, "updates %ld", u);
    fkpg::PgOptions prior;
    prior.mode = fkpg::ProposalMode::kPrior;
    prior.variant = fkpg::Variant::kPit;
    EXPECT(throws<ConfigError>([&] { ch.aux_pgibbs_step(prior); }), "PIT + prior must throw");
  });

  run_test("bench::run aux-kalman-prefix, 4 chains, exact target: rate 1, files", [&] {
    bench::RunConfig cfg;
    cfg.sampler = "aux-kalman-prefix";
    cfg.chain_length = 30;
    cfg.burn_in = 10;
    cfg.chains = 4;
    cfg.model.kind = "lgssm-synthetic";
    cfg.model.T = 20;
    cfg.model.dx = 2;
    cfg.output_dir = std::filesystem::temp_directory_path() / "auxmc_b200_run_test";
    const bench::RunResult r = bench::run(cfg);
    EXPECT(r.summary.kept == 20 && r.summary.rate == 1.0, "kept %ld rate %g", r.summary.kept,
           r.summary.rate);
    EXPECT(r.summary.probe_coords.size() == 42, "probes %zu", r.summary.probe_coords.size());
    std::ifstream tr(r.trace_path);
    std::string line;
    int rows = 0;
    while (std::getline(tr, line)) ++rows;
    EXPECT(rows == 21, "trace rows %d", rows);
    EXPECT(std::filesystem::exists(r.summary_path), "summary.json");
  });

  run_test("bench::run pgibbs-gradient: trace chain 0 equals the single-chain sweep", [&] {
    bench::RunConfig cfg;
    cfg.sampler = "pgibbs-gradient";
    cfg.chain_length = 6;
    cfg.burn_in = 2;
    cfg.particles = 8;
    cfg.chains = 2;
    cfg.model = sv;
    cfg.model.T = 10;
    cfg.output_dir = std::filesystem::temp_directory_path() / "auxmc_b200_run_pg";
    const bench::RunResult r = bench::run(cfg);
    // replay chain 0 by hand (runner.cpp:190-205)
    const bench::SimResult s2 = bench::simulate(cfg.model);
    const auxk::GenSSMTarget t2 = bench::make_target(cfg.model, s2.data);
    Trajectory x0(cfg.model.T + 1, 3);
    for (int t = 0; t <= cfg.model.T; ++t)
      for (int j = 0; j < 3; ++j) x0(t, j) = t2.m0()[j];
    fkpg::PGState st = fkpg::init_pg(x0, 1.0);
    const RngStream root = RngStream::from_seed(1).derive(stream::kChain, 0);
    std::vector<double> last;
    for (int it = 0; it < 6; ++it) {
      fkpg::aux_pgibbs_step(t2, st, 8, root);
      if (it < 2) fkpg::adapt_delta(st, 0.9);
    }
    std::ifstream tr(r.trace_path);
    std::string line, lastline;
    while (std::getline(tr, line)) lastline = line;
    char buf[64];
    std::snprintf(buf, sizeof buf, "%.17g", st.x(0, 0));
    EXPECT(lastline.rfind("5," + std::string(buf) + ",", 0) == 0, "last trace row %s vs x00 %s",
           lastline.c_str(), buf);
  });
}

static void host_tests(bool device) {
  run_test("Model dimension checks (lgssm.cpp:20-71)", [&] {
    EXPECT(throws<DimensionError>([] {
             lgssm::Model::homogeneous(5, Vec(2, 0.0), Mat::Identity(3), Mat::Identity(2),
                                       Vec(2, 0.0), Mat::Identity(2), Mat(1, 2), Vec(1, 0.0),
                                       Mat::Identity(1));
           }),
           "P0 shape");
    EXPECT(throws<DimensionError>([] {
             lgssm::Model(5, Vec(1, 0.0), Mat::Identity(1), {Mat::Identity(1), Mat::Identity(1)},
                          {Vec(1, 0.0)}, {Mat::Identity(1)}, {Mat(1, 1)}, {Vec(1, 0.0)},
                          {Mat::Identity(1)});
           }),
           "F count");
  });
  run_test("RngStream derive chain (rng.hpp:62-80) matches the oracle", [&] {
    const RngStream a = RngStream::from_seed(7).derive(6, 3).derive(1, 99);
    const ao_stream b = ao_derive(ao_derive(ao_from_seed(7), 6, 3), 1, 99);
    EXPECT(a.key() == b.key, "key");
    RngStream a2 = a;
    ao_stream b2 = b;
    EXPECT(a2.next_uniform() == ao_next_uniform(&b2), "uniform");
    EXPECT(a2.next_normal() == ao_next_normal(&b2), "normal");
  });
  run_test("make_target rejects unknown kinds (ConfigError)", [&] {
    bench::ModelSpec s;
    s.kind = "nope";
    EXPECT(throws<ConfigError>([&] { bench::make_target(s, Mat(51, 1)); }), "kind");
  });
  if (!device) {
    run_test("no device: compute calls throw CudaError (no CPU path)", [&] {
      const lgssm::Model m = lgssm::Model::homogeneous(
          4, Vec(1, 0.0), Mat::Identity(1), Mat::Identity(1), Vec(1, 0.0), Mat::Identity(1),
          Mat::Identity(1), Vec(1, 0.0), Mat::Identity(1));
      EXPECT(throws<CudaError>([&] { lgssm::kalman_filter(m, Mat(5, 1)); }), "kalman_filter");
      EXPECT(throws<CudaError>([&] { pit::parallel_filter(m, Mat(5, 1)); }), "parallel_filter");
      bench::ModelSpec s;
      s.kind = "stochvol";
      s.T = 5;
      s.dx = 2;
      EXPECT(throws<CudaError>([&] {
               const bench::SimResult r = bench::simulate(s);
               auxk::init_chain(bench::make_target(s, r.data), r.latent, 1.0);
             }),
             "init_chain");
    });
  }
}

// --run sampler kind T chain_length burn_in seed sample_param param_step delta out_dir:
// one bench::run (the facade's run driver) for the reference-parity test
// (tests/test_facade_run.py compares its files with the reference's bench::run).
static int run_mode(int argc, char** argv) {
  if (argc < 12) {
    std::printf("usage: --run sampler kind T length burn seed sample_param step delta out\n");
    return 2;
  }
  bench::RunConfig cfg;
  cfg.sampler = argv[2];
  cfg.model.kind = argv[3];
  cfg.model.T = std::atoi(argv[4]);
  cfg.chain_length = std::atol(argv[5]);
  cfg.burn_in = std::atol(argv[6]);
  cfg.seed = std::strtoull(argv[7], nullptr, 10);
  cfg.sample_param = std::atoi(argv[8]) != 0;
  cfg.param_step = std::atof(argv[9]);
  cfg.delta_init = std::atof(argv[10]);
  cfg.output_dir = argv[11];
  try {
    const bench::RunResult r = bench::run(cfg);
    std::printf("rate %.17g param_mean %.17g\n", r.summary.rate, r.summary.param_mean);
  } catch (const std::exception& e) {
    std::printf("error: %s\n", e.what());
    return 1;
  }
  return 0;
}

int main(int argc, char** argv) {
  if (argc > 1 && std::strcmp(argv[1], "--run") == 0) return run_mode(argc, argv);
  const bool no_device = argc > 1 && std::strcmp(argv[1], "--no-device") == 0;
  const bool device = auxmc_device_ok() == 1;
  if (!no_device && !device) {
    std::printf("no sm_100 device; run with --no-device for the host-only checks\n");
    return 2;
  }
  host_tests(device);
  if (!no_device) gpu_tests();
  std::printf("%d tests, %d failures\n", g_run, g_fail);
  return g_fail ? 1 : 0;
}
