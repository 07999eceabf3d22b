// C++ host facade, part 2: chain states in HBM (auxk::AuxChains, fkpg::PGChains),
// the reference's single-chain calls on top of them (auxk.hpp:59-79,
// fkpg.hpp:101-109) and the batched run driver (bench/runner.hpp, runner.cpp:112-244).
#include "auxmc_b200.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <set>

namespace auxmc {
inline namespace b200 {

using detail::DeviceBuffer;

namespace detail {

static void cuda_ok(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

static std::vector<double> replicate(const Trajectory& x0, int C, int T1, int dx) {
  require_dim(x0.rows() == T1 && x0.cols() == dx, "initial trajectory shape");
  std::vector<double> out(static_cast<size_t>(C) * T1 * dx);
  for (int c = 0; c < C; ++c)
    std::memcpy(out.data() + static_cast<size_t>(c) * T1 * dx, x0.data(),
                sizeof(double) * T1 * dx);
  return out;
}

static std::vector<std::uint64_t> root_keys(const std::vector<RngStream>& roots) {
  std::vector<std::uint64_t> k(roots.size());
  for (size_t c = 0; c < roots.size(); ++c) k[c] = roots[c].key();
  return k;
}

static std::vector<RngStream> seeded_roots(std::uint64_t seed, int C) {
  const RngStream base = RngStream::from_seed(seed);
  std::vector<RngStream> r;
  for (int c = 0; c < C; ++c) r.push_back(base.derive(stream::kChain, c));
  return r;
}

/* Column gather x[c][coord] for every chain: one strided 2-D copy per coordinate. */
static void gather_coords(const double* x, int C, size_t stride, const std::vector<long>& coords,
                          std::vector<double>& out) {
  const size_t K = coords.size();
  out.assign(static_cast<size_t>(C) * K, 0.0);
  for (size_t k = 0; k < K; ++k)
    cuda_ok(cudaMemcpy2D(out.data() + k, K * sizeof(double), x + coords[k],
                         stride * sizeof(double), sizeof(double), C, cudaMemcpyDeviceToHost),
            "gather");
}

}  // namespace detail

/* ================================ auxk ================================= */
namespace auxk {

struct AuxChains::Impl {
  GenSSMTarget target;
  int C, T1, dx;
  DeviceBuffer x, delta, log_gamma, grad, iter, stats, keys;
  detail::Workspace ws;
  auxmc_chains desc{};
  Impl(const GenSSMTarget& tg, const std::vector<RngStream>& roots)
      : target(tg), C(static_cast<int>(roots.size())), T1(tg.horizon() + 1), dx(tg.dx()),
        x(sizeof(double) * C * T1 * dx), delta(sizeof(double) * C), log_gamma(sizeof(double) * C),
        grad(sizeof(double) * C * T1 * dx), iter(sizeof(long long) * C),
        stats(sizeof(auxmc_kernel_stats) * C), keys(sizeof(std::uint64_t) * C) {
    require_dim(C > 0, "AuxChains: at least one chain");
    const std::vector<std::uint64_t> k = detail::root_keys(roots);
    keys.upload(k.data(), k.size() * sizeof(std::uint64_t));
    const std::vector<long long> zi(C, 0);
    iter.upload(zi.data(), zi.size() * sizeof(long long));
    const std::vector<auxmc_kernel_stats> zs(C, auxmc_kernel_stats{0, 0, 0, 0, 0.0, 0.0});
    stats.upload(zs.data(), zs.size() * sizeof(auxmc_kernel_stats));
    desc = {C, x.as<double>(), delta.as<double>(), log_gamma.as<double>(), grad.as<double>(),
            iter.as<long long>(), stats.as<auxmc_kernel_stats>(), keys.as<std::uint64_t>()};
  }
  void init() {  // auxk.cpp:120-128 for every chain
    const auxmc_target& t = target.device();
    auxmc_kernel_options o{0, 0, 0};
    size_t n = std::max<size_t>(auxmc_aux_kernel_workspace(&t, C, &o), 1 << 20);
    for (;;) {
      const int st = auxmc_init_chains(&t, &desc, ws.get(n), n, nullptr);
      if (st != AUXMC_E_WORKSPACE) {
        check_status(st, "init_chain");
        break;
      }
      n *= 2;
    }
  }
};

AuxChains::AuxChains(const GenSSMTarget& target, const Trajectory& x0, double delta,
                     const std::vector<RngStream>& roots)
    : impl_(new Impl(target, roots)) {
  Impl& m = *impl_;
  const std::vector<double> xs = detail::replicate(x0, m.C, m.T1, m.dx);
  m.x.upload(xs.data(), xs.size() * sizeof(double));
  const std::vector<double> d(m.C, delta);
  m.delta.upload(d.data(), d.size() * sizeof(double));
  m.init();
}

AuxChains AuxChains::seeded(const GenSSMTarget& target, const Trajectory& x0, double delta,
                            std::uint64_t seed, int C) {
  return AuxChains(target, x0, delta, detail::seeded_roots(seed, C));
}

AuxChains::~AuxChains() = default;
AuxChains::AuxChains(AuxChains&&) noexcept = default;

void AuxChains::kernel_step(const KernelOptions& opts) {
  Impl& m = *impl_;
  const auxmc_target& t = m.target.device();
  const auxmc_kernel_options o{static_cast<int>(opts.backend), opts.parallel_filter ? 1 : 0,
                               opts.zeroth_order ? 1 : 0};
  const size_t n = auxmc_aux_kernel_workspace(&t, m.C, &o);
  check_status(auxmc_aux_kernel_step(&t, &m.desc, &o, m.ws.get(n), n, nullptr), "kernel_step");
}

void AuxChains::adapt_delta(double target_rate) {
  check_status(auxmc_adapt_delta(&impl_->desc, target_rate, nullptr), "adapt_delta");
}

int AuxChains::chains() const { return impl_->C; }

static KernelStats from_c(const auxmc_kernel_stats& s) {
  KernelStats k;
  k.accepted = static_cast<long>(s.accepted);
  k.rejected = static_cast<long>(s.rejected);
  k.aborted = static_cast<long>(s.aborted);
  k.nonfinite_gamma = static_cast<long>(s.nonfinite_gamma);
  k.last_log_alpha = s.last_log_alpha;
  k.last_accept_prob = s.last_accept_prob;
  return k;
}

AuxChainState AuxChains::state(int c) const {
  const Impl& m = *impl_;
  require_dim(c >= 0 && c < m.C, "AuxChains::state: chain index");
  const size_t n = static_cast<size_t>(m.T1) * m.dx, off = static_cast<size_t>(c) * n;
  AuxChainState s;
  s.x = Trajectory(m.T1, m.dx);
  std::vector<double> g(n);
  long long it = 0;
  auxmc_kernel_stats ks;
  detail::cuda_ok(cudaMemcpy(s.x.data(), m.x.as<double>() + off, n * sizeof(double),
                             cudaMemcpyDeviceToHost), "state");
  detail::cuda_ok(cudaMemcpy(g.data(), m.grad.as<double>() + off, n * sizeof(double),
                             cudaMemcpyDeviceToHost), "state");
  detail::cuda_ok(cudaMemcpy(&s.delta, m.delta.as<double>() + c, sizeof(double),
                             cudaMemcpyDeviceToHost), "state");
  detail::cuda_ok(cudaMemcpy(&s.log_gamma, m.log_gamma.as<double>() + c, sizeof(double),
                             cudaMemcpyDeviceToHost), "state");
  detail::cuda_ok(cudaMemcpy(&it, m.iter.as<long long>() + c, sizeof(long long),
                             cudaMemcpyDeviceToHost), "state");
  detail::cuda_ok(cudaMemcpy(&ks, m.stats.as<auxmc_kernel_stats>() + c, sizeof ks,
                             cudaMemcpyDeviceToHost), "state");
  for (int t = 0; t < m.T1; ++t) s.grad_gen.emplace_back(g.begin() + t * m.dx, g.begin() + (t + 1) * m.dx);
  s.iter = static_cast<long>(it);
  s.stats = from_c(ks);
  return s;
}

void AuxChains::set_state(int c, const AuxChainState& s) {
  Impl& m = *impl_;
  require_dim(c >= 0 && c < m.C, "AuxChains::set_state: chain index");
  require_dim(s.x.rows() == m.T1 && s.x.cols() == m.dx, "AuxChainState: x shape");
  const size_t n = static_cast<size_t>(m.T1) * m.dx, off = static_cast<size_t>(c) * n;
  std::vector<double> g(n, 0.0);
  if (s.grad_gen.size() == static_cast<size_t>(m.T1))
    for (int t = 0; t < m.T1; ++t) {
      require_dim(s.grad_gen[t].size() == static_cast<size_t>(m.dx), "AuxChainState: grad_gen");
      std::memcpy(g.data() + t * m.dx, s.grad_gen[t].data(), sizeof(double) * m.dx);
    }
  const long long it = s.iter;
  const auxmc_kernel_stats ks{s.stats.accepted, s.stats.rejected, s.stats.aborted,
                              s.stats.nonfinite_gamma, s.stats.last_log_alpha,
                              s.stats.last_accept_prob};
  detail::cuda_ok(cudaMemcpy(m.x.as<double>() + off, s.x.data(), n * sizeof(double),
                             cudaMemcpyHostToDevice), "set_state");
  detail::cuda_ok(cudaMemcpy(m.grad.as<double>() + off, g.data(), n * sizeof(double),
                             cudaMemcpyHostToDevice), "set_state");
  detail::cuda_ok(cudaMemcpy(m.delta.as<double>() + c, &s.delta, sizeof(double),
                             cudaMemcpyHostToDevice), "set_state");
  detail::cuda_ok(cudaMemcpy(m.log_gamma.as<double>() + c, &s.log_gamma, sizeof(double),
                             cudaMemcpyHostToDevice), "set_state");
  detail::cuda_ok(cudaMemcpy(m.iter.as<long long>() + c, &it, sizeof it, cudaMemcpyHostToDevice),
                  "set_state");
  detail::cuda_ok(cudaMemcpy(m.stats.as<auxmc_kernel_stats>() + c, &ks, sizeof ks,
                             cudaMemcpyHostToDevice), "set_state");
}

std::vector<KernelStats> AuxChains::stats() const {
  std::vector<auxmc_kernel_stats> s(impl_->C);
  impl_->stats.download(s.data(), s.size() * sizeof(auxmc_kernel_stats));
  std::vector<KernelStats> out;
  for (const auto& k : s) out.push_back(from_c(k));
  return out;
}

std::vector<double> AuxChains::deltas() const {
  std::vector<double> d(impl_->C);
  impl_->delta.download(d.data(), d.size() * sizeof(double));
  return d;
}

static std::vector<int> device_gamma_move(const GenSSMTarget& tg, int C, const double* x,
                                          const std::uint64_t* keys, long iter, double step,
                                          std::vector<double>& gamma) {
  require_dim(static_cast<int>(gamma.size()) == C, "gamma_move: one γ per chain");
  DeviceBuffer g(sizeof(double) * C), mv(sizeof(int) * C);
  g.upload(gamma.data(), sizeof(double) * C);
  const auxmc_target& t = tg.device();
  check_status(auxmc_gamma_move(&t, C, x, keys, iter, step, g.as<double>(), mv.as<int>(), nullptr),
               "gamma_move");
  std::vector<int> moved(C);
  g.download(gamma.data(), sizeof(double) * C);
  mv.download(moved.data(), sizeof(int) * C);
  return moved;
}

std::vector<int> AuxChains::gamma_move(long iter, double step, std::vector<double>& gamma) {
  Impl& m = *impl_;
  return device_gamma_move(m.target, m.C, m.x.as<double>(), m.keys.as<std::uint64_t>(), iter,
                           step, gamma);
}

void AuxChains::retarget(const GenSSMTarget& target) {
  Impl& m = *impl_;
  require_dim(target.horizon() + 1 == m.T1 && target.dx() == m.dx, "retarget: same shape");
  m.target = target;
  m.init();  // auxk.cpp:120-128: log γ and gradients at the kept paths
}

void AuxChains::gather(const std::vector<long>& coords, std::vector<double>& out) const {
  detail::gather_coords(impl_->x.as<double>(), impl_->C,
                        static_cast<size_t>(impl_->T1) * impl_->dx, coords, out);
}

// auxk.cpp:120-128
AuxChainState init_chain(const GenSSMTarget& target, Trajectory x0, double delta) {
  AuxChains ch(target, x0, delta, {RngStream()});
  return ch.state(0);
}

// auxk.cpp:130-198: the iteration stream is rng.derive(kIteration, iter) on the device.
void kernel_step(const GenSSMTarget& target, AuxChainState& state, RngStream rng,
                 const KernelOptions& opts) {
  AuxChains ch(target, state.x, state.delta, {rng});
  ch.set_state(0, state);
  ch.kernel_step(opts);
  state = ch.state(0);
}

// auxk.cpp:213-218 (on the device, the same arithmetic as the batched chains)
void adapt_delta(AuxChainState& state, double target_rate) {
  DeviceBuffer d(&state.delta, sizeof(double));
  const long long it = state.iter;
  DeviceBuffer i(&it, sizeof it);
  const auxmc_kernel_stats ks{0, 0, 0, 0, state.stats.last_log_alpha,
                              state.stats.last_accept_prob};
  DeviceBuffer s(&ks, sizeof ks);
  auxmc_chains c{};
  c.C = 1;
  c.delta = d.as<double>();
  c.iter = i.as<long long>();
  c.stats = s.as<auxmc_kernel_stats>();
  check_status(auxmc_adapt_delta(&c, target_rate, nullptr), "adapt_delta");
  d.download(&state.delta, sizeof(double));
}

}  // namespace auxk

/* ================================ fkpg ================================= */
namespace fkpg {

struct PGChains::Impl {
  auxk::GenSSMTarget target;
  int C, N, T1, dx;
  DeviceBuffer x, keys, delta, iter, updates, last, roots, status, bad_t;
  int variant = -1;
  size_t wsb = 0;
  detail::Workspace ws;
  auxmc_pg_chains desc{};
  Impl(const auxk::GenSSMTarget& tg, const std::vector<RngStream>& r, int N_)
      : target(tg), C(static_cast<int>(r.size())), N(N_), T1(tg.horizon() + 1), dx(tg.dx()),
        x(sizeof(double) * C * T1 * dx), keys(sizeof(std::uint64_t) * C * T1),
        delta(sizeof(double) * C), iter(sizeof(long long) * C), updates(sizeof(long long) * C),
        last(sizeof(double) * C), roots(sizeof(std::uint64_t) * C), status(sizeof(int) * C),
        bad_t(sizeof(int) * C) {
    require_dim(C > 0 && N > 0, "PGChains: chains and particles must be positive");
    const std::vector<std::uint64_t> k = detail::root_keys(r);
    roots.upload(k.data(), k.size() * sizeof(std::uint64_t));
    const std::vector<std::uint64_t> zk(static_cast<size_t>(C) * T1, 0);
    keys.upload(zk.data(), zk.size() * sizeof(std::uint64_t));
    const std::vector<long long> zl(C, 0);
    iter.upload(zl.data(), zl.size() * sizeof(long long));
    updates.upload(zl.data(), zl.size() * sizeof(long long));
    const std::vector<double> zd(C, 0.0);
    last.upload(zd.data(), zd.size() * sizeof(double));
    const std::vector<int> zi(C, 0);
    status.upload(zi.data(), zi.size() * sizeof(int));
    bad_t.upload(zi.data(), zi.size() * sizeof(int));
    desc.C = C;
    desc.N = N;
    desc.x = x.as<double>();
    desc.keys = keys.as<std::uint64_t>();
    desc.delta = delta.as<double>();
    desc.iter = iter.as<long long>();
    desc.updates = updates.as<long long>();
    desc.last_update = last.as<double>();
    desc.root_keys = roots.as<std::uint64_t>();
    desc.status = status.as<int>();
    desc.bad_t = bad_t.as<int>();
  }
};

PGChains::PGChains(const auxk::GenSSMTarget& target, const Trajectory& x0, double delta,
                   const std::vector<RngStream>& roots, int N)
    : impl_(new Impl(target, roots, N)) {
  Impl& m = *impl_;
  const std::vector<double> xs = detail::replicate(x0, m.C, m.T1, m.dx);
  m.x.upload(xs.data(), xs.size() * sizeof(double));
  const std::vector<double> d(m.C, delta);
  m.delta.upload(d.data(), d.size() * sizeof(double));
}

PGChains PGChains::seeded(const auxk::GenSSMTarget& target, const Trajectory& x0, double delta,
                          std::uint64_t seed, int C, int N) {
  return PGChains(target, x0, delta, detail::seeded_roots(seed, C), N);
}

PGChains::~PGChains() = default;
PGChains::PGChains(PGChains&&) noexcept = default;

void PGChains::aux_pgibbs_step(const PgOptions& opts) {
  Impl& m = *impl_;
  if (opts.linearize != LinearizeAt::kAuxObs)
    throw ConfigError("aux_pgibbs_step: the device path linearizes at the auxiliary "
                      "observation (LinearizeAt::kAuxObs, fkpg.cpp:166-171)");
  if (opts.variant == Variant::kPit && opts.mode != ProposalMode::kGradient)
    throw ConfigError("aux_pgibbs_step: the parallel-in-time cSMC needs parent-free "
                      "(gradient) proposals");
  const auxmc_target& t = m.target.device();
  const int variant = opts.variant == Variant::kPit ? AUXMC_CSMC_PIT : AUXMC_CSMC_REFERENCE;
  if (variant != m.variant) {
    m.wsb = auxmc_aux_pgibbs_workspace(&t, m.C, m.N, variant);
    m.variant = variant;
  }
  const int mode = opts.mode == ProposalMode::kPrior      ? AUXMC_PG_PRIOR
                   : opts.mode == ProposalMode::kGradient ? AUXMC_PG_GRADIENT
                                                          : AUXMC_PG_ADAPTED;
  check_status(auxmc_aux_pgibbs_step(&t, &m.desc, mode, variant, m.ws.get(m.wsb),
                                     m.wsb, nullptr),
               "aux_pgibbs_step");
  std::vector<int> st(m.C), bt(m.C);
  m.status.download(st.data(), st.size() * sizeof(int));
  for (int c = 0; c < m.C; ++c)
    if (st[c] != AUXMC_OK) {
      m.bad_t.download(bt.data(), bt.size() * sizeof(int));
      if (st[c] == AUXMC_E_DEGENERATE)
        throw DegenerateWeightsError("all particle weights are zero at t = " +
                                     std::to_string(bt[c]) + " (chain " + std::to_string(c) + ")");
      check_status(st[c], "aux_pgibbs_step chain " + std::to_string(c));
    }
}

void PGChains::adapt_delta(double target_rate) {
  check_status(auxmc_pg_adapt_delta(&impl_->desc, target_rate, nullptr), "adapt_delta");
}

int PGChains::chains() const { return impl_->C; }

PGState PGChains::state(int c) const {
  const Impl& m = *impl_;
  require_dim(c >= 0 && c < m.C, "PGChains::state: chain index");
  const size_t n = static_cast<size_t>(m.T1) * m.dx;
  PGState s;
  s.x = Trajectory(m.T1, m.dx);
  s.keys.resize(m.T1);
  long long it = 0, up = 0;
  detail::cuda_ok(cudaMemcpy(s.x.data(), m.x.as<double>() + c * n, n * sizeof(double),
                             cudaMemcpyDeviceToHost), "state");
  detail::cuda_ok(cudaMemcpy(s.keys.data(), m.keys.as<std::uint64_t>() + static_cast<size_t>(c) * m.T1,
                             m.T1 * sizeof(std::uint64_t), cudaMemcpyDeviceToHost), "state");
  detail::cuda_ok(cudaMemcpy(&s.delta, m.delta.as<double>() + c, sizeof(double),
                             cudaMemcpyDeviceToHost), "state");
  detail::cuda_ok(cudaMemcpy(&it, m.iter.as<long long>() + c, sizeof it, cudaMemcpyDeviceToHost),
                  "state");
  detail::cuda_ok(cudaMemcpy(&up, m.updates.as<long long>() + c, sizeof up,
                             cudaMemcpyDeviceToHost), "state");
  detail::cuda_ok(cudaMemcpy(&s.last_update, m.last.as<double>() + c, sizeof(double),
                             cudaMemcpyDeviceToHost), "state");
  s.iter = static_cast<long>(it);
  s.updates = static_cast<long>(up);
  return s;
}

void PGChains::set_state(int c, const PGState& s) {
  Impl& m = *impl_;
  require_dim(c >= 0 && c < m.C, "PGChains::set_state: chain index");
  require_dim(s.x.rows() == m.T1 && s.x.cols() == m.dx, "PGState: x shape");
  const size_t n = static_cast<size_t>(m.T1) * m.dx;
  std::vector<std::uint64_t> k(m.T1, 0);
  if (s.keys.size() == static_cast<size_t>(m.T1)) k = s.keys;
  const long long it = s.iter, up = s.updates;
  detail::cuda_ok(cudaMemcpy(m.x.as<double>() + c * n, s.x.data(), n * sizeof(double),
                             cudaMemcpyHostToDevice), "set_state");
  detail::cuda_ok(cudaMemcpy(m.keys.as<std::uint64_t>() + static_cast<size_t>(c) * m.T1, k.data(),
                             m.T1 * sizeof(std::uint64_t), cudaMemcpyHostToDevice), "set_state");
  detail::cuda_ok(cudaMemcpy(m.delta.as<double>() + c, &s.delta, sizeof(double),
                             cudaMemcpyHostToDevice), "set_state");
  detail::cuda_ok(cudaMemcpy(m.iter.as<long long>() + c, &it, sizeof it, cudaMemcpyHostToDevice),
                  "set_state");
  detail::cuda_ok(cudaMemcpy(m.updates.as<long long>() + c, &up, sizeof up,
                             cudaMemcpyHostToDevice), "set_state");
  detail::cuda_ok(cudaMemcpy(m.last.as<double>() + c, &s.last_update, sizeof(double),
                             cudaMemcpyHostToDevice), "set_state");
}

std::vector<long> PGChains::updates() const {
  std::vector<long long> u(impl_->C);
  impl_->updates.download(u.data(), u.size() * sizeof(long long));
  return std::vector<long>(u.begin(), u.end());
}

std::vector<double> PGChains::deltas() const {
  std::vector<double> d(impl_->C);
  impl_->delta.download(d.data(), d.size() * sizeof(double));
  return d;
}

void PGChains::gather(const std::vector<long>& coords, std::vector<double>& out) const {
  detail::gather_coords(impl_->x.as<double>(), impl_->C,
                        static_cast<size_t>(impl_->T1) * impl_->dx, coords, out);
}

std::vector<int> PGChains::gamma_move(long iter, double step, std::vector<double>& gamma) {
  Impl& m = *impl_;
  return auxk::device_gamma_move(m.target, m.C, m.x.as<double>(), m.roots.as<std::uint64_t>(),
                                 iter, step, gamma);
}

void PGChains::retarget(const auxk::GenSSMTarget& target) {
  Impl& m = *impl_;
  require_dim(target.horizon() + 1 == m.T1 && target.dx() == m.dx, "retarget: same shape");
  m.target = target;  // runner.cpp:195: the sweep state carries nothing target-derived
}

// fkpg.cpp:252-258
PGState init_pg(Trajectory x0, double delta) {
  PGState s;
  s.keys.assign(x0.rows(), 0);
  s.x = std::move(x0);
  s.delta = delta;
  return s;
}

// fkpg.cpp:260-274
void aux_pgibbs_step(const auxk::GenSSMTarget& target, PGState& state, int N, RngStream rng,
                     const PgOptions& opts) {
  PGChains ch(target, state.x, state.delta, {rng}, N);
  ch.set_state(0, state);
  ch.aux_pgibbs_step(opts);
  state = ch.state(0);
}

// fkpg.cpp:276-280
void adapt_delta(PGState& state, double target_rate) {
  DeviceBuffer d(&state.delta, sizeof(double)), l(&state.last_update, sizeof(double));
  const long long it = state.iter;
  DeviceBuffer i(&it, sizeof it);
  auxmc_pg_chains c{};
  c.C = 1;
  c.delta = d.as<double>();
  c.iter = i.as<long long>();
  c.last_update = l.as<double>();
  check_status(auxmc_pg_adapt_delta(&c, target_rate, nullptr), "adapt_delta");
  d.download(&state.delta, sizeof(double));
}

}  // namespace fkpg

/* ============================ run driver ================================ */
namespace bench {

namespace fs = std::filesystem;
using clk = std::chrono::steady_clock;

bool is_aux_family(const std::string& s) {
  return s == "aux-kalman-seq" || s == "aux-kalman-prefix" || s == "aux-kalman-dnc";
}
bool is_pgibbs_family(const std::string& s) {
  return s == "pgibbs-prior" || s == "pgibbs-gradient" || s == "pgibbs-adapted" ||
         s == "pgibbs-pit";
}

static auxk::Backend backend_of(const std::string& s) {  // runner.cpp:31-36
  if (s == "aux-kalman-seq") return auxk::Backend::kSequential;
  if (s == "aux-kalman-prefix") return auxk::Backend::kPrefix;
  if (s == "aux-kalman-dnc") return auxk::Backend::kDnc;
  throw ConfigError("not an aux-kalman sampler: " + s);
}

static std::vector<int> choose_probes(const RunConfig& cfg, int T, int dx) {  // runner.cpp:45-56
  std::set<int> times;
  if (!cfg.probe_times.empty()) {
    for (int t : cfg.probe_times) {
      if (t < 0 || t > T) throw ConfigError("probe time out of range: " + std::to_string(t));
      times.insert(t);
    }
  } else if (static_cast<long>(T + 1) * dx <= 64) {
    for (int t = 0; t <= T; ++t) times.insert(t);
  } else {
    for (int i = 0; i < 5; ++i) times.insert(static_cast<int>(std::lround(i * T / 4.0)));
  }
  return {times.begin(), times.end()};
}

static std::string num(double v) {
  if (!std::isfinite(v)) return "null";
  char buf[64];
  std::snprintf(buf, sizeof buf, "%.17g", v);
  return buf;
}

template <class V>
static std::string arr(const V& v) {
  std::string s = "[";
  for (size_t i = 0; i < v.size(); ++i) s += (i ? ", " : "") + num(static_cast<double>(v[i]));
  return s + "]";
}

RunResult run(const RunConfig& cfg_in) {
  RunConfig cfg = cfg_in;
  if (!is_aux_family(cfg.sampler) && !is_pgibbs_family(cfg.sampler))
    throw ConfigError("unknown sampler: " + cfg.sampler);
  if (cfg.chain_length < 0 || cfg.burn_in < 0 || cfg.burn_in > cfg.chain_length)
    throw ConfigError("need 0 <= burn_in <= chain_length");
  if (cfg.chains < 1) throw ConfigError("chains must be positive");
  if (cfg.target_acceptance < 0 || cfg.target_acceptance >= 1)  // config.cpp:120-123
    throw ConfigError("target_acceptance must be in [0, 1)");
  if (cfg.target_acceptance == 0.0)
    cfg.target_acceptance = is_aux_family(cfg.sampler) ? 0.574 : 0.9;
  if (cfg.sample_param) {  // config.cpp:128-130 (+ Lorenz-96, whose γ move is the same law)
    if (cfg.model.kind != "diffusion-smoothing" && cfg.model.kind != "lorenz96")
      throw ConfigError("sample_param requires the diffusion-smoothing model");
    if (!(cfg.param_step > 0)) throw ConfigError("param_step must be > 0");
    // runner.cpp runs one chain: γ is part of the target, which the batch shares
    if (cfg.chains != 1) throw ConfigError("sample_param runs a single chain");
  }

  ModelSpec spec = cfg.model;
  const SimResult sim = simulate(spec);
  auxk::GenSSMTarget target = make_target(spec, sim.data);
  double& gam = spec.kind == "lorenz96" ? spec.l96_gamma : spec.lz_gamma;
  std::vector<double> param_draws;
  const int T = target.horizon(), dx = target.dx(), C = cfg.chains;
  const long keep = cfg.chain_length - cfg.burn_in;
  const std::vector<int> times = choose_probes(cfg, T, dx);
  std::vector<long> coords;
  for (int t : times)
    for (int j = 0; j < dx; ++j) coords.push_back(static_cast<long>(t) * dx + j);
  const size_t K = coords.size();

  fs::create_directories(cfg.output_dir);
  RunResult res;
  res.trace_path = (fs::path(cfg.output_dir) / "trace.csv").string();
  res.summary_path = (fs::path(cfg.output_dir) / "summary.json").string();
  std::ofstream trace(res.trace_path);
  if (!trace) throw ConfigError("cannot write trace file: " + res.trace_path);
  trace << "iter";
  for (long c : coords) trace << ",coord_" << c;
  trace << "\n";

  Trajectory x0(T + 1, dx);  // runner.cpp:133: m0 replicated over T+1
  for (int t = 0; t <= T; ++t)
    for (int j = 0; j < dx; ++j) x0(t, j) = target.m0()[j];

  std::vector<double> sum(K, 0.0), draws;  // draws[(k * C + c) * K + j], pooled moments
  draws.reserve(static_cast<size_t>(std::max<long>(keep, 0)) * C * K);
  std::vector<double> g;
  auto record = [&](long iter) {
    trace << iter;
    for (size_t j = 0; j < K; ++j) trace << "," << num(g[j]);  // chain 0
    trace << "\n";
    draws.insert(draws.end(), g.begin(), g.end());
    if (cfg.sample_param) param_draws.push_back(gam);  // runner.cpp:148
  };
  // runner.cpp:159-167 / :192-196: the γ move after each sweep; a new γ rebuilds the target
  auto param_move = [&](auto& ch, long iter) {
    if (!cfg.sample_param) return;
    std::vector<double> gv(1, gam);
    if (ch.gamma_move(iter, cfg.param_step, gv)[0]) {
      gam = gv[0];
      target = make_target(spec, sim.data);
      ch.retarget(target);
    }
  };

  const clk::time_point t0 = clk::now();
  double burn_seconds = 0.0, rate_num = 0.0, final_delta = cfg.delta_init;
  auto burn_end = [&]() {
    detail::synchronize();
    burn_seconds = std::chrono::duration<double>(clk::now() - t0).count();
  };
  if (is_aux_family(cfg.sampler)) {
    auxk::KernelOptions opts;
    opts.backend = backend_of(cfg.sampler);
    opts.parallel_filter = cfg.parallel_filter;
    auxk::AuxChains ch = auxk::AuxChains::seeded(target, x0, cfg.delta_init, cfg.seed, C);
    std::vector<long> mark(C, 0);
    for (long iter = 0; iter < cfg.chain_length; ++iter) {
      ch.kernel_step(opts);
      param_move(ch, iter);
      if (iter < cfg.burn_in) {
        ch.adapt_delta(cfg.target_acceptance);
        if (iter + 1 == cfg.burn_in) {
          burn_end();
          for (int c = 0; c < C; ++c) mark[c] = ch.stats()[c].accepted;
        }
      } else {
        ch.gather(coords, g);
        record(iter);
      }
    }
    const std::vector<auxk::KernelStats> st = ch.stats();
    for (int c = 0; c < C; ++c) rate_num += static_cast<double>(st[c].accepted - mark[c]);
    final_delta = ch.deltas()[0];
  } else {
    fkpg::PgOptions opts;
    opts.variant = cfg.sampler == "pgibbs-pit" ? fkpg::Variant::kPit : fkpg::Variant::kReference;
    if (cfg.sampler == "pgibbs-prior") opts.mode = fkpg::ProposalMode::kPrior;  // runner.cpp:38-43
    if (cfg.sampler == "pgibbs-adapted") opts.mode = fkpg::ProposalMode::kFullyAdapted;
    fkpg::PGChains ch =
        fkpg::PGChains::seeded(target, x0, cfg.delta_init, cfg.seed, C, cfg.particles);
    std::vector<long> mark(C, 0);
    for (long iter = 0; iter < cfg.chain_length; ++iter) {
      ch.aux_pgibbs_step(opts);
      param_move(ch, iter);
      if (iter < cfg.burn_in) {
        ch.adapt_delta(cfg.target_acceptance);
        if (iter + 1 == cfg.burn_in) {
          burn_end();
          mark = ch.updates();
        }
      } else {
        ch.gather(coords, g);
        record(iter);
      }
    }
    const std::vector<long> up = ch.updates();
    for (int c = 0; c < C; ++c) rate_num += static_cast<double>(up[c] - mark[c]);
    final_delta = ch.deltas()[0];
  }
  detail::synchronize();
  if (cfg.burn_in == 0) burn_seconds = 0.0;

  ChainSummary& s = res.summary;
  s.probe_times = times;
  s.probe_coords = coords;
  s.kept = std::max<long>(keep, 0);
  s.chains = C;
  s.final_delta = final_delta;
  s.burn_seconds = burn_seconds;
  s.sample_seconds = std::chrono::duration<double>(clk::now() - t0).count() - burn_seconds;
  const size_t n = static_cast<size_t>(s.kept) * C;  // diagnostics.cpp:48-59, pooled
  if (n > 0) {
    s.mean.assign(K, 0.0);
    s.sd.assign(K, 0.0);
    for (size_t r = 0; r < n; ++r)
      for (size_t j = 0; j < K; ++j) s.mean[j] += draws[r * K + j];
    for (size_t j = 0; j < K; ++j) s.mean[j] /= static_cast<double>(n);
    if (n > 1)
      for (size_t j = 0; j < K; ++j) {
        double ss = 0.0;
        for (size_t r = 0; r < n; ++r) ss += (draws[r * K + j] - s.mean[j]) * (draws[r * K + j] - s.mean[j]);
        s.sd[j] = std::sqrt(ss / static_cast<double>(n - 1));
      }
    s.rate = rate_num / static_cast<double>(n);
    if (cfg.sample_param && !param_draws.empty()) {  // runner.cpp:228-236
      const double pn = static_cast<double>(param_draws.size());
      double pm = 0.0, pss = 0.0;
      for (double v : param_draws) pm += v;
      pm /= pn;
      for (double v : param_draws) pss += (v - pm) * (v - pm);
      s.has_param = true;
      s.param_mean = pm;
      s.param_sd = param_draws.size() > 1 ? std::sqrt(pss / (pn - 1.0)) : 0.0;
    }
  }

  std::ofstream sf(res.summary_path);  // config.cpp:178-207 (ESS / MCSE not computed)
  if (!sf) throw ConfigError("cannot write summary file: " + res.summary_path);
  sf << "{\n  \"version\": \"" << auxmc_version() << "\",\n"
     << "  \"config\": {\"sampler\": \"" << cfg.sampler << "\", \"chain_length\": "
     << cfg.chain_length << ", \"burn_in\": " << cfg.burn_in << ", \"particles\": "
     << cfg.particles << ", \"delta_init\": " << num(cfg.delta_init)
     << ", \"target_acceptance\": " << num(cfg.target_acceptance) << ", \"seed\": " << cfg.seed
     << ", \"chains\": " << C << ", \"model\": {\"kind\": \"" << cfg.model.kind
     << "\", \"T\": " << cfg.model.T << "}},\n"
     << "  \"probe_times\": " << arr(s.probe_times) << ",\n"
     << "  \"probe_coords\": " << arr(s.probe_coords) << ",\n"
     << "  \"kept\": " << s.kept << ",\n"
     << "  \"mean\": " << (n ? arr(s.mean) : "null") << ",\n"
     << "  \"sd\": " << (n ? arr(s.sd) : "null") << ",\n"
     << "  \"rate\": " << (n ? num(s.rate) : "null") << ",\n"
     << "  \"final_delta\": " << num(s.final_delta) << ",\n"
     << (s.has_param ? "  \"param_mean\": " + num(s.param_mean) + ",\n  \"param_sd\": " +
                           num(s.param_sd) + ",\n"
                     : std::string())
     << "  \"burn_seconds\": " << num(s.burn_seconds) << ",\n"
     << "  \"sample_seconds\": " << num(s.sample_seconds) << "\n}\n";
  return res;
}

}  // namespace bench

}  // inline namespace b200
}  // namespace auxmc
