// C++ host facade over the C ABI (include/auxmc_b200.hpp): the reference's
// free-function API (lgssm.hpp, pit.hpp, auxk.hpp, fkpg.hpp, bench/models.hpp)
// with every compute call forwarded to libauxmc_b200's device entry points.
// Host work here is argument checking, host<->device copies and workspace
// management; there is no CPU compute path.
#include "auxmc_b200.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>

namespace auxmc {
inline namespace b200 {

void check_status(int status, const std::string& what) {
  if (status == AUXMC_OK) return;
  const std::string msg = what + ": " + auxmc_status_string(status);
  switch (status) {
    case AUXMC_E_DIM: throw DimensionError(msg);
    case AUXMC_E_FACTOR: throw FactorizationError(msg);
    case AUXMC_E_DEGENERATE: throw DegenerateWeightsError(msg);
    case AUXMC_E_CONTRACT: throw ContractError(msg);
    case AUXMC_E_CONFIG: throw ConfigError(msg);
    case AUXMC_E_CUDA: throw CudaError(msg + " " + auxmc_last_error());
    default: throw Error(msg);
  }
}

namespace detail {

static void cuda_try(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

static void require_device() {
  if (!auxmc_device_ok()) throw CudaError("libauxmc_b200: no usable sm_100 device");
}

DeviceBuffer::DeviceBuffer(size_t bytes) : n_(bytes) {
  require_device();
  if (bytes) cuda_try(cudaMalloc(&p_, bytes), "cudaMalloc");
}

DeviceBuffer::DeviceBuffer(const void* host, size_t bytes) : DeviceBuffer(bytes) {
  upload(host, bytes);
}

DeviceBuffer::~DeviceBuffer() {
  if (p_) cudaFree(p_);
}

DeviceBuffer& DeviceBuffer::operator=(DeviceBuffer&& o) noexcept {
  if (this != &o) {
    if (p_) cudaFree(p_);
    p_ = o.p_;
    n_ = o.n_;
    o.p_ = nullptr;
    o.n_ = 0;
  }
  return *this;
}

void DeviceBuffer::upload(const void* host, size_t bytes) {
  if (bytes) cuda_try(cudaMemcpy(p_, host, bytes, cudaMemcpyHostToDevice), "cudaMemcpy H2D");
}

void DeviceBuffer::download(void* host, size_t bytes) const {
  if (bytes) cuda_try(cudaMemcpy(host, p_, bytes, cudaMemcpyDeviceToHost), "cudaMemcpy D2H");
}

void synchronize() { cuda_try(cudaDeviceSynchronize(), "cudaDeviceSynchronize"); }

template <class T>
static DeviceBuffer upload_vec(const std::vector<T>& v) {
  return DeviceBuffer(v.data(), v.size() * sizeof(T));
}

static Mat symm(const Mat& m) {
  Mat s(m.rows(), m.cols());
  for (int i = 0; i < m.rows(); ++i)
    for (int j = 0; j < m.cols(); ++j) s(i, j) = 0.5 * (m(i, j) + m(j, i));
  return s;
}

static void append(std::vector<double>& out, const Mat& m) {
  out.insert(out.end(), m.data(), m.data() + m.size());
}

}  // namespace detail

using detail::DeviceBuffer;

/* ================================ lgssm ================================ */
namespace lgssm {

struct Model::Dev {
  DeviceBuffer m0, P0, F, b, Q, H, c, R, mask;
  auxmc_lgssm desc{};
};

// lgssm.cpp:20-71: counts 1 or T (dynamics) / T+1 (observations), square
// symmetric covariances, symmetrized on construction.
Model::Model(int T, Vec m0, Mat P0, std::vector<Mat> F, std::vector<Vec> b, std::vector<Mat> Q,
             std::vector<Mat> H, std::vector<Vec> c, std::vector<Mat> R,
             std::vector<std::uint8_t> obs_mask)
    : T_(T), dx_(static_cast<int>(m0.size())), dy_(H.empty() ? 0 : H[0].rows()),
      m0_(std::move(m0)), P0_(detail::symm(P0)), F_(std::move(F)), Q_(std::move(Q)),
      H_(std::move(H)), R_(std::move(R)), b_(std::move(b)), c_(std::move(c)),
      mask_(std::move(obs_mask)) {
  auto count_ok = [](size_t n, int want) { return n == 1 || n == static_cast<size_t>(want); };
  require_dim(T >= 0, "Model: T < 0");
  require_dim(P0_.rows() == dx_ && P0_.cols() == dx_, "Model: P0 shape");
  require_dim(count_ok(F_.size(), T) && count_ok(b_.size(), T) && count_ok(Q_.size(), T),
              "Model: F/b/Q count must be 1 or T");
  require_dim(count_ok(H_.size(), T + 1) && count_ok(c_.size(), T + 1) &&
                  count_ok(R_.size(), T + 1),
              "Model: H/c/R count must be 1 or T+1");
  require_dim(mask_.empty() || mask_.size() == static_cast<size_t>(T + 1), "Model: mask size");
  for (const Mat& f : F_) require_dim(f.rows() == dx_ && f.cols() == dx_, "Model: F shape");
  for (const Vec& v : b_) require_dim(v.size() == static_cast<size_t>(dx_), "Model: b size");
  for (Mat& q : Q_) {
    require_dim(q.rows() == dx_ && q.cols() == dx_, "Model: Q shape");
    q = detail::symm(q);
  }
  for (const Mat& h : H_) require_dim(h.rows() == dy_ && h.cols() == dx_, "Model: H shape");
  for (const Vec& v : c_) require_dim(v.size() == static_cast<size_t>(dy_), "Model: c size");
  for (Mat& r : R_) {
    require_dim(r.rows() == dy_ && r.cols() == dy_, "Model: R shape");
    r = detail::symm(r);
  }
}

Model Model::homogeneous(int T, Vec m0, Mat P0, Mat F, Vec b, Mat Q, Mat H, Vec c, Mat R,
                         std::vector<std::uint8_t> obs_mask) {
  return Model(T, std::move(m0), std::move(P0), {std::move(F)}, {std::move(b)}, {std::move(Q)},
               {std::move(H)}, {std::move(c)}, {std::move(R)}, std::move(obs_mask));
}

const auxmc_lgssm& Model::device() const {
  if (dev_) return dev_->desc;
  auto d = std::make_shared<Dev>();
  std::vector<double> F, b, Q, H, c, R;
  for (const Mat& m : F_) detail::append(F, m);
  for (const Vec& v : b_) b.insert(b.end(), v.begin(), v.end());
  for (const Mat& m : Q_) detail::append(Q, m);
  for (const Mat& m : H_) detail::append(H, m);
  for (const Vec& v : c_) c.insert(c.end(), v.begin(), v.end());
  for (const Mat& m : R_) detail::append(R, m);
  d->m0 = detail::upload_vec(m0_);
  d->P0 = DeviceBuffer(P0_.data(), P0_.size() * sizeof(double));
  d->F = detail::upload_vec(F);
  d->b = detail::upload_vec(b);
  d->Q = detail::upload_vec(Q);
  d->H = detail::upload_vec(H);
  d->c = detail::upload_vec(c);
  d->R = detail::upload_vec(R);
  if (!mask_.empty()) d->mask = detail::upload_vec(mask_);
  auxmc_lgssm& m = d->desc;
  m.T = T_;
  m.dx = dx_;
  m.dy = dy_;
  m.m0 = d->m0.as<double>();
  m.P0 = d->P0.as<double>();
  m.F = d->F.as<double>();
  m.nF = static_cast<int>(F_.size());
  m.b = d->b.as<double>();
  m.nb = static_cast<int>(b_.size());
  m.Q = d->Q.as<double>();
  m.nQ = static_cast<int>(Q_.size());
  m.H = d->H.as<double>();
  m.nH = static_cast<int>(H_.size());
  m.c = d->c.as<double>();
  m.nc = static_cast<int>(c_.size());
  m.R = d->R.as<double>();
  m.nR = static_cast<int>(R_.size());
  m.mask = mask_.empty() ? nullptr : d->mask.as<std::uint8_t>();
  dev_ = d;
  return dev_->desc;
}

}  // namespace lgssm

namespace detail {

/* One filter result in HBM (B = 1), with host <-> device conversion. */
struct DeviceFilter {
  int T1, dx;
  DeviceBuffer pm, pc, fm, fc, lm;
  auxmc_filter_result desc{};
  DeviceFilter(int T, int d)
      : T1(T + 1), dx(d), pm(sizeof(double) * T1 * d), pc(sizeof(double) * T1 * d * d),
        fm(sizeof(double) * T1 * d), fc(sizeof(double) * T1 * d * d), lm(sizeof(double)) {
    desc = {pm.as<double>(), pc.as<double>(), fm.as<double>(), fc.as<double>(), lm.as<double>()};
  }
  explicit DeviceFilter(const lgssm::FilterResult& fr, int T, int d) : DeviceFilter(T, d) {
    require_dim(fr.filt_mean.size() == static_cast<size_t>(T1) &&
                    fr.filt_cov.size() == static_cast<size_t>(T1) &&
                    fr.pred_cov.size() == static_cast<size_t>(T1),
                "FilterResult: length must be T+1");
    std::vector<double> a, b, c, e;
    for (int t = 0; t < T1; ++t) {
      if (fr.pred_mean.size() == static_cast<size_t>(T1))
        a.insert(a.end(), fr.pred_mean[t].begin(), fr.pred_mean[t].end());
      e.insert(e.end(), fr.filt_mean[t].begin(), fr.filt_mean[t].end());
      append(b, fr.pred_cov[t]);
      append(c, fr.filt_cov[t]);
    }
    require_dim(e.size() == static_cast<size_t>(T1) * d && c.size() == e.size() * d &&
                    b.size() == e.size() * d,
                "FilterResult: moment shapes");
    if (a.size() == e.size()) pm.upload(a.data(), a.size() * sizeof(double));
    fm.upload(e.data(), e.size() * sizeof(double));
    pc.upload(b.data(), b.size() * sizeof(double));
    fc.upload(c.data(), c.size() * sizeof(double));
    lm.upload(&fr.log_marginal, sizeof(double));
  }
  lgssm::FilterResult to_host() const {
    std::vector<double> a(T1 * dx), b(T1 * dx * dx), c(T1 * dx), e(T1 * dx * dx);
    lgssm::FilterResult fr;
    pm.download(a.data(), a.size() * sizeof(double));
    pc.download(b.data(), b.size() * sizeof(double));
    fm.download(c.data(), c.size() * sizeof(double));
    fc.download(e.data(), e.size() * sizeof(double));
    lm.download(&fr.log_marginal, sizeof(double));
    for (int t = 0; t < T1; ++t) {
      fr.pred_mean.emplace_back(a.begin() + t * dx, a.begin() + (t + 1) * dx);
      fr.filt_mean.emplace_back(c.begin() + t * dx, c.begin() + (t + 1) * dx);
      Mat P(dx, dx), F(dx, dx);
      std::memcpy(P.data(), b.data() + static_cast<size_t>(t) * dx * dx, sizeof(double) * dx * dx);
      std::memcpy(F.data(), e.data() + static_cast<size_t>(t) * dx * dx, sizeof(double) * dx * dx);
      fr.pred_cov.push_back(std::move(P));
      fr.filt_cov.push_back(std::move(F));
    }
    return fr;
  }
};

static lgssm::FilterResult run_filter(const lgssm::Model& model, const Mat& obs, int mode) {
  const int T = model.horizon();
  require_dim(obs.rows() == T + 1 && obs.cols() == model.dy(), "kalman_filter: obs shape");
  const auxmc_lgssm& m = model.device();
  DeviceBuffer dobs(obs.data(), obs.size() * sizeof(double));
  DeviceFilter fr(T, model.dx());
  DeviceBuffer status(sizeof(int));
  const size_t wsb = auxmc_kalman_filter_workspace(&m, 1, mode);
  DeviceBuffer ws(std::max<size_t>(wsb, 1));
  check_status(auxmc_kalman_filter(&m, dobs.as<double>(), 1, mode, &fr.desc, status.as<int>(),
                                   ws.get(), wsb, nullptr),
               mode ? "parallel_filter" : "kalman_filter");
  int st = 0;
  status.download(&st, sizeof(int));
  check_status(st, mode ? "parallel_filter" : "kalman_filter");
  return fr.to_host();
}

/* Device noise for one path: a StreamNoise runs on the counter RNG; any other
 * (address-based) NoiseSource is pre-drawn at the sampler's addresses. */
struct DeviceNoise {
  DeviceBuffer keys, terminal, backward, bridge;
  auxmc_noise desc{};
  DeviceNoise(NoiseSource& noise, int T, int dx, bool dnc) {
    if (auto* s = dynamic_cast<StreamNoise*>(&noise)) {
      const std::uint64_t k = s->base().key();
      keys = DeviceBuffer(&k, sizeof k);
      desc.kind = AUXMC_NOISE_STREAM;
      desc.keys = keys.as<std::uint64_t>();
      return;
    }
    std::vector<double> term = noise.normal(stream::kTerminalDraw, 0, dx), back;
    require_dim(term.size() == static_cast<size_t>(dx), "NoiseSource: dimension");
    for (int t = 0; t < T; ++t) {
      Vec v = noise.normal(stream::kBackwardNoise, t, dx);
      back.insert(back.end(), v.begin(), v.end());
    }
    terminal = upload_vec(term);
    backward = upload_vec(back);
    desc.kind = AUXMC_NOISE_PREDRAWN;
    desc.terminal = terminal.as<double>();
    desc.backward = backward.as<double>();
    if (dnc) {
      const long long nb = auxmc_dnc_bridge_count(T);
      std::vector<double> br;
      br.reserve(static_cast<size_t>(nb) * dx);
      for (long long id = 0; id < nb; ++id) {
        Vec v = noise.normal(stream::kDncBridge, static_cast<std::uint64_t>(id), dx);
        br.insert(br.end(), v.begin(), v.end());
      }
      bridge = upload_vec(br);
      desc.bridge = bridge.as<double>();
      desc.n_bridge = nb;
    }
  }
};

static Trajectory sample_one(const lgssm::Model& model, const lgssm::FilterResult& fr,
                             NoiseSource& noise, int sampler, const char* what) {
  const int T = model.horizon(), dx = model.dx();
  const auxmc_lgssm& m = model.device();
  DeviceFilter dfr(fr, T, dx);
  DeviceNoise nz(noise, T, dx, sampler == AUXMC_SAMPLER_DNC);
  DeviceBuffer traj(sizeof(double) * (T + 1) * dx), status(sizeof(int));
  const size_t wsb = auxmc_sample_paths_workspace(&m, 1, 1, sampler);
  DeviceBuffer ws(std::max<size_t>(wsb, 1));
  check_status(auxmc_sample_paths(&m, &dfr.desc, 1, &nz.desc, 1, sampler, traj.as<double>(),
                                  status.as<int>(), ws.get(), wsb, nullptr),
               what);
  int st = 0;
  status.download(&st, sizeof(int));
  check_status(st, what);
  Trajectory out(T + 1, dx);
  traj.download(out.data(), out.size() * sizeof(double));
  return out;
}

}  // namespace detail

namespace lgssm {

FilterResult kalman_filter(const Model& model, const Mat& obs) {
  return detail::run_filter(model, obs, 0);
}

Trajectory backward_sample(const Model& model, const FilterResult& fr, NoiseSource& noise) {
  return detail::sample_one(model, fr, noise, AUXMC_SAMPLER_SEQ, "backward_sample");
}

Trajectory backward_sample(const Model& model, const FilterResult& fr, RngStream rng) {
  StreamNoise n(rng);
  return backward_sample(model, fr, n);
}

std::vector<gauss::Gaussian> rts_smoother(const Model& model, const FilterResult& fr) {
  const int T = model.horizon(), dx = model.dx();
  const auxmc_lgssm& m = model.device();
  detail::DeviceFilter dfr(fr, T, dx);
  DeviceBuffer mean(sizeof(double) * (T + 1) * dx), cov(sizeof(double) * (T + 1) * dx * dx),
      status(sizeof(int));
  const size_t wsb = auxmc_rts_smoother_workspace(&m, 1);
  DeviceBuffer ws(std::max<size_t>(wsb, 1));
  check_status(auxmc_rts_smoother(&m, &dfr.desc, 1, mean.as<double>(), cov.as<double>(),
                                  status.as<int>(), ws.get(), wsb, nullptr),
               "rts_smoother");
  int st = 0;
  status.download(&st, sizeof(int));
  check_status(st, "rts_smoother");
  std::vector<double> hm((T + 1) * dx), hc((T + 1) * dx * dx);
  mean.download(hm.data(), hm.size() * sizeof(double));
  cov.download(hc.data(), hc.size() * sizeof(double));
  std::vector<gauss::Gaussian> out;
  for (int t = 0; t <= T; ++t) {
    gauss::Gaussian g{Vec(hm.begin() + t * dx, hm.begin() + (t + 1) * dx), Mat(dx, dx)};
    std::memcpy(g.cov.data(), hc.data() + static_cast<size_t>(t) * dx * dx,
                sizeof(double) * dx * dx);
    out.push_back(std::move(g));
  }
  return out;
}

double path_logpdf(const Model& model, const Mat& obs, const Trajectory& traj,
                   const FilterResult& fr) {
  const int T = model.horizon(), dx = model.dx();
  require_dim(obs.rows() == T + 1 && obs.cols() == model.dy(), "path_logpdf: obs shape");
  require_dim(traj.rows() == T + 1 && traj.cols() == dx, "path_logpdf: trajectory shape");
  const auxmc_lgssm& m = model.device();
  detail::DeviceFilter dfr(fr, T, dx);
  DeviceBuffer dobs(obs.data(), obs.size() * sizeof(double));
  DeviceBuffer dx_(traj.data(), traj.size() * sizeof(double));
  DeviceBuffer out(sizeof(double)), status(sizeof(int));
  check_status(auxmc_path_logpdf(&m, dobs.as<double>(), 1, dx_.as<double>(), &dfr.desc, 1, 1,
                                 out.as<double>(), status.as<int>(), nullptr),
               "path_logpdf");
  int st = 0;
  double v = 0.0;
  status.download(&st, sizeof(int));
  check_status(st, "path_logpdf");
  out.download(&v, sizeof(double));
  return v;
}

}  // namespace lgssm

/* ================================= pit ================================= */
namespace pit {

lgssm::FilterResult parallel_filter(const lgssm::Model& model, const Mat& obs, int) {
  return detail::run_filter(model, obs, 1);
}

Trajectory prefix_sample(const lgssm::Model& model, const lgssm::FilterResult& fr,
                         NoiseSource& noise, int) {
  return detail::sample_one(model, fr, noise, AUXMC_SAMPLER_PREFIX, "prefix_sample");
}

Trajectory prefix_sample(const lgssm::Model& model, const lgssm::FilterResult& fr,
                         RngStream rng, int workers) {
  StreamNoise n(rng);
  return prefix_sample(model, fr, n, workers);
}

Trajectory dnc_sample(const lgssm::Model& model, const lgssm::FilterResult& fr,
                      NoiseSource& noise, int) {
  return detail::sample_one(model, fr, noise, AUXMC_SAMPLER_DNC, "dnc_sample");
}

Trajectory dnc_sample(const lgssm::Model& model, const lgssm::FilterResult& fr, RngStream rng,
                      int workers) {
  StreamNoise n(rng);
  return dnc_sample(model, fr, n, workers);
}

gauss::Gaussian extract_affine_law(Sampler which, const lgssm::Model& model,
                                   const lgssm::FilterResult& fr) {
  const int T = model.horizon(), dx = model.dx(), n = (T + 1) * dx;
  const auxmc_lgssm& m = model.device();
  detail::DeviceFilter dfr(fr, T, dx);
  const int s = static_cast<int>(which);
  DeviceBuffer mean(sizeof(double) * n), cov(sizeof(double) * n * n), status(sizeof(int));
  const size_t wsb = auxmc_affine_law_workspace(&m, s);
  DeviceBuffer ws(std::max<size_t>(wsb, 1));
  check_status(auxmc_affine_law(&m, &dfr.desc, s, mean.as<double>(), cov.as<double>(),
                                status.as<int>(), ws.get(), wsb, nullptr),
               "extract_affine_law");
  int st = 0;
  status.download(&st, sizeof(int));
  check_status(st, "extract_affine_law");
  gauss::Gaussian g{Vec(n), Mat(n, n)};
  mean.download(g.mean.data(), sizeof(double) * n);
  cov.download(g.cov.data(), sizeof(double) * n * n);
  return g;
}

struct PathBatch::Impl {
  const lgssm::Model& model;
  detail::DeviceFilter fr;
  int sampler;
  DeviceBuffer keys, traj, status;
  detail::Workspace ws;
  size_t wsb;
  Impl(const lgssm::Model& m, const lgssm::FilterResult& f, int C, int s)
      : model(m), fr(f, m.horizon(), m.dx()), sampler(s), keys(sizeof(std::uint64_t) * C),
        traj(sizeof(double) * C * (m.horizon() + 1) * m.dx()), status(sizeof(int) * C),
        wsb(auxmc_sample_paths_workspace(&m.device(), 1, C, s)) {}
};

PathBatch::PathBatch(const lgssm::Model& model, const lgssm::FilterResult& fr, int C,
                     Sampler which)
    : impl_(new Impl(model, fr, C, static_cast<int>(which))), C_(C) {
  require_dim(C > 0, "PathBatch: C must be positive");
}

PathBatch::~PathBatch() = default;

void PathBatch::draw(const std::vector<RngStream>& roots) {
  require_dim(roots.size() == static_cast<size_t>(C_), "PathBatch::draw: one root per chain");
  std::vector<std::uint64_t> k(C_);
  for (int c = 0; c < C_; ++c) k[c] = roots[c].key();
  impl_->keys.upload(k.data(), k.size() * sizeof(std::uint64_t));
  auxmc_noise nz{};
  nz.kind = AUXMC_NOISE_STREAM;
  nz.keys = impl_->keys.as<std::uint64_t>();
  const auxmc_lgssm& m = impl_->model.device();
  check_status(auxmc_sample_paths(&m, &impl_->fr.desc, 1, &nz, C_, impl_->sampler,
                                  impl_->traj.as<double>(), impl_->status.as<int>(),
                                  impl_->ws.get(impl_->wsb), impl_->wsb, nullptr),
               "PathBatch::draw");
  std::vector<int> st(C_);
  impl_->status.download(st.data(), st.size() * sizeof(int));
  for (int c = 0; c < C_; ++c)
    check_status(st[c], "PathBatch::draw chain " + std::to_string(c));
}

Trajectory PathBatch::path(int c) const {
  const int T1 = impl_->model.horizon() + 1, dx = impl_->model.dx();
  require_dim(c >= 0 && c < C_, "PathBatch::path: chain index");
  Trajectory out(T1, dx);
  detail::cuda_try(cudaMemcpy(out.data(), impl_->traj.as<double>() + static_cast<size_t>(c) * T1 * dx,
                              out.size() * sizeof(double), cudaMemcpyDeviceToHost),
                   "PathBatch::path");
  return out;
}

const double* PathBatch::device_paths() const { return impl_->traj.as<double>(); }

}  // namespace pit

/* ============================ bench models ============================= */
namespace bench {

static int kind_code(const std::string& kind) {
  if (kind == "lgssm-synthetic") return AUXMC_KIND_LGSSM;
  if (kind == "stochvol") return AUXMC_KIND_STOCHVOL;
  if (kind == "diffusion-smoothing") return AUXMC_KIND_LORENZ63;
  if (kind == "spatio-temporal") return AUXMC_KIND_SPATIO;
  if (kind == "grid-1d-test") return AUXMC_KIND_GRID1D;
  if (kind == "lorenz96") return AUXMC_KIND_LORENZ96;
  throw ConfigError("unknown model kind: " + kind);
}

auxmc_model_spec to_c(const ModelSpec& s) {
  auxmc_model_spec c;
  auxmc_spec_default(&c);
  c.kind = kind_code(s.kind);
  c.T = s.T;
  c.dx = s.dx;
  c.dy = s.dy;
  c.grid = s.grid;
  c.data_seed = s.data_seed;
  c.sv_mu = s.sv_mu;
  c.sv_phi = s.sv_phi;
  c.sv_sig2 = s.sv_sig2;
  c.sv_rho = s.sv_rho;
  c.lz_sigma = s.lz_sigma;
  c.lz_rho = s.lz_rho;
  c.lz_beta = s.lz_beta;
  c.lz_h = s.lz_h;
  c.lz_gamma = s.lz_gamma;
  c.lz_obs_var = s.lz_obs_var;
  c.st_phi = s.st_phi;
  c.st_kappa2 = s.st_kappa2;
  c.st_tau2 = s.st_tau2;
  c.g1_phi = s.g1_phi;
  c.g1_q = s.g1_q;
  c.g1_m0 = s.g1_m0;
  c.g1_p0 = s.g1_p0;
  c.l96_F = s.l96_F;
  c.l96_h = s.l96_h;
  c.l96_gamma = s.l96_gamma;
  c.l96_obs_var = s.l96_obs_var;
  return c;
}

int latent_dim(const ModelSpec& spec) {
  auxmc_model_spec c = to_c(spec);
  return auxmc_latent_dim(&c);
}

int obs_dim(const ModelSpec& spec) {
  auxmc_model_spec c = to_c(spec);
  return auxmc_obs_dim(&c);
}

SimResult simulate(const ModelSpec& spec) {
  auxmc_model_spec c = to_c(spec);
  const int dx = auxmc_latent_dim(&c), dy = auxmc_obs_dim(&c);
  SimResult r{Trajectory(spec.T + 1, dx), Mat(spec.T + 1, dy)};
  std::vector<double> data(static_cast<size_t>(spec.T + 1) * std::max(dy, 1));
  check_status(auxmc_simulate(&c, r.latent.data(), data.data()), "simulate");
  if (dy > 0) std::memcpy(r.data.data(), data.data(), r.data.size() * sizeof(double));
  return r;
}

lgssm::Model synthetic_lgssm(const ModelSpec& spec) {
  auxmc_model_spec c = to_c(spec);
  const int dx = spec.dx, dy = spec.dy;
  Vec m0(dx), b(dx);
  Mat P0(dx, dx), F(dx, dx), Q(dx, dx), H(dy, dx), R(dy, dy);
  check_status(auxmc_synth_mats(&c, m0.data(), b.data(), P0.data(), F.data(), Q.data(), H.data(),
                                R.data()),
               "synth_mats");
  return lgssm::Model::homogeneous(spec.T, m0, P0, F, b, Q, H, Vec(dy, 0.0), R);
}

}  // namespace bench

/* =============================== targets =============================== */
namespace auxk {

struct GenSSMTarget::Impl {
  int kind = 0, T = 0, dx = 0, ydim = 0, q = 0, ne = 1;
  bool linear = true;
  Vec m0;
  std::vector<double> P0, F, b, Q, eH, ec, eR, ey, data, gH, gc, gR;
  int nF = 1;
  std::vector<std::uint8_t> emask, gmask;
  double lz_sigma = 10.0, lz_rho = 28.0, lz_beta = 8.0 / 3.0, lz_h = 0.01, l96_F = 8.0,
         l96_h = 0.01;
  DeviceBuffer dm0, dP0, dF, db, dQ, deH, dec, deR, dey, demask, ddata, dgmask, dgH, dgc, dgR;
  auxmc_target desc{};
  bool uploaded = false;

  void upload() {
    if (uploaded) return;
    auto up = [](const std::vector<double>& v) { return detail::upload_vec(v); };
    dm0 = up(m0);
    dP0 = up(P0);
    dF = up(F);
    db = up(b);
    dQ = up(Q);
    deH = up(eH);
    dec = up(ec);
    deR = up(eR);
    dey = up(ey);
    ddata = up(data);
    dgH = up(gH);
    dgc = up(gc);
    dgR = up(gR);
    demask = detail::upload_vec(emask);
    dgmask = detail::upload_vec(gmask);
    auto p = [](const DeviceBuffer& d) { return d.bytes() ? d.as<double>() : nullptr; };
    auxmc_target& t = desc;
    t.kind = kind;
    t.T = T;
    t.dx = dx;
    t.ydim = ydim;
    t.linear = linear ? 1 : 0;
    t.m0 = p(dm0);
    t.P0 = p(dP0);
    t.F = p(dF);
    t.b = p(db);
    t.Q = p(dQ);
    t.nF = nF;
    t.q = q;
    t.ne = ne;
    const bool mixed = !emask.empty() &&
                       *std::min_element(emask.begin(), emask.end()) !=
                           *std::max_element(emask.begin(), emask.end());
    t.exact_tv = (q > 0 && (ne > 1 || mixed)) ? 1 : 0;
    t.eH = p(deH);
    t.ec = p(dec);
    t.eR = p(deR);
    t.ey = p(dey);
    t.emask = demask.as<std::uint8_t>();
    t.data = p(ddata);
    t.gmask = dgmask.as<std::uint8_t>();
    t.gH = p(dgH);
    t.gc = p(dgc);
    t.gR = p(dgR);
    t.lz_sigma = lz_sigma;
    t.lz_rho = lz_rho;
    t.lz_beta = lz_beta;
    t.lz_h = lz_h;
    t.l96_F = l96_F;
    t.l96_h = l96_h;
    t.exact_sel = exact_selection() ? 1 : 0;
    uploaded = true;
  }

  // auxmc_target::exact_sel: unit selection rows, diagonal positive R_e, ne = 1
  bool exact_selection() const {
    if (q == 0) return true;
    if (ne != 1) return false;
    std::vector<int> used(dx, 0);
    for (int k = 0; k < q; ++k) {
      int nz = 0, col = -1;
      for (int j = 0; j < dx; ++j)
        if (eH[(size_t)k * dx + j] != 0.0) {
          ++nz;
          col = j;
          if (eH[(size_t)k * dx + j] != 1.0) return false;
        }
      if (nz != 1 || used[col]++) return false;
      for (int j = 0; j < q; ++j) {
        const double v = eR[(size_t)k * q + j];
        if (j == k ? !(v > 0.0) : v != 0.0) return false;
      }
    }
    return true;
  }
};

int GenSSMTarget::horizon() const { return impl_->T; }
int GenSSMTarget::dx() const { return impl_->dx; }
int GenSSMTarget::max_exact_rows() const { return impl_->q; }
const Vec& GenSSMTarget::m0() const { return impl_->m0; }
const auxmc_target& GenSSMTarget::device() const {
  impl_->upload();
  return impl_->desc;
}

// testutil.hpp:88-140 (linear_exact / linear_generic)
GenSSMTarget GenSSMTarget::from_lgssm(const lgssm::Model& m, const Mat& obs, bool generic) {
  const int T = m.horizon(), d = m.dx(), dy = m.dy();
  require_dim(obs.rows() == T + 1 && obs.cols() == dy, "from_lgssm: obs shape");
  auto im = std::make_shared<Impl>();
  im->kind = generic ? AUXMC_KIND_GAUSS_GENERIC : AUXMC_KIND_LGSSM;
  im->T = T;
  im->dx = d;
  im->m0 = m.m0();
  im->P0.assign(m.P0().data(), m.P0().data() + m.P0().size());
  bool dyn_tv = false, obs_tv = false;
  for (int t = 1; t < T && !dyn_tv; ++t)
    dyn_tv = &m.F(t) != &m.F(0) || &m.b(t) != &m.b(0) || &m.Q(t) != &m.Q(0);
  for (int t = 1; t <= T && !obs_tv; ++t)
    obs_tv = &m.H(t) != &m.H(0) || &m.c(t) != &m.c(0) || &m.R(t) != &m.R(0);
  const int nd = dyn_tv ? T : 1, ne = obs_tv ? T + 1 : 1;
  for (int t = 0; t < nd; ++t) {
    detail::append(im->F, m.F(t));
    im->b.insert(im->b.end(), m.b(t).begin(), m.b(t).end());
    detail::append(im->Q, m.Q(t));
  }
  im->nF = nd;
  std::vector<double> H, c, R;
  for (int t = 0; t < ne; ++t) {
    detail::append(H, m.H(t));
    c.insert(c.end(), m.c(t).begin(), m.c(t).end());
    detail::append(R, m.R(t));
  }
  std::vector<std::uint8_t> mask(T + 1);
  for (int t = 0; t <= T; ++t) mask[t] = m.observed(t) ? 1 : 0;
  im->ne = ne;
  if (generic) {
    im->ydim = dy;
    im->data.assign(obs.data(), obs.data() + obs.size());
    im->gmask = mask;
    im->emask.assign(T + 1, 0);
    im->gH = H;
    im->gc = c;
    im->gR = R;
  } else {
    im->q = dy;
    im->eH = H;
    im->ec = c;
    im->eR = R;
    im->ey.assign(obs.data(), obs.data() + obs.size());
    im->emask = dy > 0 ? mask : std::vector<std::uint8_t>(T + 1, 0);
    im->gmask.assign(T + 1, 0);
  }
  return GenSSMTarget(im);
}

double GenSSMTarget::log_gamma(const Trajectory& x) const {
  require_dim(x.rows() == impl_->T + 1 && x.cols() == impl_->dx, "log_gamma: trajectory shape");
  const auxmc_target& t = device();
  DeviceBuffer dx_(x.data(), x.size() * sizeof(double)), out(sizeof(double)), st(sizeof(int));
  check_status(auxmc_log_gamma(&t, dx_.as<double>(), 1, out.as<double>(), st.as<int>(), nullptr),
               "log_gamma");
  double v = 0.0;
  out.download(&v, sizeof v);
  return v;
}

}  // namespace auxk

namespace bench {

// models.cpp:240-336
auxk::GenSSMTarget make_target(const ModelSpec& spec, const Mat& data) {
  auxmc_model_spec c = to_c(spec);
  const int dx = auxmc_latent_dim(&c), dy = auxmc_obs_dim(&c), T = spec.T;
  require_dim(data.rows() == T + 1 && data.cols() == std::max(dy, 0), "make_target: data shape");
  auto im = std::make_shared<auxk::GenSSMTarget::Impl>();
  im->kind = c.kind;
  im->T = T;
  im->dx = dx;
  im->m0.assign(dx, 0.0);
  im->P0.assign(dx * dx, 0.0);
  im->F.assign(dx * dx, 0.0);
  im->b.assign(dx, 0.0);
  im->Q.assign(dx * dx, 0.0);
  check_status(auxmc_target_params(&c, im->m0.data(), im->P0.data(), im->F.data(), im->b.data(),
                                   im->Q.data()),
               "make_target");
  im->emask.assign(T + 1, 0);
  im->gmask.assign(T + 1, 0);
  const std::vector<double> d(data.data(), data.data() + data.size());
  switch (c.kind) {
    case AUXMC_KIND_LGSSM: {
      Vec m0(dx), b(dx);
      Mat P0(dx, dx), F(dx, dx), Q(dx, dx), H(dy, dx), R(dy, dy);
      check_status(auxmc_synth_mats(&c, m0.data(), b.data(), P0.data(), F.data(), Q.data(),
                                    H.data(), R.data()),
                   "make_target");
      im->q = dy;
      im->eH.assign(H.data(), H.data() + H.size());
      im->ec.assign(dy, 0.0);
      im->eR.assign(R.data(), R.data() + R.size());
      im->ey = d;
      im->emask.assign(T + 1, dy > 0 ? 1 : 0);
      break;
    }
    case AUXMC_KIND_STOCHVOL:
    case AUXMC_KIND_SPATIO:
    case AUXMC_KIND_GRID1D:
      if (dy > 0) {
        im->ydim = dy;
        im->data = d;
      }
      im->gmask.assign(T + 1, 1);
      break;
    case AUXMC_KIND_LORENZ63:
    case AUXMC_KIND_LORENZ96: {
      im->linear = false;
      im->F.clear();
      im->b.clear();
      const int q = dy;
      im->q = q;
      im->eH.assign(q * dx, 0.0);
      for (int k = 0; k < q; ++k) im->eH[k * dx + 2 * k] = 1.0;
      im->ec.assign(q, 0.0);
      im->eR.assign(q * q, 0.0);
      const double ov = c.kind == AUXMC_KIND_LORENZ63 ? spec.lz_obs_var : spec.l96_obs_var;
      for (int k = 0; k < q; ++k) im->eR[k * q + k] = ov;
      im->ey = d;
      im->emask.assign(T + 1, q > 0 ? 1 : 0);
      im->lz_sigma = spec.lz_sigma;
      im->lz_rho = spec.lz_rho;
      im->lz_beta = spec.lz_beta;
      im->lz_h = spec.lz_h;
      im->l96_F = spec.l96_F;
      im->l96_h = spec.l96_h;
      break;
    }
    default:
      throw ConfigError("make_target: unsupported kind " + spec.kind);
  }
  return auxk::GenSSMTarget(im);
}

}  // namespace bench

}  // inline namespace b200
}  // namespace auxmc
