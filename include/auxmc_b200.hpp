/*
 * auxmc_b200.hpp — C++ host facade of the B200 hot path, with the reference's
 * model / sampler API (auxmc 0.1.0, proj/include/auxmc/ headers).
 *
 * A user of the reference includes this header instead of the auxmc/ headers (lgssm, pit, auxk,
 * fkpg, bench/) and keeps the same calls: auxmc::lgssm::kalman_filter,
 * auxmc::pit::prefix_sample, auxmc::auxk::kernel_step, auxmc::fkpg::aux_pgibbs_step,
 * auxmc::bench::run, ...  Every compute call goes through the C ABI of
 * include/auxmc_gpu.h (libauxmc_b200.so) on an sm_100 device; there is no CPU
 * path, and without a device every compute call throws CudaError.
 *
 * Differences from the reference, all at the type level:
 *  - Mat is a small row-major dense matrix (Eigen is not a dependency); Vec is
 *    std::vector<double>; Trajectory is Mat with one state per row (common.hpp:11-14).
 *  - Symbols live in the inline namespace auxmc::b200, so a program can link this
 *    library and the reference side by side without ODR clashes.
 *  - Batched classes (pit::PathBatch, auxk::AuxChains, fkpg::PGChains) run many
 *    chains per call with state resident in HBM — the form the GPU is built for.
 *    The single-chain functions are those classes at C = 1 with host copies.
 *  - KernelOptions::workers and the scan worker count are accepted and ignored
 *    (the reference's fixed-tree results do not depend on them, scan.hpp:16-21).
 */
#ifndef AUXMC_B200_HPP
#define AUXMC_B200_HPP

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "auxmc_gpu.h"

namespace auxmc {
inline namespace b200 {

/* ---- common.hpp:11-43 ---- */
using Vec = std::vector<double>;

class Mat {
 public:
  Mat() = default;
  Mat(int rows, int cols, double fill = 0.0)
      : r_(rows), c_(cols), v_(static_cast<size_t>(rows) * cols, fill) {}
  static Mat Zero(int rows, int cols) { return Mat(rows, cols); }
  static Mat Identity(int n) {
    Mat m(n, n);
    for (int i = 0; i < n; ++i) m(i, i) = 1.0;
    return m;
  }
  static Mat Constant(int rows, int cols, double v) { return Mat(rows, cols, v); }
  int rows() const { return r_; }
  int cols() const { return c_; }
  size_t size() const { return v_.size(); }
  double& operator()(int i, int j) { return v_[static_cast<size_t>(i) * c_ + j]; }
  double operator()(int i, int j) const { return v_[static_cast<size_t>(i) * c_ + j]; }
  double* data() { return v_.data(); }
  const double* data() const { return v_.data(); }
  Vec row(int i) const { return Vec(v_.begin() + static_cast<size_t>(i) * c_,
                                    v_.begin() + static_cast<size_t>(i + 1) * c_); }

 private:
  int r_ = 0, c_ = 0;
  std::vector<double> v_;
};
using Trajectory = Mat;  // (T+1) x d_x, one state per row

struct Error : std::runtime_error { using std::runtime_error::runtime_error; };
struct FactorizationError : Error { using Error::Error; };
struct DimensionError : Error { using Error::Error; };
struct DegenerateWeightsError : Error { using Error::Error; };
struct ContractError : Error { using Error::Error; };
struct ConfigError : Error { using Error::Error; };
/* New: no usable sm_100 device, or a CUDA failure (the product has no CPU path). */
struct CudaError : Error { using Error::Error; };

inline void require_dim(bool ok, const std::string& what) {
  if (!ok) throw DimensionError(what);
}

/* Throws the exception class that matches an AUXMC_E_* status. */
void check_status(int status, const std::string& what);

/* ---- rng.hpp:14-137 ---- */
namespace stream {
constexpr std::uint64_t kBackwardNoise = AUXMC_L_BACKWARD_NOISE;
constexpr std::uint64_t kTerminalDraw = AUXMC_L_TERMINAL_DRAW;
constexpr std::uint64_t kAuxObs = AUXMC_L_AUX_OBS;
constexpr std::uint64_t kDncBridge = AUXMC_L_DNC_BRIDGE;
constexpr std::uint64_t kMhAccept = AUXMC_L_MH_ACCEPT;
constexpr std::uint64_t kIteration = AUXMC_L_ITERATION;
constexpr std::uint64_t kChain = AUXMC_L_CHAIN;
constexpr std::uint64_t kStep = AUXMC_L_STEP;
constexpr std::uint64_t kParticle = AUXMC_L_PARTICLE;
constexpr std::uint64_t kResample = AUXMC_L_RESAMPLE;
constexpr std::uint64_t kTerminalIndex = AUXMC_L_TERMINAL_INDEX;
constexpr std::uint64_t kBackwardIndex = AUXMC_L_BACKWARD_INDEX;
constexpr std::uint64_t kPmKey = AUXMC_L_PM_KEY;
constexpr std::uint64_t kSimulate = AUXMC_L_SIMULATE;
constexpr std::uint64_t kParam = AUXMC_L_PARAM;
}  // namespace stream

class RngStream {
 public:
  RngStream() = default;
  static RngStream from_seed(std::uint64_t seed) { return from_key(auxmc_rng_from_seed(seed)); }
  static RngStream from_key(std::uint64_t key) {
    RngStream s;
    s.key_ = key;
    return s;
  }
  RngStream derive(std::uint64_t label, std::uint64_t index) const {
    return from_key(auxmc_rng_derive(key_, label, index));
  }
  std::uint64_t key() const { return key_; }
  std::uint64_t counter() const { return counter_; }
  double next_uniform() { return auxmc_rng_uniform(key_, counter_++); }
  double next_normal() { return auxmc_rng_normal(key_, counter_++); }
  Vec normal_vec(int d) {
    Vec v(d);
    for (int i = 0; i < d; ++i) v[i] = next_normal();
    return v;
  }

 private:
  std::uint64_t key_ = 0, counter_ = 0;
};

/* NoiseSource (rng.hpp:123-137).  The device samplers read address-based noise:
 * a NoiseSource is pre-drawn at the addresses a sampler uses ((kTerminalDraw, 0),
 * (kBackwardNoise, t), (kDncBridge, id)); a StreamNoise is run on the device
 * counter RNG directly. */
struct NoiseSource {
  virtual ~NoiseSource() = default;
  virtual Vec normal(std::uint64_t label, std::uint64_t index, int dim) = 0;
};
struct StreamNoise final : NoiseSource {
  explicit StreamNoise(RngStream base) : base_(base) {}
  Vec normal(std::uint64_t label, std::uint64_t index, int dim) override {
    RngStream s = base_.derive(label, index);
    return s.normal_vec(dim);
  }
  const RngStream& base() const { return base_; }

 private:
  RngStream base_;
};

namespace detail {
/* RAII device allocation (cudaMalloc / cudaFree). */
class DeviceBuffer {
 public:
  DeviceBuffer() = default;
  explicit DeviceBuffer(size_t bytes);
  DeviceBuffer(const void* host, size_t bytes);
  ~DeviceBuffer();
  DeviceBuffer(DeviceBuffer&& o) noexcept : p_(o.p_), n_(o.n_) { o.p_ = nullptr; o.n_ = 0; }
  DeviceBuffer& operator=(DeviceBuffer&& o) noexcept;
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  void* get() const { return p_; }
  template <class T> T* as() const { return static_cast<T*>(p_); }
  size_t bytes() const { return n_; }
  void upload(const void* host, size_t bytes);
  void download(void* host, size_t bytes) const;

 private:
  void* p_ = nullptr;
  size_t n_ = 0;
};
/* Growable device workspace. */
struct Workspace {
  DeviceBuffer buf;
  void* get(size_t bytes) {
    if (buf.bytes() < bytes || !buf.get()) buf = DeviceBuffer(bytes < 256 ? 256 : bytes);
    return buf.get();
  }
};
void synchronize();
}  // namespace detail

/* ---- gauss.hpp: the Gaussian law type ---- */
namespace gauss {
struct Gaussian {
  Vec mean;
  Mat cov;
  int dim() const { return static_cast<int>(mean.size()); }
};
}  // namespace gauss

/* ---- lgssm.hpp:19-91 ---- */
namespace lgssm {

class Model {
 public:
  Model(int T, Vec m0, Mat P0, std::vector<Mat> F, std::vector<Vec> b, std::vector<Mat> Q,
        std::vector<Mat> H, std::vector<Vec> c, std::vector<Mat> R,
        std::vector<std::uint8_t> obs_mask = {});
  static Model homogeneous(int T, Vec m0, Mat P0, Mat F, Vec b, Mat Q, Mat H, Vec c, Mat R,
                           std::vector<std::uint8_t> obs_mask = {});
  int horizon() const { return T_; }
  int dx() const { return dx_; }
  int dy() const { return dy_; }
  const Vec& m0() const { return m0_; }
  const Mat& P0() const { return P0_; }
  const Mat& F(int t) const { return F_[F_.size() > 1 ? t : 0]; }
  const Vec& b(int t) const { return b_[b_.size() > 1 ? t : 0]; }
  const Mat& Q(int t) const { return Q_[Q_.size() > 1 ? t : 0]; }
  const Mat& H(int t) const { return H_[H_.size() > 1 ? t : 0]; }
  const Vec& c(int t) const { return c_[c_.size() > 1 ? t : 0]; }
  const Mat& R(int t) const { return R_[R_.size() > 1 ? t : 0]; }
  bool observed(int t) const { return mask_.empty() || mask_[t] != 0; }

  /* Device copy (uploaded once, on first use) as the C-ABI descriptor. */
  const auxmc_lgssm& device() const;

 private:
  int T_, dx_, dy_;
  Vec m0_;
  Mat P0_;
  std::vector<Mat> F_, Q_, H_, R_;
  std::vector<Vec> b_, c_;
  std::vector<std::uint8_t> mask_;
  struct Dev;
  mutable std::shared_ptr<Dev> dev_;
};

struct FilterResult {
  std::vector<Vec> pred_mean, filt_mean;  // per t = 0..T
  std::vector<Mat> pred_cov, filt_cov;
  double log_marginal = 0.0;
};

FilterResult kalman_filter(const Model& model, const Mat& obs);
/* Marginal smoothing distributions N(m_t^s, P_t^s) per t (lgssm.cpp:114-127). */
std::vector<gauss::Gaussian> rts_smoother(const Model& model, const FilterResult& fr);
Trajectory backward_sample(const Model& model, const FilterResult& fr, NoiseSource& noise);
Trajectory backward_sample(const Model& model, const FilterResult& fr, RngStream rng);
double path_logpdf(const Model& model, const Mat& obs, const Trajectory& traj,
                   const FilterResult& fr);

}  // namespace lgssm

/* ---- pit.hpp:44-87 ---- */
namespace pit {

enum class Sampler { kSequential, kPrefix, kDnc };

lgssm::FilterResult parallel_filter(const lgssm::Model& model, const Mat& obs,
                                    int workers = 1);
Trajectory prefix_sample(const lgssm::Model& model, const lgssm::FilterResult& fr,
                         NoiseSource& noise, int workers = 1);
Trajectory prefix_sample(const lgssm::Model& model, const lgssm::FilterResult& fr,
                         RngStream rng, int workers = 1);
Trajectory dnc_sample(const lgssm::Model& model, const lgssm::FilterResult& fr,
                      NoiseSource& noise, int workers = 1);
Trajectory dnc_sample(const lgssm::Model& model, const lgssm::FilterResult& fr,
                      RngStream rng, int workers = 1);

/* Exact induced law over the flattened path (index t*d_x + j), pit.cpp:303-332:
 * the zero noise and every basis noise vector pushed through the device sampler
 * as one pre-drawn batch.  Test-scale (memory grows as ((T+1) d_x)^2). */
gauss::Gaussian extract_affine_law(Sampler which, const lgssm::Model& model,
                                   const lgssm::FilterResult& fr);

/* Batched pathwise draws (new): C paths from one filter result, path c drawn with
 * StreamNoise(roots[c]) — the C2 workload (one model, many chains).  The filter
 * result and the paths stay in HBM; draw() is one launch sequence on the device. */
class PathBatch {
 public:
  PathBatch(const lgssm::Model& model, const lgssm::FilterResult& fr, int C, Sampler which);
  ~PathBatch();
  PathBatch(const PathBatch&) = delete;
  PathBatch& operator=(const PathBatch&) = delete;
  void draw(const std::vector<RngStream>& roots);   // keys uploaded per call
  Trajectory path(int c) const;                     // device -> host copy of one path
  const double* device_paths() const;               // [C][T+1][dx]
  int chains() const { return C_; }

 private:
  struct Impl;
  std::unique_ptr<Impl> impl_;
  int C_;
};

}  // namespace pit

/* ---- bench/models.hpp:16-89 (+ the Lorenz-96 model the benchmark configs name) ---- */
namespace bench {

struct ModelSpec {
  std::string kind = "lgssm-synthetic";
  // lgssm-synthetic | stochvol | diffusion-smoothing | spatio-temporal |
  // grid-1d-test | lorenz96 (new)
  int T = 50;
  int dx = 2;
  int dy = 1;
  int grid = 3;
  std::uint64_t data_seed = 1;
  double sv_mu = -1.0, sv_phi = 0.9, sv_sig2 = 0.1, sv_rho = 0.25;
  double lz_sigma = 10.0, lz_rho = 28.0, lz_beta = 8.0 / 3.0, lz_h = 0.01, lz_gamma = 2.0,
         lz_obs_var = 1.0;
  double st_phi = 0.8, st_kappa2 = 1.0, st_tau2 = 0.3;
  double g1_phi = 0.8, g1_q = 0.09, g1_m0 = 0.5, g1_p0 = 0.25;
  double l96_F = 8.0, l96_h = 0.01, l96_gamma = 1.0, l96_obs_var = 1.0;
};

int latent_dim(const ModelSpec& spec);
int obs_dim(const ModelSpec& spec);
auxmc_model_spec to_c(const ModelSpec& spec);

struct SimResult {
  Trajectory latent;  // (T+1) x latent_dim
  Mat data;           // (T+1) x obs_dim
};
SimResult simulate(const ModelSpec& spec);
lgssm::Model synthetic_lgssm(const ModelSpec& spec);

}  // namespace bench

/* ---- target.hpp:34-93 ---- */
namespace auxk {

class GenSSMTarget {
 public:
  /* testutil.hpp:88-140: an LGSSM posterior as a target, with the Gaussian
   * potentials exact (generic = false) or in generic form (generic = true). */
  static GenSSMTarget from_lgssm(const lgssm::Model& model, const Mat& obs,
                                 bool generic = false);
  int horizon() const;
  int dx() const;
  int max_exact_rows() const;
  const Vec& m0() const;
  /* log gamma(x) (target.cpp:100-108) on the device. */
  double log_gamma(const Trajectory& x) const;
  const auxmc_target& device() const;

  struct Impl;
  explicit GenSSMTarget(std::shared_ptr<Impl> impl) : impl_(std::move(impl)) {}

 private:
  std::shared_ptr<Impl> impl_;
};

}  // namespace auxk

namespace bench {
/* models.cpp:240-336 */
auxk::GenSSMTarget make_target(const ModelSpec& spec, const Mat& data);
}  // namespace bench

/* ---- auxk.hpp:15-79 ---- */
namespace auxk {

enum class Backend { kSequential, kPrefix, kDnc };

struct KernelOptions {
  Backend backend = Backend::kSequential;
  bool parallel_filter = false;
  bool zeroth_order = false;
  int workers = 1;
};

struct KernelStats {
  long accepted = 0;
  long rejected = 0;
  long aborted = 0;
  long nonfinite_gamma = 0;
  double last_log_alpha = 0.0;
  double last_accept_prob = 0.0;
};

struct AuxChainState {
  Trajectory x;
  double delta = 1.0;
  double log_gamma = 0.0;
  std::vector<Vec> grad_gen;
  long iter = 0;
  KernelStats stats;
};

AuxChainState init_chain(const GenSSMTarget& target, Trajectory x0, double delta);
void kernel_step(const GenSSMTarget& target, AuxChainState& state, RngStream rng,
                 const KernelOptions& opts = {});
void adapt_delta(AuxChainState& state, double target_rate);

/* Batched chains (new): C states resident in HBM, chain c rooted at roots[c]
 * (the batched form of runner.cpp:132 is from_seed(seed).derive(kChain, c)). */
class AuxChains {
 public:
  AuxChains(const GenSSMTarget& target, const Trajectory& x0, double delta,
            const std::vector<RngStream>& roots);
  static AuxChains seeded(const GenSSMTarget& target, const Trajectory& x0, double delta,
                          std::uint64_t seed, int C);
  ~AuxChains();
  AuxChains(AuxChains&&) noexcept;
  AuxChains(const AuxChains&) = delete;
  AuxChains& operator=(const AuxChains&) = delete;
  void kernel_step(const KernelOptions& opts = {});   // every chain, asynchronous
  void adapt_delta(double target_rate);               // every chain, asynchronous
  int chains() const;
  AuxChainState state(int c) const;                   // synchronizes, copies one chain
  void set_state(int c, const AuxChainState& s);
  std::vector<KernelStats> stats() const;
  std::vector<double> deltas() const;
  /* Gather x[c][t][j] for the given flat coordinates (t*dx + j) of every chain
   * into out[c * coords.size() + k] (one device gather + one copy). */
  void gather(const std::vector<long>& coords, std::vector<double>& out) const;
  /* bench/runner.cpp:61-85 gamma_move for every chain (device; Lorenz targets): stream
   * root_c.derive(kParam, iter); gamma[c] updated in place when chain c's move is
   * accepted; returns the accept flags. */
  std::vector<int> gamma_move(long iter, double step, std::vector<double>& gamma);
  /* Swap the target (runner.cpp:162-167: a new γ) and recompute log γ(x) and the
   * gradients for the current paths; x, δ, iteration counts and stats are kept. */
  void retarget(const GenSSMTarget& target);

 private:
  struct Impl;
  std::unique_ptr<Impl> impl_;
};

}  // namespace auxk

/* ---- fkpg.hpp:58-109 (proposals linearized at the aux observation) ---- */
namespace fkpg {

enum class ProposalMode { kPrior, kGradient, kFullyAdapted };
enum class LinearizeAt { kAuxObs, kPredictedMean };
/* Which cSMC runs the sweep: the reference's sequential cSMC (fkpg.cpp:44-152) or
 * the parallel-in-time cSMC with independent proposals (new). */
enum class Variant { kReference, kPit };

struct PgOptions {
  ProposalMode mode = ProposalMode::kGradient;
  LinearizeAt linearize = LinearizeAt::kAuxObs;
  Variant variant = Variant::kReference;
};

struct PGState {
  Trajectory x;
  std::vector<std::uint64_t> keys;
  double delta = 1.0;
  long iter = 0;
  long updates = 0;
  double last_update = 0.0;
};

PGState init_pg(Trajectory x0, double delta);
void aux_pgibbs_step(const auxk::GenSSMTarget& target, PGState& state, int N, RngStream rng,
                     const PgOptions& opts = {});
void adapt_delta(PGState& state, double target_rate);

class PGChains {
 public:
  PGChains(const auxk::GenSSMTarget& target, const Trajectory& x0, double delta,
           const std::vector<RngStream>& roots, int N);
  static PGChains seeded(const auxk::GenSSMTarget& target, const Trajectory& x0, double delta,
                         std::uint64_t seed, int C, int N);
  ~PGChains();
  PGChains(PGChains&&) noexcept;
  PGChains(const PGChains&) = delete;
  PGChains& operator=(const PGChains&) = delete;
  /* One sweep for every chain; throws DegenerateWeightsError naming the chain and
   * step when any chain's weights collapsed (fkpg.cpp:19-27). */
  void aux_pgibbs_step(const PgOptions& opts = {});
  void adapt_delta(double target_rate);
  int chains() const;
  PGState state(int c) const;
  void set_state(int c, const PGState& s);
  std::vector<long> updates() const;
  std::vector<double> deltas() const;
  void gather(const std::vector<long>& coords, std::vector<double>& out) const;
  /* runner.cpp:190-196: gamma_move on every chain's path, and the target swap */
  std::vector<int> gamma_move(long iter, double step, std::vector<double>& gamma);
  void retarget(const auxk::GenSSMTarget& target);

 private:
  struct Impl;
  std::unique_ptr<Impl> impl_;
};

}  // namespace fkpg

/* ---- bench/config.hpp, bench/runner.hpp: the run driver (runner.cpp:112-244) ---- */
namespace bench {

struct RunConfig {
  std::string sampler = "aux-kalman-seq";
  // aux-kalman-seq | aux-kalman-prefix | aux-kalman-dnc |
  // pgibbs-prior | pgibbs-gradient | pgibbs-adapted (reference cSMC) |
  // pgibbs-pit (parallel-in-time cSMC, gradient proposals; new)
  long chain_length = 1000;
  long burn_in = 100;
  int particles = 16;
  double delta_init = 1.0;
  double target_acceptance = 0.0;  // 0 = family default (0.574 / 0.9)
  std::uint64_t seed = 1;
  int workers = 1;                 // accepted, unused (device path)
  std::string output_dir = "out";
  std::vector<int> probe_times;
  bool parallel_filter = false;    // aux family: scan filter (KernelOptions)
  int chains = 1;                  // new: chains run as one batch; chain c rooted at
                                   // from_seed(seed).derive(kChain, c)
  bool sample_param = false;       // config.hpp:30 diffusion-coefficient move (Lorenz)
  double param_step = 0.2;         // config.hpp:31 random-walk scale on log gamma
  ModelSpec model;
};

bool is_aux_family(const std::string& sampler);
bool is_pgibbs_family(const std::string& sampler);

struct ChainSummary {
  std::vector<int> probe_times;
  std::vector<long> probe_coords;
  long kept = 0;
  Vec mean;   // per probe coordinate, pooled over the kept draws of all chains
  Vec sd;
  double rate = 0.0;          // acceptance / reference-update rate, kept phase, all chains
  double final_delta = 0.0;   // chain 0
  double burn_seconds = 0.0;
  double sample_seconds = 0.0;
  int chains = 1;
  bool has_param = false;     // sample_param: moments of γ over the kept iterations
  double param_mean = 0.0;
  double param_sd = 0.0;
};

struct RunResult {
  ChainSummary summary;
  std::string trace_path;
  std::string summary_path;
};

/* Burn-in with delta adaptation, then sampling with the kernel frozen; writes
 * <output_dir>/trace.csv (iter,coord_<flat>,... of chain 0, %.17g, the
 * reference's format) and <output_dir>/summary.json. */
RunResult run(const RunConfig& cfg);

}  // namespace bench

}  // inline namespace b200
}  // namespace auxmc

#endif  // AUXMC_B200_HPP
