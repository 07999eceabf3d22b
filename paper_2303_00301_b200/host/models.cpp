// models.cpp — host-side bench models of the product (bench/models.hpp:16-89):
// ModelSpec defaults, synth_mats (models.cpp:51-68), simulate (:162-238) and the
// parameter arrays of make_target (:240-336), plus the new Lorenz-96 model.
// Data generation runs once per workload on the host; the device path only
// consumes the arrays through include/auxmc_gpu.h.
#include <cmath>
#include <complex>
#include <cstring>
#include <functional>
#include <vector>

#include "../../include/auxmc_gpu.h"

namespace {

using V = std::vector<double>;

uint64_t mix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}

struct Stream {  // RngStream (rng.hpp:62-118)
  uint64_t key = 0, ctr = 0;
  static Stream seed(uint64_t s) { return {mix64(s + 0x9E3779B97F4A7C15ull), 0}; }
  Stream derive(uint64_t label, uint64_t index) const {
    uint64_t k = mix64(key ^ mix64(label ^ 0xA0761D6478BD642Full));
    k = mix64(k ^ mix64(index ^ 0xE7037ED1A0B428DBull));
    return {k, 0};
  }
  static double unit(uint64_t w) { return (static_cast<double>(w >> 11) + 0.5) * 0x1.0p-53; }
  uint64_t word(uint64_t i) const { return mix64(key + (i + 1) * 0x9E3779B97F4A7C15ull); }
  double uniform() { return unit(word(2 * ctr++)); }
  double normal() {
    const uint64_t c = ctr++;
    const double u1 = unit(word(2 * c)), u2 = unit(word(2 * c + 1));
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586476925286766559 * u2);
  }
  V normals(int d) {
    V v(d);
    for (auto& x : v) x = normal();
    return v;
  }
};

// Dense helpers (row-major n×n).
V matmul(const V& a, const V& b, int m, int k, int n) {
  V c(static_cast<size_t>(m) * n, 0.0);
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < n; ++j) {
      double s = 0.0;
      for (int l = 0; l < k; ++l) s += a[i * k + l] * b[l * n + j];
      c[i * n + j] = s;
    }
  return c;
}

// Lower Cholesky (no jitter needed for the model matrices, which are SPD by
// construction); zero matrix -> zero factor as chol_psd (gauss.cpp:45-49).
V cholesky(const V& a, int n) {
  V l(static_cast<size_t>(n) * n, 0.0);
  bool zero = true;
  for (double x : a) zero = zero && x == 0.0;
  if (zero) return l;
  for (int k = 0; k < n; ++k) {
    double x = a[k * n + k];
    for (int j = 0; j < k; ++j) x -= l[k * n + j] * l[k * n + j];
    x = std::sqrt(x);
    l[k * n + k] = x;
    for (int i = k + 1; i < n; ++i) {
      double s = a[i * n + k];
      for (int j = 0; j < k; ++j) s -= l[i * n + j] * l[k * n + j];
      l[i * n + k] = s / x;
    }
  }
  return l;
}

// (L L^T)^{-1} B, B n×r
V llt_solve(const V& l, int n, V b, int r) {
  for (int c = 0; c < r; ++c) {
    for (int i = 0; i < n; ++i) {
      double s = b[i * r + c];
      for (int j = 0; j < i; ++j) s -= l[i * n + j] * b[j * r + c];
      b[i * r + c] = s / l[i * n + i];
    }
    for (int i = n - 1; i >= 0; --i) {
      double s = b[i * r + c];
      for (int j = i + 1; j < n; ++j) s -= l[j * n + i] * b[j * r + c];
      b[i * r + c] = s / l[i * n + i];
    }
  }
  return b;
}

// Spectral radius by unshifted-then-shifted complex QR iteration on the
// Hessenberg form (Householder reduction, Wilkinson shifts, deflation).
double spectral_radius(const V& a, int n) {
  using Cx = std::complex<double>;
  std::vector<Cx> h(a.begin(), a.end());
  auto H = [&](int i, int j) -> Cx& { return h[static_cast<size_t>(i) * n + j]; };
  for (int k = 0; k + 2 < n; ++k) {  // Householder to Hessenberg
    double alpha = 0.0;
    for (int i = k + 1; i < n; ++i) alpha += std::norm(H(i, k));
    alpha = std::sqrt(alpha);
    if (alpha == 0.0) continue;
    std::vector<Cx> v(n, 0.0);
    const Cx x0 = H(k + 1, k);
    const Cx ph = std::abs(x0) > 0 ? x0 / std::abs(x0) : Cx(1.0);
    v[k + 1] = x0 + ph * alpha;
    for (int i = k + 2; i < n; ++i) v[i] = H(i, k);
    double vn = 0.0;
    for (int i = k + 1; i < n; ++i) vn += std::norm(v[i]);
    if (vn == 0.0) continue;
    for (int j = 0; j < n; ++j) {  // H = (I - 2vv*/v*v) H
      Cx s = 0.0;
      for (int i = k + 1; i < n; ++i) s += std::conj(v[i]) * H(i, j);
      s *= 2.0 / vn;
      for (int i = k + 1; i < n; ++i) H(i, j) -= v[i] * s;
    }
    for (int i = 0; i < n; ++i) {  // H = H (I - 2vv*/v*v)
      Cx s = 0.0;
      for (int j = k + 1; j < n; ++j) s += H(i, j) * v[j];
      s *= 2.0 / vn;
      for (int j = k + 1; j < n; ++j) H(i, j) -= s * std::conj(v[j]);
    }
  }
  double rad = 0.0;
  int hi = n - 1;
  int iter = 0;
  while (hi >= 0 && iter < 100 * n) {
    if (hi == 0) {
      rad = std::max(rad, std::abs(H(0, 0)));
      break;
    }
    const double sub = std::abs(H(hi, hi - 1));
    if (sub <= 1e-15 * (std::abs(H(hi, hi)) + std::abs(H(hi - 1, hi - 1))) || sub == 0.0) {
      rad = std::max(rad, std::abs(H(hi, hi)));
      --hi;
      iter = 0;
      continue;
    }
    // Wilkinson shift from the trailing 2x2
    const Cx a11 = H(hi - 1, hi - 1), a12 = H(hi - 1, hi), a21 = H(hi, hi - 1), a22 = H(hi, hi);
    const Cx tr = a11 + a22, det = a11 * a22 - a12 * a21;
    const Cx disc = std::sqrt(tr * tr - 4.0 * det);
    const Cx l1 = (tr + disc) / 2.0, l2 = (tr - disc) / 2.0;
    Cx mu = std::abs(l1 - a22) < std::abs(l2 - a22) ? l1 : l2;
    if (iter % 11 == 10) mu += Cx(sub, 0.0);  // exceptional shift
    int lo = hi;
    while (lo > 0 && std::abs(H(lo, lo - 1)) > 1e-15 * (std::abs(H(lo, lo)) + std::abs(H(lo - 1, lo - 1))))
      --lo;
    for (int i = lo; i <= hi; ++i) H(i, i) -= mu;
    std::vector<Cx> cs(n), sn(n);
    for (int k = lo; k < hi; ++k) {  // QR by Givens
      const Cx x = H(k, k), y = H(k + 1, k);
      const double r = std::sqrt(std::norm(x) + std::norm(y));
      const Cx c = r == 0 ? Cx(1.0) : x / r, s = r == 0 ? Cx(0.0) : y / r;
      cs[k] = c;
      sn[k] = s;
      for (int j = k; j < n; ++j) {
        const Cx u = H(k, j), w = H(k + 1, j);
        H(k, j) = std::conj(c) * u + std::conj(s) * w;
        H(k + 1, j) = -s * u + c * w;
      }
    }
    for (int k = lo; k < hi; ++k) {  // RQ
      const Cx c = cs[k], s = sn[k];
      for (int i = 0; i <= std::min(k + 2, hi); ++i) {
        const Cx u = H(i, k), w = H(i, k + 1);
        H(i, k) = u * c + w * s;
        H(i, k + 1) = -u * std::conj(s) + w * std::conj(c);
      }
    }
    for (int i = lo; i <= hi; ++i) H(i, i) += mu;
    ++iter;
  }
  return rad;
}

int latent(const auxmc_model_spec& s) {
  switch (s.kind) {
    case AUXMC_KIND_LGSSM: case AUXMC_KIND_STOCHVOL: case AUXMC_KIND_LORENZ96: return s.dx;
    case AUXMC_KIND_LORENZ63: return 3;
    case AUXMC_KIND_SPATIO: return s.grid * s.grid;
    case AUXMC_KIND_GRID1D: return 1;
  }
  return -1;
}
int obsdim(const auxmc_model_spec& s) {
  switch (s.kind) {
    case AUXMC_KIND_LGSSM: return s.dy;
    case AUXMC_KIND_STOCHVOL: return s.dx;
    case AUXMC_KIND_LORENZ63: return 1;
    case AUXMC_KIND_SPATIO: return s.grid * s.grid;
    case AUXMC_KIND_GRID1D: return 0;
    case AUXMC_KIND_LORENZ96: return (s.dx + 1) / 2;
  }
  return -1;
}

int check_spec(const auxmc_model_spec& s) {  // models.cpp:11-27
  if (s.T < 0 || s.dx < 1 || s.dy < 1 || s.grid < 1 || s.sv_sig2 < 0 || s.sv_rho < 0 ||
      s.sv_rho >= 1 || s.lz_h <= 0 || s.lz_gamma <= 0 || s.lz_obs_var <= 0 ||
      s.st_kappa2 <= 0 || s.st_tau2 <= 0 || std::abs(s.st_phi) >= 1 || s.g1_q <= 0 ||
      s.g1_p0 <= 0 || s.l96_h <= 0 || s.l96_gamma <= 0 || s.l96_obs_var <= 0)
    return AUXMC_E_CONFIG;
  if (latent(s) < 1) return AUXMC_E_CONFIG;
  return AUXMC_OK;
}

V random_spd(Stream& st, int d, double ridge) {  // models.cpp:39-43
  V g(static_cast<size_t>(d) * d);
  for (int i = 0; i < d; ++i) {
    V r = st.normals(d);
    for (int j = 0; j < d; ++j) g[i * d + j] = r[j];
  }
  V out(static_cast<size_t>(d) * d);
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < d; ++j) {
      double s = 0.0;
      for (int l = 0; l < d; ++l) s += g[i * d + l] * g[j * d + l];
      out[i * d + j] = s / d + (i == j ? ridge : 0.0);
    }
  return out;
}

struct Synth {
  V m0, b, P0, F, Q, H, R;
};

Synth synth(const auxmc_model_spec& s) {  // models.cpp:51-68
  Stream ms = Stream::seed(s.data_seed).derive(AUXMC_L_PARAM, 0);
  const int dx = s.dx, dy = s.dy;
  Synth m;
  m.F.resize(static_cast<size_t>(dx) * dx);
  for (int i = 0; i < dx; ++i) {
    V r = ms.normals(dx);
    for (int j = 0; j < dx; ++j) m.F[i * dx + j] = r[j] / std::sqrt(double(dx));
  }
  const double radius = spectral_radius(m.F, dx);
  const double scale = 0.7 / std::max(radius, 1e-12);
  for (auto& x : m.F) x *= scale;
  m.b = ms.normals(dx);
  for (auto& x : m.b) x *= 0.1;
  m.Q = random_spd(ms, dx, 0.1);
  m.m0 = ms.normals(dx);
  m.P0 = random_spd(ms, dx, 0.1);
  m.H.resize(static_cast<size_t>(dy) * dx);
  for (int i = 0; i < dy; ++i) {
    V r = ms.normals(dx);
    for (int j = 0; j < dx; ++j) m.H[i * dx + j] = r[j];
  }
  m.R = random_spd(ms, dy, 0.1);
  return m;
}

V lattice_laplacian(int k) {  // models.cpp:88-103
  const int n = k * k;
  V lap(static_cast<size_t>(n) * n, 0.0);
  auto link = [&](int a, int b) {
    lap[a * n + a] += 1.0;
    lap[b * n + b] += 1.0;
    lap[a * n + b] -= 1.0;
    lap[b * n + a] -= 1.0;
  };
  for (int r = 0; r < k; ++r)
    for (int c = 0; c < k; ++c) {
      if (c + 1 < k) link(r * k + c, r * k + c + 1);
      if (r + 1 < k) link(r * k + c, (r + 1) * k + c);
    }
  return lap;
}

V spatio_cov(const auxmc_model_spec& s) {  // models.cpp:105-111
  const int n = s.grid * s.grid;
  V prec = lattice_laplacian(s.grid);
  for (int i = 0; i < n; ++i) prec[i * n + i] += s.st_kappa2 * 1.0;
  V eye(static_cast<size_t>(n) * n, 0.0);
  for (int i = 0; i < n; ++i) eye[i * n + i] = 1.0;
  V cov = llt_solve(cholesky(prec, n), n, eye, n);
  for (auto& x : cov) x = s.st_tau2 * x;
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j) {
      const double v = (cov[i * n + j] + cov[j * n + i]) / 2.0;
      cov[i * n + j] = cov[j * n + i] = v;
    }
  return cov;
}

V stochvol_q(const auxmc_model_spec& s) {  // models.cpp:113-119
  const int d = s.dx;
  V q(static_cast<size_t>(d) * d);
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < d; ++j)
      q[i * d + j] = s.sv_sig2 * ((1.0 - s.sv_rho) * (i == j ? 1.0 : 0.0) + s.sv_rho * 1.0);
  return q;
}

V ar1_p0(double phi, const V& q) {  // models.cpp:123-128
  V p = q;
  if (std::abs(phi) < 1.0)
    for (auto& x : p) x = x / (1.0 - phi * phi);
  return p;
}

long poisson_draw(double lambda, Stream& s) {  // models.cpp:130-140
  const double u = s.uniform();
  double p = std::exp(-lambda), cdf = p;
  long k = 0;
  while (u > cdf && k < 100000) {
    ++k;
    p *= lambda / k;
    cdf += p;
  }
  return k;
}

V l63_drift(const auxmc_model_spec& s, const double* v) {
  return {s.lz_sigma * (v[1] - v[0]), v[0] * (s.lz_rho - v[2]) - v[1],
          v[0] * v[1] - s.lz_beta * v[2]};
}

V l96_drift(const auxmc_model_spec& s, const double* x, int d) {
  V f(d);
  for (int i = 0; i < d; ++i)
    f[i] = (x[(i + 1) % d] - x[(i + d - 2) % d]) * x[(i + d - 1) % d] - x[i] + s.l96_F;
  return f;
}

}  // namespace

extern "C" {

void auxmc_spec_default(auxmc_model_spec* s) {
  std::memset(s, 0, sizeof *s);
  s->kind = AUXMC_KIND_LGSSM;
  s->T = 50; s->dx = 2; s->dy = 1; s->grid = 3; s->data_seed = 1;
  s->sv_mu = -1.0; s->sv_phi = 0.9; s->sv_sig2 = 0.1; s->sv_rho = 0.25;
  s->lz_sigma = 10.0; s->lz_rho = 28.0; s->lz_beta = 8.0 / 3.0; s->lz_h = 0.01;
  s->lz_gamma = 2.0; s->lz_obs_var = 1.0;
  s->st_phi = 0.8; s->st_kappa2 = 1.0; s->st_tau2 = 0.3;
  s->g1_phi = 0.8; s->g1_q = 0.09; s->g1_m0 = 0.5; s->g1_p0 = 0.25;
  s->l96_F = 8.0; s->l96_h = 0.01; s->l96_gamma = 1.0; s->l96_obs_var = 1.0;
}

int auxmc_latent_dim(const auxmc_model_spec* s) { return s ? latent(*s) : -1; }
int auxmc_obs_dim(const auxmc_model_spec* s) { return s ? obsdim(*s) : -1; }

int auxmc_synth_mats(const auxmc_model_spec* s, double* m0, double* b, double* P0, double* F,
                     double* Q, double* H, double* R) {
  if (!s || s->kind != AUXMC_KIND_LGSSM) return AUXMC_E_CONFIG;
  if (int st = check_spec(*s)) return st;
  const Synth m = synth(*s);
  std::memcpy(m0, m.m0.data(), sizeof(double) * m.m0.size());
  std::memcpy(b, m.b.data(), sizeof(double) * m.b.size());
  std::memcpy(P0, m.P0.data(), sizeof(double) * m.P0.size());
  std::memcpy(F, m.F.data(), sizeof(double) * m.F.size());
  std::memcpy(Q, m.Q.data(), sizeof(double) * m.Q.size());
  std::memcpy(H, m.H.data(), sizeof(double) * m.H.size());
  std::memcpy(R, m.R.data(), sizeof(double) * m.R.size());
  return AUXMC_OK;
}

// make_target parameter arrays for every kind (models.cpp:240-336)
int auxmc_target_params(const auxmc_model_spec* s, double* m0, double* P0, double* F, double* b,
                        double* Q) {
  if (!s) return AUXMC_E_ARG;
  if (int st = check_spec(*s)) return st;
  const int dx = latent(*s);
  V vm0(dx, 0.0), vP0(static_cast<size_t>(dx) * dx, 0.0), vF(static_cast<size_t>(dx) * dx, 0.0),
      vb(dx, 0.0), vQ(static_cast<size_t>(dx) * dx, 0.0);
  switch (s->kind) {
    case AUXMC_KIND_LGSSM: {
      const Synth m = synth(*s);
      vm0 = m.m0; vP0 = m.P0; vF = m.F; vb = m.b; vQ = m.Q;
      break;
    }
    case AUXMC_KIND_STOCHVOL:
      vQ = stochvol_q(*s);
      for (int i = 0; i < dx; ++i) {
        vm0[i] = s->sv_mu;
        vF[i * dx + i] = s->sv_phi;
        vb[i] = (1.0 - s->sv_phi) * s->sv_mu;
      }
      vP0 = ar1_p0(s->sv_phi, vQ);
      break;
    case AUXMC_KIND_LORENZ63:
      vm0 = {1.0, 1.0, 25.0};
      for (int i = 0; i < 3; ++i) {
        vP0[i * 3 + i] = 1.0;
        vQ[i * 3 + i] = s->lz_h * s->lz_gamma * s->lz_gamma;
      }
      break;
    case AUXMC_KIND_LORENZ96:
      for (int i = 0; i < dx; ++i) {
        vm0[i] = s->l96_F;
        vP0[i * dx + i] = 1.0;
        vQ[i * dx + i] = s->l96_h * s->l96_gamma * s->l96_gamma;
      }
      vm0[0] += 0.01;
      break;
    case AUXMC_KIND_SPATIO:
      vQ = spatio_cov(*s);
      for (int i = 0; i < dx; ++i) vF[i * dx + i] = s->st_phi;
      vP0 = ar1_p0(s->st_phi, vQ);
      break;
    case AUXMC_KIND_GRID1D:
      vm0[0] = s->g1_m0;
      vP0[0] = s->g1_p0 * 1.0;
      vF[0] = s->g1_phi * 1.0;
      vQ[0] = s->g1_q * 1.0;
      break;
    default:
      return AUXMC_E_CONFIG;
  }
  std::memcpy(m0, vm0.data(), sizeof(double) * dx);
  std::memcpy(P0, vP0.data(), sizeof(double) * dx * dx);
  std::memcpy(F, vF.data(), sizeof(double) * dx * dx);
  std::memcpy(b, vb.data(), sizeof(double) * dx);
  std::memcpy(Q, vQ.data(), sizeof(double) * dx * dx);
  return AUXMC_OK;
}

int auxmc_simulate(const auxmc_model_spec* s, double* latent_out, double* data_out) {
  if (!s) return AUXMC_E_ARG;
  if (int st = check_spec(*s)) return st;
  const int dx = latent(*s), dy = obsdim(*s), T = s->T;
  const Stream root = Stream::seed(s->data_seed);
  V m0(dx, 0.0), p0l(static_cast<size_t>(dx) * dx, 0.0), ql(static_cast<size_t>(dx) * dx, 0.0);
  Synth sm;
  V rl;
  std::function<V(const double*)> mean;
  switch (s->kind) {
    case AUXMC_KIND_LGSSM:
      sm = synth(*s);
      m0 = sm.m0;
      p0l = cholesky(sm.P0, dx);
      ql = cholesky(sm.Q, dx);
      rl = cholesky(sm.R, dy);
      mean = [&](const double* x) {
        V o = matmul(sm.F, V(x, x + dx), dx, dx, 1);
        for (int i = 0; i < dx; ++i) o[i] += sm.b[i];
        return o;
      };
      break;
    case AUXMC_KIND_STOCHVOL: {
      for (auto& v : m0) v = s->sv_mu;
      const V q = stochvol_q(*s);
      p0l = cholesky(ar1_p0(s->sv_phi, q), dx);
      ql = cholesky(q, dx);
      mean = [&](const double* x) {
        V o(dx);
        for (int i = 0; i < dx; ++i) o[i] = s->sv_mu + s->sv_phi * (x[i] - s->sv_mu);
        return o;
      };
      break;
    }
    case AUXMC_KIND_LORENZ63:
      m0 = {1.0, 1.0, 25.0};
      for (int i = 0; i < 3; ++i) {
        p0l[i * 3 + i] = 1.0;
        ql[i * 3 + i] = std::sqrt(s->lz_h) * s->lz_gamma;
      }
      mean = [&](const double* x) {
        V f = l63_drift(*s, x), o(3);
        for (int i = 0; i < 3; ++i) o[i] = x[i] + s->lz_h * f[i];
        return o;
      };
      break;
    case AUXMC_KIND_LORENZ96:
      for (int i = 0; i < dx; ++i) {
        m0[i] = s->l96_F;
        p0l[i * dx + i] = 1.0;
        ql[i * dx + i] = std::sqrt(s->l96_h) * s->l96_gamma;
      }
      m0[0] += 0.01;
      mean = [&](const double* x) {
        V f = l96_drift(*s, x, dx), o(dx);
        for (int i = 0; i < dx; ++i) o[i] = x[i] + s->l96_h * f[i];
        return o;
      };
      break;
    case AUXMC_KIND_SPATIO: {
      const V q = spatio_cov(*s);
      p0l = cholesky(ar1_p0(s->st_phi, q), dx);
      ql = cholesky(q, dx);
      mean = [&](const double* x) {
        V o(dx);
        for (int i = 0; i < dx; ++i) o[i] = s->st_phi * x[i];
        return o;
      };
      break;
    }
    case AUXMC_KIND_GRID1D:
      m0[0] = s->g1_m0;
      p0l[0] = std::sqrt(s->g1_p0);
      ql[0] = std::sqrt(s->g1_q);
      mean = [&](const double* x) { return V{s->g1_phi * x[0]}; };
      break;
    default:
      return AUXMC_E_CONFIG;
  }
  for (int t = 0; t <= T; ++t) {
    Stream st = root.derive(AUXMC_L_SIMULATE, t);
    const V xi = st.normals(dx);
    V x(dx);
    if (t == 0) {
      const V v = matmul(p0l, xi, dx, dx, 1);
      for (int i = 0; i < dx; ++i) x[i] = m0[i] + v[i];
    } else {
      const V mu = mean(latent_out + static_cast<size_t>(t - 1) * dx);
      const V v = matmul(ql, xi, dx, dx, 1);
      for (int i = 0; i < dx; ++i) x[i] = mu[i] + v[i];
    }
    std::memcpy(latent_out + static_cast<size_t>(t) * dx, x.data(), sizeof(double) * dx);
    double* y = data_out + static_cast<size_t>(t) * dy;
    switch (s->kind) {
      case AUXMC_KIND_LGSSM: {
        const V hx = matmul(sm.H, x, dy, dx, 1);
        const V e = st.normals(dy);
        const V v = matmul(rl, e, dy, dy, 1);
        for (int i = 0; i < dy; ++i) y[i] = hx[i] + v[i];
        break;
      }
      case AUXMC_KIND_STOCHVOL:
        for (int j = 0; j < dy; ++j) y[j] = std::exp(x[j] / 2.0) * st.normal();
        break;
      case AUXMC_KIND_LORENZ63:
        y[0] = x[0] + std::sqrt(s->lz_obs_var) * st.normal();
        break;
      case AUXMC_KIND_LORENZ96:
        for (int k = 0; k < dy; ++k) y[k] = x[2 * k] + std::sqrt(s->l96_obs_var) * st.normal();
        break;
      case AUXMC_KIND_SPATIO:
        for (int j = 0; j < dy; ++j) y[j] = static_cast<double>(poisson_draw(std::exp(x[j]), st));
        break;
      default:
        break;
    }
  }
  return AUXMC_OK;
}

}  // extern "C"
