/* ao_core.c — counter RNG, noise sources and dense Gaussian primitives.
 * TEST INFRASTRUCTURE (parity oracle); see auxmc_oracle.h. */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "auxmc_oracle.h"
#include "ao_internal.h"

/* ---- rng.hpp:35-42 splitmix64 finalizer ---- */
uint64_t ao_mix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}

#define AO_GOLDEN 0x9E3779B97F4A7C15ull

/* rng.hpp:47-49 */
uint64_t ao_word_at(uint64_t key, uint64_t i) { return ao_mix64(key + (i + 1) * AO_GOLDEN); }

/* rng.hpp:51-54: (w>>11 + 0.5) * 2^-53 */
double ao_to_unit_open(uint64_t w) { return ((double)(w >> 11) + 0.5) * 0x1.0p-53; }

/* rng.hpp:66-70 */
ao_stream ao_from_seed(uint64_t seed) {
  ao_stream s = {ao_mix64(seed + AO_GOLDEN), 0};
  return s;
}

ao_stream ao_from_key(uint64_t key) {
  ao_stream s = {key, 0};
  return s;
}

/* rng.hpp:73-80 */
ao_stream ao_derive(ao_stream s, uint64_t label, uint64_t index) {
  uint64_t k = s.key;
  k = ao_mix64(k ^ ao_mix64(label ^ 0xA0761D6478BD642Full));
  k = ao_mix64(k ^ ao_mix64(index ^ 0xE7037ED1A0B428DBull));
  ao_stream o = {k, 0};
  return o;
}

/* rng.hpp:85-88 */
double ao_next_uniform(ao_stream* s) {
  uint64_t c = s->counter++;
  return ao_to_unit_open(ao_word_at(s->key, 2 * c));
}

/* rng.hpp:90-95 Box-Muller, cosine branch */
double ao_next_normal(ao_stream* s) {
  uint64_t c = s->counter++;
  double u1 = ao_to_unit_open(ao_word_at(s->key, 2 * c));
  double u2 = ao_to_unit_open(ao_word_at(s->key, 2 * c + 1));
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586476925286766559 * u2);
}

/* rng.hpp:104-108 */
uint64_t ao_next_key(ao_stream* s) {
  uint64_t c = s->counter++;
  return ao_word_at(s->key, 2 * c);
}

/* rng.hpp:97-101 */
void ao_normal_vec(ao_stream* s, int d, double* out) {
  for (int i = 0; i < d; ++i) out[i] = ao_next_normal(s);
}

/* rng.hpp:128-161 */
void ao_noise_normal(ao_noise* n, uint64_t label, uint64_t index, int dim, double* out) {
  if (n->kind == 0) {
    ao_stream s = ao_derive(n->base, label, index);
    ao_normal_vec(&s, dim, out);
    return;
  }
  if (n->kind == 2) {
    for (int i = 0; i < dim; ++i) out[i] = 0.0;
    if (n->active >= n->cursor && n->active < n->cursor + dim) out[n->active - n->cursor] = 1.0;
    n->cursor += dim;
    return;
  }
  const double* src = NULL;
  if (label == AO_L_TERMINAL_DRAW) src = n->terminal;
  else if (label == AO_L_BACKWARD_NOISE && (long)index < n->n_backward)
    src = n->backward + (size_t)index * dim;
  else if (label == AO_L_DNC_BRIDGE && (long)index < n->n_bridge)
    src = n->bridge + (size_t)index * dim;
  for (int i = 0; i < dim; ++i) out[i] = src ? src[i] : 0.0;
}

/* ---------------- small dense helpers ---------------- */
void ao_matmul(int m, int k, int n, const double* a, const double* b, double* c) {
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < n; ++j) {
      double s = 0.0;
      for (int l = 0; l < k; ++l) s += a[i * k + l] * b[l * n + j];
      c[i * n + j] = s;
    }
}
/* c = a * b^T, a m×k, b n×k */
void ao_matmul_bt(int m, int k, int n, const double* a, const double* b, double* c) {
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < n; ++j) {
      double s = 0.0;
      for (int l = 0; l < k; ++l) s += a[i * k + l] * b[j * k + l];
      c[i * n + j] = s;
    }
}
/* c = a^T * b, a k×m, b k×n */
void ao_matmul_at(int m, int k, int n, const double* a, const double* b, double* c) {
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < n; ++j) {
      double s = 0.0;
      for (int l = 0; l < k; ++l) s += a[l * m + i] * b[l * n + j];
      c[i * n + j] = s;
    }
}
void ao_matvec(int m, int n, const double* a, const double* x, double* y) {
  for (int i = 0; i < m; ++i) {
    double s = 0.0;
    for (int j = 0; j < n; ++j) s += a[i * n + j] * x[j];
    y[i] = s;
  }
}
void ao_matvec_t(int m, int n, const double* a, const double* x, double* y) {
  /* y (n) = a^T x, a m×n */
  for (int j = 0; j < n; ++j) {
    double s = 0.0;
    for (int i = 0; i < m; ++i) s += a[i * n + j] * x[i];
    y[j] = s;
  }
}
void ao_transpose(int m, int n, const double* a, double* at) {
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < n; ++j) at[j * m + i] = a[i * n + j];
}
/* symm(X) = 0.5*(X + X^T), lgssm.cpp:14 */
void ao_symm(int n, double* a) {
  for (int i = 0; i < n; ++i)
    for (int j = i; j < n; ++j) {
      double v = 0.5 * (a[i * n + j] + a[j * n + i]);
      a[i * n + j] = v;
      a[j * n + i] = v;
    }
}
int ao_all_zero(int n, const double* a) {
  for (int i = 0; i < n; ++i)
    if (a[i] != 0.0) return 0;
  return 1;
}
void ao_eye(int n, double* a) {
  memset(a, 0, sizeof(double) * n * n);
  for (int i = 0; i < n; ++i) a[i * n + i] = 1.0;
}
/* out = a * p * a^T (association (a p) a^T), a m×n, p n×n */
void ao_sandwich(int m, int n, const double* a, const double* p, double* out, double* work) {
  ao_matmul(m, n, n, a, p, work);
  ao_matmul_bt(m, n, m, work, a, out);
}

/* ---------------- Cholesky (Eigen LLT semantics) ----------------
 * Unblocked lower Cholesky reading the lower triangle; fails iff a pivot
 * x <= 0 (so NaN pivots "succeed"), gauss.cpp:13-17 via Eigen LLT::info. */
int ao_llt(int n, const double* a, double* l) {
  memset(l, 0, sizeof(double) * n * n);
  for (int k = 0; k < n; ++k) {
    double x = a[k * n + k];
    for (int j = 0; j < k; ++j) x -= l[k * n + j] * l[k * n + j];
    if (x <= 0.0) return 0;
    x = sqrt(x);
    l[k * n + k] = x;
    for (int i = k + 1; i < n; ++i) {
      double s = a[i * n + k];
      for (int j = 0; j < k; ++j) s -= l[i * n + j] * l[k * n + j];
      l[i * n + k] = s / x;
    }
  }
  return 1;
}

/* gauss.cpp:20-24 */
static double jitter_scale(int n, const double* a) {
  double tr = 0.0;
  for (int i = 0; i < n; ++i) tr += a[i * n + i];
  double s = tr / (double)n;
  if (s <= 0.0) {
    double m = 0.0;
    for (int i = 0; i < n * n; ++i) m = fabs(a[i]) > m ? fabs(a[i]) : m;
    s = m;
  }
  return s;
}

/* gauss.cpp:26-35 */
int ao_factor_psd(int n, const double* a, double* l) {
  if (ao_llt(n, a, l)) return AO_OK;
  const double s = jitter_scale(n, a);
  double* aj = (double*)malloc(sizeof(double) * n * n);
  const double eps[2] = {1e-10, 1e-8};
  for (int e = 0; e < 2; ++e) {
    memcpy(aj, a, sizeof(double) * n * n);
    for (int i = 0; i < n; ++i) aj[i * n + i] += (eps[e] * s) * 1.0;
    if (ao_llt(n, aj, l)) {
      free(aj);
      return AO_OK;
    }
  }
  free(aj);
  return AO_E_FACTOR;
}

/* gauss.cpp:45-49 */
int ao_chol_psd(int n, const double* a, double* l) {
  if (n == 0) return AO_OK;
  if (ao_all_zero(n * n, a)) {
    memset(l, 0, sizeof(double) * n * n);
    return AO_OK;
  }
  return ao_factor_psd(n, a, l);
}

/* L L^T x = b (forward then back substitution), b,x n×nrhs row-major */
void ao_llt_solve(int n, const double* l, int nrhs, const double* b, double* x) {
  for (int r = 0; r < nrhs; ++r) {
    for (int i = 0; i < n; ++i) {
      double s = b[i * nrhs + r];
      for (int j = 0; j < i; ++j) s -= l[i * n + j] * x[j * nrhs + r];
      x[i * nrhs + r] = s / l[i * n + i];
    }
    for (int i = n - 1; i >= 0; --i) {
      double s = x[i * nrhs + r];
      for (int j = i + 1; j < n; ++j) s -= l[j * n + i] * x[j * nrhs + r];
      x[i * nrhs + r] = s / l[i * n + i];
    }
  }
}

/* gauss.cpp:89-91 */
int ao_solve_spd(int n, const double* s, int nrhs, const double* b, double* x) {
  double* l = (double*)malloc(sizeof(double) * n * n);
  int st = ao_factor_psd(n, s, l);
  if (st == AO_OK) ao_llt_solve(n, l, nrhs, b, x);
  free(l);
  return st;
}

/* gauss.cpp:51-57 with the Gaussian constructor's symmetrization (:39-43) */
double ao_log_pdf(int n, const double* x, const double* mean, const double* cov, int* status) {
  static const double kLog2Pi = 1.8378770664093454835606594728112;
  double* c = (double*)malloc(sizeof(double) * (2 * n * n + 2 * n));
  double* l = c + n * n;
  double* z = l + n * n;
  double* r = z + n;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) c[i * n + j] = (cov[i * n + j] + cov[j * n + i]) * 0.5;
  int st = ao_factor_psd(n, c, l);
  if (st != AO_OK) {
    if (status) *status = st;
    free(c);
    return NAN;
  }
  for (int i = 0; i < n; ++i) r[i] = x[i] - mean[i];
  for (int i = 0; i < n; ++i) {
    double s = r[i];
    for (int j = 0; j < i; ++j) s -= l[i * n + j] * z[j];
    z[i] = s / l[i * n + i];
  }
  double sq = 0.0, ld = 0.0;
  for (int i = 0; i < n; ++i) sq += z[i] * z[i];
  for (int i = 0; i < n; ++i) ld += log(l[i * n + i]);
  free(c);
  return -0.5 * (n * kLog2Pi + sq) - ld;
}

/* gauss.cpp:59-62 */
double ao_isotropic_log_pdf(int n, const double* resid, double var) {
  static const double kLog2Pi = 1.8378770664093454835606594728112;
  double sq = 0.0;
  for (int i = 0; i < n; ++i) sq += resid[i] * resid[i];
  return -0.5 * ((double)n * (kLog2Pi + log(var)) + sq / var);
}

/* Eigen PartialPivLU::solve: row-pivoted LU, pit.cpp:41-42 */
int ao_lu_solve(int n, const double* a, int nrhs, const double* b, double* x) {
  double* lu = (double*)malloc(sizeof(double) * n * n);
  int* perm = (int*)malloc(sizeof(int) * n);
  memcpy(lu, a, sizeof(double) * n * n);
  for (int i = 0; i < n; ++i) perm[i] = i;
  for (int k = 0; k < n; ++k) {
    int p = k;
    double best = fabs(lu[k * n + k]);
    for (int i = k + 1; i < n; ++i)
      if (fabs(lu[i * n + k]) > best) {
        best = fabs(lu[i * n + k]);
        p = i;
      }
    if (p != k) {
      for (int j = 0; j < n; ++j) {
        double t = lu[k * n + j];
        lu[k * n + j] = lu[p * n + j];
        lu[p * n + j] = t;
      }
      int t = perm[k];
      perm[k] = perm[p];
      perm[p] = t;
    }
    double piv = lu[k * n + k];
    if (piv != 0.0)
      for (int i = k + 1; i < n; ++i) {
        double f = lu[i * n + k] / piv;
        lu[i * n + k] = f;
        for (int j = k + 1; j < n; ++j) lu[i * n + j] -= f * lu[k * n + j];
      }
  }
  for (int r = 0; r < nrhs; ++r) {
    for (int i = 0; i < n; ++i) {
      double s = b[perm[i] * nrhs + r];
      for (int j = 0; j < i; ++j) s -= lu[i * n + j] * x[j * nrhs + r];
      x[i * nrhs + r] = s;
    }
    for (int i = n - 1; i >= 0; --i) {
      double s = x[i * nrhs + r];
      for (int j = i + 1; j < n; ++j) s -= lu[i * n + j] * x[j * nrhs + r];
      x[i * nrhs + r] = s / lu[i * n + i];
    }
  }
  free(lu);
  free(perm);
  return AO_OK;
}

/* ---------------- spectral radius (models.cpp:58 eigenvalues().cwiseAbs().maxCoeff())
 * Reduction to upper Hessenberg form by stabilized elementary similarity
 * transforms, then the Francis double-shift QR iteration on the Hessenberg
 * matrix (textbook algorithm; Eigen uses RealSchur, equal to rounding). */
#define A1(i, j) h[((i)-1) * n + ((j)-1)]
static double sgn(double a, double b) { return b >= 0.0 ? fabs(a) : -fabs(a); }

double ao_spectral_radius(int n, const double* a) {
  if (n == 0) return 0.0;
  double* h = (double*)malloc(sizeof(double) * n * n);
  double* wr = (double*)calloc(n + 1, sizeof(double));
  double* wi = (double*)calloc(n + 1, sizeof(double));
  memcpy(h, a, sizeof(double) * n * n);
  /* Hessenberg reduction with pivoting */
  for (int m = 2; m < n; ++m) {
    double x = 0.0;
    int i = m;
    for (int j = m; j <= n; ++j)
      if (fabs(A1(j, m - 1)) > fabs(x)) {
        x = A1(j, m - 1);
        i = j;
      }
    if (i != m) {
      for (int j = m - 1; j <= n; ++j) {
        double t = A1(i, j);
        A1(i, j) = A1(m, j);
        A1(m, j) = t;
      }
      for (int j = 1; j <= n; ++j) {
        double t = A1(j, i);
        A1(j, i) = A1(j, m);
        A1(j, m) = t;
      }
    }
    if (x != 0.0) {
      for (i = m + 1; i <= n; ++i) {
        double y = A1(i, m - 1);
        if (y != 0.0) {
          y /= x;
          A1(i, m - 1) = y;
          for (int j = m; j <= n; ++j) A1(i, j) -= y * A1(m, j);
          for (int j = 1; j <= n; ++j) A1(j, m) += y * A1(j, i);
        }
      }
    }
  }
  for (int i = 3; i <= n; ++i)
    for (int j = 1; j <= i - 2; ++j) A1(i, j) = 0.0;
  /* shifted QR */
  double anorm = 0.0;
  for (int i = 1; i <= n; ++i)
    for (int j = (i - 1 > 1 ? i - 1 : 1); j <= n; ++j) anorm += fabs(A1(i, j));
  int nn = n, l = 1;
  double t = 0.0, p = 0, q = 0, r = 0, s, u, v, w, x, y, z;
  while (nn >= 1) {
    int its = 0;
    do {
      for (l = nn; l >= 2; l--) {
        s = fabs(A1(l - 1, l - 1)) + fabs(A1(l, l));
        if (s == 0.0) s = anorm;
        if (fabs(A1(l, l - 1)) + s == s) {
          A1(l, l - 1) = 0.0;
          break;
        }
      }
      x = A1(nn, nn);
      if (l == nn) {
        wr[nn] = x + t;
        wi[nn--] = 0.0;
      } else {
        y = A1(nn - 1, nn - 1);
        w = A1(nn, nn - 1) * A1(nn - 1, nn);
        if (l == nn - 1) {
          p = 0.5 * (y - x);
          q = p * p + w;
          z = sqrt(fabs(q));
          x += t;
          if (q >= 0.0) {
            z = p + sgn(z, p);
            wr[nn - 1] = wr[nn] = x + z;
            if (z != 0.0) wr[nn] = x - w / z;
            wi[nn - 1] = wi[nn] = 0.0;
          } else {
            wr[nn - 1] = wr[nn] = x + p;
            wi[nn - 1] = -(wi[nn] = z);
          }
          nn -= 2;
        } else {
          int m;
          if (its == 60) break;
          if (its == 10 || its == 20) {
            t += x;
            for (int i = 1; i <= nn; i++) A1(i, i) -= x;
            s = fabs(A1(nn, nn - 1)) + fabs(A1(nn - 1, nn - 2));
            y = x = 0.75 * s;
            w = -0.4375 * s * s;
          }
          ++its;
          for (m = nn - 2; m >= l; m--) {
            z = A1(m, m);
            r = x - z;
            s = y - z;
            p = (r * s - w) / A1(m + 1, m) + A1(m, m + 1);
            q = A1(m + 1, m + 1) - z - r - s;
            r = A1(m + 2, m + 1);
            s = fabs(p) + fabs(q) + fabs(r);
            p /= s;
            q /= s;
            r /= s;
            if (m == l) break;
            u = fabs(A1(m, m - 1)) * (fabs(q) + fabs(r));
            v = fabs(p) * (fabs(A1(m - 1, m - 1)) + fabs(z) + fabs(A1(m + 1, m + 1)));
            if (u + v == v) break;
          }
          for (int i = m + 2; i <= nn; i++) {
            A1(i, i - 2) = 0.0;
            if (i != m + 2) A1(i, i - 3) = 0.0;
          }
          for (int k = m; k <= nn - 1; k++) {
            if (k != m) {
              p = A1(k, k - 1);
              q = A1(k + 1, k - 1);
              r = 0.0;
              if (k != nn - 1) r = A1(k + 2, k - 1);
              if ((x = fabs(p) + fabs(q) + fabs(r)) != 0.0) {
                p /= x;
                q /= x;
                r /= x;
              }
            }
            if ((s = sgn(sqrt(p * p + q * q + r * r), p)) != 0.0) {
              if (k == m) {
                if (l != m) A1(k, k - 1) = -A1(k, k - 1);
              } else
                A1(k, k - 1) = -s * x;
              p += s;
              x = p / s;
              y = q / s;
              z = r / s;
              q /= p;
              r /= p;
              for (int j = k; j <= nn; j++) {
                p = A1(k, j) + q * A1(k + 1, j);
                if (k != nn - 1) {
                  p += r * A1(k + 2, j);
                  A1(k + 2, j) -= p * z;
                }
                A1(k + 1, j) -= p * y;
                A1(k, j) -= p * x;
              }
              int mmin = nn < k + 3 ? nn : k + 3;
              for (int i = l; i <= mmin; i++) {
                p = x * A1(i, k) + y * A1(i, k + 1);
                if (k != nn - 1) {
                  p += z * A1(i, k + 2);
                  A1(i, k + 2) -= p * r;
                }
                A1(i, k + 1) -= p * q;
                A1(i, k) -= p;
              }
            }
          }
        }
      }
    } while (l < nn - 1);
  }
  double rad = 0.0;
  for (int i = 1; i <= n; ++i) {
    double m = hypot(wr[i], wi[i]);
    if (m > rad) rad = m;
  }
  free(h);
  free(wr);
  free(wi);
  return rad;
}
#undef A1
