// Hessenberg + Francis double-shift QR eigenvalues for the Eigen shim (see Dense).
// TEST INFRASTRUCTURE; same algorithm as oracle/ao_core.c ao_spectral_radius.
namespace Eigen {
namespace shim {
inline double hqr_sgn(double a, double b) { return b >= 0.0 ? std::fabs(a) : -std::fabs(a); }
inline void hqr_eigenvalues(int n, std::vector<double>& hv, std::vector<double>& wro,
                            std::vector<double>& wio) {
  wro.assign(n, 0.0);
  wio.assign(n, 0.0);
  if (n == 0) return;
  std::vector<double> wr(n + 1, 0.0), wi(n + 1, 0.0);
  double* h = hv.data();
#define A1(i, j) h[((i)-1) * n + ((j)-1)]
#define fabs std::fabs
#define sqrt std::sqrt
#define sgn hqr_sgn
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
#undef A1
#undef fabs
#undef sqrt
#undef sgn
  for (int i = 0; i < n; ++i) {
    wro[i] = wr[i + 1];
    wio[i] = wi[i + 1];
  }
}
}  // namespace shim
}  // namespace Eigen
