/* ao_pit.c — parallel-in-time elements, Sklansky scans, prefix / dnc samplers
 * and the scan-based filter; restates proj/src/pit.cpp and include/auxmc/scan.hpp.
 * TEST INFRASTRUCTURE (parity oracle); see auxmc_oracle.h. */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "auxmc_oracle.h"
#include "ao_internal.h"

/* affine element: G (d×d), c (d), cov (d×d) stored contiguously */
#define EL_SZ(d) (2 * (d) * (d) + (d))
#define EL_G(e, d) (e)
#define EL_C(e, d) ((e) + (d) * (d))
#define EL_COV(e, d) ((e) + (d) * (d) + (d))

/* pit.cpp:23-30: out = a ∘ b (apply b first, then a) */
static void compose(int d, const double* a, const double* b, double* out, double* work) {
  double* tmp = work;           /* d*d */
  double* w2 = work + d * d;    /* d*d */
  ao_matmul(d, d, d, EL_G(a, d), EL_G(b, d), EL_G(out, d));
  ao_matvec(d, d, EL_G(a, d), EL_C(b, d), tmp);
  for (int i = 0; i < d; ++i) EL_C(out, d)[i] = tmp[i] + EL_C(a, d)[i];
  ao_sandwich(d, d, EL_G(a, d), EL_COV(b, d), tmp, w2);
  for (int i = 0; i < d * d; ++i) EL_COV(out, d)[i] = tmp[i] + EL_COV(a, d)[i];
  ao_symm(d, EL_COV(out, d));
}

/* scan.hpp:22-41 Sklansky fan with op(earlier, later); `flip` realizes
 * suffix_scan's flipped operator on the reversed array (scan.hpp:46-53). */
typedef void (*scan_op)(int d, const double* x, const double* y, double* out, double* work);

static void sklansky(int d, double* a, long n, size_t esz, scan_op op, int flip,
                     int* critical_path, long* applications) {
  int* depth = (int*)calloc(n > 0 ? n : 1, sizeof(int));
  double* out = (double*)malloc(sizeof(double) * esz);
  double* work = (double*)malloc(sizeof(double) * (8 * d * d + 8 * d + 64));
  long apps = 0;
  for (long stride = 1; stride < n; stride <<= 1) {
    for (long j = 0; j < n; ++j) {
      if ((j & stride) == 0) continue;
      const long pivot = (j & ~(stride - 1)) - 1;
      if (flip)
        op(d, a + j * esz, a + pivot * esz, out, work);
      else
        op(d, a + pivot * esz, a + j * esz, out, work);
      memcpy(a + j * esz, out, sizeof(double) * esz);
      depth[j] = (depth[pivot] > depth[j] ? depth[pivot] : depth[j]) + 1;
      ++apps;
    }
  }
  int cp = 0;
  for (long j = 0; j < n; ++j) cp = depth[j] > cp ? depth[j] : cp;
  if (critical_path) *critical_path = cp;
  if (applications) *applications = apps;
  free(depth);
  free(out);
  free(work);
}

static void reverse_elems(double* a, long n, size_t esz) {
  double* tmp = (double*)malloc(sizeof(double) * esz);
  for (long i = 0, j = n - 1; i < j; ++i, --j) {
    memcpy(tmp, a + i * esz, sizeof(double) * esz);
    memcpy(a + i * esz, a + j * esz, sizeof(double) * esz);
    memcpy(a + j * esz, tmp, sizeof(double) * esz);
  }
  free(tmp);
}

/* pit.cpp:53-62 */
static int build_backward_elements(const ao_lgssm* m, const ao_filter* fr, double* el) {
  const int d = m->dx;
  for (int t = 0; t < m->T; ++t) {
    double* e = el + (size_t)t * EL_SZ(d);
    int st = ao_backward_step(m, fr, t, EL_G(e, d), EL_C(e, d), EL_COV(e, d));
    if (st != AO_OK) return st;
  }
  return AO_OK;
}

/* pit.cpp:64-76 */
static int realize_noise(int d, double* el, long n, ao_noise* noise) {
  double* l = (double*)malloc(sizeof(double) * (d * d + 2 * d));
  double* xi = l + d * d;
  double* v = xi + d;
  int st = AO_OK;
  for (long t = 0; t < n; ++t) {
    double* e = el + t * EL_SZ(d);
    if (!ao_all_zero(d * d, EL_COV(e, d))) {
      st = ao_chol_psd(d, EL_COV(e, d), l);
      if (st != AO_OK) break;
      ao_noise_normal(noise, AO_L_BACKWARD_NOISE, (uint64_t)t, d, xi);
      ao_matvec(d, d, l, xi, v);
      for (int i = 0; i < d; ++i) EL_C(e, d)[i] += v[i];
    }
    memset(EL_COV(e, d), 0, sizeof(double) * d * d);
  }
  free(l);
  return st;
}

static void terminal_draw(const ao_lgssm* m, const ao_filter* fr, ao_noise* noise, double* traj,
                          int* st) {
  const int T = m->T, d = m->dx;
  double* l = (double*)malloc(sizeof(double) * (d * d + 2 * d));
  double* xi = l + d * d;
  double* v = xi + d;
  *st = ao_chol_psd(d, fr->filt_cov + (size_t)T * d * d, l);
  if (*st == AO_OK) {
    ao_noise_normal(noise, AO_L_TERMINAL_DRAW, 0, d, xi);
    ao_matvec(d, d, l, xi, v);
    for (int i = 0; i < d; ++i) traj[(size_t)T * d + i] = fr->filt_mean[(size_t)T * d + i] + v[i];
  }
  free(l);
}

/* pit.cpp:78-106 */
int ao_prefix_sample(const ao_lgssm* m, const ao_filter* fr, ao_noise* noise, double* traj,
                     int* critical_path, long* applications) {
  const int T = m->T, d = m->dx;
  int st;
  terminal_draw(m, fr, noise, traj, &st);
  if (critical_path) *critical_path = 0;
  if (applications) *applications = 0;
  if (st != AO_OK || T == 0) return st;
  const size_t esz = EL_SZ(d);
  double* el = (double*)malloc(sizeof(double) * esz * T);
  st = build_backward_elements(m, fr, el);
  if (st == AO_OK) st = realize_noise(d, el, T, noise);
  if (st == AO_OK) {
    reverse_elems(el, T, esz);
    sklansky(d, el, T, esz, compose, 1, critical_path, applications);
    reverse_elems(el, T, esz);
    const double* xT = traj + (size_t)T * d;
    for (int t = 0; t < T; ++t) {
      const double* e = el + (size_t)t * esz;
      double* x = traj + (size_t)t * d;
      ao_matvec(d, d, EL_G(e, d), xT, x);
      for (int i = 0; i < d; ++i) x[i] += EL_C(e, d)[i];
    }
  }
  free(el);
  return st;
}

/* ---------------- filtering elements (pit.cpp:36-51, :117-188) ---------------- */
#define FE_SZ(d) (3 * (d) * (d) + 2 * (d))
#define FE_A(e, d) (e)
#define FE_B(e, d) ((e) + (d) * (d))
#define FE_C(e, d) ((e) + (d) * (d) + (d))
#define FE_ETA(e, d) ((e) + 2 * (d) * (d) + (d))
#define FE_J(e, d) ((e) + 2 * (d) * (d) + 2 * (d))

void ao_filter_combine(int d, const double* uA, const double* ub, const double* uC,
                       const double* ueta, const double* uJ, const double* vA,
                       const double* vb, const double* vC, const double* veta,
                       const double* vJ, double* oA, double* ob, double* oC,
                       double* oeta, double* oJ) {
  const int dd = d * d;
  double* w = (double*)malloc(sizeof(double) * (8 * dd + 4 * d));
  double* m1 = w;            /* I + uC vJ */
  double* m2 = m1 + dd;      /* I + vJ uC */
  double* s = m2 + dd;
  double* t1 = s + dd;
  double* t2 = t1 + dd;
  double* t3 = t2 + dd;
  double* vt = t3 + dd;
  double* v2 = vt + d;
  ao_matmul(d, d, d, uC, vJ, m1);
  ao_matmul(d, d, d, vJ, uC, m2);
  for (int i = 0; i < d; ++i) {
    m1[i * d + i] += 1.0;
    m2[i * d + i] += 1.0;
  }
  /* A = vA lu.solve(uA) */
  ao_lu_solve(d, m1, d, uA, s);
  ao_matmul(d, d, d, vA, s, oA);
  /* b = vA lu.solve(ub + uC veta) + vb */
  ao_matvec(d, d, uC, veta, vt);
  for (int i = 0; i < d; ++i) vt[i] += ub[i];
  ao_lu_solve(d, m1, 1, vt, v2);
  ao_matvec(d, d, vA, v2, vt);
  for (int i = 0; i < d; ++i) ob[i] = vt[i] + vb[i];
  /* C = symm(vA lu.solve(uC) vA^T + vC) */
  ao_lu_solve(d, m1, d, uC, s);
  ao_matmul(d, d, d, vA, s, t1);
  ao_matmul_bt(d, d, d, t1, vA, t2);
  for (int i = 0; i < dd; ++i) oC[i] = t2[i] + vC[i];
  ao_symm(d, oC);
  /* eta = uA^T lu_t.solve(veta - vJ ub) + ueta */
  ao_matvec(d, d, vJ, ub, vt);
  for (int i = 0; i < d; ++i) vt[i] = veta[i] - vt[i];
  ao_lu_solve(d, m2, 1, vt, v2);
  ao_matvec_t(d, d, uA, v2, vt);
  for (int i = 0; i < d; ++i) oeta[i] = vt[i] + ueta[i];
  /* J = symm(uA^T lu_t.solve(vJ) uA + uJ) */
  ao_lu_solve(d, m2, d, vJ, s);
  ao_matmul_at(d, d, d, uA, s, t1);
  ao_matmul(d, d, d, t1, uA, t3);
  for (int i = 0; i < dd; ++i) oJ[i] = t3[i] + uJ[i];
  ao_symm(d, oJ);
  free(w);
}

static void combine_op(int d, const double* u, const double* v, double* out, double* work) {
  (void)work;
  ao_filter_combine(d, FE_A(u, d), FE_B(u, d), FE_C(u, d), FE_ETA(u, d), FE_J(u, d),
                    FE_A(v, d), FE_B(v, d), FE_C(v, d), FE_ETA(v, d), FE_J(v, d),
                    FE_A(out, d), FE_B(out, d), FE_C(out, d), FE_ETA(out, d), FE_J(out, d));
}

int ao_parallel_filter(const ao_lgssm* m, const double* obs, ao_filter* fr, int* critical_path,
                       long* applications) {
  const int T = m->T, dx = m->dx, dy = m->dy;
  const int W = dx > dy ? dx : dy;
  const size_t esz = FE_SZ(dx);
  double* el = (double*)calloc(esz * (T + 1), sizeof(double));
  double* w = (double*)malloc(sizeof(double) * (12 * W * W + 6 * W));
  double* eye = w;
  double* s = eye + W * W;
  double* hq = s + W * W;
  double* x1 = hq + W * W;    /* S^{-1} H q (dy×dx) */
  double* x2 = x1 + W * W;    /* S^{-1} H (dy×dx) */
  double* a = x2 + W * W;
  double* t1 = a + W * W;
  double* t2 = t1 + W * W;
  double* work = t2 + W * W;
  double* hsT = work + W * W;  /* hs = x2^T (dx×dy) */
  double* innov = hsT + W * W;
  double* v = innov + W;
  double* v2 = v + W;
  int st = AO_OK;
  ao_eye(dx, eye);
  for (int t = 0; t <= T && st == AO_OK; ++t) {
    const double* f = t == 0 ? eye : AO_F(m, t - 1);
    const double* bdyn = t == 0 ? m->m0 : AO_B(m, t - 1);
    const double* q = t == 0 ? m->P0 : AO_Q(m, t - 1);
    double* e = el + (size_t)t * esz;
    if (AO_OBSERVED(m, t)) {
      const double* h = AO_H(m, t);
      const double* R = AO_R(m, t);
      const double* c = AO_C(m, t);
      const double* y = obs + (size_t)t * dy;
      ao_matvec(dy, dx, h, bdyn, v);
      for (int i = 0; i < dy; ++i) innov[i] = (y[i] - v[i]) - c[i];
      ao_sandwich(dy, dx, h, q, s, work);
      for (int i = 0; i < dy * dy; ++i) s[i] += R[i];
      ao_symm(dy, s);
      ao_matmul(dy, dx, dx, h, q, hq);
      st = ao_solve_spd(dy, s, dx, hq, x1); /* gain = x1^T */
      if (st != AO_OK) break;
      st = ao_solve_spd(dy, s, dx, h, x2);  /* hs = x2^T */
      if (st != AO_OK) break;
      ao_transpose(dy, dx, x2, hsT);
      /* a = I - gain h */
      ao_matmul_at(dx, dy, dx, x1, h, a);
      for (int i = 0; i < dx * dx; ++i) a[i] = -a[i];
      for (int i = 0; i < dx; ++i) a[i * dx + i] += 1.0;
      ao_matmul(dx, dx, dx, a, f, FE_A(e, dx));
      ao_matvec_t(dy, dx, x1, innov, v);
      for (int i = 0; i < dx; ++i) FE_B(e, dx)[i] = bdyn[i] + v[i];
      ao_sandwich(dx, dx, a, q, t1, work);
      ao_matmul_at(dx, dy, dy, x1, R, t2); /* gain R */
      ao_matmul(dx, dy, dx, t2, x1, work);  /* gain R gain^T */
      for (int i = 0; i < dx * dx; ++i) FE_C(e, dx)[i] = t1[i] + work[i];
      ao_symm(dx, FE_C(e, dx));
      ao_matvec(dx, dy, hsT, innov, v);      /* hs innov */
      ao_matvec_t(dx, dx, f, v, FE_ETA(e, dx));
      /* J = symm(((f^T hs) h) f) */
      ao_matmul_at(dx, dx, dy, f, hsT, t1);  /* f^T hs: dx×dy */
      ao_matmul(dx, dy, dx, t1, h, t2);
      ao_matmul(dx, dx, dx, t2, f, FE_J(e, dx));
      ao_symm(dx, FE_J(e, dx));
    } else {
      memcpy(FE_A(e, dx), f, sizeof(double) * dx * dx);
      memcpy(FE_B(e, dx), bdyn, sizeof(double) * dx);
      memcpy(FE_C(e, dx), q, sizeof(double) * dx * dx);
      memset(FE_ETA(e, dx), 0, sizeof(double) * dx);
      memset(FE_J(e, dx), 0, sizeof(double) * dx * dx);
    }
    if (t == 0) memset(FE_A(e, dx), 0, sizeof(double) * dx * dx);
  }
  if (st == AO_OK) {
    sklansky(dx, el, T + 1, esz, combine_op, 0, critical_path, applications);
    fr->log_marginal = 0.0;
    for (int t = 0; t <= T && st == AO_OK; ++t) {
      const double* e = el + (size_t)t * esz;
      memcpy(fr->filt_mean + (size_t)t * dx, FE_B(e, dx), sizeof(double) * dx);
      memcpy(fr->filt_cov + (size_t)t * dx * dx, FE_C(e, dx), sizeof(double) * dx * dx);
      double* pm = fr->pred_mean + (size_t)t * dx;
      double* pc = fr->pred_cov + (size_t)t * dx * dx;
      if (t == 0) {
        memcpy(pm, m->m0, sizeof(double) * dx);
        memcpy(pc, m->P0, sizeof(double) * dx * dx);
      } else {
        ao_matvec(dx, dx, AO_F(m, t - 1), fr->filt_mean + (size_t)(t - 1) * dx, pm);
        const double* b = AO_B(m, t - 1);
        for (int i = 0; i < dx; ++i) pm[i] += b[i];
        ao_sandwich(dx, dx, AO_F(m, t - 1), fr->filt_cov + (size_t)(t - 1) * dx * dx, pc, work);
        const double* Q = AO_Q(m, t - 1);
        for (int i = 0; i < dx * dx; ++i) pc[i] += Q[i];
        ao_symm(dx, pc);
      }
      if (AO_OBSERVED(m, t)) {
        const double* h = AO_H(m, t);
        ao_sandwich(dy, dx, h, pc, s, work);
        const double* R = AO_R(m, t);
        for (int i = 0; i < dy * dy; ++i) s[i] += R[i];
        ao_symm(dy, s);
        ao_matvec(dy, dx, h, pm, v2);
        const double* c = AO_C(m, t);
        for (int i = 0; i < dy; ++i) v2[i] += c[i];
        fr->log_marginal += ao_log_pdf(dy, obs + (size_t)t * dy, v2, s, &st);
      }
    }
  }
  free(w);
  free(el);
  return st;
}

/* ---------------- divide and conquer (pit.cpp:192-295) ---------------- */
typedef struct { int l, m, r; uint64_t id; int left, right; } dnc_node;

int ao_dnc_sample(const ao_lgssm* m, const ao_filter* fr, ao_noise* noise, double* traj) {
  const int T = m->T, d = m->dx;
  int st;
  terminal_draw(m, fr, noise, traj, &st);
  if (st != AO_OK || T == 0) return st;
  const size_t esz = EL_SZ(d);
  double* base = (double*)malloc(sizeof(double) * esz * T);
  st = build_backward_elements(m, fr, base);
  if (st != AO_OK) {
    free(base);
    return st;
  }
  /* fixed BFS segment tree over [0, T] */
  long cap = 4L * T + 8;
  dnc_node* nodes = (dnc_node*)malloc(sizeof(dnc_node) * cap);
  long* lev_lo = (long*)malloc(sizeof(long) * 80);
  long* lev_hi = (long*)malloc(sizeof(long) * 80);
  long nn = 0;
  int nlev = 0;
  nodes[nn++] = (dnc_node){0, -1, T, 1, -1, -1};
  lev_lo[0] = 0;
  lev_hi[0] = 1;
  nlev = 1;
  for (;;) {
    long lo = lev_lo[nlev - 1], hi = lev_hi[nlev - 1];
    long begin = nn;
    for (long i = lo; i < hi; ++i) {
      dnc_node n = nodes[i];
      if (n.r - n.l < 2) continue;
      const int mid = (n.l + n.r) / 2;
      nodes[i].m = mid;
      nodes[i].left = (int)nn;
      nodes[nn++] = (dnc_node){n.l, -1, mid, 2 * n.id, -1, -1};
      nodes[i].right = (int)nn;
      nodes[nn++] = (dnc_node){mid, -1, n.r, 2 * n.id + 1, -1, -1};
    }
    if (begin == nn) break;
    lev_lo[nlev] = begin;
    lev_hi[nlev] = nn;
    ++nlev;
  }
  double* elem = (double*)malloc(sizeof(double) * esz * nn);
  double* work = (double*)malloc(sizeof(double) * (16 * d * d + 16 * d));
  for (int lev = nlev - 1; lev >= 0; --lev)
    for (long i = lev_lo[lev]; i < lev_hi[lev]; ++i) {
      const dnc_node* n = &nodes[i];
      if (n->left < 0)
        memcpy(elem + i * esz, base + (size_t)n->l * esz, sizeof(double) * esz);
      else
        compose(d, elem + (size_t)n->left * esz, elem + (size_t)n->right * esz, elem + i * esz,
                work);
    }
  /* serial noise draws: root conditional, then midpoints level by level */
  double* root_xi = (double*)malloc(sizeof(double) * d);
  double* mid_xi = (double*)calloc((size_t)nn * d, sizeof(double));
  ao_noise_normal(noise, AO_L_BACKWARD_NOISE, 0, d, root_xi);
  for (int lev = 0; lev < nlev; ++lev)
    for (long i = lev_lo[lev]; i < lev_hi[lev]; ++i)
      if (nodes[i].left >= 0) ao_noise_normal(noise, AO_L_DNC_BRIDGE, nodes[i].id, d, mid_xi + i * d);
  double* l = work;
  double* v = l + d * d;
  double* v2 = v + d;
  double* mu = v2 + d;
  double* cross = mu + d;
  double* s = cross + d * d;
  double* gain = s + d * d;
  double* a = gain + d * d;
  double* cov = a + d * d;
  double* t1 = cov + d * d;
  double* w2 = t1 + d * d;
  double* crossT = w2 + d * d;
  double* sol = crossT + d * d;
  /* root: x_0 | x_T */
  {
    const double* e = elem;
    st = ao_chol_psd(d, EL_COV(e, d), l);
    if (st == AO_OK) {
      ao_matvec(d, d, l, root_xi, v);
      for (int i = 0; i < d; ++i) v[i] += EL_C(e, d)[i];
      ao_matvec(d, d, EL_G(e, d), traj + (size_t)T * d, v2);
      for (int i = 0; i < d; ++i) traj[i] = v2[i] + v[i];
    }
  }
  for (int lev = 0; lev < nlev && st == AO_OK; ++lev)
    for (long i = lev_lo[lev]; i < lev_hi[lev] && st == AO_OK; ++i) {
      const dnc_node* n = &nodes[i];
      if (n->left < 0) continue;
      const double* elm = elem + (size_t)n->left * esz;
      const double* emr = elem + (size_t)n->right * esz;
      const double* xl = traj + (size_t)n->l * d;
      const double* xr = traj + (size_t)n->r * d;
      ao_matvec(d, d, EL_G(emr, d), xr, mu);
      for (int k = 0; k < d; ++k) mu[k] += EL_C(emr, d)[k];
      ao_matmul_bt(d, d, d, EL_COV(emr, d), EL_G(elm, d), cross);
      if (ao_all_zero(d * d, cross)) {
        memset(gain, 0, sizeof(double) * d * d);
      } else {
        ao_sandwich(d, d, EL_G(elm, d), EL_COV(emr, d), s, w2);
        for (int k = 0; k < d * d; ++k) s[k] += EL_COV(elm, d)[k];
        ao_symm(d, s);
        ao_transpose(d, d, cross, crossT);
        st = ao_solve_spd(d, s, d, crossT, sol);
        if (st != AO_OK) break;
        ao_transpose(d, d, sol, gain);
      }
      ao_matmul(d, d, d, gain, EL_G(elm, d), a);
      for (int k = 0; k < d * d; ++k) a[k] = -a[k];
      for (int k = 0; k < d; ++k) a[k * d + k] += 1.0;
      ao_sandwich(d, d, a, EL_COV(emr, d), cov, w2);
      ao_sandwich(d, d, gain, EL_COV(elm, d), t1, w2);
      for (int k = 0; k < d * d; ++k) cov[k] += t1[k];
      ao_symm(d, cov);
      /* mean = mu + gain (x_l - G_lm mu - c_lm) */
      ao_matvec(d, d, EL_G(elm, d), mu, v);
      for (int k = 0; k < d; ++k) v[k] = (xl[k] - v[k]) - EL_C(elm, d)[k];
      ao_matvec(d, d, gain, v, v2);
      st = ao_chol_psd(d, cov, l);
      if (st != AO_OK) break;
      ao_matvec(d, d, l, mid_xi + i * d, v);
      double* xm = traj + (size_t)n->m * d;
      for (int k = 0; k < d; ++k) xm[k] = (mu[k] + v2[k]) + v[k];
    }
  free(base);
  free(nodes);
  free(lev_lo);
  free(lev_hi);
  free(elem);
  free(work);
  free(root_xi);
  free(mid_xi);
  return st;
}

/* pit.cpp:303-332 */
int ao_extract_affine_law(int which, const ao_lgssm* m, const ao_filter* fr, double* mean,
                          double* cov) {
  const int n = (m->T + 1) * m->dx;
  ao_noise probe;
  memset(&probe, 0, sizeof probe);
  probe.kind = 2;
  probe.active = -1;
  probe.cursor = 0;
  int st;
#define RUN(out)                                                   \
  (which == 0   ? ao_backward_sample(m, fr, &probe, out)           \
   : which == 1 ? ao_prefix_sample(m, fr, &probe, out, NULL, NULL) \
                : ao_dnc_sample(m, fr, &probe, out))
  st = RUN(mean);
  if (st != AO_OK) return st;
  const int nd = probe.cursor;
  double* a = (double*)malloc(sizeof(double) * (size_t)n * (nd > 0 ? nd : 1));
  double* tr = (double*)malloc(sizeof(double) * n);
  for (int k = 0; k < nd && st == AO_OK; ++k) {
    probe.active = k;
    probe.cursor = 0;
    st = RUN(tr);
    for (int i = 0; i < n; ++i) a[(size_t)i * nd + k] = tr[i] - mean[i];
  }
#undef RUN
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      double s = 0.0;
      for (int k = 0; k < nd; ++k) s += a[(size_t)i * nd + k] * a[(size_t)j * nd + k];
      cov[(size_t)i * n + j] = s;
    }
  ao_symm(n, cov);
  free(a);
  free(tr);
  return st;
}
