// dnc.cu — pit::dnc_sample (pit.cpp:192-301) on B200.
//
// The reference builds a breadth-first segment tree over [0, T] (split at
// floor((l+r)/2) while r-l >= 2, heap ids 1, 2h, 2h+1; pit.cpp:214-234).  The
// tree depends only on T, so here nodes are addressed directly by heap id: the
// interval of node h follows from the bits of h, and node arrays are indexed
// by h (no host-built tree).  Levels run deepest-first for the bottom-up
// element composition (pit.cpp:237-245) and root-first for the Gaussian bridges
// (pit.cpp:265-293).  Bridge gains and factors depend only on the elements, so
// with a shared filter result they are computed once and reused by every chain.
#include "common.cuh"
#include "dense.cuh"
#include "rng.cuh"

namespace auxmc_gpu {


__host__ __device__ inline int dnc_depth(int T) {
  int depth = 0;
  long long cap = 1;
  while (cap < T) {
    cap <<= 1;
    ++depth;
  }
  return depth;
}

// Interval of heap node h; returns false if the node does not exist.
__device__ __forceinline__ bool dnc_interval(uint64_t h, int T, int& l, int& r) {
  int depth = 63 - __clzll((long long)h);
  l = 0;
  r = T;
  for (int bit = depth - 1; bit >= 0; --bit) {
    if (r - l < 2) return false;
    const int m = (l + r) / 2;
    if ((h >> bit) & 1ull) l = m;
    else r = m;
  }
  return true;
}

// Bottom-up: elem[h] = leaf ? base[l] : elem[2h] ∘ elem[2h+1] (pit.cpp:23-30).
template <bool BLOCK>
__global__ void k_dnc_compose(int T, int d, int level, int Bfr, const double* __restrict__ base,
                              double* nodes, long long n_heap) {
  extern __shared__ double smem[];
  const int dd = d * d, ES = (2 * dd + d + 1) & ~1;
  Grp g = BLOCK ? block_group() : warp_group();
  const int gid = BLOCK ? 0 : (threadIdx.x >> 5);
  const int gpb = BLOCK ? 1 : (blockDim.x >> 5);
  double* W = smem + (size_t)gid * 2 * dd;
  const long long width = 1LL << level;
  const long long n_items = width * Bfr;
  for (long long item = (long long)blockIdx.x * gpb + gid; item < n_items;
       item += (long long)gridDim.x * gpb) {
    const int b = (int)(item / width);
    const uint64_t h = (uint64_t)width + (uint64_t)(item % width);
    int l, r;
    if (!dnc_interval(h, T, l, r)) continue;
    double* out = nodes + ((size_t)b * n_heap + h) * ES;
    if (r - l < 2) {
      const double* src = base + ((size_t)b * T + l) * ES;
      g_copy(g, 2 * dd + d, src, out);
      g.sync();
      continue;
    }
    const double* a = nodes + ((size_t)b * n_heap + 2 * h) * ES;
    const double* bb = nodes + ((size_t)b * n_heap + 2 * h + 1) * ES;
    g_mm(g, d, d, d, a, bb, out);                         // G = a.G b.G
    g_mv(g, d, d, a, bb + dd, out + dd, a + dd);          // c = a.G b.c + a.c
    g_mm(g, d, d, d, a, bb + dd + d, W);                  // a.G b.cov
    g.sync();
    g_mm_nt(g, d, d, d, W, a, out + dd + d, a + dd + d);  // (.) a.G^T + a.cov
    g.sync();
    g_symm(g, d, out + dd + d);
    g.sync();
  }
}

// Bridge parameters per internal node (pit.cpp:270-291): K (gain), L = chol(cov).
// Root (h = 1): L = chol_psd(root cov) (pit.cpp:259-263).
constexpr int kBridgeBuffers = 6;
template <bool BLOCK>
__global__ void k_dnc_bridge(int T, int d, int Bfr, const double* __restrict__ nodes,
                             long long n_heap, long long n_first, long long n_last,
                             double* params, int* status) {
  extern __shared__ double smem[];
  const int dd = d * d, ES = (2 * dd + d + 1) & ~1;
  Grp g = BLOCK ? block_group() : warp_group();
  const int gid = BLOCK ? 0 : (threadIdx.x >> 5);
  const int gpb = BLOCK ? 1 : (blockDim.x >> 5);
  const int per = kBridgeBuffers * dd + 4;
  double* sm = smem + (size_t)gid * per;
  // six d*d buffers rotate with the liveness of the step (same operation
  // sequence as with one buffer per quantity): B0 cross, then K; B1 s; B2 A, then
  // the output factor; B3 W; B4 the first factor, then cov; B5 factor scratch
  double* cross = sm;
  double* s = cross + dd;
  double* A = s + dd;
  double* W = A + dd;
  double* L = W + dd;
  double* scr = L + dd;
  // Buffer liveness (each alias is written only after its previous occupant's last read):
  //   B0 cross: read by the zero test and the cross^T copy into A  -> then K (written after
  //             the solve consumed A; cross is dead)
  //   B4 L (the factor of s): last read by g_llt_solve             -> then cov (written after)
  //   B2 A = cross^T / solve rhs, then I - K G_lm: last read forming W = A S_mr and cov
  //                                                                -> then Lc (chol of cov)
  // A retry inside g_factor_psd / g_chol_psd reads only its own input (s / cov) and writes
  // its output (L / Lc) and scr, none of which alias a live buffer at that point.
  double* K = cross;
  double* cov = L;
  double* Lc = A;
  double* red = scr + dd;
  int* flag = reinterpret_cast<int*>(red + 2);
  const long long width = n_last - n_first;
  const long long n_items = width * Bfr;
  for (long long item = (long long)blockIdx.x * gpb + gid; item < n_items;
       item += (long long)gridDim.x * gpb) {
    const int b = (int)(item / width);
    const uint64_t h = (uint64_t)(n_first + item % width);
    int l, r;
    if (!dnc_interval(h, T, l, r)) continue;
    double* out = params + ((size_t)b * n_heap + h) * 2 * dd;
    int st = 0;
    if (h == 1) {  // root factor lives in the unused heap slot 0
      st = g_chol_psd(g, d, nodes + ((size_t)b * n_heap + 1) * ES + dd + d, L, scr, flag, red);
      g_copy(g, dd, L, params + (size_t)b * n_heap * 2 * dd + dd);
      g.sync();
      if (st && g.lane == 0) atomicMax(status + b, st);
    }
    if (r - l < 2) continue;
    const double* elm = nodes + ((size_t)b * n_heap + 2 * h) * ES;
    const double* emr = nodes + ((size_t)b * n_heap + 2 * h + 1) * ES;
    const double* Glm = elm;
    const double* Slm = elm + dd + d;
    const double* Smr = emr + dd + d;
    g_mm_nt(g, d, d, d, Smr, Glm, cross);  // cov(x_m, x_l | x_r)
    g.sync();
    if (g_all_zero(g, dd, cross, flag)) {
      g_zero(g, dd, K);
      g.sync();
    } else {
      g_mm(g, d, d, d, Glm, Smr, W);
      g.sync();
      g_mm_nt(g, d, d, d, W, Glm, s, Slm);
      g.sync();
      g_symm(g, d, s);
      for (int i = g.lane; i < dd; i += g.size) A[i] = cross[(i % d) * d + i / d];  // cross^T
      g.sync();
      st = g_factor_psd(g, d, s, L, scr, flag, red);
      if (st) {  // FactorizationError (gauss.cpp:34): flag the chain, poison this bridge
        if (g.lane == 0) atomicMax(status + b, st);
        for (int i = g.lane; i < 2 * dd; i += g.size) out[i] = __longlong_as_double(0x7ff8000000000000ll);
        g.sync();
        continue;
      }
      g_llt_solve(g, d, L, d, A, scr);  // scr: inverted diagonal blocks (CTA, d >= 16)
      for (int i = g.lane; i < dd; i += g.size) K[i] = A[(i % d) * d + i / d];
      g.sync();
    }
    // A = I - K G_lm ; cov = symm(A S_mr A^T + K S_lm K^T)
    g_mm(g, d, d, d, K, Glm, A);
    g.sync();
    for (int i = g.lane; i < dd; i += g.size) A[i] = (i / d == i % d ? 1.0 : 0.0) - A[i];
    g.sync();
    g_mm(g, d, d, d, A, Smr, W);
    g.sync();
    g_mm_nt(g, d, d, d, W, A, cov);
    g.sync();
    g_mm(g, d, d, d, K, Slm, W);
    g.sync();
    g_mm_nt(g, d, d, d, W, K, s);
    g.sync();
    for (int i = g.lane; i < dd; i += g.size) cov[i] += s[i];
    g.sync();
    g_symm(g, d, cov);
    g.sync();
    st = g_chol_psd(g, d, cov, Lc, scr, flag, red);
    if (st && g.lane == 0) atomicMax(status + b, st);
    g_copy(g, dd, K, out);
    g_copy(g, dd, Lc, out + dd);
    g.sync();
  }
}

template <int D>
__device__ __forceinline__ void dnc_normals(const NoiseArgs& nz, int c, uint64_t label,
                                            uint64_t index, int T, double* xi) {
  if (nz.kind == AUXMC_NOISE_PREDRAWN) {
    const double* src = label == kDncBridge ? nz.bridge + ((size_t)c * nz.n_bridge + index) * D
                        : label == kTerminalDraw ? nz.terminal + (size_t)c * D
                                                 : nz.backward + ((size_t)c * T + index) * D;
#pragma unroll
    for (int i = 0; i < D; ++i) xi[i] = src[i];
  } else {
    const uint64_t k = derive(nz.keys[c], label, index);
#pragma unroll
    for (int i = 0; i < D; ++i) xi[i] = normal_at(k, (uint64_t)i);
  }
}

// x_T (pit.cpp:206-208) and x_0 | x_T through the root (pit.cpp:259-263).
template <int D>
__global__ void k_dnc_ends(int T, int B, int fr_shared, const double* __restrict__ term,
                           const double* __restrict__ nodes, const double* __restrict__ params,
                           long long n_heap, NoiseArgs nz, double* traj) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= B) return;
  constexpr int ES = (2 * D * D + D + 1) & ~1;
  constexpr int TS = (D * D + D + 1) & ~1;
  const int b = fr_shared ? 0 : c;
  const double* tm = term + (size_t)b * TS;
  double* out = traj + (size_t)c * (T + 1) * D;
  double xi[D], x[D], v[D];
  dnc_normals<D>(nz, c, kTerminalDraw, 0, T, xi);
  r_matvec<D>(tm + D, xi, x);
#pragma unroll
  for (int i = 0; i < D; ++i) {
    x[i] = tm[i] + x[i];
    out[(size_t)T * D + i] = x[i];
  }
  if (T == 0) return;
  const double* root = nodes + ((size_t)b * n_heap + 1) * ES;
  const double* Lr = params + (size_t)b * n_heap * 2 * D * D + D * D;
  dnc_normals<D>(nz, c, kBackwardNoise, 0, T, xi);
  r_matvec<D>(Lr, xi, v);
#pragma unroll
  for (int i = 0; i < D; ++i) v[i] = root[D * D + i] + v[i];  // shifted = c + L xi
  double gx[D];
  r_matvec<D>(root, x, gx);
#pragma unroll
  for (int i = 0; i < D; ++i) out[i] = gx[i] + v[i];
}

// One level of bridges: thread per (node, chain), chains fastest.
template <int D>
__global__ void k_dnc_level(int T, int B, int fr_shared, int level,
                            const double* __restrict__ nodes, const double* __restrict__ params,
                            long long n_heap, NoiseArgs nz, double* traj) {
  constexpr int ES = (2 * D * D + D + 1) & ~1;
  const long long width = 1LL << level;
  const long long n = width * B;
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(q % B);
    const uint64_t h = (uint64_t)width + (uint64_t)(q / B);
    int l, r;
    if (!dnc_interval(h, T, l, r) || r - l < 2) continue;
    const int m = (l + r) / 2;
    const int b = fr_shared ? 0 : c;
    const double* elm = nodes + ((size_t)b * n_heap + 2 * h) * ES;
    const double* emr = nodes + ((size_t)b * n_heap + 2 * h + 1) * ES;
    const double* K = params + ((size_t)b * n_heap + h) * 2 * D * D;
    const double* L = K + D * D;
    double* out = traj + (size_t)c * (T + 1) * D;
    double xl[D], xr[D], mu[D], v[D], w[D], xi[D];
#pragma unroll
    for (int i = 0; i < D; ++i) {
      xl[i] = out[(size_t)l * D + i];
      xr[i] = out[(size_t)r * D + i];
    }
    r_matvec<D>(emr, xr, mu);
#pragma unroll
    for (int i = 0; i < D; ++i) mu[i] += emr[D * D + i];
    r_matvec<D>(elm, mu, v);
#pragma unroll
    for (int i = 0; i < D; ++i) v[i] = (xl[i] - v[i]) - elm[D * D + i];
    r_matvec<D>(K, v, w);
    dnc_normals<D>(nz, c, kDncBridge, h, T, xi);
    double lx[D];
    r_matvec<D>(L, xi, lx);
#pragma unroll
    for (int i = 0; i < D; ++i) out[(size_t)m * D + i] = (mu[i] + w[i]) + lx[i];
  }
}

// Deep levels.  Each bridge is affine in its end states:
//   x_m = mu + K (x_l - G_l mu - c_l) + L xi,  mu = G_r x_r + c_r
//       = A x_r + K x_l + a + L xi,  A = (I - K G_l) G_r,  a = (I - K G_l) c_r - K c_l,
// with (A, a) chain-independent when the filter result is shared, precomputed
// once per node (k_dnc_affine).  Every node at level L0 roots a subtree of at
// most kDncSpan steps that needs only its two end states, so one CTA (thread =
// chain) stages the subtree's node parameters in shared memory once and runs all
// remaining levels with the chain's states in shared memory; each state is
// written to HBM once, contiguously per chain, and only the subtree ends are read.
constexpr int kDncSpan = 16;
constexpr int kDncSubThreads = 128;

template <int D>
constexpr int dnc_aff_stride() {  // A | K | a | L per node, 16-B aligned
  return (3 * D * D + D + 1) & ~1;
}
template <int D>
constexpr int dnc_lane_stride() {  // odd (in doubles): conflict-free per-thread rows
  return ((kDncSpan + 1) * D) | 1;
}

template <int D>
__global__ void k_dnc_affine(int T, int Bfr, const double* __restrict__ nodes,
                             const double* __restrict__ params, long long n_heap, long long h_lo,
                             double* aff) {
  constexpr int ES = (2 * D * D + D + 1) & ~1, AS = dnc_aff_stride<D>();
  const long long n = (n_heap - h_lo) * Bfr;
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < n;
       q += (long long)gridDim.x * blockDim.x) {
    const int b = (int)(q / (n_heap - h_lo));
    const uint64_t h = (uint64_t)(h_lo + q % (n_heap - h_lo));
    int l, r;
    if (!dnc_interval(h, T, l, r) || r - l < 2) continue;
    const double* elm = nodes + ((size_t)b * n_heap + 2 * h) * ES;
    const double* emr = nodes + ((size_t)b * n_heap + 2 * h + 1) * ES;
    const double* K = params + ((size_t)b * n_heap + h) * 2 * D * D;
    const double* L = K + D * D;
    double* o = aff + ((size_t)b * n_heap + h) * AS;
    double M[D * D];  // I - K G_l
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
      for (int j = 0; j < D; ++j) {
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < D; ++k) acc += K[i * D + k] * elm[k * D + j];
        M[i * D + j] = (i == j ? 1.0 : 0.0) - acc;
      }
#pragma unroll
    for (int i = 0; i < D; ++i) {
#pragma unroll
      for (int j = 0; j < D; ++j) {
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < D; ++k) acc += M[i * D + k] * emr[k * D + j];
        o[i * D + j] = acc;                 // A
        o[D * D + i * D + j] = K[i * D + j];  // K
        o[2 * D * D + D + i * D + j] = L[i * D + j];  // L
      }
      double acc = 0.0, acc2 = 0.0;
#pragma unroll
      for (int k = 0; k < D; ++k) {
        acc += M[i * D + k] * emr[D * D + k];
        acc2 += K[i * D + k] * elm[D * D + k];
      }
      o[2 * D * D + i] = acc - acc2;  // a
    }
  }
}

template <int D>
__device__ __forceinline__ void dnc_noise_vec(const NoiseArgs& nz, int c, uint64_t h, int T,
                                              double* xi) {
  if (nz.kind == AUXMC_NOISE_PREDRAWN) {
    const double* src = nz.bridge + ((size_t)c * nz.n_bridge + h) * D;
    if constexpr (D % 2 == 0) {
#pragma unroll
      for (int i = 0; i < D; i += 2) {
        const double2 v = *reinterpret_cast<const double2*>(src + i);
        xi[i] = v.x;
        xi[i + 1] = v.y;
      }
    } else {
#pragma unroll
      for (int i = 0; i < D; ++i) xi[i] = src[i];
    }
  } else {
    dnc_normals<D>(nz, c, kDncBridge, h, T, xi);
  }
}

template <int D>
__global__ void __launch_bounds__(kDncSubThreads)
    k_dnc_subtree(int T, int B, int fr_shared, int L0, int depth, const double* __restrict__ aff,
                  long long n_heap, NoiseArgs nz, double* traj) {
  extern __shared__ __align__(16) double smx[];
  constexpr int AS = dnc_aff_stride<D>(), LSTR = dnc_lane_stride<D>();
  double* pn = smx;  // kDncSpan node parameter blocks, indexed by local heap id
  int* lrm = reinterpret_cast<int*>(smx + kDncSpan * AS);  // [kDncSpan] (l, r) or l = -1
  double* xs = smx + kDncSpan * AS + kDncSpan + (size_t)threadIdx.x * LSTR;
  const long long width = 1LL << L0;
  const int cgroups = (B + kDncSubThreads - 1) / kDncSubThreads;
  const long long n_items = width * cgroups;
  const int n_local = 1 << (depth - L0);  // local ids 1 .. n_local-1, level order
  for (long long q = blockIdx.x; q < n_items; q += gridDim.x) {
    const int c = (int)(q % cgroups) * kDncSubThreads + threadIdx.x;
    const bool live = c < B;
    const uint64_t h0 = (uint64_t)width + (uint64_t)(q / cgroups);
    int l0, r0;
    if (!dnc_interval(h0, T, l0, r0) || r0 - l0 < 2) continue;  // CTA-uniform
    const int fb = fr_shared ? 0 : (live ? c : 0);
    __syncthreads();
    for (int lid = 1 + threadIdx.x; lid < n_local; lid += blockDim.x) {
      const int lev = 31 - __clz(lid);
      const uint64_t h = (h0 << lev) + (uint64_t)(lid - (1 << lev));
      int l, r;
      const bool ok = dnc_interval(h, T, l, r) && r - l >= 2;
      lrm[2 * lid] = ok ? l : -1;
      lrm[2 * lid + 1] = r;
    }
    if (fr_shared)
      for (int e = threadIdx.x; e < (n_local - 1) * AS; e += blockDim.x) {
        const int lid = 1 + e / AS, o = e % AS;
        const int lev = 31 - __clz(lid);
        const uint64_t h = (h0 << lev) + (uint64_t)(lid - (1 << lev));
        pn[lid * AS + o] = h < (uint64_t)n_heap ? aff[(size_t)h * AS + o] : 0.0;
      }
    __syncthreads();
    if (!live) continue;
    double* out = traj + (size_t)c * (T + 1) * D;
#pragma unroll
    for (int i = 0; i < D; ++i) {
      xs[i] = out[(size_t)l0 * D + i];
      xs[(r0 - l0) * D + i] = out[(size_t)r0 * D + i];
    }
    auto hid = [&](int lid) {
      const int lev = 31 - __clz(lid);
      return (h0 << lev) + (uint64_t)(lid - (1 << lev));
    };
    double xin[D];  // noise of the next node, loaded one node ahead
    dnc_noise_vec<D>(nz, c, hid(1), T, xin);
    for (int lid = 1; lid < n_local; ++lid) {
      double xi[D];
#pragma unroll
      for (int j = 0; j < D; ++j) xi[j] = xin[j];
      if (lid + 1 < n_local) dnc_noise_vec<D>(nz, c, hid(lid + 1), T, xin);
      const int l = lrm[2 * lid], r = lrm[2 * lid + 1];
      if (l < 0) continue;
      const int m = (l + r) / 2;
      const uint64_t h = hid(lid);
      const double* P = fr_shared ? pn + lid * AS : aff + ((size_t)fb * n_heap + h) * AS;
      double xl[D], xr[D];
#pragma unroll
      for (int j = 0; j < D; ++j) {
        xl[j] = xs[(l - l0) * D + j];
        xr[j] = xs[(r - l0) * D + j];
      }
#pragma unroll
      for (int j = 0; j < D; ++j) {
        double u = 0.0, v = 0.0, w = 0.0;
#pragma unroll
        for (int k2 = 0; k2 < D; ++k2) {
          u += P[j * D + k2] * xr[k2];
          v += P[D * D + j * D + k2] * xl[k2];
          w += P[2 * D * D + D + j * D + k2] * xi[k2];
        }
        xs[(m - l0) * D + j] = ((u + v) + P[2 * D * D + j]) + w;
      }
    }
    const int nv = (r0 - l0 - 1) * D;  // x_(l0+1) .. x_(r0-1), contiguous in the path
    if constexpr (D % 2 == 0) {
      double2* o2 = reinterpret_cast<double2*>(out + (size_t)(l0 + 1) * D);
      for (int i = 0; i < nv / 2; ++i) o2[i] = make_double2(xs[D + 2 * i], xs[D + 2 * i + 1]);
    } else {
      for (int i = 0; i < nv; ++i) out[(size_t)(l0 + 1) * D + i] = xs[D + i];
    }
  }
}

// ---- any d (9..64): warp per (node, chain), lanes over rows; the dot products
// run in the register kernels' order (ascending j), so results match them.
constexpr int kDncWarps = 4;

__device__ __forceinline__ void dnc_normals_w(const NoiseArgs& nz, int c, uint64_t label,
                                              uint64_t index, int T, int d, int lane, double* xi) {
  if (nz.kind == AUXMC_NOISE_PREDRAWN) {
    const double* src = label == kDncBridge ? nz.bridge + ((size_t)c * nz.n_bridge + index) * d
                        : label == kTerminalDraw ? nz.terminal + (size_t)c * d
                                                 : nz.backward + ((size_t)c * T + index) * d;
    for (int i = lane; i < d; i += 32) xi[i] = src[i];
  } else {
    const uint64_t k = derive(nz.keys[c], label, index);
    for (int i = lane; i < d; i += 32) xi[i] = normal_at(k, (uint64_t)i);
  }
}

// y[i] = Σ_j A[i*d+j] x[j] (+ add[i]) for the lane's rows
__device__ __forceinline__ void w_matvec(int lane, int d, const double* A, const double* x,
                                         double* y) {
  for (int i = lane; i < d; i += 32) {
    double s = 0.0;
    for (int j = 0; j < d; ++j) s += A[i * d + j] * x[j];
    y[i] = s;
  }
}

__global__ void k_dnc_ends_gen(int T, int d, int B, int fr_shared, const double* __restrict__ term,
                               const double* __restrict__ nodes, const double* __restrict__ params,
                               long long n_heap, NoiseArgs nz, double* traj) {
  __shared__ double sv[kDncWarps][4][64];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x * kDncWarps + w;
  if (c >= B) return;
  const int dd = d * d, ES = (2 * dd + d + 1) & ~1, TS = (dd + d + 1) & ~1;
  const int b = fr_shared ? 0 : c;
  const double* tm = term + (size_t)b * TS;
  double* out = traj + (size_t)c * (T + 1) * d;
  double *xi = sv[w][0], *x = sv[w][1], *v = sv[w][2], *gx = sv[w][3];
  dnc_normals_w(nz, c, kTerminalDraw, 0, T, d, lane, xi);
  __syncwarp();
  w_matvec(lane, d, tm + d, xi, x);
  for (int i = lane; i < d; i += 32) {
    x[i] = tm[i] + x[i];
    out[(size_t)T * d + i] = x[i];
  }
  __syncwarp();
  if (T == 0) return;
  const double* root = nodes + ((size_t)b * n_heap + 1) * ES;
  const double* Lr = params + (size_t)b * n_heap * 2 * dd + dd;
  dnc_normals_w(nz, c, kBackwardNoise, 0, T, d, lane, xi);
  __syncwarp();
  w_matvec(lane, d, Lr, xi, v);
  w_matvec(lane, d, root, x, gx);
  for (int i = lane; i < d; i += 32) out[i] = gx[i] + (root[dd + i] + v[i]);
}

__global__ void k_dnc_level_gen(int T, int d, int B, int fr_shared, int level,
                                const double* __restrict__ nodes, const double* __restrict__ params,
                                long long n_heap, NoiseArgs nz, double* traj) {
  __shared__ double sv[kDncWarps][7][64];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int dd = d * d, ES = (2 * dd + d + 1) & ~1;
  const long long width = 1LL << level;
  const long long n = width * B;
  double *xl = sv[w][0], *xr = sv[w][1], *mu = sv[w][2], *v = sv[w][3], *wv = sv[w][4],
         *xi = sv[w][5], *lx = sv[w][6];
  for (long long q = (long long)blockIdx.x * kDncWarps + w; q < n;
       q += (long long)gridDim.x * kDncWarps) {
    const int c = (int)(q % B);
    const uint64_t h = (uint64_t)width + (uint64_t)(q / B);
    int l, r;
    if (!dnc_interval(h, T, l, r) || r - l < 2) continue;
    const int m = (l + r) / 2;
    const int b = fr_shared ? 0 : c;
    const double* elm = nodes + ((size_t)b * n_heap + 2 * h) * ES;
    const double* emr = nodes + ((size_t)b * n_heap + 2 * h + 1) * ES;
    const double* K = params + ((size_t)b * n_heap + h) * 2 * dd;
    const double* L = K + dd;
    double* out = traj + (size_t)c * (T + 1) * d;
    for (int i = lane; i < d; i += 32) {
      xl[i] = out[(size_t)l * d + i];
      xr[i] = out[(size_t)r * d + i];
    }
    dnc_normals_w(nz, c, kDncBridge, h, T, d, lane, xi);
    __syncwarp();
    w_matvec(lane, d, emr, xr, mu);
    for (int i = lane; i < d; i += 32) mu[i] += emr[dd + i];
    __syncwarp();
    w_matvec(lane, d, elm, mu, v);
    for (int i = lane; i < d; i += 32) v[i] = (xl[i] - v[i]) - elm[dd + i];
    __syncwarp();
    w_matvec(lane, d, K, v, wv);
    w_matvec(lane, d, L, xi, lx);
    for (int i = lane; i < d; i += 32) out[(size_t)m * d + i] = (mu[i] + wv[i]) + lx[i];
    __syncwarp();
  }
}

int launch_dnc(const DevModel& dm, int Bfr, int fr_shared, const double* elems,
               const double* term, const NoiseArgs& nz, int B, double* traj, Arena& ws,
               int* st_fr, cudaStream_t stream) {
  const int d = dm.dx, T = dm.T, dd = d * d;
  const int ES = (2 * dd + d + 1) & ~1;
  const int depth = dnc_depth(T);
  const long long n_heap = 2LL << depth;  // ids < 2^(depth+1)
  double* nodes = ws.take<double>((size_t)Bfr * n_heap * ES);
  double* params = ws.take<double>((size_t)Bfr * n_heap * 2 * dd);
  double* aff = d <= 8 ? ws.take<double>((size_t)Bfr * n_heap * ((3 * dd + d + 1) & ~1)) : nullptr;
  if (ws.base == nullptr) return AUXMC_OK;
  if (!nodes || !params || (d <= 8 && !aff)) return AUXMC_E_WORKSPACE;
  // CTA bridges keep 6 d*d + 4 doubles in shared memory; the warp-level draw
  // kernels stage 64-wide vectors: d <= 64
  if (d > 64 || sizeof(double) * (kBridgeBuffers * (size_t)dd + 4) > 227 * 1024)
    return AUXMC_E_DIM;
  const bool block = d > 16;  // CTA groups (blocked DMMA factor/solves) for d > 16
  const int warps = 4;
  if (T > 0) {
    for (int level = depth; level >= 0; --level) {
      const long long items = (1LL << level) * Bfr;
      if (block) {
        const int grid = (int)std::min<long long>(items, 148LL * 16);
        const size_t smem = sizeof(double) * 2 * dd;
        AUXMC_CUDA_TRY(cudaFuncSetAttribute(k_dnc_compose<true>,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        AUXMC_LAUNCH(k_dnc_compose<true>, grid, 128, smem, stream, T, d, level, Bfr, elems, nodes,
                     n_heap);
      } else {
        const int grid = (int)std::min<long long>((items + warps - 1) / warps, 148LL * 64);
        const size_t smem = sizeof(double) * 2 * dd * warps;
        AUXMC_CUDA_TRY(cudaFuncSetAttribute(k_dnc_compose<false>,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        AUXMC_LAUNCH(k_dnc_compose<false>, grid, 32 * warps, smem, stream, T, d, level, Bfr, elems,
                     nodes, n_heap);
      }
    }
    const long long items = (n_heap - 1) * Bfr;
    if (block) {
      const int grid = (int)std::min<long long>(items, 148LL * 16);
      const size_t smem = sizeof(double) * (kBridgeBuffers * dd + 4);
      AUXMC_CUDA_TRY(cudaFuncSetAttribute(k_dnc_bridge<true>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      AUXMC_LAUNCH(k_dnc_bridge<true>, grid, 128, smem, stream, T, d, Bfr, nodes, n_heap, 1LL,
                   n_heap, params, st_fr);
    } else {
      const int grid = (int)std::min<long long>((items + warps - 1) / warps, 148LL * 64);
      const size_t smem = sizeof(double) * (kBridgeBuffers * dd + 4) * warps;
      AUXMC_CUDA_TRY(cudaFuncSetAttribute(k_dnc_bridge<false>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      AUXMC_LAUNCH(k_dnc_bridge<false>, grid, 32 * warps, smem, stream, T, d, Bfr, nodes, n_heap,
                   1LL, n_heap, params, st_fr);
    }
  }
  if (d > 8) {
    AUXMC_LAUNCH(k_dnc_ends_gen, (B + kDncWarps - 1) / kDncWarps, 32 * kDncWarps, 0, stream, T, d,
                 B, fr_shared, term, nodes, params, n_heap, nz, traj);
    for (int level = 0; level < depth; ++level) {
      const long long n = (1LL << level) * B;
      const int grid = (int)std::min<long long>((n + kDncWarps - 1) / kDncWarps, 148LL * 64);
      AUXMC_LAUNCH(k_dnc_level_gen, grid, 32 * kDncWarps, 0, stream, T, d, B, fr_shared, level,
                   nodes, params, n_heap, nz, traj);
    }
    return AUXMC_OK;
  }
  // levels >= L0 run as subtrees of at most kDncSpan steps (intervals at level L
  // span at most ceil(T / 2^L) steps)
  int L0 = 0;
  while (L0 < depth && ((long long)T + (1LL << L0) - 1) / (1LL << L0) > kDncSpan) ++L0;
  switch (d) {
#define CASE(D)                                                                              \
  case D: {                                                                                  \
    AUXMC_LAUNCH(k_dnc_ends<D>, (B + 127) / 128, 128, 0, stream, T, B, fr_shared, term, nodes, \
                 params, n_heap, nz, traj);                                                  \
    for (int level = 0; level < L0; ++level) {                                               \
      const long long n = (1LL << level) * B;                                                \
      const int grid = (int)std::min<long long>((n + 255) / 256, 148LL * 32);                \
      AUXMC_LAUNCH(k_dnc_level<D>, grid, 256, 0, stream, T, B, fr_shared, level, nodes,      \
                   params, n_heap, nz, traj);                                                \
    }                                                                                        \
    if (L0 < depth) {                                                                        \
      const long long h_lo = 1LL << L0;                                                      \
      const long long na = (n_heap - h_lo) * Bfr;                                            \
      AUXMC_LAUNCH(k_dnc_affine<D>, (int)std::min<long long>((na + 255) / 256, 148LL * 32),  \
                   256, 0, stream, T, Bfr, nodes, params, n_heap, h_lo, aff);                \
      const size_t smem = sizeof(double) * (kDncSpan * dnc_aff_stride<D>() + kDncSpan +      \
                                            (size_t)dnc_lane_stride<D>() * kDncSubThreads);  \
      AUXMC_CUDA_TRY(cudaFuncSetAttribute(k_dnc_subtree<D>,                                  \
                                          cudaFuncAttributeMaxDynamicSharedMemorySize,       \
                                          (int)smem));                                       \
      const long long n = (1LL << L0) * ((B + kDncSubThreads - 1) / kDncSubThreads);         \
      const int grid = (int)std::min<long long>(n, 148LL * 16);                              \
      AUXMC_LAUNCH(k_dnc_subtree<D>, grid, kDncSubThreads, smem, stream, T, B, fr_shared, L0, \
                   depth, aff, n_heap, nz, traj);                                            \
    }                                                                                        \
    break;                                                                                   \
  }
    CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7) CASE(8)
#undef CASE
    default:
      return AUXMC_E_DIM;
  }
  return AUXMC_OK;
}

}  // namespace auxmc_gpu
