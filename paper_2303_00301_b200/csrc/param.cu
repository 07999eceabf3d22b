// param.cu — diffusion-coefficient random-walk MH within Gibbs (runner.cpp:61-85,
// called at :159-161 and :188-190) for a batch of chains.
//
// The move needs Σ_t |x_{t+1} − a(x_t)|² over the chain's path (the drift a does not
// depend on γ, runner.cpp:58-60), then one scalar MH decision.  One warp per chain:
// lanes evaluate the residuals of 32 consecutive steps in parallel and every lane
// folds them into the running sum in t order through shuffles, so the sum has the
// reference's serial rounding order (:65-70).  The path is read once (8·(T+1)·d B per
// chain), HBM-bound; lane 0 then draws from s = root.derive(kParam, iter) — normal at
// counter 0, uniform at counter 1 (rng.hpp:85-95) — and applies the strict `<` test.
#include <cmath>

#include "common.cuh"
#include "rng.cuh"
#include "target.cuh"

namespace auxmc_gpu {
namespace {

constexpr double kPi = 3.14159265358979323846;

// Products feeding a sum are rounded separately (__dmul_rn) so nvcc does not contract
// them into FMAs: the oracle (and the reference on x86-64) rounds each product.
__global__ void k_gamma_move(DevTarget tg, int C, const double* __restrict__ x,
                             const uint64_t* __restrict__ roots, long long iter, double step,
                             double* __restrict__ gamma, int* __restrict__ moved) {
  const int lane = threadIdx.x & 31;
  const int c = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (c >= C) return;
  const int T = tg.T, d = tg.dx;
  const double* xc = x + (size_t)c * (T + 1) * d;
  double sse = 0.0;
  for (int base = 0; base < T; base += 32) {
    const int t = base + lane;
    double sq = 0.0;
    if (t < T) {
      const double* xt = xc + (size_t)t * d;
      for (int i = 0; i < d; ++i) {
        const double r = xt[d + i] - dyn_mean_i(tg, t, xt, i);
        sq += __dmul_rn(r, r);
      }
    }
    const int n = T - base < 32 ? T - base : 32;
    for (int j = 0; j < n; ++j) sse += __shfl_sync(0xffffffffu, sq, j);
  }
  if (lane) return;
  const double h = tg.kind == AUXMC_KIND_LORENZ63 ? tg.lz_h : tg.l96_h;
  const double hd = 0.5 * d;  // 1.5 for Lorenz-63 (runner.cpp:71-74), exact
  const double g0 = gamma[c];
  auto loglik = [&](double g) {
    return __dmul_rn(-hd * T, log(2.0 * kPi * h * g * g)) - sse / (2.0 * h * g * g);
  };
  const uint64_t key = derive(roots[c], kParam, (uint64_t)iter);
  const double lg = log(g0);
  const double lg_prop = lg + __dmul_rn(step, normal_at(key, 0));
  const double g_prop = exp(lg_prop);
  const double log_r = (loglik(g_prop) - __dmul_rn(0.5 * lg_prop, lg_prop)) -
                       (loglik(g0) - __dmul_rn(0.5 * lg, lg));
  const int acc = log(uniform_at(key, 1)) < log_r;
  if (acc) gamma[c] = g_prop;
  moved[c] = acc;
}

}  // namespace
}  // namespace auxmc_gpu

using namespace auxmc_gpu;

extern "C" {

int auxmc_gamma_move(const auxmc_target* target, int C, const double* x,
                     const uint64_t* root_keys, long long iter, double step, double* gamma,
                     int* moved, void* stream) {
  if (!device_ok()) return AUXMC_E_CUDA;
  int st = check_target(target);
  if (st) return st;
  if (target->kind != AUXMC_KIND_LORENZ63 && target->kind != AUXMC_KIND_LORENZ96)
    return AUXMC_E_CONFIG;
  if (C < 0 || !x || !root_keys || !gamma || !moved) return AUXMC_E_ARG;
  if (C == 0) return AUXMC_OK;
  const DevTarget tg = to_dev_target(*target);
  AUXMC_LAUNCH(k_gamma_move, (C + 3) / 4, 128, 0, stream, tg, C, x, root_keys, iter, step, gamma,
               moved);
  return AUXMC_OK;
}

}  // extern "C"
