// rng.cuh — counter-based splitmix64 streams on the device.
//
// Bit-exact restatement of the integer path of proj/include/auxmc/rng.hpp:35-118:
// derive(label, index) (rng.hpp:73-80), word_at (:47-49), to_unit_open (:51-54),
// Box-Muller normals from words 2c, 2c+1 (:90-95).  Every draw is a pure
// function of (key, counter), so any thread can generate any variate of any
// chain without coordination.  FP64 log/cos/sqrt are CUDA libdevice (<= 2 ulp
// from glibc), which is the only source of difference against the CPU stream.
#pragma once
#include <cstdint>

namespace auxmc_gpu {

enum : uint64_t {
  kBackwardNoise = 1, kTerminalDraw = 2, kAuxObs = 3, kDncBridge = 4, kMhAccept = 5,
  kIteration = 6, kChain = 7, kStep = 8, kParticle = 9, kResample = 10,
  kTerminalIndex = 11, kBackwardIndex = 12, kPmKey = 13, kSimulate = 14, kParam = 15
};

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;
constexpr uint64_t kLabelSalt = 0xA0761D6478BD642Full;
constexpr uint64_t kIndexSalt = 0xE7037ED1A0B428DBull;

__host__ __device__ __forceinline__ uint64_t word_at(uint64_t key, uint64_t i) {
  return mix64(key + (i + 1) * kGolden);
}

__host__ __device__ __forceinline__ double to_unit_open(uint64_t w) {
  return (static_cast<double>(w >> 11) + 0.5) * 0x1.0p-53;
}

__host__ __device__ __forceinline__ uint64_t seed_key(uint64_t seed) { return mix64(seed + kGolden); }

// derive split into its two halves: the label half is a per-(parent,label)
// constant that kernels hoist out of their t loops.
__host__ __device__ __forceinline__ uint64_t derive_label(uint64_t key, uint64_t label) {
  return mix64(key ^ mix64(label ^ kLabelSalt));
}
__host__ __device__ __forceinline__ uint64_t derive_index(uint64_t k_label, uint64_t index) {
  return mix64(k_label ^ mix64(index ^ kIndexSalt));
}
__host__ __device__ __forceinline__ uint64_t derive(uint64_t key, uint64_t label, uint64_t index) {
  return derive_index(derive_label(key, label), index);
}

__host__ __device__ __forceinline__ double uniform_at(uint64_t key, uint64_t c) {
  return to_unit_open(word_at(key, 2 * c));
}

__device__ __forceinline__ double normal_at(uint64_t key, uint64_t c) {
  const double u1 = to_unit_open(word_at(key, 2 * c));
  const double u2 = to_unit_open(word_at(key, 2 * c + 1));
  return sqrt(-2.0 * log(u1)) * cos(6.283185307179586476925286766559 * u2);
}

__host__ __device__ __forceinline__ uint64_t key_at(uint64_t key, uint64_t c) {
  return word_at(key, 2 * c);
}

}  // namespace auxmc_gpu
