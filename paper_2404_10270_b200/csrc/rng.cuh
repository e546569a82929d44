// splitmix64 counter-based streams (pkg/src/picmc/rng.py:56-116) on the
// device: integer arithmetic, bit-exact with the reference.
#pragma once

#include "common.cuh"

namespace pb {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ uint64_t derive(uint64_t key, uint64_t n) {
  return mix64(key + (n + 1) * kGolden);
}

__device__ __forceinline__ double uniform(uint64_t key, uint64_t c) {
  return __dmul_rn((double)(derive(key, c) >> 11), 0x1p-53);
}

__device__ __forceinline__ double uniform_open(uint64_t key, uint64_t c) {
  return __dmul_rn(__dadd_rn((double)(derive(key, c) >> 11), 0.5),
                   0x1p-53);
}

}  // namespace pb
