// lpb_rng.cuh — the counter-based draw of the RPC entering rule ("Random
// Positive Coefficient"; include/lpb.h LPB_RULE_RPC, reading R15 in DESIGN.md).
//
// No random state is stored: candidate variable j of LP k at pivot t scores
//   u = mix64(mix64(mix64(seed ^ mix64(k)) ^ t) ^ j) >> 11      (an integer < 2^53)
// and the largest score enters (ties: lowest j), so the choice is uniform over the
// candidates and independent of how a size class stores its positions.
#pragma once
#include <cstdint>

namespace lpb {

// SplitMix64 finaliser.
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Per-LP part of the key (k = the LP's index in the lpb_solve_batch call).
__device__ __forceinline__ uint64_t rpc_lp_key(uint64_t seed, int64_t k) {
  return mix64(seed ^ mix64((uint64_t)k));
}

// Per-pivot part (t = phase-I + phase-II pivots done so far).
__device__ __forceinline__ uint64_t rpc_pivot_key(uint64_t lp_key, int t) {
  return mix64(lp_key ^ (uint64_t)(uint32_t)t);
}

// Score of candidate variable j.
__device__ __forceinline__ uint64_t rpc_score(uint64_t pivot_key, int j) {
  return mix64(pivot_key ^ (uint64_t)(uint32_t)j) >> 11;
}

}  // namespace lpb
