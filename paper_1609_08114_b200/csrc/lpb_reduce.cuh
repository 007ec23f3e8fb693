// lpb_reduce.cuh — warp-wide (value, tie) argmax / argmin with the sm_100 REDUX instructions
// (__reduce_*_sync), used by the simplex kernels for Step 1 (entering column, PAPER.md:93,
// 132) and Step 2 (ratio test).  The comparison order is exactly the
// oracle's: values compared as IEEE doubles (-0 == +0), ties broken by the smaller tie key.
#pragma once
#include <cuda_runtime.h>

namespace lpb {

constexpr unsigned kFullMask = 0xffffffffu;

// Order-preserving 64-bit key of a double; -0.0 is folded to +0.0 first so that IEEE
// equality (-0 == +0) remains a tie, as in the oracle's comparisons.
__device__ __forceinline__ unsigned long long okey(double d) {
  const unsigned long long u = (unsigned long long)__double_as_longlong(__dadd_rn(d, 0.0));
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ unsigned ikey(int t) { return (unsigned)t ^ 0x80000000u; }

// Warp argmax of (key desc, tie asc) over lanes with `valid`; returns the winner lane or -1.
// Must be called by all 32 lanes.  Fast path: one REDUX on the key's high word; only when
// several lanes share it (rare for real-valued data) are the low word and the tie key
// reduced as well.
__device__ __forceinline__ int warp_argmax(bool valid, unsigned long long k, unsigned tie) {
  const unsigned hi = valid ? (unsigned)(k >> 32) : 0u;
  const unsigned mhi = __reduce_max_sync(kFullMask, hi);
  const bool c1 = valid && hi == mhi;
  const unsigned b1 = __ballot_sync(kFullMask, c1);
  if (b1 == 0u) return -1;
  if ((b1 & (b1 - 1u)) == 0u) return __ffs(b1) - 1;
  const unsigned lo = c1 ? (unsigned)k : 0u;
  const unsigned mlo = __reduce_max_sync(kFullMask, lo);
  const bool c2 = c1 && (unsigned)k == mlo;
  const unsigned t = c2 ? tie : 0xffffffffu;
  const unsigned mt = __reduce_min_sync(kFullMask, t);
  return __ffs(__ballot_sync(kFullMask, c2 && tie == mt)) - 1;
}

// Warp argmin of (key asc, tie asc) over lanes with `valid`; returns the winner lane or -1.
__device__ __forceinline__ int warp_argmin(bool valid, unsigned long long k, unsigned tie) {
  const unsigned hi = valid ? (unsigned)(k >> 32) : 0xffffffffu;
  const unsigned mhi = __reduce_min_sync(kFullMask, hi);
  const bool c1 = valid && hi == mhi;
  const unsigned b1 = __ballot_sync(kFullMask, c1);
  if (b1 == 0u) return -1;
  if ((b1 & (b1 - 1u)) == 0u) return __ffs(b1) - 1;
  const unsigned lo = c1 ? (unsigned)k : 0xffffffffu;
  const unsigned mlo = __reduce_min_sync(kFullMask, lo);
  const bool c2 = c1 && (unsigned)k == mlo;
  const unsigned t = c2 ? tie : 0xffffffffu;
  const unsigned mt = __reduce_min_sync(kFullMask, t);
  return __ffs(__ballot_sync(kFullMask, c2 && tie == mt)) - 1;
}


}  // namespace lpb
