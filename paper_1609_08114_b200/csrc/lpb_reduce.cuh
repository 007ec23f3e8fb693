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

// The candidate lanes' lowest and highest lane ids by two independent REDUX (≈ 22 cycles each,
// issued back to back) instead of VOTE.ballot + FLO (≈ 60 cycles as a dependent pair on
// sm_100, scripts/ubench/lat_ops.cu): none if lo == 32, unique if lo == hi.
#define LPB_FIRST_LANE(c1, none_ret)                                                  \
  const unsigned lane_ = threadIdx.x & 31u;                                          \
  const unsigned l1 = __reduce_min_sync(kFullMask, (c1) ? lane_ : 32u);              \
  const unsigned l2 = __reduce_max_sync(kFullMask, (c1) ? lane_ : 0u);               \
  if (l1 == 32u) return none_ret;                                                    \
  if (l1 == l2) return (int)l1;

// Warp argmax of (key desc, tie asc) over lanes with `valid`; returns the winner lane or -1.
// Must be called by all 32 lanes.  Fast path: one REDUX on the key's high word (+ the lane
// REDUXes above); only when several lanes share it (rare for real-valued data) are the low
// word and the tie key reduced as well.
__device__ __forceinline__ int warp_argmax(bool valid, unsigned long long k, unsigned tie) {
  const unsigned hi = valid ? (unsigned)(k >> 32) : 0u;
  const unsigned mhi = __reduce_max_sync(kFullMask, hi);
  const bool c1 = valid && hi == mhi;
  LPB_FIRST_LANE(c1, -1)
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
  LPB_FIRST_LANE(c1, -1)
  const unsigned lo = c1 ? (unsigned)k : 0xffffffffu;
  const unsigned mlo = __reduce_min_sync(kFullMask, lo);
  const bool c2 = c1 && (unsigned)k == mlo;
  const unsigned t = c2 ? tie : 0xffffffffu;
  const unsigned mt = __reduce_min_sync(kFullMask, t);
  return __ffs(__ballot_sync(kFullMask, c2 && tie == mt)) - 1;
}


}  // namespace lpb
