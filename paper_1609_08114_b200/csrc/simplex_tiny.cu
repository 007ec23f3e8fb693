// simplex_tiny.cu — S class, register variant: one LP per THREAD with the whole condensed
// tableau in registers, for type-1 LPs (b >= 0) of m, n <= 6 (cfg1 is 5x5).
//
// The SMEM-slice kernel (simplex_thread.cu) keeps each thread's tableau in shared memory so
// that the dynamic pivot row / column are plain indexed loads; its occupancy is set by the
// slice size (~10 warps per SM at 5x5) and every step of the pivot chain waits on SMEM.
// Here the tableau is a C x C register array (C = compile-time capacity, padded positions
// hold -inf in the objective row and are never candidates) and the dynamic row l and column
// e are picked with predicated selects over the fully unrolled array: per pivot C*C DFMAs
// plus selects, no memory traffic, no barrier.  The pivot arithmetic is the SMEM kernel's
// (and the oracle's) operation for operation: Step 1 over positions (
// RPC P:133; Bland after K stalls, reading R6), ratio test by IEEE division,
// pivot row divided by PE and fma(-f_i, prow_j, T_ij) elsewhere (Listing 1).
//
// An LP with some b_i < 0 needs the two-phase method and up to m more
// positions: the thread appends it to a.defer_list and the SMEM-slice kernel, launched next
// in list mode, solves exactly those LPs (none for cfg1's type-1 batch).
#include <algorithm>
#include <climits>

#include "lpb_fp64.cuh"
#include "lpb_internal.cuh"
#include "lpb_rng.cuh"

namespace lpb {
namespace {

constexpr int TY_MAXC = 6;

__device__ __forceinline__ double ninf() { return __longlong_as_double(0xfff0000000000000ll); }

// Persistent: every thread solves LP after LP, taking the next LP index from the launch's
// ticket the moment its current LP ends (one atomicAdd per warp for all lanes that need one),
// so a warp's lanes stay busy instead of idling until the slowest of 32 fixed LPs finishes
// (pivot counts per LP vary 0..8 at 5x5, mean 1.9: the fixed mapping ran every warp for its
// maximum).  Each loop iteration is one pivot of every busy lane; the build and the extract
// of the lanes that start / finish an LP run as (divergent) branches of the same iteration.
#ifndef LPB_TINY_MINB
#define LPB_TINY_MINB 4  // 4 CTAs (16 warps) per SM: 128 registers (measured best of 1, 4, 5)
#endif
template <int C, bool RPC>  // RPC: a separate instantiation keeps LPC's registers
__global__ void __launch_bounds__(128, LPB_TINY_MINB) simplex_tiny_kernel(SimplexArgs a) {
  const int m = a.m, n = a.n;
  const unsigned lane = threadIdx.x & 31u;
  // kmax_hint = 0 (type-1 promise, include/lpb.h): an LP with some b_i < 0 is reported
  // LPB_BAD_HINT here instead of being deferred to the two-phase SMEM-slice kernel
  const bool hinted = a.khint == 0;
  double T[C][C], d[C], rhs[C];
  // basis keys and nonbasic variables packed 8 bits per entry (values <= 2 * TY_MAXC, 255 =
  // a padding position): dynamic-index reads / writes are a shift and a mask instead of
  // selects over C registers, and 2 registers each instead of C (spills 112 -> 84 bytes at
  // C = 5; cfg1m 0.152 -> 0.150 ms)
  uint64_t pbk = 0ull, pnv = 0ull;
#define BKEY(i_) ((int)((pbk >> (8 * (i_))) & 0xffull))
#define NBV(j_) ((int)((pnv >> (8 * (j_))) & 0xffull))
  double z = 0.0;  // objective row's RHS cell (obj = -z, reading R3)
  int it2 = 0, stall = 0;
  int64_t lp = 0;
  bool have = false;
  uint64_t lpkey = 0ull;
  // Step 1 (entering position) of the NEXT pivot; computed right after the build and right
  // after each update, so that an LP whose last pivot leaves no candidate is extracted in
  // the same loop iteration (an LP with p pivots takes max(p, 1) iterations, not p + 1).
  int e = -1, ev = INT_MAX;
  auto step1 = [&]() {
    // LPC: max d, lowest variable on ties; Bland: lowest variable; RPC: largest
    // counter-based score (include/lpb.h)
    const bool bland = a.bland_K > 0 && stall >= a.bland_K;
    const bool rpc = RPC && !bland;
    const uint64_t pkey = rpc ? rpc_pivot_key(lpkey, it2) : 0ull;
    e = -1;
    ev = INT_MAX;
    double best = 0.0;
    uint64_t ub = 0ull;
#pragma unroll
    for (int j = 0; j < C; ++j) {
      const int var = NBV(j);
      const double dj = d[j];
      const bool cand = dj > a.eps_enter;  // padding positions (variable 255) hold -inf forever
      bool take;
      if (rpc) {
        const uint64_t u = rpc_score(pkey, var);
        take = cand && (e < 0 || u > ub || (u == ub && var < ev));
        ub = take ? u : ub;
      } else if (bland) {
        take = cand && var < ev;
      } else {
        take = cand && (e < 0 || dj > best || (dj == best && var < ev));
      }
      e = take ? j : e;
      ev = take ? var : ev;
      best = take ? dj : best;
    }
  };
  for (;;) {
    // ---- refill: the lanes without an LP take consecutive tickets ----
    {
      const unsigned act = __activemask();
      const unsigned need = __ballot_sync(act, !have);
      if (need) {
        const int leader = __ffs(need) - 1;
        int base = 0;
        if ((int)lane == leader) base = atomicAdd(a.ticket, __popc(need));
        base = __shfl_sync(act, base, leader);
        if (!have) lp = (int64_t)base + __popc(need & ((1u << lane) - 1u));
      }
    }
    if (!have) {
      if (lp >= a.batch) break;
      // ---- build (type 1: slack basis, R7 with k = 0) ----
      const double* __restrict__ Ak = a.A + lp * a.sA;
      const double* __restrict__ bk = a.b + lp * a.sb;
      const double* __restrict__ ck = a.c + lp * (int64_t)n;
      bool neg = false;
#pragma unroll
      for (int i = 0; i < C; ++i) {
        rhs[i] = (i < m) ? __ldg(bk + i) : 0.0;
        neg |= rhs[i] < 0.0;
      }
      if (neg) {
        if (hinted) {  // the caller's type-1 promise is broken: not solved
          a.status[lp] = ST_BAD_HINT;
          a.iters[2 * lp] = 0;
          a.iters[2 * lp + 1] = 0;
          a.obj[lp] = __longlong_as_double(0x7ff8000000000000ll);
          if (a.x)
            for (int j = 0; j < n; ++j) a.x[lp * n + j] = __longlong_as_double(0x7ff8000000000000ll);
        } else {  // two-phase LP: the SMEM-slice kernel takes it
          a.defer_list[atomicAdd(a.defer_cnt, 1)] = (int)lp;
        }
        continue;
      }
#pragma unroll
      for (int i = 0; i < C; ++i) {
#pragma unroll
        for (int j = 0; j < C; ++j) T[i][j] = (i < m && j < n) ? __ldg(Ak + i * n + j) : 0.0;
        if (i == 0) pbk = 0ull;
        pbk |= (uint64_t)(n + i) << (8 * i);
      }
#pragma unroll
      for (int j = 0; j < C; ++j) {
        d[j] = (j < n) ? __ldg(ck + j) : ninf();
        if (j == 0) pnv = 0ull;
        pnv |= (uint64_t)((j < n) ? j : 0xff) << (8 * j);
      }
      z = 0.0;
      it2 = 0;
      stall = 0;
      lpkey = RPC ? rpc_lp_key(a.rpc_seed, a.lp_base + lp) : 0ull;
      have = true;
      step1();
    }

    // ---- one pivot; Step 1 was done at the build / the last update ----
    int st = -1;
    const bool bland = a.bland_K > 0 && stall >= a.bland_K;
    double theta = 0.0;
    int l = -1;
    double col[C];
    if (e < 0) {
      st = ST_OPTIMAL;
    } else if (it2 >= a.max_iter) {
      st = ST_ITER_LIMIT;
    } else {
      // Step 2: ratio test over rows i < m with T[i][e] > eps_piv (R1, R2, R5)
#pragma unroll
      for (int i = 0; i < C; ++i) {
        double v = T[i][0];
#pragma unroll
        for (int j = 1; j < C; ++j) v = (e == j) ? T[i][j] : v;
        col[i] = v;
      }
      // Pass 1: approximate quotients rhs_i * (1/v_i) (MUFU reciprocal + one Newton step,
      // relative error ~1e-12 < 2^-36) find the smallest; the exact IEEE quotient of that row is
      // the answer unless another candidate lies within the approximation's error of it (a
      // near or exact tie, e.g. several zero ratios) or Bland's rule orders ties by basis
      // key: then every candidate is divided exactly, as before.
      bool val[C];
      double qa[C];
      double amin = 0.0;
#pragma unroll
      for (int i = 0; i < C; ++i) {
        val[i] = i < m && col[i] > a.eps_piv;
        const double v = val[i] ? col[i] : 1.0;
        qa[i] = __dmul_rn(rhs[i], recip_approx(v));
        const bool take = val[i] && (l < 0 || qa[i] < amin);
        amin = take ? qa[i] : amin;
        l = take ? i : l;
      }
      // a row j can only tie with or beat row l exactly if qa_j <= amin + 4 * 2^-30 * |amin|
      // (the approximation's relative error is below 2^-36; zero ratios are exact, and
      // +-inf quotients compare equal to each other)
      const double lim = __fma_rn(fabs(amin), 0x1p-28, amin);
      bool multi = bland;
#pragma unroll
      for (int i = 0; i < C; ++i) multi |= val[i] && i != l && qa[i] <= lim;
      if (!multi && l >= 0) {
        double v = col[0], rv = rhs[0];
#pragma unroll
        for (int i = 1; i < C; ++i) {
          v = (l == i) ? col[i] : v;
          rv = (l == i) ? rhs[i] : rv;
        }
        bool slow;
        theta = div_fast(rv, v, slow);
        if (slow) theta = ddiv_slow(rv, v);
      } else if (l >= 0) {
        l = -1;
        int lkey = INT_MAX;
#pragma unroll
        for (int i = 0; i < C; ++i) {
          bool slow;
          double rr = div_fast(rhs[i], val[i] ? col[i] : 1.0, slow);
          if (slow) rr = ddiv_slow(rhs[i], val[i] ? col[i] : 1.0);
          const int key = bland ? BKEY(i) : i;
          const bool take = val[i] && (l < 0 || rr < theta || (rr == theta && key < lkey));
          l = take ? i : l;
          lkey = take ? key : lkey;
          theta = take ? rr : theta;
        }
      }
      if (l < 0) st = ST_UNBOUNDED;
    }
    if (st < 0) {
      // Step 3: pivot row / PE (IEEE division, R12), fma update of every other row incl. the
      // objective; position e becomes the leaving variable's column (R13)
      double pe = col[0], prr = rhs[0];
      double prow[C];
#pragma unroll
      for (int j = 0; j < C; ++j) prow[j] = T[0][j];
#pragma unroll
      for (int i = 1; i < C; ++i) {
        const bool s_ = (l == i);
        pe = s_ ? col[i] : pe;
        prr = s_ ? rhs[i] : prr;
#pragma unroll
        for (int j = 0; j < C; ++j) prow[j] = s_ ? T[i][j] : prow[j];
      }
      const double r = recip_of(pe);
      double pv[C];
      bool slow_any = false;
#pragma unroll
      for (int j = 0; j < C; ++j) {
        bool sl;
        pv[j] = div_with((j == e) ? 1.0 : prow[j], pe, r, sl);
        slow_any |= sl;
      }
      bool slr;
      double pr = div_with(prr, pe, r, slr);
      if (slow_any || slr) {  // rare: outside div_with's fast range -> IEEE __ddiv_rn
#pragma unroll
        for (int j = 0; j < C; ++j) pv[j] = ddiv_slow((j == e) ? 1.0 : prow[j], pe);
        pr = ddiv_slow(prr, pe);
      }
#pragma unroll
      for (int i = 0; i < C; ++i) {
        const bool piv = (i == l);
        const double f = -col[i];
#pragma unroll
        for (int j = 0; j < C; ++j)
          T[i][j] = piv ? pv[j] : __fma_rn(f, pv[j], (j == e) ? 0.0 : T[i][j]);
        rhs[i] = piv ? pr : __fma_rn(f, pr, rhs[i]);
      }
      double fd = d[0];
#pragma unroll
      for (int j = 1; j < C; ++j) fd = (e == j) ? d[j] : fd;
      fd = -fd;
#pragma unroll
      for (int j = 0; j < C; ++j) d[j] = __fma_rn(fd, pv[j], (j == e) ? 0.0 : d[j]);
      z = __fma_rn(fd, pr, z);
      // basis swap: row l's basic variable leaves into position e
      const int leaving = BKEY(l);
      pbk = (pbk & ~(0xffull << (8 * l))) | ((uint64_t)ev << (8 * l));
      pnv = (pnv & ~(0xffull << (8 * e))) | ((uint64_t)leaving << (8 * e));
      ++it2;
      stall = (theta > 0.0) ? 0 : stall + 1;
      step1();
      if (e < 0) st = ST_OPTIMAL;
      else if (it2 >= a.max_iter) st = ST_ITER_LIMIT;
      if (st < 0) continue;
    }

    // ---- extract (R10) ----
    a.status[lp] = st;
    a.iters[2 * lp] = 0;
    a.iters[2 * lp + 1] = it2;
    a.obj[lp] = (st == ST_OPTIMAL) ? -z
              : (st == ST_UNBOUNDED) ? __longlong_as_double(0x7ff0000000000000ll)
                                     : __longlong_as_double(0x7ff8000000000000ll);
    if (a.x) {
      double* xk = a.x + lp * (int64_t)n;
      const double fill = (st == ST_OPTIMAL) ? 0.0 : __longlong_as_double(0x7ff8000000000000ll);
      for (int j = 0; j < n; ++j) xk[j] = fill;
      if (st == ST_OPTIMAL) {
#pragma unroll
        for (int i = 0; i < C; ++i)
          if (i < m && BKEY(i) < n) xk[BKEY(i)] = rhs[i];
      }
    }
    have = false;
  }
}

}  // namespace

bool tiny_fits(int m, int n) { return m <= TY_MAXC && n <= TY_MAXC; }

template <int C, bool RPC>
static cudaError_t launch_tiny(const SimplexArgs& a, cudaStream_t s) {
  auto kern = simplex_tiny_kernel<C, RPC>;
  static LaunchMemo memo;
  int per_sm = 0;
  const cudaError_t em = memo.get(0, &per_sm, [&](int& v, size_t) {
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, kern, 128, 0);
  });
  if (em != cudaSuccess) return em;
  // persistent grid: the resident CTAs (or fewer 32-thread CTAs for a small batch, spread
  // over the SMs)
  const int nt = a.batch >= (int64_t)device_sm_count() * 128 ? 128 : 32;
  const int64_t resident = (int64_t)(per_sm < 1 ? 1 : per_sm) * device_sm_count() * (128 / nt);
  int64_t grid = (a.batch + nt - 1) / nt;
  if (grid > resident) grid = resident;
  kern<<<(unsigned)grid, nt, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_simplex_tiny(const SimplexArgs& a, cudaStream_t s) {
  const bool hinted = a.khint == 0;  // type-1 promise: no deferred list, one launch
  cudaError_t e = cudaMemsetAsync(a.ticket, 0, sizeof(int), s);
  if (e != cudaSuccess) return e;
  if (!hinted) {
    e = cudaMemsetAsync(a.defer_cnt, 0, sizeof(int), s);
    if (e != cudaSuccess) return e;
  }
  const int c = std::max(a.m, a.n);
#define LPB_TINY_GO(CC) \
  e = a.rpc ? launch_tiny<CC, true>(a, s) : launch_tiny<CC, false>(a, s)
  if (c <= 3) LPB_TINY_GO(3);
  else if (c == 4) LPB_TINY_GO(4);
  else if (c == 5) LPB_TINY_GO(5);
  else LPB_TINY_GO(6);
#undef LPB_TINY_GO
  if (e != cudaSuccess || hinted) return e;
  return launch_simplex_thread(a, s);  // list mode: the deferred two-phase LPs
}

}  // namespace lpb
