// simplex_reg.cu — R class: one LP per thread block (one warp for small LPs) with the
// condensed fp64 tableau RESIDENT IN REGISTERS (256 KB register file per SM).
//
// Same method and arithmetic as simplex_block.cu / the oracle (§3.1 Steps 1-3,
// Listing 1; two-phase PAPER.md:76), different storage and reductions:
//   * thread (tr, tc) of a TR x TC grid owns constraint rows i = tr + TR*a (a < A) and
//     nonbasic positions p = tc + TC*b (b < BC): double T[A][BC] in registers;
//   * the objective row(s) are REPLICATED in every thread for its positions (d2, d1), so
//     Step 1 (Dantzig argmax; or RPC) is a register scan + a
//     REDUX-based warp argmax in every warp (no barrier), computed straight-line at the end
//     of the previous pivot's update so its latency interleaves with the update's DFMAs;
//   * Step 2 (ratio test): the owners of column e publish it to SMEM; each
//     lane of a warp then takes one of the warp's rows (one IEEE division per lane), applies
//     the previous pivot's RHS update to it (the RHS column lives in SMEM and is updated
//     lazily, each row by exactly one lane), and the winning lane writes the warp's partial
//     -> barrier 1 -> every thread scans the partials;
//   * Step 3: the owners of row l publish the RAW row -> barrier 2 ->
//     every thread divides its own positions by PE (with PE's reciprocal, which the winning
//     ratio lane computed for its own division and passed along in its partial) and applies
//     T_ip = fma(f_i, prow_p, T_ip)
//     to its registers (A*BC DFMAs with no per-element branch).  Row l and position e were
//     zeroed when they were read, so the same fma produces the pivot row (f_l = 1) and the
//     leaving variable's column.
// Reductions use order-preserving integer keys and the sm_100 REDUX (__reduce_*_sync)
// instructions: (value, tie key) argmax/argmin in three warp-wide REDUX steps.
// All arithmetic matches oracle/lpb_oracle.c bit for bit (IEEE __ddiv_rn, explicit
// __fma_rn, ascending __dadd_rn sums).
#include <climits>
#include <cstdlib>

#include "lpb_async.cuh"
#include "lpb_fp64.cuh"
#include "lpb_internal.cuh"
#include "lpb_reduce.cuh"
#include "lpb_rng.cuh"
#include "lpb_tmem.cuh"

namespace lpb {
namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int DEADV = INT_MAX;

__device__ __forceinline__ double neg_inf() { return __longlong_as_double(0xfff0000000000000ll); }
__device__ __forceinline__ double pos_inf() { return __longlong_as_double(0x7ff0000000000000ll); }
__device__ __forceinline__ double qnan() { return __longlong_as_double(0x7ff8000000000000ll); }

// Barrier of the LP's thread group.
template <int NT>
__device__ __forceinline__ void gsync() {
  if constexpr (NT == 32) __syncwarp();
  else __syncthreads();
}

#define LPB_CASES(BODY)                                                                     \
  BODY(0) BODY(1) BODY(2) BODY(3) BODY(4) BODY(5) BODY(6) BODY(7) BODY(8) BODY(9) BODY(10) \
  BODY(11) BODY(12) BODY(13) BODY(14) BODY(15) BODY(16) BODY(17) BODY(18) BODY(19)         \
  BODY(20) BODY(21) BODY(22) BODY(23) BODY(24) BODY(25) BODY(26) BODY(27) BODY(28)         \
  BODY(29) BODY(30) BODY(31)

struct Part {  // a (value, tie, index) reduction partial
  double v;
  int tie;
  int idx;
  double rc;  // ratio test: recip_of(T[idx][e]), i.e. PE's reciprocal if this row wins
};

template <int TR, int TC, int AT, int BC>
struct RegSmem {
  static constexpr int RCAP = TR * AT, CCAP = TC * BC, NWARP = (TR * TC) / 32;
  double colE[2][RCAP];  // pivot column (constraint rows), double-buffered by pivot parity
  double fcol[2][RCAP];  // update multipliers: -colE, and +1 for the pivot row
  double fobj[2][2];     // pivot-column entries of the phase-II / phase-I rows
  double rhs[RCAP];      // RHS column (lazily updated)
  double prow[CCAP];     // new pivot row (positions); scratch for the phase-I row at build
  int bkey[RCAP];        // row -> basic variable key (>= 0 real, < 0 artificial)
  int nbvar[CCAP];       // position -> nonbasic variable index (DEADV: dead / padding)
  int negrows[RCAP];     // ascending rows with b_i < 0
  int wcount[NWARP];
  Part part[NWARP];      // ratio-test partial per warp
  uint64_t mbar;         // completes when the prefetched A of LP `lp` has landed
  int lp;
  int leaving;
  uint32_t tmem;         // TMEM base address (TM layouts)
};

// Optional phase profiler, compiled in only with -DLPB_PROFILE (scripts/phase_prof.py builds
// that variant): warp 0 of every CTA accumulates clock64() deltas per pivot phase into
// prof[blockIdx.x * 12 + phase] when SimplexArgs::prof is set.
#ifdef LPB_PROFILE
#define LPB_PROF_MARK(ph)                                                 \
  if (prof_on) {                                                          \
    const long long t_ = clock64();                                       \
    pacc[ph] += t_ - pt;                                                  \
    pt = t_;                                                              \
  }
#else
#define LPB_PROF_MARK(ph)
#endif

// AS > 0: each thread also owns AS more rows (i = tr + TR*(A+s)) kept in a thread-private
// SMEM slice (double2 pairs of positions, thread-interleaved: conflict-free 128-bit accesses),
// so that three LPs fit one SM (registers + SMEM) instead of two (registers only).
// TM: the AS extra rows live in TENSOR MEMORY instead (lpb_tmem.cuh): thread tid owns TMEM
// lane tid, row slot s at columns 16 s .. 16 s + 13 (BC doubles), reached with tcgen05.ld/st
// from the whole warp at a warp-uniform column; no SMEM traffic and no prefetch buffer, so
// three CTAs (LPs) share an SM: 2/3 of the tableau in registers, 1/3 in TMEM.
template <int TR, int TC, int A, int AS, int BC, bool TWO, int MINB, bool RPC, bool TM = false>
__global__ void __launch_bounds__(TR * TC, MINB) simplex_reg_kernel(SimplexArgs a) {
  constexpr int AT = A + AS;  // rows per thread-row
  constexpr int NT = TR * TC, RCAP = TR * AT, CCAP = TC * BC, NWARP = NT / 32;
  constexpr int RPW = 32 / TC;  // thread-rows per warp
  constexpr int BH = (BC + 1) / 2;  // double2 pairs per SMEM row
  static_assert(NT % 32 == 0 && 32 % TC == 0 && TR <= 32 && AT <= 32 && BC <= 32, "layout");
  static_assert(RPW * AT <= 32, "the warp's rows must fit its lanes");
  // TMEM row slot stride: 16 columns, or 14 (exactly BC = 7 doubles: column offsets need no
  // alignment, scripts/ubench/tmem_align.cu) when 16-column slots would not fit 128 columns
  // (4 register + 9 TMEM rows for cfg2's sizes: measured 6 % slower than layout 15)
  constexpr int SLOT = AS * 16 <= 128 ? 16 : 14;
  static_assert(!TM || (!TWO && (TR * TC == 128 || TR * TC == 64) && AS * SLOT <= 128 && BC == 7),
                "TMEM layout");
  constexpr int TMCOLS = AS * SLOT <= 32 ? 32 : AS * SLOT <= 64 ? 64 : 128;  // power of two
  __shared__ RegSmem<TR, TC, AT, BC> sm;
  // TM layouts (128 registers): threadIdx.x through a volatile asm, so that the compiler
  // cannot re-read it (S2R, ~20 cycles) at every use under register pressure; the derived
  // indices are rebuilt from one register (measured: cfg2 -3.8 %; neutral elsewhere)
  int tid_;
  if constexpr (TM) asm volatile("mov.u32 %0, %%tid.x;" : "=r"(tid_));
  else tid_ = threadIdx.x;
  const int tid = tid_, lane = tid & 31, w = tid >> 5;
  const int tr = tid / TC, tc = tid - (tid / TC) * TC;
  // the row this lane serves in the warp-parallel ratio test
  const int rrow = (w * RPW + lane % RPW) + TR * (lane / RPW);
  const bool rlane = lane < RPW * AT;
  const int m = a.m, n = a.n;
#ifdef LPB_PROFILE
  const bool prof_on = a.prof != nullptr && w == 0;
  long long pacc[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  long long pt = clock64();
#endif

  double T[A][BC];
  double d2[BC];
  double d1[TWO ? BC : 1];
  // the next LP's A is prefetched into SMEM (one bulk async copy) while this LP is solved
  // (register-only layouts); with AS > 0 the dynamic SMEM holds the SMEM rows instead
  extern __shared__ __align__(16) double abuf[];
  double2* const Ts2 = reinterpret_cast<double2*>(abuf) + tid;  // [(s*BH + h) * NT]
  double* const Ts1 = abuf + 2 * tid;                             // scalar view: [s][b]
  auto ts = [&](int s_, int b_) -> double& {
    return Ts1[(size_t)((s_ * BH + (b_ >> 1)) * NT) * 2 + (b_ & 1)];
  };
  const bool pf = AS == 0 && a.prefetch != 0;
  uint32_t tbase = 0;  // this thread's TMEM lane, column 0 (TM)
  if constexpr (TM) {
    if (w == 0) tm_alloc<TMCOLS>(&sm.tmem);
    tm_fence_before();
    gsync<NT>();
    tm_fence_after();
    tbase = sm.tmem + ((uint32_t)(w * 32) << 16);
  }
  const bool direct = a.ticket == nullptr;
  const uint32_t abytes = (uint32_t)((int64_t)m * n * 8);
  uint32_t mphase = 0;
  if (tid == 0) {
    mbar_init(&sm.mbar, 1);
    // direct mode (grid = batch, no ticket): CTA b solves LP b
    const int t = direct ? (int)blockIdx.x : atomicAdd(a.ticket, 1);
    sm.lp = t;
    if (pf && t < a.batch) bulk_load(abuf, a.A + (int64_t)t * a.sA, abytes, &sm.mbar);
  }
  gsync<NT>();

  for (;;) {
    const int64_t lp = sm.lp;
    if (lp >= a.batch) break;
    const double* __restrict__ bk = a.b + lp * a.sb;
    const double* __restrict__ ck = a.c + lp * (int64_t)n;
    // issue the b and c loads before waiting for A (overlapping DRAM round trips)
    const double b_pre = (tid < m) ? __ldg(bk + tid) : 0.0;
    double c_pre[BC];
#pragma unroll
    for (int b = 0; b < BC; ++b) {
      const int p = tc + TC * b;
      c_pre[b] = (p < n) ? __ldg(ck + p) : 0.0;
    }
    if (pf) {
      mbar_wait(&sm.mbar, mphase);
      mphase ^= 1u;
    }
    const double* __restrict__ Ak = pf ? abuf : a.A + lp * a.sA;

    // ---- build: negated rows (ascending), basis keys, |b|_inf, RHS (R7) ----
    int k = 0;
    double binf = 0.0;
    for (int base = 0; base < m; base += NT) {
      const int i = base + tid;
      const double bi = (i < m) ? (base == 0 ? b_pre : __ldg(bk + i)) : 0.0;
      const bool neg = (i < m) && (bi < 0.0);
      binf = fmax(binf, fabs(bi));
      const unsigned bal = __ballot_sync(FULL, neg);
      if (lane == 0) sm.wcount[w] = __popc(bal);
      gsync<NT>();
      int off = k, tot = 0;
#pragma unroll
      for (int q = 0; q < NWARP; ++q) {
        const int cq = sm.wcount[q];
        if (q < w) off += cq;
        tot += cq;
      }
      if (neg) sm.negrows[off + __popc(bal & ((1u << lane) - 1u))] = i;
      if (i < m) {
        sm.bkey[i] = neg ? (i - m) : (n + i);
        sm.rhs[i] = neg ? -bi : bi;
      }
      k += tot;
      gsync<NT>();
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) binf = fmax(binf, __shfl_xor_sync(FULL, binf, off));
    if (lane == 0) sm.part[w].v = binf;
    gsync<NT>();
#pragma unroll
    for (int q = 0; q < NWARP; ++q) binf = fmax(binf, sm.part[q].v);
    const int npos = n + k;
    int st = (a.khint >= 0 && k > a.khint) ? ST_BAD_HINT
           : (m > RCAP || npos > CCAP || (!TWO && k > 0)) ? ST_NUMERICAL : -1;
    for (int p = tid; p < CCAP; p += NT)
      sm.nbvar[p] = (p < n) ? p : (p < npos ? n + sm.negrows[p - n] : DEADV);
    for (int i = m + tid; i < RCAP; i += NT) sm.rhs[i] = 0.0;

    // a tableau element of the build: row i (negated when b_i < 0), position p (R7)
    auto elem = [&](int i, bool rowok, bool neg, int p) -> double {
      double v = 0.0;
      if (rowok && p < npos) {
        if (p < n) {
          v = Ak[i * n + p];
          v = neg ? -v : v;
        } else {
          v = (i == sm.negrows[p - n]) ? -1.0 : (neg ? -0.0 : 0.0);
        }
      }
      return v;
    };
    if constexpr (TM) {
      // TMEM rows first, while the register rows are not live yet: the loads of G row slots
      // are in flight together (one slot at a time exposed an L2 round trip per slot; cfg2
      // -0.7 %, G = 8 spills)
      constexpr int G = 4;
#pragma unroll
      for (int s0 = 0; s0 < AS; s0 += G) {
        double vv[G][BC];
#pragma unroll
        for (int g = 0; g < G; ++g) {
          if (s0 + g < AS) {
            const int i = tr + TR * (A + s0 + g);
            const bool rowok = (i < m) && st < 0;
            const bool neg = rowok && sm.bkey[i] < 0;
#pragma unroll
            for (int b = 0; b < BC; ++b) vv[g][b] = elem(i, rowok, neg, tc + TC * b);
          }
        }
#pragma unroll
        for (int g = 0; g < G; ++g) {
          if (s0 + g < AS) {
            uint32_t cell[2 * BC];
#pragma unroll
            for (int b = 0; b < BC; ++b) tm_split(vv[g][b], cell[2 * b], cell[2 * b + 1]);
            tm_st14(tbase + SLOT * (s0 + g), cell);
          }
        }
      }
    }
#pragma unroll
    for (int ai = 0; ai < A; ++ai) {
      const int i = tr + TR * ai;
      const bool rowok = (i < m) && st < 0;
      const bool neg = rowok && sm.bkey[i] < 0;
#pragma unroll
      for (int b = 0; b < BC; ++b) T[ai][b] = elem(i, rowok, neg, tc + TC * b);
    }
#pragma unroll
    for (int s_ = 0; s_ < (TM ? 0 : AS); ++s_) {  // SMEM rows (non-TM layouts with AS > 0)
      const int i = tr + TR * (A + s_);
      const bool rowok = (i < m) && st < 0;
      const bool neg = rowok && sm.bkey[i] < 0;
      uint32_t cell[TM ? 2 * BC : 1];
#pragma unroll
      for (int b = 0; b < BC; ++b) {
        const double v = elem(i, rowok, neg, tc + TC * b);
        if constexpr (TM) tm_split(v, cell[2 * b], cell[2 * b + 1]);
        else ts(s_, b) = v;
      }
      if constexpr (TM) {
        tm_st14(tbase + SLOT * s_, cell);
      }
    }
    if constexpr (TM) tm_wait_st();
    // padding positions (and, later, dead artificial positions) hold -inf in the objective
    // replicas: never a Step-1 candidate, and fma(f, p, -inf) keeps them -inf
#pragma unroll
    for (int b = 0; b < BC; ++b) {
      const int p = tc + TC * b;
      d2[b] = (p < n) ? c_pre[b] : (p < npos ? 0.0 : neg_inf());
    }
    double z2 = 0.0, z1 = 0.0;
    if constexpr (TWO) {
      // phase-I row: ascending-row sums of the negated rows, computed once by thread-row 0
      // into SMEM scratch, then replicated into every thread's positions
      if (k > 0 && st < 0) {
        if (tr == 0) {
          for (int p = tc; p < npos; p += TC) {
            double acc = 0.0;
            for (int t = 0; t < k; ++t) {
              const int r = sm.negrows[t];
              const double v = (p < n) ? -Ak[r * n + p]
                                       : ((r == sm.negrows[p - n]) ? -1.0 : -0.0);
              acc = __dadd_rn(acc, v);
            }
            sm.prow[p] = acc;
          }
        }
        gsync<NT>();
#pragma unroll
        for (int b = 0; b < BC; ++b) {
          const int p = tc + TC * b;
          d1[b] = (p < npos) ? sm.prow[p] : neg_inf();
        }
        for (int t = 0; t < k; ++t) z1 = __dadd_rn(z1, sm.rhs[sm.negrows[t]]);
      } else {
#pragma unroll
        for (int b = 0; b < BC; ++b) d1[b] = neg_inf();
      }
    }
    gsync<NT>();  // A has been consumed: the buffer may be refilled with the next LP
    if (tid == 0) {
      const int t = direct ? (int)a.batch : atomicAdd(a.ticket, 1);
      sm.lp = t;
      if (pf && t < a.batch) bulk_load(abuf, a.A + (int64_t)t * a.sA, abytes, &sm.mbar);
      // layouts without the SMEM prefetch buffer (TMEM / SMEM rows): the next LP's A is
      // bulk-prefetched into L2 instead, so its build reads hit L2 rather than HBM (ncu
      // r02f: 19 % of cfg2's stall samples were the build's A loads; cfg2 -3.4 %, cfg10 -6.8 %)
      if (AS > 0 && a.prefetch && t < a.batch)
        bulk_prefetch_l2(a.A + (int64_t)t * a.sA, abytes);
    }

    // ---- Steps 1-3, two phases ----
    int it1 = 0, it2 = 0, stall = 0, phase = (TWO && k > 0) ? 1 : 2;
    int par = 0, l_prev = -1, dl = 0;
    double prr_prev = 0.0;  // RHS of the last pivot row (lazy RHS updates, R13)
    const uint64_t lpkey = RPC ? rpc_lp_key(a.rpc_seed, a.lp_base + lp) : 0ull;
    bool pend = false, drive = false;
    bool pre = false;  // Step 1 of this pivot was computed at the end of the last update
    int pre_wl = -1, pre_e = 0, pre_evar = 0;
    while (st < 0) {
      const bool bland = a.bland_K > 0 && stall >= a.bland_K;
      const bool p1 = TWO && phase == 1;
      int e = -1, evar = 0, l = -1;
      if (drive) {
        // phase switch (R9): drive the next basic artificial out on max |T[l][p]|
        while (dl < m && sm.bkey[dl] >= 0) ++dl;
        if (dl >= m) {
          drive = false;
          phase = 2;
          stall = 0;
          continue;
        }
        l = dl++;
        bool val = false;
        double bv = 0.0;
        unsigned bvar = 0;
        int bp = -1;
        if (tr == l % TR) {
          const int al = l / TR;
#pragma unroll
          for (int b = 0; b < BC; ++b) {
            double v = T[0][b];
#pragma unroll
            for (int ai = 1; ai < A; ++ai) v = (ai == al) ? T[ai][b] : v;
            if (AS > 0 && al >= A) v = ts(al - A, b);
            v = fabs(v);
            if (d2[b] != neg_inf() && v > a.eps_piv) {  // live position
              const int p = tc + TC * b;
              const unsigned var = (unsigned)sm.nbvar[p];
              if (!val || v > bv || (v == bv && var < bvar)) {
                val = true;
                bv = v;
                bvar = var;
                bp = p;
              }
            }
          }
        }
        const int wl = warp_argmax(val, okey(bv), bvar);
        Part pw{0.0, INT_MAX, -1};
        if (wl >= 0) {
          pw.v = __shfl_sync(FULL, bv, wl);
          pw.tie = (int)__shfl_sync(FULL, bvar, wl);
          pw.idx = __shfl_sync(FULL, bp, wl);
        }
        if (lane == 0) sm.part[w] = pw;
        gsync<NT>();
        const Part q = (lane < NWARP) ? sm.part[lane] : Part{0.0, INT_MAX, -1, 1.0};
        const int ql = warp_argmax(q.idx >= 0, okey(q.v), (unsigned)q.tie);
        gsync<NT>();
        if (ql < 0) continue;  // redundant row: the artificial stays basic at 0
        e = __shfl_sync(FULL, q.idx, ql);
        evar = __shfl_sync(FULL, q.tie, ql);
      } else if (pre) {  // Step 1 done at the end of the last update (same rule and order)
        pre = false;
        if (pre_wl < 0) {
          if (phase == 2) { st = ST_OPTIMAL; break; }
          if (z1 > a.eps_phase1 * fmax(1.0, binf)) { st = ST_INFEASIBLE; break; }
          drive = true;  // phase-I optimum with w* ~ 0
          dl = 0;
          continue;
        }
        if (it1 + it2 >= a.max_iter) { st = ST_ITER_LIMIT; break; }
        e = pre_e;
        evar = pre_evar;
      } else {
        LPB_PROF_MARK(7)
        // Step 1: entering position from the replicated objective row (warp-local)
        double bv = neg_inf();
        int bb = 0;
        unsigned bvar = 0;
        bool val;
        const bool rpc = RPC && !bland;  // a separate instantiation keeps LPC's registers
        unsigned long long ukey = 0ull;
        if (rpc) {  // RPC: the candidate with the largest counter-based score (lpb_rng.cuh)
          val = false;
          bvar = 0xffffffffu;
          const uint64_t pkey = rpc_pivot_key(lpkey, it1 + it2);
#pragma unroll
          for (int b = 0; b < BC; ++b) {
            const double v = p1 ? d1[TWO ? b : 0] : d2[b];
            if (v > a.eps_enter) {
              const unsigned var = (unsigned)sm.nbvar[tc + TC * b];
              const unsigned long long u = rpc_score(pkey, (int)var);
              if (!val || u > ukey || (u == ukey && var < bvar)) {
                val = true;
                ukey = u;
                bvar = var;
                bb = b;
              }
            }
          }
        } else if (!bland) {
#pragma unroll
          for (int b = 0; b < BC; ++b) {
            const double v = p1 ? d1[TWO ? b : 0] : d2[b];
            const bool take = v > bv;  // first maximum: lowest b on ties (fixed below)
            bv = take ? v : bv;
            bb = take ? b : bb;
          }
          val = bv > a.eps_enter;
          bool tie = false;
#pragma unroll
          for (int b = 0; b < BC; ++b) {
            const double v = p1 ? d1[TWO ? b : 0] : d2[b];
            tie |= (b != bb) && (v == bv);
          }
          bvar = val ? (unsigned)sm.nbvar[tc + TC * bb] : 0u;
          if (__any_sync(FULL, val && tie)) {  // rare: exact tie inside a thread -> var index
            if (val && tie) {
#pragma unroll
              for (int b = 0; b < BC; ++b) {
                const double v = p1 ? d1[TWO ? b : 0] : d2[b];
                const unsigned var = (unsigned)sm.nbvar[tc + TC * b];
                if (v == bv && var < bvar) {
                  bvar = var;
                  bb = b;
                }
              }
            }
          }
        } else {  // Bland: the lowest variable index with d > eps_enter
          val = false;
          bvar = 0xffffffffu;
#pragma unroll
          for (int b = 0; b < BC; ++b) {
            const double v = p1 ? d1[TWO ? b : 0] : d2[b];
            if (v > a.eps_enter) {
              const unsigned var = (unsigned)sm.nbvar[tc + TC * b];
              if (var < bvar) {
                bvar = var;
                bb = b;
                bv = v;
                val = true;
              }
            }
          }
        }
        // the RPW thread-rows of a warp hold identical replicas: only the first one competes,
        // so a unique maximum takes warp_argmax's single-REDUX fast path
        val = val && (RPW == 1 || lane < TC);
        const int wl = bland ? warp_argmin(val, 0ull, bvar)
                             : warp_argmax(val, rpc ? ukey : okey(bv), bvar);
        if (wl < 0) {
          if (phase == 2) { st = ST_OPTIMAL; break; }
          if (z1 > a.eps_phase1 * fmax(1.0, binf)) { st = ST_INFEASIBLE; break; }
          drive = true;  // phase-I optimum with w* ~ 0
          dl = 0;
          continue;
        }
        if (it1 + it2 >= a.max_iter) { st = ST_ITER_LIMIT; break; }
        e = __shfl_sync(FULL, tc + TC * bb, wl);
        evar = (int)__shfl_sync(FULL, bvar, wl);
      }

      LPB_PROF_MARK(0)
      // Step 2a: the owners of position e publish column e (+ objective-row entries)
      const int be = e / TC, etc = e - be * TC;
      double* colE = sm.colE[par];
      if (tc == etc) {
#define LPB_PUB(x)                                                                    \
  case x:                                                                             \
    if constexpr ((x) < BC) {                                                         \
      _Pragma("unroll") for (int ai = 0; ai < A; ++ai) {                             \
        colE[tr + TR * ai] = T[ai][x];                                                \
        T[ai][x] = 0.0;                                                               \
      }                                                                               \
      if (tr == 0) {                                                                  \
        sm.fobj[par][0] = d2[x];                                                      \
        if constexpr (TWO) sm.fobj[par][1] = d1[x];                                   \
      }                                                                               \
      d2[x] = 0.0;                                                                    \
      if constexpr (TWO) d1[x] = 0.0;                                                 \
    }                                                                                 \
    break;
        switch (be) { LPB_CASES(LPB_PUB) default: break; }
#undef LPB_PUB
        if constexpr (!TM) {
#pragma unroll
          for (int s_ = 0; s_ < AS; ++s_) {  // SMEM rows: dynamic position index
            double& t = ts(s_, be);
            colE[tr + TR * (A + s_)] = t;
            t = 0.0;
          }
        }
      }
      if constexpr (TM) {  // TMEM rows: the whole warp loads column be, the owners publish it
        uint32_t lo[AS > 0 ? AS : 1], hi[AS > 0 ? AS : 1];
#pragma unroll
        for (int s_ = 0; s_ < AS; ++s_) tm_ld2(tbase + SLOT * s_ + 2 * be, lo[s_], hi[s_]);
        tm_wait_ld();
        const bool own = tc == etc;
#pragma unroll
        for (int s_ = 0; s_ < AS; ++s_) {
          if (own) colE[tr + TR * (A + s_)] = tm_d(lo[s_], hi[s_]);
          tm_st2(tbase + SLOT * s_ + 2 * be, own ? 0u : lo[s_], own ? 0u : hi[s_]);
        }
        tm_wait_st();  // the pivot-row load below may read these columns
      }
      __syncwarp();
      LPB_PROF_MARK(1)
      // Step 2b: lane-parallel lazy RHS update + ratio test over the warp's rows; each lane
      // also writes its row's update multiplier f_i = -colE_i
      {
        bool val = false;
        double ratio = 0.0;
        double rc = 1.0;
        int tie = INT_MAX;
        const int i = rrow;
        if (rlane) {
          const double v = colE[i];
          sm.fcol[par][i] = -v;
          if (i < m) {
            double r = sm.rhs[i];
            if (pend) {
              r = (i == l_prev) ? prr_prev : __fma_rn(sm.fcol[par ^ 1][i], prr_prev, r);
              sm.rhs[i] = r;
            }
            if (!drive) {
              val = v > a.eps_piv;
              bool slow;
              rc = recip_of(val ? v : 1.0);
              ratio = div_with(r, val ? v : 1.0, rc, slow);  // == div_fast(r, v)
              if (slow) ratio = ddiv_slow(r, val ? v : 1.0);  // rare: outside the fast range
              tie = bland ? sm.bkey[i] : i;
            }
          }
        }
        if (!drive) {
          // the winning lane writes the warp's partial itself (no shuffles)
          const int wl = warp_argmin(val, okey(ratio), ikey(tie));
          if (lane == (wl < 0 ? 0 : wl)) sm.part[w] = wl < 0 ? Part{0.0, INT_MAX, -1, 1.0}
                                                             : Part{ratio, tie, i, rc};
        }
      }
      LPB_PROF_MARK(2)
      gsync<NT>();  // barrier 1
      LPB_PROF_MARK(3)
      double theta = 0.0;
      double qrc = 1.0;
      if (!drive) {  // Step 2c: the NWARP warp partials
        if constexpr (NWARP >= 4) {
          // lanes < NWARP hold one partial each; the same (ratio, tie) argmin by REDUX
          // (measured: cfg2 -0.6 %; with 2 warps the serial compare is shorter)
          Part q = (lane < NWARP) ? sm.part[lane] : Part{0.0, INT_MAX, -1, 1.0};
          const int ql = warp_argmin(q.idx >= 0, okey(q.v), ikey(q.tie));
          if (ql < 0) { st = (phase == 2) ? ST_UNBOUNDED : ST_NUMERICAL; break; }
          l = __shfl_sync(FULL, q.idx, ql);
          theta = __shfl_sync(FULL, q.v, ql);
          qrc = __shfl_sync(FULL, q.rc, ql);
        } else {  // every thread scans the partials (ascending warp)
          Part q = sm.part[0];
#pragma unroll
          for (int u = 1; u < NWARP; ++u) {
            const Part o = sm.part[u];
            // (ratio, tie) order of warp_argmin: IEEE compare (-0 == +0), then the smaller key
            if (o.idx >= 0 && (q.idx < 0 || o.v < q.v || (o.v == q.v && o.tie < q.tie))) q = o;
          }
          if (q.idx < 0) { st = (phase == 2) ? ST_UNBOUNDED : ST_NUMERICAL; break; }
          l = q.idx;
          theta = q.v;
          qrc = q.rc;
        }
      }

      LPB_PROF_MARK(4)
      // Step 3 (Listing 1): the owners of row l publish the RAW row (position
      // e carries 1, the leaving variable's column) and zero their copy; after barrier 2
      // every thread divides its own positions by PE (one reciprocal, taken before the
      // barrier), so no single warp holds the others on the divisions and the owner-only
      // code stays a few stores per case.
      const double pe = colE[l];
      if (tid == 0) {
        const int lv = sm.bkey[l];
        sm.bkey[l] = evar;
        sm.nbvar[e] = lv >= 0 ? lv : DEADV;
        sm.leaving = lv;
        sm.fcol[par][l] = 1.0;  // the pivot row: fma(1, prow, 0) = prow
      }
      const int ltr = l % TR, al = l / TR;
      if (tr == ltr) {
#define LPB_PROW(x)                                                                 \
  case x:                                                                           \
    if constexpr ((x) < A) {                                                        \
      _Pragma("unroll") for (int b = 0; b < BC; ++b) {                              \
        sm.prow[tc + TC * b] = (tc + TC * b == e) ? 1.0 : T[x][b];                  \
        T[x][b] = 0.0;                                                              \
      }                                                                             \
    }                                                                               \
    break;
        switch (al) { LPB_CASES(LPB_PROW) default: break; }
#undef LPB_PROW
        if (!TM && AS > 0 && al >= A) {  // pivot row in SMEM
          const int s_ = al - A;
#pragma unroll
          for (int b = 0; b < BC; ++b) {
            sm.prow[tc + TC * b] = (tc + TC * b == e) ? 1.0 : ts(s_, b);
            ts(s_, b) = 0.0;
          }
        }
      }
      if constexpr (TM) {
        if (al >= A) {  // pivot row in TMEM (warp-uniform): whole-warp load, owners publish
          const int s_ = al - A;
          uint32_t cell[14];
          tm_ld14(tbase + SLOT * s_, cell);
          tm_wait_ld();
          const bool own = tr == ltr;
#pragma unroll
          for (int b = 0; b < BC; ++b) {
            if (own) sm.prow[tc + TC * b] = (tc + TC * b == e) ? 1.0 : tm_d(cell[2 * b], cell[2 * b + 1]);
            cell[2 * b] = own ? 0u : cell[2 * b];
            cell[2 * b + 1] = own ? 0u : cell[2 * b + 1];
          }
          tm_st14(tbase + SLOT * s_, cell);
          tm_wait_st();
        }
      }
      const double rpe = drive ? recip_of(pe) : qrc;  // the winning ratio lane's reciprocal
      const double rhs_l = sm.rhs[l];  // current: its lane applied the lazy update in Step 2b
      LPB_PROF_MARK(5)
      gsync<NT>();  // barrier 2
      LPB_PROF_MARK(6)
      {
        const int leaving = sm.leaving;
        double pv[BC];
        double prr;
        // the RPW thread-rows of a warp hold the same positions: each divides every RPW-th of
        // the BC positions and the RHS (g = k*RPW + group), and the quotients travel by
        // shuffle from the lane with the same tc in the owning group
        constexpr int QN = (BC + 1 + RPW - 1) / RPW;
        const int grp = lane / TC;
        double q[QN];
        bool sl_any = false;
#pragma unroll
        for (int k = 0; k < QN; ++k) {
          const int g = k * RPW + grp;
          const double raw = (g < BC) ? sm.prow[tc + TC * (g < BC ? g : 0)] : rhs_l;
          bool sl;
          q[k] = div_with(raw, pe, rpe, sl);
          sl_any |= sl && g <= BC;
        }
#pragma unroll
        for (int b = 0; b <= BC; ++b) {
          const double v = __shfl_sync(FULL, q[b / RPW], (lane % TC) + TC * (b % RPW));
          if (b < BC) pv[b] = v;
          else prr = v;
        }
        if (__any_sync(FULL, sl_any)) {  // rare: outside div_with's fast range -> IEEE __ddiv_rn
#pragma unroll
          for (int b = 0; b < BC; ++b) pv[b] = ddiv_slow(sm.prow[tc + TC * b], pe);
          prr = ddiv_slow(rhs_l, pe);
        }
        prr_prev = prr;
        const double f2 = -sm.fobj[par][0];
        const bool upd1 = TWO && phase == 1;
        const double f1 = TWO ? -sm.fobj[par][1] : 0.0;
#pragma unroll
        for (int b = 0; b < BC; ++b) {
          d2[b] = __fma_rn(f2, pv[b], d2[b]);
          if constexpr (TWO) {
            if (upd1) d1[b] = __fma_rn(f1, pv[b], d1[b]);
          }
        }
        z2 = __fma_rn(f2, prr, z2);
        if constexpr (TWO) {
          if (upd1) z1 = __fma_rn(f1, prr, z1);
        }
        // Row l and position e were zeroed when they were read (Step 2a / Step 3), so one
        // fma per element yields the pivot row (f_l = 1: fma(1, prow, 0) = prow) and the
        // leaving variable's column (fma(-f_i, rl, 0)) without any per-element branch.
#pragma unroll
        for (int ai = 0; ai < A; ++ai) {
          const double fi = sm.fcol[par][tr + TR * ai];
#pragma unroll
          for (int b = 0; b < BC; ++b) T[ai][b] = __fma_rn(fi, pv[b], T[ai][b]);
        }
        if constexpr (TM) {  // TMEM rows: load, fma, store one slot at a time
          // each slot's 2 BC = 14 columns as x8 + x4 + x2 accesses: with x16 tuples ptxas loads
          // each slot into a second tuple and copies it (16 moves per slot) and spills (316
          // bytes).  Measured slower: the next slot's load issued before this
          // slot's fmas (2 or 3 rotating buffers: +12 %, spills), 4 + 9 rows in 14-column slots
#pragma unroll
          for (int s_ = 0; s_ < AS; ++s_) {
            const double fi = sm.fcol[par][tr + TR * (A + s_)];
            uint32_t cell[14];
            tm_ld14(tbase + SLOT * s_, cell);
            tm_wait_ld();
#pragma unroll
            for (int b = 0; b < BC; ++b)
              tm_split(__fma_rn(fi, pv[b], tm_d(cell[2 * b], cell[2 * b + 1])), cell[2 * b],
                       cell[2 * b + 1]);
            tm_st14(tbase + SLOT * s_, cell);
          }
          tm_wait_st();
        }
#pragma unroll
        for (int s_ = 0; s_ < (TM ? 0 : AS); ++s_) {  // SMEM rows, two positions per 128-bit access
          const double fi = sm.fcol[par][tr + TR * (A + s_)];
#pragma unroll
          for (int h = 0; h < BH; ++h) {
            double2 v = Ts2[(s_ * BH + h) * NT];
            v.x = __fma_rn(fi, pv[2 * h], v.x);
            if (2 * h + 1 < BC) v.y = __fma_rn(fi, pv[(2 * h + 1 < BC) ? 2 * h + 1 : 0], v.y);
            Ts2[(s_ * BH + h) * NT] = v;
          }
        }
        if constexpr (TWO) {  // an artificial left: position e is dead (-inf), branch-free
          const bool dead = leaving < 0 && tc == etc;
#pragma unroll
          for (int b = 0; b < BC; ++b) {
            const bool z = dead && b == be;
            d2[b] = z ? neg_inf() : d2[b];
            d1[b] = z ? neg_inf() : d1[b];
          }
        }
        // Step 1 of the NEXT pivot (LPC or RPC, no Bland), straight-line in the same block as
        // the update's DFMAs so the compiler fills its latency chain with them; the loop head
        // uses the result when the next pivot is not a Bland pivot (pre).
        {
          const bool p1n = TWO && phase == 1;
          // RPC: the next pivot's draw is keyed on the pivot count after this pivot
          const uint64_t pkey = RPC ? rpc_pivot_key(lpkey, it1 + it2 + 1) : 0ull;
          double bv = neg_inf();
          unsigned long long bu = 0ull;
          bool bval = false;
          int bb = 0;
          unsigned bvar = 0xffffffffu;
          if constexpr (!RPC) {
            // the first maximum over b, then this thread's variable at it; an exact tie
            // inside a thread (rare) redoes the scan with the variable-index rule
#pragma unroll
            for (int b = 0; b < BC; ++b) {
              const double v = p1n ? d1[TWO ? b : 0] : d2[b];
              const bool take = v > bv;
              bv = take ? v : bv;
              bb = take ? b : bb;
            }
            int neq = 0;
#pragma unroll
            for (int b = 0; b < BC; ++b) neq += ((p1n ? d1[TWO ? b : 0] : d2[b]) == bv);
            bvar = (unsigned)sm.nbvar[tc + TC * bb];
            if (__any_sync(FULL, neq > 1 && bv > a.eps_enter)) {
              bv = neg_inf();
              bvar = 0xffffffffu;
#pragma unroll
              for (int b = 0; b < BC; ++b) {
                const double v = p1n ? d1[TWO ? b : 0] : d2[b];
                const unsigned var = (unsigned)sm.nbvar[tc + TC * b];
                const bool take = v > bv || (v == bv && var < bvar);
                bv = take ? v : bv;
                bb = take ? b : bb;
                bvar = take ? var : bvar;
              }
            }
          } else {
#pragma unroll
          for (int b = 0; b < BC; ++b) {
            const double v = p1n ? d1[TWO ? b : 0] : d2[b];
            const unsigned var = (unsigned)sm.nbvar[tc + TC * b];
            bool take;
            if constexpr (RPC) {
              const bool cand = v > a.eps_enter;
              const unsigned long long u = rpc_score(pkey, (int)var);
              take = cand && (!bval || u > bu || (u == bu && var < bvar));
              bu = take ? u : bu;
              bval = bval || cand;
            } else {
              take = v > bv || (v == bv && var < bvar);
              bv = take ? v : bv;
            }
            bb = take ? b : bb;
            bvar = take ? var : bvar;
          }
          }
          const bool val = (RPC ? bval : bv > a.eps_enter) && (RPW == 1 || lane < TC);
          const unsigned long long key = RPC ? bu : okey(bv);
          // branch-free (key, variable) warp argmax: three REDUX steps
          const unsigned hi = val ? (unsigned)(key >> 32) : 0u;
          const unsigned mhi = __reduce_max_sync(FULL, hi);
          const bool c1 = val && hi == mhi;
          const unsigned lo = c1 ? (unsigned)key : 0u;
          const unsigned mlo = __reduce_max_sync(FULL, lo);
          const bool c2 = c1 && (unsigned)key == mlo;
          const unsigned mt = __reduce_min_sync(FULL, c2 ? bvar : 0xffffffffu);
          const unsigned win = __ballot_sync(FULL, c2 && bvar == mt);
          pre_wl = win ? __ffs(win) - 1 : -1;
          pre_e = __shfl_sync(FULL, tc + TC * bb, pre_wl & 31);
          pre_evar = (int)__shfl_sync(FULL, bvar, pre_wl & 31);
        }
      }
      LPB_PROF_MARK(8)
      pend = true;
      l_prev = l;
      par ^= 1;
      if (drive) {
        ++it1;
        pre = false;
        gsync<NT>();  // the next drive-out scan reads bkey
      } else {
        if (phase == 1) ++it1; else ++it2;
        stall = (theta > 0.0) ? 0 : stall + 1;
        pre = !(a.bland_K > 0 && stall >= a.bland_K);
      }
    }

    // ---- extract (R10) ----
    gsync<NT>();
    if (st == ST_OPTIMAL && pend) {  // apply the last pending RHS update
      for (int i = tid; i < m; i += NT)
        sm.rhs[i] = (i == l_prev) ? prr_prev
                                  : __fma_rn(sm.fcol[par ^ 1][i], prr_prev, sm.rhs[i]);
    }
    if (tid == 0) {
      a.status[lp] = st;
      a.iters[2 * lp] = it1;
      a.iters[2 * lp + 1] = it2;
      a.obj[lp] = (st == ST_OPTIMAL) ? -z2
                : (st == ST_UNBOUNDED) ? pos_inf() : (st == ST_INFEASIBLE) ? neg_inf() : qnan();
    }
    if (a.x) {
      double* xk = a.x + lp * (int64_t)n;
      const double fill = (st == ST_OPTIMAL) ? 0.0 : qnan();
      for (int j = tid; j < n; j += NT) xk[j] = fill;
      gsync<NT>();
      if (st == ST_OPTIMAL)
        for (int i = tid; i < m; i += NT) {
          const int key = sm.bkey[i];
          if (key >= 0 && key < n) xk[key] = sm.rhs[i];
        }
    }
    gsync<NT>();
  }
  if constexpr (TM) {
    tm_fence_before();
    gsync<NT>();
    tm_fence_after();
    if (w == 0) tm_dealloc<TMCOLS>(sm.tmem);
  }
#ifdef LPB_PROFILE
  if (prof_on && lane == 0)
    for (int q = 0; q < 12; ++q)
      atomicAdd((unsigned long long*)&a.prof[blockIdx.x * 12 + q], (unsigned long long)pacc[q]);
#endif
}

struct RegCfg {
  int rcap, ccap, two, id;
};

// Instantiated layouts: {id, TR, TC, A (register rows), AS (SMEM rows), BC, TWO, MINB}.
// (An AS > 0 layout with 3 LPs/SM, {8,16,7,6,7,false,3}, is correct but measured 15% slower
// than {8,16,13,0,7} on cfg2: 1.63e6 vs 1.92e6 LPs/s; none is instantiated by default.)
#define LPB_REG_CONFIGS(X)              \
  X(0, 8, 4, 1, 0, 3, true, 16)         \
  X(1, 8, 4, 2, 0, 6, true, 12)         \
  X(2, 8, 4, 4, 0, 8, true, 6)          \
  X(8, 8, 8, 7, 0, 7, false, 4)         \
  X(9, 8, 8, 7, 0, 7, true, 4)          \
  X(10, 8, 8, 8, 0, 8, false, 4)        \
  X(11, 8, 8, 8, 0, 8, true, 4)         \
  X(6, 8, 16, 13, 0, 7, false, 2)       \
  X(4, 16, 16, 7, 0, 7, false, 1)       \
  X(5, 16, 16, 7, 0, 7, true, 1)
// TMEM layouts (TM = true): A register rows + AS rows in tensor memory.  Layout 15 replaces
// layout 6 (type-1 LPs up to 104 x 112, cfg2): 5 of each thread's 13 rows in registers, 8 in
// TMEM (8 x 16 columns), 128 registers, FOUR CTAs (LPs) per SM instead of two.  Measured on
// cfg2: 4 LPs/SM 19.7 ms (then 19.0 with the tid register) vs 20.4 ms for layout 6; 3 LPs/SM
// with 8 or 5 register rows: 21.4 / 23.4 ms.  Layout 17 replaces layout 8 (up to 56 x 56,
// cfg10): 3 + 4 rows, 64-thread CTAs with 64 TMEM columns each, EIGHT LPs per SM instead of
// four (TMEM's 512 columns are the limit): cfg10 3.47 -> 2.95 ms.
#define LPB_REG_TM_CONFIGS(X)           \
  X(15, 8, 16, 5, 8, 7, false, 4)       \
  X(17, 8, 8, 3, 4, 7, false, 8)

template <int TR, int TC, int A, int AS, int BC, bool TWO, int MINB, bool RPC, bool TM = false>
cudaError_t launch_one(const SimplexArgs& a, int grid_override, cudaStream_t s, int* ctas) {
  auto kern = simplex_reg_kernel<TR, TC, A, AS, BC, TWO, MINB, RPC, TM>;
  const size_t dsm = TM ? 0
                   : AS > 0 ? (size_t)AS * ((BC + 1) / 2) * TR * TC * 16
                            : (a.prefetch ? (size_t)a.m * a.n * 8 : 0);
  // attribute + occupancy queries are host round trips: cache them per (device, smem size)
  static LaunchMemo memo;
  int per_sm = 0;
  const cudaError_t em = memo.get(dsm, &per_sm, [&](int& v, size_t attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)attr);
    if (e != cudaSuccess) return e;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, kern, TR * TC, dsm);
  });
  if (em != cudaSuccess) return em;
  // TMEM layouts: the occupancy query reports 1 CTA/SM for tcgen05 kernels; MINB CTAs are
  // co-resident (registers) and their TMEM columns (MINB x 128 <= 512) fit
  if (TM) per_sm = MINB;
  int64_t grid = (int64_t)(per_sm < 1 ? 1 : per_sm) * device_sm_count();
  SimplexArgs d = a;
  if (a.batch <= grid && grid_override <= 0) {
    d.ticket = nullptr;  // one resident wave: CTA b solves LP b, no ticket round trips
    grid = a.batch;
  }
  if (grid > a.batch) grid = a.batch;
  if (grid_override > 0) grid = grid_override;
  if (ctas) *ctas = (int)grid;
  if (d.ticket) {  // persistent launch: zero the LP ticket (direct launches need none)
    const cudaError_t e = cudaMemsetAsync(d.ticket, 0, sizeof(int), s);
    if (e != cudaSuccess) return e;
  }
  kern<<<(unsigned)grid, TR * TC, dsm, s>>>(d);
  return cudaGetLastError();
}

}  // namespace

static const RegCfg kCfgs[] = {
#define X(id, TR, TC, A, AS, BC, TWO, MINB) {TR * (A + AS), TC * BC, TWO ? 1 : 0, id},
    LPB_REG_CONFIGS(X)
#undef X
};
static const RegCfg kTmCfgs[] = {
#define X(id, TR, TC, A, AS, BC, TWO, MINB) {TR * (A + AS), TC * BC, TWO ? 1 : 0, id},
    LPB_REG_TM_CONFIGS(X)
#undef X
};

static int pick_cfg(int m, int n, int kmax) {
#ifdef LPB_DEV_HOOKS
  // experiment hook (development build): LPB_REG_CFG=<id> forces one layout when it fits
  if (const char* f = getenv("LPB_REG_CFG")) {
    const int id = atoi(f);
    for (const RegCfg& c : kCfgs)
      if (c.id == id && m <= c.rcap && n + kmax <= c.ccap && (kmax == 0 || c.two)) return id;
    for (const RegCfg& c : kTmCfgs)
      if (c.id == id && m <= c.rcap && n + kmax <= c.ccap && (kmax == 0 || c.two)) return id;
  }
#endif
  for (const RegCfg& c : kCfgs) {
    if (m > c.rcap || n + kmax > c.ccap) continue;
    if (kmax > 0 && !c.two) continue;
    // layout 6's sizes run on the TMEM layout 15 (same capacity, 4 LPs/SM instead of 2),
    // layout 8's on layout 17 (same capacity, 8 LPs/SM instead of 4)
    if (c.id == 6 && !dev_flag("LPB_NO_TMEM")) return 15;
    if (c.id == 8 && !dev_flag("LPB_NO_TMEM")) return 17;
    return c.id;
  }
  return -1;
}

bool reg_fits(int m, int n, int kmax) { return pick_cfg(m, n, kmax) >= 0; }

int reg_layout(int m, int n, int kmax) { return pick_cfg(m, n, kmax); }

cudaError_t launch_simplex_reg(const SimplexArgs& a, int grid_override, cudaStream_t s,
                               int* ctas_out) {
  switch (pick_cfg(a.m, a.n, a.kmax)) {
#define X(id, TR, TC, A, AS, BC, TWO, MINB) \
  case id:                                                                        \
    return a.rpc ? launch_one<TR, TC, A, AS, BC, TWO, MINB, true>(a, grid_override, s, ctas_out) \
                 : launch_one<TR, TC, A, AS, BC, TWO, MINB, false>(a, grid_override, s, ctas_out);
    LPB_REG_CONFIGS(X)
#undef X
#define X(id, TR, TC, A, AS, BC, TWO, MINB) \
  case id:                                                                        \
    return a.rpc ? launch_one<TR, TC, A, AS, BC, TWO, MINB, true, true>(a, grid_override, s, ctas_out) \
                 : launch_one<TR, TC, A, AS, BC, TWO, MINB, false, true>(a, grid_override, s, ctas_out);
    LPB_REG_TM_CONFIGS(X)
#undef X
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace lpb
