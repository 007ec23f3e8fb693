// simplex_warp.cu — W class: one LP per WARP for small LPs (up to 32 x 32 condensed), the
// tableau in registers and every exchange a warp shuffle (no shared memory, no barrier).
//
// Same method and arithmetic as the oracle (§3.1 Steps 1-3, Listing 1; two-phase
// PAPER.md:76; readings R1-R15 in DESIGN.md), laid out for latency: a small LP's pivot is a
// chain of dependent steps, so each step is the shortest exchange that does it.
//   * lane = (tr, tc) with tr = lane / 4 (8 thread-rows), tc = lane % 4 (4 thread-cols);
//     lane owns rows i = tr + 8a (a < A) and positions p = tc + 4b (b < BC) of the condensed
//     tableau; the objective row(s) are replicated per thread-row (d2, d1); lane L owns row L
//     for the ratio test (its RHS and basic-variable key live in its registers);
//   * Step 1: a register scan on the 4 lanes of thread-row 0 + a REDUX warp argmax;
//   * column e: its owner lanes pick T[.][e] with a uniform switch and the ratio lanes and
//     update multipliers fetch it with A shuffles; the ratio test is one IEEE division per
//     lane + a REDUX warp argmin;
//   * pivot row l: picked with a uniform switch, BC shuffles bring each lane its positions;
//     every lane divides its own positions by PE and applies fma(f_i, prow_p, T_ip).
// One warp (LP) per CTA: 32-thread CTAs let the register file hold the most LPs per SM.
#include <climits>

#include "lpb_fp64.cuh"
#include "lpb_internal.cuh"
#include "lpb_reduce.cuh"
#include "lpb_rng.cuh"

namespace lpb {
namespace {

constexpr unsigned WFULL = 0xffffffffu;
constexpr int W_WARPS = 1;  // LPs (warps) per CTA: a 32-thread CTA packs the SM to its register limit
constexpr int DEADW = INT_MAX;

__device__ __forceinline__ double w_neg_inf() {
  return __longlong_as_double(0xfff0000000000000ll);
}

// warp argmax of (64-bit key desc, tie asc) over valid lanes, branch-free; -1 if none
__device__ __forceinline__ int w_argmax(bool valid, unsigned long long key, unsigned tie) {
  const unsigned hi = valid ? (unsigned)(key >> 32) : 0u;
  const unsigned mhi = __reduce_max_sync(WFULL, hi);
  const bool c1 = valid && hi == mhi;
  LPB_FIRST_LANE(c1, -1)
  const unsigned lo = c1 ? (unsigned)key : 0u;
  const unsigned mlo = __reduce_max_sync(WFULL, lo);
  const bool c2 = c1 && (unsigned)key == mlo;
  const unsigned mt = __reduce_min_sync(WFULL, c2 ? tie : 0xffffffffu);
  return __ffs(__ballot_sync(WFULL, c2 && tie == mt)) - 1;
}

// ---- element layout: type-1 LPs with m, n <= 7, one tableau element (two rows) per lane ----
// lane = 8r + j owns T[r][j] (v0) and T[r+4][j] (v1): rows 0..6 are the constraints, row 7 the
// objective row; columns 0..6 are positions, column 7 the RHS.  Every exchange of a pivot is
// one shuffle (column e, pivot row l, PE), so the chain is Step 1 (one REDUX argmax), one
// division per RHS lane + one REDUX argmin, PE's reciprocal, one div_with and one fma per
// element -- the generic layout's switches and per-slot shuffles drop out.  The arithmetic is
// the oracle's operation for operation (Step 1 PAPER.md:93/132, ratio test P:97/126, pivot
// P:163-172, R5/R6/R12/R13/R15 in DESIGN.md).
constexpr int EL_CAP = 7;

template <bool RPC>
__device__ __forceinline__ void solve_elem(const SimplexArgs& a, int64_t lp, int lane) {
  const int m = a.m, n = a.n;
  const int r = lane >> 3, j = lane & 7;
  const int i0 = r, i1 = r + 4;  // the lane's rows (i1 == 7: the objective row)
  const double* __restrict__ Ak = a.A + lp * a.sA;
  const double* __restrict__ bk = a.b + lp * a.sb;
  const double* __restrict__ ck = a.c + lp * (int64_t)n;
  double v0, v1;
  if (j < 7) {
    v0 = (i0 < m && j < n) ? __ldg(Ak + i0 * n + j) : 0.0;
    v1 = (i1 == 7) ? ((j < n) ? __ldg(ck + j) : w_neg_inf())
                   : ((i1 < m && j < n) ? __ldg(Ak + i1 * n + j) : 0.0);
  } else {  // RHS column; the objective row's RHS cell z starts at 0 (obj = -z, R3)
    v0 = (i0 < m) ? __ldg(bk + i0) : 0.0;
    v1 = (i1 < m) ? __ldg(bk + i1) : 0.0;
  }
  int bk0 = n + i0, bk1 = n + i1;       // basic variables of the lane's rows (slack basis)
  int nbv = (j < n) ? j : DEADW;        // nonbasic variable of the lane's position
  int st = -1, it2 = 0, stall = 0;
  const uint64_t lpkey = RPC ? rpc_lp_key(a.rpc_seed, a.lp_base + lp) : 0ull;
  for (;;) {
    const bool bland = a.bland_K > 0 && stall >= a.bland_K;
    // Step 1 over the objective row (lanes 24..30)
    const bool cand = r == 3 && nbv != DEADW && v1 > a.eps_enter;
    int wl;
    if (bland) {
      wl = warp_argmin(cand, 0ull, (unsigned)nbv);
    } else if (RPC) {
      const uint64_t u = rpc_score(rpc_pivot_key(lpkey, it2), nbv);
      wl = w_argmax(cand, u, (unsigned)nbv);
    } else {
      wl = w_argmax(cand, okey(v1), (unsigned)nbv);
    }
    if (wl < 0) { st = ST_OPTIMAL; break; }
    if (it2 >= a.max_iter) { st = ST_ITER_LIMIT; break; }
    const int e = wl & 7;
    const int ev = __shfl_sync(WFULL, nbv, wl);
    // column e for the lane's rows
    const double c0 = __shfl_sync(WFULL, v0, (r << 3) | e);
    const double c1 = __shfl_sync(WFULL, v1, (r << 3) | e);
    // Step 2: the RHS lanes (j == 7) divide their two rows, keep the better, REDUX argmin
    // (div_with with recip_of(c) is div_fast(v, c); the winner's reciprocal is PE's, so it
    // travels with the partial instead of being recomputed after the argmin)
    bool val = false;
    double rr = 0.0, rc = 1.0;
    int li = -1, key = 0;
    if (j == 7) {
      const bool ok0 = i0 < m && c0 > a.eps_piv, ok1 = i1 < m && c1 > a.eps_piv;
      const double d0 = ok0 ? c0 : 1.0, d1 = ok1 ? c1 : 1.0;
      const double rc0 = recip_of(d0), rc1 = recip_of(d1);
      bool s0, s1;
      double q0 = div_with(v0, d0, rc0, s0);
      double q1 = div_with(v1, d1, rc1, s1);
      if (s0) q0 = ddiv_slow(v0, d0);
      if (s1) q1 = ddiv_slow(v1, d1);
      const int k0 = bland ? bk0 : i0, k1 = bland ? bk1 : i1;
      const bool take1 = ok1 && (!ok0 || q1 < q0 || (q1 == q0 && k1 < k0));
      val = ok0 || ok1;
      rr = take1 ? q1 : q0;
      rc = take1 ? rc1 : rc0;
      li = take1 ? i1 : i0;
      key = take1 ? k1 : k0;
    }
    const int wr = warp_argmin(val, okey(rr), ikey(key));
    if (wr < 0) { st = ST_UNBOUNDED; break; }
    const int l = __shfl_sync(WFULL, li, wr);
    const double theta = __shfl_sync(WFULL, rr, wr);
    const double rp = __shfl_sync(WFULL, rc, wr);  // recip_of(PE)
    // Step 3: row l's entries for the lane's position (PE at position e), divided by PE
    const bool hi = l >= 4;
    const double srcv = hi ? v1 : v0;
    const int lbase = (l & 3) << 3;
    const double pe = __shfl_sync(WFULL, srcv, lbase | e);
    const double prow = __shfl_sync(WFULL, srcv, lbase | j);
    const int leaving = __shfl_sync(WFULL, hi ? bk1 : bk0, lbase);
    const double num = (j == e) ? 1.0 : prow;
    bool sl;
    double pv = div_with(num, pe, rp, sl);
    if (sl) pv = ddiv_slow(num, pe);
    const bool ze = j == e;
    v0 = (i0 == l) ? pv : __fma_rn(-c0, pv, ze ? 0.0 : v0);
    v1 = (i1 == l) ? pv : __fma_rn(-c1, pv, ze ? 0.0 : v1);
    // basis swap: row l's variable leaves into position e
    if (i0 == l) bk0 = ev;
    if (i1 == l) bk1 = ev;
    if (ze) nbv = leaving;
    ++it2;
    stall = (theta > 0.0) ? 0 : stall + 1;
  }
  // ---- extract (R10) ----
  if (lane == 0) {
    a.status[lp] = st;
    a.iters[2 * lp] = 0;
    a.iters[2 * lp + 1] = it2;
  }
  if (lane == 31)  // holds z (row 7, RHS column)
    a.obj[lp] = (st == ST_OPTIMAL) ? -v1
              : (st == ST_UNBOUNDED) ? __longlong_as_double(0x7ff0000000000000ll)
                                     : __longlong_as_double(0x7ff8000000000000ll);
  if (a.x) {
    double* xk = a.x + lp * (int64_t)n;
    const double fill = (st == ST_OPTIMAL) ? 0.0 : __longlong_as_double(0x7ff8000000000000ll);
    if (lane < n) xk[lane] = fill;
    __syncwarp();
    if (st == ST_OPTIMAL && j == 7) {
      if (i0 < m && bk0 < n) xk[bk0] = v0;
      if (i1 < m && bk1 < n) xk[bk1] = v1;
    }
  }
}

// Optional phase profiler (-DLPB_PROFILE, scripts/wphase_prof.py): warp 0 of the grid adds
// clock64() deltas per phase into prof[phase]; prof[15] counts pivots.
#ifdef LPB_PROFILE
#define W_MARK(ph)                                   \
  if (prof_on) {                                     \
    const long long t_ = clock64();                  \
    pacc[ph] += t_ - pt;                             \
    pt = t_;                                         \
  }
#else
#define W_MARK(ph)
#endif

template <int A, int BC, bool TWO, bool RPC, bool EL>
__global__ void __launch_bounds__(32 * W_WARPS) simplex_warp_kernel(SimplexArgs a) {
  const int lane = threadIdx.x & 31;
#ifdef LPB_PROFILE
  const bool prof_on = a.prof != nullptr && blockIdx.x == 0 && threadIdx.x < 32;
  long long pacc[16] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  long long pt = clock64();
#endif
  const int tr = lane >> 2, tc = lane & 3;
  const int m = a.m, n = a.n;
  const int64_t gw = (int64_t)blockIdx.x * W_WARPS + (threadIdx.x >> 5);
  const int64_t nw = (int64_t)gridDim.x * W_WARPS;
  const bool direct = a.ticket == nullptr;

  // persistent warps take their next LP's ticket one LP ahead and prefetch its A, b, c into
  // L2 while the current LP is solved (the build's loads then miss HBM only once)
  auto take_ticket = [&]() -> int64_t {
    int t = 0;
    if (lane == 0) t = atomicAdd(a.ticket, 1);
    return __shfl_sync(WFULL, t, 0);
  };
  auto prefetch_lp = [&](int64_t q) {
    if (q >= a.batch) return;
    const char* pa = reinterpret_cast<const char*>(a.A + q * a.sA);
    const int64_t abytes = a.sA ? (int64_t)m * n * 8 : 0;
    for (int64_t off = (int64_t)lane * 128; off < abytes; off += 32 * 128)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(pa + off));
    if (lane == 0 && a.sb) asm volatile("prefetch.global.L2 [%0];" ::"l"(a.b + q * a.sb));
    if (lane == 1) asm volatile("prefetch.global.L2 [%0];" ::"l"(a.c + q * (int64_t)n));
  };
  int64_t lp = direct ? gw : take_ticket();
  int64_t lp_next = direct ? lp + nw : take_ticket();
  if (!direct) prefetch_lp(lp_next);
  while (lp < a.batch) {
    const double* __restrict__ Ak = a.A + lp * a.sA;
    const double* __restrict__ bk = a.b + lp * a.sb;
    const double* __restrict__ ck = a.c + lp * (int64_t)n;

    W_MARK(0)  // ticket / loop
    // ---- build (R7) ----
    const bool rowL = lane < m;
    const double bL = rowL ? __ldg(bk + lane) : 0.0;
    const bool negL = rowL && bL < 0.0;
    const unsigned negmask = __ballot_sync(WFULL, negL);
    const int k = __popc(negmask);
    if constexpr (EL) {  // a type-1 LP up to 7 x 7: the element layout (solve_elem)
      if (k == 0 && m <= EL_CAP && n <= EL_CAP) {
        solve_elem<RPC>(a, lp, lane);
        lp = lp_next;
        if (!direct && lp < a.batch) {
          lp_next = take_ticket();
          prefetch_lp(lp_next);
        } else {
          lp_next = lp + nw;
        }
        continue;
      }
    }
    const int npos = n + k;
    double binf = fabs(bL);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) binf = fmax(binf, __shfl_xor_sync(WFULL, binf, off));
    int st = (a.khint >= 0 && k > a.khint) ? ST_BAD_HINT
           : (m > 8 * A || npos > 4 * BC || (!TWO && k > 0)) ? ST_NUMERICAL : -1;
    double rhs = negL ? -bL : bL;                 // RHS of row `lane`
    int bkey = negL ? (lane - m) : (n + lane);    // key of row `lane`'s basic variable
    double T[A][BC];
    int nbv[BC];  // position -> variable (replicated across thread-rows)
#pragma unroll
    for (int b = 0; b < BC; ++b) {
      const int p = tc + 4 * b;
      int var = DEADW;
      if (p < n) {
        var = p;
      } else if (p < npos) {  // slack of the (p-n)-th negated row (ascending)
        unsigned mk = negmask;
        for (int t = 0; t < p - n; ++t) mk &= mk - 1u;
        var = n + (__ffs(mk) - 1);
      }
      nbv[b] = var;
    }
#pragma unroll
    for (int ai = 0; ai < A; ++ai) {
      const int i = tr + 8 * ai;
      const bool neg = (negmask >> (i & 31)) & 1u;
#pragma unroll
      for (int b = 0; b < BC; ++b) {
        const int p = tc + 4 * b;
        double v = 0.0;
        if (st < 0 && i < m && p < npos) {
          if (p < n) {
            v = __ldg(Ak + (int64_t)i * n + p);
            v = neg ? -v : v;
          } else {
            v = (nbv[b] == n + i) ? -1.0 : (neg ? -0.0 : 0.0);
          }
        }
        T[ai][b] = v;
      }
    }
    double d2[BC], d1[TWO ? BC : 1];
#pragma unroll
    for (int b = 0; b < BC; ++b) {
      const int p = tc + 4 * b;
      d2[b] = (p < n) ? __ldg(ck + p) : (p < npos ? 0.0 : w_neg_inf());
    }
    double z2 = 0.0, z1 = 0.0;
    if constexpr (TWO) {
      // phase-I row: ascending-row sums of the negated rows (R7), each lane for its positions
#pragma unroll
      for (int b = 0; b < BC; ++b) d1[b] = (tc + 4 * b < npos) ? 0.0 : w_neg_inf();
      if (k == 0) {
#pragma unroll
        for (int b = 0; b < BC; ++b) d1[b] = w_neg_inf();
      }
      unsigned mk = negmask;
      while (mk) {
        const int r = __ffs(mk) - 1;
        mk &= mk - 1u;
        const int ar = r >> 3, src = ((r & 7) << 2) | tc;
        double rv[BC];
#pragma unroll
        for (int b = 0; b < BC; ++b) {
          double v = T[0][b];
#pragma unroll
          for (int ai = 1; ai < A; ++ai) v = (ai == ar) ? T[ai][b] : v;
          rv[b] = __shfl_sync(WFULL, v, src);
        }
#pragma unroll
        for (int b = 0; b < BC; ++b)
          if (tc + 4 * b < npos) d1[b] = __dadd_rn(d1[b], rv[b]);
        z1 = __dadd_rn(z1, __shfl_sync(WFULL, rhs, r));
      }
    }

    W_MARK(1)  // loads + build
    // ---- Steps 1-3, two phases ----
    int it1 = 0, it2 = 0, stall = 0, phase = (TWO && k > 0) ? 1 : 2, dl = 0;
    bool drive = false;
    const uint64_t lpkey = RPC ? rpc_lp_key(a.rpc_seed, a.lp_base + lp) : 0ull;
    while (st < 0) {
      const bool bland = a.bland_K > 0 && stall >= a.bland_K;
      const bool p1 = TWO && phase == 1;
      int e, evar, l;
      double dE2 = 0.0, dE1 = 0.0;  // the objective rows' entries at position e
      W_MARK(10)  // loop head
      if (drive) {
        // R9: drive the next basic artificial out on max |T[l][p]| over live positions
        const unsigned art = __ballot_sync(WFULL, lane < m && bkey < 0);
        const unsigned rest = art & ~((dl >= 32) ? 0xffffffffu : ((1u << dl) - 1u));
        if (rest == 0u) {
          drive = false;
          phase = 2;
          stall = 0;
          continue;
        }
        l = __ffs(rest) - 1;
        dl = l + 1;
        const int al = l >> 3;
        bool val = false;
        double bv = 0.0;
        unsigned bvar = 0xffffffffu;
        int bb = 0;
        double bd2 = 0.0, bd1 = 0.0;
        if (tr == (l & 7)) {
#pragma unroll
          for (int b = 0; b < BC; ++b) {
            double v = T[0][b];
#pragma unroll
            for (int ai = 1; ai < A; ++ai) v = (ai == al) ? T[ai][b] : v;
            v = fabs(v);
            const unsigned var = (unsigned)nbv[b];
            if (d2[b] != w_neg_inf() && v > a.eps_piv &&
                (!val || v > bv || (v == bv && var < bvar))) {
              val = true;
              bv = v;
              bvar = var;
              bb = b;
              bd2 = d2[b];
              if constexpr (TWO) bd1 = d1[b];
            }
          }
        }
        const int wl = w_argmax(val, okey(bv), bvar);
        if (wl < 0) continue;  // redundant row: the artificial stays basic at 0
        e = __shfl_sync(WFULL, tc + 4 * bb, wl);
        evar = (int)__shfl_sync(WFULL, bvar, wl);
        dE2 = __shfl_sync(WFULL, bd2, wl);
        if constexpr (TWO) dE1 = __shfl_sync(WFULL, bd1, wl);
      } else {
        // Step 1 on thread-row 0 (the replicas are identical across thread-rows)
        bool val = false;
        double bv = w_neg_inf();
        unsigned long long bu = 0ull;
        unsigned bvar = 0xffffffffu;
        int bb = 0;
        double bd2 = 0.0, bd1 = 0.0;  // d2 / d1 at the chosen position (static indices only)
        const bool rpc = RPC && !bland;
        const uint64_t pkey = RPC ? rpc_pivot_key(lpkey, it1 + it2) : 0ull;
#define W_SCAN(RULE)                                                \
  _Pragma("unroll") for (int b = 0; b < BC; ++b) {                 \
    const double v = p1 ? d1[TWO ? b : 0] : d2[b];                  \
    const unsigned var = (unsigned)nbv[b];                          \
    const bool take = v > a.eps_enter && (RULE);                    \
    val = val || take;                                              \
    bv = take ? v : bv;                                             \
    bvar = take ? var : bvar;                                       \
    bb = take ? b : bb;                                             \
    bd2 = take ? d2[b] : bd2;                                       \
    if constexpr (TWO) bd1 = take ? d1[b] : bd1;                    \
  }
        if (bland) {  // the lowest variable index (R6)
          W_SCAN(var < bvar)
        } else if (rpc) {  // the largest counter-based score (R15)
#pragma unroll
          for (int b = 0; b < BC; ++b) {
            const double v = p1 ? d1[TWO ? b : 0] : d2[b];
            const unsigned var = (unsigned)nbv[b];
            const unsigned long long u = rpc_score(pkey, (int)var);
            const bool take = v > a.eps_enter && (!val || u > bu || (u == bu && var < bvar));
            val = val || take;
            bu = take ? u : bu;
            bv = take ? v : bv;
            bvar = take ? var : bvar;
            bb = take ? b : bb;
            bd2 = take ? d2[b] : bd2;
            if constexpr (TWO) bd1 = take ? d1[b] : bd1;
          }
        } else {  // LPC: the largest reduced cost, ties to the lowest variable index (R5):
                  // a pairwise tree (depth log2 BC) -- each level is a chain of dependent fp64
                  // compares, so the depth, not the count, sets the latency
          bool tv[BC];
          double tx[BC], t2[BC], t1[TWO ? BC : 1];
          unsigned tvr[BC];
          int tb[BC];
#pragma unroll
          for (int b = 0; b < BC; ++b) {
            tx[b] = p1 ? d1[TWO ? b : 0] : d2[b];
            tv[b] = tx[b] > a.eps_enter;
            tvr[b] = (unsigned)nbv[b];
            tb[b] = b;
            t2[b] = d2[b];
            if constexpr (TWO) t1[b] = d1[b];
          }
#pragma unroll
          for (int st_ = 1; st_ < BC; st_ *= 2) {
#pragma unroll
            for (int b = 0; b + st_ < BC; b += 2 * st_) {
              const int o = b + st_;
              const bool take = tv[o] && (!tv[b] || tx[o] > tx[b] ||
                                          (tx[o] == tx[b] && tvr[o] < tvr[b]));
              tv[b] = tv[b] || tv[o];
              tx[b] = take ? tx[o] : tx[b];
              tvr[b] = take ? tvr[o] : tvr[b];
              tb[b] = take ? tb[o] : tb[b];
              t2[b] = take ? t2[o] : t2[b];
              if constexpr (TWO) t1[b] = take ? t1[o] : t1[b];
            }
          }
          val = tv[0];
          bv = tx[0];
          bvar = tvr[0];
          bb = tb[0];
          bd2 = t2[0];
          if constexpr (TWO) bd1 = t1[0];
        }
#undef W_SCAN
        W_MARK(11)  // scan
        val = val && tr == 0;
        const int wl = bland ? warp_argmin(val, 0ull, bvar)
                             : w_argmax(val, rpc ? bu : okey(bv), bvar);
        W_MARK(12)  // argmax
        if (wl < 0) {
          if (phase == 2) { st = ST_OPTIMAL; break; }
          if (z1 > a.eps_phase1 * fmax(1.0, binf)) { st = ST_INFEASIBLE; break; }
          drive = true;  // phase-I optimum with w* ~ 0
          dl = 0;
          continue;
        }
        if (it1 + it2 >= a.max_iter) { st = ST_ITER_LIMIT; break; }
        e = __shfl_sync(WFULL, tc + 4 * bb, wl);
        evar = (int)__shfl_sync(WFULL, bvar, wl);
        dE2 = __shfl_sync(WFULL, bd2, wl);
        if constexpr (TWO) dE1 = __shfl_sync(WFULL, bd1, wl);
        l = -1;
      }

      W_MARK(2)  // Step 1
      // ---- column e: owners (tc == e%4) pick it; shuffles bring it to the ratio lanes and
      //      to every lane's update multipliers ----
      const int be = e >> 2, etc = e & 3;
      const bool mine = tc == etc;  // this lane holds position e
      double col[A];
      // uniform switch on the position slot: read column e, then the owners zero it (the
      // update's fma then yields the leaving variable's column, R13)
#define W_COL(x)                                                    \
  case x:                                                           \
    if constexpr ((x) < BC) {                                       \
      _Pragma("unroll") for (int ai = 0; ai < A; ++ai) {           \
        col[ai] = T[ai][x];                                         \
      }                                                             \
    }                                                               \
    break;
      switch (be) {
        W_COL(0) W_COL(1) W_COL(2) W_COL(3) W_COL(4) W_COL(5) W_COL(6) W_COL(7)
        default: break;
      }
#undef W_COL
      double f[A];  // -T[i][e] for the lane's rows
#pragma unroll
      for (int ai = 0; ai < A; ++ai) f[ai] = -__shfl_sync(WFULL, col[ai], (tr << 2) | etc);
      // ratio lane L = row L: T[L][e] comes from lane ((L & 7) << 2 | etc), register L >> 3
      double vL = 0.0;
      {
        const int src = ((lane & 7) << 2) | etc, aL = lane >> 3;
#pragma unroll
        for (int ai = 0; ai < A; ++ai) {
          const double v = __shfl_sync(WFULL, col[ai], src);
          vL = (ai == aL) ? v : vL;
        }
      }
      W_MARK(3)  // column e shuffles
      double theta = 0.0;
      if (!drive) {  // Step 2: ratio test, one row per lane (R1, R2, R5)
        const bool cand = lane < m && vL > a.eps_piv;
        bool slow;
        double r = div_fast(rhs, cand ? vL : 1.0, slow);
        if (slow) r = ddiv_slow(rhs, cand ? vL : 1.0);
        const int tie = bland ? bkey : lane;
        const int wr = warp_argmin(cand, okey(r), ikey(tie));
        if (wr < 0) { st = (phase == 2) ? ST_UNBOUNDED : ST_NUMERICAL; break; }
        l = wr;
        theta = __shfl_sync(WFULL, r, wr);
      }

      W_MARK(4)  // ratio test + argmin
      // ---- Step 3: pivot row l / PE, rank-1 update ----
      const double pe = __shfl_sync(WFULL, vL, l);
      const double rhs_l = __shfl_sync(WFULL, rhs, l);
      const int leaving = __shfl_sync(WFULL, bkey, l);
      const int al = l >> 3, ltr = l & 7;
      double prow[BC];
      {
        double rv[BC];
        const bool lrow = tr == ltr;  // this lane holds row l
#define W_ROW(x)                                                    \
  case x:                                                           \
    if constexpr ((x) < A) {                                        \
      _Pragma("unroll") for (int b = 0; b < BC; ++b) {             \
        rv[b] = T[x][b];                                            \
      }                                                             \
    }                                                               \
    break;
        switch (al) {
          W_ROW(0) W_ROW(1) W_ROW(2) W_ROW(3)
          default: break;
        }
#undef W_ROW
#pragma unroll
        for (int b = 0; b < BC; ++b) rv[b] = __shfl_sync(WFULL, rv[b], (ltr << 2) | tc);
        W_MARK(5)  // pe / row shuffles
        const double rpe = recip_of(pe);
        bool slow_any = false;
#pragma unroll
        for (int b = 0; b < BC; ++b) {
          const double num = (tc + 4 * b == e) ? 1.0 : rv[b];
          bool sl;
          prow[b] = div_with(num, pe, rpe, sl);
          slow_any |= sl;
        }
        bool slr;
        double prr = div_with(rhs_l, pe, rpe, slr);
        if (slow_any || slr) {
#pragma unroll
          for (int b = 0; b < BC; ++b) prow[b] = ddiv_slow((tc + 4 * b == e) ? 1.0 : rv[b], pe);
          prr = ddiv_slow(rhs_l, pe);
        }
        W_MARK(6)  // divisions
        // the lane's row L: RHS and basic variable
        rhs = (lane == l) ? prr : __fma_rn(-vL, prr, rhs);
        bkey = (lane == l) ? evar : bkey;
        // objective rows: position e restarts from 0, fma(-d_e, prow_p, d_p)
#pragma unroll
        for (int b = 0; b < BC; ++b) {
          const bool z = mine && b == be;
          d2[b] = __fma_rn(-dE2, prow[b], z ? 0.0 : d2[b]);
          if constexpr (TWO) {
            if (p1) d1[b] = __fma_rn(-dE1, prow[b], z ? 0.0 : d1[b]);
          }
        }
        z2 = __fma_rn(-dE2, prr, z2);
        if constexpr (TWO) {
          if (p1) z1 = __fma_rn(-dE1, prr, z1);
        }
        // tableau: row l and column e restart from 0, multiplier of row l = 1
#pragma unroll
        for (int ai = 0; ai < A; ++ai) {
          const bool isl = lrow && ai == al;
          const double fi = isl ? 1.0 : f[ai];
#pragma unroll
          for (int b = 0; b < BC; ++b) {
            const bool z = isl || (mine && b == be);
            T[ai][b] = __fma_rn(fi, prow[b], z ? 0.0 : T[ai][b]);
          }
        }
        // position e now holds the leaving variable (dead if artificial, R7)
        if (mine) {
          const int nv = leaving >= 0 ? leaving : DEADW;
#define W_NBV(x)                                                    \
  case x:                                                           \
    if constexpr ((x) < BC) {                                       \
      nbv[x] = nv;                                                  \
      if (leaving < 0) {                                            \
        d2[x] = w_neg_inf();                                        \
        if constexpr (TWO) d1[x] = w_neg_inf();                     \
      }                                                             \
    }                                                               \
    break;
          switch (be) {
            W_NBV(0) W_NBV(1) W_NBV(2) W_NBV(3) W_NBV(4) W_NBV(5) W_NBV(6) W_NBV(7)
            default: break;
          }
#undef W_NBV
        }
      }
      if (drive) {
        ++it1;
      } else {
        if (phase == 1) ++it1; else ++it2;
        stall = (theta > 0.0) ? 0 : stall + 1;
      }
      W_MARK(7)  // update
#ifdef LPB_PROFILE
      if (prof_on) pacc[15] += 1;
#endif
    }
    W_MARK(8)  // loop exit

    // ---- extract (R10) ----
    if (lane == 0) {
      a.status[lp] = st;
      a.iters[2 * lp] = it1;
      a.iters[2 * lp + 1] = it2;
      a.obj[lp] = (st == ST_OPTIMAL) ? -z2
                : (st == ST_UNBOUNDED) ? __longlong_as_double(0x7ff0000000000000ll)
                : (st == ST_INFEASIBLE) ? w_neg_inf()
                                        : __longlong_as_double(0x7ff8000000000000ll);
    }
    if (a.x) {
      double* xk = a.x + lp * (int64_t)n;
      const double fill = (st == ST_OPTIMAL) ? 0.0 : __longlong_as_double(0x7ff8000000000000ll);
      for (int j = lane; j < n; j += 32) xk[j] = fill;
      __syncwarp();
      if (st == ST_OPTIMAL && lane < m && bkey >= 0 && bkey < n) xk[bkey] = rhs;
    }
    W_MARK(9)  // extract
    lp = lp_next;  // direct: grid-stride (one pass when the grid covers the batch)
    if (!direct && lp < a.batch) {
      lp_next = take_ticket();
      prefetch_lp(lp_next);
    } else {
      lp_next = lp + nw;
    }
  }
#ifdef LPB_PROFILE
  if (prof_on && lane == 0)
    for (int q = 0; q < 16; ++q) atomicAdd((unsigned long long*)&a.prof[q], (unsigned long long)pacc[q]);
#endif
}

struct WarpCfg {
  int rcap, ccap, two, id;
};

// {id, A (row slots per thread-row), BC (positions per thread-col), TWO}
#define LPB_WARP_CONFIGS(X) \
  X(0, 1, 3, true)          \
  X(1, 2, 6, true)          \
  X(2, 4, 8, false)         \
  X(3, 4, 8, true)

template <int A, int BC, bool TWO, bool RPC>
cudaError_t launch_w(const SimplexArgs& a, int grid_override, cudaStream_t s, int* ctas) {
  // the smallest layout also carries the element layout for type-1 LPs up to 7 x 7
  constexpr bool EL = (A == 1) && (BC == 3);
  auto kern = simplex_warp_kernel<A, BC, TWO, RPC, EL>;
  static LaunchMemo memo;
  int per_sm = 0;
  const cudaError_t em = memo.get(0, &per_sm, [&](int& v, size_t) {
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, kern, 32 * W_WARPS, 0);
  });
  if (em != cudaSuccess) return em;
  const int64_t resident = (int64_t)(per_sm < 1 ? 1 : per_sm) * device_sm_count();
  const int64_t need = (a.batch + W_WARPS - 1) / W_WARPS;
  SimplexArgs d = a;
  int64_t grid;
  if (need <= resident && grid_override <= 0) {
    d.ticket = nullptr;  // one resident wave: warp w solves LP w
    grid = need;
  } else {
    grid = grid_override > 0 ? grid_override : resident;
    if (grid > need) grid = need;
    const cudaError_t e = cudaMemsetAsync(d.ticket, 0, sizeof(int), s);
    if (e != cudaSuccess) return e;
  }
  if (ctas) *ctas = (int)grid;
  kern<<<(unsigned)grid, 32 * W_WARPS, 0, s>>>(d);
  return cudaGetLastError();
}

}  // namespace

static const WarpCfg kWarpCfgs[] = {
#define X(id, A, BC, TWO) {8 * A, 4 * BC, TWO ? 1 : 0, id},
    LPB_WARP_CONFIGS(X)
#undef X
};

static int pick_warp(int m, int n, int kmax) {
  for (const WarpCfg& c : kWarpCfgs) {
    if (m > c.rcap || m > 32 || n + kmax > c.ccap) continue;
    if (kmax > 0 && !c.two) continue;
    return c.id;
  }
  return -1;
}

bool warp_fits(int m, int n, int kmax) { return pick_warp(m, n, kmax) >= 0; }
int warp_layout(int m, int n, int kmax) { return pick_warp(m, n, kmax); }

cudaError_t launch_simplex_warp(const SimplexArgs& a, int grid_override, cudaStream_t s,
                                int* ctas_out) {
  switch (pick_warp(a.m, a.n, a.kmax)) {
#define X(id, A, BC, TWO)                                                         \
  case id:                                                                        \
    return a.rpc ? launch_w<A, BC, TWO, true>(a, grid_override, s, ctas_out)      \
                 : launch_w<A, BC, TWO, false>(a, grid_override, s, ctas_out);
    LPB_WARP_CONFIGS(X)
#undef X
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace lpb
