// simplex_block.cu — M and L size classes: one LP per thread block (cl = 1) or per
// thread-block cluster of cl CTAs (cl = 2, 4, 8, 16) with the CONDENSED fp64 simplex tableau
// resident in shared memory (distributed shared memory across the cluster).
//
// The method is the paper's dense-tableau simplex (§3.1 Steps 1-3, lines 91-103;
// §4.2 "we assign a CUDA block of threads to solve an LP", line 114), re-laid out for
// sm_100a:
//   * condensed (dictionary) tableau: only the nonbasic columns + RHS are stored, (R) x (W)
//     with R = m+1 (+1 phase-I row when some b_i < 0) and W = n + k + 1 (k = #{b_i < 0});
//     the column of the leaving variable is swapped into the entering position.  Every
//     stored value is bit-identical to the corresponding full-tableau entry of the oracle
//     (readings R12/R13).
//   * the tableau never touches HBM: A, b, c are read once, status/obj/x/iters written once.
//   * Step 1 / Step 2 reductions ("parallel reduction ... two auxiliary
//     arrays Data and Indices") are (value, key) warp-shuffle butterflies + one SMEM slot
//     per warp, + one DSMEM slot per CTA for clusters.
//   * the L class splits the nonbasic positions across the cluster's CTAs (the paper's
//     "mapping an LP problem with more than one thread blocks"); the RHS
//     column is replicated in every CTA, so the pivot row stays CTA-local and only the
//     pivot column (R doubles) and two reduction partials cross DSMEM per pivot.
//   * persistent CTAs/clusters pull LP indices from an atomic ticket (pivot counts per LP
//     vary by 10x).
// Arithmetic contract (parity with oracle/lpb_oracle.c): IEEE __ddiv_rn for ratios and the
// pivot row, explicit __fma_rn(-f, r, t) for the update, __dadd_rn in ascending row order
// for the phase-I row; compiled with -fmad=false so nothing else is contracted.
#include <cooperative_groups.h>

#include <cfloat>
#include <climits>

#include "lpb_async.cuh"
#include "lpb_fp64.cuh"
#include "lpb_internal.cuh"
#include "lpb_reduce.cuh"
#include "lpb_rng.cuh"
#include "lpb_tmem.cuh"

namespace cg = cooperative_groups;

namespace lpb {
namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int DEAD = INT_MAX;  // a dead (left artificial) nonbasic position
constexpr int NT = 256;        // threads per CTA
constexpr int NW = NT / 32;

struct Cand {
  double v;
  int key;  // tie-break key: variable index / row / basis key
  int pos;  // < 0: no candidate
};

enum { MAX_V = 0, MIN_KEY = 1, MIN_V = 2 };

template <int MODE>
__device__ __forceinline__ bool better(const Cand& a, const Cand& b) {
  if (a.pos < 0) return false;
  if (b.pos < 0) return true;
  if (MODE == MAX_V) return a.v > b.v || (a.v == b.v && a.key < b.key);
  if (MODE == MIN_KEY) return a.key < b.key;
  return a.v < b.v || (a.v == b.v && a.key < b.key);
}

// Warp (value, key) reduction over the lanes' candidates (pos < 0: none), identical result
// in every lane; REDUX-based (lpb_reduce.cuh) with the MODE's order.
template <int MODE>
__device__ __forceinline__ Cand warp_reduce(Cand c) {
  const bool valid = c.pos >= 0;
  int wl;
  if (MODE == MAX_V) wl = warp_argmax(valid, okey(c.v), (unsigned)c.key);
  else if (MODE == MIN_KEY) wl = warp_argmin(valid, 0ull, ikey(c.key));
  else wl = warp_argmin(valid, okey(c.v), ikey(c.key));
  if (wl < 0) return Cand{0.0, 0, -1};
  Cand r;
  r.v = __shfl_sync(FULL, c.v, wl);
  r.key = __shfl_sync(FULL, c.key, wl);
  r.pos = __shfl_sync(FULL, c.pos, wl);
  return r;
}

// One CTA's speculative pivot proposal: its best local entering candidate and the ratio-test
// result on that column (the global winner is one of the CL proposals).
struct Rec {
  Cand ce;
  double theta;
  int l;
  int pad;
};

struct Ctl {
  double theta;
  double binf;
  int lp;
  int l;
  int k;
  int pad;
};

// Tableau row stride (doubles): even, so rows are 128-bit pair arrays, with S/2 odd so that a
// column read by 32 consecutive rows spreads over the banks.
__host__ __device__ __forceinline__ int row_stride(int Q) { return 2 * (((Q + 2) >> 1) | 1); }

struct Smem {
  // Tableau row i: SMEM row i - h0 for i >= h0; rows below h0 (hybrid TMR variants only) keep
  // their storage of record in a per-CTA global (L2-resident) scratch gT (the pivot loop holds
  // them in TMEM)
  __device__ __forceinline__ double* row(int i) const {
    return i < h0 ? gT + (size_t)i * S : T + (size_t)(i - h0) * S;
  }
  int h0 = 0, S = 0;
  double* gT = nullptr;
  double* T;      // rows x S
  double* colE;   // pivot column (all rows), filled by the owner CTA
  double* fcol;   // update multipliers: -colE_i, +1 for the pivot row
  double* prow;   // new pivot row (local columns)
  double* lraw;   // TMR: raw pivot row fetched from TMEM (S doubles)
  int* nbvar;     // local position -> variable index (or DEAD)
  int* bkey;      // row -> key of its basic variable (>= 0 real, < 0 artificial)
  int* negrows;   // ascending list of rows with b_i < 0
  int* wcount;    // NW ints
  Cand* wslots;   // 2 x NW
  Cand* cslots;   // 2 x CL
  Rec* rec;       // 2 x CL proposals (parity-buffered), written by every CTA of the cluster
  double* colC;   // 2 x CL x RC proposal columns (parity-buffered)
  Ctl* ctl;
  uint64_t* xbar; // 2 mbarriers (by parity): the peers' proposals have landed (PUSH, CL > 1)
  double* rbuf;   // 2 x (n + kmax + 1): phase-II row replay (warm start, mode 2)
};

template <int CL>
struct Cluster {
  int rank;
  __device__ Cluster() {
    if constexpr (CL > 1) rank = (int)cg::this_cluster().block_rank();
    else rank = 0;
  }
  __device__ __forceinline__ void sync() const {
    if constexpr (CL > 1) cg::this_cluster().sync();
    else __syncthreads();
  }
  template <class T>
  __device__ __forceinline__ T* remote(T* p, int q) const {
    if constexpr (CL > 1) return cg::this_cluster().map_shared_rank(p, q);
    else return p;
  }
};

// Block-wide (value,key) reduction; result identical in every thread.
template <int MODE>
__device__ __forceinline__ int warp_winner(const Cand& c) {
  const bool valid = c.pos >= 0;
  if (MODE == MAX_V) return warp_argmax(valid, okey(c.v), (unsigned)c.key);
  if (MODE == MIN_KEY) return warp_argmin(valid, 0ull, ikey(c.key));
  return warp_argmin(valid, okey(c.v), ikey(c.key));
}

template <int MODE>
__device__ __forceinline__ Cand block_reduce(Cand c, Cand* slots) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // the warp's winning lane writes the partial itself (no shuffles before the barrier)
  const int wl = warp_winner<MODE>(c);
  if (lane == (wl < 0 ? 0 : wl)) slots[w] = wl < 0 ? Cand{0.0, 0, -1} : c;
  __syncthreads();
  Cand r{0.0, 0, -1};
  if (lane < NW) r = slots[lane];
  return warp_reduce<MODE>(r);
}

// Cluster-wide reduction: block reduce, publish the CTA partial into every CTA's slot
// `rank`, cluster barrier, reduce the CL partials.
template <int MODE, int CL>
__device__ __forceinline__ Cand cluster_reduce(Cand c, const Smem& s, int& par,
                                               const Cluster<CL>& cl) {
  Cand* ws = s.wslots + par * NW;
  Cand* cs = s.cslots + par * CL;
  par ^= 1;
  Cand r = block_reduce<MODE>(c, ws);
  if constexpr (CL == 1) {
    return r;
  } else {
    if (threadIdx.x == 0)
#pragma unroll 1
      for (int q = 0; q < CL; ++q) *cl.remote(cs + cl.rank, q) = r;
    cl.sync();
    Cand best = cs[0];
#pragma unroll 4
    for (int q = 1; q < CL; ++q) {
      const Cand o = cs[q];
      if (better<MODE>(o, best)) best = o;
    }
    return best;
  }
}

// Step 3 (Listing 1) on the condensed tableau, CTA-local part.
// colE[] (pivot column, all rows) is already in this CTA's SMEM.  Row l becomes the pivot
// row divided by PE; the entering position e (owned by CTA `owner` at local column jloc)
// receives the leaving variable's column: rl = 1/PE in row l, fma(-f_i, rl, 0) elsewhere.
// Implementation: row l and column jloc are zeroed once their values are captured, and the
// multiplier of row l is +1, so ONE fma per element, T_ij = fma(fcol_i, prow_j, T_ij), yields
// the pivot row (fma(1, prow, 0)), the swapped column (fma(-f_i, rl, 0)) and every other
// element -- no per-element branch.  Warps walk rows, lanes walk columns (conflict-free
// SMEM rows, odd stride), the lane's prow values stay in registers.
// rec (mode 1): the new pivot row is also written to the record, local column j at global
// position g0 + j and the RHS (local column Wa - 1) at npos by rank 0.
struct RecRow {
  double* row;  // null: no recording
  int g0, npos;
  bool rank0;
};

__device__ __forceinline__ void pivot_local(const Smem& s, const double* colE, int S, int Wa,
                                            int nrow, int l, bool own, int jloc, int ent_var,
                                            const RecRow& rec = RecRow{nullptr, 0, 0, false}) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const double pe = colE[l];
  const double rpe = recip_of(pe);
  for (int j = tid; j < Wa; j += NT) {
    const bool sw = own && j == jloc;
    double* tl = s.row(l) + j;
    const double num = sw ? 1.0 : *tl;
    bool slow;
    double q = div_with(num, pe, rpe, slow);
    if (slow) q = ddiv_slow(num, pe);
    s.prow[j] = q;
    *tl = 0.0;
    if (rec.row) {
      if (j < Wa - 1) rec.row[rec.g0 + j] = q;
      else if (rec.rank0) rec.row[rec.npos] = q;
    }
  }
  for (int i = tid; i < nrow; i += NT) {
    s.fcol[i] = (i == l) ? 1.0 : -colE[i];
    if (own) s.row(i)[jloc] = 0.0;
  }
  if (tid == 0) {
    const int leaving = s.bkey[l];
    s.bkey[l] = ent_var;
    if (own) s.nbvar[jloc] = leaving < 0 ? DEAD : leaving;
    if (Wa & 1) s.prow[Wa] = 0.0;  // pad of the last pair (Wa + 1 <= S)
  }
  __syncthreads();
  // 128-bit pairs of columns: lane handles pairs lane + 32c (Wa <= 256 -> <= 4 chunks)
  constexpr int MAXC = 4;
  const int Wa2 = (Wa + 1) >> 1, S2 = S >> 1;
  const double2* prow2 = reinterpret_cast<const double2*>(s.prow);
  double2 pr[MAXC];
#pragma unroll
  for (int c = 0; c < MAXC; ++c) {
    const int j = lane + 32 * c;
    pr[c] = (j < Wa2) ? prow2[j] : make_double2(0.0, 0.0);
  }
  if (Wa2 <= 64) {  // the common case: two chunks
    for (int i = w; i < nrow; i += NW) {
      const double f = s.fcol[i];
      double2* row = reinterpret_cast<double2*>(s.row(i)) + lane;
      if (lane < Wa2) {
        double2 v0 = row[0];
        v0.x = __fma_rn(f, pr[0].x, v0.x);
        v0.y = __fma_rn(f, pr[0].y, v0.y);
        row[0] = v0;
      }
      if (lane + 32 < Wa2) {
        double2 v1 = row[32];
        v1.x = __fma_rn(f, pr[1].x, v1.x);
        v1.y = __fma_rn(f, pr[1].y, v1.y);
        row[32] = v1;
      }
    }
  } else {
    for (int i = w; i < nrow; i += NW) {
      const double f = s.fcol[i];
      double2* row = reinterpret_cast<double2*>(s.row(i)) + lane;
#pragma unroll
      for (int c = 0; c < MAXC; ++c) {
        if (lane + 32 * c < Wa2) {
          double2 v = row[32 * c];
          v.x = __fma_rn(f, pr[c].x, v.x);
          v.y = __fma_rn(f, pr[c].y, v.y);
          row[32 * c] = v;
        }
      }
    }
  }
  __syncthreads();
}

// Phase-II compaction ("dead positions and the phase-I row skipped"; the
// artificials are dropped after phase I).  Once phase I is over, the positions
// whose nonbasic variable is a left artificial (nbvar == DEAD) can never enter again, so each
// CTA moves its live columns (and the RHS) left, in order, and phase II updates cnt' + 1
// columns instead of cnt + 1.  Row-local moves: every warp owns whole rows, so a row is read
// into registers, then written back shifted.  Positions keep their global numbering
// g0 + local column (the owner CTA of a position is still pos / Q).  Returns the new count.
__device__ __forceinline__ int compact_live(const Smem& s, int S, int cnt, int nrows) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int j = tid;  // cnt <= Q <= 255 < NT: one column per thread
  const bool live = j < cnt && s.nbvar[j] != DEAD;
  const int var = j < cnt ? s.nbvar[j] : DEAD;
  const unsigned bal = __ballot_sync(FULL, live);
  if (lane == 0) s.wcount[w] = __popc(bal);
  __syncthreads();
  int off = 0, tot = 0;
#pragma unroll
  for (int q = 0; q < NW; ++q) {
    const int cq = s.wcount[q];
    if (q < w) off += cq;
    tot += cq;
  }
  if (tot == cnt) {  // nothing dead on this CTA
    __syncthreads();
    return cnt;
  }
  int* map = reinterpret_cast<int*>(s.prow);  // scratch: prow holds S >= cnt + 1 doubles
  if (j < cnt) map[j] = live ? off + __popc(bal & ((1u << lane) - 1u)) : -1;
  if (j == cnt) map[j] = tot;  // the RHS column
  __syncthreads();
  if (live) s.nbvar[map[j]] = var;
  constexpr int CH = (NT + 31) / 32;  // column chunks of a row (cnt + 1 <= NT)
  for (int i = w; i < nrows; i += NW) {
    double v[CH];
    int dst[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      const int jj = lane + 32 * c;
      dst[c] = jj <= cnt ? map[jj] : -1;
      v[c] = dst[c] >= 0 ? s.row(i)[jj] : 0.0;
    }
    __syncwarp();
#pragma unroll
    for (int c = 0; c < CH; ++c)
      if (dst[c] >= 0) s.row(i)[dst[c]] = v[c];
    __syncwarp();
  }
  __syncthreads();
  return tot;
}

// ---- TMR variants: the constraint rows live in TENSOR MEMORY during the pivot loop ----
// The L class is bound by SMEM bandwidth in its rank-1 update (16 B of SMEM traffic per
// element, 128 B/clk/SM).  TMEM (128 lanes x 512 columns x 32 bit per SM) has its own
// datapath (scripts/ubench/tmem_bw.cu: ~155 B/clk/SM read plus as much written), so the TMR
// variants keep constraint row r in TMEM lane r % 128, row slot r / 128, position j of the
// CTA's range at columns slot * sc + 2j, 2j + 1 (one fp64 per column pair).  Warp w reaches
// lanes 32 (w % 4) .. + 31 (the 32x32b shapes), so the 8 warps of a CTA form two halves
// (h = w / 4) over the same lanes: half h updates the 8-position chunks c = h, h + 2, ... of
// every row of its lanes, and serves the row slots s = h, h + 2, ... in the ratio test.  The
// objective rows (Step 1) stay in SMEM.  The SMEM rows are still the storage of record for
// the build, the phase switch (drive-out + compaction) and the extraction: the rows are
// copied TMEM <-> SMEM at those points (once or twice per LP), and the pivot loop in between
// never touches the SMEM copies of the constraint rows.
constexpr int TM_NS = 4;     // row slots (m <= 512)
#ifndef LPB_HYB_MT
#define LPB_HYB_MT 128
#endif
constexpr int HYB_MT = LPB_HYB_MT;  // hybrid layout: constraint rows [0, HYB_MT) in TMEM
// row slots a TMR variant is compiled for (register arrays): 2-CTA clusters m <= 256, 4-CTA
// m <= 384, larger clusters m <= 512
__host__ __device__ constexpr int tm_ns_max(int cl) { return cl <= 2 ? 2 : cl <= 4 ? 3 : 4; }
constexpr int TM_COLS = 512; // the whole TMEM of the SM: TMR launches run 1 CTA per SM

struct TmRows {
  uint32_t tb;  // TMEM address of this warp's lane quarter, column 0
  int ns, sc;   // row slots in use, columns per slot (16 per 8-position chunk)
  int q, h;     // lane quarter (w % 4), half (w / 4)
  int mt;       // rows [0, mt) live in TMEM (m, or 128 in the hybrid layout); the rest in SMEM
};

__host__ __device__ __forceinline__ int tm_slot_cols(int Q) { return 16 * ((Q + 1 + 7) / 8); }
__host__ __device__ __forceinline__ int tm_slots(int m) { return (m + 127) / 128; }

// Every TMEM write of this thread has landed, and a barrier orders it before the other
// threads' TMEM accesses (and theirs before ours).
__device__ __forceinline__ void tm_sync() {
  tm_wait_st();
  tm_fence_before();
  __syncthreads();
  tm_fence_after();
}

// SMEM rows [0, m) -> TMEM (nch chunks of 8 positions); ends with tm_sync().
__device__ __forceinline__ void tm_rows_from_smem(const Smem& s, const TmRows& t, int S, int,
                                                  int nch) {
  const int lane = threadIdx.x & 31, m = t.mt;
  for (int sl = 0; sl < t.ns; ++sl) {
    if (128 * sl + 32 * t.q >= m) break;  // warp-uniform: no row of this warp
    const int r = 128 * sl + 32 * t.q + lane;
    const double* row = s.row(r < m ? r : 0);
    for (int c = t.h; c < nch; c += 2) {
      uint32_t v[16];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int j = 8 * c + k;
        tm_split((r < m && j < S) ? row[j] : 0.0, v[2 * k], v[2 * k + 1]);
      }
      tm_st16(t.tb + sl * t.sc + 16 * c, v);
    }
  }
  tm_sync();
}

// TMEM rows [0, m) -> SMEM; ends with a barrier.
__device__ __forceinline__ void tm_rows_to_smem(const Smem& s, const TmRows& t, int S, int,
                                                int nch) {
  const int lane = threadIdx.x & 31, m = t.mt;
  for (int sl = 0; sl < t.ns; ++sl) {
    if (128 * sl + 32 * t.q >= m) break;
    const int r = 128 * sl + 32 * t.q + lane;
    double* row = s.row(r < m ? r : 0);
    for (int c = t.h; c < nch; c += 2) {
      uint32_t v[16];
      tm_ld16(t.tb + sl * t.sc + 16 * c, v);
      tm_wait_ld();
      if (r < m) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int j = 8 * c + k;
          if (j < S) row[j] = tm_d(v[2 * k], v[2 * k + 1]);
        }
      }
    }
  }
  tm_fence_before();
  __syncthreads();
  tm_fence_after();
}

// Step 3 of the TMR variants (same arithmetic as pivot_local): row l (< m) is fetched from
// TMEM into its SMEM row by the two warps of its lane quarter (the owner lane stores, every
// lane writes back, the owner zeros), then the divisions by PE run as in pivot_local, column
// jloc is zeroed in TMEM (owner CTA), and the update runs chunk by chunk over the TMEM rows
// (the 8 pivot-row quotients of a chunk are SMEM broadcasts) and row by row over the SMEM
// objective rows [m, nrow).
template <int NSX, bool HYB>
__device__ __forceinline__ void pivot_local_tm(const Smem& s, const TmRows& t, const double* colE,
                                               int S, int Wa, int m, int nrow, int l, bool own,
                                               int jloc, int ent_var, const RecRow& rec) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int nch = (Wa + 7) >> 3;
  const int mt = HYB ? t.mt : m;
  const bool ltm = !HYB || l < mt;  // row l in TMEM (else an SMEM row of the hybrid layout)
  if (ltm && t.q == ((l >> 5) & 3)) {  // the pivot row's lane quarter (warp-uniform)
    const int sl = l >> 7;
    const bool ol = lane == (l & 31);
    constexpr int FB = 1;  // chunks in flight per wait (measured: 4 is no faster)
    for (int c0 = t.h; c0 < nch; c0 += 2 * FB) {
      uint32_t v[FB][16];
#pragma unroll
      for (int u = 0; u < FB; ++u)
        if (c0 + 2 * u < nch) tm_ld16(t.tb + sl * t.sc + 16 * (c0 + 2 * u), v[u]);
      tm_wait_ld();
#pragma unroll
      for (int u = 0; u < FB; ++u) {
        const int c = c0 + 2 * u;
        if (c < nch) {
          if (ol) {  // 128-bit stores (S is even: pairs never straddle the row end)
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const int j = 8 * c + 2 * k;
              if (j < S)
                *reinterpret_cast<double2*>(s.lraw + j) =
                    make_double2(tm_d(v[u][4 * k], v[u][4 * k + 1]),
                                 tm_d(v[u][4 * k + 2], v[u][4 * k + 3]));
            }
          }
#pragma unroll
          for (int k = 0; k < 16; ++k) v[u][k] = ol ? 0u : v[u][k];
          tm_st16(t.tb + sl * t.sc + 16 * c, v[u]);
        }
      }
    }
  }
  if (own && t.h == ((jloc >> 3) & 1))  // the swapped column starts from 0 (as pivot_local)
    for (int sl = 0; sl < t.ns; ++sl)
      if (128 * sl + 32 * t.q < mt) tm_st2(t.tb + sl * t.sc + 2 * jloc, 0u, 0u);
  tm_sync();
  double* const lrow = ltm ? s.lraw : s.row(l);
  const double pe = colE[l];
  const double rpe = recip_of(pe);
  for (int j = tid; j < Wa; j += NT) {
    const bool sw = own && j == jloc;
    const double num = sw ? 1.0 : lrow[j];
    if (!ltm) lrow[j] = 0.0;  // an SMEM row l starts from 0 (fcol_l = 1), as in pivot_local
    bool slow;
    double q = div_with(num, pe, rpe, slow);
    if (slow) q = ddiv_slow(num, pe);
    s.prow[j] = q;
    if (rec.row) {
      if (j < Wa - 1) rec.row[rec.g0 + j] = q;
      else if (rec.rank0) rec.row[rec.npos] = q;
    }
  }
  for (int i = tid; i < nrow; i += NT) {
    s.fcol[i] = (i == l) ? 1.0 : -colE[i];
    if (own && i >= mt) s.row(i)[jloc] = 0.0;
  }
  if (tid == 0) {
    const int leaving = s.bkey[l];
    s.bkey[l] = ent_var;
    if (own) s.nbvar[jloc] = leaving < 0 ? DEAD : leaving;
    if (Wa & 1) s.prow[Wa] = 0.0;
  }
  __syncthreads();
  // objective rows (SMEM): lanes walk 128-bit column pairs
  {
    const int Wa2 = (Wa + 1) >> 1;
    const double2* prow2 = reinterpret_cast<const double2*>(s.prow);
    for (int i = mt + w; i < nrow; i += NW) {  // SMEM rows: the objective rows (+ hybrid rows)
      const double f = s.fcol[i];
      double2* T2 = reinterpret_cast<double2*>(s.row(i));
      for (int j = lane; j < Wa2; j += 32) {
        const double2 p = prow2[j];
        double2 v = T2[j];
        v.x = __fma_rn(f, p.x, v.x);
        v.y = __fma_rn(f, p.y, v.y);
        T2[j] = v;
      }
    }
  }
  // constraint rows (TMEM): chunk c = h, h + 2, ...; the chunk's 8 quotients are loaded once
  // and applied to every row slot of the lane
  // chunk by chunk: the chunk's 8 quotients are loaded once and applied to every row slot of
  // the lane (measured: batching several TMEM loads per wait is slower, cfg3 +10..20 %)
  double f[NSX];
#pragma unroll
  for (int sl = 0; sl < NSX; ++sl) {
    const int r = 128 * sl + 32 * t.q + lane;
    f[sl] = (sl < t.ns && r < mt) ? s.fcol[r] : 0.0;
  }
  const double2* prow2 = reinterpret_cast<const double2*>(s.prow);
  for (int c = t.h; c < nch; c += 2) {
    double2 p[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) p[k] = prow2[4 * c + k];
#pragma unroll
    for (int sl = 0; sl < NSX; ++sl) {
      if (sl < t.ns && 128 * sl + 32 * t.q < mt) {  // warp-uniform
        uint32_t v[16];
        const uint32_t ad = t.tb + sl * t.sc + 16 * c;
        tm_ld16(ad, v);
        tm_wait_ld();
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          tm_split(__fma_rn(f[sl], p[k].x, tm_d(v[4 * k], v[4 * k + 1])), v[4 * k], v[4 * k + 1]);
          tm_split(__fma_rn(f[sl], p[k].y, tm_d(v[4 * k + 2], v[4 * k + 3])), v[4 * k + 2],
                   v[4 * k + 3]);
        }
        tm_st16(ad, v);
      }
    }
  }
  tm_sync();
}

// PULL (proposal columns read over DSMEM after the barrier) is used for CL >= 8, and for
// CL = 2/4 whenever its smaller SMEM footprint fits more CTAs per SM than PUSH (launch_cl).
template <int CL, bool PULL, bool TMR>
__device__ __forceinline__ void simplex_block_body(const SimplexArgs& a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const Cluster<CL> cl;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int m = a.m, n = a.n;
  const int Q = (n + a.kmax + CL - 1) / CL;  // nonbasic positions per CTA (capacity)
  const int S = row_stride(Q);  // even (128-bit rows), S/2 odd (spread column reads)
  const int RC = m + 2;

  // hybrid TMR layout: rows 0..127 live in TMEM during the pivot loop and in the CTA's global
  // scratch otherwise; SMEM holds rows 128.. only
  const bool hyb = TMR && CL == 2 && a.tm_hyb != 0;
  Smem s;
  s.S = S;
  s.h0 = hyb ? HYB_MT : 0;
  s.gT = hyb ? a.tm_scr + (size_t)blockIdx.x * HYB_MT * S : nullptr;
  s.T = reinterpret_cast<double*>(smem_raw);
  s.colE = s.T + (size_t)(RC - s.h0) * S;
  s.fcol = s.colE + RC;
  s.prow = s.fcol + RC;
  s.lraw = s.prow + S;
  s.nbvar = reinterpret_cast<int*>(s.lraw + S);
  s.bkey = s.nbvar + (Q + 1);
  // negrows is needed only while the LP is built, before colE is first written: alias
  s.negrows = reinterpret_cast<int*>(s.colE);
  s.wcount = s.bkey + m;
  uintptr_t p = reinterpret_cast<uintptr_t>(s.wcount + NW);
  p = (p + 15) & ~uintptr_t(15);
  s.wslots = reinterpret_cast<Cand*>(p);
  s.cslots = s.wslots + 2 * NW;
  s.rec = reinterpret_cast<Rec*>(s.cslots + 2 * CL);
  s.colC = reinterpret_cast<double*>(s.rec + 2 * CL);
  s.ctl = reinterpret_cast<Ctl*>(s.colC + 2 * (PULL ? 1 : CL) * RC);
  s.xbar = reinterpret_cast<uint64_t*>(s.ctl + 1);
  s.rbuf = reinterpret_cast<double*>(s.xbar + 2);  // allocated for mode 2 (warm start) only
  // PUSH clusters exchange the per-pivot proposals with st.async into the peers' slots, each
  // completing on the receiver's mbarrier of that parity: no cluster barrier (and no release
  // fence over every outstanding memory operation) per pivot.
  constexpr bool XASYNC = !PULL && CL > 1;
  if (XASYNC && tid == 0) {
    mbar_init(&s.xbar[0], 1);
    mbar_init(&s.xbar[1], 1);
  }
  uint32_t xph = 0;  // bit q: parity of the next phase of xbar[q]

  // DSMEM may only be touched once every CTA of the cluster is running: one
  // cluster barrier before the first remote ticket write (racecheck finding); it also
  // publishes the initialised mbarriers.
  TmRows tm{0u, hyb ? 1 : tm_slots(m), tm_slot_cols(Q), w & 3, w >> 2, hyb ? (m < HYB_MT ? m : HYB_MT) : m};
  const uint32_t tmcols = hyb ? TM_COLS / 2 : TM_COLS;  // hybrid: two CTAs share the SM's TMEM
  if constexpr (TMR) {
    if (w == 0) tm_alloc_n(reinterpret_cast<uint32_t*>(&s.ctl->pad), tmcols);
    tm_fence_before();
  }
  if constexpr (CL > 1) cl.sync();
  else if (XASYNC || TMR) __syncthreads();
  if constexpr (TMR) {
    tm_fence_after();
    tm.tb = (uint32_t)s.ctl->pad + ((uint32_t)(32 * tm.q) << 16);
  }

  int par = 0;
  for (;;) {
    if (cl.rank == 0 && tid == 0) {
      const int t = atomicAdd(a.ticket, 1);
#pragma unroll 1
      for (int q = 0; q < CL; ++q) cl.remote(s.ctl, q)->lp = t;
    }
    cl.sync();
    const int64_t lp = s.ctl->lp;
    if (lp >= a.batch) break;

    const double* __restrict__ Ak = a.A + lp * a.sA;
    const double* __restrict__ bk = a.b + lp * a.sb;
    const double* __restrict__ ck = a.c + lp * (int64_t)n;

    // ---- build (reading R7): negated rows, basis keys, |b|_inf ----
    const bool warm = a.mode == 2;
    int k = warm ? a.rec_info[3] : 0;
    double binf = 0.0;
    for (int base = 0; base < (warm ? 0 : m); base += NT) {
      const int i = base + tid;
      const double bi = (i < m) ? __ldg(bk + i) : 0.0;
      const bool neg = (i < m) && (bi < 0.0);
      binf = fmax(binf, fabs(bi));
      const unsigned bal = __ballot_sync(FULL, neg);
      if (lane == 0) s.wcount[w] = __popc(bal);
      __syncthreads();
      int off = k, tot = 0;
      for (int q = 0; q < NW; ++q) {
        const int cq = s.wcount[q];
        if (q < w) off += cq;
        tot += cq;
      }
      if (neg) s.negrows[off + __popc(bal & ((1u << lane) - 1u))] = i;
      if (i < m) s.bkey[i] = neg ? (i - m) : (n + i);
      k += tot;
      __syncthreads();
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) binf = fmax(binf, __shfl_xor_sync(FULL, binf, off));
    if (lane == 0) s.wslots[w].v = binf;
    __syncthreads();
    binf = s.wslots[0].v;
    for (int q = 1; q < NW; ++q) binf = fmax(binf, s.wslots[q].v);
    __syncthreads();

    int st = -1, it1 = 0, it2 = 0;
    bool tm_live = false;  // TMR: the constraint rows are in TMEM (not their SMEM copies)
    const uint64_t lpkey = a.rpc ? rpc_lp_key(a.rpc_seed, a.lp_base + lp) : 0ull;
    int cnt = max(0, min(Q, n + k - cl.rank * Q));  // live local positions
    int Wa = cnt + 1;                               // + RHS at local column cnt
    const int Wp = (Wa + 1) & ~1;                   // whole 128-bit pairs (build)
    const int g0 = cl.rank * Q;
    if (k > a.kmax) st = ST_NUMERICAL;  // cannot happen: kmax comes from the prepass / hint
    if (a.khint >= 0 && k > a.khint) st = ST_BAD_HINT;
    const int npos = n + k, Wr = npos + 1;              // record row: positions, then RHS
    int phase = (k > 0) ? 1 : 2;

    if (warm && st < 0) {
      // Warm start (mode 2): phase I of this polytope was solved once (mode 1).  Terminal
      // phase-I outcomes apply to every LP; otherwise load the recorded tableau and rebuild
      // this LP's carried phase-II row by replaying the recorded pivots on c -- the same
      // fma(-f, prow_j, T_mj) sequence phase I applies to it (R7, R13): bit-identical.
      const int rst = a.rec_info[0];
      it1 = a.rec_info[1];
      if (rst >= 0) {
        st = rst;
      } else {
        const int npiv = a.rec_info[2];
        phase = 2;
        for (int i = w; i < m; i += NW)
          for (int j = lane; j < Wp; j += 32)
            s.row(i)[j] = (j < cnt) ? a.rec_T[(size_t)i * Wr + g0 + j]
                                       : (j == cnt ? a.rec_T[(size_t)i * Wr + npos] : 0.0);
        for (int j = tid; j < cnt; j += NT) s.nbvar[j] = a.rec_nbvar[g0 + j];
        for (int i = tid; i < m; i += NT) s.bkey[i] = a.rec_bkey[i];
        double* cur = s.rbuf;
        double* nxt = s.rbuf + Wr;
        for (int p = tid; p < Wr; p += NT) cur[p] = (p < n) ? __ldg(ck + p) : 0.0;
        __syncthreads();
        for (int t = 0; t < npiv; ++t) {
          const int e = __ldg(a.rec_e + t);
          const double f = cur[e];
          const double* __restrict__ pr = a.rec_rows + (size_t)t * Wr;
          for (int p = tid; p < Wr; p += NT) nxt[p] = __fma_rn(-f, __ldg(pr + p), p == e ? 0.0 : cur[p]);
          double* tmp = cur;
          cur = nxt;
          nxt = tmp;
          __syncthreads();
        }
        for (int j = tid; j < Wp; j += NT)
          s.row(m)[j] = (j < cnt) ? cur[g0 + j] : (j == cnt ? cur[npos] : 0.0);
        __syncthreads();
        cnt = compact_live(s, S, cnt, m + 1);  // phase II from here on: drop dead positions
        Wa = cnt + 1;
        if constexpr (TMR) {
          tm_rows_from_smem(s, tm, S, m, (Wa + 7) >> 3);
          tm_live = true;
        }
      }
    } else if (st < 0) {
      for (int i = w; i < m; i += NW) {
        const bool neg = s.bkey[i] < 0;
        for (int j = lane; j < Wp; j += 32) {
          const int gp = g0 + j;
          double v;
          if (j >= Wa) {
            v = 0.0;  // pad column of the last 128-bit pair
          } else if (j == cnt) {
            v = __ldg(bk + i);
            v = neg ? -v : v;
          } else if (gp < n) {
            v = __ldg(Ak + (int64_t)i * n + gp);
            v = neg ? -v : v;
          } else {
            v = (i == s.negrows[gp - n]) ? -1.0 : (neg ? -0.0 : 0.0);
          }
          s.row(i)[j] = v;
        }
      }
      for (int j = tid; j < Wp; j += NT) {
        const int gp = g0 + j;
        s.row(m)[j] = (j < cnt && gp < n) ? __ldg(ck + gp) : 0.0;
        if (j < cnt) s.nbvar[j] = gp < n ? gp : n + s.negrows[gp - n];
      }
      __syncthreads();
      if (k > 0) {  // phase-I row: ascending-row sums of the negated rows (R7)
        for (int j = tid; j < Wp; j += NT) {
          double acc = 0.0;
          for (int t = 0; t < k; ++t) acc = __dadd_rn(acc, s.row(s.negrows[t])[j]);
          s.row(m + 1)[j] = acc;
        }
      }
      __syncthreads();
      if constexpr (TMR) {
          tm_rows_from_smem(s, tm, S, m, (Wa + 7) >> 3);
          tm_live = true;
        }
    }

    // ---- Steps 1-3 loop, two phases ----
    int stall = 0, pp = 0;
    const bool record = a.mode == 1;  // record phase I (LP 0 only), then stop
    bool recorded = false;
    while (st < 0) {
      const int objrow = (phase == 1) ? m + 1 : m;
      const int nrow = (phase == 1) ? m + 2 : m + 1;
      const bool bland = a.bland_K > 0 && stall >= a.bland_K;
      // Step 1: this CTA's entering candidate (LPC/Dantzig, lowest variable index on ties;
      // Bland), then Step 2 on that candidate column, speculatively: the global winner is
      // one of the CL proposals, so ONE cluster barrier per pivot publishes them all.
      // RPC: the candidate's value is its counter-based score u < 2^53 (exact as a double,
      // lpb_rng.cuh), so the same max-value reductions pick the largest score.
      Cand ce{0.0, 0, -1};
      const bool rpc = a.rpc && !bland;
      const uint64_t pkey = rpc ? rpc_pivot_key(lpkey, it1 + it2) : 0ull;
      for (int j = tid; j < cnt; j += NT) {
        const int var = s.nbvar[j];
        const double d = s.row(objrow)[j];
        if (var != DEAD && d > a.eps_enter) {
          const Cand cd{rpc ? (double)rpc_score(pkey, var) : d, var, g0 + j};
          if (bland ? better<MIN_KEY>(cd, ce) : better<MAX_V>(cd, ce)) ce = cd;
        }
      }
      ce = bland ? block_reduce<MIN_KEY>(ce, s.wslots) : block_reduce<MAX_V>(ce, s.wslots);
      Cand cr{0.0, 0, -1};
      const int jc = ce.pos - g0;  // local column of the proposal
      const int jcs = ce.pos >= 0 ? jc : 0;  // the column sent (ignored without a candidate)
      double cv[TMR ? TM_NS : 1];  // TMR: column jcs of this thread's TMEM rows
      if constexpr (TMR) {
#pragma unroll
        for (int sl = 0; sl < TM_NS; ++sl) {
          cv[sl] = 0.0;
          if (sl < tm.ns && (sl & 1) == tm.h && 128 * sl + 32 * tm.q < tm.mt) {  // warp-uniform
            uint32_t a0, a1, b0, b1;
            tm_ld2(tm.tb + sl * tm.sc + 2 * jcs, a0, a1);
            tm_ld2(tm.tb + sl * tm.sc + 2 * cnt, b0, b1);
            tm_wait_ld();
            const int i = 128 * sl + 32 * tm.q + lane;
            const double ai = tm_d(a0, a1);
            cv[sl] = ai;
            if (ce.pos >= 0 && i < tm.mt && ai > a.eps_piv) {
              const double ri = tm_d(b0, b1);
              bool slow;
              double r = div_fast(ri, ai, slow);
              if (slow) r = ddiv_slow(ri, ai);
              const Cand cc{r, bland ? s.bkey[i] : i, i};
              if (better<MIN_V>(cc, cr)) cr = cc;
            }
          }
        }
        tm_fence_before();  // these loads precede the update's stores (after the barriers)
      }
      // SMEM constraint rows (all of them, or the hybrid's rows 128..): in the hybrid layout the
      // half-0 warps serve the TMEM slot above, so the half-1 warps take these rows
      // (measured: cfg3 -1.4 %, and -1.6 % more for the column publish below)
      const int st0 = hyb ? tid - NT / 2 : tid;
      const int sstep = hyb ? NT / 2 : NT;
      if (ce.pos >= 0 && st0 >= 0) {
        for (int i = (TMR ? tm.mt : 0) + st0; i < m; i += sstep) {
          const double ai = s.row(i)[jc];
          if (ai > a.eps_piv) {
            bool slow;
            double r = div_fast(s.row(i)[cnt], ai, slow);
            if (slow) r = ddiv_slow(s.row(i)[cnt], ai);
            const Cand cc{r, bland ? s.bkey[i] : i, i};
            if (better<MIN_V>(cc, cr)) cr = cc;
          }
        }
      }
      cr = block_reduce<MIN_V>(cr, s.wslots + NW);
      // PUSH (CL <= 4): the proposal column goes into every CTA's slot `rank`;
      // PULL (CL >= 8): it stays in this CTA's own parity slot and the CTAs read the winner's
      // slot over DSMEM after the barrier (SMEM for CL columns would not fit at m ~ 500).
      // The PULL slot of parity pp is rewritten two pivots later, after the next cluster
      // barrier, which every reader has passed only once its pivot_local read is done.
      double* const myc = PULL ? s.colC + (size_t)pp * RC
                               : s.colC + (size_t)(pp * CL + cl.rank) * RC;
      if constexpr (XASYNC) {
        // every CTA sends a column (column 0 when it has no candidate, then ignored), so
        // each receiver expects exactly (CL - 1) columns + records
        if (tid == 0) mbar_arrive_expect(&s.xbar[pp], (CL - 1) * (nrow * 8 + (int)sizeof(Rec)));
        uint32_t rb[CL], rc[CL];
#pragma unroll
        for (int q = 0; q < CL; ++q) {
          rb[q] = cluster_addr(myc, q);
          rc[q] = cluster_addr(&s.xbar[pp], q);
        }
        if constexpr (TMR) {
#pragma unroll
          for (int sl = 0; sl < TM_NS; ++sl) {
            const int i = 128 * sl + 32 * tm.q + lane;
            if (sl < tm.ns && (sl & 1) == tm.h && i < tm.mt) {
              myc[i] = cv[sl];
#pragma unroll
              for (int q = 0; q < CL; ++q)
                if (q != cl.rank) st_async_f64(rb[q] + 8u * i, cv[sl], rc[q]);
            }
          }
        }
        for (int i = (TMR ? tm.mt : 0) + st0; st0 >= 0 && i < nrow; i += sstep) {
          const double v = s.row(i)[jcs];
          myc[i] = v;
#pragma unroll
          for (int q = 0; q < CL; ++q)
            if (q != cl.rank) st_async_f64(rb[q] + 8u * i, v, rc[q]);
        }
        if (tid == 0) {
          const Rec r{ce, cr.v, cr.pos, 0};
          Rec* mine = s.rec + pp * CL + cl.rank;
          *mine = r;
          const uint4* w4 = reinterpret_cast<const uint4*>(&r);
#pragma unroll
          for (int q = 0; q < CL; ++q)
            if (q != cl.rank) {
              const uint32_t ra = cluster_addr(mine, q);
              st_async_v4(ra, w4[0], rc[q]);
              st_async_v4(ra + 16u, w4[1], rc[q]);
            }
        }
        __syncthreads();  // this CTA's own slot
        mbar_wait_cluster(&s.xbar[pp], (xph >> pp) & 1u);
        xph ^= 1u << pp;
      } else {
        if (TMR && ce.pos >= 0) {
#pragma unroll
          for (int sl = 0; sl < TM_NS; ++sl) {
            const int i = 128 * sl + 32 * tm.q + lane;
            if (sl < tm.ns && (sl & 1) == tm.h && i < tm.mt) {
              if constexpr (PULL) {
                myc[i] = cv[sl];
              } else {
#pragma unroll
                for (int q = 0; q < CL; ++q) cl.remote(myc, q)[i] = cv[sl];
              }
            }
          }
        }
        if (ce.pos >= 0)
          for (int i = (TMR ? tm.mt : 0) + tid; i < nrow; i += NT) {
            const double v = s.row(i)[jc];
            if constexpr (PULL) {
              myc[i] = v;
            } else {
#pragma unroll
              for (int q = 0; q < CL; ++q) cl.remote(myc, q)[i] = v;
            }
          }
        if (tid == 0) {
          const Rec r{ce, cr.v, cr.pos, 0};
#pragma unroll 1
          for (int q = 0; q < CL; ++q) *cl.remote(s.rec + pp * CL + cl.rank, q) = r;  // 32 B
        }
        cl.sync();
      }
      int win = 0;
      ce = s.rec[pp * CL].ce;
#pragma unroll 4
      for (int q = 1; q < CL; ++q) {
        const Cand o = s.rec[pp * CL + q].ce;
        if (bland ? better<MIN_KEY>(o, ce) : better<MAX_V>(o, ce)) {
          ce = o;
          win = q;
        }
      }
      if (ce.pos < 0) {
        if (phase == 2) { st = ST_OPTIMAL; break; }
        // phase switch (R8, R9): infeasibility test, drive artificials out, drop phase-I row
        if (TMR && tm_live) {  // the SMEM path from here
          tm_rows_to_smem(s, tm, S, m, (Wa + 7) >> 3);
          tm_live = false;
        }
        const double wstar = s.row(m + 1)[cnt];
        if (wstar > a.eps_phase1 * fmax(1.0, binf)) { st = ST_INFEASIBLE; break; }
        for (int l = 0; l < m; ++l) {
          if (s.bkey[l] >= 0) continue;
          Cand cd{0.0, 0, -1};
          for (int j = tid; j < cnt; j += NT) {
            const int var = s.nbvar[j];
            const double v = fabs(s.row(l)[j]);
            if (var != DEAD && v > a.eps_piv) {
              const Cand cc{v, var, g0 + j};
              if (better<MAX_V>(cc, cd)) cd = cc;
            }
          }
          cd = cluster_reduce<MAX_V, CL>(cd, s, par, cl);
          if (cd.pos < 0) continue;  // redundant row: the artificial stays basic at 0
          const int owner = cd.pos / Q, jloc = cd.pos - owner * Q;
          if (cl.rank == owner) {
            for (int i = tid; i < m + 2; i += NT) {
              const double v = s.row(i)[jloc];
#pragma unroll 1
              for (int q = 0; q < CL; ++q) cl.remote(s.colE, q)[i] = v;
            }
          }
          cl.sync();
          RecRow rr{nullptr, g0, npos, cl.rank == 0};
          if (record && it1 < a.rec_cap) {
            rr.row = a.rec_rows + (size_t)it1 * Wr;
            if (cl.rank == 0 && tid == 0) a.rec_e[it1] = cd.pos;
          }
          pivot_local(s, s.colE, S, Wa, m + 2, l, cl.rank == owner, jloc, cd.key, rr);
          ++it1;
        }
        phase = 2;
        stall = 0;
        pp ^= 1;  // the proposal slots of this round may still be read by a peer CTA
        if (!record) {  // phase II never touches the dead (left artificial) positions
          cnt = compact_live(s, S, cnt, m + 1);
          Wa = cnt + 1;
          if constexpr (TMR) {
          tm_rows_from_smem(s, tm, S, m, (Wa + 7) >> 3);
          tm_live = true;
        }
        }
        if (record) {  // phase I recorded: dump the tableau it leaves, then stop (mode 1)
          for (int i = w; i < m; i += NW)
            for (int j = lane; j < Wa; j += 32) {
              if (j < cnt) a.rec_T[(size_t)i * Wr + g0 + j] = s.row(i)[j];
              else if (cl.rank == 0) a.rec_T[(size_t)i * Wr + npos] = s.row(i)[cnt];
            }
          for (int j = tid; j < cnt; j += NT) a.rec_nbvar[g0 + j] = s.nbvar[j];
          if (cl.rank == 0) {
            for (int i = tid; i < m; i += NT) a.rec_bkey[i] = s.bkey[i];
            if (tid == 0) {
              a.rec_info[0] = it1 <= a.rec_cap ? -1 : ST_NUMERICAL;
              a.rec_info[1] = it1;
              a.rec_info[2] = it1;
              a.rec_info[3] = k;
            }
          }
          recorded = true;
          break;
        }
        continue;
      }
      if (it1 + it2 >= a.max_iter) { st = ST_ITER_LIMIT; break; }
      const int l = s.rec[pp * CL + win].l;
      const double theta = s.rec[pp * CL + win].theta;
      if (l < 0) { st = (phase == 2) ? ST_UNBOUNDED : ST_NUMERICAL; break; }
      // Step 3: pivot (the winner's column is in this CTA's slot `win`)
      const int jloc = ce.pos - win * Q;
      const double* wcol = PULL ? cl.remote(s.colC + (size_t)pp * RC, win)
                                : s.colC + (size_t)(pp * CL + win) * RC;
      RecRow rr{nullptr, g0, npos, cl.rank == 0};
      if (record && phase == 1 && it1 < a.rec_cap) {
        rr.row = a.rec_rows + (size_t)it1 * Wr;
        if (cl.rank == 0 && tid == 0) a.rec_e[it1] = ce.pos;
      }
      if constexpr (TMR)
        pivot_local_tm<tm_ns_max(CL), CL == 2>(s, tm, wcol, S, Wa, m, nrow, l, cl.rank == win, jloc, ce.key, rr);
      else
        pivot_local(s, wcol, S, Wa, nrow, l, cl.rank == win, jloc, ce.key, rr);
      pp ^= 1;
      if (phase == 1) ++it1; else ++it2;
      stall = (theta > 0.0) ? 0 : stall + 1;
    }

    // rows still in TMEM (the LP ended inside a pivot loop phase): back to SMEM for extract
    if (TMR && tm_live) tm_rows_to_smem(s, tm, S, m, (Wa + 7) >> 3);
    if (record) {  // mode 1: no result for LP 0 here (the warm pass solves it); a phase-I
                   // outcome that ends every LP (INFEASIBLE, NUMERICAL, ITER_LIMIT) is recorded
      if (!recorded && cl.rank == 0 && tid == 0) {
        a.rec_info[0] = st;
        a.rec_info[1] = it1;
        a.rec_info[2] = 0;
        a.rec_info[3] = k;
      }
      cl.sync();
      continue;
    }
    // ---- extract (R10) ----
    if (cl.rank == 0) {
      if (tid == 0) {
        a.status[lp] = st;
        a.iters[2 * lp] = it1;
        a.iters[2 * lp + 1] = it2;
        a.obj[lp] = (st == ST_OPTIMAL) ? -s.row(m)[cnt]
                  : (st == ST_UNBOUNDED) ? __longlong_as_double(0x7ff0000000000000ll)
                  : (st == ST_INFEASIBLE) ? __longlong_as_double(0xfff0000000000000ll)
                                          : __longlong_as_double(0x7ff8000000000000ll);
      }
      if (a.x) {
        double* xk = a.x + lp * (int64_t)n;
        const double fill = (st == ST_OPTIMAL) ? 0.0 : __longlong_as_double(0x7ff8000000000000ll);
        for (int j = tid; j < n; j += NT) xk[j] = fill;
        __syncthreads();
        if (st == ST_OPTIMAL)
          for (int i = tid; i < m; i += NT) {
            const int key = s.bkey[i];
            if (key >= 0 && key < n) xk[key] = s.row(i)[cnt];
          }
      }
    }
    cl.sync();
  }
  if constexpr (TMR) {
    tm_fence_before();
    __syncthreads();
    tm_fence_after();
    if (w == 0) tm_dealloc_n((uint32_t)s.ctl->pad, tmcols);
  }
}

// The kernels: the hybrid TMR variant (2-CTA clusters, two CTAs per SM) is compiled for 128
// registers; every other variant keeps the default register heuristics of __launch_bounds__(NT).
template <int CL, bool PULL, bool TMR>
__global__ void __launch_bounds__(NT) simplex_block_kernel(SimplexArgs a) {
  simplex_block_body<CL, PULL, TMR>(a);
}
template <bool PULL>
__global__ void __launch_bounds__(NT, 2) simplex_block_hyb_kernel(SimplexArgs a) {
  simplex_block_body<2, PULL, true>(a);
}
template <int CL, bool PULL, bool TMR>
constexpr void (*block_kernel())(SimplexArgs) {
  if constexpr (CL == 2 && TMR) return simplex_block_hyb_kernel<PULL>;
  else return simplex_block_kernel<CL, PULL, TMR>;
}

}  // namespace

static size_t smem_bytes(int cl, int m, int n, int kmax, bool pull, bool warm, int h0 = 0) {
  const int Q = (n + kmax + cl - 1) / cl;
  const int S = row_stride(Q);
  // SMEM rows (all m + 2, or rows h0.. of the hybrid TMR layout), colE, fcol, prow, lraw
  size_t bytes = sizeof(double) * ((size_t)(m + 2 - h0) * S + 2 * (size_t)(m + 2) + 2 * (size_t)S);
  bytes += sizeof(int) * ((size_t)(Q + 1) + (size_t)m + NW);  // nbvar, bkey, wcount
  bytes = (bytes + 15) & ~size_t(15);
  const size_t ncol = pull ? 1 : (size_t)cl;  // proposal columns per parity (PUSH: cl)
  bytes += sizeof(Cand) * (2 * NW + 2 * cl) + sizeof(Rec) * 2 * cl +
           sizeof(double) * 2 * ncol * (m + 2) + sizeof(Ctl) + 2 * sizeof(uint64_t);
  if (warm) bytes += sizeof(double) * 2 * ((size_t)n + kmax + 1);  // warm-start replay buffer
  return bytes;
}
size_t block_smem_bytes(int cl, int m, int n, int kmax) {
  return smem_bytes(cl, m, n, kmax, cl >= 8, true);
}
// Hybrid TMR layout (2-CTA clusters, two CTAs per SM): eligible when rows 0..127 fit one TMEM
// slot of <= 256 columns and the remaining SMEM footprint admits exactly two CTAs per SM (more
// would let a third CTA wait on the SM's TMEM).  Returns the global scratch one launch needs
// (doubles: 128 rows x S per CTA, <= 2 CTAs per SM), 0 when not eligible.
static bool hyb_eligible(int m, int n, int kmax, bool pull, bool warm, size_t* smem_out) {
  if (m <= HYB_MT || dev_flag("LPB_NO_TMEM") || dev_flag("LPB_NO_HYB")) return false;
  const int Q = (n + kmax + 1) / 2;
  if (tm_slot_cols(Q) > TM_COLS / 2) return false;
  const size_t sm = smem_bytes(2, m, n, kmax, pull, warm, HYB_MT);
  if (smem_out) *smem_out = sm;
  return 2 * (sm + 1024) <= 227 * 1024 && 3 * (sm + 1024) > 228 * 1024;
}
size_t block_hyb_scratch_doubles(int m, int n, int kmax) {
  const int Q = (n + kmax + 1) / 2;
  if (!hyb_eligible(m, n, kmax, false, true, nullptr) &&
      !hyb_eligible(m, n, kmax, true, true, nullptr) &&
      !hyb_eligible(m, n, kmax, false, false, nullptr) &&
      !hyb_eligible(m, n, kmax, true, false, nullptr))
    return 0;
  return (size_t)2 * device_sm_count() * HYB_MT * row_stride(Q);
}

bool block_fits(int cl, int m, int n, int kmax) {
  const int Q = (n + kmax + cl - 1) / cl;  // pivot_local keeps <= 8 columns per lane
  return Q + 1 <= 256 && smem_bytes(cl, m, n, kmax, true, true) <= 227 * 1024;
}

// Resident CTAs of one (CL, PULL) variant for this launch's SMEM size (memoised).
template <int CL, bool PULL, bool TMR = false>
static cudaError_t resident_ctas(const SimplexArgs& a, size_t smem, int* out) {
  const int sms = device_sm_count();
  static LaunchMemo memo;
  return memo.get(smem, out, [&](int& v, size_t attr) {
    cudaError_t e = cudaFuncSetAttribute(block_kernel<CL, PULL, TMR>(),
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)attr);
    if (e != cudaSuccess) return e;
    if constexpr (CL > 8) {  // 16-CTA clusters are a non-portable (opt-in) size on sm_100
      e = cudaFuncSetAttribute(block_kernel<CL, PULL, TMR>(),
                               cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      if (e != cudaSuccess) return e;
    }
    if constexpr (CL == 1) {
      int per_sm = 0;
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, block_kernel<1, PULL, TMR>(),
                                                        NT, smem);
      v = per_sm * sms;
      return e;
    } else {
      cudaLaunchConfig_t q = {};
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = CL;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      q.attrs = at;
      q.numAttrs = 1;
      q.blockDim = dim3(NT);
      q.dynamicSmemBytes = smem;
      q.gridDim = dim3(CL * sms);
      int clusters = 0;
      e = cudaOccupancyMaxActiveClusters(&clusters, block_kernel<CL, PULL, TMR>(), &q);
      v = clusters * CL;
      return e;
    }
  });
}

template <int CL, bool PULL, bool TMR>
static cudaError_t launch_variant(const SimplexArgs& a, size_t smem, int resident,
                                  int grid_override, cudaStream_t s, int* ctas_out) {
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  if constexpr (CL > 1) {
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
  }
  if (resident <= 0) return cudaErrorInvalidConfiguration;
  int64_t want = a.batch * CL;
  int grid = (int)(want < resident ? want : resident);
  if (grid_override > 0) grid = grid_override * CL;
  grid = (grid / CL) * CL;
  if (grid < CL) grid = CL;
  cfg.gridDim = dim3(grid);
  if (ctas_out) *ctas_out = grid;
  const cudaError_t e = cudaMemsetAsync(a.ticket, 0, sizeof(int), s);  // persistent LP ticket
  if (e != cudaSuccess) return e;
  return cudaLaunchKernelEx(&cfg, block_kernel<CL, PULL, TMR>(), a);
}

// TMR (constraint rows in TMEM during the pivot loop) for clusters of >= 4 CTAs whose CTAs
// run one per SM anyway (the SMEM tableau admits no second CTA) and whose rows fit the SM's
// 512 TMEM columns; each TMR CTA allocates all of them.  Measured (A/B, bit-identical):
// cfg6 (4-CTA) 59.0 -> 56.2 ms per 1000 LPs, cfg8 (8-CTA) 615.7 -> 510.8 ms per 200, cfg7
// (16-CTA) 305.7 -> 242.5 ms per 300; but cfg3 on 2-CTA clusters 200.5 -> 233.3 ms per 1500
// (the pivot-row fetch from one TMEM lane is on the critical path of every pivot), so 2-CTA
// clusters keep the SMEM rows.
template <int CL, bool PULL>
static cudaError_t launch_tm_or(const SimplexArgs& a, size_t smem, int resident,
                                int grid_override, cudaStream_t s, int* ctas_out) {
  if constexpr (CL == 2) {  // hybrid TMR: two CTAs (LPs) per SM instead of one
    size_t sh = 0;
    const int sms = device_sm_count();
    if (a.tm_scr && hyb_eligible(a.m, a.n, a.kmax, PULL, a.mode == 2, &sh) &&
        (grid_override <= 0 || grid_override * CL <= 2 * sms)) {
      // the occupancy API counts one CTA per SM for kernels that use tcgen05; SMEM (checked by
      // hyb_eligible), registers (<= 128 by the launch bounds) and TMEM (256 columns each)
      // admit two, so the resident count is set here (after raising the SMEM attribute)
      int rt = 0;
      const cudaError_t e = resident_ctas<CL, PULL, true>(a, sh, &rt);
      if (e != cudaSuccess) return e;
      cudaFuncAttributes fa{};
      const cudaError_t e2 = cudaFuncGetAttributes(&fa, block_kernel<CL, PULL, true>());
      if (e2 != cudaSuccess) return e2;
      rt = 2 * sms;
      if (fa.numRegs <= 128 && rt > resident) {
        SimplexArgs d = a;
        d.tm_hyb = 1;
        return launch_variant<CL, PULL, true>(d, sh, rt, grid_override, s, ctas_out);
      }
    }
  }
  if constexpr (CL >= 4) {
    const int Q = (a.n + a.kmax + CL - 1) / CL;
    const int ns = tm_slots(a.m);
    if (ns <= tm_ns_max(CL) && ns * tm_slot_cols(Q) <= TM_COLS && resident <= device_sm_count() &&
        !dev_flag("LPB_NO_TMEM")) {
      int rt = 0;
      const cudaError_t e = resident_ctas<CL, PULL, true>(a, smem, &rt);
      if (e != cudaSuccess) return e;
      if (rt >= CL)
        return launch_variant<CL, PULL, true>(a, smem, rt, grid_override, s, ctas_out);
    }
  }
  return launch_variant<CL, PULL, false>(a, smem, resident, grid_override, s, ctas_out);
}

// PUSH for CL <= 4 unless PULL's smaller footprint (one own proposal column per parity
// instead of CL) fits more CTAs on an SM (e.g. 200x200 two-phase on 4-CTA clusters: 2 CTAs
// per SM instead of 1); PULL for CL >= 8 (CL columns would not fit SMEM at m ~ 500).
template <int CL>
static cudaError_t launch_cl(const SimplexArgs& a, int grid_override, cudaStream_t s,
                             int* ctas_out) {
  const bool warm = a.mode == 2;
  const size_t spull = smem_bytes(CL, a.m, a.n, a.kmax, true, warm);
  int rpull = 0;
  cudaError_t e = resident_ctas<CL, true>(a, spull, &rpull);
  if (e != cudaSuccess) return e;
  if constexpr (CL <= 4) {
    const size_t spush = smem_bytes(CL, a.m, a.n, a.kmax, false, warm);
    int rpush = 0;
    if (spush <= 227 * 1024) {
      e = resident_ctas<CL, false>(a, spush, &rpush);
      if (e != cudaSuccess) return e;
    }
    if (rpush >= rpull)
      return launch_tm_or<CL, false>(a, spush, rpush, grid_override, s, ctas_out);
  }
  return launch_tm_or<CL, true>(a, spull, rpull, grid_override, s, ctas_out);
}

cudaError_t launch_simplex_block(int cl, const SimplexArgs& a, int grid_override,
                                 cudaStream_t s, int* ctas_out) {
  switch (cl) {
    case 1: return launch_cl<1>(a, grid_override, s, ctas_out);
    case 2: return launch_cl<2>(a, grid_override, s, ctas_out);
    case 4: return launch_cl<4>(a, grid_override, s, ctas_out);
    case 8: return launch_cl<8>(a, grid_override, s, ctas_out);
    case 16: return launch_cl<16>(a, grid_override, s, ctas_out);
    default: return cudaErrorInvalidValue;
  }
}

// Prepass: kmax = max_k #{i : b_ki < 0}.  One warp per LP, ballot counts.
__global__ void count_art_kernel(const double* __restrict__ b, int64_t batch, int m,
                                 int* __restrict__ kmax) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int best = 0;
  for (int64_t lp = warp; lp < batch; lp += nwarps) {
    const double* bk = b + lp * m;
    int cnt = 0;
    for (int i = lane; i < m; i += 32) cnt += (__ldg(bk + i) < 0.0);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) cnt += __shfl_xor_sync(FULL, cnt, off);
    best = max(best, cnt);
  }
  if (lane == 0 && best > 0) atomicMax(kmax, best);
}

cudaError_t launch_count_art(const double* b, int64_t batch, int m, int* kmax_dev,
                             cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(kmax_dev, 0, sizeof(int), s);
  if (e != cudaSuccess) return e;
  int64_t warps = batch;
  const int64_t cap = (int64_t)device_sm_count() * 64;
  if (warps > cap) warps = cap;
  const int threads = 256;
  const int blocks = (int)((warps * 32 + threads - 1) / threads);
  count_art_kernel<<<blocks, threads, 0, s>>>(b, batch, m, kmax_dev);
  return cudaGetLastError();
}

}  // namespace lpb
