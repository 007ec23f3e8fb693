// simplex_thread.cu — S class: one LP per THREAD for tiny LPs (m, n <= 8; cfg1 is 5x5).
//
// For a 5x5 LP a pivot touches ~40 tableau elements; any cooperative mapping spends its time
// in warp reductions and barriers.  Here each thread runs the whole method (§3.1
// Steps 1-3, two phases PAPER.md:76) sequentially on its own condensed tableau, held in a
// thread-private slice of shared memory (odd stride: the 32 threads of a warp hit 32 distinct
// banks at every step, dynamic indexing is free).  No barrier, no shuffle; warps run 32 LPs in
// lock step (the batch-interleaved SIMT the paper's one-thread-per-LP hyperbox kernel uses,
// PAPER.md:303).  The worst-case width n+m+1 is reserved, so no prepass is needed.
// Arithmetic is the oracle's, element for element (same division, fma and sum order).
#include <algorithm>
#include <climits>

#include "lpb_fp64.cuh"
#include "lpb_internal.cuh"
#include "lpb_rng.cuh"

namespace lpb {
namespace {

constexpr int S_NT = 32;       // threads (LPs) per CTA: spreads small batches over many SMs
constexpr int S_MAXM = 8, S_MAXN = 8;
constexpr int DEADV = INT_MAX;

__device__ __forceinline__ double sdiv(double a, double b) {
  bool slow;
  const double q = div_fast(a, b, slow);
  return slow ? __ddiv_rn(a, b) : q;
}

// Solve LP `lp` of the launch on thread `tid`'s SMEM slice.
__device__ __forceinline__ void s_solve(const SimplexArgs& a, int64_t lp, int tid, double* ssm) {
  const int m = a.m, n = a.n;
  const int W = n + m + 1;     // positions n+m (worst case k = m) + RHS
  const int S = ((m + 2) * W) | 1;
  double* T = ssm + (size_t)tid * S;                                // (m+2) x W, row stride W
  int* ib = reinterpret_cast<int*>(ssm + (size_t)S_NT * S) + tid;  // int slices, stride S_NT
  // int arrays (interleaved across threads: element q of thread t at ib[q * S_NT])
  auto bkey = [&](int i) -> int& { return ib[i * S_NT]; };
  auto nbv = [&](int p) -> int& { return ib[(S_MAXM + p) * S_NT]; };
  auto neg = [&](int t) -> int& { return ib[(S_MAXM + S_MAXM + S_MAXN + t) * S_NT]; };
  const double* Ak = a.A + lp * a.sA;
  const double* bk = a.b + lp * a.sb;
  const double* ck = a.c + lp * (int64_t)n;

  // ---- build (R7) ----
  int k = 0;
  double binf = 0.0;
  for (int i = 0; i < m; ++i) {
    const double bi = __ldg(bk + i);
    binf = fmax(binf, fabs(bi));
    if (bi < 0.0) {
      neg(k++) = i;
      bkey(i) = i - m;
    } else {
      bkey(i) = n + i;
    }
  }
  const int npos = n + k, rhs = npos;  // RHS at column npos
  const bool bad_hint = a.khint >= 0 && k > a.khint;
  for (int i = 0; i < m; ++i) {
    const bool ng = bkey(i) < 0;
    double* row = T + i * W;
    for (int j = 0; j < n; ++j) {
      const double v = __ldg(Ak + i * n + j);
      row[j] = ng ? -v : v;
    }
    for (int t = 0; t < k; ++t) row[n + t] = (i == neg(t)) ? -1.0 : (ng ? -0.0 : 0.0);
    const double bi = __ldg(bk + i);
    row[rhs] = ng ? -bi : bi;
  }
  for (int j = 0; j <= npos; ++j) T[m * W + j] = (j < n) ? __ldg(ck + j) : 0.0;
  for (int p = 0; p < npos; ++p) nbv(p) = p < n ? p : n + neg(p - n);
  if (k > 0)
    for (int j = 0; j <= npos; ++j) {
      double acc = 0.0;
      for (int t = 0; t < k; ++t) acc = __dadd_rn(acc, T[neg(t) * W + j]);
      T[(m + 1) * W + j] = acc;
    }

  int st = bad_hint ? ST_BAD_HINT : -1, it1 = 0, it2 = 0, stall = 0, phase = k > 0 ? 1 : 2;
  const uint64_t lpkey = a.rpc ? rpc_lp_key(a.rpc_seed, a.lp_base + lp) : 0ull;
  auto pivot = [&](int l, int e, int nrow) {
    const double pe = T[l * W + e];
    const double r = recip_of(pe);
    double* rowl = T + l * W;
    for (int j = 0; j <= npos; ++j) {
      const double num = (j == e) ? 1.0 : rowl[j];
      bool slow;
      const double q = div_with(num, pe, r, slow);
      rowl[j] = slow ? __ddiv_rn(num, pe) : q;
    }
    for (int i = 0; i < nrow; ++i) {
      if (i == l) continue;
      double* row = T + i * W;
      const double f = -row[e];
      for (int j = 0; j <= npos; ++j)
        row[j] = __fma_rn(f, rowl[j], (j == e) ? 0.0 : row[j]);
    }
    const int leaving = bkey(l);
    bkey(l) = nbv(e);
    nbv(e) = leaving < 0 ? DEADV : leaving;
  };
  while (st < 0) {
    const int orow = phase == 1 ? m + 1 : m;
    const int nrow = phase == 1 ? m + 2 : m + 1;
    const bool bland = a.bland_K > 0 && stall >= a.bland_K;
    // Step 1 (LPC / Dantzig, lowest variable index on ties; RPC: largest counter-based
    // score u_j, include/lpb.h; Bland)
    int e = -1, ev = INT_MAX;
    double best = 0.0;
    const bool rpc = a.rpc && !bland;
    const uint64_t pkey = rpc ? rpc_pivot_key(lpkey, it1 + it2) : 0ull;
    uint64_t ubest = 0;
    for (int p = 0; p < npos; ++p) {
      const int var = nbv(p);
      const double d = T[orow * W + p];
      if (var == DEADV || !(d > a.eps_enter)) continue;
      if (rpc) {
        const uint64_t u = rpc_score(pkey, var);
        if (e < 0 || u > ubest || (u == ubest && var < ev)) {
          e = p;
          ev = var;
          ubest = u;
        }
        continue;
      }
      if (bland ? (var < ev) : (e < 0 || d > best || (d == best && var < ev))) {
        e = p;
        ev = var;
        best = d;
      }
    }
    if (e < 0) {
      if (phase == 2) { st = ST_OPTIMAL; break; }
      if (T[(m + 1) * W + rhs] > a.eps_phase1 * fmax(1.0, binf)) { st = ST_INFEASIBLE; break; }
      for (int l = 0; l < m; ++l) {  // drive-out (R9)
        if (bkey(l) >= 0) continue;
        int ed = -1, edv = INT_MAX;
        double bv = 0.0;
        for (int p = 0; p < npos; ++p) {
          const int var = nbv(p);
          const double v = fabs(T[l * W + p]);
          if (var == DEADV || !(v > a.eps_piv)) continue;
          if (ed < 0 || v > bv || (v == bv && var < edv)) { ed = p; edv = var; bv = v; }
        }
        if (ed < 0) continue;
        pivot(l, ed, m + 2);
        ++it1;
      }
      phase = 2;
      stall = 0;
      continue;
    }
    if (it1 + it2 >= a.max_iter) { st = ST_ITER_LIMIT; break; }
    // Step 2 (ratio test, R1/R2/R5)
    int l = -1, lkey = INT_MAX;
    double theta = 0.0;
    for (int i = 0; i < m; ++i) {
      const double ai = T[i * W + e];
      if (!(ai > a.eps_piv)) continue;
      const double rr = sdiv(T[i * W + rhs], ai);
      const int key = bland ? bkey(i) : i;
      if (l < 0 || rr < theta || (rr == theta && key < lkey)) { l = i; lkey = key; theta = rr; }
    }
    if (l < 0) { st = phase == 2 ? ST_UNBOUNDED : ST_NUMERICAL; break; }
    pivot(l, e, nrow);
    if (phase == 1) ++it1; else ++it2;
    stall = (theta > 0.0) ? 0 : stall + 1;
  }
  a.status[lp] = st;
  a.iters[2 * lp] = it1;
  a.iters[2 * lp + 1] = it2;
  a.obj[lp] = (st == ST_OPTIMAL) ? -T[m * W + rhs]
            : (st == ST_UNBOUNDED) ? __longlong_as_double(0x7ff0000000000000ll)
            : (st == ST_INFEASIBLE) ? __longlong_as_double(0xfff0000000000000ll)
                                    : __longlong_as_double(0x7ff8000000000000ll);
  if (a.x) {
    double* xk = a.x + lp * (int64_t)n;
    const double fill = (st == ST_OPTIMAL) ? 0.0 : __longlong_as_double(0x7ff8000000000000ll);
    for (int j = 0; j < n; ++j) xk[j] = fill;
    if (st == ST_OPTIMAL)
      for (int i = 0; i < m; ++i) {
        const int key = bkey(i);
        if (key >= 0 && key < n) xk[key] = T[i * W + rhs];
      }
  }
}

// One LP per thread; in list mode (a.defer_cnt set) a grid-stride loop over the LPs the
// register kernel (simplex_tiny.cu) deferred.
__global__ void __launch_bounds__(S_NT) simplex_thread_kernel(SimplexArgs a) {
  extern __shared__ __align__(16) double ssm[];
  const int tid = threadIdx.x;
  if (a.defer_cnt != nullptr) {
    const int cnt = *a.defer_cnt;
    for (int64_t q = (int64_t)blockIdx.x * S_NT + tid; q < cnt; q += (int64_t)gridDim.x * S_NT)
      s_solve(a, a.defer_list[q], tid, ssm);
    return;
  }
  const int64_t lp = (int64_t)blockIdx.x * S_NT + tid;
  if (lp < a.batch) s_solve(a, lp, tid, ssm);
}

size_t thread_smem_bytes(int m, int n) {
  const int S = ((m + 2) * (n + m + 1)) | 1;
  return (size_t)S_NT * S * 8 + (size_t)S_NT * (2 * S_MAXM + S_MAXN + S_MAXM) * 4;
}

}  // namespace

bool thread_fits(int m, int n) { return m <= S_MAXM && n <= S_MAXN; }

cudaError_t launch_simplex_thread(const SimplexArgs& a, cudaStream_t s) {
  const size_t smem = thread_smem_bytes(a.m, a.n);
  static LaunchMemo memo;
  int ok = 0;
  const cudaError_t em = memo.get(smem, &ok, [&](int& v, size_t attr) {
    v = 1;
    return cudaFuncSetAttribute(simplex_thread_kernel,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)attr);
  });
  if (em != cudaSuccess) return em;
  int64_t grid = (a.batch + S_NT - 1) / S_NT;
  // list mode: the deferred count is only known on the device; a few CTAs per SM cover it
  if (a.defer_cnt != nullptr) grid = std::min<int64_t>(grid, (int64_t)device_sm_count() * 4);
  simplex_thread_kernel<<<(unsigned)grid, S_NT, smem, s>>>(a);
  return cudaGetLastError();
}

}  // namespace lpb
