// hyperbox.cu — H class: the closed-form hyperbox LP (§6, Eq. 6):
//     max_{x in B} l.x = sum_i l_i h_i,  h_i = lo_i if l_i < 0 else hi_i   (l_i = 0 -> hi_i)
// One LP per thread (the paper also uses one thread per LP), but the
// HBM traffic is staged through shared memory so that every global access is coalesced:
//   1. the CTA's tile of TILE LPs x n directions (a contiguous TILE*n*8-byte run) is read
//      with consecutive 8-byte loads across the block into a padded SMEM tile (odd row
//      stride: the per-thread row reads in step 2 are bank-conflict free);
//   2. each thread evaluates its LP: the sequential chain acc = fma(l_i, h_i, acc),
//      i = 0..n-1 from acc = 0 (the oracle's order, bit-exact), writes h back in place;
//   3. obj/status are stored per thread (coalesced) and x = h leaves through the same
//      coalesced walk.
// The box (2n fp64) is shared by the batch (LPB_SHARED_BOX, the paper's experiment,
// PAPER.md:313) and lives in SMEM; a per-LP box is read from global memory.
// This kernel is HBM-bound: 8n bytes in + (8n + 12) bytes out per LP.
#include <algorithm>
#include <cstdlib>

#include "lpb_async.cuh"

#include "lpb_internal.cuh"

namespace lpb {
namespace {

constexpr int HB_NT = 256;  // threads = LPs per tile

__global__ void __launch_bounds__(HB_NT) hyperbox_kernel(HyperboxArgs a) {
  extern __shared__ __align__(16) double hsm[];
  const int n = a.n;
  const int S = n | 1;
  double* tile = hsm;                      // HB_NT x S
  double* blo = tile + (size_t)HB_NT * S;  // n
  double* bhi = blo + n;                   // n
  const int tid = threadIdx.x;
  if (a.shared_box) {
    for (int i = tid; i < n; i += HB_NT) {
      bhi[i] = a.box[i];
      blo[i] = -a.box[n + i];
    }
  }
  // incremental divmod of the flat tile index by n
  const int r0 = tid / n, j0 = tid - r0 * n;
  const int dq = HB_NT / n, dr = HB_NT - dq * n;
  const int64_t ntiles = (a.batch + HB_NT - 1) / HB_NT;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t lp0 = t * HB_NT;
    const int64_t left = a.batch - lp0;
    const int rows = left < HB_NT ? (int)left : HB_NT;
    const int total = rows * n;
    const double* __restrict__ src = a.l + lp0 * n;
    {
      // batches of UNR independent streaming loads per thread before the SMEM stores, so that
      // UNR x 256 x (CTAs/SM) 8-byte loads are in flight per SM (latency x bandwidth)
      constexpr int UNR = 8;
      int r = r0, j = j0;
      for (int f0 = 0; f0 < total; f0 += UNR * HB_NT) {
        double v[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
          const int f = f0 + u * HB_NT + tid;
          v[u] = (f < total) ? __ldcs(src + f) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
          const int f = f0 + u * HB_NT + tid;
          if (f < total) tile[r * S + j] = v[u];
          j += dr;
          r += dq;
          if (j >= n) { j -= n; ++r; }
        }
      }
    }
    __syncthreads();
    if (tid < rows) {
      const int64_t lp = lp0 + tid;
      const double* lo = blo;
      const double* hi = bhi;
      if (!a.shared_box) {
        // per-LP box from global memory (b = [hi; -lo] per LP)
        const double* bx = a.box + lp * 2 * (int64_t)n;
        double* row = tile + tid * S;
        bool empty = false;
        double acc = 0.0;
        for (int i = 0; i < n; ++i) {
          const double h_hi = __ldg(bx + i), h_lo = -__ldg(bx + n + i);
          empty |= (h_lo > h_hi);
          const double li = row[i];
          const double h = (li < 0.0) ? h_lo : h_hi;
          acc = __fma_rn(li, h, acc);
          row[i] = h;
        }
        a.status[lp] = empty ? ST_INFEASIBLE : ST_OPTIMAL;
        a.obj[lp] = empty ? __longlong_as_double(0xfff0000000000000ll) : acc;
        if (empty)
          for (int i = 0; i < n; ++i) row[i] = __longlong_as_double(0x7ff8000000000000ll);
      } else {
        double* row = tile + tid * S;
        bool empty = false;
        double acc = 0.0;
        for (int i = 0; i < n; ++i) {
          const double li = row[i];
          const double h = (li < 0.0) ? lo[i] : hi[i];
          empty |= (lo[i] > hi[i]);
          acc = __fma_rn(li, h, acc);
          row[i] = h;
        }
        __stcs(a.status + lp, empty ? ST_INFEASIBLE : ST_OPTIMAL);
        __stcs(a.obj + lp, empty ? __longlong_as_double(0xfff0000000000000ll) : acc);
        if (empty)
          for (int i = 0; i < n; ++i) row[i] = __longlong_as_double(0x7ff8000000000000ll);
      }
    }
    __syncthreads();
    if (a.x) {
      double* __restrict__ dst = a.x + lp0 * n;
      int r = r0, j = j0;
      for (int f = tid; f < total; f += HB_NT) {
        __stcs(dst + f, tile[r * S + j]);
        j += dr;
        r += dq;
        if (j >= n) { j -= n; ++r; }
      }
    }
    __syncthreads();
  }
}


// Shared-box fast path: tiles of LPT*256 directions stream HBM -> SMEM with bulk async copies
// (cp.async.bulk, one per tile) through a STAGES-deep ring, so several tiles per SM are in
// flight while the current one is evaluated (HBM latency x bandwidth needs ~44 KB in flight
// per SM).  Each thread evaluates its LPs from its SMEM row (128-bit reads when n is even)
// and writes h back in place; x then leaves the SM as ONE bulk async store per tile
// (cp.async.bulk shared -> global, TMA engine), so the SM issues no per-element global
// stores.  The ragged tail (< one tile) is evaluated by the next CTA in round-robin order
// straight from global memory, inside the same launch.
__device__ __forceinline__ double hb_eval_row(double* row, int n, const double* blo,
                                              const double* bhi, bool empty, bool wb) {
  // acc = fma(l_i, h_i, acc) over i = 0..n-1 from 0 (the oracle's order); h written back
  const double nan = __longlong_as_double(0x7ff8000000000000ll);
  double acc = 0.0;
  if ((n & 1) == 0) {
    double2* r2 = reinterpret_cast<double2*>(row);
    for (int i2 = 0; i2 < (n >> 1); ++i2) {
      double2 v = r2[i2];
      const double h0 = (v.x < 0.0) ? blo[2 * i2] : bhi[2 * i2];
      acc = __fma_rn(v.x, h0, acc);
      const double h1 = (v.y < 0.0) ? blo[2 * i2 + 1] : bhi[2 * i2 + 1];
      acc = __fma_rn(v.y, h1, acc);
      if (wb) r2[i2] = make_double2(empty ? nan : h0, empty ? nan : h1);
    }
  } else {
    for (int i = 0; i < n; ++i) {
      const double li = row[i];
      const double h = (li < 0.0) ? blo[i] : bhi[i];
      acc = __fma_rn(li, h, acc);
      if (wb) row[i] = empty ? nan : h;
    }
  }
  return acc;
}

__global__ void __launch_bounds__(HB_NT, 1)
hyperbox_tma_kernel(HyperboxArgs a, int lpt, int stages, int bulk_x) {
  extern __shared__ __align__(16) unsigned char hraw[];
  const int n = a.n, tid = threadIdx.x;
  const int tile_lps = lpt * HB_NT;
  const size_t tile_elems = (size_t)tile_lps * n;
  const uint32_t tile_bytes = (uint32_t)(tile_elems * 8);
  uint64_t* mbar = reinterpret_cast<uint64_t*>(hraw);                 // [stages]
  double* blo = reinterpret_cast<double*>(hraw + 16 * 8);            // [n]
  double* bhi = blo + n;                                              // [n]
  double* buf = bhi + n + ((2 * n) & 1);                              // [stages][tile]
  buf = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(buf) + 15) & ~uintptr_t(15));
  for (int i = tid; i < n; i += HB_NT) {
    bhi[i] = a.box[i];
    blo[i] = -a.box[n + i];
  }
  bool empty = false;
  for (int i = 0; i < n; ++i) empty |= (-a.box[n + i] > a.box[i]);
  const double ninf = __longlong_as_double(0xfff0000000000000ll);
  const int64_t nfull = a.batch / tile_lps;  // full tiles go through the TMA ring
  const int64_t G = gridDim.x;
  if (tid == 0) {
    for (int st = 0; st < stages; ++st) mbar_init(&mbar[st], 1);
    for (int st = 0; st < stages; ++st) {
      const int64_t t = blockIdx.x + (int64_t)st * G;
      if (t < nfull) bulk_load(buf + st * tile_elems, a.l + t * tile_elems, tile_bytes, &mbar[st]);
    }
  }
  __syncthreads();
  const bool wx = a.x != nullptr;
  const int j0 = tid % n, dr = HB_NT % n;
  int k = 0;
  for (int64_t t = blockIdx.x; t < nfull; t += G, ++k) {
    const int st = k % stages;
    mbar_wait(&mbar[st], (uint32_t)((k / stages) & 1));
    double* tb = buf + st * tile_elems;
    const int64_t lp0 = t * tile_lps;
    for (int q = 0; q < lpt; ++q) {
      const int r = q * HB_NT + tid;
      const double acc = hb_eval_row(tb + (size_t)r * n, n, blo, bhi, empty, wx && bulk_x);
      __stcs(a.status + lp0 + r, empty ? ST_INFEASIBLE : ST_OPTIMAL);
      __stcs(a.obj + lp0 + r, empty ? ninf : acc);
    }
    if (wx && bulk_x) {
      fence_proxy_async_smem();  // the in-place h writes, before the async-proxy store reads
      __syncthreads();
      if (tid == 0) {
        bulk_store(a.x + lp0 * n, tb, tile_bytes);
        bulk_commit();
        // the store of the previous tile has finished reading its stage: refill that stage
        bulk_wait_read<1>();
        if (k > 0) {
          const int sp = (k - 1) % stages;
          const int64_t tn = t - G + (int64_t)stages * G;
          if (tn < nfull)
            bulk_load(buf + sp * tile_elems, a.l + tn * tile_elems, tile_bytes, &mbar[sp]);
        }
      }
    } else {
      if (wx) {  // coalesced per-thread stores of x from the sign of l
        double* __restrict__ dst = a.x + lp0 * n;
        const int total = tile_lps * n;
        int j = j0;
        for (int f = tid; f < total; f += HB_NT) {
          const double li = tb[f];
          __stcs(dst + f, empty ? __longlong_as_double(0x7ff8000000000000ll)
                                : ((li < 0.0) ? blo[j] : bhi[j]));
          j += dr;
          if (j >= n) j -= n;
        }
      }
      __syncthreads();  // every read of this stage is done: refill it
      if (tid == 0) {
        const int64_t tn = t + (int64_t)stages * G;
        if (tn < nfull) bulk_load(tb, a.l + tn * tile_elems, tile_bytes, &mbar[st]);
      }
    }
  }
  if (wx && bulk_x && tid == 0) {
    // the last tile's stage was never refilled; make every store complete before exit
    bulk_wait_all();
  }
  // ragged tail (< one tile): the next CTA in round-robin order, straight from global memory
  const int64_t done = nfull * tile_lps;
  if (done < a.batch && blockIdx.x == nfull % G) {
    const double nan = __longlong_as_double(0x7ff8000000000000ll);
    for (int64_t lp = done + tid; lp < a.batch; lp += HB_NT) {
      const double* li = a.l + lp * n;
      double acc = 0.0;
      for (int i = 0; i < n; ++i) {
        const double l_i = __ldg(li + i);
        const double h = (l_i < 0.0) ? blo[i] : bhi[i];
        acc = __fma_rn(l_i, h, acc);
        if (wx) a.x[lp * n + i] = empty ? nan : h;
      }
      a.status[lp] = empty ? ST_INFEASIBLE : ST_OPTIMAL;
      a.obj[lp] = empty ? ninf : acc;
    }
  }
}

}  // namespace

static cudaError_t launch_hyperbox_plain(const HyperboxArgs& a, cudaStream_t s) {
  const int S = a.n | 1;
  const size_t smem = sizeof(double) * ((size_t)HB_NT * S + 2 * (size_t)a.n);
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  static LaunchMemo memo;
  int per_sm = 0;
  const cudaError_t em = memo.get(smem, &per_sm, [&](int& v, size_t attr) {
    cudaError_t e = cudaFuncSetAttribute(hyperbox_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)attr);
    if (e != cudaSuccess) return e;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, hyperbox_kernel, HB_NT, smem);
  });
  if (em != cudaSuccess) return em;
  const int64_t ntiles = (a.batch + HB_NT - 1) / HB_NT;
  int64_t grid = (int64_t)per_sm * device_sm_count();
  if (grid > ntiles) grid = ntiles;
  if (grid < 1) grid = 1;
  hyperbox_kernel<<<(unsigned)grid, HB_NT, smem, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_hyperbox(const HyperboxArgs& a, cudaStream_t s) {
  // Shared box and 16-byte aligned directions: TMA-ring kernel over the full tiles, the plain
  // kernel over the ragged tail (and for per-LP boxes).
  const int n = a.n;
  int lpt = 1;
  // tiles of ~20-56 KB: measured best on cfg4 (n=5: 2x256 LPs, 20 KB, 0.070 vs 0.076 ms at
  // 40 KB and 0.087 ms at 10 KB) and cfg5 (n=28: 256 LPs, 56 KB, 3 stages)
  while (lpt < 8 && (size_t)(2 * lpt) * HB_NT * n * 8 <= 32 * 1024) lpt *= 2;
#ifdef LPB_DEV_HOOKS
  if (const char* v = getenv("LPB_HB_LPT")) {  // tuning hook: a power of two in [1, 8]
    const int q = atoi(v);
    lpt = q >= 8 ? 8 : q >= 4 ? 4 : q >= 2 ? 2 : 1;
  }
#endif
  const size_t tile_bytes = (size_t)lpt * HB_NT * n * 8;
  int stages = (int)((200 * 1024) / tile_bytes);
  int smax = 4;
#ifdef LPB_DEV_HOOKS
  if (const char* v = getenv("LPB_HB_STAGES")) smax = std::max(2, std::min(8, atoi(v)));  // tuning hook
#endif
  if (stages > smax) stages = smax;
  const bool tma = a.shared_box && stages >= 2 && (tile_bytes % 16) == 0 &&
                   (reinterpret_cast<uintptr_t>(a.l) & 15) == 0 && !dev_flag("LPB_NO_TMA");
  const int64_t tile_lps = (int64_t)lpt * HB_NT;
  const int64_t nfull = tma ? a.batch / tile_lps : 0;
  if (nfull > 0) {
    // x leaves by bulk store when its tiles are 16-byte aligned (always for cudaMalloc'd x
    // and tile-aligned chunks); otherwise by coalesced per-thread stores
    const int bulk_x = (a.x != nullptr && (reinterpret_cast<uintptr_t>(a.x) & 15) == 0 &&
                        !dev_flag("LPB_NO_BULK_X")) ? 1 : 0;
    const size_t smem = 16 * 8 + 16 * (size_t)((2 * n + 2 + 1) / 2) + 16 + stages * tile_bytes;
    static LaunchMemo memo;
    int ok = 0;
    const cudaError_t em = memo.get(smem, &ok, [&](int& v, size_t attr) {
      v = 1;
      return cudaFuncSetAttribute(hyperbox_tma_kernel,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)attr);
    });
    if (em != cudaSuccess) return em;
    int64_t grid = device_sm_count();
    if (grid > nfull) grid = nfull;
    hyperbox_tma_kernel<<<(unsigned)grid, HB_NT, smem, s>>>(a, lpt, stages, bulk_x);
    return cudaGetLastError();  // the ragged tail is handled inside the same launch
  }
  const int64_t done = nfull * tile_lps;
  if (done < a.batch) {
    HyperboxArgs t = a;
    t.batch = a.batch - done;
    t.l = a.l + done * n;
    t.status = a.status + done;
    t.obj = a.obj + done;
    t.x = a.x ? a.x + done * n : nullptr;
    if (!a.shared_box) t.box = a.box + done * 2 * (int64_t)n;
    return launch_hyperbox_plain(t, s);
  }
  return cudaSuccess;
}

}  // namespace lpb
