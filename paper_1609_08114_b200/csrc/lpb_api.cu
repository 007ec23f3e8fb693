// lpb_api.cu — the C ABI (include/lpb.h): contexts, size-class dispatch, the host<->device
// stream pipeline and device-event timing.  No torch types, plain pointers only.
//
// Host pipeline (§4.4: H2D-ST -> kernel -> D2H-res on CUDA streams,
// 10 streams above 100 LPs): the batch is cut into n_chunks contiguous chunks; chunk c
// runs H2D(A,b,c) -> solve kernel -> D2H(results) on its own stream, so chunk c+1's copy
// overlaps chunk c's kernel.  Unlike the paper, only the raw A, b, c cross PCIe (the
// tableau is built on the device), which halves the bytes of a full-tableau H2D.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <vector>

#include "../../include/lpb.h"
#include "lpb_internal.cuh"

namespace lpb {
int device_sm_count() {
  static std::atomic<int> cache[64];  // zero-initialised (static storage)
  int dev = 0;
  cudaGetDevice(&dev);
  int v = 0;
  if (dev >= 0 && dev < 64) v = cache[dev].load(std::memory_order_relaxed);
  if (v == 0) {
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    v = v > 0 ? v : 1;
    if (dev >= 0 && dev < 64) cache[dev].store(v, std::memory_order_relaxed);
  }
  return v;
}
}  // namespace lpb

using namespace lpb;

struct lpb_ctx {
  int64_t batch = 0;
  int m = 0, n = 0, kind = 0;
  lpb_options opt{};
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  // context-owned device results
  int32_t* d_status = nullptr;
  double* d_obj = nullptr;
  double* d_x = nullptr;
  int32_t* d_iters = nullptr;
  // device input buffers for host-pointer solves (allocated on first use)
  double* d_A = nullptr;
  double* d_b = nullptr;
  double* d_c = nullptr;
  int64_t d_A_elems = 0, d_b_elems = 0;  // allocated sizes (shared-constraint solves need one A, b)
  int* d_ticket = nullptr;  // one counter per chunk
  int* d_kmax = nullptr;
  int* d_defer = nullptr;      // S class register kernel: deferred (two-phase) LPs, [batch]
  int* d_defer_cnt = nullptr;  // one counter per chunk
  // L class hybrid TMR layout: per-chunk global scratch for rows 0..127 (allocated on use)
  double* d_tmscr[64] = {};
  size_t tmscr_n[64] = {};
  int* h_kmax = nullptr;    // pinned
  std::vector<cudaStream_t> chunk_streams;
  std::vector<cudaEvent_t> chunk_done;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  cudaEvent_t kev0 = nullptr, kev1 = nullptr;  // around the dominant (solve) kernel
  bool kev_valid = false;
  bool no_timing = false, timing_valid = false;  // LPB_NO_TIMING on the last solve
  bool solved = false, last_nox = false, host_path = false;
  int last_launches = 0, last_class = 0, last_cluster = 0, last_grid = 0;
  long long* prof = nullptr;  // diagnostics: per-CTA phase counters (lpb_set_profile_buffer)
  // phase-I record of a shared-constraint two-phase batch (warm start, NEXT-1)
  double* rec_rows = nullptr;
  double* rec_T = nullptr;
  int* rec_ints = nullptr;  // rec_e[cap] | nbvar[n+kmax] | bkey[m] | info[4]
  int rec_cap = 0, rec_W = 0;
  cudaEvent_t rec_ev = nullptr;  // host pipeline: the phase-I record is complete
  // development build: per-chunk event timeline of the host pipeline (lpb_set_timeline)
  std::vector<cudaEvent_t> tl;
  bool tl_on = false;
  int tl_n = 0;
  char err[256] = {0};
};

static int set_cuda_err(lpb_ctx* c, cudaError_t e, const char* where) {
  if (c) std::snprintf(c->err, sizeof(c->err), "%s: %s", where, cudaGetErrorString(e));
  return LPB_ECUDA;
}

#define LPB_CUDA(ctx, call)                                  \
  do {                                                       \
    cudaError_t e_ = (call);                                 \
    if (e_ != cudaSuccess) return set_cuda_err(ctx, e_, #call); \
  } while (0)

extern "C" int lpb_default_options(lpb_options* o) {
  if (!o) return LPB_EINVAL;
  std::memset(o, 0, sizeof(*o));
  o->struct_size = (int32_t)sizeof(lpb_options);
  o->eps_enter = 1e-9;
  o->eps_piv = 1e-9;
  o->eps_phase1 = 1e-9;
  o->max_iter = 0;
  o->bland_after = 0;
  o->device = -1;
  o->stream = nullptr;
  o->n_chunks = 0;
  o->kernel_class = 0;
  o->grid_ctas = 0;
  o->cluster_ctas = 0;
  o->pivot_rule = LPB_RULE_LPC;
  o->rpc_seed = 0;
  o->lp_index_base = 0;
  o->warm_start = 0;
  o->kmax_hint = -1;
  return LPB_OK;
}

extern "C" const char* lpb_strerror(int err) {
  switch (err) {
    case LPB_OK: return "ok";
    case LPB_EINVAL: return "invalid argument";
    case LPB_ENOMEM: return "out of memory";
    case LPB_ECUDA: return "CUDA error";
    case LPB_ESTATE: return "results requested before a solve";
    case LPB_ETOOBIG: return "no compiled size class fits this LP size";
    default: return "unknown error";
  }
}

extern "C" const char* lpb_last_error(lpb_ctx* c) { return c ? c->err : ""; }

// Size-class capacity check at the best case (no artificial rows).
static bool general_fits_any(int m, int n) {
  return thread_fits(m, n) || warp_fits(m, n, 0) || reg_fits(m, n, 0) || block_fits(1, m, n, 0) ||
         block_fits(2, m, n, 0) || block_fits(4, m, n, 0) || block_fits(8, m, n, 0) ||
         block_fits(16, m, n, 0);
}

extern "C" int lpb_create(lpb_ctx** out, int64_t batch, int32_t m, int32_t n, int32_t kind,
                          const lpb_options* o) {
  if (!out) return LPB_EINVAL;
  *out = nullptr;
  if (batch <= 0 || m <= 0 || n <= 0) return LPB_EINVAL;
  if (kind != LPB_GENERAL && kind != LPB_HYPERBOX) return LPB_EINVAL;
  if (kind == LPB_HYPERBOX && m != 2 * n) return LPB_EINVAL;
  // the simplex kernels hand out LPs with 32-bit ticket counters
  if (kind == LPB_GENERAL && batch > (int64_t)(INT_MAX / 2)) return LPB_EINVAL;
  lpb_options opt;
  lpb_default_options(&opt);
  if (o) {
    if (o->struct_size != (int32_t)sizeof(lpb_options)) return LPB_EINVAL;
    opt = *o;
  }
  if (!(opt.eps_enter >= 0) || !(opt.eps_piv >= 0) || !(opt.eps_phase1 >= 0)) return LPB_EINVAL;
  if (opt.pivot_rule != LPB_RULE_LPC && opt.pivot_rule != LPB_RULE_RPC) return LPB_EINVAL;
  if (opt.cluster_ctas != 0 && opt.cluster_ctas != 2 && opt.cluster_ctas != 4 &&
      opt.cluster_ctas != 8 && opt.cluster_ctas != 16)
    return LPB_EINVAL;
  if (opt.kmax_hint < -1 || opt.kmax_hint > m) return LPB_EINVAL;
  {  // kernel_class: a defined class of this kind (an unknown value would silently run auto)
    const int k = opt.kernel_class;
    const bool ok = kind == LPB_GENERAL
                        ? (k == CLASS_AUTO || k == CLASS_S || k == CLASS_M || k == CLASS_L ||
                           k == CLASS_R || k == CLASS_W)
                        : (k == CLASS_AUTO || k == CLASS_H);
    if (!ok) return LPB_EINVAL;
  }
  if (kind == LPB_GENERAL && !general_fits_any(m, n)) return LPB_ETOOBIG;
  if (kind == LPB_HYPERBOX && (size_t)(n | 1) * 256 * 8 > 200 * 1024) return LPB_ETOOBIG;

  lpb_ctx* c = new (std::nothrow) lpb_ctx();
  if (!c) return LPB_ENOMEM;
  c->batch = batch;
  c->m = m;
  c->n = n;
  c->kind = kind;
  c->opt = opt;
  int dev = opt.device;
  if (dev < 0) {
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) { set_cuda_err(c, e, "cudaGetDevice"); delete c; return LPB_ECUDA; }
  }
  c->device = dev;
  cudaError_t e = cudaSetDevice(dev);
  if (e == cudaSuccess) {
    if (opt.stream) {
      c->stream = (cudaStream_t)opt.stream;
    } else {
      e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
      c->own_stream = true;
    }
  }
  if (e == cudaSuccess) e = cudaMalloc(&c->d_status, sizeof(int32_t) * batch);
  if (e == cudaSuccess) e = cudaMalloc(&c->d_obj, sizeof(double) * batch);
  if (e == cudaSuccess) e = cudaMalloc(&c->d_x, sizeof(double) * batch * (int64_t)n);
  if (e == cudaSuccess) e = cudaMalloc(&c->d_iters, sizeof(int32_t) * 2 * batch);
  // hyperbox LPs take no pivots: their iteration counts read as 0 (never uninitialised)
  if (e == cudaSuccess && kind == LPB_HYPERBOX) e = cudaMemset(c->d_iters, 0, sizeof(int32_t) * 2 * batch);
  if (e == cudaSuccess) e = cudaMalloc(&c->d_ticket, sizeof(int) * 64);
  if (e == cudaSuccess) e = cudaMalloc(&c->d_kmax, sizeof(int));
  if (e == cudaSuccess) e = cudaMallocHost(&c->h_kmax, sizeof(int));
  if (e == cudaSuccess) e = cudaEventCreate(&c->ev0);
  if (e == cudaSuccess) e = cudaEventCreate(&c->ev1);
  if (e == cudaSuccess) e = cudaEventCreate(&c->kev0);
  if (e == cudaSuccess) e = cudaEventCreate(&c->kev1);
  if (e != cudaSuccess) {
    const bool oom = (e == cudaErrorMemoryAllocation);
    set_cuda_err(c, e, "lpb_create");
    lpb_destroy(c);
    return oom ? LPB_ENOMEM : LPB_ECUDA;
  }
  *out = c;
  return LPB_OK;
}

extern "C" int lpb_destroy(lpb_ctx* c) {
  if (!c) return LPB_OK;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (auto s : c->chunk_streams) { cudaStreamSynchronize(s); cudaStreamDestroy(s); }
  for (auto ev : c->chunk_done) cudaEventDestroy(ev);
  for (auto ev : c->tl) cudaEventDestroy(ev);
  cudaFree(c->d_status);
  cudaFree(c->d_obj);
  cudaFree(c->d_x);
  cudaFree(c->d_iters);
  cudaFree(c->d_A);
  cudaFree(c->d_b);
  cudaFree(c->d_c);
  cudaFree(c->d_ticket);
  cudaFree(c->d_kmax);
  cudaFree(c->d_defer);
  cudaFree(c->d_defer_cnt);
  for (double* p : c->d_tmscr) cudaFree(p);
  cudaFree(c->rec_rows);
  cudaFree(c->rec_T);
  cudaFree(c->rec_ints);
  if (c->rec_ev) cudaEventDestroy(c->rec_ev);
  if (c->h_kmax) cudaFreeHost(c->h_kmax);
  if (c->ev0) cudaEventDestroy(c->ev0);
  if (c->ev1) cudaEventDestroy(c->ev1);
  if (c->kev0) cudaEventDestroy(c->kev0);
  if (c->kev1) cudaEventDestroy(c->kev1);
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  delete c;
  return LPB_OK;
}

// Choose the simplex size class for a known kmax (forced class honoured when it fits).
static int choose_class(const lpb_ctx* c, int kmax, int* cl) {
  const int m = c->m, n = c->n;
  const int forced = c->opt.kernel_class;
  *cl = 1;
  if (forced == CLASS_W) return warp_fits(m, n, kmax) ? CLASS_W : -1;
  if (forced == CLASS_R) return reg_fits(m, n, kmax) ? CLASS_R : -1;
  if (forced == CLASS_M) return block_fits(1, m, n, kmax) ? CLASS_M : -1;
  const int fcl = c->opt.cluster_ctas;
  if (fcl > 0 && (forced == CLASS_L || forced == CLASS_AUTO)) {
    if (!block_fits(fcl, m, n, kmax)) return -1;
    *cl = fcl;
    return CLASS_L;
  }
  if (forced == CLASS_L) {
    for (int q : {2, 4, 8, 16})
      if (block_fits(q, m, n, kmax)) { *cl = q; return CLASS_L; }
    return -1;
  }
  if (warp_fits(m, n, kmax)) return CLASS_W;
  if (reg_fits(m, n, kmax)) return CLASS_R;
  if (block_fits(1, m, n, kmax)) return CLASS_M;
  for (int q : {2, 4, 8, 16})
    if (block_fits(q, m, n, kmax)) { *cl = q; return CLASS_L; }
  return -1;
}

static void fill_args(const lpb_ctx* c, SimplexArgs& a, int64_t lp0, int64_t cnt,
                      const double* A, const double* b, const double* cv, bool nox,
                      int kmax, int* ticket, bool sab) {
  const int m = c->m, n = c->n;
  a.batch = cnt;
  a.m = m;
  a.n = n;
  a.A = A;
  a.b = b;
  a.sA = sab ? 0 : (int64_t)c->m * c->n;
  a.sb = sab ? 0 : (int64_t)c->m;
  a.c = cv;
  a.status = c->d_status + lp0;
  a.obj = c->d_obj + lp0;
  a.x = nox ? nullptr : c->d_x + lp0 * n;
  a.iters = c->d_iters + 2 * lp0;
  a.eps_enter = c->opt.eps_enter;
  a.eps_piv = c->opt.eps_piv;
  a.eps_phase1 = c->opt.eps_phase1;
  a.max_iter = c->opt.max_iter > 0 ? c->opt.max_iter : 50 * (n + m);
  a.bland_K = c->opt.bland_after == 0 ? n + m : c->opt.bland_after;
  a.kmax = kmax;
  a.khint = c->opt.kmax_hint;
  a.ticket = ticket;
  a.mode = 0;
  a.rec_cap = 0;
  a.rec_rows = a.rec_T = nullptr;
  a.rec_e = a.rec_nbvar = a.rec_bkey = a.rec_info = nullptr;
  a.rpc = c->opt.pivot_rule == LPB_RULE_RPC ? 1 : 0;
  a.rpc_seed = c->opt.rpc_seed;
  a.lp_base = c->opt.lp_index_base + lp0;
  a.defer_list = nullptr;
  a.defer_cnt = nullptr;
  a.tm_hyb = 0;
  a.tm_scr = nullptr;
  // bulk-copy prefetch needs every LP's A to start 16-byte aligned and be a multiple of 16
  // bytes (m*n even), and to fit SMEM next to the register layouts' small SMEM state
  const int64_t bytes = (int64_t)m * n * 8;
  a.prof = c->prof;
  a.prefetch = (((uintptr_t)A & 15) == 0 && (m * (int64_t)n) % 2 == 0 && bytes <= 100 * 1024 &&
                !dev_flag("LPB_NO_PREFETCH")) ? 1 : 0;
}

// Enqueue the general-LP kernels for one resident chunk on stream s.
// The size class depends on kmax = max #{b_i < 0} (it sets the condensed width n + k):
// when a register layout holds even the worst case k = m, no prepass is needed; otherwise
// one tiny prepass kernel + a 4-byte D2H give kmax first.
// rec_role (shared-constraint warm start only): REC_SELF records phase I and solves on s;
// REC_FIRST also signals c->rec_ev after the record; REC_WAIT solves from the record made
// by the REC_FIRST chunk (waits on rec_ev, no second record).
enum { REC_SELF = 0, REC_FIRST = 1, REC_WAIT = 2 };
static int run_general(lpb_ctx* c, cudaStream_t s, int64_t lp0, int64_t cnt, const double* A,
                       const double* b, const double* cv, bool nox, bool sab, int kmax_known,
                       int* ticket, int* launches, int rec_role = REC_SELF) {
  int kmax = kmax_known >= 0 ? kmax_known : c->opt.kmax_hint;  // the hint: no prepass
  const int forced = c->opt.kernel_class;
  // S (thread per LP) wins on throughput once every SM has a few warps of LPs (measured: 3-4x
  // over the warp-per-LP register layout at 1e5-1e6 LPs of 5x5); below that the warp-per-LP
  // layout has the shorter per-LP latency (cfg1: 1000 LPs).
  const bool s_auto = forced == CLASS_AUTO && thread_fits(c->m, c->n) && cnt >= 8192;
  if (forced == CLASS_S || s_auto) {
    if (!thread_fits(c->m, c->n)) return LPB_ETOOBIG;
    SimplexArgs a;  // worst-case width reserved: no prepass
    fill_args(c, a, lp0, cnt, A, b, cv, nox, c->m, ticket, sab);
    // m, n <= 6: the register kernel, which defers two-phase LPs to the SMEM-slice kernel
    const bool tiny = tiny_fits(c->m, c->n) && !dev_flag("LPB_NO_TINY");
    if (tiny) {
      if (!c->d_defer) {
        LPB_CUDA(c, cudaMalloc(&c->d_defer, sizeof(int) * c->batch));
        LPB_CUDA(c, cudaMalloc(&c->d_defer_cnt, sizeof(int) * 64));
      }
      a.defer_list = c->d_defer + lp0;
      a.defer_cnt = c->d_defer_cnt + (ticket - c->d_ticket);  // the chunk's own counter
    }
    const bool timed = (s == c->stream) && !c->no_timing;
    if (timed) LPB_CUDA(c, cudaEventRecord(c->kev0, s));
    LPB_CUDA(c, tiny ? launch_simplex_tiny(a, s) : launch_simplex_thread(a, s));
    if (timed) {
      LPB_CUDA(c, cudaEventRecord(c->kev1, s));
      c->kev_valid = true;
    }
    *launches += (tiny && c->opt.kmax_hint != 0) ? 2 : 1;  // + list-mode two-phase kernel
    c->last_class = CLASS_S;
    c->last_cluster = 0;
    c->last_grid = 0;
    return LPB_OK;
  }
  // Worst-case capacity (k = m) saves the kmax prepass (a tiny kernel + a 4-byte D2H round
  // trip) -- worth it only when the worst-case register layout is already the one the
  // smallest k would get (tiny LPs); otherwise the exact kmax buys a denser layout (e.g. a
  // warp per LP at 28x28 instead of a 128-thread CTA).
  const int worst_layout = reg_layout(c->m, c->n, c->m);
  const bool r_ok_worst = worst_layout >= 0 && worst_layout == reg_layout(c->m, c->n, 0);
  const int w_worst = warp_layout(c->m, c->n, c->m);
  const bool w_ok_worst = w_worst >= 0 && w_worst == warp_layout(c->m, c->n, 0);
  if (kmax < 0 && w_ok_worst && (forced == CLASS_AUTO || forced == CLASS_W))
    kmax = c->m;  // worst-case capacity, no prepass
  if (kmax < 0 && r_ok_worst && (forced == CLASS_AUTO || forced == CLASS_R))
    kmax = c->m;
  if (kmax < 0) {  // device prepass: kmax over the chunk (one tiny kernel + 4-byte D2H)
    LPB_CUDA(c, launch_count_art(b, sab ? 1 : cnt, c->m, c->d_kmax, s));
    LPB_CUDA(c, cudaMemcpyAsync(c->h_kmax, c->d_kmax, sizeof(int), cudaMemcpyDeviceToHost, s));
    LPB_CUDA(c, cudaStreamSynchronize(s));
    kmax = *c->h_kmax;
    *launches += 1;
  }
  int cl = 1;
  const int klass = choose_class(c, kmax, &cl);
  if (klass < 0) return LPB_ETOOBIG;
  SimplexArgs a;
  fill_args(c, a, lp0, cnt, A, b, cv, nox, kmax, ticket, sab);
  int ctas = 0;
  const bool timed = (s == c->stream) && !c->no_timing;
  if (timed) LPB_CUDA(c, cudaEventRecord(c->kev0, s));
  if (klass == CLASS_W) {
    LPB_CUDA(c, launch_simplex_warp(a, c->opt.grid_ctas, s, &ctas));
  } else if (klass == CLASS_R) {
    LPB_CUDA(c, launch_simplex_reg(a, c->opt.grid_ctas, s, &ctas));
  } else {
    if (klass == CLASS_L && cl == 2) {  // hybrid TMR layout: the chunk's row-0..127 scratch
      const size_t need = block_hyb_scratch_doubles(c->m, c->n, kmax);
      const int slot = (int)(ticket - c->d_ticket);
      if (need > 0 && slot >= 0 && slot < 64) {
        if (c->tmscr_n[slot] < need) {
          cudaFree(c->d_tmscr[slot]);
          c->d_tmscr[slot] = nullptr;
          c->tmscr_n[slot] = 0;
          LPB_CUDA(c, cudaMalloc(&c->d_tmscr[slot], sizeof(double) * need));
          c->tmscr_n[slot] = need;
        }
        a.tm_scr = c->d_tmscr[slot];
      }
    }
    // Shared constraints with an infeasible slack basis (LPB_SHARED_AB, k > 0): phase I
    // depends on A and b only, so it is solved once (mode 1, LP 0) and every LP starts at
    // phase II from that record (mode 2).  Under RPC the phase-I path
    // depends on the LP index, so RPC batches take the cold path.
    const bool warm = sab && kmax > 0 && c->opt.warm_start >= 0 &&
                      c->opt.pivot_rule == LPB_RULE_LPC;
    if (warm) {
      const int W = c->n + kmax + 1;
      const int cap = a.max_iter + c->m;
      if (rec_role == REC_WAIT && (c->rec_cap < cap || c->rec_W < W)) return LPB_ESTATE;
      if (c->rec_cap < cap || c->rec_W < W) {
        cudaFree(c->rec_rows);
        cudaFree(c->rec_T);
        cudaFree(c->rec_ints);
        c->rec_rows = nullptr;
        c->rec_T = nullptr;
        c->rec_ints = nullptr;
        c->rec_cap = c->rec_W = 0;
        LPB_CUDA(c, cudaMalloc(&c->rec_rows, sizeof(double) * (size_t)cap * W));
        LPB_CUDA(c, cudaMalloc(&c->rec_T, sizeof(double) * (size_t)c->m * W));
        LPB_CUDA(c, cudaMalloc(&c->rec_ints, sizeof(int) * ((size_t)cap + W + c->m + 4)));
        c->rec_cap = cap;
        c->rec_W = W;
      }
      a.rec_cap = c->rec_cap;
      a.rec_rows = c->rec_rows;
      a.rec_T = c->rec_T;
      a.rec_e = c->rec_ints;
      a.rec_nbvar = c->rec_ints + c->rec_cap;
      a.rec_bkey = a.rec_nbvar + W;
      a.rec_info = a.rec_bkey + c->m;
      if (rec_role == REC_WAIT) {
        LPB_CUDA(c, cudaStreamWaitEvent(s, c->rec_ev, 0));
      } else {
        SimplexArgs r = a;
        r.mode = 1;
        r.batch = 1;
        LPB_CUDA(c, launch_simplex_block(cl, r, 0, s, &ctas));
        *launches += 1;
        if (rec_role == REC_FIRST) {
          if (!c->rec_ev) LPB_CUDA(c, cudaEventCreateWithFlags(&c->rec_ev, cudaEventDisableTiming));
          LPB_CUDA(c, cudaEventRecord(c->rec_ev, s));
        }
      }
      a.mode = 2;
    }
    LPB_CUDA(c, launch_simplex_block(cl, a, c->opt.grid_ctas, s, &ctas));
  }
  if (timed) {
    LPB_CUDA(c, cudaEventRecord(c->kev1, s));
    c->kev_valid = true;
  }
  *launches += 1;
  c->last_class = klass;
  c->last_cluster = klass == CLASS_L ? cl : 1;
  c->last_grid = ctas;
  return LPB_OK;
}

static int run_hyperbox(lpb_ctx* c, cudaStream_t s, int64_t lp0, int64_t cnt, const double* l,
                        const double* box, bool shared, bool nox, int* launches) {
  HyperboxArgs h;
  h.batch = cnt;
  h.n = c->n;
  h.l = l;
  h.box = box;
  h.shared_box = shared ? 1 : 0;
  h.status = c->d_status + lp0;
  h.obj = c->d_obj + lp0;
  h.x = nox ? nullptr : c->d_x + lp0 * c->n;
  const bool timed = (s == c->stream) && !c->no_timing;
  if (timed) LPB_CUDA(c, cudaEventRecord(c->kev0, s));
  LPB_CUDA(c, launch_hyperbox(h, s));
  if (timed) {
    LPB_CUDA(c, cudaEventRecord(c->kev1, s));
    c->kev_valid = true;
  }
  *launches += 1;
  c->last_class = CLASS_H;
  c->last_cluster = 0;
  c->last_grid = 0;
  return LPB_OK;
}

static int ensure_host_path(lpb_ctx* c, int nch, bool shared) {
  const int64_t B = c->batch;
  // LPB_SHARED_AB / LPB_SHARED_BOX stage one A, b (box); a later per-LP solve grows the buffers
  const int64_t needb = (shared ? 1 : B) * (int64_t)c->m;
  if (c->kind == LPB_GENERAL) {
    const int64_t needA = (shared ? 1 : B) * (int64_t)c->m * c->n;
    if (c->d_A_elems < needA) {
      cudaFree(c->d_A);
      c->d_A = nullptr;
      c->d_A_elems = 0;
      LPB_CUDA(c, cudaMalloc(&c->d_A, sizeof(double) * needA));
      c->d_A_elems = needA;
    }
  }
  if (c->d_b_elems < needb) {
    cudaFree(c->d_b);
    c->d_b = nullptr;
    c->d_b_elems = 0;
    LPB_CUDA(c, cudaMalloc(&c->d_b, sizeof(double) * needb));
    c->d_b_elems = needb;
  }
  if (!c->d_c) LPB_CUDA(c, cudaMalloc(&c->d_c, sizeof(double) * B * (int64_t)c->n));
  while ((int)c->chunk_streams.size() < nch) {
    cudaStream_t s;
    cudaEvent_t ev;
    LPB_CUDA(c, cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    LPB_CUDA(c, cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    c->chunk_streams.push_back(s);
    c->chunk_done.push_back(ev);
  }
  return LPB_OK;
}

static int solve_impl(lpb_ctx* c, const double* A, const double* b, const double* cv,
                      uint32_t flags, int32_t* o_status, double* o_obj, double* o_x,
                      int32_t* o_iters) {
  if (!c) return LPB_EINVAL;
  const bool general = c->kind == LPB_GENERAL;
  if ((general && (!A || !b || !cv)) || (!general && (A || !b || !cv))) return LPB_EINVAL;
  const bool nox = (flags & LPB_NO_X) != 0;
  const bool shared = (flags & LPB_SHARED_BOX) != 0;
  const bool sab = general && (flags & LPB_SHARED_AB) != 0;
  if (o_x && nox) return LPB_EINVAL;
  LPB_CUDA(c, cudaSetDevice(c->device));
  c->solved = false;
  c->kev_valid = false;
  c->no_timing = (flags & LPB_NO_TIMING) && (flags & LPB_DEVICE_PTRS);
  c->timing_valid = true;
  c->last_launches = 0;
  c->last_nox = nox;
  const int64_t B = c->batch;
  const int m = c->m, n = c->n;

  if (flags & LPB_DEVICE_PTRS) {
    c->host_path = false;
    if (!c->no_timing) LPB_CUDA(c, cudaEventRecord(c->ev0, c->stream));
    int rc = general ? run_general(c, c->stream, 0, B, A, b, cv, nox, sab, -1, c->d_ticket,
                                   &c->last_launches)
                     : run_hyperbox(c, c->stream, 0, B, cv, b, shared, nox, &c->last_launches);
    if (rc != LPB_OK) return rc;
    if (!c->no_timing) LPB_CUDA(c, cudaEventRecord(c->ev1, c->stream));
    c->timing_valid = !c->no_timing;
    if (o_status) LPB_CUDA(c, cudaMemcpyAsync(o_status, c->d_status, 4 * B, cudaMemcpyDefault, c->stream));
    if (o_obj) LPB_CUDA(c, cudaMemcpyAsync(o_obj, c->d_obj, 8 * B, cudaMemcpyDefault, c->stream));
    if (o_x) LPB_CUDA(c, cudaMemcpyAsync(o_x, c->d_x, 8 * B * (int64_t)n, cudaMemcpyDefault, c->stream));
    if (o_iters) LPB_CUDA(c, cudaMemcpyAsync(o_iters, c->d_iters, 8 * B, cudaMemcpyDefault, c->stream));
    c->solved = true;
    if (!(flags & LPB_ASYNC)) LPB_CUDA(c, cudaStreamSynchronize(c->stream));
    return LPB_OK;
  }

  // ---- host pointers: chunked H2D -> kernel -> D2H pipeline on n_chunks streams ----
  c->host_path = true;
  // default pipeline depth: the paper's 10 streams for batches > 100 when the
  // inputs are big enough to overlap; a chunk's copies and launch cost ~10 us of fixed
  // latency, so inputs under 1 MiB go as one chunk (reading R16)
  const int64_t in_bytes = 8 * (general ? (sab ? (int64_t)m * n + m + B * (int64_t)n
                                               : B * ((int64_t)m * n + m + n))
                                        : (shared ? 2 * (int64_t)n : 2 * B * (int64_t)n) + B * (int64_t)n);
  int nch = c->opt.n_chunks > 0 ? c->opt.n_chunks
                                : ((B > 100 && in_bytes >= (1 << 20)) ? 10 : 1);
  if (nch > 64) nch = 64;
  if (nch > B) nch = (int)B;
  int rc = ensure_host_path(c, nch, general ? sab : shared);
  if (rc != LPB_OK) return rc;
  // e2e time starts here: the host scan of b below (when there is no kmax_hint) is part of
  // the end-to-end solve
  LPB_CUDA(c, cudaEventRecord(c->ev0, c->stream));
  int kmax = c->opt.kmax_hint;
  if (general && kmax < 0) {  // kmax from the host copy of b (no device round trip inside the pipeline)
    int best = 0;
    for (int64_t k = 0; k < (sab ? 1 : B); ++k) {
      int cnt = 0;
      const double* bk = b + k * m;
      for (int i = 0; i < m; ++i) cnt += (bk[i] < 0.0);
      best = std::max(best, cnt);
    }
    kmax = best;
  }
#ifdef LPB_DEV_HOOKS
  // timeline marks per chunk: [0] before its H2D, [1] H2D done, [2] kernel done, [3] D2H done
#define LPB_TL(q, k) \
  if (c->tl_on) LPB_CUDA(c, cudaEventRecord(c->tl[4 * (q) + (k)], s))
  if (c->tl_on) {
    while ((int)c->tl.size() < 4 * nch) {
      cudaEvent_t ev;
      LPB_CUDA(c, cudaEventCreate(&ev));
      c->tl.push_back(ev);
    }
    c->tl_n = nch;
  }
#else
#define LPB_TL(q, k)
#endif
  for (int q = 0; q < nch; ++q) {
    const int64_t lp0 = B * q / nch, lp1 = B * (q + 1) / nch, cnt = lp1 - lp0;
    cudaStream_t s = c->chunk_streams[q];
    LPB_CUDA(c, cudaStreamWaitEvent(s, c->ev0, 0));
    LPB_TL(q, 0);
    if (general) {
      // shared constraints (LPB_SHARED_AB): A and b cross PCIe once, on the first chunk's
      // stream; the other chunks wait for that copy
      const int64_t sA = sab ? 0 : m * (int64_t)n, sb = sab ? 0 : m;
      if (q == 0 || !sab) {
        LPB_CUDA(c, cudaMemcpyAsync(c->d_A + lp0 * sA, A + lp0 * sA,
                                    8 * (sab ? m * (int64_t)n : cnt * sA),
                                    cudaMemcpyHostToDevice, s));
        LPB_CUDA(c, cudaMemcpyAsync(c->d_b + lp0 * sb, b + lp0 * sb, 8 * (sab ? m : cnt * sb),
                                    cudaMemcpyHostToDevice, s));
      }
      if (sab && q == 0) LPB_CUDA(c, cudaEventRecord(c->chunk_done[0], s));
      if (sab && q > 0) LPB_CUDA(c, cudaStreamWaitEvent(s, c->chunk_done[0], 0));
      LPB_CUDA(c, cudaMemcpyAsync(c->d_c + lp0 * n, cv + lp0 * n, 8 * cnt * n,
                                  cudaMemcpyHostToDevice, s));
      LPB_TL(q, 1);
      rc = run_general(c, s, lp0, cnt, c->d_A + lp0 * sA, c->d_b + lp0 * sb, c->d_c + lp0 * n,
                       nox, sab, kmax, c->d_ticket + q, &c->last_launches,
                       sab ? (q == 0 ? REC_FIRST : REC_WAIT) : REC_SELF);
    } else {
      const int64_t bstride = shared ? 0 : 2 * (int64_t)n;
      if (q == 0 || !shared)
        LPB_CUDA(c, cudaMemcpyAsync(c->d_b + lp0 * bstride, b + lp0 * bstride,
                                    8 * (shared ? 2 * (int64_t)n : cnt * bstride),
                                    cudaMemcpyHostToDevice, s));
      if (shared && q == 0) LPB_CUDA(c, cudaEventRecord(c->chunk_done[0], s));
      if (shared && q > 0) LPB_CUDA(c, cudaStreamWaitEvent(s, c->chunk_done[0], 0));
      LPB_CUDA(c, cudaMemcpyAsync(c->d_c + lp0 * n, cv + lp0 * n, 8 * cnt * n,
                                  cudaMemcpyHostToDevice, s));
      LPB_TL(q, 1);
      rc = run_hyperbox(c, s, lp0, cnt, c->d_c + lp0 * n, c->d_b + lp0 * bstride, shared, nox,
                        &c->last_launches);
    }
    if (rc != LPB_OK) return rc;
    LPB_TL(q, 2);
    if (o_status) LPB_CUDA(c, cudaMemcpyAsync(o_status + lp0, c->d_status + lp0, 4 * cnt, cudaMemcpyDefault, s));
    if (o_obj) LPB_CUDA(c, cudaMemcpyAsync(o_obj + lp0, c->d_obj + lp0, 8 * cnt, cudaMemcpyDefault, s));
    if (o_x) LPB_CUDA(c, cudaMemcpyAsync(o_x + lp0 * n, c->d_x + lp0 * n, 8 * cnt * (int64_t)n, cudaMemcpyDefault, s));
    if (o_iters) LPB_CUDA(c, cudaMemcpyAsync(o_iters + 2 * lp0, c->d_iters + 2 * lp0, 8 * cnt, cudaMemcpyDefault, s));
    LPB_TL(q, 3);
    cudaEvent_t done;
    LPB_CUDA(c, cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
    LPB_CUDA(c, cudaEventRecord(done, s));
    LPB_CUDA(c, cudaStreamWaitEvent(c->stream, done, 0));
    cudaEventDestroy(done);  // destruction is deferred until the event completes
  }
  LPB_CUDA(c, cudaEventRecord(c->ev1, c->stream));
  c->solved = true;
  if (!(flags & LPB_ASYNC)) LPB_CUDA(c, cudaStreamSynchronize(c->stream));
  return LPB_OK;
}

extern "C" int lpb_solve_batch(lpb_ctx* c, const double* A, const double* b, const double* cv,
                               uint32_t flags) {
  return solve_impl(c, A, b, cv, flags, nullptr, nullptr, nullptr, nullptr);
}

extern "C" int lpb_solve_batch_into(lpb_ctx* c, const double* A, const double* b,
                                    const double* cv, uint32_t flags, int32_t* status,
                                    double* obj, double* x, int32_t* iters) {
  return solve_impl(c, A, b, cv, flags, status, obj, x, iters);
}

extern "C" int lpb_results(lpb_ctx* c, int32_t* status, double* obj, double* x,
                           int32_t* iters) {
  if (!c) return LPB_EINVAL;
  if (!c->solved) return LPB_ESTATE;
  if (x && c->last_nox) return LPB_EINVAL;
  LPB_CUDA(c, cudaSetDevice(c->device));
  const int64_t B = c->batch;
  if (status) LPB_CUDA(c, cudaMemcpyAsync(status, c->d_status, 4 * B, cudaMemcpyDefault, c->stream));
  if (obj) LPB_CUDA(c, cudaMemcpyAsync(obj, c->d_obj, 8 * B, cudaMemcpyDefault, c->stream));
  if (x) LPB_CUDA(c, cudaMemcpyAsync(x, c->d_x, 8 * B * (int64_t)c->n, cudaMemcpyDefault, c->stream));
  if (iters) LPB_CUDA(c, cudaMemcpyAsync(iters, c->d_iters, 8 * B, cudaMemcpyDefault, c->stream));
  LPB_CUDA(c, cudaStreamSynchronize(c->stream));
  return LPB_OK;
}

extern "C" int lpb_result_device_ptrs(lpb_ctx* c, int32_t** status, double** obj, double** x,
                                      int32_t** iters) {
  if (!c) return LPB_EINVAL;
  if (status) *status = c->d_status;
  if (obj) *obj = c->d_obj;
  if (x) *x = c->d_x;
  if (iters) *iters = c->d_iters;
  return LPB_OK;
}

extern "C" int lpb_sync(lpb_ctx* c) {
  if (!c) return LPB_EINVAL;
  LPB_CUDA(c, cudaSetDevice(c->device));
  LPB_CUDA(c, cudaStreamSynchronize(c->stream));
  return LPB_OK;
}

extern "C" int lpb_last_timing(lpb_ctx* c, double* solve_ms, double* e2e_ms) {
  if (!c) return LPB_EINVAL;
  if (!c->solved || !c->timing_valid) return LPB_ESTATE;
  LPB_CUDA(c, cudaSetDevice(c->device));
  LPB_CUDA(c, cudaEventSynchronize(c->ev1));
  float ms = 0.f;
  LPB_CUDA(c, cudaEventElapsedTime(&ms, c->ev0, c->ev1));
  if (solve_ms) *solve_ms = c->host_path ? std::nan("") : (double)ms;
  if (e2e_ms) *e2e_ms = (double)ms;
  return LPB_OK;
}

#ifdef LPB_DEV_HOOKS  // development build only (include/dev/lpb_selftest.h)
extern "C" int lpb_set_timeline(lpb_ctx* c, int on) {
  if (!c) return LPB_EINVAL;
  c->tl_on = on != 0;
  return LPB_OK;
}

extern "C" int lpb_last_timeline(lpb_ctx* c, float* out, int max_chunks, int* n_chunks) {
  if (!c || !out || !n_chunks) return LPB_EINVAL;
  if (!c->solved || !c->host_path || !c->tl_on) return LPB_ESTATE;
  LPB_CUDA(c, cudaSetDevice(c->device));
  LPB_CUDA(c, cudaEventSynchronize(c->ev1));
  const int nq = std::min(c->tl_n, max_chunks);
  for (int q = 0; q < nq; ++q)
    for (int k = 0; k < 4; ++k)
      LPB_CUDA(c, cudaEventElapsedTime(out + 4 * q + k, c->ev0, c->tl[4 * q + k]));
  *n_chunks = nq;
  return LPB_OK;
}

extern "C" int lpb_set_profile_buffer(lpb_ctx* c, long long* dev_buf) {
  if (!c) return LPB_EINVAL;
  c->prof = dev_buf;
  return LPB_OK;
}
#endif

extern "C" int lpb_last_kernel_timing(lpb_ctx* c, double* kernel_ms) {
  if (!c || !kernel_ms) return LPB_EINVAL;
  if (!c->solved || !c->kev_valid) return LPB_ESTATE;
  LPB_CUDA(c, cudaSetDevice(c->device));
  LPB_CUDA(c, cudaEventSynchronize(c->kev1));
  float ms = 0.f;
  LPB_CUDA(c, cudaEventElapsedTime(&ms, c->kev0, c->kev1));
  *kernel_ms = (double)ms;
  return LPB_OK;
}

extern "C" int lpb_last_launch_info(lpb_ctx* c, int32_t* launches, int32_t* kernel_class) {
  if (!c) return LPB_EINVAL;
  if (launches) *launches = c->last_launches;
  if (kernel_class) *kernel_class = c->last_class;
  return LPB_OK;
}

extern "C" int lpb_last_launch_shape(lpb_ctx* c, int32_t* cluster_ctas, int32_t* grid_ctas) {
  if (!c) return LPB_EINVAL;
  if (cluster_ctas) *cluster_ctas = c->last_cluster;
  if (grid_ctas) *grid_ctas = c->last_grid;
  return LPB_OK;
}
