// lpb_internal.cuh — kernel argument blocks and launcher declarations shared by the
// translation units of liblpb.so (never installed; the public ABI is include/lpb.h).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#include <mutex>

namespace lpb {

// Per-LP status codes (must equal LPB_OPTIMAL.. in include/lpb.h).
enum : int32_t { ST_OPTIMAL = 0, ST_UNBOUNDED = 1, ST_INFEASIBLE = 2, ST_ITER_LIMIT = 3,
                 ST_NUMERICAL = 4, ST_BAD_HINT = 5 };

// Size classes (lpb_options.kernel_class / lpb_last_launch_info).
// (6 was a row-per-thread register class, removed in round 2: never auto-selected and
// measured 6 % slower than R on its only candidate sizes; the value stays unused)
enum : int32_t { CLASS_AUTO = 0, CLASS_S = 1, CLASS_M = 2, CLASS_L = 3, CLASS_R = 4,
                 CLASS_H = 5, CLASS_W = 7 };

struct SimplexArgs {
  int64_t batch;
  int m, n;
  const double* A;  // batch x m x n (LP k at A + k * sA)
  const double* b;  // batch x m     (LP k at b + k * sb)
  int64_t sA, sb;   // per-LP strides in elements: m*n and m, or 0 (LPB_SHARED_AB)
  const double* c;  // batch x n
  int32_t* status;
  double* obj;
  double* x;        // may be null (LPB_NO_X)
  int32_t* iters;   // batch x 2
  double eps_enter, eps_piv, eps_phase1;
  int max_iter;     // > 0
  int bland_K;      // > 0: Bland mode after K consecutive degenerate pivots; <= 0: never
  int kmax;         // layout capacity for artificial (b_i < 0) rows
  int khint;        // lpb_options.kmax_hint (-1: none): an LP with more b_i < 0 reports
                    // ST_BAD_HINT unsolved (the caller broke its promise)
  int* ticket;      // persistent-scheduler counter, zeroed before each launch
  int prefetch;     // R class: A (m*n*8 bytes, 16-B aligned per LP) is bulk-prefetched to SMEM
  long long* prof;  // optional per-CTA phase cycle counters (diagnostics), normally null
  int rpc;           // Step 1 rule: 0 LPC (Dantzig), 1 RPC (include/lpb.h LPB_RULE_RPC)
  uint64_t rpc_seed;
  int64_t lp_base;   // index in the lpb_solve_batch call of this launch's LP 0 (RPC key)
  // Phase-I warm start for shared-constraint two-phase batches (M/L classes; SURVEY §8(f)
  // NEXT-1): phase I depends on A and b only, so it runs once (mode 1, LP 0) and records its
  // pivot rows; mode 2 starts every LP at phase II from the recorded tableau, its carried
  // phase-II row rebuilt by replaying the recorded pivots (the same fma sequence, bit-exact).
  int mode;            // 0 normal, 1 record phase I of LP 0, 2 warm start from the record
  int rec_cap;         // pivot rows the record can hold
  double* rec_rows;    // [rec_cap][W] pivot rows / PE (W = n + kmax + 1: positions, RHS)
  int* rec_e;          // [rec_cap] entering (global) position of each recorded pivot
  double* rec_T;       // [m][W] constraint rows after phase I (positions, then RHS)
  int* rec_nbvar;      // [n + kmax] position -> nonbasic variable (DEAD: left artificial)
  int* rec_bkey;       // [m] row -> basic-variable key
  int* rec_info;       // {status after phase I (-1: phase II follows), it1, pivots, k}
  // S class (thread per LP): the register kernel (type-1 LPs) appends the LPs it cannot hold
  // (b has a negative entry) to defer_list; the SMEM-slice kernel then solves exactly those
  // (list mode when defer_cnt != nullptr).
  int* defer_list;     // [batch] launch-relative LP indices
  int* defer_cnt;      // number of entries, zeroed before the register kernel
  // L class, hybrid TMR layout (2-CTA clusters at 2 CTAs per SM): constraint rows 0..127 in
  // TMEM during the pivot loop, their storage of record in tm_scr (per CTA: 128 x S doubles,
  // CTA b at tm_scr + b * 128 * S) instead of SMEM
  int tm_hyb;
  double* tm_scr;
};

struct HyperboxArgs {
  int64_t batch;
  int n;
  const double* l;    // batch x n directions (the objective c)
  const double* box;  // [hi(n); -lo(n)] shared, or batch x 2n
  int shared_box;
  int32_t* status;
  double* obj;
  double* x;          // may be null
};

// ---- M / L classes: one LP per CTA (cl = 1) or per cl-CTA cluster, tableau in SMEM ----
size_t block_smem_bytes(int cl, int m, int n, int kmax);
bool block_fits(int cl, int m, int n, int kmax);
size_t block_hyb_scratch_doubles(int m, int n, int kmax);  // 0: no hybrid TMR layout
cudaError_t launch_simplex_block(int cl, const SimplexArgs& a, int grid_override,
                                 cudaStream_t s, int* ctas_out);

// ---- S class: one LP per thread (tiny LPs), tableau in a thread-private SMEM slice ----
bool thread_fits(int m, int n);
cudaError_t launch_simplex_thread(const SimplexArgs& a, cudaStream_t s);
// register variant for m, n <= 6: type-1 LPs in registers, the rest deferred to the SMEM-slice
// kernel (a.defer_list / a.defer_cnt must be set; two launches, the count memset first)
bool tiny_fits(int m, int n);
cudaError_t launch_simplex_tiny(const SimplexArgs& a, cudaStream_t s);

// ---- R class: one LP per CTA (one warp for small LPs), tableau resident in registers ----
bool reg_fits(int m, int n, int kmax);
int reg_layout(int m, int n, int kmax);  // the layout id the R class would use (-1: none)
cudaError_t launch_simplex_reg(const SimplexArgs& a, int grid_override, cudaStream_t s,
                               int* ctas_out);

// ---- W class: one LP per warp (m <= 32, n + kmax <= 32), tableau in registers, shuffles ----
bool warp_fits(int m, int n, int kmax);
int warp_layout(int m, int n, int kmax);  // the layout id the W class would use (-1: none)
cudaError_t launch_simplex_warp(const SimplexArgs& a, int grid_override, cudaStream_t s,
                                int* ctas_out);

// ---- prepass: kmax = max over LPs of #{i : b_i < 0} ----
cudaError_t launch_count_art(const double* b, int64_t batch, int m, int* kmax_dev,
                             cudaStream_t s);

// ---- H class: hyperbox closed form (Eq. 6) ----
cudaError_t launch_hyperbox(const HyperboxArgs& a, cudaStream_t s);

int device_sm_count();

// Development-build switches (A/B experiments, tests of alternative paths): read from the
// environment only when compiled with -DLPB_DEV_HOOKS (build.py --dev); the product library
// never reads the environment.
#ifdef LPB_DEV_HOOKS
inline bool dev_flag(const char* name) { return std::getenv(name) != nullptr; }
#else
inline constexpr bool dev_flag(const char*) { return false; }
#endif

// Thread-safe memo of a launch-configuration query per (device, key): function attributes
// and occupancy are host round trips worth doing once.  compute(v, attr) runs under the lock
// and must set cudaFuncAttributeMaxDynamicSharedMemorySize to `attr`, which is the largest
// key (dynamic SMEM size) this memo has seen on the device: the attribute is only ever RAISED,
// so a launch that another host thread configured for a larger size is never invalidated by
// a concurrent smaller one (the launch itself happens after the lock is released).  The
// occupancy result is computed for the key's own size.  Up to kSlots keys per device are
// kept (round-robin replacement).
class LaunchMemo {
 public:
  template <class F>
  cudaError_t get(size_t key, int* out, F&& compute) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> g(mu_);
    if (dev < 0 || dev >= kDevs) {  // beyond the table: no memo (the attribute still only grows)
      size_t& mx = spill_attr_;
      if (key > mx) mx = key;
      int v = 0;
      e = compute(v, mx);
      *out = v;
      return e;
    }
    Dev& d = dev_[dev];
    for (const Entry& en : d.ent)
      if (en.valid && en.key == key) {
        *out = en.val;
        return cudaSuccess;
      }
    const size_t attr = key > d.attr_max ? key : d.attr_max;
    int v = 0;
    e = compute(v, attr);
    if (e != cudaSuccess) return e;
    d.attr_max = attr;
    Entry& en = d.ent[d.next];
    d.next = (d.next + 1) % kSlots;
    en.valid = true;
    en.key = key;
    en.val = v;
    *out = v;
    return cudaSuccess;
  }

 private:
  struct Entry {
    bool valid = false;
    size_t key = 0;
    int val = 0;
  };
  static constexpr int kDevs = 64, kSlots = 8;
  struct Dev {
    Entry ent[kSlots];
    int next = 0;
    size_t attr_max = 0;
  };
  std::mutex mu_;
  size_t spill_attr_ = 0;
  Dev dev_[kDevs];
};

}  // namespace lpb
