/*
 * lpb.h — C ABI of the B200-native batched LP solver (paper_1609_08114_b200/liblpb.so).
 *
 * Solves a batch of independent linear programs in standard form
 *     maximize c.x  subject to  A x <= b,  x >= 0                (Eq. 1-3)
 * with the dense-tableau simplex method (Dantzig's "Largest Positive Coefficient" entering
 * rule, or the "Random Positive Coefficient" rule, see
 * lpb_options.pivot_rule; ratio test PAPER.md:97,126; pivot PAPER.md:163-172), the two-phase
 * method when the slack basis is infeasible, and the closed-form hyperbox LP
 * (Eq. 6).  One LP per CUDA thread block (or thread-block cluster, or
 * warp, or thread), as in PAPER.md:114 ("We assign a CUDA block of threads to solve an LP").
 *
 * Conventions
 *   - Every call returns int: LPB_OK (0) or a negative error code.  No C++ exception crosses
 *     the ABI.  Per-LP outcomes (optimal / unbounded / infeasible / ...) are DATA returned in
 *     the status array, never call errors (a pathological LP does not fail the batch).
 *   - All floating point is IEEE fp64.  Inputs must be finite (caller contract; no NaN scan).
 *   - One context is used by one host thread at a time.  Contexts are independent (e.g. one
 *     per GPU / torch.distributed rank).
 *
 * Layouts (LP-contiguous, index-aligned: output k belongs to input LP k)
 *   A    : batch x m x n, row-major        A[(k*m + i)*n + j]
 *   b    : batch x m                       b[k*m + i]
 *   c    : batch x n                       c[k*n + j]
 *   status: int32[batch]   obj: f64[batch]   x: f64[batch*n]   iters: int32[batch*2]
 *          (iters[2k] = phase-I pivots incl. artificial drive-outs, iters[2k+1] = phase-II)
 *   Non-optimal LPs report obj = +inf (UNBOUNDED), -inf (INFEASIBLE), NaN (ITER_LIMIT,
 *   NUMERICAL) and x = NaN.
 *
 * Hyperbox kind (LPB_HYPERBOX): the feasible region is the box [lo_1,hi_1] x ... x [lo_n,hi_n]
 *   encoded literally as A x <= b with A = [I; -I] (implicit: pass A = NULL), m = 2n and
 *   b = [hi_1..hi_n, -lo_1..-lo_n]; c holds the direction l.  With LPB_SHARED_BOX one box is
 *   shared by the whole batch (b has 2n entries; the paper's experiment).  NOTE:
 *   x >= 0 is NOT implied for this kind; the box is the whole feasible region.
 *   Result: obj = sum_i l_i h_i, h_i = lo_i if l_i < 0 else hi_i, x = h, status OPTIMAL, or
 *   INFEASIBLE when some lo_i > hi_i.
 *
 * Ownership
 *   The caller owns every array.  Without LPB_ASYNC, lpb_solve_batch has consumed its
 *   inputs when it returns (the library keeps no caller pointer).  With LPB_ASYNC the work is
 *   only enqueued on the context's stream: the caller keeps inputs alive until lpb_results /
 *   lpb_sync returns.  Results live in context-owned device memory until the next solve.
 */
#ifndef LPB_H_
#define LPB_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct lpb_ctx lpb_ctx; /* opaque, owned by the library */

enum { LPB_GENERAL = 0, LPB_HYPERBOX = 1 }; /* problem kind */

enum { /* per-LP status (data, not an error) */
  LPB_OPTIMAL = 0,    /* no entering variable: reduced costs all <= eps_enter  */
  LPB_UNBOUNDED = 1,  /* no leaving variable in phase II                       */
  LPB_INFEASIBLE = 2, /* phase-I optimum w* > eps_phase1*max(1,|b|_inf)         */
  LPB_ITER_LIMIT = 3, /* phase-I + phase-II pivots reached max_iter                           */
  LPB_NUMERICAL = 4,  /* phase I reported unbounded (impossible in exact arithmetic)          */
  LPB_BAD_HINT = 5    /* not solved: the LP has more b_i < 0 than lpb_options.kmax_hint
                         promised (obj = NaN, x = NaN, iters = 0)                            */
};

enum { /* call errors */
  LPB_OK = 0,
  LPB_EINVAL = -1,  /* batch <= 0, m or n <= 0, NULL required pointer, bad kind / options     */
  LPB_ENOMEM = -2,  /* device or pinned-host allocation failed                                */
  LPB_ECUDA = -3,   /* a CUDA runtime error (text via lpb_strerror / lpb_last_error)          */
  LPB_ESTATE = -4,  /* results requested before any solve                                     */
  LPB_ETOOBIG = -5  /* no compiled size class fits (m, n)                                     */
};

enum { /* lpb_solve_batch flags */
  LPB_DEVICE_PTRS = 1u, /* A, b, c are device pointers (e.g. torch CUDA tensors)              */
  LPB_SHARED_BOX = 2u,  /* hyperbox: one box (2n entries of b) for the whole batch             */
  LPB_NO_X = 4u,        /* do not produce x (saves 8n bytes per LP of HBM / D2H traffic)       */
  LPB_ASYNC = 8u,       /* enqueue only; do not synchronize before returning                   */
  LPB_SHARED_AB = 16u,  /* general LPs: one constraint system (A: m x n, b: m) for the whole
                           batch, only c varies per LP -- many objectives over one polytope,
                           the support-function sampling of PAPER.md:313,330 (SURVEY §8(f)
                           NEXT-1); A and b are read with stride 0                            */
  LPB_NO_TIMING = 32u   /* device-pointer solves: record no timing events (lpb_last_timing /
                           lpb_last_kernel_timing then return LPB_ESTATE).  For back-to-back
                           solves timed by the caller: each event record is GPU work        */
};

typedef struct {
  int32_t struct_size; /* = sizeof(lpb_options); ABI versioning                               */
  double eps_enter;    /* 1e-9: Step 1 candidates have reduced cost d_j > eps_enter          */
  double eps_piv;      /* 1e-9: Step 2 candidates have pivot-column entry a_ie > eps_piv     */
  double eps_phase1;   /* 1e-9: infeasible iff w* > eps_phase1 * max(1, |b|_inf)             */
  int32_t max_iter;    /* 0 -> 50*(n+m) pivots (phase I + phase II), then LPB_ITER_LIMIT     */
  int32_t bland_after; /* 0 -> n+m consecutive degenerate pivots switch to Bland's rule;
                          < 0 -> never (pure Dantzig)                                         */
  int32_t device;      /* CUDA device ordinal; -1 -> the current device                       */
  void* stream;        /* cudaStream_t to run on (cudaStreamLegacy = 0x1 for the legacy default
                          stream); NULL -> a non-blocking stream owned by the context          */
  int32_t n_chunks;    /* host-pointer pipeline depth; 0 -> 10 if batch > 100 and the inputs
                          are >= 1 MiB, else 1 (the paper's stream count; tiny
                          inputs cannot pay for per-chunk copy latency)                       */
  int32_t kernel_class;/* 0 auto; 1 S (thread/LP, m,n <= 8), 2 M (block/LP, SMEM tableau),
                          3 L (2/4-CTA cluster/LP, DSMEM), 4 R (block or warp/LP, register-
                          resident tableau tiles), 7 W (warp/LP, m <= 32 and n + k <= 32,
                          tableau in registers, shuffle exchanges); for tests / benches.
                          Hyperbox contexts accept 0 or 5 (H).  Any other value (or a class
                          of the other kind) is LPB_EINVAL at lpb_create                    */
  int32_t grid_ctas;   /* 0 auto; persistent grid size override (scheduling-invariance tests) */
  int32_t cluster_ctas;/* L class cluster size: 0 auto (the smallest of 2/4/8/16 CTAs whose
                          distributed SMEM holds the tableau); 2/4/8/16 forces that size when
                          the tableau fits it (tests / benches); 16 is a non-portable size    */
  int32_t pivot_rule;  /* Step 1 entering rule: LPB_RULE_LPC (0, default)
                          = Largest Positive Coefficient (Dantzig); LPB_RULE_RPC (1) = Random
                          Positive Coefficient.  Bland's rule still takes over after
                          bland_after degenerate pivots under either rule.                   */
  uint64_t rpc_seed;   /* RPC: seed of the counter-based choice (see LPB_RULE_RPC)            */
  int64_t lp_index_base;/* index, in the caller's numbering, of this context's LP 0 (RPC keys
                          k = lp_index_base + position in the call): a rank solving LPs
                          [lo, hi) of a sharded batch passes lo and follows exactly the pivot
                          path of an unsharded run; default 0                                */
  int32_t warm_start;  /* LPB_SHARED_AB batches with an infeasible slack basis (b has negative
                          entries): phase I depends on A and b only, so by default (0) it is
                          solved ONCE and every LP starts phase II from the recorded tableau,
                          its carried objective row rebuilt by replaying the recorded pivots
                          (bit-identical to solving each LP from scratch; M/L classes, LPC).
                          -1: solve every LP from scratch                                     */
  int32_t kmax_hint;   /* -1 (default): unknown.  >= 0: the caller promises that no LP of a
                          solve has more than kmax_hint rows with b_i < 0 -- the paper's LP
                          "type" (type 1 = feasible slack basis, b >= 0, is
                          kmax_hint 0; type 2 = infeasible basis, two-phase).  The size class
                          and register layout depend on k (the condensed width is n + k + 1),
                          so without a hint a device-pointer solve whose layout depends on k
                          first runs a tiny prepass kernel and reads its 4-byte result back
                          (the only host synchronisation inside an LPB_ASYNC solve); with a
                          hint the solve is ONE kernel launch and never blocks.  An LP that
                          breaks the promise is not solved: status LPB_BAD_HINT.  Host-pointer
                          solves scan the host b instead (inside the e2e time) when no hint
                          is given.  Must be in [-1, m]; else LPB_EINVAL at lpb_create.       */
} lpb_options;

/* Entering rules (lpb_options.pivot_rule).
 * LPB_RULE_RPC picks uniformly among the Step-1 candidates (reduced cost > eps_enter, never a
 * left artificial) without a stored random state: with mix64 the SplitMix64 finaliser
 * (z += 0x9E3779B97F4A7C15; z = (z^(z>>30))*0xBF58476D1CE4E5B9; z = (z^(z>>27))*
 * 0x94D049BB133111EB; z ^= z>>31), candidate variable j (0..n-1 structural, n+i slack of row
 * i) of LP k (lp_index_base + its 0-based index in the lpb_solve_batch call) at pivot t (= phase-I + phase-II
 * pivots done so far) scores  u = mix64(mix64(mix64(rpc_seed ^ mix64(k)) ^ t) ^ j) >> 11
 * (an integer < 2^53), and the candidate with the largest u enters (ties: lowest j).  Every
 * candidate is equally likely to win, the choice depends only on (seed, k, t, j) -- not on
 * the storage order of a size class -- and identical seeds give identical pivot sequences.
 * An undefined rule value is LPB_EINVAL at lpb_create. */
enum { LPB_RULE_LPC = 0, LPB_RULE_RPC = 1 };

/* Fill *o with the defaults above.  Returns LPB_EINVAL if o is NULL. */
int lpb_default_options(lpb_options* o);

/* Create a context for batches of up to `batch` LPs of size m x n of the given kind.
 * o may be NULL (defaults).  Allocates device result buffers for `batch` LPs.
 * Errors: LPB_EINVAL (batch <= 0, m/n <= 0, kind invalid, hyperbox with m != 2n, a general
 *         batch above 2^30 LPs -- split it over several calls / contexts),
 *         LPB_ETOOBIG (no size class holds m x n), LPB_ENOMEM, LPB_ECUDA. */
int lpb_create(lpb_ctx** out, int64_t batch, int32_t m, int32_t n, int32_t kind,
               const lpb_options* o);

/* Solve the context's batch (size given at create).  A must be NULL for LPB_HYPERBOX.
 * Host pointers (default): inputs are copied host->device straight from the caller's arrays
 * in n_chunks chunks on separate streams, each chunk's kernel overlapping the next chunk's
 * copy.  Pinned (page-locked) caller arrays give asynchronous, overlapped
 * copies; pageable ones are staged by the driver and overlap less.  The device input buffers
 * are allocated by the first host-pointer solve and kept by the context (one A and b -- one
 * box -- for LPB_SHARED_AB / LPB_SHARED_BOX; grown if a later call needs per-LP arrays).
 * With LPB_DEVICE_PTRS the kernels read the caller's device arrays.
 * Errors: LPB_EINVAL (NULL required pointer), LPB_ECUDA, LPB_ENOMEM. */
int lpb_solve_batch(lpb_ctx* c, const double* A, const double* b, const double* cvec,
                    uint32_t flags);

/* lpb_solve_batch + results in one call: the result arrays (host or device pointers; any may
 * be NULL) are filled per chunk, so on the host-pointer path chunk c's D2H overlaps chunk
 * c+1's kernel (the paper's "D2H-res").  This is the end-to-end entry point.
 * Errors: as lpb_solve_batch. */
int lpb_solve_batch_into(lpb_ctx* c, const double* A, const double* b, const double* cvec,
                         uint32_t flags, int32_t* status, double* obj, double* x,
                         int32_t* iters);

/* Copy results out (host or device pointers; cudaMemcpyDefault).  Any pointer may be NULL
 * to skip that output.  Synchronizes the context's stream.  x is not available when the
 * last solve used LPB_NO_X (x must then be NULL).  Errors: LPB_ESTATE, LPB_EINVAL,
 * LPB_ECUDA. */
int lpb_results(lpb_ctx* c, int32_t* status, double* obj, double* x, int32_t* iters);

/* Zero-copy access: device pointers of the context-owned result arrays (valid until the
 * next solve or destroy).  Any out-pointer may be NULL.  Does not synchronize. */
int lpb_result_device_ptrs(lpb_ctx* c, int32_t** status, double** obj, double** x,
                           int32_t** iters);

/* Wait for all work enqueued by this context.  Errors: LPB_ECUDA. */
int lpb_sync(lpb_ctx* c);

/* Device-event timing of the last solve (synchronizes): solve_ms brackets the kernel
 * launches only (inputs resident on the device); e2e_ms brackets first H2D copy -> last D2H
 * copy for host-pointer solves (equal to solve_ms for device-pointer solves). */
int lpb_last_timing(lpb_ctx* c, double* solve_ms, double* e2e_ms);

/* Device-event duration of the last device-pointer solve's dominant kernel alone (the
 * simplex or hyperbox kernel, without the size prepass).  Errors: LPB_ESTATE when the last
 * solve was not a device-pointer solve. */
int lpb_last_kernel_timing(lpb_ctx* c, double* kernel_ms);

/* Number of kernel launches the last solve issued (for the bench's gpu_launches count),
 * and the size class it dispatched to (1 S, 2 M, 3 L, 4 R, 5 H, 6 T, 7 W). */
int lpb_last_launch_info(lpb_ctx* c, int32_t* launches, int32_t* kernel_class);

/* Launch shape of the last solve's dominant kernel: CTAs per LP (the L class's cluster size
 * 2/4/8/16; 1 for one LP per CTA; 0 for the per-thread S and H classes) and the grid size
 * in CTAs (of the last chunk's launch).  Either pointer may be NULL.  Errors: LPB_EINVAL. */
int lpb_last_launch_shape(lpb_ctx* c, int32_t* cluster_ctas, int32_t* grid_ctas);

/* Release every resource of the context.  NULL is accepted. */
int lpb_destroy(lpb_ctx* c);

/* Static text for an error code. */
const char* lpb_strerror(int err);

/* Text of the last CUDA error seen by this context ("" if none). */
const char* lpb_last_error(lpb_ctx* c);

#ifdef __cplusplus
}
#endif
#endif /* LPB_H_ */
