/*
 * lpb_oracle.c — CPU fp64 reference ("oracle") for the batched LP hot path of
 * Gurung & Ray, "Solving Batched Linear Programs on GPU and Multicore CPU"
 * (arXiv 1609.08114; "D1").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code, header,
 * table or helper with the CUDA path (paper_1609_08114_b200/, include/); the two only
 * consume the same seeded arrays from lpgen/.
 *
 * What it computes, written the plain way (no blocking, no fusion, no reordering):
 *   - a FULL-tableau textbook simplex (§3, lines 71-103; Listing 1)
 *     with every slack and artificial column stored explicitly;
 *   - the two-phase method for an infeasible slack basis;
 *   - the hyperbox closed form, Eq. (6).
 * Where the paper is silent the readings of SURVEY.md §8(c) are taken; each is listed in
 * DESIGN.md §"Readings" (R1..R12 below refer to that list).
 *
 * Arithmetic contract: compiled with -O2 -ffp-contract=off (no implicit FMA), explicit
 * fma() for the pivot update, IEEE division for the ratio test and the pivot row.
 *
 * Parity status: pinned (tests/test_oracle_*.py): SPEC worked examples, Klee-Minty closed
 * form, Chvatal's cycling LP, drive-out fixtures, fractional knapsack / diagonal closed
 * forms, LP certificates (dual / Farkas / ray) from the original data, exact-rational brute
 * force on m,n <= 4, scipy HiGHS (presolve off); hyperbox against exact 2^n-vertex brute
 * force.  Nothing here is "parity unpinned".
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { OR_OPTIMAL = 0, OR_UNBOUNDED = 1, OR_INFEASIBLE = 2, OR_ITER_LIMIT = 3, OR_NUMERICAL = 4 };

typedef struct {
  double eps_enter;   /* Step 1 threshold (R4): d_j > eps_enter is an improving column   */
  double eps_piv;     /* Step 2 threshold (R1): a_ie > eps_piv is a ratio candidate       */
  double eps_phase1;  /* phase-I zero test (R8): w* > eps_phase1*max(1,|b|_inf) infeasible */
  int max_iter;       /* <= 0 -> 50(n+m)                                     */
  int bland_after;    /* 0 -> n+m ; < 0 -> never (pure Dantzig) (R6)                       */
  int pivot_rule;     /* 0 LPC, 1 RPC (reading R15)             */
  uint64_t rpc_seed;  /* RPC: seed of the counter-based choice (R15)                          */
  int64_t lp_base;    /* RPC: the batch's LP k is LP lp_base + k of the caller's numbering     */
} oracle_opts;

/* One LP's full tableau.  Rows 0..m-1 constraints, row m the phase-II (original objective)
 * row, row m+1 the phase-I row.  Columns: x_0..x_{n-1} | s_0..s_{m-1} | art_0..art_{k-1} |
 * RHS  ("p = m+1 ... q = n + slack + artificial + 2"; the two auxiliary
 * columns are the basis index (kept in basis[]) and b (the RHS column)). */
typedef struct {
  int m, n, k, ncol, rhs;
  double* T;    /* (m+2) x ncol, row-major */
  int* basis;   /* row -> column index of its basic variable */
} tableau;

#define TT(t, i, j) ((t)->T[(size_t)(i) * (size_t)(t)->ncol + (size_t)(j)])

/* Bland tie-break key of a basic variable (R5): artificials rank below every real
 * variable, ordered by their row; real variables by their index. */
static int var_key(const tableau* t, int col) {
  if (col < t->n + t->m) return col;
  return (col - (t->n + t->m)) - t->k; /* in [-k, -1], ascending with the artificial's row */
}

/* Build (Eq. 4 slack form; two-phase auxiliary LP, R7):
 * row i = [a_i1..a_in | e_i | b_i]; if b_i < 0 the whole row is multiplied by -1 and an
 * artificial with coefficient +1 becomes its basic variable. */
static int build(tableau* t, int m, int n, const double* A, const double* b, const double* c) {
  int k = 0;
  for (int i = 0; i < m; ++i) k += (b[i] < 0.0);
  t->m = m; t->n = n; t->k = k;
  t->ncol = n + m + k + 1;
  t->rhs = n + m + k;
  t->T = (double*)calloc((size_t)(m + 2) * (size_t)t->ncol, sizeof(double));
  t->basis = (int*)malloc(sizeof(int) * (size_t)m);
  if (!t->T || !t->basis) return -1;
  int a = 0;
  for (int i = 0; i < m; ++i) {
    for (int j = 0; j < n; ++j) TT(t, i, j) = A[(size_t)i * n + j];
    for (int r = 0; r < m; ++r) TT(t, i, n + r) = (r == i) ? 1.0 : 0.0;
    TT(t, i, t->rhs) = b[i];
    if (b[i] < 0.0) {
      for (int j = 0; j < n + m; ++j) TT(t, i, j) = -1.0 * TT(t, i, j);
      TT(t, i, t->rhs) = -1.0 * TT(t, i, t->rhs);
      TT(t, i, n + m + a) = 1.0;
      t->basis[i] = n + m + a;
      ++a;
    } else {
      t->basis[i] = n + i;
    }
  }
  /* Phase-II row: reduced costs c_j - z_j = c_j at the slack basis; RHS = -objective = 0
   * ("the last row stores ... the coefficients of the non-basic variables in the objective
   * function"; sign convention R3). */
  for (int j = 0; j < n; ++j) TT(t, m, j) = c[j];
  /* Phase-I row (R7): maximise -sum(art); its reduced costs are the column sums of the
   * negated rows over the non-artificial columns and the RHS, summed in ascending row
   * order starting from 0.0. */
  if (k > 0) {
    for (int j = 0; j < t->ncol; ++j) {
      if (j >= n + m && j < t->rhs) continue; /* artificial columns: 0 */
      double acc = 0.0;
      for (int i = 0; i < m; ++i)
        if (b[i] < 0.0) acc = acc + TT(t, i, j);
      TT(t, m + 1, j) = acc;
    }
  }
  return 0;
}

/* Step 3 (Listing 1): NewPivotRow = OldPivotRow / PE; then for every
 * other active row NewRow_ij = OldRow_ij - PivotCol_i * NewPivotRow_j, written as one
 * fma(-f, r, T) per element (R12).  Rows 0..nrow-1 are updated (both objective rows while
 * the phase-I row is live). */
static void pivot(tableau* t, int l, int e, int nrow) {
  const double pe = TT(t, l, e);
  for (int j = 0; j < t->ncol; ++j) TT(t, l, j) = TT(t, l, j) / pe;
  TT(t, l, e) = 1.0;
  for (int i = 0; i < nrow; ++i) {
    if (i == l) continue;
    const double f = TT(t, i, e);
    for (int j = 0; j < t->ncol; ++j) TT(t, i, j) = fma(-f, TT(t, l, j), TT(t, i, j));
    TT(t, i, e) = 0.0;
  }
  t->basis[l] = e;
}

/* Step 1 ("Largest Positive Coefficient"): the non-artificial column with
 * the largest reduced cost > eps_enter, ties to the lowest column (= variable) index (R5);
 * in Bland mode the lowest-index such column (R6).  Artificial columns never enter (R7). */
static int entering(const tableau* t, int row, double eps, int bland) {
  int e = -1;
  double best = 0.0;
  for (int j = 0; j < t->n + t->m; ++j) {
    const double d = TT(t, row, j);
    if (!(d > eps)) continue;
    if (bland) return j;
    if (e < 0 || d > best) { e = j; best = d; }
  }
  return e;
}

/* SplitMix64 finaliser (R15): z += golden gamma; two xor-shift-multiply rounds; xor-shift. */
static uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

/* Step 1 under RPC ("we choose a random index having a positive coefficient
 * from the last row"; reading R15): every column j with reduced cost > eps_enter (artificials
 * excluded, R7) draws the score u_j = mix64(mix64(mix64(seed ^ mix64(k)) ^ t) ^ j) >> 11 --
 * k = the LP's index in the batch, t = pivots done so far -- and the largest score enters
 * (ties to the lowest j).  Each candidate is equally likely to win. */
static int entering_rpc(const tableau* t, int row, double eps, uint64_t seed, int64_t k,
                        int pivots) {
  const uint64_t base = mix64(mix64(seed ^ mix64((uint64_t)k)) ^ (uint64_t)pivots);
  int e = -1;
  uint64_t best = 0;
  for (int j = 0; j < t->n + t->m; ++j) {
    const double d = TT(t, row, j);
    if (!(d > eps)) continue;
    const uint64_t u = mix64(base ^ (uint64_t)j) >> 11;
    if (e < 0 || u > best) { e = j; best = u; }
  }
  return e;
}

/* Step 2 ("minimum positive ratio ... a large positive number in place of
 * ratios that are negative or undefined"; readings R1, R2): rows with a_ie > eps_piv give
 * r_i = b_i / a_ie (IEEE division); other rows are excluded (the +inf sentinel); argmin r,
 * ties to the lowest row (Dantzig mode) or the lowest basic-variable key (Bland mode). */
static int leaving(const tableau* t, int e, double eps, int bland, double* theta) {
  int l = -1;
  double best = 0.0;
  for (int i = 0; i < t->m; ++i) {
    const double a = TT(t, i, e);
    if (!(a > eps)) continue;
    const double r = TT(t, i, t->rhs) / a;
    if (l < 0 || r < best ||
        (r == best && bland && var_key(t, t->basis[i]) < var_key(t, t->basis[l]))) {
      l = i;
      best = r;
    }
  }
  *theta = best;
  return l;
}

/* Certificates read off the final tableau (used by the tests):
 *   y_i = -T[row][slack_i]  (dual for OPTIMAL with row = phase-II; Farkas for INFEASIBLE with
 *   row = phase-I);  ray for UNBOUNDED: d_e = 1 (if e < n), d_basis[i] = -T[i][e];
 *   xb = the basic point (structural part) at termination. */
static void certs(const tableau* t, int status, int e_unb, double* y, double* ray, double* xb) {
  const int m = t->m, n = t->n;
  if (xb) { /* basic point at termination: feasible for OPTIMAL / UNBOUNDED (certifies the ray) */
    for (int j = 0; j < n; ++j) xb[j] = 0.0;
    for (int i = 0; i < m; ++i)
      if (t->basis[i] < n) xb[t->basis[i]] = TT(t, i, t->rhs);
  }
  if (y) {
    const int row = (status == OR_INFEASIBLE) ? m + 1 : m;
    for (int i = 0; i < m; ++i) y[i] = (status == OR_OPTIMAL || status == OR_INFEASIBLE)
                                           ? -TT(t, row, n + i) : NAN;
  }
  if (ray) {
    for (int j = 0; j < n; ++j) ray[j] = (status == OR_UNBOUNDED) ? 0.0 : NAN;
    if (status == OR_UNBOUNDED) {
      if (e_unb < n) ray[e_unb] = 1.0;
      for (int i = 0; i < m; ++i)
        if (t->basis[i] < n) ray[t->basis[i]] = -TT(t, i, e_unb);
    }
  }
}

/* Solve one LP: max c.x s.t. A x <= b, x >= 0 (Eq. 1-3).
 * Outputs: status; obj (= -T[m][RHS] when OPTIMAL, +inf UNBOUNDED, -inf INFEASIBLE, NaN
 * otherwise; R10); x[n] (basic values read from the RHS column, NaN when not OPTIMAL);
 * iters[2] = (phase-I pivots incl. drive-outs, phase-II pivots).  y[m], ray[n] optional. */
int oracle_solve_lp(int m, int n, const double* A, const double* b, const double* c,
                    const oracle_opts* o, int64_t lp_index, int* status, double* obj,
                    double* x, int* iters, double* y, double* ray, double* xb) {
  tableau tb;
  tableau* t = &tb;
  if (build(t, m, n, A, b, c) != 0) return -1;
  const int max_iter = o->max_iter > 0 ? o->max_iter : 50 * (n + m);
  const int K = o->bland_after == 0 ? n + m : o->bland_after; /* < 0: never */
  int it[2] = {0, 0};
  int phase = t->k > 0 ? 1 : 2;
  int stall = 0, st = OR_OPTIMAL, e_unb = -1;
  for (;;) {
    const int row = (phase == 1) ? m + 1 : m;
    const int nrow = (phase == 1) ? m + 2 : m + 1;
    const int bland = (K > 0 && stall >= K);
    const int e = (o->pivot_rule == 1 && !bland)
                      ? entering_rpc(t, row, o->eps_enter, o->rpc_seed, lp_index, it[0] + it[1])
                      : entering(t, row, o->eps_enter, bland);
    if (e < 0) {
      if (phase == 2) { st = OR_OPTIMAL; break; }
      /* Phase switch ("checked if the optimal solution ... is 0"; R8, R9). */
      double binf = 0.0;
      for (int i = 0; i < m; ++i) binf = fmax(binf, fabs(b[i]));
      const double w = TT(t, m + 1, t->rhs); /* = sum of the artificials' values */
      if (w > o->eps_phase1 * fmax(1.0, binf)) { st = OR_INFEASIBLE; break; }
      for (int l = 0; l < m; ++l) {
        if (t->basis[l] < n + m) continue;  /* not artificial */
        int ed = -1;
        double best = 0.0;
        for (int j = 0; j < n + m; ++j) {
          const double a = fabs(TT(t, l, j));
          if (a > o->eps_piv && (ed < 0 || a > best)) { ed = j; best = a; }
        }
        if (ed < 0) continue; /* redundant row: artificial stays basic at 0 */
        pivot(t, l, ed, m + 2);
        it[0]++;
      }
      phase = 2;
      stall = 0;
      continue;
    }
    if (it[0] + it[1] >= max_iter) { st = OR_ITER_LIMIT; break; }
    double theta = 0.0;
    const int l = leaving(t, e, o->eps_piv, bland, &theta);
    if (l < 0) {
      st = (phase == 2) ? OR_UNBOUNDED : OR_NUMERICAL;
      e_unb = e;
      break;
    }
    pivot(t, l, e, nrow);
    it[phase - 1]++;
    stall = (theta > 0.0) ? 0 : stall + 1;
  }
  *status = st;
  iters[0] = it[0];
  iters[1] = it[1];
  if (st == OR_OPTIMAL) {
    *obj = -TT(t, m, t->rhs);
    for (int j = 0; j < n; ++j) x[j] = 0.0;
    for (int i = 0; i < m; ++i)
      if (t->basis[i] < n) x[t->basis[i]] = TT(t, i, t->rhs);
  } else {
    *obj = (st == OR_UNBOUNDED) ? INFINITY : (st == OR_INFEASIBLE) ? -INFINITY : NAN;
    for (int j = 0; j < n; ++j) x[j] = NAN;
  }
  certs(t, st, e_unb, y, ray, xb);
  free(t->T);
  free(t->basis);
  return 0;
}

/* Hyperbox LP, Eq. (6): max l.x over [lo_1,hi_1] x ... x [lo_n,hi_n]
 * = sum_i l_i h_i with h_i = lo_i if l_i < 0 else hi_i (R11: l_i = 0 and -0.0 take hi).
 * The sum is the sequential chain acc = fma(l_i, h_i, acc), i = 0..n-1, from acc = 0.
 * INFEASIBLE when some lo_i > hi_i (empty box). */
void oracle_hyperbox(int n, const double* lo, const double* hi, const double* l, int* status,
                     double* obj, double* x) {
  int empty = 0;
  for (int i = 0; i < n; ++i) empty |= (lo[i] > hi[i]);
  if (empty) {
    *status = OR_INFEASIBLE;
    *obj = -INFINITY;
    if (x) for (int i = 0; i < n; ++i) x[i] = NAN;
    return;
  }
  double acc = 0.0;
  for (int i = 0; i < n; ++i) {
    const double h = (l[i] < 0.0) ? lo[i] : hi[i];
    acc = fma(l[i], h, acc);
    if (x) x[i] = h;
  }
  *status = OR_OPTIMAL;
  *obj = acc;
}

/* ---- batch drivers: one LP per task over a pthread pool (the paper's multicore-CPU
 * baseline role, PAPER.md:264 / Algorithm 1; each thread solves one LP at a time). ---- */

typedef struct {
  int64_t batch;
  int m, n;
  const double *A, *b, *c;
  const oracle_opts* o;
  int* status;
  double *obj, *x;
  int* iters;
  double *y, *ray, *xb;
  int64_t next;
} batch_job;

static void* batch_worker(void* arg) {
  batch_job* j = (batch_job*)arg;
  for (;;) {
    const int64_t k = __atomic_fetch_add(&j->next, 1, __ATOMIC_RELAXED);
    if (k >= j->batch) break;
    const size_t mn = (size_t)j->m * (size_t)j->n;
    oracle_solve_lp(j->m, j->n, j->A + (size_t)k * mn, j->b + (size_t)k * j->m,
                    j->c + (size_t)k * j->n, j->o, j->o->lp_base + k, j->status + k, j->obj + k,
                    j->x + (size_t)k * j->n, j->iters + 2 * k,
                    j->y ? j->y + (size_t)k * j->m : NULL,
                    j->ray ? j->ray + (size_t)k * j->n : NULL,
                    j->xb ? j->xb + (size_t)k * j->n : NULL);
  }
  return NULL;
}

int oracle_solve_batch(int64_t batch, int m, int n, const double* A, const double* b,
                       const double* c, const oracle_opts* o, int nthreads, int* status,
                       double* obj, double* x, int* iters, double* y, double* ray,
                       double* xb) {
  batch_job j = {batch, m, n, A, b, c, o, status, obj, x, iters, y, ray, xb, 0};
  if (nthreads <= 1) { batch_worker(&j); return 1; }
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nthreads);
  int started = 0;
  for (int i = 0; i < nthreads; ++i)
    if (pthread_create(&th[i], NULL, batch_worker, &j) == 0) ++started;
  if (started == 0) batch_worker(&j);
  for (int i = 0; i < started; ++i) pthread_join(th[i], NULL);
  free(th);
  return started > 0 ? started : 1;
}

typedef struct {
  int64_t batch;
  int n;
  const double *lo, *hi, *l;
  int64_t box_stride; /* 0: one shared box; n: one box per LP */
  int* status;
  double *obj, *x;
  int64_t next;
} hbox_job;

static void* hbox_worker(void* arg) {
  hbox_job* j = (hbox_job*)arg;
  const int64_t chunk = 4096;
  for (;;) {
    const int64_t k0 = __atomic_fetch_add(&j->next, chunk, __ATOMIC_RELAXED);
    if (k0 >= j->batch) break;
    const int64_t k1 = k0 + chunk < j->batch ? k0 + chunk : j->batch;
    for (int64_t k = k0; k < k1; ++k)
      oracle_hyperbox(j->n, j->lo + k * j->box_stride, j->hi + k * j->box_stride,
                      j->l + k * j->n, j->status + k, j->obj + k,
                      j->x ? j->x + k * j->n : NULL);
  }
  return NULL;
}

int oracle_hyperbox_batch(int64_t batch, int n, const double* lo, const double* hi,
                          int64_t box_stride, const double* l, int nthreads, int* status,
                          double* obj, double* x) {
  hbox_job j = {batch, n, lo, hi, l, box_stride, status, obj, x, 0};
  if (nthreads <= 1) { hbox_worker(&j); return 1; }
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nthreads);
  int started = 0;
  for (int i = 0; i < nthreads; ++i)
    if (pthread_create(&th[i], NULL, hbox_worker, &j) == 0) ++started;
  if (started == 0) hbox_worker(&j);
  for (int i = 0; i < started; ++i) pthread_join(th[i], NULL);
  free(th);
  return started > 0 ? started : 1;
}
