/* Sanitizer driver for the oracle's pthread pool (tests/test_sanitizers_cpu.py; SURVEY.md
 * §4 "race detection"): solves seeded random batches (type 1, type 2 and unbounded /
 * infeasible mixes, plus hyperbox batches) on 1 and 8 threads and checks that the results
 * are identical, under -fsanitize=address,undefined or -fsanitize=thread.  Links
 * oracle/lpb_oracle.c directly.  Exit code 0 = identical results (the sanitizers report on
 * stderr and abort on their own). */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  double eps_enter, eps_piv, eps_phase1;
  int max_iter, bland_after, pivot_rule;
  uint64_t rpc_seed;
  int64_t lp_base;
} oracle_opts;
int oracle_solve_batch(int64_t batch, int m, int n, const double* A, const double* b,
                       const double* c, const oracle_opts* o, int nthreads, int* status,
                       double* obj, double* x, int* iters, double* y, double* ray, double* xb);
int oracle_hyperbox_batch(int64_t batch, int n, const double* lo, const double* hi,
                          int64_t box_stride, const double* l, int nthreads, int* status,
                          double* obj, double* x);

static uint64_t st = 0x9E3779B97F4A7C15ull;
static double unif(double lo, double hi) {
  st ^= st << 13; st ^= st >> 7; st ^= st << 17;
  return lo + (hi - lo) * (double)(st >> 11) * (1.0 / 9007199254740992.0);
}

static int run_general(int B, int m, int n, int neg, int rule) {
  double* A = malloc(sizeof(double) * B * m * n);
  double* b = malloc(sizeof(double) * B * m);
  double* c = malloc(sizeof(double) * B * n);
  for (int64_t i = 0; i < (int64_t)B * m * n; ++i) A[i] = unif(-10, 10);
  for (int64_t i = 0; i < (int64_t)B * m; ++i) b[i] = unif(1, 100) * (neg && unif(0, 1) < 0.25 ? -1 : 1);
  for (int64_t i = 0; i < (int64_t)B * n; ++i) c[i] = unif(-10, 10);
  oracle_opts o = {1e-9, 1e-9, 1e-9, 0, 0, rule, 7, 0};
  int *s1 = malloc(sizeof(int) * B), *s8 = malloc(sizeof(int) * B);
  int *i1 = malloc(sizeof(int) * 2 * B), *i8 = malloc(sizeof(int) * 2 * B);
  double *o1 = malloc(sizeof(double) * B), *o8 = malloc(sizeof(double) * B);
  double *x1 = malloc(sizeof(double) * B * n), *x8 = malloc(sizeof(double) * B * n);
  double *y8 = malloc(sizeof(double) * B * m), *r8 = malloc(sizeof(double) * B * n);
  double *xb8 = malloc(sizeof(double) * B * n);
  oracle_solve_batch(B, m, n, A, b, c, &o, 1, s1, o1, x1, i1, NULL, NULL, NULL);
  oracle_solve_batch(B, m, n, A, b, c, &o, 8, s8, o8, x8, i8, y8, r8, xb8);
  int bad = memcmp(s1, s8, sizeof(int) * B) || memcmp(i1, i8, sizeof(int) * 2 * B) ||
            memcmp(o1, o8, sizeof(double) * B) || memcmp(x1, x8, sizeof(double) * B * n);
  int hist[5] = {0};
  for (int k = 0; k < B; ++k) hist[s1[k] >= 0 && s1[k] < 5 ? s1[k] : 4]++;
  printf("general B=%d %dx%d neg=%d rule=%d: statuses %d %d %d %d %d %s\n", B, m, n, neg, rule,
         hist[0], hist[1], hist[2], hist[3], hist[4], bad ? "MISMATCH" : "identical");
  free(A); free(b); free(c); free(s1); free(s8); free(i1); free(i8); free(o1); free(o8);
  free(x1); free(x8); free(y8); free(r8); free(xb8);
  return bad;
}

static int run_hyperbox(int B, int n) {
  double *lo = malloc(sizeof(double) * n), *hi = malloc(sizeof(double) * n);
  double* l = malloc(sizeof(double) * B * n);
  for (int i = 0; i < n; ++i) { lo[i] = unif(-1, 0); hi[i] = lo[i] + unif(0.01, 1); }
  for (int64_t i = 0; i < (int64_t)B * n; ++i) l[i] = unif(-1, 1);
  int *s1 = malloc(sizeof(int) * B), *s8 = malloc(sizeof(int) * B);
  double *o1 = malloc(sizeof(double) * B), *o8 = malloc(sizeof(double) * B);
  double *x1 = malloc(sizeof(double) * B * n), *x8 = malloc(sizeof(double) * B * n);
  oracle_hyperbox_batch(B, n, lo, hi, 0, l, 1, s1, o1, x1);
  oracle_hyperbox_batch(B, n, lo, hi, 0, l, 8, s8, o8, x8);
  int bad = memcmp(s1, s8, sizeof(int) * B) || memcmp(o1, o8, sizeof(double) * B) ||
            memcmp(x1, x8, sizeof(double) * B * n);
  printf("hyperbox B=%d n=%d: %s\n", B, n, bad ? "MISMATCH" : "identical");
  free(lo); free(hi); free(l); free(s1); free(s8); free(o1); free(o8); free(x1); free(x8);
  return bad;
}

int main(void) {
  int bad = 0;
  bad |= run_general(3000, 5, 5, 0, 0);
  bad |= run_general(3000, 6, 6, 1, 0);
  bad |= run_general(400, 20, 20, 1, 1);
  bad |= run_general(40, 60, 60, 1, 0);
  bad |= run_hyperbox(100003, 28);
  return bad;
}
