/* tests/csrc/oracle_sanitize.c -- test driver: the C oracle (oracle/nrmf_oracle.c)
 * built with -fsanitize=address,undefined and run over small, ragged, empty,
 * special-value and column inputs (tests/test_oracle_sanitize.py).  Any
 * out-of-bounds access, leak, signed overflow or other UB aborts the run; a
 * handful of closed forms (not the oracle's own arithmetic) are checked too. */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

double oracle_v1_hypot_d(double x, double y);
float oracle_v1_hypot_s(float x, float y);
double oracle_R_H_d(int64_t n, const double *x);
float oracle_R_H_s(int64_t n, const float *x);
double oracle_R_A_d(int64_t n, const double *x);
double oracle_cr_hypot_d(double x, double y);
double oracle_nrmf_tree_d(const double *x, int64_t n, int64_t lanes, int64_t J, int64_t p2_min, int top_cr, int *ok);
float oracle_nrmf_tree_s(const float *x, int64_t n, int64_t lanes, int64_t J, int64_t p2_min, int top_cr, int *ok);
int oracle_tiles_d(const double *x, int64_t n, int64_t lanes, int64_t J, int64_t tau0, int64_t count, double *out);
int oracle_nrmf_cols_d(int64_t r, int64_t c, int64_t ld, const double *A, int64_t lanes, int64_t J, int top_cr,
                       double *col_norms, double *frob);
int oracle_nrmf_cols_s(int64_t r, int64_t c, int64_t ld, const float *A, int64_t lanes, int64_t J, int top_cr,
                       float *col_norms, float *frob);
double exact_nrm_d(const double *x, int64_t n);
float exact_nrm_s(const float *x, int64_t n);

static int fails = 0;
#define CHECK(c) do { if (!(c)) { fprintf(stderr, "FAIL %s:%d %s\n", __FILE__, __LINE__, #c); ++fails; } } while (0)

static uint64_t st = 0x9E3779B97F4A7C15ull;
static double urand(void) { st ^= st << 13; st ^= st >> 7; st ^= st << 17; return (double)(st >> 11) * 0x1p-53; }

int main(void) {
  /* closed forms (Listing 2 on Pythagorean pairs and zeros) */
  CHECK(oracle_v1_hypot_d(3.0, 4.0) == 5.0);
  CHECK(oracle_v1_hypot_d(-5.0, 12.0) == 13.0);
  CHECK(oracle_v1_hypot_d(0.0, 0.0) == 0.0 && !signbit(oracle_v1_hypot_d(-0.0, 0.0)));
  CHECK(oracle_v1_hypot_s(6.0f, 8.0f) == 10.0f);
  CHECK(oracle_cr_hypot_d(3.0, 4.0) == 5.0);
  CHECK(isinf(oracle_v1_hypot_d(INFINITY, 1.0)));
  CHECK(oracle_v1_hypot_d(0x1p-1074, 0.0) == 0x1p-1074);
  /* trees: every length 0..300 (ragged tails, empty), both dtypes, both tops */
  for (int64_t n = 0; n <= 300; ++n) {
    double *x = (double *)malloc((size_t)(n ? n : 1) * sizeof(double));
    float *xs = (float *)malloc((size_t)(n ? n : 1) * sizeof(float));
    for (int64_t i = 0; i < n; ++i) { x[i] = 2.0 * urand() - 1.0; xs[i] = (float)x[i]; }
    int ok = 0;
    const double r = oracle_nrmf_tree_d(x, n, 4, 8, 1, 0, &ok);
    CHECK(ok);
    const double rc = oracle_nrmf_tree_d(x, n, 4, 8, 1, 1, &ok);
    CHECK(ok);
    (void)rc;
    const float rs = oracle_nrmf_tree_s(xs, n, 8, 4, 1, 0, &ok);
    CHECK(ok);
    (void)rs;
    const double e = exact_nrm_d(x, n);
    CHECK(n == 0 ? r == 0.0 : fabs(r - e) <= 64 * 0x1p-53 * e);
    if (n > 0) {  /* Listing 1 is defined for n >= 1 (the tree calls it on P2 >= 1 tiles) */
      (void)oracle_R_H_d(n, x);
      (void)oracle_R_A_d(n, x);
      (void)oracle_R_H_s(n, xs);
    }
    (void)exact_nrm_s(xs, n);
    /* one-hot: the result is |c| for every position (neutral +0 padding) */
    if (n > 0) {
      for (int64_t i = 0; i < n; ++i) x[i] = 0.0;
      x[n / 2] = -0.75;
      CHECK(oracle_nrmf_tree_d(x, n, 4, 8, 1, 0, &ok) == 0.75);
    }
    free(x);
    free(xs);
  }
  /* the real tree shape at a few thousand elements, tiles and the tile API */
  {
    const int64_t n = 3 * 4096 + 17;
    double *x = (double *)malloc((size_t)n * sizeof(double));
    for (int64_t i = 0; i < n; ++i) x[i] = urand();
    int ok = 0;
    (void)oracle_nrmf_tree_d(x, n, 64, 64, 1, 0, &ok);
    CHECK(ok);
    double tv[4];
    CHECK(oracle_tiles_d(x, n, 64, 64, 0, 4, tv) == 1);
    free(x);
  }
  /* columns: ragged rows, ld > rows, empty shapes */
  {
    const int64_t r = 37, c = 5, ld = 41;
    double *A = (double *)malloc((size_t)(ld * c) * sizeof(double));
    float *As = (float *)malloc((size_t)(ld * c) * sizeof(float));
    for (int64_t i = 0; i < ld * c; ++i) { A[i] = 2.0 * urand() - 1.0; As[i] = (float)A[i]; }
    double cn[5], fr;
    float cns[5], frs;
    CHECK(oracle_nrmf_cols_d(r, c, ld, A, 4, 8, 0, cn, &fr) == 1);
    CHECK(oracle_nrmf_cols_s(r, c, ld, As, 8, 4, 0, cns, &frs) == 1);
    CHECK(oracle_nrmf_cols_d(0, c, ld, A, 4, 8, 0, cn, &fr) == 1 && fr == 0.0);
    CHECK(oracle_nrmf_cols_d(r, 0, ld, A, 4, 8, 0, cn, &fr) == 1 && fr == 0.0);
    free(A);
    free(As);
  }
  if (fails) return 1;
  printf("oracle under ASan/UBSan: ok\n");
  return 0;
}
