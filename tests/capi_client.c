/* capi_client.c — a plain-C caller of libgk_b200.so through include/gk_capi.h
 * only (no Python, no torch): the drop-in boundary exercised the way a
 * reference-side binding would drive it.
 *
 * Pipeline (GpModel on D-SKI, gp.cpp:117-187): the C1 workload's first 200
 * points (gk_make_dataset), Grid::cover, DskiOperator with noise (0.3, 0.3),
 * one MVM of the stacked targets, the rank-60 pivoted-Cholesky
 * preconditioner of the kernel part, GpModel::solve and
 * log_marginal_likelihood (SLQ 8 probes × 25 steps), and the predictive mean
 * + gradient at 5 points. Results go to a little-endian binary file
 * (argv[1]) that tests/test_gpu_capi_client.py checks against the oracle.
 *
 * Build: gcc -std=c99 -I include tests/capi_client.c -L<lib> -lgk_b200 -lm */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "gk_capi.h"

#define CHECK(call)                                                              \
  do {                                                                           \
    gk_status s_ = (call);                                                       \
    if (s_ != GK_OK) {                                                           \
      fprintf(stderr, "%s failed: status %d: %s\n", #call, (int)s_, gk_last_error()); \
      return 2;                                                                  \
    }                                                                            \
  } while (0)

static int put(FILE* f, const char* tag, const double* v, int64_t n) {
  /* record: 8-byte tag, int64 count, n doubles */
  char t[8] = {0};
  size_t len = strlen(tag);
  memcpy(t, tag, len < 8 ? len : 8);
  if (fwrite(t, 1, 8, f) != 8 || fwrite(&n, sizeof n, 1, f) != 1) return 1;
  return fwrite(v, sizeof(double), (size_t)n, f) != (size_t)n;
}

int main(int argc, char** argv) {
  if (argc != 2) {
    fprintf(stderr, "usage: %s OUT.bin\n", argv[0]);
    return 1;
  }
  int64_t nfull = 0;
  int d = 0;
  CHECK(gk_make_dataset(1, 0, &nfull, &d, NULL, NULL, NULL));
  double* Xf = malloc(sizeof(double) * nfull * d);
  double* yf = malloc(sizeof(double) * nfull);
  double* dYf = malloc(sizeof(double) * nfull * d);
  CHECK(gk_make_dataset(1, 0, &nfull, &d, Xf, yf, dYf));

  const int64_t n = 200;
  double* X = malloc(sizeof(double) * n * d);
  for (int j = 0; j < d; ++j) memcpy(X + j * n, Xf + j * nfull, sizeof(double) * n);
  /* stacked targets [y - mean; dY_1; ...; dY_d] (observations.hpp:29-35, gp.cpp:43) */
  const int64_t N = n * (d + 1);
  double mean = 0;
  for (int64_t i = 0; i < n; ++i) mean += yf[i];
  mean /= (double)n;
  double* t = malloc(sizeof(double) * N);
  for (int64_t i = 0; i < n; ++i) t[i] = yf[i] - mean;
  for (int j = 0; j < d; ++j)
    for (int64_t i = 0; i < n; ++i) t[(j + 1) * n + i] = dYf[j * nfull + i];

  gk_kernel ker = {0, 0.15, 1.0, 0.0, 0.0, 0};
  gk_grid grid;
  CHECK(gk_grid_cover(X, n, d, 1e-3, 3, 40, &grid));
  gk_op* op = NULL;
  CHECK(gk_dski_create(&ker, &grid, X, n, 0.3, 0.3, 0, 1, 0, &op));
  if (gk_op_size(op) != N) {
    fprintf(stderr, "operator size %lld != %lld\n", (long long)gk_op_size(op), (long long)N);
    return 2;
  }

  double* Kt = malloc(sizeof(double) * N);
  CHECK(gk_op_mvm(op, t, N, Kt, N, 1));

  gk_pivchol* f = NULL;
  CHECK(gk_pivoted_cholesky(op, 1, 60, 0.0, &f));
  const int64_t rank = gk_pivchol_rank(f);
  int64_t* piv = malloc(sizeof(int64_t) * rank);
  double* pivd = malloc(sizeof(double) * rank);
  CHECK(gk_pivchol_get(f, NULL, piv, NULL, NULL));
  for (int64_t k = 0; k < rank; ++k) pivd[k] = (double)piv[k];
  gk_precond* M = NULL;
  CHECK(gk_precond_from_pivchol(op, f, &M));

  double* alpha = malloc(sizeof(double) * N);
  int its = 0;
  CHECK(gk_gp_solve(op, M, t, N, 1, 1e-8, 2000, alpha, N, &its));
  double lml = 0, fit = 0, logdet = 0;
  CHECK(gk_gp_log_marginal_likelihood(op, M, t, 1e-8, 2000, 8, 25, 0, 0.3, 0.3, 1, &lml, &fit,
                                      &logdet, NULL));

  const int64_t T = 5;
  double* Xt = malloc(sizeof(double) * T * d);
  for (int j = 0; j < d; ++j)
    for (int64_t i = 0; i < T; ++i) Xt[j * T + i] = X[j * n + 10 * i + 3];
  double* mu = malloc(sizeof(double) * T);
  double* grad = malloc(sizeof(double) * T * d);
  CHECK(gk_dski_predict_mean_grad(op, alpha, mean, Xt, T, mu, grad));

  /* an error path: a row index out of range is std::out_of_range (dski.cpp:293) */
  double* row = malloc(sizeof(double) * N);
  gk_status rs = gk_op_row(op, N, row);
  double err_code = (double)rs;

  FILE* out = fopen(argv[1], "wb");
  if (!out) return 3;
  double meta[4] = {(double)n, (double)d, (double)its, (double)rank};
  double scal[3] = {lml, fit, logdet};
  int bad = put(out, "meta", meta, 4) | put(out, "Kt", Kt, N) | put(out, "pivots", pivd, rank) |
            put(out, "alpha", alpha, N) | put(out, "lml", scal, 3) | put(out, "mu", mu, T) |
            put(out, "grad", grad, T * d) | put(out, "rowerr", &err_code, 1);
  fclose(out);
  printf("capi_client: N=%lld rank=%lld its=%d lml=%.12g launches=%lld\n", (long long)N,
         (long long)rank, its, lml, (long long)gk_kernel_launch_count());

  gk_precond_destroy(M);
  gk_pivchol_destroy(f);
  gk_op_destroy(op);
  free(Xf); free(yf); free(dYf); free(X); free(t); free(Kt); free(piv); free(pivd);
  free(alpha); free(Xt); free(mu); free(grad); free(row);
  return bad ? 4 : 0;
}
