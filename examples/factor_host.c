/* Plain-C use of the C ABI (include/rcholqr.h): Algorithm 2 of a tall-and-skinny host matrix
 * through rcholqr_factor_host -- no CUDA headers, no Python.  Builds a seeded X = G diag(sigma) (cond 1e3), factors
 * it with a Gaussian and a sparse-sign Theta, and checks on the host that X = QR to rounding, that R is upper
 * triangular with a positive diagonal, and that cond(Q) is small (sketched orthogonality).
 *
 *   gcc -O2 -Iinclude examples/factor_host.c -Lpaper_2210_09953_b200/lib -lrcholqr -Wl,-rpath,$PWD/paper_2210_09953_b200/lib -lm -o factor_host
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include "rcholqr.h"

static double lcg_normal(unsigned long long* s) {   /* sum of 12 uniforms - 6: enough for a test matrix */
  double a = 0.0;
  for (int t = 0; t < 12; ++t) {
    *s = *s * 6364136223846793005ULL + 1442695040888963407ULL;
    a += (double)(*s >> 11) * (1.0 / 9007199254740992.0);
  }
  return a - 6.0;
}

static int run(int sketch, const char* name) {
  const long long m = 200000;
  const int n = 32, k = 64;
  double* X = malloc(sizeof(double) * m * n);
  double* Q = malloc(sizeof(double) * m * n);
  double* R = malloc(sizeof(double) * n * n);
  unsigned long long s = 12345;
  for (long long i = 0; i < m; ++i)
    for (int j = 0; j < n; ++j) X[i * n + j] = lcg_normal(&s) * pow(10.0, -3.0 * j / (n - 1));
  rcholqr_desc d = {n, k, RCHOLQR_F64, sketch, 8, 0, 7ULL, NULL};
  rcholqr_plan plan = NULL;
  rcholqr_status st = rcholqr_create(&d, &plan);
  if (st != RCHOLQR_OK) { printf("%s: create failed: %s\n", name, rcholqr_strerror(st)); return 1; }
  st = rcholqr_factor_host(plan, X, m, 0, n, Q, n, R, NULL, NULL);
  if (st != RCHOLQR_OK) { printf("%s: factor failed: %s\n", name, rcholqr_strerror(st)); return 1; }
  uint32_t path = 0;
  rcholqr_last_path(plan, &path, NULL);
  double res = 0.0, nx = 0.0, lower = 0.0, mind = 1e300;
  for (long long i = 0; i < m; i += 97)                /* sampled rows: X_i = Q_i R */
    for (int j = 0; j < n; ++j) {
      double a = 0.0;
      for (int l = 0; l <= j; ++l) a += Q[i * n + l] * R[l * n + j];
      res += (a - X[i * n + j]) * (a - X[i * n + j]);
      nx += X[i * n + j] * X[i * n + j];
    }
  for (int i = 0; i < n; ++i) {
    if (R[i * n + i] < mind) mind = R[i * n + i];
    for (int j = 0; j < i; ++j) lower += fabs(R[i * n + j]);
  }
  /* Gram of Q: its extreme eigenvalues bound cond(Q)^2; Gershgorin-free check through the trace and the
   * largest off-diagonal entry is enough for an example: for k = 2n the squared column norms of Q lie in [0.34, 11.7] (eq:sketchedcond with eps = sqrt(n/k)) */
  double offmax = 0.0, dmin = 1e300, dmax = 0.0;
  for (int a = 0; a < n; ++a)
    for (int b = a; b < n; ++b) {
      double g = 0.0;
      for (long long i = 0; i < m; ++i) g += Q[i * n + a] * Q[i * n + b];
      if (a == b) { if (g < dmin) dmin = g; if (g > dmax) dmax = g; }
      else if (fabs(g) > offmax) offmax = fabs(g);
    }
  printf("%s: status=%s path=0x%x residual=%.3e lower(R)=%.1e min diag(R)=%.3e diag(Q^T Q) in [%.3f, %.3f] offdiag<=%.3f\n",
         name, rcholqr_strerror(st), path, sqrt(res / nx), lower, mind, dmin, dmax, offmax);
  const int ok = sqrt(res / nx) <= 1e-13 && lower == 0.0 && mind > 0.0 && dmin > 0.2 && dmax < 12.0;
  rcholqr_destroy(plan);
  free(X); free(Q); free(R);
  return ok ? 0 : 1;
}

int main(void) {
  int bad = run(RCHOLQR_GAUSSIAN, "gaussian") + run(RCHOLQR_SPARSE_SIGN, "sparse-sign") + run(RCHOLQR_SRHT, "srht");
  printf(bad ? "FAILED\n" : "c abi example ok\n");
  return bad;
}
