/*
 * Minimal C caller of the hjb200 C ABI (include/hjb200.h): what a non-Python
 * host (or the reference's own FFI) would bind.  Builds with any C99 compiler:
 *
 *   gcc -std=c99 -Iinclude examples/solve_c.c -o solve_c \
 *       -Lpaper_1008_4166_b200 -l:libhjb200.so -Wl,-rpath,$PWD/paper_1008_4166_b200 -lm
 *
 * Solves a small seeded problem (G 96 x 64, 40 positive and 24 negative
 * signs) with p = 4 ring workers and prints the DiagInfo fields and the
 * extreme eigenvalues lambda_k = j_k ||g_k||^2.
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "hjb200.h"

int main(void) {
  const int64_t m = 96, n = 64;
  double *G = malloc(sizeof(double) * m * n), *Gout = malloc(sizeof(double) * m * n);
  int8_t *J = malloc(n);
  unsigned s = 12345u;
  for (int64_t k = 0; k < m * n; ++k) { /* column-major, LCG noise in [-1, 1) */
    s = s * 1664525u + 1013904223u;
    G[k] = (double)(s >> 8) / 8388608.0 - 1.0;
  }
  for (int64_t k = 0; k < n; ++k) J[k] = k < 40 ? 1 : -1;
  if (hjb_device_count() < 1) {
    fprintf(stderr, "no CUDA device: the library has no CPU fallback\n");
    return 2;
  }
  hjb_problem pr = {0};
  pr.dtype = HJB_F64;
  pr.memspace = HJB_HOST;
  pr.m = m;
  pr.n = n;
  pr.ldg = m;
  pr.G_in = G;
  pr.G_out = Gout;
  pr.signs = J;
  pr.p = 4;
  pr.strategy = HJB_ROUND_ROBIN;
  pr.orth_tol = (double)n * 2.220446049250313e-16;
  pr.quad_tol = -1.0;
  pr.max_sweeps = 30;
  hjb_result res;
  const int rc = hjb_solve(&pr, &res);
  if (rc != HJB_OK) {
    fprintf(stderr, "hjb_solve: status %d: %s\n", rc, hjb_last_error());
    return 1;
  }
  double lo = INFINITY, hi = -INFINITY;
  for (int64_t c = 0; c < n; ++c) {
    double d = 0.0;
    for (int64_t r = 0; r < m; ++r) d += Gout[r + c * m] * Gout[r + c * m];
    d *= J[c];
    lo = d < lo ? d : lo;
    hi = d > hi ? d : hi;
  }
  printf("sweeps %d converged %d rotations %lld lambda in [%.6g, %.6g]\n", res.sweeps, res.converged,
         (long long)res.rotations, lo, hi);
  free(G);
  free(Gout);
  free(J);
  return res.converged ? 0 : 3;
}
