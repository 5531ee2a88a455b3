/* certify.c -- the C ABI used from plain C (no Python): robust stability of x' = A(alpha) x on the
 * simplex by the Polya relaxation (Sec. III, Algorithm 2), for a 2-vertex, 4-state system
 * and an unstable copy of it.  Set-up (polya_setup), Algorithm 2 to its stopping rule
 * (polya_ipm_solve: apply / adjoint / Schur kernels + the K x K factorisation) and the grid check
 * of the certificate (polya_verdict), all on the GPU.
 *
 * Build: gcc -O2 -I include examples/certify.c -L paper_1411_3769_b200 -lpolya \
 *            -Wl,-rpath,$PWD/paper_1411_3769_b200 -L /usr/local/cuda/lib64 -lcudart -o build/certify
 * Run:   build/certify          (prints one line per system; exit 0 iff stable certified, unstable not) */
#include <stdio.h>
#include <stdlib.h>

#include <cuda_runtime_api.h>

#include "polya.h"

#define N 4
#define L 2

static int certify(const double* A, const char* name) {
  polya_config cfg = {N, L, /*dp*/ 1, /*da*/ 1, /*d1*/ 1, /*d2*/ 1, /*delta*/ 1e-3, /*rank*/ 0, /*nranks*/ 1,
                      POLYA_SHARD_TILES};
  polya_ctx* ctx = NULL;
  polya_status st = polya_setup(&cfg, A, &ctx);
  if (st != POLYA_OK) {
    fprintf(stderr, "polya_setup: %s\n", polya_strerror(st));
    return -1;
  }
  polya_dims d;
  polya_dims_get(ctx, &d);
  const size_t blk = (size_t)d.nblocks * d.block_n * d.block_n * sizeof(double);
  double *X = NULL, *Z = NULL, *y = NULL;
  if (cudaMalloc((void**)&X, blk) != cudaSuccess || cudaMalloc((void**)&Z, blk) != cudaSuccess ||
      cudaMalloc((void**)&y, (size_t)d.K * sizeof(double)) != cudaSuccess) {
    fprintf(stderr, "cudaMalloc failed\n");
    return -1;
  }
  polya_ipm_state s = {X, Z, y, 0.0, 0};
  polya_solve_opts opt = {1e-8, 1e-8, 60, 1, NULL};
  polya_solve_result res;
  st = polya_ipm_solve(ctx, &s, &opt, &res, NULL);
  if (st != POLYA_OK) {
    fprintf(stderr, "polya_ipm_solve: %s (%s)\n", polya_strerror(st), polya_last_error(ctx));
    return -1;
  }
  /* vertices, edge midpoint and a few interior points of the simplex */
  const double pts[][L] = {{1, 0}, {0, 1}, {0.5, 0.5}, {0.1, 0.9}, {0.3, 0.7}, {0.7, 0.3}, {0.9, 0.1}};
  int32_t nfail = -1;
  if (res.converged) polya_verdict(ctx, y, (int32_t)(sizeof(pts) / sizeof(pts[0])), &pts[0][0], &nfail, NULL);
  const int certified = res.converged && nfail == 0;
  printf("%s: K=%lld blocks=%lld iterations=%d gap=%.2e status=%s grid_failures=%d certified=%d\n", name,
         (long long)d.K, (long long)d.nblocks, res.iterations, res.gap, polya_strerror((polya_status)res.status),
         nfail, certified);
  cudaFree(X);
  cudaFree(Z);
  cudaFree(y);
  polya_destroy(ctx);
  return certified;
}

int main(void) {
  /* A_1 = -2 I + S_1 + K_1, A_2 = -2 I + S_2 + K_2 (symmetric part < -I: robustly stable) */
  double A[L][N][N];
  for (int v = 0; v < L; ++v)
    for (int i = 0; i < N; ++i)
      for (int j = 0; j < N; ++j) {
        const double sym = 0.05 * (double)((i + 2 * j + 3 * v) % 5 - 2) + 0.05 * (double)((j + 2 * i + 3 * v) % 5 - 2);
        const double skew = (i < j ? 1.0 : i > j ? -1.0 : 0.0) * (0.3 + 0.2 * v + 0.1 * (i + j));
        A[v][i][j] = (i == j ? -2.0 : 0.0) + sym + skew;
      }
  const int stable = certify(&A[0][0][0], "stable");
  for (int i = 0; i < N; ++i) A[1][i][i] += 3.0; /* vertex 2 shifted by +3 I: unstable */
  const int unstable = certify(&A[0][0][0], "unstable");
  return (stable == 1 && unstable == 0) ? 0 : 1;
}
