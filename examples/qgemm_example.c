/*
 * qgemm_example.c -- calling libqgemm.so from plain C (include/qgemm.h).
 *
 *   C <- alpha * A * B^H + beta * C   over the quaternions, FP64, M=5 N=3 K=4
 *
 * Build (from the repo root, after `python -c "import __graft_entry__ as g; g.build()"`):
 *   gcc -std=c11 -O2 -Iinclude -I/usr/local/cuda/include examples/qgemm_example.c \
 *       -Lpaper_1903_05575_b200 -lqgemm -L/usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,$PWD/paper_1903_05575_b200 -o qgemm_example
 * The result is checked against a direct evaluation of the Hamilton product
 * written here (a usage demo, not the test oracle).
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <cuda_runtime_api.h>

#include "qgemm.h"

enum { M = 5, N = 3, K = 4 };

/* out = p q (Hamilton product) */
static void hamilton(const double *p, const double *q, double *out) {
  out[0] = p[0] * q[0] - p[1] * q[1] - p[2] * q[2] - p[3] * q[3];
  out[1] = p[0] * q[1] + p[1] * q[0] + p[2] * q[3] - p[3] * q[2];
  out[2] = p[0] * q[2] - p[1] * q[3] + p[2] * q[0] + p[3] * q[1];
  out[3] = p[0] * q[3] + p[1] * q[2] - p[2] * q[1] + p[3] * q[0];
}

int main(void) {
  /* column-major, interleaved: X(i, j) at X[4 * (i + j * ld)] */
  double A[4 * M * K], B[4 * N * K], C[4 * M * N], ref[4 * M * N];
  const double alpha[4] = {0.5, 0.0, 0.0, 0.0}, beta[4] = {1.0, 0.0, 0.0, 0.0};
  for (int i = 0; i < 4 * M * K; ++i) A[i] = (double)((i * 7) % 11) / 5.0 - 1.0;
  for (int i = 0; i < 4 * N * K; ++i) B[i] = (double)((i * 5) % 13) / 6.0 - 1.0;
  for (int i = 0; i < 4 * M * N; ++i) C[i] = ref[i] = (double)(i % 9) / 4.0 - 1.0;

  /* reference: C(i,j) = alpha * sum_k A(i,k) conj(B(j,k)) + beta * C(i,j)   (op(B) = B^H) */
  for (int j = 0; j < N; ++j)
    for (int i = 0; i < M; ++i) {
      double t[4] = {0, 0, 0, 0}, pr[4], bc[4], s[4];
      for (int k = 0; k < K; ++k) {
        const double *b = &B[4 * (j + k * N)];
        bc[0] = b[0]; bc[1] = -b[1]; bc[2] = -b[2]; bc[3] = -b[3];
        hamilton(&A[4 * (i + k * M)], bc, pr);
        for (int c = 0; c < 4; ++c) t[c] += pr[c];
      }
      hamilton(alpha, t, s);
      for (int c = 0; c < 4; ++c) ref[4 * (i + j * M) + c] = s[c] + beta[0] * ref[4 * (i + j * M) + c];
    }

  double *dA, *dB, *dC;
  void *ws = NULL;
  const size_t wsb = qgemm_workspace_bytes('N', 'H', M, N, K, 0); /* 0 here: small-problem path */
  if (cudaMalloc((void **)&dA, sizeof A) || cudaMalloc((void **)&dB, sizeof B) ||
      cudaMalloc((void **)&dC, sizeof C) || (wsb && cudaMalloc(&ws, wsb))) {
    fprintf(stderr, "cudaMalloc failed\n");
    return 2;
  }
  cudaMemcpy(dA, A, sizeof A, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B, sizeof B, cudaMemcpyHostToDevice);
  cudaMemcpy(dC, C, sizeof C, cudaMemcpyHostToDevice);
  const int rc = qgemm('N', 'H', M, N, K, alpha, dA, M, dB, N, beta, dC, M, ws, wsb, NULL);
  if (rc != 0) {
    fprintf(stderr, "qgemm returned %d\n", rc);
    return 3;
  }
  cudaMemcpy(C, dC, sizeof C, cudaMemcpyDeviceToHost); /* synchronises the legacy stream */
  double err = 0.0;
  for (int i = 0; i < 4 * M * N; ++i) err = fmax(err, fabs(C[i] - ref[i]));
  printf("%s: %s, max |C - ref| = %.3e, %d kernel(s)\n", qgemm_version(), err < 1e-12 ? "OK" : "MISMATCH", err,
         qgemm_last_launch_count());
  cudaFree(dA); cudaFree(dB); cudaFree(dC);
  if (ws) cudaFree(ws);
  return err < 1e-12 ? 0 : 1;
}
