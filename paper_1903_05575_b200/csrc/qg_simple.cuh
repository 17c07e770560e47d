// qg_simple.cuh -- the two elementwise kernels of the library:
//   * qgemm_scale_kernel: C <- beta (x) C, the quick-return path for alpha == 0
//     or K == 0 (BLAS convention, R4); beta == 0 writes zeros without
//     reading C (R3).  HBM-bound.
//   * qgemm_naive_kernel: one thread per output quaternion, reading op(A) and
//     op(B) in place -- Alg. 1's arithmetic without packing.  A
//     debug / cross-check path exported as qgemm_naive(); qgemm() never uses it.
#pragma once
#include "qg_common.cuh"

namespace qg {

// tri = 1/2: only the lower/upper triangle (incl. diagonal) is touched and the
// diagonal's vector part is set to 0 (QHERK, R18).
template <typename T>
__global__ void qgemm_scale_kernel(T *C, int64_t ldc, int64_t M, int64_t N, Scalars<T> sc, int tri) {
  const int64_t total = M * N;
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
       idx += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = idx % M, j = idx / M;
    if (tri == 1 && i < j) continue;
    if (tri == 2 && i > j) continue;
    T *p = C + 4 * (i + j * ldc);
    T out[4] = {T(0), T(0), T(0), T(0)};
    if (!sc.beta_zero) {
      T c[4];
      ldq_c(p, c);
      left_scale(sc.beta, sc.beta_real, c, out);
    }
    if (tri != 0 && i == j) out[1] = out[2] = out[3] = T(0);
    stq(p, out);
  }
}

// Y <- Y + beta (x) X (left quaternion product): folds the caller's C into the
// accumulated alpha op(A) op(B) of the host-streamed path (qgemm_host).  HBM-bound.
template <typename T>
__global__ void qgemm_axpby_kernel(T *Y, int64_t ldy, const T *X, int64_t ldx, int64_t M, int64_t N,
                                   Scalars<T> sc) {
  const int64_t total = M * N;
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
       idx += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = idx % M, j = idx / M;
    T x[4], bx[4], y[4];
    ldq(X + 4 * (i + j * ldx), x);
    ldq_c(Y + 4 * (i + j * ldy), y);
    left_scale(sc.beta, sc.beta_real, x, bx);
#pragma unroll
    for (int c = 0; c < 4; ++c) y[c] += bx[c];
    stq(Y + 4 * (i + j * ldy), y);
  }
}

template <typename T>
__global__ void qgemm_naive_kernel(int opA, int opB, int64_t M, int64_t N, int64_t K, const T *A, int64_t lda,
                                   const T *B, int64_t ldb, T *C, int64_t ldc, Scalars<T> sc) {
  const int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (i >= M) return;
  for (int64_t j = blockIdx.y; j < N; j += gridDim.y) {
    T t[4] = {T(0), T(0), T(0), T(0)};
    for (int64_t k = 0; k < K; ++k) {
      T a[4], b[4], pr[4];
      ldq(opA == 0 ? A + 4 * (i + k * lda) : A + 4 * (k + i * lda), a);
      ldq(opB == 0 ? B + 4 * (k + j * ldb) : B + 4 * (j + k * ldb), b);
      if (opA == 2) { a[1] = -a[1]; a[2] = -a[2]; a[3] = -a[3]; }
      if (opB == 2) { b[1] = -b[1]; b[2] = -b[2]; b[3] = -b[3]; }
      hmul(a, b, pr);
#pragma unroll
      for (int c = 0; c < 4; ++c) t[c] += pr[c];
    }
    epilogue_one(sc, t, C + 4 * (i + j * ldc));
  }
}

}  // namespace qg
