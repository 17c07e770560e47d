// qgemm_api.cu -- C ABI of libqgemm.so (include/qgemm.h); the library's one
// translation unit (kernels: qg_*.cuh; host runtime: qg_runtime.cuh; host-
// resident operands: qg_host_path.cuh).
//
// Device-operand calls: validation and quick returns (row a1), then the small
// kernel, the direct path, or the K-panel loop (row a6, Alg. 2's kappa loop,
// PAPER.md P:906-911) of pack A + B (a2, a3) and mainloop with fused epilogue
// (a4 + a5) -- all enqueued on the caller's stream.
#include <algorithm>
#include <atomic>
#include <climits>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <cuda_runtime.h>

#include "../../include/qgemm.h"
#include "qg_dmma.cuh"
#include "qg_pack.cuh"
#include "qg_simple.cuh"
#include "qg_small.cuh"
#include "qg_tc32.cuh"
#include "qg_tc32_2cta.cuh"


namespace {

#include "qg_runtime.cuh"

// Rows (r) x K panel of an operand as the pack kernel sees it (qg_pack.cuh).
template <typename T>
struct PackSpec {
  const T *X;
  int64_t ldx;
  int row_contig, conj;
};
template <typename T>
int panel_loop(const PackSpec<T> &pa, const PackSpec<T> &pb, int64_t M, int64_t N, int64_t K,
               const qg::Scalars<T> &sc, T *C, int64_t ldc, void *workspace, size_t workspace_bytes,
               cudaStream_t st, int tri);

template <typename T>
int qgemm_impl(char transA, char transB, int64_t M, int64_t N, int64_t K, const T *alpha, const T *A,
               int64_t lda, const T *B, int64_t ldb, const T *beta, T *C, int64_t ldc, void *workspace,
               size_t workspace_bytes, void *stream) {
  g_last_launches = 0;
  Shape sh;
  bool reads_ab = false;
  int rc = validate<T>(transA, transB, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, sh, reads_ab);
  if (rc != 0) return rc;
  if (M == 0 || N == 0) return 0;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  qg::Scalars<T> sc = make_scalars(alpha, beta);
  if (!reads_ab) {  // C <- beta C; nothing to do for beta = 1 (BLAS quick return)
    if (sc.beta_real && sc.beta[0] == T(1)) return 0;
    return launch_scale(C, ldc, M, N, sc, st);
  }
  PackSpec<T> pa{A, lda, sh.oa == 0 ? 1 : 0, sh.oa == 2 ? 1 : 0};
  PackSpec<T> pb{B, ldb, sh.ob == 0 ? 0 : 1, sh.ob == 2 ? 1 : 0};
  if (use_small<T>(M, N, K))  // one launch, no workspace (NEXT item 4)
    return launch_small<T>(A, lda, pa.row_contig, pa.conj, B, ldb, pb.row_contig, pb.conj, C, ldc, M, N, K,
                           alpha, beta, st);
  if (const int feed = direct_feed<T>(sh.oa, sh.ob, M, N, K)) {  // one launch; workspace = scratch only
    if (workspace == nullptr || (reinterpret_cast<uintptr_t>(workspace) & 255u)) return -14;
    if (workspace_bytes < sk_reserve<T>(M, N, cdiv(K, Geo<T>::kq))) return -15;
    if constexpr (sizeof(T) == 8)
      return launch_mainloop_direct(feed, A, lda, pa.row_contig, pa.conj, B, ldb, pb.row_contig, pb.conj, C,
                                    ldc, M, N, K, sc, workspace, st);
    else
      return launch_mainloop_direct_f32(A, lda, pa.row_contig, pa.conj, B, ldb, pb.row_contig, pb.conj, C, ldc, M,
                                        N, K, sc, workspace, st);
  }
  return panel_loop<T>(pa, pb, M, N, K, sc, C, ldc, workspace, workspace_bytes, st, 0);
}

// K-panel loop (row a6): pack A, pack B, mainloop per panel that fits.
template <typename T>
int panel_loop(const PackSpec<T> &pa, const PackSpec<T> &pb, int64_t M, int64_t N, int64_t K,
               const qg::Scalars<T> &sc, T *C, int64_t ldc, void *workspace, size_t workspace_bytes,
               cudaStream_t st, int tri) {
  int rc = 0;
  const int64_t KT_total = cdiv(K, Geo<T>::kq);
  const size_t min_ws = workspace_for<T>(M, N, K, 1);
  if (workspace == nullptr || (reinterpret_cast<uintptr_t>(workspace) & 255u)) return -14;
  if (workspace_bytes < min_ws) return -15;
  int64_t KTp = KT_total;
  while (KTp > 1 && workspace_for<T>(M, N, K, KTp) > workspace_bytes) {
    // largest panel that fits; start from a proportional estimate
    const size_t res = sk_reserve<T>(M, N, KT_total);
    int64_t est = int64_t((workspace_bytes - res) / bytes_per_ktile<T>(M, N));
    KTp = std::max<int64_t>(1, std::min<int64_t>(KTp - 1, est));
  }
  const int64_t MT = Geo<T>::a_tiles(M), NT = cdiv(N, Geo<T>::rows);
  T *Ap = reinterpret_cast<T *>(workspace);
  T *Bp = reinterpret_cast<T *>(reinterpret_cast<char *>(workspace) +
                                align256(size_t(MT) * size_t(KTp) * Geo<T>::chunk));
  void *sk_scratch = reinterpret_cast<char *>(Bp) + align256(size_t(NT) * size_t(KTp) * Geo<T>::chunk);
  qg::Scalars<T> sc_acc = sc;  // later panels accumulate: beta = 1
  for (int c = 0; c < 4; ++c) sc_acc.beta[c] = T(c == 0 ? 1 : 0);
  sc_acc.beta_real = 1;
  sc_acc.beta_zero = 0;
  for (int64_t kt0 = 0; kt0 < KT_total; kt0 += KTp) {
    const int64_t k_begin = kt0 * Geo<T>::kq;
    const int64_t k_end = std::min<int64_t>(K, (kt0 + KTp) * Geo<T>::kq);
    const int64_t ktn = cdiv(k_end - k_begin, Geo<T>::kq);
    rc = launch_pack2<T>(pack_job<T>(pa.X, pa.ldx, pa.row_contig, pa.conj, M, k_begin, k_end, ktn, Ap, true),
                         pack_job<T>(pb.X, pb.ldx, pb.row_contig, pb.conj, N, k_begin, k_end, ktn, Bp, false),
                         st);
    if (rc) return rc;
    rc = launch_mainloop(Ap, Bp, C, ldc, M, N, ktn, kt0 == 0 ? sc : sc_acc, sk_scratch, st, tri);
    if (rc) return rc;
  }
  return 0;
}

template <typename T>
size_t ws_bytes(char transA, char transB, int64_t M, int64_t N, int64_t K, bool minimum);

// QHERK: C <- alpha op(A) op(A)^H + beta C on one
// triangle, alpha/beta real; same pack + DMMA mainloop, triangular tile list.
int qherk_impl(char uplo, char trans, int64_t N, int64_t K, double alpha, const double *A, int64_t lda,
               double beta, double *C, int64_t ldc, void *workspace, size_t workspace_bytes, void *stream) {
  g_last_launches = 0;
  const int tri = (uplo == 'L' || uplo == 'l') ? 1 : (uplo == 'U' || uplo == 'u') ? 2 : 0;
  if (!tri) return -1;
  const int ot = op_code(trans);
  if (ot != 0 && ot != 2) return -2;  // 'N' or 'H'/'C' (no plain transpose, as BLAS xHERK)
  if (N < 0) return -3;
  if (K < 0) return -4;
  const int64_t a_rows = ot == 0 ? N : K, a_cols = ot == 0 ? K : N;
  if (lda < std::max<int64_t>(1, a_rows)) return -7;
  if (ldc < std::max<int64_t>(1, N)) return -10;
  if (N == 0) return 0;
  if (C == nullptr || (reinterpret_cast<uintptr_t>(C) & 15u)) return -9;
  const bool reads_a = K > 0 && alpha != 0.0;
  if (!reads_a && beta == 1.0) return 0;  // BLAS quick return
  if (reads_a) {
    if (A == nullptr || (reinterpret_cast<uintptr_t>(A) & 15u)) return -6;
    uintptr_t c0, c1, a0, a1;
    extent(C, N, N, ldc, c0, c1);
    extent(A, a_rows, a_cols, lda, a0, a1);
    if (overlaps(c0, c1, a0, a1)) return -9;
  }
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const double al[4] = {alpha, 0, 0, 0}, be[4] = {beta, 0, 0, 0};
  qg::Scalars<double> sc = make_scalars(al, be);
  if (!reads_a) return launch_scale(C, ldc, N, N, sc, st, tri);
  if (workspace == nullptr || (reinterpret_cast<uintptr_t>(workspace) & 255u)) return -11;
  if (const int feed = direct_feed<double>(ot, ot == 0 ? 2 : 0, N, N, K)) {
    if (workspace_bytes < sk_reserve<double>(N, N, cdiv(K, qg::kBK))) return -12;
    // same operand views as the packed path below (conj folded into the signs)
    return launch_mainloop_direct(feed, A, lda, ot == 0 ? 1 : 0, ot == 0 ? 0 : 1, A, lda, ot == 0 ? 1 : 0,
                                  ot == 0 ? 1 : 0, C, ldc, N, N, K, sc, workspace, st, tri);
  }
  if (workspace_bytes < workspace_for<double>(N, N, K, 1)) return -12;
  // op(A) as the A operand; op(B) = op(A)^H as the B operand (same buffer):
  //   trans N: op(A)(n,k) = A(n,k) -> rows contiguous;  B~(k,n) = conj(A(n,k))
  //   trans H: op(A)(n,k) = conj(A(k,n));                B~(k,n) = A(k,n)
  PackSpec<double> pa{A, lda, ot == 0 ? 1 : 0, ot == 0 ? 0 : 1};
  PackSpec<double> pb{A, lda, ot == 0 ? 1 : 0, ot == 0 ? 1 : 0};
  return panel_loop<double>(pa, pb, N, N, K, sc, C, ldc, workspace, workspace_bytes, st, tri);
}

template <typename T>
size_t ws_bytes(char transA, char transB, int64_t M, int64_t N, int64_t K, bool minimum) {
  if (op_code(transA) < 0 || op_code(transB) < 0 || M <= 0 || N <= 0 || K <= 0) return 0;
  if (use_small<T>(M, N, K)) return 0;  // the small kernel needs no workspace
  if (direct_feed<T>(op_code(transA), op_code(transB), M, N, K))
    return sk_reserve<T>(M, N, cdiv(K, Geo<T>::kq));  // stream-K scratch only
  return workspace_for<T>(M, N, K, minimum ? 1 : cdiv(K, Geo<T>::kq));
}

#include "qg_host_path.cuh"

}  // namespace

extern "C" {

int qgemm(char transA, char transB, int64_t M, int64_t N, int64_t K, const double alpha[4], const double *A,
          int64_t lda, const double *B, int64_t ldb, const double beta[4], double *C, int64_t ldc,
          void *workspace, size_t workspace_bytes, void *stream) {
  return qgemm_impl<double>(transA, transB, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, workspace,
                            workspace_bytes, stream);
}

int qgemm_f32(char transA, char transB, int64_t M, int64_t N, int64_t K, const float alpha[4], const float *A,
              int64_t lda, const float *B, int64_t ldb, const float beta[4], float *C, int64_t ldc,
              void *workspace, size_t workspace_bytes, void *stream) {
  return qgemm_impl<float>(transA, transB, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, workspace,
                           workspace_bytes, stream);
}

size_t qgemm_workspace_bytes(char transA, char transB, int64_t M, int64_t N, int64_t K, int dtype) {
  if (dtype == 0) return ws_bytes<double>(transA, transB, M, N, K, false);
  if (dtype == 1) return ws_bytes<float>(transA, transB, M, N, K, false);
  return 0;
}

size_t qgemm_workspace_min_bytes(char transA, char transB, int64_t M, int64_t N, int64_t K, int dtype) {
  if (dtype == 0) return ws_bytes<double>(transA, transB, M, N, K, true);
  if (dtype == 1) return ws_bytes<float>(transA, transB, M, N, K, true);
  return 0;
}

int qgemm_naive(char transA, char transB, int64_t M, int64_t N, int64_t K, const double alpha[4],
                const double *A, int64_t lda, const double *B, int64_t ldb, const double beta[4], double *C,
                int64_t ldc, void *stream) {
  g_last_launches = 0;
  Shape sh;
  bool reads_ab = false;
  int rc = validate<double>(transA, transB, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, sh, reads_ab);
  if (rc != 0) return rc;
  if (M == 0 || N == 0) return 0;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  qg::Scalars<double> sc = make_scalars(alpha, beta);
  if (!reads_ab) return launch_scale(C, ldc, M, N, sc, st);
  dim3 grid(unsigned(cdiv(M, 128)), unsigned(std::min<int64_t>(N, 65535)));
  { int ti = tstart(kNaive, st);
  qg::qgemm_naive_kernel<double><<<grid, 128, 0, st>>>(sh.oa, sh.ob, M, N, K, A, lda, B, ldb, C, ldc, sc);
  tstop(ti, st); }
  ++g_last_launches;
  return int(cudaGetLastError());
}

int qgemm_pack_panel(char trans, int operand, int64_t R, int64_t K, const double *X, int64_t ldx, double *out,
                     size_t out_bytes, void *stream) {
  g_last_launches = 0;
  const int op = op_code(trans);
  if (op < 0) return -1;
  if (operand != 0 && operand != 1) return -2;
  if (R < 0) return -3;
  if (K < 0) return -4;
  // operand A: op N reads rows contiguously; operand B: op T/H does (qg_pack.cuh)
  const int rc = operand == 0 ? (op == 0) : (op != 0);
  if (ldx < std::max<int64_t>(1, rc ? R : K)) return -6;
  if (R == 0 || K == 0) return 0;
  if (X == nullptr || (reinterpret_cast<uintptr_t>(X) & 15u)) return -5;
  const int64_t KT = cdiv(K, qg::kBK);
  const size_t need = size_t(cdiv(R, qg::kBR)) * size_t(KT) * size_t(qg::kChunkElems) * sizeof(double);
  if (out == nullptr || (reinterpret_cast<uintptr_t>(out) & 15u)) return -7;
  if (out_bytes < need) return -8;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  qg::PackJob<double> none{};
  none.blocks = 0;
  return launch_pack2<double>(pack_job<double>(X, ldx, rc, op == 2, R, 0, K, KT, out, operand == 0), none, st);
}

int qherk(char uplo, char trans, int64_t N, int64_t K, double alpha, const double *A, int64_t lda, double beta,
          double *C, int64_t ldc, void *workspace, size_t workspace_bytes, void *stream) {
  return qherk_impl(uplo, trans, N, K, alpha, A, lda, beta, C, ldc, workspace, workspace_bytes, stream);
}

size_t qherk_workspace_bytes(char uplo, char trans, int64_t N, int64_t K) {
  const int ot = op_code(trans);
  if (!(uplo == 'L' || uplo == 'l' || uplo == 'U' || uplo == 'u') || (ot != 0 && ot != 2) || N <= 0 || K <= 0)
    return 0;
  if (direct_feed<double>(ot, ot == 0 ? 2 : 0, N, N, K)) return sk_reserve<double>(N, N, cdiv(K, qg::kBK));
  return workspace_for<double>(N, N, K, cdiv(K, qg::kBK));
}

int qgemm_host(char transA, char transB, int64_t M, int64_t N, int64_t K, const double alpha[4],
               const double *A, int64_t lda, const double *B, int64_t ldb, const double beta[4], double *C,
               int64_t ldc, void *workspace, size_t workspace_bytes, void *stream) {
  return qgemm_host_impl<double>(transA, transB, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, workspace,
                                 workspace_bytes, stream);
}

int qgemm_host_f32(char transA, char transB, int64_t M, int64_t N, int64_t K, const float alpha[4],
                   const float *A, int64_t lda, const float *B, int64_t ldb, const float beta[4], float *C,
                   int64_t ldc, void *workspace, size_t workspace_bytes, void *stream) {
  return qgemm_host_impl<float>(transA, transB, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, workspace,
                                workspace_bytes, stream);
}

size_t qgemm_host_workspace_bytes(char transA, char transB, int64_t M, int64_t N, int64_t K, int dtype) {
  if (dtype == 0) return host_ws_bytes<double>(transA, transB, M, N, K);
  if (dtype == 1) return host_ws_bytes<float>(transA, transB, M, N, K);
  return 0;
}

int qgemm_last_launch_count(void) { return g_last_launches; }

int qgemm_set_path_policy(int policy) {
  if (policy < 0 || policy > 5) return -1;
  return g_path_policy.exchange(policy);
}

void qgemm_timing_enable(int on) { g_timing.on = on != 0; }

int qgemm_timing_collect(double ms[5], int counts[5]) {
  for (int k = 0; k < kKinds; ++k) { ms[k] = 0.0; counts[k] = 0; }
  int rc = 0;
  for (const TimingRec &r : g_timing.recs) {
    cudaError_t e = cudaEventSynchronize(r.e1);
    float t = 0.f;
    if (e == cudaSuccess) e = cudaEventElapsedTime(&t, r.e0, r.e1);
    if (e != cudaSuccess && rc == 0) rc = int(e);
    ms[r.kind] += double(t);
    counts[r.kind] += 1;
    g_timing.pool.push_back(r.e0);
    g_timing.pool.push_back(r.e1);
  }
  g_timing.recs.clear();
  return rc;
}

const char *qgemm_version(void) {
  return "qgemm-b200 0.3 (sm_100a; FP64 DMMA.8x8x4 persistent stream-K, packed or TMA-fed; "
         "FP32 tcgen05 3xTF32; one-launch small kernel)";
}

#ifdef QG_TRACE
// Diagnostic builds only (-DQG_TRACE, not declared in include/qgemm.h): copy the
// DMMA kernel's phase trace (256 CTAs x 48 events, see qg_dmma.cuh) to host and
// clear it.
int qgemm_debug_trace(unsigned long long *host, int n) {
  const size_t bytes = std::min(size_t(n), size_t(256 * qg::kTraceEv)) * sizeof(unsigned long long);
  cudaError_t e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaMemcpyFromSymbol(host, qg::g_trace, bytes);
  static unsigned long long zeros[256 * qg::kTraceEv];
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(qg::g_trace, zeros, sizeof(zeros));
  return int(e);
}
#endif

}  // extern "C"
