/*
 * qgemm.h -- C ABI of the B200-native quaternion GEMM library (libqgemm.so).
 *
 * Operation (arXiv 1903.05575 = PAPER.md; "P:n" = PAPER.md line n):
 *
 *     C <- alpha * op(A) * op(B) + beta * C                Eq. general_gemm
 *
 * over the Hamilton quaternions H (Eq. quaternion_def, product
 * Eq. quaternion_prod), op(X) in {X, X^T, X^H}, where
 * (X^H)_{mu nu} = conj(X_{nu mu}) and conj is Eq. quaternion_conj
 * (P:330-334).  op(A) is M x K, op(B) is K x N, C is M x N.
 *
 * Scalars: alpha and beta are quaternions applied FROM THE LEFT,
 *     (q P Q)_{mu nu} = q * sum_k P_{mu k} Q_{k nu}
 * (reading R2).  A real scalar r is passed as {r, 0, 0, 0}.
 *
 * Storage: column-major; element (i, j) of a stored
 * matrix X with leading dimension ldx occupies the 4 consecutive scalars
 *     X[4*(i + j*ldx) + c],  c = 0..3  (components q^0, q^1, q^2, q^3).
 * Leading dimensions are counted in QUATERNIONS:
 *     lda >= max(1, M) for transA = 'N', else lda >= max(1, K)
 *     ldb >= max(1, K) for transB = 'N', else ldb >= max(1, N)
 *     ldc >= max(1, M)
 * Rows beyond the logical extent (the ld padding) are never read or written.
 *
 * op characters: 'N' (no-op), 'T' (transpose, no conjugation), 'H' or 'C'
 * (conjugate transpose), case-insensitive (reading R6).
 *
 * Ownership: A, B, C and workspace are caller-owned DEVICE pointers on the
 * device current for the calling thread; alpha and beta are HOST pointers to 4
 * scalars, read before the call returns.  The library allocates nothing, and
 * keeps no reference to any argument once the enqueued work has completed.
 * `stream` is a cudaStream_t (NULL = legacy default stream).
 *
 * Asynchrony: the call validates, enqueues the pack / mainloop / epilogue
 * kernels on `stream` and returns.  Faults that happen while the kernels run
 * surface at the caller's next synchronisation on that stream.
 *
 * Quick returns (BLAS convention; reading R4):
 *     M == 0 or N == 0      -> returns 0, enqueues nothing;
 *     alpha == 0 or K == 0  -> C <- beta * C (one elementwise kernel; nothing
 *                              is enqueued when beta == 1);
 *     beta == 0             -> C is overwritten and never read (NaN in C does
 *                              not propagate; reading R3).
 *
 * Error convention (LAPACK "info" style; reading R7):
 *     0   success (work enqueued)
 *    -i   the i-th argument is invalid, numbering
 *           transA=1 transB=2 M=3 N=4 K=5 alpha=6 A=7 lda=8 B=9 ldb=10
 *           beta=11 C=12 ldc=13 workspace=14 workspace_bytes=15 stream=16;
 *         a C extent overlapping the A or B extent returns -12;
 *         NULL A/B are accepted only when they are not read (K == 0 or alpha == 0);
 *         A, B and C must be 16-byte aligned (every kernel moves whole
 *         quaternions with 16-byte vector accesses): otherwise -7/-9/-12;
 *         the workspace must be 256-byte aligned: otherwise -14.
 *    >0   a cudaError_t raised while enqueueing.
 * Nothing is enqueued when the return value is non-zero.
 *
 * Workspace: qgemm_workspace_bytes() returns the size that lets the call pack
 * all of op(A) and op(B) at once.  A smaller workspace is accepted down to the
 * size of a single K-panel (qgemm_workspace_min_bytes); the call then loops over
 * K-panels (Alg. 2 kappa loop), applying beta on the first panel and
 * accumulating onto C afterwards.  Smaller -> -15.
 * The workspace must be 256-byte aligned (-14 otherwise).  When an FP64 call
 * takes the direct path (no pack; see the path policy below), both functions
 * return the stream-K scratch size only (~33 MB) and no K-panel loop runs.
 *
 * Small problems: below the library's measured
 * crossover (FP64: M*N*K <= 2^25 quaternion multiply-adds, K <= 16, or at most
 * 64 output tiles of 64 x 64 with K >= 4 max(M, N); FP32: <= 2^25, or
 * M <= 256, N <= 128 with K >= 8 max(M, N)), qgemm/qgemm_f32 run ONE kernel that reads
 * op(A)/op(B) in place (no pack, no workspace);
 * qgemm_workspace_bytes() then returns 0 and `workspace` may be NULL.  The
 * path is a pure function of (transA, M, N, K), the precision and the path
 * policy below, so qgemm_workspace_bytes() with the same arguments sizes it.
 */
#ifndef QGEMM_B200_H
#define QGEMM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* FP64: computes in double on the FP64 tensor pipe (DMMA). */
int qgemm(char transA, char transB, int64_t M, int64_t N, int64_t K,
          const double alpha[4], const double *A, int64_t lda,
          const double *B, int64_t ldb, const double beta[4],
          double *C, int64_t ldc,
          void *workspace, size_t workspace_bytes, void *stream);

/* FP32: same contract with float storage.  Arithmetic: 3xTF32 on the tcgen05
 * tensor cores with FP32 accumulation (hi/lo split of both operands), which
 * meets the FP32 tolerance where 1xTF32 does not; the small-
 * problem path below computes in FP64 and rounds once on store.
 * Environment (read once per process): QG_TC2_L2_PERSIST=1 launches the FP32
 * mainloop under a persisting-L2 access-policy window over its running-sum
 * scratch and raises cudaLimitPersistingL2CacheSize on the device once
 * (device-wide state, hence opt-in); results are identical. */
int qgemm_f32(char transA, char transB, int64_t M, int64_t N, int64_t K,
              const float alpha[4], const float *A, int64_t lda,
              const float *B, int64_t ldb, const float beta[4],
              float *C, int64_t ldc,
              void *workspace, size_t workspace_bytes, void *stream);

/* Workspace bytes for a single-panel call (dtype 0 = FP64, 1 = FP32).
 * Returns 0 for quick-return shapes and for invalid arguments. */
size_t qgemm_workspace_bytes(char transA, char transB, int64_t M, int64_t N, int64_t K, int dtype);

/* Smallest accepted workspace (one K-panel), same arguments. */
size_t qgemm_workspace_min_bytes(char transA, char transB, int64_t M, int64_t N, int64_t K, int dtype);

/* End-to-end call on HOST-resident operands (the call a user with host data
 * makes).  Same arguments, semantics, quick returns and error codes as
 * qgemm()/qgemm_f32(), except:
 *   A, B, C   may be host memory (pinned -- cudaHostAlloc / cudaHostRegister --
 *             for the transfers to overlap compute; pageable memory is correct
 *             but serialises) or device memory: every access is a
 *             cudaMemcpy2DAsync with cudaMemcpyDefault;
 *   workspace DEVICE memory of at least qgemm_host_workspace_bytes() bytes,
 *             256-byte aligned; it holds the device accumulator of C, a device
 *             copy of the caller's C, and double-buffered staging and packed
 *             chunks of op(A)/op(B).
 * The call streams K in chunks (Alg. 2's kappa loop) host->device
 * on a private upload stream while `stream` packs and multiplies the previous
 * chunk.  The accumulator starts from beta = 0, the caller's C is uploaded
 * behind the first chunks and folded in (C += beta (x) C_old) before the last
 * chunk, which runs per column panel so each finished panel downloads while
 * the next computes.  It returns
 * after enqueueing; the result is in the caller's C once `stream` has
 * synchronised (host buffers must stay valid until then).  The library creates
 * two streams and a few events per call and releases them once their work
 * completes.  A positive return (cudaError_t) can leave part of the work
 * enqueued. */
int qgemm_host(char transA, char transB, int64_t M, int64_t N, int64_t K,
               const double alpha[4], const double *A, int64_t lda,
               const double *B, int64_t ldb, const double beta[4],
               double *C, int64_t ldc,
               void *workspace, size_t workspace_bytes, void *stream);
int qgemm_host_f32(char transA, char transB, int64_t M, int64_t N, int64_t K,
                   const float alpha[4], const float *A, int64_t lda,
                   const float *B, int64_t ldb, const float beta[4],
                   float *C, int64_t ldc,
                   void *workspace, size_t workspace_bytes, void *stream);

/* Device workspace bytes of qgemm_host (dtype 0) / qgemm_host_f32 (dtype 1);
 * 0 for invalid op characters or M, N <= 0. */
size_t qgemm_host_workspace_bytes(char transA, char transB, int64_t M, int64_t N, int64_t K, int dtype);

/* Quaternion Hermitian rank-K update (the paper
 * names rank-k updates as a reuse target of its GEMM kernels, and
 * defines quaternion hermiticity Q = Q^H at P:483-492):
 *     trans = 'N':        C <- alpha * A * A^H + beta * C,   A is N x K (lda >= max(1,N))
 *     trans = 'H' or 'C': C <- alpha * A^H * A + beta * C,   A is K x N (lda >= max(1,K))
 * alpha, beta REAL (so a Hermitian C stays Hermitian).  Only the `uplo`
 * triangle of C ('L' lower or 'U' upper, diagonal included) is read and
 * written; the other triangle is never touched.  The vector part of every
 * diagonal entry is set to 0 on output (the diagonal of a Hermitian matrix is
 * real; R18).  Tiles of the other triangle are not computed: about
 * half the flops of the equivalent qgemm(N, H).
 * Storage, ownership, asynchrony, workspace and K-panel behaviour as qgemm.
 * Quick returns: N == 0, or (alpha == 0 or K == 0) with beta == 1.
 * Errors: uplo=-1 trans=-2 N=-3 K=-4 A=-6 lda=-7 C=-9 (also: C overlaps A)
 * ldc=-10 workspace=-11 workspace_bytes=-12; >0 cudaError_t. */
int qherk(char uplo, char trans, int64_t N, int64_t K, double alpha, const double *A, int64_t lda,
          double beta, double *C, int64_t ldc, void *workspace, size_t workspace_bytes, void *stream);

/* Workspace bytes for a single-panel qherk call (0 for invalid/quick-return shapes). */
size_t qherk_workspace_bytes(char uplo, char trans, int64_t N, int64_t K);

/* Peer memory (multi-GPU driver).  The
 * row-sharded QGEMM fuses its collection step into the epilogue: each rank
 * passes root's C, mapped into its own address space, as the `C` argument of
 * qgemm() (row offset r0, ldc = root's leading dimension), so finished tiles
 * are stored over NVLink / NVSwitch while the rest of the mainloop runs.
 *
 * qgemm_ipc_handle: CUDA IPC handle (64 bytes, written to `handle`) of the
 *   device allocation containing `dptr`, and the byte offset of `dptr` inside
 *   it (*offset; *alloc_bytes = allocation size if non-NULL).  Works for
 *   interior pointers of caching allocators.  Returns 0, -1 (dptr NULL),
 *   -2 (handle NULL), -3 (offset NULL), or a cudaError_t.
 * qgemm_ipc_open: map a handle from another process of this node into this
 *   process (cudaIpcMemLazyEnablePeerAccess); *dptr = mapped base + offset,
 *   *base = the mapping to pass to qgemm_ipc_close.  Returns 0, -1/-3/-4 for
 *   NULL arguments, or a cudaError_t (e.g. opening in the exporting process).
 * qgemm_ipc_close: unmap a base returned by qgemm_ipc_open. */
int qgemm_ipc_handle(const void *dptr, unsigned char handle[64], uint64_t *offset, uint64_t *alloc_bytes);
int qgemm_ipc_open(const unsigned char handle[64], uint64_t offset, void **dptr, void **base);
int qgemm_ipc_close(void *base);

/* Debug/cross-check path: one thread per output quaternion, reads op(A) and
 * op(B) in place (no pack, no workspace).  Same arguments, errors and
 * semantics as qgemm() minus the workspace.  Not used by qgemm(). */
int qgemm_naive(char transA, char transB, int64_t M, int64_t N, int64_t K,
                const double alpha[4], const double *A, int64_t lda,
                const double *B, int64_t ldb, const double beta[4],
                double *C, int64_t ldc, void *stream);

/* Pack A / pack B alone (test hook for SURVEY.md §8(a) rows a2/a3; the packed
 * path of qgemm() runs the same kernel, Alg. 4 PACK1 / Alg. 5 PACK2,
 * P:1164-1202).  Packs the R x K panel X~ of op(X) into FP64 chunks:
 *   operand 0 (A): X~(r, k) = op(X)(r, k), op(X) is R x K (X stored R x K for
 *                  trans 'N', K x R for 'T'/'H');
 *   operand 1 (B): X~(r, k) = op(X)(k, r), op(X) is K x R (X stored K x R for
 *                  'N', R x K for 'T'/'H');
 * trans 'H' (alias 'C') conjugates (components 1..3 negated).
 * out: ceil(R/64) * ceil(K/16) chunks of 64 x 16 quaternions, chunk index
 * rt * ceil(K/16) + kt; inside a chunk, component c of X~(64 rt + r, 16 kt + k)
 * is the double at offset ((((k/4)*8 + r/8)*2 + c/2)*32 + 4(r%8) + k%4)*2 + c%2
 * (the DMMA m8n8k4 fragment order); rows r >= R and k >= K are 0 (Alg. 2
 * padding).  Device pointers X (16-byte aligned) and out; enqueued
 * on `stream`.  Errors: trans=-1 operand=-2 R=-3 K=-4 X=-5 ldx=-6 out=-7
 * out_bytes=-8 (too small); >0 cudaError_t.  R == 0 or K == 0: no-op. */
int qgemm_pack_panel(char trans, int operand, int64_t R, int64_t K, const double *X, int64_t ldx,
                     double *out, size_t out_bytes, void *stream);

/* Path policy (process-wide): 0 = auto (default), 1 = always the packed
 * path (pack launch + persistent mainloop), 2 = always the one-launch small
 * kernel, 3 = direct (FP64: the persistent mainloop fed by TMA straight from
 * the interleaved storage -- one launch, no pack, workspace = stream-K scratch
 * only; FP32: the tcgen05 pair kernel fed with raw tiles by TMA and split into
 * tf32 hi/lo planes in shared memory -- no pack launch, workspace = the
 * accumulation-chunk slots and split-K partials), 4 = direct restricted to the
 * 32-byte-swizzle tile feed (3 and auto load both operands as conflict-free
 * 4-quaternion-group tiles when the groups are whole: M, resp. N, a multiple
 * of 4 for op(A) = A, resp. op(B) = B^T / B^H, else K), 5 = as 2 but never the
 * tile-exact variant of the small kernel (taken when M % 8 == N % 8 == K % 4
 * == 0 and, for FP64, A, B, C are 32-byte aligned).  Auto = small kernel below the
 * crossover; above it FP64 takes the direct path whenever the group tiles
 * apply (op(A) = A: M % 4 == 0 and N % 4 (op(B) = B^T/B^H) resp. K % 4 == 0),
 * when op(A) is T/H, and otherwise up to M*N*K <= 2^37; else packed; FP32
 * packed (pack launch + the tcgen05 pair kernel, split over K below one wave:
 * faster than the direct feed, whose in-SM split saturates shared memory;
 * DESIGN.md §6).  FP32 on the tensor cores accumulates K in chunks of 256
 * added with round-to-nearest (the tensor core's own accumulation truncates).
 * Returns the previous policy, or -1 (policy unchanged) for other values.
 * For tests and benchmarks; the result is correct under every policy. */
int qgemm_set_path_policy(int policy);

/* Number of kernels the last successful call on this host thread enqueued
 * (for the bench's gpu_launches count). */
int qgemm_last_launch_count(void);

/* Instrumentation (off by default).  While enabled, every kernel this host
 * thread enqueues is bracketed by two CUDA events recorded on the same stream.
 * qgemm_timing_collect() synchronises on those events, writes the summed
 * milliseconds and launch counts per kernel kind into ms[5] / counts[5]
 * (0 = pack, 1 = mainloop (DMMA or FP32), 2 = beta-scale, 3 = naive,
 * 4 = small-problem kernel), clears the record and returns 0 (or a
 * cudaError_t).  Host arrays of 5 entries, caller-owned. */
void qgemm_timing_enable(int on);
int qgemm_timing_collect(double ms[5], int counts[5]);

/* Library version string. */
const char *qgemm_version(void);

#ifdef __cplusplus
}
#endif

#endif /* QGEMM_B200_H */
