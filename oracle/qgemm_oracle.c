/*
 * oracle/qgemm_oracle.c -- CPU correctness oracle for quaternion GEMM.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_1903_05575_b200/) never imports, links or calls it,
 * and this file shares no code, header, table or constant with the CUDA path.
 *
 * What it computes (PAPER.md = arXiv 1903.05575, LaTeX source):
 *   C <- alpha * op(A) * op(B) + beta * C                       Eq. general_gemm
 * over the Hamilton quaternions, with
 *   - the Hamilton product written exactly as Eq. quaternion_prod,
 *     the Levi-Civita tensor of Eq. quaternion_alg;
 *   - conjugate of Eq. quaternion_conj;
 *   - op(X) in {X, X^T, X^H}, (X^H)_{mu nu} = conj(X_{nu mu});
 *   - scalar products taken from the LEFT: (qPQ)_{mu nu} = q sum_k P Q,
 *     so alpha and beta multiply from the left (reading R2);
 *   - column-major storage with leading dimension in quaternions,
 *     quaternion components interleaved [q0;q1;q2;q3];
 *   - the loop order of Alg. 1, the reference GEMM: columns nu of C,
 *     then kappa over K, then an axpy over the rows of the column.
 *
 * Departures from Alg. 1, all allowed by the plain definition:
 *   - the sum T = op(A) op(B) is accumulated from zero and alpha, beta are applied
 *     once at the end (C = alpha*T + beta*C), i.e. alpha applied once to the sum
 *     (reading R9); beta == 0 means C is overwritten and never read (reading R3);
 *   - op(A), op(B) are materialised as explicit host copies before the loop so the
 *     loop body is identical for all nine (opA, opB) pairs;
 *   - columns of C are distributed over OpenMP threads; every column is computed
 *     by exactly one thread in the same order, so the result is independent of
 *     the thread count.
 *
 * Everything is FP64, compiled with -O3 -fno-fast-math -ffp-contract=off (IEEE
 * semantics, no reassociation, no FMA contraction).
 *
 * Parity pins: see tests/test_oracle_pins.py (basis table, worked product, norm,
 * associativity, (AB)^H = B^H A^H, chi-embedding vs numpy complex GEMM, complex and
 * real sub-algebras, closed forms).  oracle_qgemm_entries() (sampled entries) is
 * pinned by equality with oracle_qgemm on small sizes.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* Levi-Civita symbol eps_{ij}^k for i,j,k in {1,2,3} (Eq. quaternion_alg). */
static inline int levi_civita(int i, int j, int k) {
  if (i == j || j == k || i == k) return 0;
  /* even permutations of (1,2,3): (1,2,3), (2,3,1), (3,1,2) */
  if ((i == 1 && j == 2 && k == 3) || (i == 2 && j == 3 && k == 1) ||
      (i == 3 && j == 1 && k == 2))
    return 1;
  return -1;
}

/* Hamilton product pq, Eq. quaternion_prod:
 *   pq = (p^0 q^0 - sum_i p^i q^i) e0
 *      + sum_k (p^0 q^k + p^k q^0 + sum_{i,j} eps_{ij}^k p^i q^j) e_k            */
void oracle_hmul(const double *p, const double *q, double *out) {
  double r0 = p[0] * q[0];
  for (int i = 1; i <= 3; ++i) r0 -= p[i] * q[i];
  double r[4];
  r[0] = r0;
  for (int k = 1; k <= 3; ++k) {
    double v = p[0] * q[k] + p[k] * q[0];
    for (int i = 1; i <= 3; ++i)
      for (int j = 1; j <= 3; ++j) {
        int e = levi_civita(i, j, k);
        if (e != 0) v += (double)e * p[i] * q[j];
      }
    r[k] = v;
  }
  out[0] = r[0]; out[1] = r[1]; out[2] = r[2]; out[3] = r[3];
}

/* Conjugate, Eq. quaternion_conj. */
void oracle_hconj(const double *q, double *out) {
  out[0] = q[0]; out[1] = -q[1]; out[2] = -q[2]; out[3] = -q[3];
}

static int op_code(char t) {
  switch (t) {
    case 'N': case 'n': return 0;
    case 'T': case 't': return 1;
    case 'H': case 'h': case 'C': case 'c': return 2;
    default: return -1;
  }
}

/* Materialise op(X) (rows x cols, column-major, ld = rows) from stored X.
 * For op N stored X is rows x cols; for T/H stored X is cols x rows. */
static double *materialise_op(int op, int64_t rows, int64_t cols, const double *X, int64_t ldx) {
  double *Y = (double *)malloc(sizeof(double) * 4 * (size_t)(rows > 0 ? rows : 1) * (size_t)(cols > 0 ? cols : 1));
  if (!Y) return NULL;
  for (int64_t c = 0; c < cols; ++c)
    for (int64_t r = 0; r < rows; ++r) {
      const double *src = (op == 0) ? X + 4 * (r + c * ldx) : X + 4 * (c + r * ldx);
      double *dst = Y + 4 * (r + c * rows);
      if (op == 2) oracle_hconj(src, dst);
      else memcpy(dst, src, 4 * sizeof(double));
    }
  return Y;
}

static int is_zero_q(const double *q) { return q[0] == 0.0 && q[1] == 0.0 && q[2] == 0.0 && q[3] == 0.0; }

/* Finish one entry: C_ij <- alpha*T_ij + beta*C_ij (left products). */
static void finish_entry(const double *alpha, const double *t, const double *beta, double *c) {
  double at[4];
  oracle_hmul(alpha, t, at);
  if (is_zero_q(beta)) {           /* reading R3: beta == 0 -> C not read */
    c[0] = at[0]; c[1] = at[1]; c[2] = at[2]; c[3] = at[3];
  } else {
    double bc[4];
    oracle_hmul(beta, c, bc);
    c[0] = at[0] + bc[0]; c[1] = at[1] + bc[1]; c[2] = at[2] + bc[2]; c[3] = at[3] + bc[3];
  }
}

/* Full GEMM.  Returns 0 on success, -1/-2 for bad op characters, -3..-5 for
 * negative sizes, -20 on allocation failure.  No other validation: the oracle
 * is called only by tests with well-formed arguments. */
int oracle_qgemm(char transA, char transB, int64_t M, int64_t N, int64_t K,
                 const double *alpha, const double *A, int64_t lda,
                 const double *B, int64_t ldb, const double *beta,
                 double *C, int64_t ldc, int nthreads) {
  int oa = op_code(transA), ob = op_code(transB);
  if (oa < 0) return -1;
  if (ob < 0) return -2;
  if (M < 0) return -3;
  if (N < 0) return -4;
  if (K < 0) return -5;
  if (M == 0 || N == 0) return 0;
  double *opA = NULL, *opB = NULL;
  if (K > 0) {
    opA = materialise_op(oa, M, K, A, lda);   /* op(A): M x K, ld = M */
    opB = materialise_op(ob, K, N, B, ldb);   /* op(B): K x N, ld = K */
    if (!opA || !opB) { free(opA); free(opB); return -20; }
  }
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#else
  (void)nthreads;
#endif
  int fail = 0;
#pragma omp parallel
  {
    double *T = (double *)malloc(sizeof(double) * 4 * (size_t)M);
    if (!T) {
#pragma omp atomic write
      fail = 1;
    }
#pragma omp for schedule(dynamic, 1)
    for (int64_t nu = 0; nu < N; ++nu) {          /* Alg. 1: for nu = 1:N */
      if (!T) continue;
      for (int64_t i = 0; i < 4 * M; ++i) T[i] = 0.0;
      for (int64_t ka = 0; ka < K; ++ka) {        /* for kappa = 1:K */
        const double *b = opB + 4 * (ka + nu * K); /* B_{kappa nu} */
        const double *acol = opA + 4 * (ka * M);   /* A(:, kappa) */
        for (int64_t mu = 0; mu < M; ++mu) {      /* column axpy: T(:,nu) += A(:,kappa) B_{kappa nu} */
          double prod[4];
          oracle_hmul(acol + 4 * mu, b, prod);
          T[4 * mu + 0] += prod[0];
          T[4 * mu + 1] += prod[1];
          T[4 * mu + 2] += prod[2];
          T[4 * mu + 3] += prod[3];
        }
      }
      for (int64_t mu = 0; mu < M; ++mu)
        finish_entry(alpha, T + 4 * mu, beta, C + 4 * (mu + nu * ldc));
    }
    free(T);
  }
  free(opA);
  free(opB);
  return fail ? -20 : 0;
}

/* Sampled entries: for each (rows[s], cols[s]) compute
 *   out[s] = alpha * sum_k op(A)_{i k} op(B)_{k j} + beta * C0_{ij}
 * without materialising anything (direct index into stored A, B).  C0 is the
 * pre-call C (may be NULL when beta == 0).  Used for the parity check at
 * BASELINE.json's full sizes, where the full oracle is too slow. */
int oracle_qgemm_entries(char transA, char transB, int64_t M, int64_t N, int64_t K,
                         const double *alpha, const double *A, int64_t lda,
                         const double *B, int64_t ldb, const double *beta,
                         const double *C0, int64_t ldc,
                         int64_t nsamples, const int64_t *rows, const int64_t *cols,
                         double *out, int nthreads) {
  int oa = op_code(transA), ob = op_code(transB);
  if (oa < 0) return -1;
  if (ob < 0) return -2;
  if (M < 0 || N < 0 || K < 0) return -3;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#else
  (void)nthreads;
#endif
  int bad = 0;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t s = 0; s < nsamples; ++s) {
    int64_t i = rows[s], j = cols[s];
    if (i < 0 || i >= M || j < 0 || j >= N) {
#pragma omp atomic write
      bad = 1;
      continue;
    }
    double t[4] = {0.0, 0.0, 0.0, 0.0};
    for (int64_t k = 0; k < K; ++k) {
      double a[4], b[4], p[4];
      const double *as = (oa == 0) ? A + 4 * (i + k * lda) : A + 4 * (k + i * lda);
      const double *bs = (ob == 0) ? B + 4 * (k + j * ldb) : B + 4 * (j + k * ldb);
      if (oa == 2) oracle_hconj(as, a); else memcpy(a, as, sizeof a);
      if (ob == 2) oracle_hconj(bs, b); else memcpy(b, bs, sizeof b);
      oracle_hmul(a, b, p);
      t[0] += p[0]; t[1] += p[1]; t[2] += p[2]; t[3] += p[3];
    }
    double c[4] = {0.0, 0.0, 0.0, 0.0};
    if (!is_zero_q(beta)) memcpy(c, C0 + 4 * (i + j * ldc), sizeof c);
    finish_entry(alpha, t, beta, c);
    memcpy(out + 4 * s, c, sizeof c);
  }
  return bad ? -14 : 0;
}

/* Quaternion matrix-vector product y = op(X) x (x, y column vectors of
 * quaternions, x multiplied from the RIGHT), used by the Freivalds check of
 * tests (P11): C x  vs  alpha (op(A) (op(B) x)) + beta (C0 x), valid over H by
 * associativity. */
int oracle_qgemv(char trans, int64_t rows, int64_t cols, const double *X, int64_t ldx,
                 const double *x, double *y, int nthreads) {
  int o = op_code(trans);
  if (o < 0) return -1;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#else
  (void)nthreads;
#endif
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < rows; ++r) {
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int64_t c = 0; c < cols; ++c) {
      double a[4], p[4];
      const double *s = (o == 0) ? X + 4 * (r + c * ldx) : X + 4 * (c + r * ldx);
      if (o == 2) oracle_hconj(s, a); else memcpy(a, s, sizeof a);
      oracle_hmul(a, x + 4 * c, p);
      acc[0] += p[0]; acc[1] += p[1]; acc[2] += p[2]; acc[3] += p[3];
    }
    memcpy(y + 4 * r, acc, sizeof acc);
  }
  return 0;
}

int oracle_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
