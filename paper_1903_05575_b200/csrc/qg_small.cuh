// qg_small.cuh -- one-launch QGEMM for small problems (SURVEY.md §8(f) NEXT 4:
// "fuse the pack into the mainloop ... to drop the extra launches at small N").
//
// The packed path (pack A + pack B + persistent 64x64 DMMA mainloop) costs three
// launches and, below ~ one wave of 64x64 tiles, runs on a handful of SMs: at
// c1 (64^3) one tile exists and the mainloop's split-K still reaches only two
// SMs.  This kernel reads op(A) and op(B) IN PLACE (interleaved, column-major,
// any of N/T/H) and spreads the work over 8x8-quaternion warp tiles with an
// intra-CTA split over K, so a 64^3 problem occupies 64 SMs in one launch.
//
// Arithmetic: the same 16-product rule as the packed mainloop
// (D^{p XOR s} += eps(p,s) A^p B^s, Eq. quaternion_prod) on the FP64
// tensor pipe (mma.sync.m8n8k4.f64 -> DMMA.8x8x4).  The m8n8k4 fragments are
// whole quaternions: lane l holds A(m0 + l/4, k0 + l%4) and B(k0 + l%4, n0 + l/4),
// so ONE 32-byte load per operand per lane gives the fragments of all four
// components (no shared-memory de-interleave is needed).  op = H conjugates the
// loaded quaternion; op = T only swaps the index roles.
//
// FP32 storage: quaternions are widened to double on load and the FP64 result
// is rounded once on store -- more accurate than the FP32 tolerance requires.
//
// CTA = W = QG_SMALL_WARPS warps.  With split factor S in {1, 2, .., W} (host: as
// large as keeps the grid within one wave of resident CTAs), warp w computes the
// 8x8 tile (w / S) of the CTA's (W/S) M-stacked tiles over the (w % S)-th of S equal
// ranges of k4 steps; partials are summed in a fixed order through shared
// memory (deterministic), then lane l applies the alpha/beta epilogue (left
// products) to the two quaternions it owns: C(m0 + l/4, n0 + 2(l%4) + i).
#pragma once
#include "qg_common.cuh"

namespace qg {

#ifndef QG_SMALL_WARPS
#define QG_SMALL_WARPS 4
#endif
constexpr int kSmallWarps = QG_SMALL_WARPS;
constexpr int kSmallThreads = kSmallWarps * 32;
constexpr int kSmallUnroll = 4;  // k4 steps whose loads are issued together

struct SmallArgs {
  const void *A, *B;
  void *C;
  int64_t lda, ldb, ldc, M, N, K;
  int a_rc, a_cj, b_rc, b_cj;  // operand views of load_rk (from opA, opB)
  int S;                       // warps per 8x8 tile splitting K
  int Z;                       // CTAs per 8x8 tile splitting K (a thread-block cluster; S == W when > 1)
  int64_t m_blocks;            // CTAs along M (1-D grid: m fastest)
  Scalars<double> sc;
  int pdl_trigger;             // tiny kernel, launched with PDL: 1 = let the next kernel launch at
                               // entry, 2 = after this CTA's stores (0: no PDL attribute)
  int64_t per;                 // tiny kernel: k4 steps per warp (ceil(K / 4 / S))
};

template <typename T>
__device__ __forceinline__ void ld_quat_d(const T *p, double (&q)[4]) {
  T t[4];
  ldq(p, t);
#pragma unroll
  for (int c = 0; c < 4; ++c) q[c] = double(t[c]);
}

// Quaternion (r, k) of an operand viewed as R x K: rows_contig -> X(r, k) at
// X + 4(r + k ldx), else X(k, r) at X + 4(k + r ldx); conj flips q^1..q^3.
// Out of range -> 0 (the zero padding of Alg. 2).
//   A: op(A)(m, k) = A(m, k) [N] | A(k, m) [T] | conj A(k, m) [H]
//   B: op(B)(k, n) = B(k, n) [N] | B(n, k) [T] | conj B(n, k) [H]  (r = n)
template <typename T>
__device__ __forceinline__ void load_rk(const T *X, int64_t ldx, int rows_contig, int conj, int64_t r,
                                        int64_t k, int64_t R, int64_t K, double (&q)[4]) {
  if (r < R && k < K) {
    ld_quat_d(rows_contig ? X + 4 * (r + k * ldx) : X + 4 * (k + r * ldx), q);
    if (conj) { q[1] = -q[1]; q[2] = -q[2]; q[3] = -q[3]; }
  } else {
    q[0] = q[1] = q[2] = q[3] = 0.0;
  }
}

// The same element in two halves, so that every load of an unrolled group is
// issued before any is consumed (a load inside a range branch followed by its
// conj fix-up serialised the round trips: ncu long-scoreboard stalls on the
// fix-ups, ~4x the DMMA time at c1): rk_addr clamps an out-of-range (r, k) to
// the base pointer (a valid address; the value is discarded), rk_fix zeroes or
// conjugates after all loads are in flight.
template <typename T>
__device__ __forceinline__ const T *rk_addr(const T *X, int64_t ldx, int rows_contig, int64_t r, int64_t k,
                                            int64_t R, int64_t K, bool &ok) {
  ok = r < R && k < K;
  return ok ? (rows_contig ? X + 4 * (r + k * ldx) : X + 4 * (k + r * ldx)) : X;
}
__device__ __forceinline__ void rk_fix(bool ok, int conj, double (&q)[4]) {
  const double s = conj ? -1.0 : 1.0;
  q[0] = ok ? q[0] : 0.0;
#pragma unroll
  for (int c = 1; c < 4; ++c) q[c] = ok ? s * q[c] : 0.0;
}

// One k4 step of the 8x8 warp tile: 16 DMMA.8x8x4, acc^{p^s} += eps(p,s) A^p B^s.
__device__ __forceinline__ void small_step(double (&acc)[4][2], const double (&qa)[4], const double (&qb)[4]) {
  double nb[4];
#pragma unroll
  for (int s = 0; s < 4; ++s) nb[s] = -qb[s];
#pragma unroll
  for (int p = 0; p < 4; ++p)
#pragma unroll
    for (int s = 0; s < 4; ++s) dmma_8x8x4(acc[p ^ s], qa[p], hneg(p, s) ? nb[s] : qb[s]);
}

constexpr int kSmallMaxCluster = 8;

__device__ __forceinline__ void cluster_arrive_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void cluster_arrive_release() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory"); }
// Store a double into CTA `rank`'s shared memory at the address of `p` in this CTA.
__device__ __forceinline__ void st_dsmem(const double *p, uint32_t rank, double v) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(remote) : "r"(smem_u32(p)), "r"(rank));
  asm volatile("st.shared::cluster.f64 [%0], %1;\n" ::"r"(remote), "d"(v) : "memory");
}

// Z > 1 (host: only when S == W, i.e. one 8x8 tile per CTA, for long K): the Z
// CTAs of a thread-block cluster split the tile's k4 steps; ranks 1..Z-1 store
// their CTA-reduced partial into rank 0's shared memory (DSMEM), rank 0 adds
// them in rank order (deterministic) and runs the epilogue.
// (kZ: a separate instantiation, so the Z = 1 kernel carries none of it.)
template <typename T, bool kZ>
// (<= 128 registers: 4 CTAs per SM -- occupancy, not ILP, sets its speed; measured)
__global__ void __launch_bounds__(kSmallThreads, 512 / kSmallThreads) qgemm_small_kernel(SmallArgs a) {
  __shared__ double red[kSmallThreads / 32][8][32];  // [warp][component, e][lane]: conflict-free
  __shared__ double zred[kZ ? kSmallMaxCluster - 1 : 1][8][32];
  const T *A = static_cast<const T *>(a.A);
  const T *B = static_cast<const T *>(a.B);
  T *C = static_cast<T *>(a.C);
  // Programmatic dependent launch (host: QG_SMALL_PDL): let the next kernel of
  // the stream start launching now, so its CTA dispatch and prologue overlap
  // this grid; and wait for the previous kernel's completion (and memory) only
  // here, right before the first global access.  Without the launch attribute
  // both are no-ops.
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = a.S, tiles_per_cta = kSmallWarps / S, Z = kZ ? a.Z : 1;
  const int tile = warp / S, part = warp % S;
  const uint32_t z = kZ ? cluster_rank() : 0u;
  if constexpr (kZ) cluster_arrive_relaxed();  // (waited on before the first DSMEM store)
  const int64_t cta = int64_t(blockIdx.x) / Z;
  const int64_t mb = cta % a.m_blocks, nb = cta / a.m_blocks;
  const int64_t m0 = (mb * tiles_per_cta + tile) * 8;
  const int64_t n0 = nb * 8;
  const int lr = lane >> 2, lk = lane & 3;

  // this warp's k4 steps: rank z's share of the tile, then part `part` of it
  const int64_t steps_all = (a.K + 3) / 4;
  const int64_t perz = (steps_all + Z - 1) / Z;
  const int64_t z0 = min(steps_all, int64_t(z) * perz), z1 = min(steps_all, z0 + perz);
  const int64_t per = (z1 - z0 + S - 1) / S;
  const int64_t s0 = min(z1, z0 + int64_t(part) * per), s1 = min(z1, s0 + per);

  // C is independent of the k loop: the epilogue warps prefetch their two
  // quaternions into L1 first, so the C read latency overlaps the mainloop
  // (a prefetch, not a load: no registers held across the loop)
  if (part == 0 && z == 0 && !a.sc.beta_zero && m0 + lr < a.M) {
#pragma unroll
    for (int i = 0; i < 2; ++i)
      if (n0 + 2 * lk + i < a.N)
        asm volatile("prefetch.global.L1 [%0];" ::"l"(C + 4 * (m0 + lr + (n0 + 2 * lk + i) * a.ldc)));
  }

  double acc[4][2];
#pragma unroll
  for (int c = 0; c < 4; ++c) acc[c][0] = acc[c][1] = 0.0;

  if (m0 < a.M) {
    int64_t st = s0;
    for (; st + kSmallUnroll <= s1; st += kSmallUnroll) {  // loads of 4 steps in flight
      double qa[kSmallUnroll][4], qb[kSmallUnroll][4];
      bool oka[kSmallUnroll], okb[kSmallUnroll];
#pragma unroll
      for (int u = 0; u < kSmallUnroll; ++u) {
        const int64_t k = (st + u) * 4 + lk;
        ld_quat_d(rk_addr(A, a.lda, a.a_rc, m0 + lr, k, a.M, a.K, oka[u]), qa[u]);
        ld_quat_d(rk_addr(B, a.ldb, a.b_rc, n0 + lr, k, a.N, a.K, okb[u]), qb[u]);
      }
#pragma unroll
      for (int u = 0; u < kSmallUnroll; ++u) {
        rk_fix(oka[u], a.a_cj, qa[u]);
        rk_fix(okb[u], a.b_cj, qb[u]);
      }
#pragma unroll
      for (int u = 0; u < kSmallUnroll; ++u) small_step(acc, qa[u], qb[u]);
    }
    for (; st < s1; ++st) {  // tail: one step at a time (no DMMAs on zero fill)
      double qa[4], qb[4];
      load_rk(A, a.lda, a.a_rc, a.a_cj, m0 + lr, st * 4 + lk, a.M, a.K, qa);
      load_rk(B, a.ldb, a.b_rc, a.b_cj, n0 + lr, st * 4 + lk, a.N, a.K, qb);
      small_step(acc, qa, qb);
    }
  }

  // fixed-order reduction of the S partial tiles (deterministic)
  if (S > 1) {
    if (part != 0) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        red[warp][2 * c][lane] = acc[c][0];
        red[warp][2 * c + 1][lane] = acc[c][1];
      }
    }
    __syncthreads();
    if (part == 0)
      for (int w = 1; w < S; ++w)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          acc[c][0] += red[warp + w][2 * c][lane];
          acc[c][1] += red[warp + w][2 * c + 1][lane];
        }
  }
  // then across the cluster (every thread takes part in the cluster barriers)
  if constexpr (kZ) {
    cluster_wait();  // every CTA of the cluster is running: DSMEM is live
    if (z > 0 && part == 0)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        st_dsmem(&zred[z - 1][2 * c][lane], 0, acc[c][0]);
        st_dsmem(&zred[z - 1][2 * c + 1][lane], 0, acc[c][1]);
      }
    cluster_arrive_release();
    cluster_wait();
    if (z > 0) return;
    if (part == 0)
      for (int r = 0; r < Z - 1; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          acc[c][0] += zred[r][2 * c][lane];
          acc[c][1] += zred[r][2 * c + 1][lane];
        }
  }
  if (part != 0) return;

  const int64_t row = m0 + lr;
  if (row >= a.M) return;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int64_t col = n0 + 2 * lk + i;
    if (col >= a.N) continue;
    T *cp = C + 4 * (row + col * a.ldc);
    double t[4] = {acc[0][i], acc[1][i], acc[2][i], acc[3][i]};
    double out[4];
    left_scale(a.sc.alpha, a.sc.alpha_real, t, out);
    if (!a.sc.beta_zero) {
      T c0[4];
      ldq_c(cp, c0);
      double cd[4] = {double(c0[0]), double(c0[1]), double(c0[2]), double(c0[3])}, bc[4];
      left_scale(a.sc.beta, a.sc.beta_real, cd, bc);
#pragma unroll
      for (int k = 0; k < 4; ++k) out[k] += bc[k];
    }
    T o[4] = {T(out[0]), T(out[1]), T(out[2]), T(out[3])};
    stq(cp, o);
  }
}

// ---------------------------------------------------------------------------
// Tile-exact variant (host: M % 8 == N % 8 == K % 4 == 0, no cluster split;
// c1 and every power-of-two small shape): the same work split and arithmetic as
// qgemm_small_kernel, with everything the general kernel decides per element
// moved to compile time or out of the loop -- the op pair (rows-contiguous /
// conj flags, kOps) is a template parameter, so op H is a sign in the product
// table (eps(p,s) sigma_A(p) sigma_B(s)) instead of a fix-up per loaded
// component; no range checks (every fragment is in range); each operand walks
// one pointer with a fixed per-k4-step stride; FP64 quaternions move as one
// 256-bit access (LDG/STG.E.ENL2.256; 32-byte aligned A, B, C).  ncu at c1 on
// the general kernel: 810 issued instructions per warp for 64 DMMAs, ~6.6
// cycles per issue (fixed-latency "wait" and short-scoreboard stalls) -- the
// instruction stream, not the DMMA pipe, set the time.
// kOps: bit 0 op(A) rows contiguous (A = N), bit 1 conj A (H), bit 2 op(B) rows
// contiguous (B = T/H), bit 3 conj B (H).
__device__ __forceinline__ void ld_quat_wide(const double *p, double (&q)[4]) {
  asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];\n"
               : "=d"(q[0]), "=d"(q[1]), "=d"(q[2]), "=d"(q[3])
               : "l"(p));
}
__device__ __forceinline__ void ld_quat_wide(const float *p, double (&q)[4]) {
  float t[4];
  asm volatile("ld.global.nc.v4.f32 {%0, %1, %2, %3}, [%4];\n"
               : "=f"(t[0]), "=f"(t[1]), "=f"(t[2]), "=f"(t[3])
               : "l"(p));
#pragma unroll
  for (int c = 0; c < 4; ++c) q[c] = double(t[c]);
}
__device__ __forceinline__ void ld_c_wide(const double *p, double (&q)[4]) {
  asm volatile("ld.global.v4.f64 {%0, %1, %2, %3}, [%4];\n"
               : "=d"(q[0]), "=d"(q[1]), "=d"(q[2]), "=d"(q[3])
               : "l"(p)
               : "memory");
}
__device__ __forceinline__ void ld_c_wide(const float *p, double (&q)[4]) {
  float t[4];
  ldq_c(p, t);
#pragma unroll
  for (int c = 0; c < 4; ++c) q[c] = double(t[c]);
}
__device__ __forceinline__ void st_c_wide(double *p, const double (&q)[4]) {
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};\n" ::"l"(p), "d"(q[0]), "d"(q[1]), "d"(q[2]), "d"(q[3])
               : "memory");
}
__device__ __forceinline__ void st_c_wide(float *p, const double (&q)[4]) {
  const float t[4] = {float(q[0]), float(q[1]), float(q[2]), float(q[3])};
  stq(p, t);
}

// One k4 step with the conj signs folded in: acc^{p^s} += eps(p,s) sa(p) sb(s) A^p B^s.
template <bool CA, bool CB>
__device__ __forceinline__ void tiny_step(double (&acc)[4][2], const double (&qa)[4], const double (&qb)[4]) {
  double nb[4];
#pragma unroll
  for (int s = 0; s < 4; ++s) nb[s] = -qb[s];
#pragma unroll
  for (int p = 0; p < 4; ++p)
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const bool neg = hneg(p, s) ^ (CA && p != 0) ^ (CB && s != 0);
      dmma_8x8x4(acc[p ^ s], qa[p], neg ? nb[s] : qb[s]);
    }
}

#ifndef QG_TINY_WARPS
#define QG_TINY_WARPS 4  // warps per CTA of the tile-exact kernel (c1: 2.37 us back to back vs 2.82 with 8)
#endif
#ifndef QG_TINY_DUAL
#define QG_TINY_DUAL 0  // 1: two accumulator sets (even / odd k4 steps), 8 independent DMMA chains per warp
#endif
constexpr int kTinyWarps = QG_TINY_WARPS;
constexpr int kTinyThreads = kTinyWarps * 32;
template <typename T, int kOps>
__global__ void __launch_bounds__(kTinyThreads, (QG_TINY_DUAL ? 384 : 512) / kTinyThreads) qgemm_tiny_kernel(SmallArgs a) {
  constexpr bool a_rc = kOps & 1, a_cj = (kOps >> 1) & 1, b_rc = (kOps >> 2) & 1, b_cj = (kOps >> 3) & 1;
  __shared__ double red[kTinyWarps][8][32];  // [warp][component, e][lane]: conflict-free
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // grid (m blocks, n tiles); S a power of two (host), so no divisions here
  const int S = a.S, lgS = __ffs(S) - 1;
  const int tile = warp >> lgS, part = warp & (S - 1);
  const int64_t m0 = (int64_t(blockIdx.x) * (kTinyWarps >> lgS) + tile) * 8;
  const int64_t n0 = int64_t(blockIdx.y) * 8;
  const int lr = lane >> 2, lk = lane & 3;
  const int64_t steps_all = a.K >> 2;
  // (the last CTA row may hold tiles past M: no loads, no stores, but they take
  // part in the reduction barrier)
  const bool live = m0 < a.M;
  const int64_t s0 = live ? min(steps_all, int64_t(part) * a.per) : 0;
  const int64_t s1 = live ? min(steps_all, s0 + a.per) : 0;
  const T *A = static_cast<const T *>(a.A);
  const T *B = static_cast<const T *>(a.B);
  T *C = static_cast<T *>(a.C);
  // this lane's quaternion of op(A) (row m0 + lr) / op(B) (column n0 + lr) at k = 4 s0 + lk,
  // and the step to the next k4 step
  const int64_t ka = 4 * s0 + lk;
  const T *pa = a_rc ? A + 4 * ((m0 + lr) + ka * a.lda) : A + 4 * (ka + (m0 + lr) * a.lda);
  const T *pb = b_rc ? B + 4 * ((n0 + lr) + ka * a.ldb) : B + 4 * (ka + (n0 + lr) * a.ldb);
  const int64_t da = a_rc ? 16 * a.lda : 16, db = b_rc ? 16 * a.ldb : 16;
  T *cp0 = C + 4 * ((m0 + lr) + (n0 + 2 * lk) * a.ldc);
  // PDL (host QG_SMALL_PDL): the previous kernel's results are visible from here
  if (a.pdl_trigger == 1) asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  if (part == 0 && live && !a.sc.beta_zero) {
    asm volatile("prefetch.global.L1 [%0];" ::"l"(cp0));
    asm volatile("prefetch.global.L1 [%0];" ::"l"(cp0 + 4 * a.ldc));
  }

  double acc[4][2];
#pragma unroll
  for (int c = 0; c < 4; ++c) acc[c][0] = acc[c][1] = 0.0;
#if QG_TINY_DUAL
  double acc2[4][2];
#pragma unroll
  for (int c = 0; c < 4; ++c) acc2[c][0] = acc2[c][1] = 0.0;
#endif
  int64_t st = s0;
  for (; st + kSmallUnroll <= s1; st += kSmallUnroll) {  // loads of 4 steps in flight
    double qa[kSmallUnroll][4], qb[kSmallUnroll][4];
#pragma unroll
    for (int u = 0; u < kSmallUnroll; ++u) {
      ld_quat_wide(pa + u * da, qa[u]);
      ld_quat_wide(pb + u * db, qb[u]);
    }
#pragma unroll
    for (int u = 0; u < kSmallUnroll; ++u) {
#if QG_TINY_DUAL
      if (u & 1) { tiny_step<a_cj, b_cj>(acc2, qa[u], qb[u]); continue; }
#endif
      tiny_step<a_cj, b_cj>(acc, qa[u], qb[u]);
    }
    pa += kSmallUnroll * da;
    pb += kSmallUnroll * db;
  }
#if QG_TINY_DUAL
#pragma unroll
  for (int c = 0; c < 4; ++c) { acc[c][0] += acc2[c][0]; acc[c][1] += acc2[c][1]; }
#endif
  for (; st < s1; ++st) {
    double qa[4], qb[4];
    ld_quat_wide(pa, qa);
    ld_quat_wide(pb, qb);
    tiny_step<a_cj, b_cj>(acc, qa, qb);
    pa += da;
    pb += db;
  }

  if (S > 1) {  // fixed-order reduction of the S partial tiles (deterministic)
    if (part != 0) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        red[warp][2 * c][lane] = acc[c][0];
        red[warp][2 * c + 1][lane] = acc[c][1];
      }
    }
    __syncthreads();
    if (part != 0) return;
    for (int w = 1; w < S; ++w)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        acc[c][0] += red[warp + w][2 * c][lane];
        acc[c][1] += red[warp + w][2 * c + 1][lane];
      }
  }
  if (!live) return;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    T *cp = cp0 + i * 4 * a.ldc;
    const double t[4] = {acc[0][i], acc[1][i], acc[2][i], acc[3][i]};
    double out[4];
    left_scale(a.sc.alpha, a.sc.alpha_real, t, out);
    if (!a.sc.beta_zero) {
      double c0[4], bc[4];
      ld_c_wide(cp, c0);
      left_scale(a.sc.beta, a.sc.beta_real, c0, bc);
#pragma unroll
      for (int k = 0; k < 4; ++k) out[k] += bc[k];
    }
    st_c_wide(cp, out);
  }
  if (a.pdl_trigger == 2) asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}

}  // namespace qg
