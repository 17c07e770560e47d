// qg_common.cuh -- shared device helpers of the B200 QGEMM library (product path).
//
// Quaternion algebra used by every kernel, restated from PAPER.md:
//   basis products e_p e_s (Eq. quaternion_alg) all have the form
//       e_p e_s = eps(p,s) e_{p XOR s},   eps(p,s) in {+1,-1},
//   with eps = -1 exactly for (p,s) in {(1,1),(1,3),(2,1),(2,2),(3,2),(3,3)}
//   (e_i e_i = -e0; e1e3 = -e2; e2e1 = -e3; e3e2 = -e1).  Hence the Hamilton
//   product (Eq. quaternion_prod) is the 16-FMA rule
//       (a b)^{p XOR s} += eps(p,s) a^p b^s,
//   the form every kernel below evaluates (one sign-table lookup, no branches).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace qg {

// bit (4p+s) set <=> eps(p,s) = -1
constexpr unsigned kNegMask = (1u << 5) | (1u << 7) | (1u << 9) | (1u << 10) | (1u << 14) | (1u << 15)
#ifdef QG_NEGATIVE_CONTROL
    // test-suite sensitivity check only: eps(1,2) flipped, so
    // every kernel computes a wrong Hamilton product; never in libqgemm.so
    ^ (1u << 6)
#endif
    ;

__host__ __device__ constexpr bool hneg(int p, int s) { return (kNegMask >> (4 * p + s)) & 1u; }

// out = a (x) b (left factor a), all four components.
template <typename T>
__device__ __forceinline__ void hmul(const T (&a)[4], const T (&b)[4], T (&out)[4]) {
#pragma unroll
  for (int c = 0; c < 4; ++c) out[c] = T(0);
#pragma unroll
  for (int p = 0; p < 4; ++p)
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      if (hneg(p, s)) out[p ^ s] = fma(-a[p], b[s], out[p ^ s]);
      else out[p ^ s] = fma(a[p], b[s], out[p ^ s]);
    }
}

// Scalars of the epilogue (alpha, beta applied from the LEFT).
template <typename T>
struct Scalars {
  T alpha[4];
  T beta[4];
  int alpha_real;  // alpha^1 = alpha^2 = alpha^3 = 0
  int beta_real;
  int beta_zero;   // beta == 0: C is write-only (R3)
};

template <typename T>
__device__ __forceinline__ void left_scale(const T (&s)[4], int s_real, const T (&q)[4], T (&out)[4]) {
  if (s_real) {
#pragma unroll
    for (int c = 0; c < 4; ++c) out[c] = s[0] * q[c];
  } else {
    hmul(s, q, out);
  }
}

// Load / store one interleaved quaternion (32 B for double, 16 B for float);
// base pointers are 16-byte aligned (checked by the planner).
__device__ __forceinline__ void ldq(const double *p, double (&q)[4]) {
  double2 a = __ldg(reinterpret_cast<const double2 *>(p));
  double2 b = __ldg(reinterpret_cast<const double2 *>(p) + 1);
  q[0] = a.x; q[1] = a.y; q[2] = b.x; q[3] = b.y;
}
__device__ __forceinline__ void ldq(const float *p, float (&q)[4]) {
  float4 a = __ldg(reinterpret_cast<const float4 *>(p));
  q[0] = a.x; q[1] = a.y; q[2] = a.z; q[3] = a.w;
}
// C may be read and then written by the same thread: plain (coherent) loads.
__device__ __forceinline__ void ldq_c(const double *p, double (&q)[4]) {
  double2 a = *reinterpret_cast<const double2 *>(p);
  double2 b = *(reinterpret_cast<const double2 *>(p) + 1);
  q[0] = a.x; q[1] = a.y; q[2] = b.x; q[3] = b.y;
}
__device__ __forceinline__ void ldq_c(const float *p, float (&q)[4]) {
  float4 a = *reinterpret_cast<const float4 *>(p);
  q[0] = a.x; q[1] = a.y; q[2] = a.z; q[3] = a.w;
}
__device__ __forceinline__ void stq(double *p, const double (&q)[4]) {
  reinterpret_cast<double2 *>(p)[0] = make_double2(q[0], q[1]);
  reinterpret_cast<double2 *>(p)[1] = make_double2(q[2], q[3]);
}
__device__ __forceinline__ void stq(float *p, const float (&q)[4]) {
  *reinterpret_cast<float4 *>(p) = make_float4(q[0], q[1], q[2], q[3]);
}

// Epilogue of one output quaternion: C_ij <- alpha (x) acc + beta (x) C_ij.
template <typename T>
__device__ __forceinline__ void epilogue_one(const Scalars<T> &sc, const T (&acc)[4], T *cptr) {
  T out[4];
  left_scale(sc.alpha, sc.alpha_real, acc, out);
  if (!sc.beta_zero) {
    T c[4], bc[4];
    ldq_c(cptr, c);
    left_scale(sc.beta, sc.beta_real, c, bc);
#pragma unroll
    for (int k = 0; k < 4; ++k) out[k] += bc[k];
  }
  stq(cptr, out);
}

// ----------------------------------------------------------------------------
// mbarrier + bulk-copy (TMA engine, non-tensor form) helpers, sm_90+/sm_100a.
// ----------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// Rank of this CTA in its thread-block cluster (0 without a cluster launch).
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// 1-D bulk copy global -> shared, completion counted on `bar` (bytes % 16 == 0).
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void dmma_8x8x4(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

}  // namespace qg
