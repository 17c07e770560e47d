// qg_tc32_2cta.cuh -- FP32 (3xTF32) QGEMM on CTA pairs: tcgen05.mma.cta_group::2.
//
// Same method as qg_tc32.cuh (16 real products per quaternion MAC, D^{p XOR s}
// += eps(p,s) A^p B^s, Eq. quaternion_prod; three tf32 MMAs per
// product, A_hi B_hi + A_hi B_lo + A_lo B_hi; eps = -1 as the negate-A bit),
// but a cluster of two CTAs on one TPC computes a 256 x 128 quaternion tile
// with M = 256 MMAs issued by the leader CTA: each CTA holds its own 128 rows
// of A and HALF (64 columns) of B in shared memory, and receives its 128 x 128
// block of the four accumulators in its own TMEM.  Per CTA that halves the B
// bytes staged and read per MMA flop, and the M = 256, N = 128 shape issues at
// the tf32 pipe's full rate (tools/microbench/tf32_peak.cu: 1097 TF vs 1042 TF
// for the 1-CTA M = 128, N = 128 shape).
//
// Operands stream with 2-D TMA over the packed chunk arrays (no swizzle: the
// chunks are byte images of the canonical K-major UMMA layout): both CTAs load
// their own A chunk and B half, completing transaction bytes on the LEADER's
// full barrier (peer bit of the barrier address cleared, .cta_group::2); the
// leader's commits arrive on both CTAs' empty / accumulator barriers
// (.multicast::cluster).  The B chunks are packed with split_halves so each
// CTA's 64-column half is one contiguous 16 KB block.
#pragma once
#include <cuda.h>
#include "qg_tc32.cuh"

namespace qg {

constexpr int kTc2Stages = 4;
#ifndef QG_TC2_GROUP
#define QG_TC2_GROUP 4  // swept 2-16 at c3: 4 reads 38 GB from DRAM (8: 56, 16: 105) and is fastest
#endif
constexpr int kTc2GroupM = QG_TC2_GROUP;  // pair-rows (256 rows each) per raster group
constexpr uint32_t kTc2ABytes = kTcChunkBytes;       // 32 KB: this CTA's 128 rows, 8 planes
constexpr uint32_t kTc2BBytes = kTcChunkBytes / 2;   // 16 KB: this CTA's 64 columns, 8 planes
constexpr int kTc2AFloats = kTcChunkFloats;
constexpr int kTc2BFloats = kTcChunkFloats / 2;
constexpr size_t kTc2SmemBytes = size_t(kTc2Stages) * (kTc2ABytes + kTc2BBytes) + 256 + 1024;  // + barriers
constexpr uint32_t kPeerBitMask = 0xFEFFFFFFu;  // shared::cluster address of the leader's copy
// Direct feed (no pack launch): raw interleaved FP32 tiles by TMA into a raw
// ring, split into the tf32 hi/lo planes by two converter warps per CTA.
constexpr int kTc2DStages = 3;                       // plane stages (the MMA's ring)
constexpr int kTc2RawStages = 3;                     // raw stages
constexpr uint32_t kTc2RawABytes = kTcBM * kTcBK * 16;      // 16 KB: 128 rows x 8 k quaternions
constexpr uint32_t kTc2RawBBytes = kTcBM / 2 * kTcBK * 16;  // 8 KB: 64 columns x 8 k
constexpr size_t kTc2DSmemBytes =
    size_t(kTc2DStages) * (kTc2ABytes + kTc2BBytes) + size_t(kTc2RawStages) * (kTc2RawABytes + kTc2RawBBytes) +
    256 + 1024;
static_assert(kTc2DSmemBytes <= 232448, "direct FP32 pair kernel exceeds 227 KB of shared memory");

struct alignas(64) Tc2Args {
  CUtensorMap tmA;   // packed A viewed as [rows of 256 floats]; a chunk = 32 rows
  CUtensorMap tmB;   // packed B (split halves): a half = 16 rows
  float *C;
  int64_t ldc, M, N, MT2, NT, KT;  // MT2 = 256-row tile pairs
  Scalars<float> sc;
  int S;             // K splits of each pair past `full` (1: the epilogue updates C)
  int64_t full;      // pairs [0, full) of the raster are computed whole, the rest split S ways
  float *part;       // S > 1: raw accumulators of the split pairs, kTc2PartFloats per CTA, summed by tc2_reduce_kernel
  // direct feed: tmA / tmB are 2-D maps of the user's interleaved op(A) / op(B)
  // (rc: rows contiguous -> {4 R floats, K}, boxes of 32 rows x 8 k; else
  // {4 K floats, R}, one box of all rows x 8 k, 128-byte swizzle); cj: op H
  int a_rc, b_rc, a_cj, b_cj;
  int kc;            // k-tiles per TMEM accumulation chunk (promotion, see below)
  float *tmp;        // chunk promotion: one kTc2PartFloats slot per SM id (%smid) ...
  int nslots;        // ... for SM ids < nslots
};
// One CTA's raw partial: 4 components x 128 columns x 128 rows, rows fastest.
constexpr int64_t kTc2PartFloats = 4 * int64_t(kTcBN) * kTcBM;

// ---- Accumulation chunks ("promotion").  The tensor core adds each MMA's
// products into the TMEM accumulator with truncating FP32 arithmetic, so the
// error of one accumulation chain grows like (steps) x |D| ~ K^1.5, faster
// than the north-star tolerance's sqrt(K) (tools/f32_accuracy.py; one 8192-deep
// chain of uniform data errs by ~7 x tol).  A unit's k-tiles are therefore
// accumulated in chunks of kc k-tiles (error ~ sqrt(K / kc) kc^1.5: a constant
// fraction of the tolerance, proportional to kc): after every chunk but the last
// the epilogue warps read TMEM component by component, release each component
// to the MMA issuer at once (it waits per component before the next chunk's
// first MMA into it, so the next chunk overlaps the drain) and add the values
// into their SM's slot with L2 reductions (round-to-nearest FP32; the first
// chunk stores).  The last chunk adds the slot to its TMEM values and folds
// into the target: C <- alpha sum + beta C, or, for a split-K unit, the raw
// partial.  (QG_TC2_RED = 0: every chunk stored to the slot and folded into the
// target behind the next chunk's MMAs -- four times the L2 traffic.)  Each thread only touches its own TMEM lane (row) of the
// slot, so the slot needs no synchronisation beyond program order;
// one CTA per SM (shared memory) makes the %smid-indexed slot private to the
// running CTA (the host sizes the slots by the SM count; a CTA on an SM id past
// it -- ids need not be contiguous -- folds every chunk into the target
// straight from TMEM, holding TMEM during the fold).
#ifndef QG_TC2_RED
// 1: chunks summed in the slot by L2 reductions (red.global.add.f32), C written
// once; 0: each chunk stored to the slot and folded into C behind the next one.
// c3 FP32 67.7-68.0 vs 71.1-74.5 ms (same box; the clock under the power cap
// 1605-1620 vs 1466-1485 MHz: a quarter of the L2 traffic), same accuracy.
#define QG_TC2_RED 1
#endif
#ifndef QG_TC2_CHUNK_KT
#define QG_TC2_CHUNK_KT 32  // 256 quaternion k per chunk
#endif
__device__ __forceinline__ uint32_t smid() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%smid;\n" : "=r"(r));
  return r;
}
// Arrive on the barrier at this smem offset in CTA `rank` of the cluster (release, cluster scope).
__device__ __forceinline__ void mbar_arrive_cluster(uint64_t *bar, uint32_t rank) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(remote) : "r"(smem_u32(bar)), "r"(rank));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(remote) : "memory");
}
// Wait with cluster-scope acquire (arrivals from the peer CTA).
__device__ __forceinline__ void mbar_wait_cluster(uint64_t *bar, uint32_t parity) {
  const long long t0 = clock64();
  uint32_t done = 0;
  while (true) {
    asm volatile(
        "{\n.reg .pred P1;\nmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%1], %2;\n"
        "selp.b32 %0, 1, 0, P1;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (done) return;
    if (clock64() - t0 > 20000000000LL) __trap();
  }
}

// Tile pair `pid` of the grouped raster (kTc2GroupM pair-rows per group).
__device__ __forceinline__ void tc2_tile(int64_t pid, int64_t MT2, int64_t NT, int64_t &pm, int64_t &pn) {
  const int64_t per_group = int64_t(kTc2GroupM) * NT;
  const int64_t g = pid / per_group;
  const int64_t first_m = g * kTc2GroupM;
  const int64_t gsz = (MT2 - first_m) < kTc2GroupM ? (MT2 - first_m) : kTc2GroupM;
  const int64_t in = pid - g * per_group;
  pm = first_m + in % gsz;
  pn = in / gsz;
}

// kind::tf32, D f32, K-major A/B, M = 256 (pair), N = 128.
__host__ __device__ constexpr uint32_t tc2_idesc(bool negate_a) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((negate_a ? 1u : 0u) << 13) | (uint32_t(kTcBN >> 3) << 17) |
         (uint32_t(256 >> 4) << 24);
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

// 2-D TMA load into this CTA's smem; transaction bytes counted on the leader's barrier.
__device__ __forceinline__ void tma2_load_2d(void *dst, const CUtensorMap *tm, int c0, int c1, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3}], [%4];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(smem_u32(bar) & kPeerBitMask)
      : "memory");
}

__device__ __forceinline__ void tc2_mma(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

// Arrive (once the leader's prior MMAs complete) on the barrier at this smem
// offset in BOTH CTAs of the pair.
__device__ __forceinline__ void tc2_commit_both(uint64_t *bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
          smem_u32(bar)),
      "h"((unsigned short)3)
      : "memory");
}

// The 48 MMAs of one k-tile (4 output components x 4 products x 3xTF32), with
// the chunk bookkeeping: before the first MMA into component c of a new chunk,
// wait until both CTAs' epilogue warps have read that component of the previous
// chunk; after the last k-tile's MMAs into c, commit "component c complete".
// (Issued from an elect.sync branch of a whole warp: run by a lane-0-only branch
// next to the chunk epilogue's register arrays, ptxas moved the descriptors out
// of uniform registers -- an R2UR per operand per MMA -- and the single issuing
// thread fell behind the pipe: c3 FP32 67 vs 61 ms with chunks off.)
// 2-D TMA tile load into this CTA's smem completing on its own barrier.
__device__ __forceinline__ void tma_load_2d_local(void *dst, const CUtensorMap *tm, int c0, int c1, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// Split one raw tile (R rows x 8 k quaternions, as the direct feed's TMA left
// it) into the 8 tf32 planes [p][hi, lo] of the canonical K-major layout the
// MMA descriptors expect -- the pack kernel's arithmetic (conj, x_hi =
// tf32(x), x_lo = tf32(x - x_hi), qg_tc32.cuh), done in shared memory.
// Thread items: (row r, k quad kq); rows contiguous: raw (r, k, c) at
// ((r / 32) * 8 + k) * 128 + (r % 32) * 4 + c floats; k contiguous (128-byte
// swizzled rows of 8 quaternions): r * 32 + ((k ^ (r % 8)) * 4) + c.
template <int R>
__device__ __forceinline__ void tc2_convert(const float *raw, float *planes, int rc, int cj, int t, int nt) {
  constexpr int kPlane = R * kTcBK;  // floats per plane
  const float sg = cj ? -1.f : 1.f;
  for (int item = t; item < 2 * R; item += nt) {
    const int r = item % R, kq = item / R;
    float4 q[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int k = 4 * kq + e;
      const int off = rc ? ((r >> 5) * 8 + k) * 128 + (r & 31) * 4 : r * 32 + ((k ^ (r & 7)) << 2);
      q[e] = *reinterpret_cast<const float4 *>(raw + off);
    }
    const int poff = (r >> 3) * 64 + kq * 32 + (r & 7) * 4;
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      float x[4], hi[4], lo[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float v = p == 0 ? q[e].x : p == 1 ? q[e].y : p == 2 ? q[e].z : q[e].w;
        x[e] = p == 0 ? v : sg * v;
        hi[e] = tf32_rna(x[e]);
        lo[e] = tf32_rna(x[e] - hi[e]);
      }
      *reinterpret_cast<float4 *>(planes + (p * 2 + 0) * kPlane + poff) = make_float4(hi[0], hi[1], hi[2], hi[3]);
      *reinterpret_cast<float4 *>(planes + (p * 2 + 1) * kPlane + poff) = make_float4(lo[0], lo[1], lo[2], lo[3]);
    }
  }
}

__device__ __forceinline__ bool elect_one() {
  uint32_t pred;
  asm volatile("{\n.reg .pred p;\nelect.sync _|p, 0xffffffff;\nselp.u32 %0, 1, 0, p;\n}\n" : "=r"(pred));
  return pred != 0;
}
__device__ __forceinline__ void tc2_issue_ktile(uint32_t a0, uint32_t b0, uint32_t tmem, bool fresh, bool wait_empty,
                                             uint32_t empty_parity, uint64_t *acc_empty, bool ends,
                                             uint64_t *acc_full) {
  // descriptors of the stage's first A / B plane; the others differ only in the
  // start-address field (address >> 4, 14 bits: every smem address fits), so
  // each is the base plus a compile-time constant
  const uint64_t da = tc_sdesc(a0), db = tc_sdesc(b0);
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const uint32_t d = tmem + uint32_t(c * kTcBN);
    if (wait_empty) {  // both CTAs' epilogue warps have read component c of the previous chunk
      mbar_wait_cluster(&acc_empty[c], empty_parity);
      tc_fence_after();
    }
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      const int s = p ^ c;
      const uint32_t id = tc2_idesc(hneg(p, s));
      const uint64_t ahi = da + uint64_t(((p * 2 + 0) * kTcPlaneFloats * 4) >> 4);
      const uint64_t alo = da + uint64_t(((p * 2 + 1) * kTcPlaneFloats * 4) >> 4);
      const uint64_t bhi = db + uint64_t(((s * 2 + 0) * (kTcPlaneFloats / 2) * 4) >> 4);
      const uint64_t blo = db + uint64_t(((s * 2 + 1) * (kTcPlaneFloats / 2) * 4) >> 4);
      tc2_mma(d, ahi, bhi, id, (!fresh || p > 0) ? 1u : 0u);
      tc2_mma(d, ahi, blo, id, 1u);
      tc2_mma(d, alo, bhi, id, 1u);
    }
    // component c of this chunk complete once these MMAs are: the epilogue can
    // drain it while the pipe still runs the other components
    if (ends) tc2_commit_both(&acc_full[c]);
  }
}

// Fold W columns (n0..) of one thread's row into the target: the split-K
// partial (raw sums, coalesced over the warp's rows) or C (alpha; beta on the
// first contribution, else + C).
template <int W>
__device__ __forceinline__ void tc2_fold(const Tc2Args &args, float *part, int64_t row, int64_t pn, int lr, int n0,
                                         const float (&d)[4][W], bool first_chunk) {
  if (part) {
    float old[4][W];
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int jj = 0; jj < W; ++jj)  // every load before any store (they may alias as far as the compiler knows)
        old[c][jj] = first_chunk ? 0.f : __ldcg(part + (int64_t(c) * kTcBN + n0 + jj) * kTcBM + lr);
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int jj = 0; jj < W; ++jj)
        __stcg(part + (int64_t(c) * kTcBN + n0 + jj) * kTcBM + lr, first_chunk ? d[c][jj] : old[c][jj] + d[c][jj]);
    return;
  }
  if (row >= args.M) return;
  float cold[W][4];
  if (!args.sc.beta_zero || !first_chunk) {  // (beta = 0: C is never read, R3)
#pragma unroll
    for (int jj = 0; jj < W; ++jj) {
      const int64_t col = pn * kTcBN + n0 + jj;
      if (col < args.N) ldq_c(args.C + 4 * (row + col * args.ldc), cold[jj]);
    }
  }
#pragma unroll
  for (int jj = 0; jj < W; ++jj) {
    const int64_t col = pn * kTcBN + n0 + jj;
    if (col >= args.N) continue;
    const float acc[4] = {d[0][jj], d[1][jj], d[2][jj], d[3][jj]};
    float out[4];
    left_scale(args.sc.alpha, args.sc.alpha_real, acc, out);
    if (!first_chunk) {
#pragma unroll
      for (int k = 0; k < 4; ++k) out[k] += cold[jj][k];
    } else if (!args.sc.beta_zero) {
      float bc[4];
      left_scale(args.sc.beta, args.sc.beta_real, cold[jj], bc);
#pragma unroll
      for (int k = 0; k < 4; ++k) out[k] += bc[k];
    }
    stq(args.C + 4 * (row + col * args.ldc), out);
  }
}

// kDirect: operands read in place from the user's storage (raw TMA ring +
// converter warps 2-3); else from the pack kernel's chunks.
template <bool kDirect>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kTcThreads, 1)
    qgemm_tc32_2cta_kernel(const __grid_constant__ Tc2Args args) {
  constexpr int P = kDirect ? kTc2DStages : kTc2Stages;  // plane stages
  constexpr int RS = kTc2RawStages;
  extern __shared__ __align__(128) unsigned char smem_dyn[];
  unsigned char *smem = smem_dyn + ((1024u - (smem_u32(smem_dyn) & 1023u)) & 1023u);
  float *sA = reinterpret_cast<float *>(smem);
  float *sB = sA + P * kTc2AFloats;
  float *rA = sB + P * kTc2BFloats;                                   // direct: raw A tiles
  float *rB = rA + (kDirect ? RS * kTc2RawABytes / 4 : 0);            // direct: raw B halves
  uint64_t *full = reinterpret_cast<uint64_t *>(rB + (kDirect ? RS * kTc2RawBBytes / 4 : 0));  // leader's
  uint64_t *empty = full + P;
  uint64_t *acc_full = empty + P;     // [4] component c of a chunk complete (both CTAs, multicast)
  uint64_t *acc_empty = acc_full + 4; // [4] leader: component c of TMEM drained by both CTAs
  uint64_t *raw_full = acc_empty + 4; // direct [RS]: raw tile landed (TMA bytes)
  uint64_t *raw_empty = raw_full + RS;  // direct [RS]: converters done with the raw tile
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(raw_empty + RS);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  // tile pair of this cluster (grouped rasterisation as the 1-CTA kernel): the
  // first `full` clusters each take a whole pair; past them, pair full + r / S
  // and its share [k0, k1) of the k-tiles (split ks = r % S)
  const int64_t cid = int64_t(blockIdx.x) >> 1;
  const bool split = cid >= args.full;
  const int64_t Su = split ? args.S : 1;
  const int64_t pid = split ? args.full + (cid - args.full) / Su : cid, ks = split ? (cid - args.full) % Su : 0;
  int64_t pm, pn;
  tc2_tile(pid, args.MT2, args.NT, pm, pn);
  const int64_t mt = 2 * pm + rank;  // this CTA's 128-row A tile
  const int64_t KT = args.KT;
  const int64_t k0 = ks * KT / Su, k1 = (ks + 1) * KT / Su;

  if (threadIdx.x == 0) {
    for (int s = 0; s < P; ++s) {
      mbar_init(&full[s], kDirect ? 4 : 1);  // direct: 2 converter warps x 2 CTAs arrive
      mbar_init(&empty[s], 1);
    }
    if (kDirect)
      for (int s = 0; s < RS; ++s) {
        mbar_init(&raw_full[s], 1);
        mbar_init(&raw_empty[s], 2);
      }
    for (int c = 0; c < 4; ++c) mbar_init(&acc_full[c], 1);
    for (int c = 0; c < 4; ++c) mbar_init(&acc_empty[c], 8);  // 4 epilogue warps x 2 CTAs
    fence_mbar_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 && lane == 0) {
    // ---------------- producer (both CTAs) ----------------
    int slot = 0;
    uint32_t phase = 0;
    for (int64_t kt = k0; kt < k1; ++kt) {
      if constexpr (kDirect) {
        // raw interleaved tiles of this CTA's 128 rows of op(A) and 64 columns of op(B)
        if (kt - k0 >= RS) mbar_wait_guarded(&raw_empty[slot], phase ^ 1u);
        mbar_arrive_expect_tx(&raw_full[slot], kTc2RawABytes + kTc2RawBBytes);
        float *ra = rA + slot * (kTc2RawABytes / 4), *rb = rB + slot * (kTc2RawBBytes / 4);
        const int ka = int(kt * kTcBK), r0 = int(mt * kTcBM), n0 = int(pn * kTcBN + rank * (kTcBN / 2));
        if (args.a_rc)
          for (int j = 0; j < kTcBM / 32; ++j)
            tma_load_2d_local(ra + j * (32 * 4 * kTcBK), &args.tmA, 4 * (r0 + 32 * j), ka, &raw_full[slot]);
        else
          tma_load_2d_local(ra, &args.tmA, 4 * ka, r0, &raw_full[slot]);
        if (args.b_rc)
          for (int j = 0; j < kTcBN / 64; ++j)
            tma_load_2d_local(rb + j * (32 * 4 * kTcBK), &args.tmB, 4 * (n0 + 32 * j), ka, &raw_full[slot]);
        else
          tma_load_2d_local(rb, &args.tmB, 4 * ka, n0, &raw_full[slot]);
        if (++slot == RS) { slot = 0; phase ^= 1u; }
      } else {
        if (kt - k0 >= P) mbar_wait_guarded(&empty[slot], phase ^ 1u);
        if (rank == 0) mbar_arrive_expect_tx(&full[slot], 2 * (kTc2ABytes + kTc2BBytes));
        tma2_load_2d(sA + slot * kTc2AFloats, &args.tmA, 0, int((mt * KT + kt) * 32), &full[slot]);
        tma2_load_2d(sB + slot * kTc2BFloats, &args.tmB, 0, int((pn * KT + kt) * 32 + rank * 16), &full[slot]);
        if (++slot == P) { slot = 0; phase ^= 1u; }
      }
    }
  } else if (kDirect && (warp == 2 || warp == 3)) {
    // ---------------- converters (both CTAs): raw tile -> tf32 hi / lo planes ----------------
    int rs = 0, ps = 0;
    uint32_t rph = 0, pph = 0;
    const int t = threadIdx.x - 64;
    for (int64_t kt = k0; kt < k1; ++kt) {
      mbar_wait_guarded(&raw_full[rs], rph);
      if (kt - k0 >= P) mbar_wait_guarded(&empty[ps], pph ^ 1u);  // the MMAs have read this plane stage
      tc2_convert<kTcBM>(rA + rs * (kTc2RawABytes / 4), sA + ps * kTc2AFloats, args.a_rc, args.a_cj, t, 64);
      tc2_convert<kTcBM / 2>(rB + rs * (kTc2RawBBytes / 4), sB + ps * kTc2BFloats, args.b_rc, args.b_cj, t, 64);
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // generic writes -> the MMA's reads
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&raw_empty[rs]);
        mbar_arrive_cluster(&full[ps], 0);  // the leader's stage barrier (both CTAs' planes ready)
      }
      if (++rs == RS) { rs = 0; rph ^= 1u; }
      if (++ps == P) { ps = 0; pph ^= 1u; }
    }
  } else if (warp == 1 && rank == 0) {
    // ---------------- MMA issuer (leader only) ----------------
    // The whole warp walks the loop (its control values are warp-uniform, so
    // ptxas keeps the descriptors in uniform registers); one elected lane issues.
    int slot = 0;
    uint32_t phase = 0;
    const int kc = args.kc;
    uint32_t chunk = 0;
    int kk = 0;  // k-tile index inside the current accumulation chunk (no divisions in this loop)
    for (int64_t kt = k0; kt < k1; ++kt) {
      const bool fresh = kk == 0;                         // first k-tile of an accumulation chunk
      const bool ends = kk == kc - 1 || kt + 1 == k1;     // last k-tile of a chunk
      if (++kk == kc) kk = 0;
      if (kDirect) mbar_wait_cluster(&full[slot], phase);  // converters of both CTAs (release.cluster)
      else mbar_wait_guarded(&full[slot], phase);
      tc_fence_after();
      if (elect_one())
        tc2_issue_ktile(smem_u32(sA + slot * kTc2AFloats), smem_u32(sB + slot * kTc2BFloats), tmem, fresh,
                        fresh && kt > k0, (chunk - 1) & 1u, acc_empty, ends, acc_full);
      __syncwarp();
      if (lane == 0) tc2_commit_both(&empty[slot]);  // both CTAs may refill this stage
      if (++slot == P) { slot = 0; phase ^= 1u; }
      if (ends) ++chunk;
    }
  } else if (warp >= 4) {
    // ---------------- epilogue (both CTAs): TMEM -> registers -> C ----------------
    const int q = warp - 4;
    const int64_t row = mt * kTcBM + q * 32 + lane;
    const uint32_t tbase = tmem + (uint32_t(q * 32) << 16);
    float *part = Su > 1 ? args.part + (((pid - args.full) * Su + ks) * 2 + rank) * kTc2PartFloats : nullptr;
    const int64_t nchunks = (k1 - k0 + args.kc - 1) / args.kc;
    // this SM's running-sum slot, [c][col / 4][row][col % 4]: each thread's 4
    // consecutive columns are one 16-byte vector (one vector reduction; a warp's
    // 32 rows are 512 contiguous bytes); without a slot (SM id past the slots)
    // every chunk folds into the target straight from TMEM
    const uint32_t sm = smid();
    float *slotp = sm < uint32_t(args.nslots) ? args.tmp + int64_t(sm) * kTc2PartFloats + 4 * (q * 32 + lane) : nullptr;
    auto slot_off = [](int c, int n) { return (int64_t(c) * (kTcBN / 4) + (n >> 2)) * (4 * kTcBM) + (n & 3); };
    auto ld_tmem16 = [&](int n0, float (&d)[4][16]) {
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld16(tbase + uint32_t(c * kTcBN + n0), d[c]);
      tmem_ld_wait();
    };
    auto release = [&](int c) {  // component c of TMEM may be overwritten by the next chunk
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(&acc_empty[c], 0);
    };
    for (int64_t j = 0; j < nchunks; ++j) {
      if (j + 1 < nchunks && slotp) {
        // component by component: TMEM -> registers, release the component (the
        // next chunk's MMAs into it may start), registers -> slot (plain stores);
        // then fold the slot into the target while the next chunk runs
#pragma unroll 1
        for (int c = 0; c < 4; ++c) {
          mbar_wait_guarded(&acc_full[c], uint32_t(j & 1));
          tc_fence_after();
          float v[kTcBN];
#pragma unroll
          for (int n0 = 0; n0 < kTcBN; n0 += 16) {
            float (&d)[16] = *reinterpret_cast<float (*)[16]>(&v[n0]);
            tmem_ld16(tbase + uint32_t(c * kTcBN + n0), d);
          }
          tmem_ld_wait();
          release(c);
          float *sp = slotp + slot_off(c, 0);
#if QG_TC2_RED
          // running sum in the slot: the first chunk stores, later ones add in L2
          // (red.global.add.v4.f32, round-to-nearest; no round trip, nothing to
          // wait for; one 16-byte reduction per 4 columns: a quarter of the L2
          // operations of scalar reductions)
          if (j == 0) {
#pragma unroll
            for (int n = 0; n < kTcBN; n += 4)
              __stcg(reinterpret_cast<float4 *>(sp + slot_off(0, n)), make_float4(v[n], v[n + 1], v[n + 2], v[n + 3]));
          } else {
#pragma unroll
            for (int n = 0; n < kTcBN; n += 4)
              asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};\n" ::"l"(sp + slot_off(0, n)), "f"(v[n]),
                           "f"(v[n + 1]), "f"(v[n + 2]), "f"(v[n + 3])
                           : "memory");
          }
#else
#pragma unroll
          for (int n = 0; n < kTcBN; n += 4)
            __stcg(reinterpret_cast<float4 *>(sp + slot_off(0, n)), make_float4(v[n], v[n + 1], v[n + 2], v[n + 3]));
#endif
        }
#if !QG_TC2_RED
        for (int n0 = 0; n0 < kTcBN; n0 += 8) {
          float d[4][8];
#pragma unroll
          for (int c = 0; c < 4; ++c)
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) d[c][jj] = __ldcg(slotp + slot_off(c, n0 + jj));
          tc2_fold<8>(args, part, row, pn, q * 32 + lane, n0, d, j == 0);
        }
#endif
        continue;
      }
      // the last chunk (or any chunk without a slot) folds straight from TMEM
      // (QG_TC2_RED: plus the running sum of the earlier chunks from the slot)
      for (int c = 0; c < 4; ++c) mbar_wait_guarded(&acc_full[c], uint32_t(j & 1));
      tc_fence_after();
      const bool with_slot = QG_TC2_RED && slotp && nchunks > 1;
      for (int n0 = 0; n0 < kTcBN; n0 += 16) {
        float d[4][16];
        ld_tmem16(n0, d);
        if (with_slot) {
          float4 o[4][4];
#pragma unroll
          for (int c = 0; c < 4; ++c)
#pragma unroll
            for (int g = 0; g < 4; ++g) o[c][g] = __ldcg(reinterpret_cast<const float4 *>(slotp + slot_off(c, n0 + 4 * g)));
#pragma unroll
          for (int c = 0; c < 4; ++c)
#pragma unroll
            for (int g = 0; g < 4; ++g) {
              d[c][4 * g] += o[c][g].x;
              d[c][4 * g + 1] += o[c][g].y;
              d[c][4 * g + 2] += o[c][g].z;
              d[c][4 * g + 3] += o[c][g].w;
            }
        }
        tc2_fold<16>(args, part, row, pn, q * 32 + lane, n0, d, with_slot || j == 0);
      }
      if (j + 1 < nchunks)
        for (int c = 0; c < 4; ++c) release(c);
    }
  }
  tc_fence_before();
  cluster_sync_all();  // no CTA frees TMEM / exits while its peer's MMAs may still target it
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;\n" ::"r"(tmem) : "memory");
  }
}

// Split-K epilogue of the split pairs (raster positions full..): C(row, col) <-
// alpha (x) sum_ks part_ks + beta (x) C, the S partials added in split order
// (deterministic).  Block = one CTA tile's 128 rows (threads) x 16 columns;
// grid = (2 * split pairs, 8).
__global__ void __launch_bounds__(kTcBM) tc2_reduce_kernel(const __grid_constant__ Tc2Args args) {
  const int64_t cta = blockIdx.x, sp = cta >> 1, pid = args.full + sp;
  const int rank = int(cta & 1);
  int64_t pm, pn;
  tc2_tile(pid, args.MT2, args.NT, pm, pn);
  const int64_t row = (2 * pm + rank) * kTcBM + threadIdx.x;
  if (row >= args.M) return;
  const float *p0 = args.part + (sp * args.S * 2 + rank) * kTc2PartFloats + threadIdx.x;
  const int64_t stride = 2 * kTc2PartFloats;  // next split, same rank
  for (int j = 0; j < 16; ++j) {
    const int cl = int(blockIdx.y) * 16 + j;
    const int64_t col = pn * kTcBN + cl;
    if (col >= args.N) break;
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    for (int k = 0; k < args.S; ++k)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[c] += __ldcg(p0 + k * stride + (int64_t(c) * kTcBN + cl) * kTcBM);
    float *cp = args.C + 4 * (row + col * args.ldc);
    float out[4];
    left_scale(args.sc.alpha, args.sc.alpha_real, acc, out);
    if (!args.sc.beta_zero) {
      float cold[4], bc[4];
      ldq_c(cp, cold);
      left_scale(args.sc.beta, args.sc.beta_real, cold, bc);
#pragma unroll
      for (int c = 0; c < 4; ++c) out[c] += bc[c];
    }
    stq(cp, out);
  }
}

}  // namespace qg
