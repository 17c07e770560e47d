// qg_tc32.cuh -- FP32 QGEMM on the 5th-generation tensor cores (tcgen05, TMEM)
// with 3xTF32 error compensation.
//
// Method (same algebra as qg_dmma.cuh): with component planes the quaternion
// product is 16 real products per output tile, D^{p XOR s} += eps(p,s) A^p B^s
// (Eq. quaternion_prod P:299-309 restated as a sign rule, qg_common.cuh).  Each
// real product is one tcgen05.mma.kind::tf32 (M = 128 quaternion rows, N = 128
// quaternion columns, K = 8); the sign eps(p,s) = -1 is the instruction
// descriptor's negate-A bit, so no signed copies exist anywhere.  The four
// output components live in four 128-column TMEM accumulators (all 512 columns).
//
// 3xTF32: every FP32 operand x is split by the pack into x_hi = tf32(x) and
// x_lo = tf32(x - x_hi) (round-to-nearest); per real product three MMAs,
// A_hi B_hi + A_hi B_lo + A_lo B_hi, accumulate in FP32.  1xTF32 misses the
// FP32 tolerance at config 3 (simulated max error 0.31 vs 0.30);
// 3xTF32 is accurate to about FP32 (the dropped A_lo B_lo term is ~2^-22 relative).
//
// Operands come from shared memory in the canonical no-swizzle K-major layout
// ("core matrices" of 8 rows x 16 bytes): element (r, k) of a 128 x 8 plane at
// byte (r/8)*256 + (k/4)*128 + (r%8)*16 + (k%4)*4 (LBO = 128 B between the two
// K core matrices, SBO = 256 B between 8-row groups).  The pack (pack_tc32_kernel)
// writes chunks that are byte images of a pipeline stage -- 8 planes
// [p][hi, lo] of 4 KB for one 128-row tile and 8 k -- so a stage is two 1-D bulk
// copies (A chunk, B chunk) completing on an mbarrier, as in the FP64 path.
//
// Warp roles (256 threads, one tile per CTA): warp 0 allocates TMEM and its
// lane 0 streams stages; warp 1 lane 0 issues the MMAs (48 per stage) and
// commits each stage back to the producer and the finished accumulators to the
// epilogue; warps 4..7 (one TMEM lane quarter each) read the accumulators with
// tcgen05.ld, apply alpha/beta from the left and store whole quaternions.
#pragma once
#include "qg_common.cuh"
#include "qg_pack.cuh"  // PackJob

namespace qg {

constexpr int kTcBM = 128;  // quaternion rows per tile (= UMMA M)
constexpr int kTcBN = 128;  // quaternion columns per tile (= UMMA N)
constexpr int kTcBK = 8;    // quaternion k per stage (= UMMA K for tf32)
constexpr int kTcGroupM = 8;  // tile rasterisation group (L2 reuse of A/B panels)
constexpr int kTcPlaneFloats = 128 * kTcBK;            // one 128 x 8 plane
constexpr int kTcChunkFloats = 8 * kTcPlaneFloats;     // planes [p 4][hi, lo]
constexpr uint32_t kTcChunkBytes = kTcChunkFloats * 4; // 32 KiB
constexpr int kTcStages = 3;
constexpr int kTcPackSub = 4;  // chunks packed per block
constexpr int kTcThreads = 256;
constexpr size_t kTcSmemBytes = size_t(kTcStages) * 2 * kTcChunkBytes + 256;

// Float offset of element (r, k) (r < 128, k < 8) inside a plane.
__host__ __device__ constexpr int tc_plane_offset(int r, int k) {
  return (r >> 3) * 64 + (k >> 2) * 32 + (r & 7) * 4 + (k & 3);
}

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// Pack for the tensor-core path: rows r of op(X) (R of them) x k in
// [k_begin, k_end), conj applied, split into tf32 hi/lo, one 32 KiB chunk per
// (128-row tile, 8-k tile).  A block packs kTcPackSub consecutive chunks of one
// row tile: grid = RT * ceil(KT / kTcPackSub) blocks of 256 threads.
// grid = ja.blocks + jb.blocks: A and B in one launch (as pack_kernel).
__global__ void __launch_bounds__(256) pack_tc32_kernel(const PackJob<float> ja, const PackJob<float> jb) {
  const bool second = int64_t(blockIdx.x) >= ja.blocks;
  const PackJob<float> &j = second ? jb : ja;
  const int64_t bid = second ? int64_t(blockIdx.x) - ja.blocks : int64_t(blockIdx.x);
  const float *__restrict__ X = j.X;
  const int64_t ldx = j.ldx, R = j.R, k_end = j.k_end, KT = j.KT;
  const int row_contig = j.row_contig, conj = j.conj;
  float *__restrict__ out = j.out;
  // [k][component][row], rows padded to 129: conflict-free for both the
  // staging writes (consecutive rows, or consecutive k) and the per-plane reads
  constexpr int kPitch = kTcBM + 1;
  __shared__ float tile[kTcBK][4][kPitch];
  const int64_t KTS = (KT + kTcPackSub - 1) / kTcPackSub;  // blocks per row tile
  const int64_t rt = bid / KTS;
  const int64_t r0 = rt * kTcBM;
  const float sgn = conj ? -1.f : 1.f;
  for (int sub = 0; sub < kTcPackSub; ++sub) {
    const int64_t kt = (bid % KTS) * kTcPackSub + sub;
    if (kt >= KT) break;
    const int64_t k0 = j.k_begin + kt * kTcBK;
    if (sub) __syncthreads();  // the previous chunk's reads of `tile` are done
#pragma unroll
    for (int it = 0; it < (kTcBM * kTcBK) / 256; ++it) {
      const int q = threadIdx.x + 256 * it;
      int r, k;
      if (row_contig) { r = q % kTcBM; k = q / kTcBM; }
      else            { k = q % kTcBK; r = q / kTcBK; }
      const int64_t rg = r0 + r, kg = k0 + k;
      float v[4] = {0.f, 0.f, 0.f, 0.f};
      if (rg < R && kg < k_end) {
        ldq(row_contig ? X + 4 * (rg + kg * ldx) : X + 4 * (kg + rg * ldx), v);
        v[1] *= sgn; v[2] *= sgn; v[3] *= sgn;
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) tile[k][c][r] = v[c];
    }
    __syncthreads();
    float4 *o = reinterpret_cast<float4 *>(out + (rt * KT + kt) * int64_t(kTcChunkFloats));
    for (int o4 = threadIdx.x; o4 < kTcChunkFloats / 4; o4 += 256) {
      const int plane = o4 >> 8, rem = o4 & 255;
      const int rg = rem >> 4, kh = (rem >> 3) & 1, r8 = rem & 7;
      const int r = rg * 8 + r8, kb = kh * 4, p = plane >> 1, lo = plane & 1;
      float w[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float x = tile[kb + e][p][r];
        const float hi = tf32_rna(x);
        w[e] = lo ? tf32_rna(x - hi) : hi;
      }
      // split_halves: rows 64h.. of every plane grouped per half h -> [h][plane][64 x 8]
      const int dst = j.split_halves ? (rg >> 3) * 1024 + plane * 128 + (rem & 127) : o4;
      o[dst] = make_float4(w[0], w[1], w[2], w[3]);
    }
  }
}

// ---------------------------------------------------------------- tcgen05 helpers
__device__ __forceinline__ uint64_t tc_sdesc(uint32_t saddr) {
  uint64_t d = uint64_t((saddr >> 4) & 0x3FFFu);
  d |= uint64_t(128 >> 4) << 16;  // LBO: next core matrix along K
  d |= uint64_t(256 >> 4) << 32;  // SBO: next 8-row group
  d |= uint64_t(1) << 46;         // descriptor version 1 (sm_100)
  return d;                       // base offset 0, SWIZZLE_NONE
}

// kind::tf32 instruction descriptor: D f32, A/B tf32, K-major, M = 128, N = 128.
__host__ __device__ constexpr uint32_t tc_idesc(bool negate_a) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((negate_a ? 1u : 0u) << 13) | (uint32_t(kTcBN >> 3) << 17) |
         (uint32_t(kTcBM >> 4) << 24);
}

__device__ __forceinline__ void tc_mma(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void tc_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }

struct Tc32Args {
  const float *Ap;  // MT x KT chunks (128-row tiles)
  const float *Bp;  // NT x KT chunks
  float *C;
  int64_t ldc, M, N, MT, NT, KT;
  Scalars<float> sc;
};

// mbarrier wait that traps after ~10 s instead of hanging the GPU if an
// asynchronous (tensor-core / bulk-copy) completion never arrives.
__device__ __forceinline__ void mbar_wait_guarded(uint64_t *bar, uint32_t parity) {
  const long long t0 = clock64();
  uint32_t done = 0;
  while (true) {
    asm volatile(
        "{\n.reg .pred P1;\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\nselp.b32 %0, 1, 0, P1;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (done) return;
    if (clock64() - t0 > 20000000000LL) __trap();
  }
}

__global__ void __launch_bounds__(kTcThreads, 1) qgemm_tc32_kernel(const Tc32Args args) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float *sA = reinterpret_cast<float *>(smem_raw);
  float *sB = sA + kTcStages * kTcChunkFloats;
  uint64_t *full = reinterpret_cast<uint64_t *>(sB + kTcStages * kTcChunkFloats);
  uint64_t *empty = full + kTcStages;
  uint64_t *acc_full = empty + kTcStages;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(acc_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // grouped rasterisation (groups of kTcGroupM M-tiles, M fastest inside a
  // group): a wave of 148 CTAs touches ~8 A + ~18 B panels, which L2 holds,
  // instead of every A panel (measured 131 GB of DRAM reads per c3 launch
  // with plain M-fastest order)
  int64_t mt, nt;
  {
    const int64_t per_group = int64_t(kTcGroupM) * args.NT;
    const int64_t g = int64_t(blockIdx.x) / per_group;
    const int64_t first_m = g * kTcGroupM;
    const int64_t gsz = (args.MT - first_m) < kTcGroupM ? (args.MT - first_m) : kTcGroupM;
    const int64_t in = int64_t(blockIdx.x) - g * per_group;
    mt = first_m + in % gsz;
    nt = in / gsz;
  }
  const int64_t KT = args.KT;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kTcStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(acc_full, 1);
    fence_mbar_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 && lane == 0) {
    // ---------------- producer ----------------
    const float *a_src = args.Ap + mt * KT * kTcChunkFloats;
    const float *b_src = args.Bp + nt * KT * kTcChunkFloats;
    int slot = 0;
    uint32_t phase = 0;
    for (int64_t kt = 0; kt < KT; ++kt) {
      if (kt >= kTcStages) mbar_wait_guarded(&empty[slot], phase ^ 1u);
      mbar_arrive_expect_tx(&full[slot], 2 * kTcChunkBytes);
      bulk_g2s(sA + slot * kTcChunkFloats, a_src + kt * kTcChunkFloats, kTcChunkBytes, &full[slot]);
      bulk_g2s(sB + slot * kTcChunkFloats, b_src + kt * kTcChunkFloats, kTcChunkBytes, &full[slot]);
      if (++slot == kTcStages) { slot = 0; phase ^= 1u; }
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer ----------------
    int slot = 0;
    uint32_t phase = 0;
    for (int64_t kt = 0; kt < KT; ++kt) {
      mbar_wait_guarded(&full[slot], phase);
      tc_fence_after();
      const uint32_t a0 = smem_u32(sA + slot * kTcChunkFloats);
      const uint32_t b0 = smem_u32(sB + slot * kTcChunkFloats);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const uint32_t d = tmem + uint32_t(c * kTcBN);
#pragma unroll
        for (int p = 0; p < 4; ++p) {
          const int s = p ^ c;
          const uint32_t id = tc_idesc(hneg(p, s));
          const uint64_t ahi = tc_sdesc(a0 + (p * 2 + 0) * kTcPlaneFloats * 4);
          const uint64_t alo = tc_sdesc(a0 + (p * 2 + 1) * kTcPlaneFloats * 4);
          const uint64_t bhi = tc_sdesc(b0 + (s * 2 + 0) * kTcPlaneFloats * 4);
          const uint64_t blo = tc_sdesc(b0 + (s * 2 + 1) * kTcPlaneFloats * 4);
          tc_mma(d, ahi, bhi, id, (kt > 0 || p > 0) ? 1u : 0u);
          tc_mma(d, ahi, blo, id, 1u);
          tc_mma(d, alo, bhi, id, 1u);
        }
      }
      tc_commit(&empty[slot]);  // frees the stage once these MMAs have read it
      if (++slot == kTcStages) { slot = 0; phase ^= 1u; }
    }
    tc_commit(acc_full);  // accumulators complete
  } else if (warp >= 4) {
    // ---------------- epilogue: TMEM -> registers -> C ----------------
    const int q = warp - 4;                    // TMEM lanes 32q .. 32q+31
    const int row_in_tile = q * 32 + lane;
    const int64_t row = mt * kTcBM + row_in_tile;
    mbar_wait_guarded(acc_full, 0);
    tc_fence_after();
    const uint32_t tbase = tmem + (uint32_t(q * 32) << 16);
    for (int n0 = 0; n0 < kTcBN; n0 += 16) {
      float d[4][16];
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld16(tbase + uint32_t(c * kTcBN + n0), d[c]);
      tmem_ld_wait();
      if (row < args.M) {
        float cold[16][4];
        if (!args.sc.beta_zero) {
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int64_t col = nt * kTcBN + n0 + j;
            if (col < args.N) ldq_c(args.C + 4 * (row + col * args.ldc), cold[j]);
          }
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int64_t col = nt * kTcBN + n0 + j;
          if (col >= args.N) continue;
          const float acc[4] = {d[0][j], d[1][j], d[2][j], d[3][j]};
          float out[4];
          left_scale(args.sc.alpha, args.sc.alpha_real, acc, out);
          if (!args.sc.beta_zero) {
            float bc[4];
            left_scale(args.sc.beta, args.sc.beta_real, cold[j], bc);
#pragma unroll
            for (int k = 0; k < 4; ++k) out[k] += bc[k];
          }
          stq(args.C + 4 * (row + col * args.ldc), out);
        }
      }
    }
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem) : "memory");
  }
}

}  // namespace qg
