// qg_simt_f32.cuh -- FP32 mainloop on the FP32 FMA pipe with fused epilogue.
//
// Same method as qg_dmma.cuh (Alg. 3 P:1004-1028 rank-1 updates,
// Hamilton rule P:299-309 as D^{p^s} += eps(p,s) A^p B^s), on FFMA: each
// thread owns a 4x4 block of output quaternions (64 fp32 accumulators) and per
// k loads 4 A quaternions + 4 B quaternions as component planes (8 LDS.128),
// then issues 256 FMAs: every loaded component feeds 4 rows x 4 output
// components (the register blocking the north star asks for).  FP32 on the
// tensor cores (1xTF32) misses the FP32 tolerance, so this path
// stays on FFMA.
//
// CTA: 64x64 quaternions = 16x16 threads (8 warps, each 4 thread-rows x 8
// thread-cols) + 1 producer warp; packed chunks (PlanarLayout [k][c][r]) are
// streamed through a 4-stage ring with cp.async.bulk + mbarriers.
#pragma once
#include "qg_dmma.cuh"

namespace qg {

constexpr int kF32Stages = 4;
constexpr int kF32ConsumerWarps = 8;
constexpr int kF32Threads = (kF32ConsumerWarps + 1) * 32;
constexpr size_t kF32SmemBytes = size_t(kF32Stages) * 2 * kChunkElems * sizeof(float) + 2 * kF32Stages * 8;

struct F32Args {
  const float *Ap;
  const float *Bp;
  float *C;
  int64_t ldc, M, N, MT, NT, KT;
  Scalars<float> sc;
};

__global__ void __launch_bounds__(kF32Threads, 1) qgemm_simt_f32_kernel(const F32Args args) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float *sA = reinterpret_cast<float *>(smem_raw);
  float *sB = sA + kF32Stages * kChunkElems;
  uint64_t *full = reinterpret_cast<uint64_t *>(sB + kF32Stages * kChunkElems);
  uint64_t *empty = full + kF32Stages;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  int64_t mt, nt;
  tile_coords(blockIdx.x, args.MT, args.NT, mt, nt);
  const int64_t KT = args.KT;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kF32Stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kF32ConsumerWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == kF32ConsumerWarps) {
    if (lane == 0) {
      const float *a_src = args.Ap + mt * KT * kChunkElems;
      const float *b_src = args.Bp + nt * KT * kChunkElems;
      constexpr uint32_t kBytes = kChunkElems * sizeof(float);
      for (int64_t kt = 0; kt < KT; ++kt) {
        const int slot = int(kt % kF32Stages);
        if (kt >= kF32Stages) mbar_wait(&empty[slot], uint32_t((kt / kF32Stages) - 1) & 1u);
        mbar_arrive_expect_tx(&full[slot], 2 * kBytes);
        bulk_g2s(sA + slot * kChunkElems, a_src + kt * kChunkElems, kBytes, &full[slot]);
        bulk_g2s(sB + slot * kChunkElems, b_src + kt * kChunkElems, kBytes, &full[slot]);
      }
    }
    return;
  }

  const int tm = (warp & 3) * 4 + (lane & 3);   // thread-row 0..15 -> rows 4tm..4tm+3
  const int tn = (warp >> 2) * 8 + (lane >> 2);  // thread-col 0..15 -> cols 4tn..4tn+3
  float acc[4][4][4];  // [row][col][component]
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[i][j][c] = 0.f;

  int slot = 0;
  uint32_t phase = 0;
  for (int64_t kt = 0; kt < KT; ++kt) {
    mbar_wait(&full[slot], phase);
    const float *a = sA + slot * kChunkElems;
    const float *b = sB + slot * kChunkElems;
#pragma unroll 4
    for (int k = 0; k < kBK; ++k) {
      float af[4][4], bf[4][4];  // [component][row or col]
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        float4 va = *reinterpret_cast<const float4 *>(a + (k * 4 + c) * kBR + 4 * tm);
        float4 vb = *reinterpret_cast<const float4 *>(b + (k * 4 + c) * kBR + 4 * tn);
        af[c][0] = va.x; af[c][1] = va.y; af[c][2] = va.z; af[c][3] = va.w;
        bf[c][0] = vb.x; bf[c][1] = vb.y; bf[c][2] = vb.z; bf[c][3] = vb.w;
      }
#pragma unroll
      for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int s = 0; s < 4; ++s)
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              if (hneg(p, s)) acc[i][j][p ^ s] = fmaf(-af[p][i], bf[s][j], acc[i][j][p ^ s]);
              else acc[i][j][p ^ s] = fmaf(af[p][i], bf[s][j], acc[i][j][p ^ s]);
            }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[slot]);
    if (++slot == kF32Stages) { slot = 0; phase ^= 1u; }
  }

#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t row = mt * kBR + 4 * tm + i;
    if (row >= args.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t col = nt * kBR + 4 * tn + j;
      if (col >= args.N) continue;
      const float q[4] = {acc[i][j][0], acc[i][j][1], acc[i][j][2], acc[i][j][3]};
      epilogue_one(args.sc, q, args.C + 4 * (row + col * args.ldc));
    }
  }
}

}  // namespace qg
