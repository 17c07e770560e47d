// qg_pack.cuh -- pack kernels (SURVEY.md §8(a) rows a2 "Pack A" and a3 "Pack B").
//
// PAPER.md Alg. 4 PACK1 / Alg. 5 PACK2: copy a panel of op(X)
// into contiguous auxiliary storage in exactly the order the micro-kernel
// consumes it, applying PACKOP.  The paper's central quaternion
// idea -- move the AoS->SoA rearrangement of the interleaved
// [q0;q1;q2;q3] elements out of the micro-kernel and into the bandwidth-bound
// pack -- is kept; the register-transpose choreography of the AVX kernels is not.
//
// One pack kernel serves A and B: both operands are handled as an R x K panel
// X~(r, k) (r = row of op(A), or column of op(B)), with
//     stored address of X~(r, k) = X + 4 * (r + k*ldx)   (row_contig = 1)
//                               or X + 4 * (k + r*ldx)   (row_contig = 0)
//   A: op N -> row_contig=1;  op T/H -> row_contig=0
//   B: op N -> row_contig=0;  op T/H -> row_contig=1
// and conj (op H) negating components 1..3 (Eq. quaternion_conj).
// Rows r >= R and k >= K are zero-filled up to tile multiples, so
// the mainloop needs no bounds checks; only the epilogue masks.
//
// Output: one contiguous CHUNK per (row tile rt, k tile kt), chunk index
// rt*KT + kt, so a pipeline stage is ONE bulk copy.  Chunk layouts:
//   FragLayout   (FP64, DMMA m8n8k4): [ks 4][i 8][pp 2][lane 32][e 2]
//       value = X~(8i + lane/4, 4ks + lane%4) component 2pp+e; a lane's 16-byte
//       word holds its A (or B) fragments of two components, for both operands
//       (the m8n8k4 A fragment is A[lane/4][lane%4], B fragment B[lane%4][lane/4]).
// (the FP32 tcgen05 path has its own pack, qg_tc32.cuh pack_tc32_kernel)
#pragma once
#include <type_traits>
#include "qg_common.cuh"

namespace qg {

constexpr int kBR = 64;   // rows of a tile (BM = BN)
constexpr int kBK = 16;   // k of a tile (quaternions)
constexpr int kChunkElems = kBR * kBK * 4;

struct FragLayout {
  // element offset inside a chunk of (r, k, c)
  __device__ __forceinline__ static int offset(int r, int k, int c) {
    int ks = k >> 2, i = r >> 3, lane = ((r & 7) << 2) | (k & 3), pp = c >> 1, e = c & 1;
    return ((((ks * 8 + i) * 2 + pp) * 32 + lane) << 1) | e;
  }
};

// One operand panel to pack: rows [0, R) x k in [k_begin, k_end) of op(X), as
// RT*KT chunks (RT = ceil(R / tile rows)); `blocks` = RT*KT.
template <typename T>
struct PackJob {
  const T *X;
  int64_t ldx;
  int row_contig, conj;
  int64_t R, k_begin, k_end, KT;
  T *out;
  int64_t blocks;
  int split_halves;  // FP32 tcgen05 pack only: each 64-row half of a chunk contiguous (2-CTA B operand)
};

// grid: ja.blocks + jb.blocks blocks (1-D), 256 threads: A and B are packed by
// ONE launch (jb.blocks may be 0).  Tile staged through shared memory so both
// the global reads (along the stored contiguous axis) and the chunk writes
// (linear) are coalesced.
template <typename T, class Layout>
__global__ void __launch_bounds__(256) pack_kernel(const PackJob<T> ja, const PackJob<T> jb) {
  const bool second = int64_t(blockIdx.x) >= ja.blocks;
  const PackJob<T> &j = second ? jb : ja;
  const int64_t bid = second ? int64_t(blockIdx.x) - ja.blocks : int64_t(blockIdx.x);
  const T *__restrict__ X = j.X;
  const int64_t ldx = j.ldx, R = j.R, k_end = j.k_end, KT = j.KT;
  const int row_contig = j.row_contig, conj = j.conj;
  T *__restrict__ out = j.out;
  __shared__ __align__(16) T tile[kBK * kBR * 4 + 4 * kBK];  // [k][r][c], rows padded by 4 elems per k
  constexpr int kPitch = kBR * 4 + 4;
  const int64_t rt = bid / KT;
  const int64_t kt = bid % KT;
  const int64_t r0 = rt * kBR;
  const int64_t k0 = j.k_begin + kt * kBK;
  const T sgn = conj ? T(-1) : T(1);

#pragma unroll
  for (int it = 0; it < (kBR * kBK) / 256; ++it) {
    int q = threadIdx.x + 256 * it;
    int r, k;
    if (row_contig) { r = q % kBR; k = q / kBR; }
    else            { k = q % kBK; r = q / kBK; }
    int64_t rg = r0 + r, kg = k0 + k;
    T v[4] = {T(0), T(0), T(0), T(0)};
    if (rg < R && kg < k_end) {
      const T *src = row_contig ? X + 4 * (rg + kg * ldx) : X + 4 * (kg + rg * ldx);
      ldq(src, v);
      v[1] *= sgn; v[2] *= sgn; v[3] *= sgn;
    }
    T *d = tile + k * kPitch + r * 4;
    d[0] = v[0]; d[1] = v[1]; d[2] = v[2]; d[3] = v[3];
  }
  __syncthreads();
  T *o = out + bid * (int64_t)kChunkElems;
  // Walk the chunk linearly, 2 elements per step (16 B for double, 8 B for float).
  for (int w = threadIdx.x; w < kChunkElems / 2; w += 256) {
    // invert the layout for the element pair at offset 2w, 2w+1
    T pair[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      int off = 2 * w + e, r, k, c;
      static_assert(std::is_same<Layout, FragLayout>::value, "FP64 packs use the fragment layout");
      int ee = off & 1, lane = (off >> 1) & 31, pp = (off >> 6) & 1, i = (off >> 7) & 7, ks = off >> 10;
      r = i * 8 + (lane >> 2); k = ks * 4 + (lane & 3); c = pp * 2 + ee;
      pair[e] = tile[k * kPitch + r * 4 + c];
    }
    if constexpr (sizeof(T) == 8) {
      reinterpret_cast<double2 *>(o)[w] = make_double2(pair[0], pair[1]);
    } else {
      reinterpret_cast<float2 *>(o)[w] = make_float2(pair[0], pair[1]);
    }
  }
}

}  // namespace qg
