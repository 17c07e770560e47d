// qg_dmma.cuh -- FP64 mainloop on the FP64 tensor pipe (DMMA.8x8x4) with the
// alpha/beta epilogue fused (SURVEY.md §8(a) rows a4 "Mainloop" and a5 "Epilogue").
//
// PAPER.md: the micro-kernel of Alg. 3 accumulates a register
// block C_r as a sum of rank-1 updates over k (Eq. micro_kernel);
// the quaternion product of each update is the 16-FMA Hamilton rule
// (Eq. quaternion_prod; batch form Eqs. simd_batch_mul*).
//
// B200 form.  Component planes make the quaternion product a sum of 16 real
// matrix products per output tile (derived from P:274-309):
//     D^{p XOR s} += eps(p,s) * A^p * B^s,     p, s in {0,1,2,3},
// evaluated with mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4), which measured
// 37.0 TFLOP/s on B200 vs 33.8 for DFMA (tools/microbench/fp64_pipes.cu).
// The sign is applied by feeding -B^s (one sign flip per fragment, reused by
// every m8 tile of the warp), so each A^p/B^s fragment loaded from shared
// memory is reused across all four output components (north star).
//
// CTA: 64x64 output quaternions, 8 consumer warps (2 in m x 4 in n, each a
// 32x16 warp tile = 4x2 m8n8 tiles x 4 components = 64 f64 accumulators per
// lane) + a producer warpgroup, one lane of which fills a 3-stage shared-memory
// ring completing on mbarriers -- with TMA tensor-map loads of the user's
// interleaved tiles (the direct path, the default: kFeedTma128 4-quaternion
// groups or kFeedTma 32-byte tiles), de-interleaved by the consumers' fragment
// addresses, or with 1-D bulk copies of packed chunks (qg_pack.cuh FragLayout;
// SASS UBLKCP).  Epilogue: alpha (x) acc + beta (x) C, left products
// (P:493-500), masked at the M/N edges, each lane owning whole quaternions; in
// the direct kernels the C tile travels through the same ring by TMA
// (produce_c_stage).
//
// Schedule: persistent (one CTA per SM), "data-parallel + stream-K" hybrid.
// Whole tiles are dealt round-robin for every full wave; the remainder's
// k-iterations are split evenly over all CTAs (stream-K), so no SM idles in a
// partial last wave (c2: 256 tiles on 148 SMs).  A tile split
// across CTAs is finished by the CTA holding its k = 0 segment (the "owner"):
// the others park their partial accumulators in the workspace and bump the
// tile's arrival counter; the owner adds them and runs the epilogue (the host
// launches such grids cooperatively, so every CTA is resident).  The producer
// walks the same work list, so the ring keeps streaming across tile boundaries
// while the consumers run an epilogue.
#pragma once
#include <cuda.h>  // CUtensorMap (the TMA feed)
#include "qg_pack.cuh"

namespace qg {

#ifndef QG_DMMA_STAGES
#define QG_DMMA_STAGES 3
#endif
constexpr int kStages = QG_DMMA_STAGES;
constexpr int kConsumerWarps = 8;
constexpr int kConsumerThreads = kConsumerWarps * 32;
// 8 consumer warps + a producer warpgroup; setmaxnreg moves registers from the
// producer (40/thread) to the consumers (232/thread): 128*40 + 256*232 <= 64K.
constexpr int kDmmaThreads = (kConsumerWarps + 4) * 32;
constexpr int kProducerRegs = 40;
constexpr int kConsumerRegs = 232;
#ifndef QG_GROUP_M
#define QG_GROUP_M 8
#endif
#ifndef QG_RING_BETA0
#define QG_RING_BETA0 1  // beta == 0 tiles take the ring too (no C stage loads; the store warp TMA-stores the boxes)
#endif
#ifndef QG_C_RING
#define QG_C_RING 1  // epilogue C tiles through the ring by TMA (see produce_c_stage)
#endif
#ifndef QG_C_STORE_WARP
// 1: a producer-warpgroup warp issues the ring epilogue's TMA stores, waits for
// the TMA unit to read each box and hands the slot back to the producer, so the
// consumers go on to the next tile as soon as they have written their
// quaternions (no CTA-wide barriers, no wait for the store's reads); 0: consumer
// thread 0 stores behind two consumer barriers and all consumers wait for the reads
#define QG_C_STORE_WARP 1
#endif
#ifndef QG_C_PREFETCH_BULK
#define QG_C_PREFETCH_BULK 1  // 1: the producer lane bulk-prefetches C tiles; 0: consumer lanes prefetch per quaternion
#endif
#ifndef QG_C_PREFETCH_KT
#define QG_C_PREFETCH_KT 2  // k-tiles before the end of a tile at which its C tile is prefetched to L2
#endif
constexpr int kGroupM = QG_GROUP_M;  // rasterisation: M-tiles per group (L2 reuse of panels)
// ring + barriers + 1 KB so the ring can start on a 1024-byte boundary
// (barriers: full, empty and, for the ring epilogue's store warp, cdone per slot)
constexpr size_t kDmmaSmemBytes = size_t(kStages) * 2 * kChunkElems * sizeof(double) + 3 * kStages * 8 + 1024;

// How the ring is fed (kernel template parameter).
// (a third feed -- all 128 producer threads de-interleaving with 16-byte
// cp.async -- was measured 3% slower than packed at c3 and removed)
enum Feed : int {
  kFeedPacked = 0,  // bulk copies of pre-packed chunks (pack_kernel)
  kFeedTma = 2,     // TMA tensor-map tiles of the interleaved storage, 32-byte swizzle
  kFeedTma128 = 3,  // TMA tiles of 4-quaternion groups, 128-byte swizzle, permuted k (conflict-free)
};
constexpr int kAccPerThread = 64;                      // doubles
constexpr size_t kPartialBytes = size_t(kConsumerThreads) * kAccPerThread * sizeof(double);  // 128 KiB
constexpr int kMaxPersistentCTAs = 256;

// ---- optional phase trace (diagnostic builds only, -DQG_TRACE; read back with
// qgemm_debug_trace): consumer thread 0 of every CTA stamps %globaltimer at
// phase boundaries; event = (code << 56) | ns.  Codes: 1 consumers start,
// 2 unit start, 3 unit k-loop done, 4 stream-K fixup done (contributor parked /
// owner summed), 5 epilogue done, 6 consumers done, 7/8 per-lane epilogue C
// batch landed, 9 the unit's first stage landed.
#ifdef QG_TRACE
constexpr int kTraceEv = 48;
__device__ unsigned long long g_trace[256][kTraceEv];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// (the last slot always holds the final event, so long unit lists keep it)
#define QG_TR(code)                                                                                 \
  do {                                                                                              \
    if (threadIdx.x == 0 && (tr_n < kTraceEv - 1 || (code) == 6))                                   \
      g_trace[blockIdx.x][(code) == 6 ? kTraceEv - 1 : tr_n++] =                                    \
          ((unsigned long long)(code) << 56) | (gtimer() & ((1ull << 56) - 1));                     \
  } while (0)
// stamp once `dep` (a loaded value) is available: the asm takes it as an input
#define QG_TR_DEP(code, dep)                                                                        \
  do {                                                                                              \
    if (threadIdx.x == 0 && tr_n < kTraceEv - 1) {                                                  \
      unsigned long long t_;                                                                        \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_) : "d"(dep));                             \
      g_trace[blockIdx.x][tr_n++] = ((unsigned long long)(code) << 56) | (t_ & ((1ull << 56) - 1)); \
    }                                                                                               \
  } while (0)
#else
#define QG_TR(code) \
  do {              \
  } while (0)
#define QG_TR_DEP(code, dep) \
  do {                       \
  } while (0)
#endif

struct alignas(64) DmmaArgs {
  CUtensorMap tmA, tmB;  // TMA feed: 3-D maps (component, view row, k) or (component, k, view row)
  CUtensorMap tmC;       // QG_C_RING: C as (component, column, row), box 4 x 64 x 16, 32-byte swizzle
  int c_ring;            // host: C tiles through the ring for this launch (see launch_dmma)
  int c_remote;          // host: C is not in this GPU's memory (multi-GPU epilogue stores): no L2 prefetch of C
  int c_reduce;          // host: ring epilogue with beta == 1: boxes of alpha (x) acc added into C by TMA reductions
  const double *Ap;  // packed path: packed A panel, MT x KT chunks
  const double *Bp;  // packed path: packed B panel, NT x KT chunks
  // TMA feed: op(A) / op(B) read in place as R x K views -- X~(r, k) at
  // X + 4(r + k ldx) (rc = 1) or X + 4(k + r ldx) (rc = 0)
  const double *A, *B;
  int64_t lda, ldb, K;
  int a_rc, b_rc;
  double *C;
  int64_t ldc, M, N, MT, NT, KT;
  Scalars<double> sc;
  // persistent stream-K schedule
  int64_t T;          // tiles
  int64_t dp_tiles;   // tiles dealt whole, round-robin
  int64_t sk_iters;   // (T - dp_tiles) * KT k-iterations split over the grid
  double *partials;   // gridDim.x slots of kPartialBytes
  int *flags;         // T - dp_tiles arrival counters (zero on entry; owners reset them)
  int64_t grid;       // host side: CTAs launched
  int tri;            // 0: all tiles; 1/2: only tiles of the lower/upper triangle (QHERK)
};

__device__ __forceinline__ void tile_coords(int64_t pid, int64_t MT, int64_t NT, int64_t &mt, int64_t &nt) {
  const int64_t per_group = int64_t(kGroupM) * NT;
  const int64_t g = pid / per_group;
  const int64_t first_m = g * kGroupM;
  const int64_t gsz = (MT - first_m) < kGroupM ? (MT - first_m) : kGroupM;
  const int64_t in = pid - g * per_group;
  mt = first_m + in % gsz;
  nt = in / gsz;
}

// Tile t of the work list: full grid (grouped raster) or, for the triangular
// (QHERK) schedule, the lower triangle in bands of kGroupM tile rows, each band
// column by column (rows inner) like the grouped raster: band b (rows
// [8b, 8b + h), h <= 8) holds 8b*h tiles left of its diagonal block, then the
// h(h+1)/2 tiles of that block; bands start at t = 32 b^2 + 4 b (kGroupM = 8).
__device__ __forceinline__ void work_tile(const DmmaArgs &a, int64_t t, int64_t &mt, int64_t &nt) {
  if (a.tri == 0) {
    tile_coords(t, a.MT, a.NT, mt, nt);
    return;
  }
  constexpr int64_t G = kGroupM;
  auto band_start = [](int64_t b) { return (G * G / 2) * b * b + (G * (G + 1) / 2 - G * G / 2) * b; };
  int64_t b = int64_t((-double(G * (G + 1) / 2 - G * G / 2) +
                       sqrt(double(G * (G + 1) / 2 - G * G / 2) * double(G * (G + 1) / 2 - G * G / 2) +
                            2.0 * double(G * G) * double(t))) / double(G * G));
  while (b > 0 && band_start(b) > t) --b;
  while (band_start(b + 1) <= t) ++b;
  const int64_t r0 = G * b, h = (a.MT - r0) < G ? (a.MT - r0) : G;
  const int64_t u = t - band_start(b);
  int64_t r, c;
  if (u < r0 * h) {
    c = u / h;
    r = r0 + u % h;
  } else {  // diagonal block: column j has rows j..h-1
    int64_t v = u - r0 * h, j = 0;
    while (v >= h - j) { v -= h - j; ++j; }
    c = r0 + j;
    r = r0 + j + v;
  }
  if (a.tri == 1) { mt = r; nt = c; }
  else            { mt = c; nt = r; }
}

// Stream-K range of CTA c: [begin, end) in the SK iteration space.
struct SkSplit {
  int64_t per, extra;
  __device__ __forceinline__ int64_t begin(int64_t c) const { return c * per + (c < extra ? c : extra); }
  __device__ __forceinline__ int64_t end(int64_t c) const { return begin(c) + per + (c < extra ? 1 : 0); }
  __device__ __forceinline__ int64_t owner_of(int64_t i) const {  // CTA whose range holds iteration i
    const int64_t big = extra * (per + 1);
    if (i < big) return i / (per + 1);
    return extra + (i - big) / per;
  }
};

// One unit of work: k-tiles [kb, ke) of tile t.
struct Unit {
  int64_t t, kb, ke;
};

// Enumerate this CTA's units in order; returns false when exhausted.
struct WorkIter {
  int64_t next_dp, sk_i, sk_end;
  __device__ __forceinline__ bool next(const DmmaArgs &a, Unit &u) {
    if (next_dp < a.dp_tiles) {
      u.t = next_dp;
      u.kb = 0;
      u.ke = a.KT;
      next_dp += gridDim.x;
      return true;
    }
    if (sk_i < sk_end) {
      const int64_t lt = sk_i / a.KT;
      u.t = a.dp_tiles + lt;
      u.kb = sk_i - lt * a.KT;
      const int64_t tile_end = (lt + 1) * a.KT;
      const int64_t stop = sk_end < tile_end ? sk_end : tile_end;
      u.ke = u.kb + (stop - sk_i);
      sk_i = stop;
      return true;
    }
    return false;
  }
};

__device__ __forceinline__ WorkIter make_iter(const DmmaArgs &a, const SkSplit &sp) {
  WorkIter w;
  w.next_dp = blockIdx.x;
  w.sk_i = a.sk_iters ? sp.begin(blockIdx.x) : 0;
  w.sk_end = a.sk_iters ? sp.end(blockIdx.x) : 0;
  return w;
}

__device__ __forceinline__ void consumer_bar() {
  asm volatile("bar.sync 1, %0;\n" ::"n"(kConsumerThreads) : "memory");
}

__device__ __forceinline__ int ld_acquire(const int *p) {
  int v;
  asm volatile("ld.global.acquire.gpu.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// 3-D TMA tile load completing on an mbarrier (transaction bytes).
__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *tm, int c0, int c1, int c2,
                                            uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tm)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

// 3-D TMA tile store from shared memory (bulk-group completion).
__device__ __forceinline__ void tma_store_3d(const CUtensorMap *tm, const void *src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];\n" ::"l"(
                   reinterpret_cast<uint64_t>(tm)),
               "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(src))
               : "memory");
}

// 3-D TMA reduction from shared memory into global: dst += box, element-wise in
// the map's type (FP64 here), performed in L2 (bulk-group completion).
__device__ __forceinline__ void tma_reduce_add_3d(const CUtensorMap *tm, const void *src, int c0, int c1, int c2) {
  asm volatile("cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2, %3}], [%4];\n" ::"l"(
                   reinterpret_cast<uint64_t>(tm)),
               "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(src))
               : "memory");
}

// Producer cursor over the CTA's (unit, k-tile) sequence.
struct Producer {
  WorkIter it;
  int64_t kt, ke;
  int64_t mt, nt;  // TMA feed: tile coordinates of the current unit
  const double *a_src, *b_src;
  int slot;
  uint32_t phase;
  int64_t fills;
  int64_t c_pref_kt;  // k-tile at which to L2-prefetch the unit's C tile (-1: none)
  int c_left;         // QG_C_RING: C stages still to issue for the current unit
  bool c_load;        // ... and whether they load C (beta != 0)
};

// ---- C through the ring (QG_C_RING): a unit that runs the epilogue is
// followed in the ring by two C stages -- batch h = rows 16h.. and 32 + 16h..
// of the 64 x 64 tile, one 32 KB TMA box each ([row 16][col 64][4 comps],
// 32-byte swizzle) into the slot's A and B halves, i.e. the quaternions consumer
// half wm of batch h owns.  The consumers read C from shared memory, write the
// results back in place and one thread TMA-stores the boxes (the TMA unit clips
// the M / N edges): the epilogue's global traffic runs at TMA rates instead of
// 128-bit per-lane loads and stores with 64 KB in flight per batch.
// Without a C read (beta = 0) the C stages load nothing and the consumers
// overwrite the boxes whole (QG_RING_BETA0; with the store warp this beats the
// per-lane stores); with a real beta == 1 they load nothing either
// and the store warp adds the boxes into C by TMA reductions (QG_C_REDUCE).
// QHERK's off-diagonal tiles lie wholly inside its triangle; its diagonal tiles
// never take the ring.
constexpr uint32_t kCBoxBytes = 16u * 64u * 32u;  // 32 KB = one slot half
__device__ __forceinline__ void produce_c_stage(Producer &p, const DmmaArgs &args, double *sA, double *sB,
                                                uint64_t *full, uint64_t *empty) {
  const int h = 2 - p.c_left;
  if (p.fills >= kStages) mbar_wait(&empty[p.slot], p.phase ^ 1u);
  if (p.c_load) {
    mbar_arrive_expect_tx(&full[p.slot], 2 * kCBoxBytes);
    const int n0 = int(p.nt * kBR), r0 = int(p.mt * kBR) + 16 * h;
    tma_load_3d(sA + p.slot * kChunkElems, &args.tmC, 0, n0, r0, &full[p.slot]);
    tma_load_3d(sB + p.slot * kChunkElems, &args.tmC, 0, n0, r0 + 32, &full[p.slot]);
  } else {  // beta = 0 (QHERK off-diagonal tile): the box is overwritten whole
    mbar_arrive(&full[p.slot]);
  }
  if (++p.slot == kStages) { p.slot = 0; p.phase ^= 1u; }
  --p.c_left;
  ++p.fills;
}
// Whether a tile's epilogue takes the ring: beta != 0 or QHERK, except QHERK's
// diagonal tiles -- a TMA store writes the whole box back, so the strict other
// triangle (which qherk must never touch, qgemm.h) would be rewritten with the
// values loaded earlier, losing a concurrent writer's update; those few tiles
// (MT of MT(MT+1)/2) take the per-lane masked store epilogue instead.
__device__ __forceinline__ bool ring_epilogue(const DmmaArgs &a, int64_t mt, int64_t nt) {
  return a.c_ring && (!a.sc.beta_zero || a.tri != 0 || QG_RING_BETA0) && !(a.tri != 0 && mt == nt);
}
template <bool kRing>
__device__ __forceinline__ void producer_unit_c(Producer &p, const DmmaArgs &a, const Unit &u) {
  p.c_load = !a.sc.beta_zero && !a.c_reduce;  // (c_reduce: C is read by the TMA reduction, in L2)
  p.c_left = (kRing && u.kb == 0 && ring_epilogue(a, p.mt, p.nt)) ? 2 : 0;
}

// L2 prefetch of the C tile (mt, nt) by the TMA engine: one bulk prefetch per
// column (up to 64 quaternions = 2 KB contiguous).  Issued by the producer lane
// QG_C_PREFETCH_KT k-tiles before a unit that runs the epilogue ends.
__device__ __forceinline__ void prefetch_c_tile(const DmmaArgs &a, int64_t mt, int64_t nt) {
  const int64_t r0 = mt * kBR, c0 = nt * kBR;
  const int64_t rows = (a.M - r0) < kBR ? (a.M - r0) : kBR;
  const int64_t cols = (a.N - c0) < kBR ? (a.N - c0) : kBR;
  const uint32_t bytes = uint32_t(rows) * 32u;
  for (int64_t j = 0; j < cols; ++j) {
    const double *p = a.C + 4 * (r0 + (c0 + j) * a.ldc);
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(p), "r"(bytes) : "memory");
  }
}
template <bool kRing>
__device__ __forceinline__ void producer_unit_prefetch(Producer &p, const DmmaArgs &a, const Unit &u) {
  p.c_pref_kt = (!(kRing && a.c_ring) && !a.c_remote && QG_C_PREFETCH_BULK && QG_C_PREFETCH_KT > 0 && u.kb == 0 &&
                 !a.sc.beta_zero)
                    ? (u.ke - QG_C_PREFETCH_KT > u.kb ? u.ke - QG_C_PREFETCH_KT : u.kb)
                    : int64_t(-1);
}

// Issue the next fill (bulk copies of one A and one B chunk); false when done.
__device__ __forceinline__ bool produce_next(Producer &p, const DmmaArgs &args, double *sA, double *sB,
                                             uint64_t *full, uint64_t *empty) {
  constexpr uint32_t kBytes = kChunkElems * sizeof(double);
  while (p.kt >= p.ke) {
    Unit u;
    if (!p.it.next(args, u)) return false;
    work_tile(args, u.t, p.mt, p.nt);
    p.a_src = args.Ap + p.mt * args.KT * kChunkElems;
    p.b_src = args.Bp + p.nt * args.KT * kChunkElems;
    p.kt = u.kb;
    p.ke = u.ke;
    producer_unit_prefetch<false>(p, args, u);
  }
  if (p.kt == p.c_pref_kt) prefetch_c_tile(args, p.mt, p.nt);
  if (p.fills >= kStages) mbar_wait(&empty[p.slot], p.phase ^ 1u);
  mbar_arrive_expect_tx(&full[p.slot], 2 * kBytes);
  bulk_g2s(sA + p.slot * kChunkElems, p.a_src + p.kt * kChunkElems, kBytes, &full[p.slot]);
  bulk_g2s(sB + p.slot * kChunkElems, p.b_src + p.kt * kChunkElems, kBytes, &full[p.slot]);
  if (++p.slot == kStages) { p.slot = 0; p.phase ^= 1u; }
  ++p.kt;
  ++p.fills;
  return true;
}

// ---- TMA feed: one lane loads each operand tile straight from the user's
// interleaved storage with a 3-D tensor map (component, row, k) or (component,
// k, row); out-of-range rows / k are zero-filled by the TMA unit (the padding
// of Alg. 2).  The tile lands in smem in storage order, 32-byte
// swizzled (one quaternion = one 32-byte swizzle row; the 128-byte mode would
// pad every 32-byte row to 128 bytes): element (r, k, c) of the 64 x 16 tile at
//   lin = ((k*64 + r)*4 + c)*8   (rows contiguous)   or   ((r*16 + k)*4 + c)*8
//   swz = lin ^ (((lin >> 7) & 1) << 4)   (16-byte half swapped on odd 128 B)
// so the de-interleave into DMMA fragments is done by the consumers' addresses
// (layout verified element by element by tools/microbench/tma_probe.cu).  A
// 128-bit shared load is served a quarter-warp (8 lanes = 2 rows x 4 k) at a
// time, and those 8 lanes hit only 2 bank groups when rows are contiguous
// (4-way conflicts; ncu) or 4 when k is contiguous (2-way) -- the price of not
// packing, which auto pays only where the sweep shows it wins.

template <bool kG4>
__device__ __forceinline__ bool produce_next_tma(Producer &p, const DmmaArgs &args, double *sA, double *sB,
                                                 uint64_t *full, uint64_t *empty) {
  constexpr uint32_t kBytes = kChunkElems * sizeof(double);
  while (p.kt >= p.ke && p.c_left == 0) {
    Unit u;
    if (!p.it.next(args, u)) return false;
    work_tile(args, u.t, p.mt, p.nt);
    p.kt = u.kb;
    p.ke = u.ke;
    producer_unit_prefetch<QG_C_RING>(p, args, u);
    producer_unit_c<QG_C_RING>(p, args, u);
  }
  if (p.kt >= p.ke) {
    produce_c_stage(p, args, sA, sB, full, empty);
    return true;
  }
  if (p.kt == p.c_pref_kt) prefetch_c_tile(args, p.mt, p.nt);
  if (p.fills >= kStages) mbar_wait(&empty[p.slot], p.phase ^ 1u);
  mbar_arrive_expect_tx(&full[p.slot], 2 * kBytes);
  const int k0 = int(p.kt * kBK), ra = int(p.mt * kBR), rb = int(p.nt * kBR);
  if constexpr (kG4) {  // group maps (16 doubles, k, row/4) or (16 doubles, k/4, row)
    if (args.a_rc) tma_load_3d(sA + p.slot * kChunkElems, &args.tmA, 0, k0, ra / 4, &full[p.slot]);
    else           tma_load_3d(sA + p.slot * kChunkElems, &args.tmA, 0, k0 / 4, ra, &full[p.slot]);
    if (args.b_rc) tma_load_3d(sB + p.slot * kChunkElems, &args.tmB, 0, k0, rb / 4, &full[p.slot]);
    else           tma_load_3d(sB + p.slot * kChunkElems, &args.tmB, 0, k0 / 4, rb, &full[p.slot]);
  } else {
    if (args.a_rc) tma_load_3d(sA + p.slot * kChunkElems, &args.tmA, 0, ra, k0, &full[p.slot]);
    else           tma_load_3d(sA + p.slot * kChunkElems, &args.tmA, 0, k0, ra, &full[p.slot]);
    if (args.b_rc) tma_load_3d(sB + p.slot * kChunkElems, &args.tmB, 0, rb, k0, &full[p.slot]);
    else           tma_load_3d(sB + p.slot * kChunkElems, &args.tmB, 0, k0, rb, &full[p.slot]);
  }
  if (++p.slot == kStages) { p.slot = 0; p.phase ^= 1u; }
  ++p.kt;
  ++p.fills;
  return true;
}

__device__ __forceinline__ void mbar_arrive_n(uint64_t *bar, uint32_t n) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(n) : "memory");
}
// QG_C_STORE_WARP: the ring epilogue's stores.  This lane walks the CTA's work
// list like the producer, tracking the ring slot (a unit of k-tiles [kb, ke)
// occupies ke - kb fills, then two C stages if it runs the ring epilogue); per
// C stage it waits until all consumer warps have written their quaternions
// (cdone), TMA-stores the two boxes, waits until the TMA unit has read them and
// returns the slot to the producer (one arrival counting for every consumer
// warp).  Its bulk-store groups are completed before the CTA exits.
__device__ __forceinline__ void c_store_loop(const DmmaArgs &args, const SkSplit &sp, double *sA, double *sB,
                                             uint64_t *empty, uint64_t *cdone) {
  WorkIter it = make_iter(args, sp);
  Unit u;
  int slot = 0;
  uint32_t cph = 0;  // parity of each slot's cdone barrier
  while (it.next(args, u)) {
    slot = int((int64_t(slot) + (u.ke - u.kb)) % kStages);
    if (u.kb != 0) continue;  // stream-K contributor: no epilogue here
    int64_t mt, nt;
    work_tile(args, u.t, mt, nt);
    if (!ring_epilogue(args, mt, nt)) continue;
#pragma unroll 1
    for (int h = 0; h < 2; ++h) {
      mbar_wait(&cdone[slot], (cph >> slot) & 1u);
      cph ^= 1u << slot;
      const int n0 = int(nt * kBR), r0 = int(mt * kBR) + 16 * h;
      if (args.c_reduce) {  // C += box (beta == 1): the add happens in L2
        tma_reduce_add_3d(&args.tmC, sA + slot * kChunkElems, 0, n0, r0);
        tma_reduce_add_3d(&args.tmC, sB + slot * kChunkElems, 0, n0, r0 + 32);
      } else {
        tma_store_3d(&args.tmC, sA + slot * kChunkElems, 0, n0, r0);
        tma_store_3d(&args.tmC, sB + slot * kChunkElems, 0, n0, r0 + 32);
      }
      asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
      mbar_arrive_n(&empty[slot], kConsumerWarps);
      if (++slot == kStages) slot = 0;
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}

// Byte offset of the 16-byte pair (components 2pp, 2pp+1) of (r, k) in a TMA tile.
__device__ __forceinline__ uint32_t tma_tile_off(int rc, int r, int k, int pp) {
  const uint32_t lin = rc ? uint32_t(((k * kBR + r) * 4 + 2 * pp) * 8) : uint32_t(((r * kBK + k) * 4 + 2 * pp) * 8);
  return lin ^ (((lin >> 7) & 1u) << 4);
}

// Per-lane part of the fragment offsets in a TMA tile.  A lane reads rows
// r0 + 8i (r0 = its first row) at k = 4ks + kl.  Rows contiguous: the swizzle
// bit (address bit 7) is bit 2 of the row, the same for every i, so
//   off = r0*32 + kl*2048 + ks*8192 + i*256 + ((16 pp) ^ x),   x = 16 * bit2(r0);
// k contiguous: the swizzle bit is bit 2 of k = bit 0 of ks, so
//   off = r0*512 + kl*32 + i*4096 + ks*128 + 16 (pp ^ (ks & 1)).
// Everything but `base` / `x` is a compile-time constant of the unrolled loops.
struct TmaLane {
  uint32_t base, x;
  int rc;
};
__device__ __forceinline__ TmaLane tma_lane(int rc, int r0, int kl) {
  TmaLane t;
  t.rc = rc;
  t.base = rc ? uint32_t(r0 * 32 + kl * 2048) : uint32_t(r0 * 512 + kl * 32);
  t.x = rc ? uint32_t(((r0 >> 2) & 1) << 4) : 0u;
  return t;
}
__device__ __forceinline__ uint32_t tma_frag_off(const TmaLane &t, int ks, int i, int pp) {
  return t.rc ? t.base + uint32_t(ks * 8192 + i * 256) + (uint32_t(pp << 4) ^ t.x)
              : t.base + uint32_t(i * 4096 + ks * 128 + ((pp ^ (ks & 1)) << 4));
}

// ---- kFeedTma128: both operands as tiles of 4-quaternion groups.  The map's
// inner dimension is 16 doubles = 4 consecutive quaternions along the
// operand's contiguous index = one 128-byte row of the 128-byte swizzle (no
// padding); the outer dimensions are the other index and the group index
// (layouts checked element by element by tools/microbench/tma_probe_g4.cu):
//   rows contiguous: smem [r/4][k][r%4][c]   lin = ((r>>2)*16 + k)*128 + (r&3)*32 + 8c
//   k contiguous:    smem [r][k/4][k%4][c]   lin = (r*4 + (k>>2))*128 + (k&3)*32 + 8c
//   swz = lin ^ (((lin >> 7) & 7) << 4)      (16-byte chunk ^= 128-byte row & 7)
// A quarter-warp's 128-bit loads cover fragment rows rho, rho+1 (rho even) x
// the 4 k of a k4 step.  In the natural k order those 4 k XOR the chunks with
// {0,1,2,3} (rows contiguous) or sit in one 128-byte row (k contiguous), and
// the two rows collide.  This kernel therefore feeds k4 step ks with tile k =
// kperm(ks, kl) = 8(ks>>1) + 2(ks&1) + kk, kk = (kl&1) + 4(kl>>1) in {0,1,4,5}
// -- a bijection of the tile's 16 k applied to A and B alike, so the k-sum is
// unchanged -- and the 8 lanes hit 8 distinct bank groups in both layouts
// (rows contiguous: chunks 2q ^ kk, q = rho & 3 in {0,1} or {2,3}; k
// contiguous: the 4 k span two 128-byte rows and rho & 1 flips chunk bit 2).
// (Permuting rows instead needs the permutation in the epilogue: measured
// slower at c4.)  The host takes this feed when the group extents are whole:
// M (N) % 4 == 0 for a rows-contiguous op(A) (op(B)), K % 4 == 0 for a
// k-contiguous one; otherwise kFeedTma.
struct G4Lane {
  uint32_t base, x;
};
// rb: first row of the warp's fragments (a multiple of 8); rho = lane / 4, kl = lane % 4
__device__ __forceinline__ G4Lane g4_lane(int rc, int rb, int rho, int kl) {
  const int kk = (kl & 1) + 4 * (kl >> 1);
  G4Lane t;
  if (rc) {  // chunk = (2q + pp) ^ (k & 7), k & 7 = 2(ks & 1) + kk
    t.base = uint32_t(((rb >> 2) + (rho >> 2)) * 2048 + kk * 128);
    t.x = uint32_t(((2 * (rho & 3)) ^ kk) << 4);
  } else {   // k = 4h + q: h = 2(ks >> 1) + (kl >> 1), q = 2(ks & 1) + (kl & 1);
             // chunk = (2q + pp) ^ (4(rho & 1) + (h & 3))
    t.base = uint32_t((rb + rho) * 512 + (kl >> 1) * 128);
    t.x = uint32_t((2 * (kl & 1) ^ 4 * (rho & 1) ^ (kl >> 1)) << 4);
  }
  return t;
}
// Byte offset of the 16-byte pair (components 2pp, 2pp+1) of fragment i
// (rows rb + 8i + rho) at k = kperm(ks, kl); rc is a compile-time constant.
__device__ __forceinline__ uint32_t g4_frag_off(int rc, const G4Lane &t, int ks, int i, int pp) {
  return rc ? t.base + uint32_t(i * 4096 + (8 * (ks >> 1) + 2 * (ks & 1)) * 128) +
                  (t.x ^ uint32_t((pp ^ (2 * (ks & 1))) << 4))
            : t.base + uint32_t(i * 4096 + (ks >> 1) * 256) +
                  (t.x ^ uint32_t((4 * (ks & 1) ^ 2 * ((ks >> 1) & 1) ^ pp) << 4));
}

// kFeed: kFeedPacked (conj applied by the pack kernel; CA = CB = false), or a
// direct feed reading op(A)/op(B) in place (CA / CB: op H on
// A / B, folded into the sign of each of the 16 products: conj flips the sign
// of components 1-3); otherwise from packed chunks (conj applied by
// the pack kernel; CA = CB = false).
// kRC (TMA feed only): bit 0 = op(A) rows contiguous, bit 1 = op(B) rows
// contiguous -- compile-time, so the fragment offsets fold into immediates.
template <int kFeed, bool CA, bool CB, int kRC = 0>
__global__ void __launch_bounds__(kDmmaThreads, 1) qgemm_dmma_kernel(const __grid_constant__ DmmaArgs args) {
  // C tiles through the ring only in the direct-feed instantiations: it speeds
  // up c2 (direct, 1.3%) but slowed the packed kernel at c3 / c4 (A/B in one run,
  // DESIGN.md §6) -- and code it does not use changed the packed kernel's code
  constexpr bool kRing = QG_C_RING && kFeed != kFeedPacked;
  extern __shared__ __align__(128) unsigned char smem_dyn[];
  // (offset arithmetic on the shared array, not an integer round trip, so the
  // compiler keeps shared-space loads: LDS, not generic LD)
  unsigned char *smem_raw = smem_dyn + ((1024u - (smem_u32(smem_dyn) & 1023u)) & 1023u);
  double *sA = reinterpret_cast<double *>(smem_raw);
  double *sB = sA + kStages * kChunkElems;
  uint64_t *full = reinterpret_cast<uint64_t *>(sB + kStages * kChunkElems);
  uint64_t *empty = full + kStages;
  uint64_t *cdone = empty + kStages;  // QG_C_STORE_WARP: consumers wrote a C stage (ring epilogue)

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t KT = args.KT;
  SkSplit sp;
  sp.per = args.sk_iters / gridDim.x;
  sp.extra = args.sk_iters - sp.per * gridDim.x;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
      mbar_init(&cdone[s], kConsumerWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();

  // ---------------- producer warpgroup, kStages fills ahead ----------------
  // One lane streams packed chunks (bulk copies) or interleaved tiles (TMA);
  // setmaxnreg hands the warpgroup's registers to the consumers.
  Producer prod;
  prod.it = make_iter(args, sp);
  prod.kt = 0;
  prod.ke = 0;
  prod.slot = 0;
  prod.phase = 0;
  prod.fills = 0;
  prod.c_pref_kt = -1;
  prod.c_left = 0;
  prod.c_load = false;
  prod.mt = prod.nt = 0;
  if (warp >= kConsumerWarps) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(kProducerRegs));
    if constexpr (kFeed == kFeedTma || kFeed == kFeedTma128) {
      if (warp == kConsumerWarps && lane == 0)
        while (produce_next_tma<kFeed == kFeedTma128>(prod, args, sA, sB, full, empty)) {
        }
      if (kRing && QG_C_STORE_WARP && args.c_ring && warp == kConsumerWarps + 1 && lane == 0)
        c_store_loop(args, sp, sA, sB, empty, cdone);
    } else {
      if (warp == kConsumerWarps && lane == 0)
        while (produce_next(prod, args, sA, sB, full, empty)) {
        }
    }
    return;
  }
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(kConsumerRegs));

  // ---------------- consumers ----------------
  const int wm = warp & 1;   // 32-row half of the CTA tile
  const int wn = warp >> 1;  // 16-column quarter
  [[maybe_unused]] const TmaLane ta = tma_lane(kRC & 1, wm * 32 + (lane >> 2), lane & 3);
  [[maybe_unused]] const TmaLane tb = tma_lane((kRC >> 1) & 1, wn * 16 + (lane >> 2), lane & 3);
  [[maybe_unused]] const G4Lane ga = g4_lane(kRC & 1, wm * 32, lane >> 2, lane & 3);
  [[maybe_unused]] const G4Lane gb = g4_lane((kRC >> 1) & 1, wn * 16, lane >> 2, lane & 3);
  const int tid = threadIdx.x;
  int slot = 0;
  uint32_t phase = 0;
  WorkIter it = make_iter(args, sp);
  Unit u;
  [[maybe_unused]] int tr_n = 0;
  QG_TR(1);
  while (it.next(args, u)) {
    QG_TR(2);
    double acc[4][2][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[i][j][c][0] = acc[i][j][c][1] = 0.0;

    // k-tile at which to warm L2 with this unit's C tile (beta != 0, epilogue here)
    const int64_t kt_prefetch = (!(kRing && args.c_ring) && !args.c_remote && !QG_C_PREFETCH_BULK &&
                                 QG_C_PREFETCH_KT > 0 && u.kb == 0 &&
                                 !args.sc.beta_zero)
                                    ? (u.ke - QG_C_PREFETCH_KT > u.kb ? u.ke - QG_C_PREFETCH_KT : u.kb)
                                    : int64_t(-1);
    for (int64_t kt = u.kb; kt < u.ke; ++kt) {
      if (kt == kt_prefetch) {
        int64_t pmt, pnt;
        work_tile(args, u.t, pmt, pnt);
#pragma unroll
        for (int ii = 0; ii < 4; ++ii)
#pragma unroll
          for (int jj = 0; jj < 2; ++jj)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int64_t row = pmt * kBR + (wm * 4 + ii) * 8 + (lane >> 2);
              const int64_t col = pnt * kBR + (wn * 2 + jj) * 8 + 2 * (lane & 3) + e;
              if (row < args.M && col < args.N)
                asm volatile("prefetch.global.L2 [%0];\n" ::"l"(args.C + 4 * (row + col * args.ldc)));
            }
      }
      mbar_wait(&full[slot], phase);
      if (kt == u.kb) QG_TR(9);  // the unit's first stage has landed
      const double2 *a2 = reinterpret_cast<const double2 *>(sA + slot * kChunkElems);
      const double2 *b2 = reinterpret_cast<const double2 *>(sB + slot * kChunkElems);
      [[maybe_unused]] const unsigned char *a8 = reinterpret_cast<const unsigned char *>(a2);
      [[maybe_unused]] const unsigned char *b8 = reinterpret_cast<const unsigned char *>(b2);
#pragma unroll
      for (int ks = 0; ks < kBK / 4; ++ks) {
        double af[4][4], bf[2][4], bn[2][4];
#pragma unroll
        for (int ii = 0; ii < 4; ++ii)
#pragma unroll
          for (int pp = 0; pp < 2; ++pp) {
            double2 v;
            if constexpr (kFeed == kFeedTma)
              v = *reinterpret_cast<const double2 *>(a8 + tma_frag_off(ta, ks, ii, pp));
            else if constexpr (kFeed == kFeedTma128)
              v = *reinterpret_cast<const double2 *>(a8 + g4_frag_off(kRC & 1, ga, ks, ii, pp));
            else
              v = a2[((ks * 8 + wm * 4 + ii) * 2 + pp) * 32 + lane];
            af[ii][2 * pp] = v.x;
            af[ii][2 * pp + 1] = v.y;
          }
#pragma unroll
        for (int jj = 0; jj < 2; ++jj)
#pragma unroll
          for (int pp = 0; pp < 2; ++pp) {
            double2 v;
            if constexpr (kFeed == kFeedTma)
              v = *reinterpret_cast<const double2 *>(b8 + tma_frag_off(tb, ks, jj, pp));
            else if constexpr (kFeed == kFeedTma128)
              v = *reinterpret_cast<const double2 *>(b8 + g4_frag_off((kRC >> 1) & 1, gb, ks, jj, pp));
            else
              v = b2[((ks * 8 + wn * 2 + jj) * 2 + pp) * 32 + lane];
            bf[jj][2 * pp] = v.x;
            bf[jj][2 * pp + 1] = v.y;
          }
#pragma unroll
        for (int jj = 0; jj < 2; ++jj)
#pragma unroll
          for (int s = 0; s < 4; ++s) bn[jj][s] = -bf[jj][s];

        // 16 DMMA per (m8, n8) tile; p outermost so consecutive DMMAs hit
        // different accumulators.
#pragma unroll
        for (int p = 0; p < 4; ++p)
#pragma unroll
          for (int ii = 0; ii < 4; ++ii)
#pragma unroll
            for (int jj = 0; jj < 2; ++jj)
#pragma unroll
              for (int c = 0; c < 4; ++c) {
                const int s = p ^ c;
                const bool neg = hneg(p, s) ^ (CA && p != 0) ^ (CB && s != 0);
                dmma_8x8x4(acc[ii][jj][c], af[ii][p], neg ? bn[jj][s] : bf[jj][s]);
              }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
      if (++slot == kStages) { slot = 0; phase ^= 1u; }
    }

    QG_TR(3);
    const bool whole = (u.kb == 0 && u.ke == KT);
    if (!whole) {
      // stream-K fixup (only tiles >= dp_tiles are ever split)
      const int64_t lt = u.t - args.dp_tiles;
      double2 *mine = reinterpret_cast<double2 *>(args.partials + size_t(blockIdx.x) * (kPartialBytes / 8));
      if (u.kb != 0) {
        // contributor: park the partial sums, then signal the owner
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int c = 0; c < 4; ++c)
              __stcg(&mine[((i * 2 + j) * 4 + c) * kConsumerThreads + tid],
                     make_double2(acc[i][j][c][0], acc[i][j][c][1]));
        __threadfence();
        consumer_bar();
        if (tid == 0) atomicAdd(&args.flags[lt], 1);
        QG_TR(4);
        continue;
      }
      // owner: wait for every other CTA holding a piece of this tile, add their partials
      const int64_t first = lt * KT;
      const int64_t c_last = sp.owner_of(first + KT - 1);
      const int expected = int(c_last - blockIdx.x);
      if (tid == 0) {
        // contributors are co-resident (grid <= resident CTAs) and never wait
        // on anything, so this terminates; the trap turns a broken schedule
        // into a launch error instead of a hung GPU.
        uint32_t spins = 0;
        while (ld_acquire(&args.flags[lt]) < expected) {
          __nanosleep(100);
          if (++spins == (1u << 27)) __trap();
        }
        args.flags[lt] = 0;  // ready for the next call
      }
      consumer_bar();
      for (int64_t src = blockIdx.x + 1; src <= c_last; ++src) {
        const double2 *p = reinterpret_cast<const double2 *>(args.partials + size_t(src) * (kPartialBytes / 8));
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              const double2 v = __ldcg(&p[((i * 2 + j) * 4 + c) * kConsumerThreads + tid]);
              acc[i][j][c][0] += v.x;
              acc[i][j][c][1] += v.y;
            }
      }
    }

    QG_TR(4);
    // ---------------- epilogue ----------------
    // D fragment of m8n8k4: lane holds D[lane/4][2*(lane%4) + e], e = 0, 1.
    int64_t mt, nt;
    work_tile(args, u.t, mt, nt);
    // (beta = 0 outside QHERK: no C read -- the plain store path below is faster;
    // QHERK's diagonal tiles: masked per-lane stores, see ring_epilogue)
    if (kRing && ring_epilogue(args, mt, nt)) {
      // C tile through the ring (produce_c_stage): read, update in place, TMA store.
      int slots[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        slots[h] = slot;
        mbar_wait(&full[slot], phase);
        unsigned char *box = reinterpret_cast<unsigned char *>((wm ? sB : sA) + slot * kChunkElems);
#pragma unroll
        for (int i2 = 0; i2 < 2; ++i2)
#pragma unroll
          for (int jj = 0; jj < 2; ++jj)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int ii = 2 * h + i2;
              const int rl = i2 * 8 + (lane >> 2);                    // row in the 16-row box
              const int cl = (wn * 2 + jj) * 8 + 2 * (lane & 3) + e;  // column in the tile
              const uint32_t lin = uint32_t(rl * 64 + cl) * 32u;
              double2 *q0 = reinterpret_cast<double2 *>(box + (lin ^ (((lin >> 7) & 1u) << 4)));
              double2 *q1 = reinterpret_cast<double2 *>(box + ((lin + 16u) ^ ((((lin + 16u) >> 7) & 1u) << 4)));
              const double q[4] = {acc[ii][jj][0][e], acc[ii][jj][1][e], acc[ii][jj][2][e], acc[ii][jj][3][e]};
              double out[4];
              left_scale(args.sc.alpha, args.sc.alpha_real, q, out);
              if (!args.sc.beta_zero && !args.c_reduce) {
                const double2 c01 = *q0, c23 = *q1;
                const double cold[4] = {c01.x, c01.y, c23.x, c23.y};
                double bc[4];
                left_scale(args.sc.beta, args.sc.beta_real, cold, bc);
#pragma unroll
                for (int k = 0; k < 4; ++k) out[k] += bc[k];
              }
              *q0 = make_double2(out[0], out[1]);
              *q1 = make_double2(out[2], out[3]);
            }
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // smem writes -> TMA store
        if (QG_C_STORE_WARP) {  // the store warp takes it from here (c_store_loop)
          __syncwarp();
          if (lane == 0) mbar_arrive(&cdone[slot]);
          if (++slot == kStages) { slot = 0; phase ^= 1u; }
          continue;
        }
        consumer_bar();
        if (tid == 0) {
          const int n0 = int(nt * kBR), r0 = int(mt * kBR) + 16 * h;
          tma_store_3d(&args.tmC, sA + slot * kChunkElems, 0, n0, r0);
          tma_store_3d(&args.tmC, sB + slot * kChunkElems, 0, n0, r0 + 32);
          asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
        }
        if (++slot == kStages) { slot = 0; phase ^= 1u; }
      }
      if (QG_C_STORE_WARP) {
        QG_TR(5);
        continue;
      }
      // the slots return to the producer once the TMA unit has read them
      if (tid == 0) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
      consumer_bar();
      if (lane == 0) {
        mbar_arrive(&empty[slots[0]]);
        mbar_arrive(&empty[slots[1]]);
      }
      QG_TR(5);
      continue;
    }
    // Two batches of 8 quaternions: all C loads of a batch are issued before
    // any store, so the 8 round trips overlap (the compiler cannot reorder
    // loads of C above stores to C on its own).
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      double cold[2][2][2][4];
      bool ok[2][2][2];
      double *cp[2][2][2];
#pragma unroll
      for (int i2 = 0; i2 < 2; ++i2)
#pragma unroll
        for (int jj = 0; jj < 2; ++jj)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int ii = 2 * h + i2;
            const int64_t row = mt * kBR + (wm * 4 + ii) * 8 + (lane >> 2);
            const int64_t col = nt * kBR + (wn * 2 + jj) * 8 + 2 * (lane & 3) + e;
            ok[i2][jj][e] = row < args.M && col < args.N &&
                            (args.tri == 0 || (args.tri == 1 ? row >= col : row <= col));
            cp[i2][jj][e] = args.C + 4 * (row + col * args.ldc);
            if (!args.sc.beta_zero && ok[i2][jj][e]) ldq_c(cp[i2][jj][e], cold[i2][jj][e]);
          }
      QG_TR_DEP(7 + h, cold[0][0][0][0]);  // batch h's first C load has landed
#pragma unroll
      for (int i2 = 0; i2 < 2; ++i2)
#pragma unroll
        for (int jj = 0; jj < 2; ++jj)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            if (!ok[i2][jj][e]) continue;
            const int ii = 2 * h + i2;
            const double q[4] = {acc[ii][jj][0][e], acc[ii][jj][1][e], acc[ii][jj][2][e], acc[ii][jj][3][e]};
            double out[4];
            left_scale(args.sc.alpha, args.sc.alpha_real, q, out);
            if (!args.sc.beta_zero) {
              double bc[4];
              left_scale(args.sc.beta, args.sc.beta_real, cold[i2][jj][e], bc);
#pragma unroll
              for (int k = 0; k < 4; ++k) out[k] += bc[k];
            }
            if (args.tri != 0) {
              // QHERK: the diagonal of a Hermitian matrix is real (R18)
              const int64_t row = mt * kBR + (wm * 4 + 2 * h + i2) * 8 + (lane >> 2);
              const int64_t col = nt * kBR + (wn * 2 + jj) * 8 + 2 * (lane & 3) + e;
              if (row == col) out[1] = out[2] = out[3] = 0.0;
            }
            stq(cp[i2][jj][e], out);
          }
    }
    QG_TR(5);
  }
  if (kRing && args.c_ring && tid == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
  // Per-lane C stores may target another GPU's memory (the multi-GPU driver's
  // epilogue stores into root's C over NVLink, dist.qgemm_rowsharded_p2p):
  // make them visible at system scope before this CTA retires, so whatever the
  // rank signals next (the completion all_reduce) is ordered after them.
  if (!(kRing && args.c_ring)) asm volatile("fence.acq_rel.sys;\n" ::: "memory");
  QG_TR(6);
}

}  // namespace qg
