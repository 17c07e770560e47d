// qg_runtime.cuh -- host-side runtime of libqgemm.so (internal; included once, by
// qgemm_api.cu, inside its anonymous namespace -- one translation unit).
//
// SURVEY.md §8(a) row a1 "Plan / validate": per-thread launch counting and the
// optional CUDA-event timing of every launch, BLAS-style argument validation,
// packed-operand geometry and workspace sizing, the persistent-grid schedule,
// the path policy (packed / direct / one-launch small kernel) and one launcher
// per kernel.
#pragma once

thread_local int g_last_launches = 0;

// ---- path choice: packed (pack launch + persistent mainloop), direct (FP64:
// the persistent mainloop fed by TMA from the interleaved storage, no pack) or
// the one-launch small kernel.  0 = auto, 1 = always packed, 2 = small kernel
// whenever the call reads A and B, 3 = direct for FP64 (packed for FP32), 4 =
// direct with the 32-byte-swizzle tiles only (never kFeedTma128), 5 = small
// kernel, general variant only (never the tile-exact one) --
// qgemm_set_path_policy; the tests run every shape under each.
std::atomic<int> g_path_policy{0};

// ---- optional per-launch event timing (qgemm_timing_enable / _collect)
struct TimingRec {
  int kind;
  cudaEvent_t e0, e1;
};
struct Timing {
  bool on = false;
  std::vector<TimingRec> recs;
  std::vector<cudaEvent_t> pool;
  cudaEvent_t get() {
    if (!pool.empty()) {
      cudaEvent_t e = pool.back();
      pool.pop_back();
      return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
  }
};
thread_local Timing g_timing;

enum Kind { kPack = 0, kMain = 1, kScale = 2, kNaive = 3, kSmall = 4, kKinds = 5 };

// Bracket one launch: call before (returns the record index or -1) and after.
int tstart(int kind, cudaStream_t st) {
  if (!g_timing.on) return -1;
  TimingRec r{kind, g_timing.get(), g_timing.get()};
  cudaEventRecord(r.e0, st);
  g_timing.recs.push_back(r);
  return int(g_timing.recs.size()) - 1;
}
void tstop(int idx, cudaStream_t st) {
  if (idx >= 0) cudaEventRecord(g_timing.recs[size_t(idx)].e1, st);
}

int op_code(char t) {
  switch (t) {
    case 'N': case 'n': return 0;
    case 'T': case 't': return 1;
    case 'H': case 'h': case 'C': case 'c': return 2;
    default: return -1;
  }
}

template <typename T>
bool is_zero_q(const T *q) { return q[0] == T(0) && q[1] == T(0) && q[2] == T(0) && q[3] == T(0); }

template <typename T>
qg::Scalars<T> make_scalars(const T *alpha, const T *beta) {
  qg::Scalars<T> s;
  for (int c = 0; c < 4; ++c) { s.alpha[c] = alpha[c]; s.beta[c] = beta[c]; }
  s.alpha_real = alpha[1] == T(0) && alpha[2] == T(0) && alpha[3] == T(0);
  s.beta_real = beta[1] == T(0) && beta[2] == T(0) && beta[3] == T(0);
  s.beta_zero = is_zero_q(beta);
  return s;
}

int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }
size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// Byte extent [lo, hi) touched by a stored rows x cols matrix with leading dim ld.
template <typename T>
void extent(const T *p, int64_t rows, int64_t cols, int64_t ld, uintptr_t &lo, uintptr_t &hi) {
  lo = reinterpret_cast<uintptr_t>(p);
  hi = lo + uintptr_t(4 * sizeof(T)) * uintptr_t((cols - 1) * ld + rows);
}
bool overlaps(uintptr_t a0, uintptr_t a1, uintptr_t b0, uintptr_t b1) { return a0 < b1 && b0 < a1; }

struct Shape {
  int oa, ob;
  int64_t M, N, K;
};

// Packed-operand geometry per precision: rows per tile, k per tile, bytes per chunk.
template <typename T>
struct Geo;
// a_tiles: row tiles of packed A (FP32 with CTA pairs: an even count, the
// pair's second tile zero-filled past M); B is packed with split halves then.
#ifndef QG_TC32_2CTA
#define QG_TC32_2CTA 1  // FP32 mainloop on CTA pairs (qg_tc32_2cta.cuh); 0: one CTA per tile
#endif
template <>
struct Geo<double> {  // DMMA path (qg_dmma.cuh)
  static constexpr int64_t rows = qg::kBR, kq = qg::kBK;
  static constexpr size_t chunk = size_t(qg::kChunkElems) * sizeof(double);
  static int64_t a_tiles(int64_t M) { return cdiv(M, rows); }
  static constexpr int split_b = 0;
  static constexpr int64_t pack_sub = 1;  // chunks per pack block
};
template <>
struct Geo<float> {  // tcgen05 3xTF32 path (qg_tc32.cuh): hi + lo planes
  static constexpr int64_t rows = qg::kTcBM, kq = qg::kTcBK;
  static constexpr size_t chunk = qg::kTcChunkBytes;
  static int64_t a_tiles(int64_t M) { return QG_TC32_2CTA ? 2 * cdiv(M, 2 * rows) : cdiv(M, rows); }
  static constexpr int split_b = QG_TC32_2CTA;
  static constexpr int64_t pack_sub = qg::kTcPackSub;
};

// Bytes of one K-tile column of packed panels (all MT + NT row tiles).
template <typename T>
size_t bytes_per_ktile(int64_t M, int64_t N) {
  return size_t(Geo<T>::a_tiles(M) + cdiv(N, Geo<T>::rows)) * Geo<T>::chunk;
}

// Upper bound of the persistent grid for a panel of `ktiles` k-tiles: the
// schedule (plan_schedule) never launches more CTAs than this.
int64_t max_grid(int64_t tiles, int64_t ktiles) {
  return std::max<int64_t>(1, std::min<int64_t>(qg::kMaxPersistentCTAs, std::max<int64_t>(tiles, tiles * ktiles / 2)));
}

// Stream-K scratch of the persistent FP64 mainloop: one partial-accumulator slot
// per CTA + the arrival counters (at most 2 per CTA).
template <typename T>
size_t sk_slots_bytes(int64_t M, int64_t N, int64_t ktiles) {
  const int64_t tiles = cdiv(M, qg::kBR) * cdiv(N, qg::kBR);
  return align256(size_t(max_grid(tiles, ktiles)) * qg::kPartialBytes);
}
int num_sms();

// FP32 pair kernel: K splits per 256 x 128 tile pair when there are fewer pairs
// than one wave (one pair per 2 SMs) -- as many as fill the wave, at most 8
// (16 measured 10-19% slower at 320^3-512^3), each split >= 4 k-tiles.  Monotone in ktiles, so a reserve sized for the
// whole K covers every K-panel launch.
//
// At one wave or more the whole waves run whole tile pairs (epilogue into C) and
// only the R pairs of the partial last wave split K, S ways: S minimises the
// partial wave's cost in units of one whole-pair wave, ceil(R S / wave) / S, over
// 2 <= S <= 8 with R S <= kTc2SplitMaxWaves waves, and is taken when that cost is
// <= 0.85 and every split keeps >= kTc2SplitMinKt k-tiles (the partial stores and
// the reduce launch stay small against it).  2048^3: 128 pairs = 74 + 54, and
// 54 pairs x 4 splits fill 3 waves of quarter-K units (cost 0.75).  S depends
// on K only through the k-tile floor, so a reserve for the whole K covers every
// K-panel / host-chunk launch (tc2_part_bytes).  The environment variable
// QG_TC2_S (read once) forces S for the sub-wave / remainder case, for A/B
// measurements (within the same reserve bound).
struct Tc2Split {
  int64_t full;  // leading tile pairs of the raster computed whole (epilogue into C)
  int64_t S;     // splits of each remaining pair (1: none)
};
constexpr int64_t kTc2SplitMinKt = 16;    // >= 128 k per split unit above one wave
constexpr int64_t kTc2SplitMaxWaves = 3;  // remainder split units <= 3 waves
int tc2_forced_splits() {
  static const int v = [] {
    const char *e = std::getenv("QG_TC2_S");
    return e ? std::atoi(e) : 0;
  }();
  return v;
}
// Remainder split of R pairs above one wave (K-independent part of the rule).
int64_t tc2_rem_splits(int64_t R, int64_t wave) {
  if (R <= 0) return 1;
  const int64_t smax = std::min<int64_t>(8, kTc2SplitMaxWaves * wave / R);
  if (const int f = tc2_forced_splits()) return std::max<int64_t>(1, std::min<int64_t>(f, smax));
  int64_t best = 1;
  double cbest = 0.85;
  for (int64_t S = 2; S <= smax; ++S) {
    const double c = double(cdiv(R * S, wave)) / double(S);
    if (c < cbest - 1e-9) { cbest = c; best = S; }
  }
  return best;
}
Tc2Split tc2_split(int64_t M, int64_t N, int64_t ktiles) {
  const int64_t pairs = cdiv(M, 2 * qg::kTcBM) * cdiv(N, qg::kTcBN);
  if (!QG_TC32_2CTA) return {pairs, 1};
  const int64_t wave = std::max<int64_t>(1, num_sms() / 2);
  if (pairs < wave) {
    const int f = tc2_forced_splits();
    int64_t S = f > 0 ? f : std::min<int64_t>({wave / pairs, 8, ktiles / 4});
    S = std::max<int64_t>(1, std::min<int64_t>({S, wave / pairs, 8, ktiles}));  // within the reserve, >= 1 k-tile each
    return {S > 1 ? 0 : pairs, S};
  }
  const int64_t full = pairs / wave * wave, S = tc2_rem_splits(pairs - full, wave);
  const int64_t floor_kt = tc2_forced_splits() ? 1 : kTc2SplitMinKt;
  if (S <= 1 || ktiles < floor_kt * S) return {pairs, 1};
  return {full, S};
}
int64_t tc2_splits(int64_t M, int64_t N, int64_t ktiles) { return tc2_split(M, N, ktiles).S; }
// Split-K partials: pairs x S of the largest split any launch with <= ktiles
// k-tiles takes (sub-wave: S is monotone in ktiles; above: S or none).
size_t tc2_part_bytes(int64_t M, int64_t N, int64_t ktiles) {
  const Tc2Split sp = tc2_split(M, N, ktiles);
  if (sp.S <= 1) return 0;
  const int64_t pairs = cdiv(M, 2 * qg::kTcBM) * cdiv(N, qg::kTcBN);
  return align256(size_t(pairs - sp.full) * size_t(sp.S) * 2 * size_t(qg::kTc2PartFloats) * sizeof(float));
}

// FP32 pair kernel, chunk promotion (qg_tc32_2cta.cuh): one raw 4 x 128 x 128
// FP32 slot per SM (indexed by %smid; 37.9 MB on 148 SMs).
size_t tc2_slot_bytes() { return align256(size_t(num_sms()) * size_t(qg::kTc2PartFloats) * sizeof(float)); }

template <typename T>
size_t sk_reserve(int64_t M, int64_t N, int64_t ktiles) {
  if (sizeof(T) != 8) return (QG_TC32_2CTA ? tc2_slot_bytes() : 0) + tc2_part_bytes(M, N, ktiles);
  return sk_slots_bytes<T>(M, N, ktiles) + align256(size_t(2 * qg::kMaxPersistentCTAs) * sizeof(int));
}

template <typename T>
size_t workspace_for(int64_t M, int64_t N, int64_t K, int64_t ktiles) {
  // the stream-K reserve is sized for the whole K (an upper bound for any panel),
  // so the workspace grows linearly with the panel depth `ktiles`
  const size_t a = size_t(Geo<T>::a_tiles(M)) * size_t(ktiles) * Geo<T>::chunk;
  const size_t b = size_t(cdiv(N, Geo<T>::rows)) * size_t(ktiles) * Geo<T>::chunk;
  return align256(a) + align256(b) + sk_reserve<T>(M, N, cdiv(K, Geo<T>::kq));
}

// Argument validation common to all entry points.  Returns 0 or -i.
template <typename T>
int validate(char transA, char transB, int64_t M, int64_t N, int64_t K, const T *alpha, const T *A,
             int64_t lda, const T *B, int64_t ldb, const T *beta, const T *C, int64_t ldc, Shape &sh,
             bool &reads_ab) {
  sh.oa = op_code(transA);
  sh.ob = op_code(transB);
  if (sh.oa < 0) return -1;
  if (sh.ob < 0) return -2;
  if (M < 0) return -3;
  if (N < 0) return -4;
  if (K < 0) return -5;
  if (alpha == nullptr) return -6;
  const int64_t a_rows = sh.oa == 0 ? M : K, a_cols = sh.oa == 0 ? K : M;
  const int64_t b_rows = sh.ob == 0 ? K : N, b_cols = sh.ob == 0 ? N : K;
  if (lda < std::max<int64_t>(1, a_rows)) return -8;
  if (ldb < std::max<int64_t>(1, b_rows)) return -10;
  if (beta == nullptr) return -11;
  if (ldc < std::max<int64_t>(1, M)) return -13;
  sh.M = M; sh.N = N; sh.K = K;
  reads_ab = false;
  if (M == 0 || N == 0) return 0;
  if (C == nullptr || (reinterpret_cast<uintptr_t>(C) & 15u)) return -12;
  reads_ab = K > 0 && !is_zero_q(alpha);
  if (reads_ab) {
    if (A == nullptr || (reinterpret_cast<uintptr_t>(A) & 15u)) return -7;
    if (B == nullptr || (reinterpret_cast<uintptr_t>(B) & 15u)) return -9;
    uintptr_t c0, c1, a0, a1, b0, b1;
    extent(C, M, N, ldc, c0, c1);
    extent(A, a_rows, a_cols, lda, a0, a1);
    extent(B, b_rows, b_cols, ldb, b0, b1);
    if (overlaps(c0, c1, a0, a1) || overlaps(c0, c1, b0, b1)) return -12;
  }
  return 0;
}

template <typename T>
int launch_scale(T *C, int64_t ldc, int64_t M, int64_t N, const qg::Scalars<T> &sc, cudaStream_t st,
                 int tri = 0) {
  const int64_t total = M * N;
  const int threads = 256;
  const int64_t blocks = std::min<int64_t>(cdiv(total, threads), 148 * 16);
  { int ti = tstart(kScale, st);
  qg::qgemm_scale_kernel<T><<<unsigned(blocks), threads, 0, st>>>(C, ldc, M, N, sc, tri);
  tstop(ti, st); }
  ++g_last_launches;
  return int(cudaGetLastError());
}

// Y <- Y + beta (x) X over an M x N block (beta from sc, left product); HBM-bound.
template <typename T>
int launch_axpby(T *Y, int64_t ldy, const T *X, int64_t ldx, int64_t M, int64_t N, const qg::Scalars<T> &sc,
                 cudaStream_t st) {
  const int64_t total = M * N;
  const int threads = 256;
  const int64_t blocks = std::min<int64_t>(cdiv(total, threads), 148 * 16);
  { int ti = tstart(kScale, st);
  qg::qgemm_axpby_kernel<T><<<unsigned(blocks), threads, 0, st>>>(Y, ldy, X, ldx, M, N, sc);
  tstop(ti, st); }
  ++g_last_launches;
  return int(cudaGetLastError());
}

// is_a: the A operand (row tiles per Geo::a_tiles); B takes Geo::split_b.
template <typename T>
qg::PackJob<T> pack_job(const T *X, int64_t ldx, int row_contig, int conj, int64_t R, int64_t k_begin,
                        int64_t k_end, int64_t KT, T *out, bool is_a) {
  qg::PackJob<T> j;
  j.X = X; j.ldx = ldx; j.row_contig = row_contig; j.conj = conj; j.R = R;
  j.k_begin = k_begin; j.k_end = k_end; j.KT = KT; j.out = out;
  j.blocks = (is_a ? Geo<T>::a_tiles(R) : cdiv(R, Geo<T>::rows)) * cdiv(KT, Geo<T>::pack_sub);
  j.split_halves = is_a ? 0 : Geo<T>::split_b;
  return j;
}

// Pack both operands' panels (rows a2 and a3) in ONE launch.
template <typename T>
int launch_pack2(const qg::PackJob<T> &ja, const qg::PackJob<T> &jb, cudaStream_t st) {
  const int64_t blocks = ja.blocks + jb.blocks;
  if (blocks <= 0) return 0;
  if (blocks > INT32_MAX) return int(cudaErrorInvalidConfiguration);
  int ti = tstart(kPack, st);
  if constexpr (sizeof(T) == 8)
    qg::pack_kernel<T, qg::FragLayout><<<unsigned(blocks), 256, 0, st>>>(ja, jb);
  else
    qg::pack_tc32_kernel<<<unsigned(blocks), 256, 0, st>>>(ja, jb);
  tstop(ti, st);
  ++g_last_launches;
  return int(cudaGetLastError());
}

// Per-device caches below are atomics: any host thread may make the first call
// on a device; racing initialisations store the same value.
constexpr int kMaxDev = 64;

// Resident CTAs of the persistent FP64 mainloop on the current device.
// (cached per device: the query costs microseconds, which matter at c1 sizes)
int persistent_ctas() {
  static std::atomic<int> cache[kMaxDev];
  int dev = 0, sms = 0, per_sm = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  if (dev < kMaxDev) {
    const int c = cache[dev].load(std::memory_order_relaxed);
    if (c > 0) return c;
  }
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, qg::qgemm_dmma_kernel<qg::kFeedPacked, false, false>,
                                                    qg::kDmmaThreads, qg::kDmmaSmemBytes) != cudaSuccess)
    return 0;
  const int r = std::min(qg::kMaxPersistentCTAs, sms * std::max(1, per_sm));
  if (dev < kMaxDev) cache[dev].store(r, std::memory_order_relaxed);
  return r;
}

// Full waves folded into the stream-K part (besides the partial last wave):
// 0 = data-parallel for every full wave, stream-K over the remainder only
// (c2: 35.32-35.51 vs 35.24-35.41 TFLOP/s graph-replayed with 1).
#ifndef QG_G4_KROWS
#define QG_G4_KROWS 1  // group tiles also for k-contiguous op(A) x rows-contiguous op(B)
                        // (0.6-0.9% slower before the C ring, 0-0.5% faster with it)
#endif
#ifndef QG_RING_TRI
#define QG_RING_TRI 1  // QHERK launches take the ring whatever their K (c4 QHERK 125.0 vs 125.8 ms)
#endif
#ifndef QG_C_RING_MIN_KT
// ring epilogue for launches of >= this many k-tiles (beta != 0).  32 while the
// consumers barriered and waited for the TMA store's reads (c4's 16 k-tiles:
// 248.4 vs 245.5 ms per-lane); with the store warp (QG_C_STORE_WARP) the ring
// wins at c4 too: 241.8 vs 245.9 ms (profiles/r02w_ab.txt)
#define QG_C_RING_MIN_KT 1
#endif
#ifndef QG_C_REDUCE
#define QG_C_REDUCE 1
#endif
#ifndef QG_SK_FULL_WAVES
#define QG_SK_FULL_WAVES 0
#endif
// Persistent "data-parallel + stream-K" schedule (see qg_dmma.cuh).
void plan_schedule(qg::DmmaArgs &a, int resident) {
  a.T = a.tri ? a.MT * (a.MT + 1) / 2 : a.MT * a.NT;
  // fewer tiles than SMs: split k too, but keep >= 2 k-tiles per CTA
  const int64_t G = std::max<int64_t>(1, std::min<int64_t>(resident, std::max<int64_t>(a.T, (a.T * a.KT) / 2)));
  const int64_t waves = a.T / G, rem = a.T % G;
  if (rem == 0) {
    a.dp_tiles = a.T;
  } else if (waves >= QG_SK_FULL_WAVES) {
    a.dp_tiles = (waves - QG_SK_FULL_WAVES) * G;  // the last QG_SK_FULL_WAVES full waves + remainder go stream-K
  } else {
    a.dp_tiles = 0;
  }
  a.sk_iters = (a.T - a.dp_tiles) * a.KT;
  a.grid = G;
}

using DmmaKernel = void (*)(const qg::DmmaArgs);  // (__grid_constant__ is not part of the type)

// Instantiations: packed; TMA x the op pairs (rows-contiguous and conj flags of
// A and B are compile-time there).
// One instantiation per op pair (9 per feed).  op H implies k-contiguous
// storage for A (rows of op(A) = columns of A) and rows-contiguous for B, so
// conj A => arc = 0 and conj B => brc = 1.
// (kFeedTma128 is never used with a k-contiguous op(A) and a rows-contiguous
// op(B), kRC = 2: see launch_mainloop_direct; no such instantiation.)
template <int F, bool CA, bool CB, int RC>
DmmaKernel tma_inst() {
  if constexpr (F == qg::kFeedTma128 && RC == 2 && !QG_G4_KROWS) return nullptr;
  else return qg::qgemm_dmma_kernel<F, CA, CB, RC>;
}
template <int F>
DmmaKernel tma_kernel_op(bool ca, bool cb, int arc, int brc) {
  if (ca && cb) return tma_inst<F, true, true, 2>();
  if (ca) return brc ? tma_inst<F, true, false, 2>() : tma_inst<F, true, false, 0>();
  if (cb) return arc ? tma_inst<F, false, true, 3>() : tma_inst<F, false, true, 2>();
  switch (arc | (brc << 1)) {
    case 0: return tma_inst<F, false, false, 0>();
    case 1: return tma_inst<F, false, false, 1>();
    case 2: return tma_inst<F, false, false, 2>();
    default: return tma_inst<F, false, false, 3>();
  }
}
DmmaKernel dmma_kernel(int feed, bool ca, bool cb, int arc = 0, int brc = 0) {
  using namespace qg;
  if (feed == kFeedPacked) return qgemm_dmma_kernel<kFeedPacked, false, false>;
  if (feed == kFeedTma128) return tma_kernel_op<kFeedTma128>(ca, cb, arc, brc);
  return tma_kernel_op<kFeedTma>(ca, cb, arc, brc);
}

int dmma_set_attributes() {
  static std::atomic<bool> done[kMaxDev];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return int(e);
  if (dev < kMaxDev && done[dev].load(std::memory_order_acquire)) return 0;
  for (int feed : {int(qg::kFeedPacked), int(qg::kFeedTma), int(qg::kFeedTma128)})
    for (int c = 0; c < 16; ++c) {
      const bool ca = c & 1, cb = c & 2;
      const int arc = (c >> 2) & 1, brc = (c >> 3) & 1;
      if (feed == qg::kFeedPacked && c) continue;
      if ((ca && arc) || (cb && !brc)) continue;  // no such op
      const DmmaKernel k = dmma_kernel(feed, ca, cb, arc, brc);
      if (!k) continue;
      e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(qg::kDmmaSmemBytes));
      if (e != cudaSuccess) return int(e);
    }
  if (dev < kMaxDev) done[dev].store(true, std::memory_order_release);
  return 0;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (the library
// does not link libcuda).
using EncodeTiledFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                   const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_tiled() {
  static std::atomic<EncodeTiledFn> fn{nullptr};
  if (EncodeTiledFn f = fn.load(std::memory_order_acquire)) return f;
  void *p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess)
    return nullptr;
  fn.store(reinterpret_cast<EncodeTiledFn>(p), std::memory_order_release);
  return reinterpret_cast<EncodeTiledFn>(p);
}

// 3-D map of an R x K operand view over interleaved FP64 storage (ld in
// quaternions): (component, row, k) when rows are contiguous, else
// (component, k, row); box = one 64-row x 16-k tile, 32-byte swizzle.
int encode_view(CUtensorMap *tm, const double *X, int64_t ldx, int rc, int64_t R, int64_t K) {
  EncodeTiledFn fn = encode_tiled();
  if (!fn) return int(cudaErrorNotSupported);
  const cuuint64_t dims[3] = {4, cuuint64_t(rc ? R : K), cuuint64_t(rc ? K : R)};
  const cuuint64_t strides[2] = {32, cuuint64_t(32) * cuuint64_t(ldx)};
  const cuuint32_t box[3] = {4, cuuint32_t(rc ? qg::kBR : qg::kBK), cuuint32_t(rc ? qg::kBK : qg::kBR)};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = fn(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double *>(X), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : int(cudaErrorInvalidValue);
}

// kFeedTma128 group maps (qg_dmma.cuh): (16 doubles, k, row/4) when rows are
// contiguous, else (16 doubles, k/4, row); box = one 64-row x 16-k tile;
// 128-byte swizzle.  The inner dimension is 4 quaternions along the
// contiguous index, so it needs R % 4 == 0, resp. K % 4 == 0 (then no read
// leaves the operand's extent).
bool g4_ok(int rc, int64_t R, int64_t K) { return rc ? (R % 4 == 0) : (K % 4 == 0); }
int encode_view_g4(CUtensorMap *tm, const double *X, int64_t ldx, int rc, int64_t R, int64_t K) {
  EncodeTiledFn fn = encode_tiled();
  if (!fn) return int(cudaErrorNotSupported);
  const cuuint64_t col = cuuint64_t(32) * cuuint64_t(ldx);
  const cuuint64_t dims[3] = {16, cuuint64_t(rc ? K : K / 4), cuuint64_t(rc ? R / 4 : R)};
  const cuuint64_t strides[2] = {rc ? col : 128, rc ? 128 : col};
  const cuuint32_t box[3] = {16, cuuint32_t(rc ? qg::kBK : qg::kBK / 4), cuuint32_t(rc ? qg::kBR / 4 : qg::kBR)};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = fn(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double *>(X), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : int(cudaErrorInvalidValue);
}

// The ring epilogue moves C with the TMA unit; C in another GPU's memory (the
// multi-GPU driver stores row blocks straight into root's C over peer memory,
// dist.qgemm_rowsharded_p2p) keeps the per-lane load / store epilogue.
// QG_FORCE_REMOTE_C=1 (test hook, read once): treat every C as remote, so the
// multi-GPU epilogue (per-lane loads / stores, no ring, no L2 prefetch of C) is
// checked against the oracle on a one-GPU box (tests/test_gpu_parity.py).
bool force_remote_c() {
  static const bool v = [] {
    const char *e = std::getenv("QG_FORCE_REMOTE_C");
    return e && std::atoi(e) != 0;
  }();
  return v;
}
bool c_is_local(const void *C) {
  if (force_remote_c()) return false;
  cudaPointerAttributes at{};
  int dev = 0;
  // a failed query leaves an error behind: clear only that one, never an error
  // the caller had pending before this call
  const bool pending = cudaPeekAtLastError() != cudaSuccess;
  if (cudaPointerGetAttributes(&at, C) != cudaSuccess || cudaGetDevice(&dev) != cudaSuccess) {
    if (!pending) cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice && at.device == dev;
}

// C as (component, column, row) for the ring epilogue: box 4 x 64 columns x 16
// rows = 32 KB, 32-byte swizzle (smem [row][col][component]).
int encode_c(CUtensorMap *tm, const double *C, int64_t ldc, int64_t M, int64_t N) {
  EncodeTiledFn fn = encode_tiled();
  if (!fn) return int(cudaErrorNotSupported);
  const cuuint64_t dims[3] = {4, cuuint64_t(N), cuuint64_t(M)};
  const cuuint64_t strides[2] = {cuuint64_t(32) * cuuint64_t(ldc), 32};
  const cuuint32_t box[3] = {4, 64, 16};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = fn(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double *>(C), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : int(cudaErrorInvalidValue);
}

// Schedule + stream-K scratch + launch of a filled-in DmmaArgs (operands set).
int launch_dmma(qg::DmmaArgs &a, DmmaKernel kernel, bool direct, void *sk_scratch, cudaStream_t st) {
  // the direct kernels' epilogue C tiles go through the ring (qg_dmma.cuh
  // produce_c_stage) -- except for short-K full grids: at c4 (16 k-tiles per
  // tile) the C boxes' TMA requests compete with the A/B stream (DMMA-active
  // 94.7% vs 96.0%, 250.1 vs 247.4 ms), while c2 / c3 / QHERK gain (DESIGN.md
  // §6).  The packed kernel never takes the ring: no pointer query, no map.
  // (one pointer query per launch that reads C or may take the ring; C in
  // another GPU's memory -- the multi-GPU driver's epilogue stores -- gets
  // neither the ring nor the L2 prefetch of C tiles)
  const bool query = (direct && QG_C_RING) || !a.sc.beta_zero;
  a.c_remote = query ? !c_is_local(a.C) : 0;
  a.c_ring = direct && QG_C_RING && ((QG_RING_TRI && a.tri != 0) || a.KT >= QG_C_RING_MIN_KT) && !a.c_remote;
  // beta == 1 (real): the ring epilogue writes alpha (x) acc and the store warp
  // adds the boxes into C with TMA reductions, so no C stage is loaded through
  // the ring and no C value passes through shared memory (QG_C_REDUCE)
  a.c_reduce = a.c_ring && QG_C_REDUCE && a.sc.beta_real && a.sc.beta[0] == 1.0;
  if (a.c_ring) {
    const int e = encode_c(&a.tmC, a.C, a.ldc, a.M, a.N);
    if (e) return e;
  }
  int rc = dmma_set_attributes();
  if (rc) return rc;
  const int resident = persistent_ctas();
  if (resident <= 0) return int(cudaErrorInvalidConfiguration);
  a.MT = cdiv(a.M, qg::kBR); a.NT = cdiv(a.N, qg::kBR);
  plan_schedule(a, resident);
  // scratch layout: [2*kMaxPersistentCTAs arrival counters][grid partial slots]
  a.flags = reinterpret_cast<int *>(sk_scratch);
  a.partials = reinterpret_cast<double *>(reinterpret_cast<char *>(sk_scratch) +
                                          align256(size_t(2 * qg::kMaxPersistentCTAs) * sizeof(int)));
  if (a.sk_iters) {
    cudaError_t e = cudaMemsetAsync(a.flags, 0, size_t(a.T - a.dp_tiles) * sizeof(int), st);
    if (e != cudaSuccess) return int(e);
  }
  // Stream-K owners wait for the CTAs holding the rest of their tile, which is
  // only safe if the whole grid is resident at once.  A cooperative launch
  // guarantees that even when other kernels share the GPU (e.g. qgemm calls on
  // two streams at once, each with a persistent grid that fills every SM);
  // data-parallel-only schedules have no inter-CTA waits and launch plainly.
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(a.grid));
  cfg.blockDim = dim3(qg::kDmmaThreads);
  cfg.dynamicSmemBytes = qg::kDmmaSmemBytes;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
#ifndef QG_COOP
#define QG_COOP 1  // (0: plain launch, for the regression check in DESIGN.md §6)
#endif
  cfg.numAttrs = (QG_COOP && a.sk_iters) ? 1 : 0;
  cudaError_t le;
  { int ti = tstart(kMain, st);
  le = cudaLaunchKernelEx(&cfg, kernel, a);
  tstop(ti, st); }
  if (le != cudaSuccess) return int(le);
  ++g_last_launches;
  return int(cudaGetLastError());
}

// Packed path: operands from packed chunks (pack_kernel).
int launch_mainloop(const double *Ap, const double *Bp, double *C, int64_t ldc, int64_t M, int64_t N,
                    int64_t KT, const qg::Scalars<double> &sc, void *sk_scratch, cudaStream_t st, int tri = 0) {
  qg::DmmaArgs a{};
  a.Ap = Ap; a.Bp = Bp; a.C = C; a.ldc = ldc; a.M = M; a.N = N; a.KT = KT; a.sc = sc; a.tri = tri;
  return launch_dmma(a, dmma_kernel(qg::kFeedPacked, false, false), false, sk_scratch, st);
}

// Direct path: op(A), op(B) read in place by the producer warpgroup (no pack
// launch, no packed workspace).  rc / cj as PackSpec (row_contig, conj).
int launch_mainloop_direct(int feed, const double *A, int64_t lda, int a_rc, int a_cj, const double *B,
                           int64_t ldb, int b_rc, int b_cj, double *C, int64_t ldc, int64_t M, int64_t N,
                           int64_t K, const qg::Scalars<double> &sc, void *sk_scratch, cudaStream_t st,
                           int tri = 0) {
  qg::DmmaArgs a{};
  a.A = A; a.B = B; a.lda = lda; a.ldb = ldb; a.K = K; a.a_rc = a_rc; a.b_rc = b_rc;
  a.C = C; a.ldc = ldc; a.M = M; a.N = N; a.KT = cdiv(K, qg::kBK); a.sc = sc; a.tri = tri;
  // 4-quaternion-group tiles (conflict-free fragment loads, qg_dmma.cuh
  // kFeedTma128) where both operands' group extents are whole (for a
  // k-contiguous op(A) with a rows-contiguous op(B) only since the C tiles go
  // through the ring: before, the group tiles were 0.6-0.9% slower there,
  // profiles/r01p_feed_sweep_g4.jsonl; now 0-0.5% faster, QG_G4_KROWS)
  if (feed == qg::kFeedTma && g_path_policy.load(std::memory_order_relaxed) != 4 && g4_ok(a_rc, M, K) &&
      g4_ok(b_rc, N, K) && (QG_G4_KROWS || a_rc || !b_rc))
    feed = qg::kFeedTma128;
  if (feed == qg::kFeedTma128) {
    int rc = encode_view_g4(&a.tmA, A, lda, a_rc, M, K);
    if (!rc) rc = encode_view_g4(&a.tmB, B, ldb, b_rc, N, K);
    if (rc) return rc;
  } else if (feed == qg::kFeedTma) {
    int rc = encode_view(&a.tmA, A, lda, a_rc, M, K);
    if (!rc) rc = encode_view(&a.tmB, B, ldb, b_rc, N, K);
    if (rc) return rc;
  }
  return launch_dmma(a, dmma_kernel(feed, a_cj != 0, b_cj != 0, a_rc, b_rc), true, sk_scratch, st);
}

// 2-D view of a packed FP32 chunk array for the pair kernel's TMA: rows of
// 256 floats (1 KB); a chunk = 32 rows, a split B half = 16 rows.
int encode_packed_2d(CUtensorMap *tm, const float *base, int64_t chunks, int box_rows) {
  EncodeTiledFn fn = encode_tiled();
  if (!fn) return int(cudaErrorNotSupported);
  const cuuint64_t dims[2] = {256, cuuint64_t(chunks) * 32};
  const cuuint64_t strides[1] = {1024};
  const cuuint32_t box[2] = {256, cuuint32_t(box_rows)};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = fn(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(base), dims, strides, box,
                        estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : int(cudaErrorInvalidValue);
}

int tc32_set_attributes() {
  static std::atomic<bool> attr_set[kMaxDev];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return int(cudaErrorInvalidDevice);
  if (dev < kMaxDev && attr_set[dev].load(std::memory_order_acquire)) return 0;
  cudaError_t e = cudaFuncSetAttribute(qg::qgemm_tc32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       int(qg::kTcSmemBytes));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(qg::qgemm_tc32_2cta_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(qg::kTc2SmemBytes));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(qg::qgemm_tc32_2cta_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(qg::kTc2DSmemBytes));
  if (e != cudaSuccess) return int(e);
  if (dev < kMaxDev) attr_set[dev].store(true, std::memory_order_release);
  return 0;
}

// QG_TC2_L2_PERSIST=1 (environment, read once; off by default because it changes
// device-wide state): the per-SM running-sum slots of the FP32 pair kernel are
// launched under a persisting-L2 access-policy window, with the persisting
// carve-out (cudaLimitPersistingL2CacheSize) raised once to the slots' size.
bool tc2_l2_persist() {
  static const bool v = [] {
    const char *e = std::getenv("QG_TC2_L2_PERSIST");
    return e && std::atoi(e) != 0;
  }();
  return v;
}
// Returns the window size to use (0: not available), raising the carve-out once per device.
size_t tc2_persist_window(size_t want) {
  static std::atomic<int64_t> got[kMaxDev];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev >= kMaxDev) return 0;
  int64_t g = got[dev].load(std::memory_order_acquire);
  if (g == 0) {
    int max_persist = 0, max_window = 0;
    cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev);
    cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, dev);
    const size_t n = std::min({want, size_t(max_persist), size_t(max_window)});
    g = (n > 0 && cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, n) == cudaSuccess) ? int64_t(n) : -1;
    got[dev].store(g, std::memory_order_release);
  }
  return g > 0 ? size_t(g) : 0;
}

// Pair kernel launch (+ the split-K reduce) for a filled-in Tc2Args.
template <bool kDirect>
int launch_tc2(qg::Tc2Args &t, int64_t M, int64_t N, int64_t KT, void *sk_scratch, cudaStream_t st) {
  // sk_scratch = [per-SM chunk slots][split-K partials] (sk_reserve<float>):
  // fewer tile pairs than a wave -> split K, then one reduce + epilogue launch
  t.kc = QG_TC2_CHUNK_KT;
  t.tmp = static_cast<float *>(sk_scratch);
  t.nslots = num_sms();
  const Tc2Split sp = tc2_split(M, N, KT);
  t.S = int(sp.S);
  t.full = sp.full;
  t.part = reinterpret_cast<float *>(static_cast<char *>(sk_scratch) + tc2_slot_bytes());
  const int64_t rest = t.MT2 * t.NT - t.full;  // pairs split over K
  const int64_t grid = 2 * (t.full + rest * t.S);
  if (grid > INT32_MAX) return int(cudaErrorInvalidConfiguration);
  const size_t window = tc2_l2_persist() ? tc2_persist_window(tc2_slot_bytes()) : 0;
  { int ti = tstart(kMain, st);
  if (window) {
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeAccessPolicyWindow;
    at[0].val.accessPolicyWindow.base_ptr = t.tmp;
    at[0].val.accessPolicyWindow.num_bytes = window;
    at[0].val.accessPolicyWindow.hitRatio = 1.0f;
    at[0].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    at[0].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(unsigned(grid));
    cfg.blockDim = dim3(qg::kTcThreads);
    cfg.dynamicSmemBytes = kDirect ? qg::kTc2DSmemBytes : qg::kTc2SmemBytes;
    cfg.stream = st;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, qg::qgemm_tc32_2cta_kernel<kDirect>, t);
  } else {
    qg::qgemm_tc32_2cta_kernel<kDirect><<<unsigned(grid), qg::kTcThreads,
                                         kDirect ? qg::kTc2DSmemBytes : qg::kTc2SmemBytes, st>>>(t);
  }
  tstop(ti, st); }
  ++g_last_launches;
  if (t.S > 1) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return int(e);
    { int ti = tstart(kMain, st);
    qg::tc2_reduce_kernel<<<dim3(unsigned(2 * rest), qg::kTcBN / 16), qg::kTcBM, 0, st>>>(t);
    tstop(ti, st); }
    ++g_last_launches;
  }
  return int(cudaGetLastError());
}

// Raw interleaved FP32 operand view for the direct pair kernel: rows
// contiguous -> {4 R floats, K}, box 32 rows x 8 k (no swizzle); k contiguous
// -> {4 K floats, R}, box 8 k x box_rows rows, 128-byte swizzle (conflict-free
// converter reads; qg_tc32_2cta.cuh tc2_convert).
int encode_raw_f32(CUtensorMap *tm, const float *X, int64_t ldx, int rc, int64_t R, int64_t K, int box_rows) {
  EncodeTiledFn fn = encode_tiled();
  if (!fn) return int(cudaErrorNotSupported);
  const cuuint64_t dims[2] = {cuuint64_t(4 * (rc ? R : K)), cuuint64_t(rc ? K : R)};
  const cuuint64_t strides[1] = {cuuint64_t(16) * cuuint64_t(ldx)};
  const cuuint32_t box[2] = {rc ? 128u : 32u, rc ? cuuint32_t(qg::kTcBK) : cuuint32_t(box_rows)};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = fn(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(X), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, rc ? CU_TENSOR_MAP_SWIZZLE_NONE : CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : int(cudaErrorInvalidValue);
}

// FP32 direct path: op(A) / op(B) read in place (rc / cj as PackSpec), no pack
// launch; K is one launch (the accumulation chunks bound the error, §6).
int launch_mainloop_direct_f32(const float *A, int64_t lda, int a_rc, int a_cj, const float *B, int64_t ldb,
                               int b_rc, int b_cj, float *C, int64_t ldc, int64_t M, int64_t N, int64_t K,
                               const qg::Scalars<float> &sc, void *sk_scratch, cudaStream_t st) {
  if (int e = tc32_set_attributes()) return e;
  qg::Tc2Args t{};
  t.C = C; t.ldc = ldc; t.M = M; t.N = N; t.sc = sc;
  t.KT = cdiv(K, qg::kTcBK);
  t.MT2 = cdiv(M, 2 * qg::kTcBM); t.NT = cdiv(N, qg::kTcBN);
  t.a_rc = a_rc; t.a_cj = a_cj; t.b_rc = b_rc; t.b_cj = b_cj;
  int rc = encode_raw_f32(&t.tmA, A, lda, a_rc, M, K, qg::kTcBM);
  if (!rc) rc = encode_raw_f32(&t.tmB, B, ldb, b_rc, N, K, qg::kTcBN / 2);
  if (rc) return rc;
  return launch_tc2<true>(t, M, N, t.KT, sk_scratch, st);
}

int launch_mainloop(const float *Ap, const float *Bp, float *C, int64_t ldc, int64_t M, int64_t N, int64_t KT,
                    const qg::Scalars<float> &sc, void *sk_scratch, cudaStream_t st,
                    int /*tri: FP64 only*/ = 0) {
  if (int e = tc32_set_attributes()) return e;
  if (QG_TC32_2CTA) {
    qg::Tc2Args t{};
    t.C = C; t.ldc = ldc; t.M = M; t.N = N; t.KT = KT; t.sc = sc;
    t.MT2 = cdiv(M, 2 * qg::kTcBM); t.NT = cdiv(N, qg::kTcBN);
    int rc = encode_packed_2d(&t.tmA, Ap, 2 * t.MT2 * KT, 32);
    if (!rc) rc = encode_packed_2d(&t.tmB, Bp, t.NT * KT, 16);
    if (rc) return rc;
    return launch_tc2<false>(t, M, N, KT, sk_scratch, st);
  }
  qg::Tc32Args t;
  t.Ap = Ap; t.Bp = Bp; t.C = C; t.ldc = ldc; t.M = M; t.N = N;
  t.MT = cdiv(M, qg::kTcBM); t.NT = cdiv(N, qg::kTcBN); t.KT = KT; t.sc = sc;
  { int ti = tstart(kMain, st);
  qg::qgemm_tc32_kernel<<<unsigned(t.MT * t.NT), qg::kTcThreads, qg::kTcSmemBytes, st>>>(t);
  tstop(ti, st); }
  ++g_last_launches;
  return int(cudaGetLastError());
}


// Direct (TMA-fed) FP64 mainloop vs pack launch + mainloop.  With the
// 4-quaternion-group tiles (conflict-free fragment loads) and the C tiles
// through the ring, the direct path wins at every size measured
// (profiles/r01q_feed_sweep_ring.jsonl, r01q_ab_policy.txt): 384^3 1.08x, c2
// 1.04x, 4096^3 1.010x, c3 1.006x, c4 (K = 256) 1.012x, QHERK at c4 1.018x.
// Auto: direct whenever the group tiles apply (op(A) = N needs M % 4 == 0 and,
// with op(B) = T/H, N % 4 == 0, else K % 4 == 0), and for op(A) = T/H always
// (k-contiguous A: 2-way conflicts at worst); otherwise (32-byte tiles, 4-way
// conflicts on a rows-contiguous op(A)) only up to 2^37 quaternion MACs.
template <typename T>
int direct_feed(int opA, int opB, int64_t M, int64_t N, int64_t K) {
  const int pol = g_path_policy.load(std::memory_order_relaxed);
  // FP32 (tcgen05 pair kernel): the direct feed (raw tiles by TMA + the hi/lo
  // split in shared memory) only under policies 3 / 4.  Auto keeps the pack
  // launch: the in-SM split adds 48 KB of shared-memory traffic per stage to the
  // MMAs' ~290 KB and the SM's shared-memory port saturates -- c3 FP32 86.6 vs
  // 75.4 ms (pack + mainloop), tensor pipe 69% vs 92% active (ncu), DESIGN.md §6
  if (sizeof(T) != 8) return (pol == 3 || pol == 4) ? 1 : 0;
  if (pol == 3 || pol == 4) return qg::kFeedTma;
  if (pol != 0) return 0;
  if (opA != 0) return qg::kFeedTma;
  const bool g4 = M % 4 == 0 && (opB != 0 ? N % 4 == 0 : K % 4 == 0);
  return (g4 || double(M) * double(N) * double(K) <= double(int64_t(1) << 37)) ? qg::kFeedTma : 0;
}

// Auto policy (crossover measured on B200 with tools/small_sweep.py, DESIGN.md §6;
// profiles/r01p_small_sweep_f64.jsonl):
//  * FP64: the small kernel up to 2^25 quaternion multiply-adds (320^3: 49 us vs
//    60 direct; tie at 384^3), for K <= 16 (C-traffic bound: 4096^2 x 2 takes
//    350 us vs 564), and for few output tiles with long K (<= 64 tiles of 64x64,
//    K >= 4 max(M, N): the cluster split over K beats stream-K's owner
//    reductions, 64x64x8192: 53 us vs 332; 128x128x4096: 96 vs 153);
//  * FP32: up to 2^25 (320^3: 49 us vs 53 for the split-K pair kernel; 384^3:
//    74 vs 55), and up to 2^28 for a single 256x128 tile pair with
//    K >= 8 max(M, N) (profiles/r01p_small_sweep_f32.jsonl);
//    but not for K <= 16 with M*N >= 2^20: there the FP32 call is C-traffic
//    bound and the packed tcgen05 epilogue streams C better.
constexpr int64_t kSmallMaxMacs = int64_t(1) << 25;

int num_sms();

template <typename T>
bool use_small(int64_t M, int64_t N, int64_t K) {
  const int pol = g_path_policy.load(std::memory_order_relaxed);
  if (pol == 1 || pol == 3 || pol == 4) return false;
  if (pol == 2 || pol == 5) return true;
  constexpr int64_t kCap = int64_t(1) << 28;
  if (M > kCap || N > kCap || K > kCap) return false;  // keeps M*N*K from overflowing below
  const double macs = double(M) * double(N) * double(K);
  if (macs > double(kCap)) return false;
  if (sizeof(T) == 8) {
    if (macs <= double(kSmallMaxMacs) || K <= 16) return true;
    return cdiv(M, 64) * cdiv(N, 64) <= 64 && K >= 4 * std::max(M, N);
  }
  if (K <= 16 && double(M) * double(N) >= double(1 << 20)) return false;
  if (macs <= double(kSmallMaxMacs)) return true;
  // one 256 x 128 tile pair and a long K: even split 8 ways the pair kernel
  // fills a tenth of the GPU (64x64x4096: small 31 us vs 148)
  return cdiv(M, 256) * cdiv(N, 128) == 1 && K >= 8 * std::max(M, N);
}

int num_sms() {
  static std::atomic<int> cache[kMaxDev];
  int dev = 0, v = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  if (dev < kMaxDev && (v = cache[dev].load(std::memory_order_relaxed)) > 0) return v;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) return 148;
  if (dev < kMaxDev) cache[dev].store(v, std::memory_order_relaxed);
  return v;
}

#ifndef QG_SMALL_CLUSTER_MIN_STEPS
#define QG_SMALL_CLUSTER_MIN_STEPS 16
#endif
#ifndef QG_SMALL_MIN_STEPS
#define QG_SMALL_MIN_STEPS 1  // k4 steps per warp at least (after the split; 64x64x16: 3.5 -> 3.1 us at 1 vs 2)
#endif
#ifndef QG_SMALL_CTAS_PER_SM
#define QG_SMALL_CTAS_PER_SM (16 / QG_SMALL_WARPS)  // resident at <= 128 registers
#endif

#ifndef QG_SMALL_PDL
#define QG_SMALL_PDL 2  // c1 2.81 -> 2.37 us back to back vs no PDL; 1 (trigger at entry) slowed 128^3
#endif
// Programmatic dependent launch for the one-launch small kernel: default
// QG_SMALL_PDL, overridable at run time with the environment variable
// QG_SMALL_PDL=0/1 (read once; for A/B measurements).
// 0: plain launches; 1: PDL, the next kernel may launch at this one's entry;
// 2: PDL, triggered after each CTA's stores (tiny kernel; the general small
// kernel triggers at entry for 1 and 2).
int small_pdl() {
  static const int v = [] {
    const char *e = std::getenv("QG_SMALL_PDL");
    return e ? std::atoi(e) : QG_SMALL_PDL;
  }();
  return v;
}

template <typename T>
using SmallKernel = void (*)(qg::SmallArgs);
// Tile-exact small kernel for this op pair (qg_small.cuh qgemm_tiny_kernel).
template <typename T>
SmallKernel<T> tiny_kernel(int ops) {
  switch (ops) {
    case 0: return qg::qgemm_tiny_kernel<T, 0>;
    case 1: return qg::qgemm_tiny_kernel<T, 1>;
    case 2: return qg::qgemm_tiny_kernel<T, 2>;
    case 4: return qg::qgemm_tiny_kernel<T, 4>;
    case 5: return qg::qgemm_tiny_kernel<T, 5>;
    case 6: return qg::qgemm_tiny_kernel<T, 6>;
    case 12: return qg::qgemm_tiny_kernel<T, 12>;
    case 13: return qg::qgemm_tiny_kernel<T, 13>;
    case 14: return qg::qgemm_tiny_kernel<T, 14>;
    default: return nullptr;
  }
}

template <typename T>
int launch_small(const T *A, int64_t lda, int a_rc, int a_cj, const T *B, int64_t ldb, int b_rc, int b_cj, T *C,
                 int64_t ldc, int64_t M, int64_t N, int64_t K, const T *alpha, const T *beta, cudaStream_t st) {
  qg::SmallArgs a;
  a.A = A; a.B = B; a.C = C; a.lda = lda; a.ldb = ldb; a.ldc = ldc; a.M = M; a.N = N; a.K = K;
  a.a_rc = a_rc; a.a_cj = a_cj; a.b_rc = b_rc; a.b_cj = b_cj;
  double al[4], be[4];
  for (int c = 0; c < 4; ++c) { al[c] = double(alpha[c]); be[c] = double(beta[c]); }
  a.sc = make_scalars<double>(al, be);
  // split K over more warps until the grid covers the SMs (keeping >= 2 k4 steps per warp)
  const int64_t tm = cdiv(M, 8), tn = cdiv(N, 8), steps = cdiv(K, 4);
  const int64_t sms = num_sms();
  // split K over more warps while the grid still fits one wave of resident
  // CTAs (QG_SMALL_CTAS_PER_SM per SM) and each warp keeps >= QG_SMALL_MIN_STEPS k4 steps:
  // shorter per-warp load->DMMA chains, same number of waves
  constexpr int W = qg::kSmallWarps;
  int S = 1;
  while (S < W && cdiv(tm, W / (2 * S)) * tn <= QG_SMALL_CTAS_PER_SM * sms && steps >= 2 * QG_SMALL_MIN_STEPS * S)
    S *= 2;
  a.S = S;
  a.m_blocks = cdiv(tm, W / S);
  const int64_t blocks = a.m_blocks * tn;
  // long K with few tiles: split each tile's K over a cluster of Z CTAs too
  // (partials summed through distributed shared memory) while the grid fits one
  // wave and every warp keeps >= QG_SMALL_CLUSTER_MIN_STEPS k4 steps (below
  // that the cluster launch and barriers cost more than they save: c1 4.0 us
  // at Z = 1 vs 4.7 at Z = 2)
  int Z = 1;
  if (S == W)
    while (Z < qg::kSmallMaxCluster && blocks * 2 * Z <= QG_SMALL_CTAS_PER_SM * sms &&
           steps >= QG_SMALL_CLUSTER_MIN_STEPS * S * 2 * Z)
      Z *= 2;
  a.Z = Z;
  if (blocks * Z > INT32_MAX) return int(cudaErrorInvalidConfiguration);
  // tile-exact shapes (every 8x8 fragment and k4 step in range) take the
  // specialised kernel; FP64 moves whole quaternions as 256-bit accesses there,
  // which needs 32-byte aligned bases (FP32: the ABI's 16 bytes suffice)
  auto aligned = [](const void *p) { return (reinterpret_cast<uintptr_t>(p) & (sizeof(T) == 8 ? 31u : 15u)) == 0; };
  const bool tiny = Z == 1 && M % 8 == 0 && N % 8 == 0 && K % 4 == 0 && tn <= 65535 && aligned(A) &&
                    aligned(B) && aligned(C) &&
                    g_path_policy.load(std::memory_order_relaxed) != 5;
  const int pdl = small_pdl();
  a.pdl_trigger = pdl;
  a.per = cdiv(steps, S);
  if (tiny) {
    // the tile-exact kernel has kTinyWarps warps per CTA (2 per SM sub-partition:
    // two warps' DMMA chains interleave): its own split, by the same rule
    constexpr int WT = qg::kTinyWarps, per_sm = 16 / WT;
    S = 1;
    while (S < WT && cdiv(tm, WT / (2 * S)) * tn <= per_sm * sms && steps >= 2 * QG_SMALL_MIN_STEPS * S) S *= 2;
    a.S = S;
    a.m_blocks = cdiv(tm, WT / S);
    a.per = cdiv(steps, S);
  }
  cudaError_t e = cudaSuccess;
  { int ti = tstart(kSmall, st);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(blocks * Z));
  if (tiny) cfg.gridDim = dim3(unsigned(a.m_blocks), unsigned(tn));
  cfg.blockDim = dim3(tiny ? qg::kTinyThreads : qg::kSmallThreads);
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (Z > 1) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = unsigned(Z);
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  if (pdl) {  // programmatic dependent launch (qg_small.cuh griddepcontrol)
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = unsigned(na);
  if (tiny)
    e = cudaLaunchKernelEx(&cfg, tiny_kernel<T>(a_rc | (a_cj << 1) | (b_rc << 2) | (b_cj << 3)), a);
  else
    e = Z == 1 ? cudaLaunchKernelEx(&cfg, qg::qgemm_small_kernel<T, false>, a)
               : cudaLaunchKernelEx(&cfg, qg::qgemm_small_kernel<T, true>, a);
  tstop(ti, st); }
  if (e != cudaSuccess) return int(e);
  ++g_last_launches;
  return int(cudaGetLastError());
}

