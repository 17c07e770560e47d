// qgemm_api.cu -- C ABI and host planner of libqgemm.so (include/qgemm.h).
//
// SURVEY.md §8(a) row a1 "Plan / validate": BLAS-style argument checks, quick
// returns, workspace carving and the K-panel loop (row a6, Alg. 2's kappa loop,
// PAPER.md P:906-911), then per panel: pack A (a2), pack B (a3), mainloop with
// fused epilogue (a4 + a5) -- all enqueued on the caller's stream.
#include <algorithm>
#include <atomic>
#include <climits>
#include <cstdint>
#include <cstring>
#include <vector>
#include <cuda_runtime.h>

#include "../../include/qgemm.h"
#include "qg_dmma.cuh"
#include "qg_pack.cuh"
#include "qg_simple.cuh"
#include "qg_small.cuh"
#include "qg_simt_f32.cuh"
#include "qg_tc32.cuh"

// FP32 mainloop: 1 = tcgen05 3xTF32 (qg_tc32.cuh), 0 = FFMA (qg_simt_f32.cuh)
#ifndef QG_F32_TC
#define QG_F32_TC 1
#endif

namespace {

thread_local int g_last_launches = 0;

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
template <>
struct Geo<double> {  // DMMA path (qg_dmma.cuh)
  static constexpr int64_t rows = qg::kBR, kq = qg::kBK;
  static constexpr size_t chunk = size_t(qg::kChunkElems) * sizeof(double);
};
#if QG_F32_TC
template <>
struct Geo<float> {  // tcgen05 3xTF32 path (qg_tc32.cuh): hi + lo planes
  static constexpr int64_t rows = qg::kTcBM, kq = qg::kTcBK;
  static constexpr size_t chunk = qg::kTcChunkBytes;
};
#else
template <>
struct Geo<float> {  // FFMA path (qg_simt_f32.cuh)
  static constexpr int64_t rows = qg::kBR, kq = qg::kBK;
  static constexpr size_t chunk = size_t(qg::kChunkElems) * sizeof(float);
};
#endif

// Bytes of one K-tile column of packed panels (all MT + NT row tiles).
template <typename T>
size_t bytes_per_ktile(int64_t M, int64_t N) {
  return size_t(cdiv(M, Geo<T>::rows) + cdiv(N, Geo<T>::rows)) * Geo<T>::chunk;
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
template <typename T>
size_t sk_reserve(int64_t M, int64_t N, int64_t ktiles) {
  if (sizeof(T) != 8) return 0;
  return sk_slots_bytes<T>(M, N, ktiles) + align256(size_t(2 * qg::kMaxPersistentCTAs) * sizeof(int));
}

template <typename T>
size_t workspace_for(int64_t M, int64_t N, int64_t K, int64_t ktiles) {
  // the stream-K reserve is sized for the whole K (an upper bound for any panel),
  // so the workspace grows linearly with the panel depth `ktiles`
  const size_t a = size_t(cdiv(M, Geo<T>::rows)) * size_t(ktiles) * Geo<T>::chunk;
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

template <typename T>
qg::PackJob<T> pack_job(const T *X, int64_t ldx, int row_contig, int conj, int64_t R, int64_t k_begin,
                        int64_t k_end, int64_t KT, T *out) {
  qg::PackJob<T> j;
  j.X = X; j.ldx = ldx; j.row_contig = row_contig; j.conj = conj; j.R = R;
  j.k_begin = k_begin; j.k_end = k_end; j.KT = KT; j.out = out;
  j.blocks = cdiv(R, Geo<T>::rows) * KT;
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
#if QG_F32_TC
    qg::pack_tc32_kernel<<<unsigned(blocks), 256, 0, st>>>(ja, jb);
#else
    qg::pack_kernel<T, qg::PlanarLayout><<<unsigned(blocks), 256, 0, st>>>(ja, jb);
#endif
  tstop(ti, st);
  ++g_last_launches;
  return int(cudaGetLastError());
}

// Resident CTAs of the persistent FP64 mainloop on the current device.
// (cached per device: the query costs microseconds, which matter at c1 sizes)
int persistent_ctas() {
  constexpr int kMaxDev = 64;
  static int cache[kMaxDev] = {0};
  int dev = 0, sms = 0, per_sm = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  if (dev < kMaxDev && cache[dev] > 0) return cache[dev];
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, qg::qgemm_dmma_kernel<false, false, false>,
                                                    qg::kDmmaThreads, qg::kDmmaSmemBytes) != cudaSuccess)
    return 0;
  const int r = std::min(qg::kMaxPersistentCTAs, sms * std::max(1, per_sm));
  if (dev < kMaxDev) cache[dev] = r;
  return r;
}

// Persistent "data-parallel + stream-K" schedule (see qg_dmma.cuh).
void plan_schedule(qg::DmmaArgs &a, int resident) {
  a.T = a.tri ? a.MT * (a.MT + 1) / 2 : a.MT * a.NT;
  // fewer tiles than SMs: split k too, but keep >= 2 k-tiles per CTA
  const int64_t G = std::max<int64_t>(1, std::min<int64_t>(resident, std::max<int64_t>(a.T, (a.T * a.KT) / 2)));
  const int64_t waves = a.T / G, rem = a.T % G;
  if (rem == 0) {
    a.dp_tiles = a.T;
  } else if (waves >= 2) {
    a.dp_tiles = (waves - 1) * G;  // last full wave + remainder go stream-K
  } else {
    a.dp_tiles = 0;
  }
  a.sk_iters = (a.T - a.dp_tiles) * a.KT;
  a.grid = G;
}

using DmmaKernel = void (*)(const qg::DmmaArgs);

// The five instantiations: packed, and direct x (conj A, conj B).
DmmaKernel dmma_kernel(bool direct, bool ca, bool cb) {
  if (!direct) return qg::qgemm_dmma_kernel<false, false, false>;
  if (ca) return cb ? qg::qgemm_dmma_kernel<true, true, true> : qg::qgemm_dmma_kernel<true, true, false>;
  return cb ? qg::qgemm_dmma_kernel<true, false, true> : qg::qgemm_dmma_kernel<true, false, false>;
}

int dmma_set_attributes() {
  constexpr int kMaxDev = 64;
  static bool done[kMaxDev] = {false};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return int(e);
  if (dev < kMaxDev && done[dev]) return 0;
  const DmmaKernel ks[5] = {dmma_kernel(false, false, false), dmma_kernel(true, false, false),
                            dmma_kernel(true, true, false), dmma_kernel(true, false, true),
                            dmma_kernel(true, true, true)};
  for (DmmaKernel k : ks) {
    e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(qg::kDmmaSmemBytes));
    if (e != cudaSuccess) return int(e);
  }
  if (dev < kMaxDev) done[dev] = true;
  return 0;
}

// Schedule + stream-K scratch + launch of a filled-in DmmaArgs (operands set).
int launch_dmma(qg::DmmaArgs &a, DmmaKernel kernel, void *sk_scratch, cudaStream_t st) {
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
  { int ti = tstart(kMain, st);
  kernel<<<unsigned(a.grid), qg::kDmmaThreads, qg::kDmmaSmemBytes, st>>>(a);
  tstop(ti, st); }
  ++g_last_launches;
  return int(cudaGetLastError());
}

// Packed path: operands from packed chunks (pack_kernel).
int launch_mainloop(const double *Ap, const double *Bp, double *C, int64_t ldc, int64_t M, int64_t N,
                    int64_t KT, const qg::Scalars<double> &sc, void *sk_scratch, cudaStream_t st, int tri = 0) {
  qg::DmmaArgs a{};
  a.Ap = Ap; a.Bp = Bp; a.C = C; a.ldc = ldc; a.M = M; a.N = N; a.KT = KT; a.sc = sc; a.tri = tri;
  return launch_dmma(a, dmma_kernel(false, false, false), sk_scratch, st);
}

// Direct path: op(A), op(B) read in place by the producer warpgroup (no pack
// launch, no packed workspace).  rc / cj as PackSpec (row_contig, conj).
int launch_mainloop_direct(const double *A, int64_t lda, int a_rc, int a_cj, const double *B, int64_t ldb,
                           int b_rc, int b_cj, double *C, int64_t ldc, int64_t M, int64_t N, int64_t K,
                           const qg::Scalars<double> &sc, void *sk_scratch, cudaStream_t st, int tri = 0) {
  qg::DmmaArgs a{};
  a.A = A; a.B = B; a.lda = lda; a.ldb = ldb; a.K = K; a.a_rc = a_rc; a.b_rc = b_rc;
  a.C = C; a.ldc = ldc; a.M = M; a.N = N; a.KT = cdiv(K, qg::kBK); a.sc = sc; a.tri = tri;
  return launch_dmma(a, dmma_kernel(true, a_cj != 0, b_cj != 0), sk_scratch, st);
}

int launch_mainloop(const float *Ap, const float *Bp, float *C, int64_t ldc, int64_t M, int64_t N, int64_t KT,
                    const qg::Scalars<float> &sc, void * /*sk_scratch*/, cudaStream_t st,
                    int /*tri: FP64 only*/ = 0) {
#if QG_F32_TC
  static bool tc_attr_set = false;
  if (!tc_attr_set) {
    cudaError_t e = cudaFuncSetAttribute(qg::qgemm_tc32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(qg::kTcSmemBytes));
    if (e != cudaSuccess) return int(e);
    tc_attr_set = true;
  }
  qg::Tc32Args t;
  t.Ap = Ap; t.Bp = Bp; t.C = C; t.ldc = ldc; t.M = M; t.N = N;
  t.MT = cdiv(M, qg::kTcBM); t.NT = cdiv(N, qg::kTcBN); t.KT = KT; t.sc = sc;
  { int ti = tstart(kMain, st);
  qg::qgemm_tc32_kernel<<<unsigned(t.MT * t.NT), qg::kTcThreads, qg::kTcSmemBytes, st>>>(t);
  tstop(ti, st); }
  ++g_last_launches;
  return int(cudaGetLastError());
#endif
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(qg::qgemm_simt_f32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(qg::kF32SmemBytes));
    if (e != cudaSuccess) return int(e);
    attr_set = true;
  }
  qg::F32Args a;
  a.Ap = Ap; a.Bp = Bp; a.C = C; a.ldc = ldc; a.M = M; a.N = N;
  a.MT = cdiv(M, qg::kBR); a.NT = cdiv(N, qg::kBR); a.KT = KT; a.sc = sc;
  { int ti = tstart(kMain, st);
  qg::qgemm_simt_f32_kernel<<<unsigned(a.MT * a.NT), qg::kF32Threads, qg::kF32SmemBytes, st>>>(a);
  tstop(ti, st); }
  ++g_last_launches;
  return int(cudaGetLastError());
}

// ---- path choice: packed (pack launch + persistent mainloop), direct (FP64:
// the pack fused into the mainloop's producer warpgroup) or the one-launch
// small kernel.  0 = auto, 1 = always packed, 2 = small kernel whenever the call
// reads A and B, 3 = direct for FP64 (packed for FP32) -- qgemm_set_path_policy;
// the tests run every shape under each.
std::atomic<int> g_path_policy{0};

// Direct path only on request: measured 3.3% slower than pack + mainloop at c3
// (494.7 vs 478.9 ms) and c4 (255.1 vs 247.1 ms), equal at c2;
// its merit is memory: the workspace is the stream-K scratch only.
template <typename T>
bool use_direct() {
  if (sizeof(T) != 8) return false;
  return g_path_policy.load(std::memory_order_relaxed) == 3;
}
// Auto policy (crossover measured on B200 with tools/small_sweep.py):
//  * FP64: the small kernel up to 2^24 quaternion multiply-adds (256^3), where
//    the packed path's persistent DMMA mainloop catches up;
//  * FP32: up to 2^25 (the tcgen05 path has a 128x128 tile and no split-K), and
//    up to 2^28 when that path would launch fewer than 1/4 as many CTAs as
//    there are SMs and K >= 4 max(M, N) (small M x N, long K);
//    but not for K <= 16 with M*N >= 2^20: there the FP32 call is C-traffic
//    bound and the packed tcgen05 epilogue streams C better.
constexpr int64_t kSmallMaxMacs = int64_t(1) << 24;

int num_sms();

template <typename T>
bool use_small(int64_t M, int64_t N, int64_t K) {
  const int pol = g_path_policy.load(std::memory_order_relaxed);
  if (pol == 1 || pol == 3) return false;
  if (pol == 2) return true;
  constexpr int64_t kCap = int64_t(1) << 28;
  if (M > kCap || N > kCap || K > kCap) return false;  // keeps M*N*K from overflowing below
  const double macs = double(M) * double(N) * double(K);
  if (macs > double(kCap)) return false;
  if (sizeof(T) == 8) return macs <= double(kSmallMaxMacs);
  if (K <= 16 && double(M) * double(N) >= double(1 << 20)) return false;
  if (macs <= double(2 * kSmallMaxMacs)) return true;
  const int64_t tc_ctas = cdiv(M, 128) * cdiv(N, 128);
  return 4 * tc_ctas < num_sms() && K >= 4 * std::max(M, N);
}

int num_sms() {
  static int sms = 0;
  if (sms > 0) return sms;
  int dev = 0, v = 0;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0)
    return 148;
  sms = v;
  return sms;
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
  int S = 1;
  while (S < 4 && cdiv(tm, 4 / S) * tn < sms && steps >= 4 * S) S *= 2;
  a.S = S;
  a.m_blocks = cdiv(tm, 4 / S);
  const int64_t blocks = a.m_blocks * tn;
  if (blocks > INT32_MAX) return int(cudaErrorInvalidConfiguration);
  { int ti = tstart(kSmall, st);
  qg::qgemm_small_kernel<T><<<unsigned(blocks), qg::kSmallThreads, 0, st>>>(a);
  tstop(ti, st); }
  ++g_last_launches;
  return int(cudaGetLastError());
}

// Rows (r) x K panel of an operand as the pack kernel sees it (qg_pack.cuh).
template <typename T>
struct PackSpec {
  const T *X;
  int64_t ldx;
  int row_contig, conj;
};
template <typename T>
int panel_loop(const PackSpec<T> &pa, const PackSpec<T> &pb, int64_t M, int64_t N, int64_t K,
               const qg::Scalars<T> &sc, T *C, int64_t ldc, void *workspace, size_t workspace_bytes,
               cudaStream_t st, int tri);

template <typename T>
int qgemm_impl(char transA, char transB, int64_t M, int64_t N, int64_t K, const T *alpha, const T *A,
               int64_t lda, const T *B, int64_t ldb, const T *beta, T *C, int64_t ldc, void *workspace,
               size_t workspace_bytes, void *stream) {
  g_last_launches = 0;
  Shape sh;
  bool reads_ab = false;
  int rc = validate<T>(transA, transB, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, sh, reads_ab);
  if (rc != 0) return rc;
  if (M == 0 || N == 0) return 0;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  qg::Scalars<T> sc = make_scalars(alpha, beta);
  if (!reads_ab) return launch_scale(C, ldc, M, N, sc, st);
  PackSpec<T> pa{A, lda, sh.oa == 0 ? 1 : 0, sh.oa == 2 ? 1 : 0};
  PackSpec<T> pb{B, ldb, sh.ob == 0 ? 0 : 1, sh.ob == 2 ? 1 : 0};
  if (use_small<T>(M, N, K))  // one launch, no workspace (NEXT item 4)
    return launch_small<T>(A, lda, pa.row_contig, pa.conj, B, ldb, pb.row_contig, pb.conj, C, ldc, M, N, K,
                           alpha, beta, st);
  if constexpr (sizeof(T) == 8) {
    if (use_direct<T>()) {  // one launch; the workspace holds only the stream-K scratch
      if (workspace == nullptr || (reinterpret_cast<uintptr_t>(workspace) & 255u)) return -14;
      if (workspace_bytes < sk_reserve<T>(M, N, cdiv(K, Geo<T>::kq))) return -15;
      return launch_mainloop_direct(A, lda, pa.row_contig, pa.conj, B, ldb, pb.row_contig, pb.conj, C, ldc, M,
                                    N, K, sc, workspace, st);
    }
  }
  return panel_loop<T>(pa, pb, M, N, K, sc, C, ldc, workspace, workspace_bytes, st, 0);
}

// K-panel loop (row a6): pack A, pack B, mainloop per panel that fits.
template <typename T>
int panel_loop(const PackSpec<T> &pa, const PackSpec<T> &pb, int64_t M, int64_t N, int64_t K,
               const qg::Scalars<T> &sc, T *C, int64_t ldc, void *workspace, size_t workspace_bytes,
               cudaStream_t st, int tri) {
  int rc = 0;
  const int64_t KT_total = cdiv(K, Geo<T>::kq);
  const size_t min_ws = workspace_for<T>(M, N, K, 1);
  if (workspace == nullptr || (reinterpret_cast<uintptr_t>(workspace) & 255u)) return -14;
  if (workspace_bytes < min_ws) return -15;
  int64_t KTp = KT_total;
  while (KTp > 1 && workspace_for<T>(M, N, K, KTp) > workspace_bytes) {
    // largest panel that fits; start from a proportional estimate
    const size_t res = sk_reserve<T>(M, N, KT_total);
    int64_t est = int64_t((workspace_bytes - res) / bytes_per_ktile<T>(M, N));
    KTp = std::max<int64_t>(1, std::min<int64_t>(KTp - 1, est));
  }
  const int64_t MT = cdiv(M, Geo<T>::rows), NT = cdiv(N, Geo<T>::rows);
  T *Ap = reinterpret_cast<T *>(workspace);
  T *Bp = reinterpret_cast<T *>(reinterpret_cast<char *>(workspace) +
                                align256(size_t(MT) * size_t(KTp) * Geo<T>::chunk));
  void *sk_scratch = reinterpret_cast<char *>(Bp) + align256(size_t(NT) * size_t(KTp) * Geo<T>::chunk);
  qg::Scalars<T> sc_acc = sc;  // later panels accumulate: beta = 1
  for (int c = 0; c < 4; ++c) sc_acc.beta[c] = T(c == 0 ? 1 : 0);
  sc_acc.beta_real = 1;
  sc_acc.beta_zero = 0;
  for (int64_t kt0 = 0; kt0 < KT_total; kt0 += KTp) {
    const int64_t k_begin = kt0 * Geo<T>::kq;
    const int64_t k_end = std::min<int64_t>(K, (kt0 + KTp) * Geo<T>::kq);
    const int64_t ktn = cdiv(k_end - k_begin, Geo<T>::kq);
    rc = launch_pack2<T>(pack_job<T>(pa.X, pa.ldx, pa.row_contig, pa.conj, M, k_begin, k_end, ktn, Ap),
                         pack_job<T>(pb.X, pb.ldx, pb.row_contig, pb.conj, N, k_begin, k_end, ktn, Bp), st);
    if (rc) return rc;
    rc = launch_mainloop(Ap, Bp, C, ldc, M, N, ktn, kt0 == 0 ? sc : sc_acc, sk_scratch, st, tri);
    if (rc) return rc;
  }
  return 0;
}

template <typename T>
size_t ws_bytes(char transA, char transB, int64_t M, int64_t N, int64_t K, bool minimum);

// QHERK: C <- alpha op(A) op(A)^H + beta C on one
// triangle, alpha/beta real; same pack + DMMA mainloop, triangular tile list.
int qherk_impl(char uplo, char trans, int64_t N, int64_t K, double alpha, const double *A, int64_t lda,
               double beta, double *C, int64_t ldc, void *workspace, size_t workspace_bytes, void *stream) {
  g_last_launches = 0;
  const int tri = (uplo == 'L' || uplo == 'l') ? 1 : (uplo == 'U' || uplo == 'u') ? 2 : 0;
  if (!tri) return -1;
  const int ot = op_code(trans);
  if (ot != 0 && ot != 2) return -2;  // 'N' or 'H'/'C' (no plain transpose, as BLAS xHERK)
  if (N < 0) return -3;
  if (K < 0) return -4;
  const int64_t a_rows = ot == 0 ? N : K, a_cols = ot == 0 ? K : N;
  if (lda < std::max<int64_t>(1, a_rows)) return -7;
  if (ldc < std::max<int64_t>(1, N)) return -10;
  if (N == 0) return 0;
  if (C == nullptr || (reinterpret_cast<uintptr_t>(C) & 15u)) return -9;
  const bool reads_a = K > 0 && alpha != 0.0;
  if (!reads_a && beta == 1.0) return 0;  // BLAS quick return
  if (reads_a) {
    if (A == nullptr || (reinterpret_cast<uintptr_t>(A) & 15u)) return -6;
    uintptr_t c0, c1, a0, a1;
    extent(C, N, N, ldc, c0, c1);
    extent(A, a_rows, a_cols, lda, a0, a1);
    if (overlaps(c0, c1, a0, a1)) return -9;
  }
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const double al[4] = {alpha, 0, 0, 0}, be[4] = {beta, 0, 0, 0};
  qg::Scalars<double> sc = make_scalars(al, be);
  if (!reads_a) return launch_scale(C, ldc, N, N, sc, st, tri);
  if (workspace == nullptr || (reinterpret_cast<uintptr_t>(workspace) & 255u)) return -11;
  if (use_direct<double>()) {
    if (workspace_bytes < sk_reserve<double>(N, N, cdiv(K, qg::kBK))) return -12;
    // same operand views as the packed path below (conj folded into the signs)
    return launch_mainloop_direct(A, lda, ot == 0 ? 1 : 0, ot == 0 ? 0 : 1, A, lda, ot == 0 ? 1 : 0,
                                  ot == 0 ? 1 : 0, C, ldc, N, N, K, sc, workspace, st, tri);
  }
  if (workspace_bytes < workspace_for<double>(N, N, K, 1)) return -12;
  // op(A) as the A operand; op(B) = op(A)^H as the B operand (same buffer):
  //   trans N: op(A)(n,k) = A(n,k) -> rows contiguous;  B~(k,n) = conj(A(n,k))
  //   trans H: op(A)(n,k) = conj(A(k,n));                B~(k,n) = A(k,n)
  PackSpec<double> pa{A, lda, ot == 0 ? 1 : 0, ot == 0 ? 0 : 1};
  PackSpec<double> pb{A, lda, ot == 0 ? 1 : 0, ot == 0 ? 1 : 0};
  return panel_loop<double>(pa, pb, N, N, K, sc, C, ldc, workspace, workspace_bytes, st, tri);
}

template <typename T>
size_t ws_bytes(char transA, char transB, int64_t M, int64_t N, int64_t K, bool minimum) {
  if (op_code(transA) < 0 || op_code(transB) < 0 || M <= 0 || N <= 0 || K <= 0) return 0;
  if (use_small<T>(M, N, K)) return 0;  // the small kernel needs no workspace
  if (use_direct<T>()) return sk_reserve<T>(M, N, cdiv(K, Geo<T>::kq));  // stream-K scratch only
  return workspace_for<T>(M, N, K, minimum ? 1 : cdiv(K, Geo<T>::kq));
}

// ---------------------------------------------------------------------------
// Host-resident operands (qgemm_host / qgemm_host_f32): the end-to-end call.
//
// A, B and C live in host memory (pinned for overlap; any memory cudaMemcpy
// can address works).  The call streams them through device staging buffers
// so that the PCIe transfers hide behind the FP64 mainloop:
//   * K is cut into Q chunks (Alg. 2's kappa loop, P:906-911 = row a6): chunk p
//     of op(A) and op(B) is copied host->device on an upload stream H while the
//     compute stream S packs / multiplies chunk p-1 (double-buffered staging);
//   * C is the accumulator of the kappa loop and stays on the device; the
//     first chunk runs per column panel of C so each panel's mainloop starts
//     as soon as that panel of C has arrived (beta != 0), and the last chunk
//     runs per column panel so each finished panel is copied device->host on a
//     download stream D while the next one computes.
// Exposed on the caller's stream: chunk 0 of A/B + one C panel before the first
// mainloop, one C panel after the last.
// ---------------------------------------------------------------------------
template <typename T>
struct HostPlan {
  bool small = false;       // one-launch kernel on the whole problem (Q = P = 1)
  int64_t Kc0 = 0, Kc = 0, Q = 0;  // first K chunk (short: compute starts early), later chunks, count
  int64_t Nj = 0, P = 0;    // C column panel width and count (last chunk / downloads)
  size_t off_cold = 0;      // device copy of the caller's C (beta != 0); off_C = 0
  size_t off_sa[2], off_sb[2], off_pa[2], off_pb[2], off_sk = 0, total = 0;
  int64_t k_begin(int64_t p) const { return p == 0 ? 0 : Kc0 + (p - 1) * Kc; }
};

template <typename T>
HostPlan<T> host_plan(int64_t M, int64_t N, int64_t K) {
  HostPlan<T> h;
  constexpr size_t qb = 4 * sizeof(T);
  const int64_t kq = Geo<T>::kq, rows = 128;  // panel width: multiple of both tile sizes (64, 128)
  h.small = use_small<T>(M, N, K);
  if (h.small || K == 0) {
    h.Kc0 = h.Kc = std::max<int64_t>(K, 1); h.Q = 1; h.Nj = N; h.P = 1;
  } else {
    // chunks of ~K/8 (256..2048); the first one a quarter of that, so the first
    // mainloop waits only for a small upload
    h.Kc = std::min<int64_t>(cdiv(K, kq) * kq, std::max<int64_t>(256, std::min<int64_t>(2048, cdiv(cdiv(K, 8), kq) * kq)));
    h.Kc0 = std::min<int64_t>(h.Kc, std::max<int64_t>(kq, cdiv(cdiv(h.Kc, 4), kq) * kq));
    h.Q = K <= h.Kc0 ? 1 : 1 + cdiv(K - h.Kc0, h.Kc);
    h.Nj = std::min<int64_t>(cdiv(N, rows) * rows, std::max<int64_t>(256, cdiv(cdiv(N, 16), rows) * rows));
    h.P = cdiv(N, h.Nj);
  }
  const size_t csz = align256(size_t(M) * size_t(N) * qb);  // C, compact ld = M
  size_t off = csz;
  h.off_cold = off;
  if (!h.small && K > 0) off += csz;  // the caller's C waits here until the axpby pass
  const size_t sa = align256(size_t(M) * size_t(h.Kc) * qb), sb = align256(size_t(N) * size_t(h.Kc) * qb);
  const int nbuf = (h.Q > 1) ? 2 : 1;
  for (int i = 0; i < 2; ++i) { h.off_sa[i] = off; if (i < nbuf) off += sa; }
  for (int i = 0; i < 2; ++i) { h.off_sb[i] = off; if (i < nbuf) off += sb; }
  if (!h.small && K > 0) {
    const int64_t ktc = cdiv(h.Kc, kq);
    const size_t pa = align256(size_t(cdiv(M, Geo<T>::rows)) * size_t(ktc) * Geo<T>::chunk);
    const size_t pb = align256(size_t(cdiv(N, Geo<T>::rows)) * size_t(ktc) * Geo<T>::chunk);
    for (int i = 0; i < 2; ++i) { h.off_pa[i] = off; if (i < nbuf) off += pa; }
    for (int i = 0; i < 2; ++i) { h.off_pb[i] = off; if (i < nbuf) off += pb; }
    h.off_sk = off;
    off += sk_reserve<T>(M, N, cdiv(K, kq));
  } else {
    for (int i = 0; i < 2; ++i) h.off_pa[i] = h.off_pb[i] = off;
    h.off_sk = off;
  }
  h.total = off;
  return h;
}

// RAII set of the call's private streams/events (released once their work completes).
struct HostStreams {
  cudaStream_t H = nullptr, D = nullptr;
  std::vector<cudaEvent_t> evs;
  cudaError_t err = cudaSuccess;
  HostStreams() {
    if (err == cudaSuccess) err = cudaStreamCreateWithFlags(&H, cudaStreamNonBlocking);
    if (err == cudaSuccess) err = cudaStreamCreateWithFlags(&D, cudaStreamNonBlocking);
  }
  cudaEvent_t ev() {
    cudaEvent_t e = nullptr;
    cudaError_t r = cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    if (r != cudaSuccess) { if (err == cudaSuccess) err = r; return nullptr; }
    evs.push_back(e);
    return e;
  }
  // `waiter` waits for all work enqueued so far on `from`
  void link(cudaStream_t from, cudaStream_t waiter) {
    cudaEvent_t e = ev();
    if (!e) return;
    cudaError_t r = cudaEventRecord(e, from);
    if (r == cudaSuccess) r = cudaStreamWaitEvent(waiter, e, 0);
    if (r != cudaSuccess && err == cudaSuccess) err = r;
  }
  ~HostStreams() {
    for (cudaEvent_t e : evs) cudaEventDestroy(e);
    if (H) cudaStreamDestroy(H);
    if (D) cudaStreamDestroy(D);
  }
};

template <typename T>
int copy2d(T *dst, int64_t dld, const T *src, int64_t sld, int64_t rows, int64_t cols, cudaStream_t st) {
  constexpr size_t qb = 4 * sizeof(T);
  if (rows <= 0 || cols <= 0) return 0;
  return int(cudaMemcpy2DAsync(dst, size_t(dld) * qb, src, size_t(sld) * qb, size_t(rows) * qb, size_t(cols),
                               cudaMemcpyDefault, st));
}

template <typename T>
int qgemm_host_impl(char transA, char transB, int64_t M, int64_t N, int64_t K, const T *alpha, const T *A,
                    int64_t lda, const T *B, int64_t ldb, const T *beta, T *C, int64_t ldc, void *workspace,
                    size_t workspace_bytes, void *stream) {
  g_last_launches = 0;
  Shape sh;
  bool reads_ab = false;
  int rc = validate<T>(transA, transB, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, sh, reads_ab);
  if (rc != 0) return rc;
  if (M == 0 || N == 0) return 0;
  const int64_t Ke = reads_ab ? K : 0;  // alpha == 0 behaves as K == 0
  const HostPlan<T> h = host_plan<T>(M, N, Ke);
  if (workspace == nullptr || (reinterpret_cast<uintptr_t>(workspace) & 255u)) return -14;
  if (workspace_bytes < h.total) return -15;
  cudaStream_t S = reinterpret_cast<cudaStream_t>(stream);
  const qg::Scalars<T> sc = make_scalars(alpha, beta);
  char *ws = static_cast<char *>(workspace);
  T *Cd = reinterpret_cast<T *>(ws);
  const bool need_c = !sc.beta_zero;
  int launches = 0;

  HostStreams hs;
  if (hs.err != cudaSuccess) return int(hs.err);
  hs.link(S, hs.H);  // all transfers come after the caller's prior work
  hs.link(S, hs.D);
#define QH_TRY(x) do { int _r = (x); if (_r) return _r; if (hs.err) return int(hs.err); } while (0)

  if (!reads_ab) {  // C <- beta C
    if (need_c) QH_TRY(copy2d(Cd, M, C, ldc, M, N, hs.H));
    hs.link(hs.H, S);
    QH_TRY(launch_scale(Cd, M, M, N, sc, S));
    hs.link(S, hs.D);
    QH_TRY(copy2d(C, ldc, Cd, M, M, N, hs.D));
    hs.link(hs.D, S);
    g_last_launches = 1;
    return int(hs.err);
  }

  // staged operand views (compact): chunk p of op(A) and op(B) over k in [k0, k1)
  const int a_rc = sh.oa == 0, a_cj = sh.oa == 2, b_rc = sh.ob != 0, b_cj = sh.ob == 2;
  auto chunk = [&](int64_t p, int64_t &k0, int64_t &kc) {
    k0 = h.k_begin(p);
    kc = std::min<int64_t>(K, p == 0 ? h.Kc0 : k0 + h.Kc) - k0;
  };
  auto stage = [&](int64_t p) -> int {  // on H
    const int sl = int(p & 1);
    int64_t k0, kc;
    chunk(p, k0, kc);
    T *sa = reinterpret_cast<T *>(ws + h.off_sa[sl]);
    T *sb = reinterpret_cast<T *>(ws + h.off_sb[sl]);
    int r = a_rc ? copy2d(sa, M, A + 4 * (k0 * lda), lda, M, kc, hs.H)     // A(:, k0:k1), ld M
                 : copy2d(sa, h.Kc, A + 4 * k0, lda, kc, M, hs.H);         // A(k0:k1, :), ld Kc
    if (r) return r;
    return b_rc ? copy2d(sb, N, B + 4 * (k0 * ldb), ldb, N, kc, hs.H)      // B(:, k0:k1), ld N
                : copy2d(sb, h.Kc, B + 4 * k0, ldb, kc, N, hs.H);          // B(k0:k1, :), ld Kc
  };
  const int64_t lda_s = a_rc ? M : h.Kc, ldb_s = b_rc ? N : h.Kc;

  if (h.small) {
    QH_TRY(stage(0));
    if (need_c) QH_TRY(copy2d(Cd, M, C, ldc, M, N, hs.H));
    hs.link(hs.H, S);
    const T *sa = reinterpret_cast<const T *>(ws + h.off_sa[0]);
    const T *sb = reinterpret_cast<const T *>(ws + h.off_sb[0]);
    QH_TRY(launch_small<T>(sa, lda_s, a_rc, a_cj, sb, ldb_s, b_rc, b_cj, Cd, M, M, N, K, alpha, beta, S));
    hs.link(S, hs.D);
    QH_TRY(copy2d(C, ldc, Cd, M, M, N, hs.D));
    hs.link(hs.D, S);
    g_last_launches = 1;
    return int(hs.err);
  }

  // Cd accumulates T = alpha sum_p op(A)_p op(B)_p from beta = 0 (the caller's C
  // is not needed for that); the caller's C is uploaded behind the first two
  // chunks into Cold and folded in with one axpby pass, Cd += beta Cold, before
  // the last chunk (or per panel inside it when there are fewer than 3 chunks).
  qg::Scalars<T> sc0 = sc, sc_acc = sc;
  for (int c = 0; c < 4; ++c) {
    sc0.beta[c] = T(0);
    sc_acc.beta[c] = T(c == 0 ? 1 : 0);
  }
  sc0.beta_real = 1; sc0.beta_zero = 1;
  sc_acc.beta_real = 1; sc_acc.beta_zero = 0;
  T *Cold = reinterpret_cast<T *>(ws + h.off_cold);
  void *sk = ws + h.off_sk;
  std::vector<cudaEvent_t> packed(size_t(h.Q), nullptr);
  cudaEvent_t c_up = nullptr;
  bool folded = !need_c;
  const int64_t p_fold = h.Q >= 3 ? h.Q - 2 : -1;  // fold after this chunk's mainloop

  for (int64_t p = 0; p < h.Q; ++p) {
    const int sl = int(p & 1);
    // ---- H: staging slot sl is free once the pack of chunk p-2 has run
    if (p >= 2) QH_TRY(int(cudaStreamWaitEvent(hs.H, packed[size_t(p - 2)], 0)));
    QH_TRY(stage(p));
    cudaEvent_t staged = hs.ev();
    QH_TRY(int(cudaEventRecord(staged, hs.H)));
    if (need_c && p == std::min<int64_t>(1, h.Q - 1)) {  // the caller's C, behind chunks 0 and 1
      QH_TRY(copy2d(Cold, M, C, ldc, M, N, hs.H));
      c_up = hs.ev();
      QH_TRY(int(cudaEventRecord(c_up, hs.H)));
    }
    // ---- S: pack chunk p, then its mainloop(s)
    QH_TRY(int(cudaStreamWaitEvent(S, staged, 0)));
    int64_t k0, kc;
    chunk(p, k0, kc);
    const int64_t ktn = cdiv(kc, Geo<T>::kq);
    T *pa = reinterpret_cast<T *>(ws + h.off_pa[sl]);
    T *pb = reinterpret_cast<T *>(ws + h.off_pb[sl]);
    QH_TRY(launch_pack2<T>(pack_job<T>(reinterpret_cast<const T *>(ws + h.off_sa[sl]), lda_s, a_rc, a_cj, M, 0, kc, ktn, pa),
                           pack_job<T>(reinterpret_cast<const T *>(ws + h.off_sb[sl]), ldb_s, b_rc, b_cj, N, 0, kc, ktn, pb), S));
    ++launches;
    packed[size_t(p)] = hs.ev();
    QH_TRY(int(cudaEventRecord(packed[size_t(p)], S)));
    const qg::Scalars<T> &scp = p == 0 ? sc0 : sc_acc;
    if (p != h.Q - 1) {
      QH_TRY(launch_mainloop(pa, pb, Cd, M, M, N, ktn, scp, sk, S));
      ++launches;
      if (!folded && p == p_fold) {
        QH_TRY(int(cudaStreamWaitEvent(S, c_up, 0)));
        QH_TRY(launch_axpby(Cd, M, Cold, M, M, N, sc, S));
        ++launches;
        folded = true;
      }
      continue;
    }
    if (!folded) QH_TRY(int(cudaStreamWaitEvent(S, c_up, 0)));
    for (int64_t j = 0; j < h.P; ++j) {  // last chunk: per column panel, each downloaded at once
      const int64_t n0 = j * h.Nj, nj = std::min<int64_t>(N, n0 + h.Nj) - n0;
      const T *pbj = pb + size_t(n0 / Geo<T>::rows) * size_t(ktn) * (Geo<T>::chunk / sizeof(T));
      T *Cdj = Cd + 4 * (n0 * M);
      QH_TRY(launch_mainloop(pa, pbj, Cdj, M, M, nj, ktn, scp, sk, S));
      ++launches;
      if (!folded) {
        QH_TRY(launch_axpby(Cdj, M, Cold + 4 * (n0 * M), M, M, nj, sc, S));
        ++launches;
      }
      hs.link(S, hs.D);
      QH_TRY(copy2d(C + 4 * (n0 * ldc), ldc, Cdj, M, M, nj, hs.D));
    }
  }
  hs.link(hs.D, S);  // the call is complete when the caller's stream is
  g_last_launches = launches;
  return int(hs.err);
#undef QH_TRY
}

template <typename T>
size_t host_ws_bytes(char transA, char transB, int64_t M, int64_t N, int64_t K) {
  if (op_code(transA) < 0 || op_code(transB) < 0 || M <= 0 || N <= 0 || K < 0) return 0;
  return host_plan<T>(M, N, K).total;
}

}  // namespace

extern "C" {

int qgemm(char transA, char transB, int64_t M, int64_t N, int64_t K, const double alpha[4], const double *A,
          int64_t lda, const double *B, int64_t ldb, const double beta[4], double *C, int64_t ldc,
          void *workspace, size_t workspace_bytes, void *stream) {
  return qgemm_impl<double>(transA, transB, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, workspace,
                            workspace_bytes, stream);
}

int qgemm_f32(char transA, char transB, int64_t M, int64_t N, int64_t K, const float alpha[4], const float *A,
              int64_t lda, const float *B, int64_t ldb, const float beta[4], float *C, int64_t ldc,
              void *workspace, size_t workspace_bytes, void *stream) {
  return qgemm_impl<float>(transA, transB, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, workspace,
                           workspace_bytes, stream);
}

size_t qgemm_workspace_bytes(char transA, char transB, int64_t M, int64_t N, int64_t K, int dtype) {
  if (dtype == 0) return ws_bytes<double>(transA, transB, M, N, K, false);
  if (dtype == 1) return ws_bytes<float>(transA, transB, M, N, K, false);
  return 0;
}

size_t qgemm_workspace_min_bytes(char transA, char transB, int64_t M, int64_t N, int64_t K, int dtype) {
  if (dtype == 0) return ws_bytes<double>(transA, transB, M, N, K, true);
  if (dtype == 1) return ws_bytes<float>(transA, transB, M, N, K, true);
  return 0;
}

int qgemm_naive(char transA, char transB, int64_t M, int64_t N, int64_t K, const double alpha[4],
                const double *A, int64_t lda, const double *B, int64_t ldb, const double beta[4], double *C,
                int64_t ldc, void *stream) {
  g_last_launches = 0;
  Shape sh;
  bool reads_ab = false;
  int rc = validate<double>(transA, transB, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, sh, reads_ab);
  if (rc != 0) return rc;
  if (M == 0 || N == 0) return 0;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  qg::Scalars<double> sc = make_scalars(alpha, beta);
  if (!reads_ab) return launch_scale(C, ldc, M, N, sc, st);
  dim3 grid(unsigned(cdiv(M, 128)), unsigned(std::min<int64_t>(N, 65535)));
  { int ti = tstart(kNaive, st);
  qg::qgemm_naive_kernel<double><<<grid, 128, 0, st>>>(sh.oa, sh.ob, M, N, K, A, lda, B, ldb, C, ldc, sc);
  tstop(ti, st); }
  ++g_last_launches;
  return int(cudaGetLastError());
}

int qherk(char uplo, char trans, int64_t N, int64_t K, double alpha, const double *A, int64_t lda, double beta,
          double *C, int64_t ldc, void *workspace, size_t workspace_bytes, void *stream) {
  return qherk_impl(uplo, trans, N, K, alpha, A, lda, beta, C, ldc, workspace, workspace_bytes, stream);
}

size_t qherk_workspace_bytes(char uplo, char trans, int64_t N, int64_t K) {
  const int ot = op_code(trans);
  if (!(uplo == 'L' || uplo == 'l' || uplo == 'U' || uplo == 'u') || (ot != 0 && ot != 2) || N <= 0 || K <= 0)
    return 0;
  if (use_direct<double>()) return sk_reserve<double>(N, N, cdiv(K, qg::kBK));
  return workspace_for<double>(N, N, K, cdiv(K, qg::kBK));
}

int qgemm_host(char transA, char transB, int64_t M, int64_t N, int64_t K, const double alpha[4],
               const double *A, int64_t lda, const double *B, int64_t ldb, const double beta[4], double *C,
               int64_t ldc, void *workspace, size_t workspace_bytes, void *stream) {
  return qgemm_host_impl<double>(transA, transB, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, workspace,
                                 workspace_bytes, stream);
}

int qgemm_host_f32(char transA, char transB, int64_t M, int64_t N, int64_t K, const float alpha[4],
                   const float *A, int64_t lda, const float *B, int64_t ldb, const float beta[4], float *C,
                   int64_t ldc, void *workspace, size_t workspace_bytes, void *stream) {
  return qgemm_host_impl<float>(transA, transB, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, workspace,
                                workspace_bytes, stream);
}

size_t qgemm_host_workspace_bytes(char transA, char transB, int64_t M, int64_t N, int64_t K, int dtype) {
  if (dtype == 0) return host_ws_bytes<double>(transA, transB, M, N, K);
  if (dtype == 1) return host_ws_bytes<float>(transA, transB, M, N, K);
  return 0;
}

int qgemm_last_launch_count(void) { return g_last_launches; }

int qgemm_set_path_policy(int policy) {
  if (policy < 0 || policy > 3) return -1;
  return g_path_policy.exchange(policy);
}

void qgemm_timing_enable(int on) { g_timing.on = on != 0; }

int qgemm_timing_collect(double ms[5], int counts[5]) {
  for (int k = 0; k < kKinds; ++k) { ms[k] = 0.0; counts[k] = 0; }
  int rc = 0;
  for (const TimingRec &r : g_timing.recs) {
    cudaError_t e = cudaEventSynchronize(r.e1);
    float t = 0.f;
    if (e == cudaSuccess) e = cudaEventElapsedTime(&t, r.e0, r.e1);
    if (e != cudaSuccess && rc == 0) rc = int(e);
    ms[r.kind] += double(t);
    counts[r.kind] += 1;
    g_timing.pool.push_back(r.e0);
    g_timing.pool.push_back(r.e1);
  }
  g_timing.recs.clear();
  return rc;
}

const char *qgemm_version(void) {
#if QG_F32_TC
  return "qgemm-b200 0.2 (sm_100a; FP64 DMMA.8x8x4 persistent stream-K; FP32 tcgen05 3xTF32)";
#else
  return "qgemm-b200 0.2 (sm_100a; FP64 DMMA.8x8x4 persistent stream-K; FP32 FFMA)";
#endif
}

}  // extern "C"
