// qg_host_path.cuh -- qgemm_host / qgemm_host_f32 (internal; included once, by
// qgemm_api.cu, inside its anonymous namespace, after qg_runtime.cuh).
#pragma once

// Chunking of the host-streamed path (tuned on c3): K chunks of
// ~K/QG_HOST_KC_DIV, the first one QG_HOST_KC0_DIV times shorter; the last
// chunk in QG_HOST_PANELS column panels.
#ifndef QG_HOST_KC_DIV
#define QG_HOST_KC_DIV 8
#endif
#ifndef QG_HOST_KC0_DIV
#define QG_HOST_KC0_DIV 4
#endif
#ifndef QG_HOST_PANELS
#define QG_HOST_PANELS 16
#endif
// Chunk p > 0 is QG_HOST_GROWTH^(p-1) times the second one (capped at
// QG_HOST_KC_MAX): uploads run ~6x faster than the mainloop consumes K at c3,
// so later chunks can grow, and every chunk fewer saves one C pass + relaunch
// (c3: chunks 256, 1024, 2048, 4096, 768; 489.4 ms per call vs 493.1 with
// uniform 1024-chunks; growth 3-4 up to 8192 exposes 12-16 ms of uploads).
#ifndef QG_HOST_GROWTH
#define QG_HOST_GROWTH 2
#endif
#ifndef QG_HOST_BIG_LAST
#define QG_HOST_BIG_LAST 1
#endif
#ifndef QG_HOST_LAST_SPLIT
#define QG_HOST_LAST_SPLIT 4  // the last column panel is cut into this many (its download is exposed)
#endif
#ifndef QG_HOST_KC_MAX
#define QG_HOST_KC_MAX 4096
#endif
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
  bool direct = false;      // FP64 chunks on the TMA-fed mainloop (no pack)
  int64_t Kc0 = 0, Kc = 0, Q = 0;  // first K chunk (short: compute starts early), largest chunk, count
  int64_t Nj = 0, P = 0;    // C column panel width and count (last chunk / downloads)
  size_t off_cold = 0;      // device copy of the caller's C (beta != 0); off_C = 0
  size_t off_sa[2], off_sb[2], off_pa[2], off_pb[2], off_sk = 0, total = 0;
  std::vector<int64_t> kb;  // chunk p covers k in [kb[p], kb[p+1])
  // the last chunk's launches: (first column, width) per column panel -- the very
  // last panel in QG_HOST_LAST_SPLIT pieces (multiples of 128 columns: a packed
  // FP32 B panel starts on a 128-column tile) so less of its download is exposed
  std::vector<std::pair<int64_t, int64_t>> panels;
  int64_t k_begin(int64_t p) const { return kb[size_t(p)]; }
  int64_t k_len(int64_t p) const { return kb[size_t(p) + 1] - kb[size_t(p)]; }
};

template <typename T>
HostPlan<T> host_plan(int oa, int ob, int64_t M, int64_t N, int64_t K) {
  HostPlan<T> h;
  // FP64: each chunk's mainloop reads the staged operands in place (TMA-fed,
  // no pack launch, no packed buffers) where the device path would
  h.direct = K > 0 && direct_feed<T>(oa, ob, M, N, K) != 0;
  constexpr size_t qb = 4 * sizeof(T);
  const int64_t kq = Geo<T>::kq, rows = 128;  // panel width: multiple of both tile sizes (64, 128)
  h.small = use_small<T>(M, N, K);
  if (h.small || K == 0) {
    h.Kc0 = h.Kc = std::max<int64_t>(K, 1); h.Q = 1; h.Nj = N; h.P = 1;
    h.kb = {0, K};
  } else {
    // chunks of ~K/8 (256..2048); the first one a quarter of that, so the first
    // mainloop waits only for a small upload; later ones growing by QG_HOST_GROWTH
    const int64_t kc1 = std::min<int64_t>(cdiv(K, kq) * kq,
                             std::max<int64_t>(256, std::min<int64_t>(2048, cdiv(cdiv(K, QG_HOST_KC_DIV), kq) * kq)));
    h.Kc0 = std::min<int64_t>(kc1, std::max<int64_t>(kq, cdiv(cdiv(kc1, QG_HOST_KC0_DIV), kq) * kq));
    h.kb.push_back(0);
    int64_t k = std::min<int64_t>(K, h.Kc0), len = kc1;
    h.kb.push_back(k);
    h.Kc = h.Kc0;
    while (k < K) {
      const int64_t l = std::min<int64_t>(K - k, len);
      h.Kc = std::max(h.Kc, l);
      k += l;
      h.kb.push_back(k);
      len = std::max<int64_t>(kc1, std::min<int64_t>(int64_t(QG_HOST_KC_MAX), len * QG_HOST_GROWTH));
    }
    h.Q = int64_t(h.kb.size()) - 1;
    // the last chunk runs per column panel with each panel's download behind the
    // next panel's compute: make it the longest chunk (a short remainder moves one
    // place forward) so the compute per column dwarfs the download per column
    if (QG_HOST_BIG_LAST && h.Q >= 3) {
      const int64_t last = h.kb[size_t(h.Q)] - h.kb[size_t(h.Q - 1)];
      const int64_t prev = h.kb[size_t(h.Q - 1)] - h.kb[size_t(h.Q - 2)];
      if (last < prev) h.kb[size_t(h.Q - 1)] = h.kb[size_t(h.Q - 2)] + last;
    }
    h.Nj = std::min<int64_t>(cdiv(N, rows) * rows, std::max<int64_t>(256, cdiv(cdiv(N, QG_HOST_PANELS), rows) * rows));
    h.P = cdiv(N, h.Nj);
    for (int64_t j = 0; j < h.P; ++j) {
      const int64_t n0 = j * h.Nj, nj = std::min<int64_t>(N, n0 + h.Nj) - n0;
      const int64_t piece = (j == h.P - 1) ? std::max<int64_t>(128, cdiv(cdiv(nj, QG_HOST_LAST_SPLIT), 128) * 128) : nj;
      for (int64_t c = 0; c < nj; c += piece) h.panels.emplace_back(n0 + c, std::min(piece, nj - c));
    }
  }
  // stream-K / split-K scratch for EVERY mainloop width launched: N (chunks
  // before the last) and each panel / piece width of the last chunk.  (The FP32
  // split count is not monotone in the width: a narrow piece has fewer tile
  // pairs than a wave and splits K where N and Nj did not.)
  size_t sk_need = 0;
  if (!h.small && K > 0) {
    sk_need = sk_reserve<T>(M, N, cdiv(K, kq));
    for (const auto &pn : h.panels) sk_need = std::max(sk_need, sk_reserve<T>(M, pn.second, cdiv(K, kq)));
  }
  const size_t csz = align256(size_t(M) * size_t(N) * qb);  // C, compact ld = M
  size_t off = csz;
  h.off_cold = off;
  if (!h.small && K > 0) off += csz;  // the caller's C waits here until the axpby pass
  const size_t sa = align256(size_t(M) * size_t(h.Kc) * qb), sb = align256(size_t(N) * size_t(h.Kc) * qb);
  const int nbuf = (h.Q > 1) ? 2 : 1;
  for (int i = 0; i < 2; ++i) { h.off_sa[i] = off; if (i < nbuf) off += sa; }
  for (int i = 0; i < 2; ++i) { h.off_sb[i] = off; if (i < nbuf) off += sb; }
  if (!h.small && K > 0 && !h.direct) {
    const int64_t ktc = cdiv(h.Kc, kq);
    const size_t pa = align256(size_t(Geo<T>::a_tiles(M)) * size_t(ktc) * Geo<T>::chunk);
    const size_t pb = align256(size_t(cdiv(N, Geo<T>::rows)) * size_t(ktc) * Geo<T>::chunk);
    for (int i = 0; i < 2; ++i) { h.off_pa[i] = off; if (i < nbuf) off += pa; }
    for (int i = 0; i < 2; ++i) { h.off_pb[i] = off; if (i < nbuf) off += pb; }
    h.off_sk = off;
    off += sk_need;
  } else if (!h.small && K > 0) {  // direct: stream-K scratch only
    for (int i = 0; i < 2; ++i) h.off_pa[i] = h.off_pb[i] = off;
    h.off_sk = off;
    off += sk_need;
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
  const HostPlan<T> h = host_plan<T>(op_code(transA), op_code(transB), M, N, Ke);
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
    kc = h.k_len(p);
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
    const T *sa = reinterpret_cast<const T *>(ws + h.off_sa[sl]);
    const T *sb = reinterpret_cast<const T *>(ws + h.off_sb[sl]);
    if (!h.direct) {
      QH_TRY(launch_pack2<T>(pack_job<T>(sa, lda_s, a_rc, a_cj, M, 0, kc, ktn, pa, true),
                             pack_job<T>(sb, ldb_s, b_rc, b_cj, N, 0, kc, ktn, pb, false), S));
      ++launches;
    }
    // staging slot sl is free again once the pack (or, direct, the chunk's mainloop) has run
    auto release_slot = [&]() -> int {
      packed[size_t(p)] = hs.ev();
      return int(cudaEventRecord(packed[size_t(p)], S));
    };
    // one mainloop over columns [n0, n0 + nj) of this chunk into Cdj
    auto mainloop = [&](int64_t n0, int64_t nj, T *Cdj, const qg::Scalars<T> &s_) -> int {
      if (h.direct) {
        if constexpr (sizeof(T) == 8)
          return launch_mainloop_direct(qg::kFeedTma, sa, lda_s, a_rc, a_cj, sb + 4 * (b_rc ? n0 : n0 * ldb_s),
                                        ldb_s, b_rc, b_cj, Cdj, M, M, nj, kc, s_, sk, S);
        else
          return launch_mainloop_direct_f32(sa, lda_s, a_rc, a_cj, sb + 4 * (b_rc ? n0 : n0 * ldb_s), ldb_s, b_rc,
                                            b_cj, Cdj, M, M, nj, kc, s_, sk, S);
      }
      const T *pbj = pb + size_t(n0 / Geo<T>::rows) * size_t(ktn) * (Geo<T>::chunk / sizeof(T));
      return launch_mainloop(pa, pbj, Cdj, M, M, nj, ktn, s_, sk, S);
    };
    if (!h.direct) QH_TRY(release_slot());
    const qg::Scalars<T> &scp = p == 0 ? sc0 : sc_acc;
    if (p != h.Q - 1) {
      QH_TRY(mainloop(0, N, Cd, scp));
      ++launches;
      if (h.direct) QH_TRY(release_slot());
      if (!folded && p == p_fold) {
        QH_TRY(int(cudaStreamWaitEvent(S, c_up, 0)));
        QH_TRY(launch_axpby(Cd, M, Cold, M, M, N, sc, S));
        ++launches;
        folded = true;
      }
      continue;
    }
    if (!folded) QH_TRY(int(cudaStreamWaitEvent(S, c_up, 0)));
    // last chunk: per column panel (h.panels), each downloaded at once
    for (const auto &pn : h.panels) {
      const int64_t n0 = pn.first, nj = pn.second;
      T *Cdj = Cd + 4 * (n0 * M);
      QH_TRY(mainloop(n0, nj, Cdj, scp));
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
  return host_plan<T>(op_code(transA), op_code(transB), M, N, K).total;
}

