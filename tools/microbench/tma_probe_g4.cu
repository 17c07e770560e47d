// Probe: the "4-quaternion group" TMA tiles of the DMMA kernel's feed
// kFeedTma128 (qg_dmma.cuh), checked element by element against the offset
// formulas the consumers use.  The inner box dimension is 16 doubles = 4 whole
// quaternions = one 128-byte swizzle row, so SWIZZLE_128B applies without
// padding:
//   rows contiguous (stored R x K, ld):  dims (16, K, ceil(R/4)), strides
//     (32 ld, 128) bytes, box (16, 16, 16)  -> smem [r/4][k][r%4][c]
//   k contiguous (stored K x R, ld):     dims (16, ceil(K/4), R), strides
//     (128, 32 ld), box (16, 4, 64)         -> smem [r][k/4][k%4][c]
//   swz = lin ^ (((lin >> 7) & 7) << 4)
// (an earlier k-contiguous variant with dims (16, R, ceil(K/4)) -> smem
// [k/4][r] also checked out but was slower).  A non-monotonic stride order
// (128 B for the outer dim) is part of what is being checked.  Scratch verification tool; not product code.
//   ./tma_probe_g4
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tma_probe_g4 tma_probe_g4.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return uint32_t(__cvta_generic_to_shared(p)); }

__global__ void probe(const __grid_constant__ CUtensorMap tm, int c1, int c2, double *out) {
  extern __shared__ __align__(128) unsigned char dyn[];
  unsigned char *tile = dyn + ((1024u - (smem_u32(dyn) & 1023u)) & 1023u);
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(&bar)), "r"(32768)
                 : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];\n" ::"r"(smem_u32(tile)),
        "l"(reinterpret_cast<uint64_t>(&tm)), "r"(0), "r"(c1), "r"(c2), "r"(smem_u32(&bar))
        : "memory");
  }
  asm volatile(
      "{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@!P1 bra W;\n}\n" ::"r"(
          smem_u32(&bar)) : "memory");
  const double *t = reinterpret_cast<const double *>(tile);
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) out[i] = t[i];
}

int main() {
  void *p = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
  auto enc = reinterpret_cast<CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                           const cuuint64_t *, const cuuint32_t *, const cuuint32_t *,
                                           CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                           CUtensorMapFloatOOBfill)>(p);
  const int ld = 103, ncols = 40;  // buffer: ncols columns of ld quaternions
  double *h = (double *)malloc(sizeof(double) * 4 * ld * ncols);
  for (int j = 0; j < ncols; ++j)
    for (int i = 0; i < ld; ++i)
      for (int c = 0; c < 4; ++c) h[4 * (i + j * ld) + c] = i * 1000 + j * 10 + c + (i >= 100 ? 0.5 : 0.0);
  double *d, *o;
  CK(cudaMalloc(&d, sizeof(double) * 4 * ld * ncols));
  CK(cudaMalloc(&o, sizeof(double) * 4096));
  CK(cudaMemcpy(d, h, sizeof(double) * 4 * ld * ncols, cudaMemcpyHostToDevice));
  CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768 + 1024));
  int bad = 0;
  for (int rc = 1; rc >= 0; --rc) {
    // rc = 1: stored R x K with R = 100 rows (ld 103), K = 40 columns
    // rc = 0: stored K x R with K = 40 (k = 0..39 of each column), R = 40 columns
    const int R = rc ? 100 : 40, K = 40;
    CUtensorMap tm;
    const cuuint64_t dims[3] = {16, cuuint64_t(rc ? K : (K + 3) / 4), cuuint64_t(rc ? (R + 3) / 4 : R)};
    const cuuint64_t strides[2] = {rc ? cuuint64_t(32) * ld : 128, rc ? 128 : cuuint64_t(32) * ld};
    const cuuint32_t box[3] = {16, cuuint32_t(rc ? 16 : 4), cuuint32_t(rc ? 16 : 64)};
    const cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("rc=%d encode failed %d\n", rc, int(r)); return 1; }
    // a tile crossing the edges: rows 64..127 (R = 100), k 32..47 (K = 40)
    const int r0 = rc ? 64 : 32, k0 = 32;
    const int c1 = rc ? k0 : k0 / 4, c2 = rc ? r0 / 4 : r0;
    probe<<<1, 128, 32768 + 1024>>>(tm, c1, c2, o);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    double t[4096];
    CK(cudaMemcpy(t, o, sizeof(t), cudaMemcpyDeviceToHost));
    for (int rl = 0; rl < 64; ++rl)
      for (int kl = 0; kl < 16; ++kl)
        for (int c = 0; c < 4; ++c) {
          const int rr = r0 + rl, kk = k0 + kl;
          double want = 0.0;
          if (rc) {  // rows past R inside the last 4-row group are real memory (ld padding)
            if (kk < K && rr / 4 < (R + 3) / 4) want = h[4 * (rr + kk * ld) + c];
          } else {   // k past K inside the last 4-k group likewise
            if (rr < R && kk / 4 < (K + 3) / 4) want = h[4 * (kk + rr * ld) + c];
          }
          const uint32_t lin = rc ? uint32_t((((rl / 4) * 16 + kl) * 16 + (rl % 4) * 4 + c) * 8)
                                  : uint32_t(((rl * 4 + kl / 4) * 16 + (kl % 4) * 4 + c) * 8);
          const uint32_t swz = lin ^ (((lin >> 7) & 7u) << 4);
          if (t[swz / 8] != want) {
            if (bad < 8) printf("rc=%d mismatch at (r%d,k%d,c%d): got %g want %g\n", rc, rl, kl, c, t[swz / 8], want);
            ++bad;
          }
        }
    printf("rc=%d checked, bad=%d\n", rc, bad);
  }
  printf(bad ? "FAIL\n" : "OK\n");
  return bad != 0;
}
