// tcgen05.mma kind::tf32 throughput yardstick on sm_100a (the roofline
// denominator of the FP32 3xTF32 path, qg_tc32.cuh).  Context measurement
// only; not product code.  One CTA per SM; one thread issues back-to-back
// tcgen05.mma (M = 128, N = 128 or 256, K = 8) on operands resident in shared
// memory into alternating TMEM accumulators, committing every 64 MMAs.
// Reports dense tf32 TFLOP/s (2*M*N*K per MMA) best-of and sustained (~1 s).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tf32_peak tf32_peak.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  uint64_t d = uint64_t((saddr >> 4) & 0x3FFFu);
  d |= uint64_t(128 >> 4) << 16;
  d |= uint64_t(256 >> 4) << 32;
  d |= uint64_t(1) << 46;
  return d;
}
template <int N>
__host__ __device__ constexpr uint32_t idesc() {
  return (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(128 >> 4) << 24);
}

template <int N>
__global__ void __launch_bounds__(128, 1) tf32_loop(int iters, float *out) {
  __shared__ __align__(1024) float sA[128 * 8];
  __shared__ __align__(1024) float sB[256 * 8];
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 128 * 8; i += blockDim.x) sA[i] = 1e-3f * (i & 7);
  for (int i = threadIdx.x; i < 256 * 8; i += blockDim.x) sB[i] = 1e-3f * (i & 5);
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    const uint64_t a = sdesc(smem_u32(sA)), b = sdesc(smem_u32(sB));
    constexpr uint32_t id = idesc<N>();
    uint32_t phase[2] = {0, 0};
    for (int it = 0; it < iters; ++it) {
#pragma unroll 8
      for (int j = 0; j < 64; ++j) {
        const uint32_t d = tmem + uint32_t((j & 1) * N);
        const uint32_t acc = (it | j) ? 1u : 0u;
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
            "l"(a), "l"(b), "r"(id), "r"(acc));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                       smem_u32(&bar[it & 1])) : "memory");
      // two commit groups in flight: wait for the previous one
      if (it > 0) {
        const int pb = (it - 1) & 1;
        asm volatile(
            "{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W;\n}\n" ::"r"(
                smem_u32(&bar[pb])), "r"(phase[pb]) : "memory");
        phase[pb] ^= 1u;
      }
    }
    const int pb = (iters - 1) & 1;
    asm volatile(
        "{\n.reg .pred P1;\nW2:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W2;\n}\n" ::"r"(
            smem_u32(&bar[pb])), "r"(phase[pb]) : "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  if (warp == 0) {
    uint32_t r;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];\n" : "=r"(r) : "r"(tmem + ((threadIdx.x & 31) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
    if (__uint_as_float(r) == 12345.f) out[threadIdx.x] = __uint_as_float(r);
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
  }
}

// 2-CTA variant: a cluster of 2 CTAs on one TPC; the leader issues
// tcgen05.mma.cta_group::2 with M = 256 (128 rows from each CTA's smem), N
// columns (N/2 from each CTA's smem), D = 128 x N in each CTA's TMEM.
template <int N>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) tf32_loop_2cta(int iters, float *out) {
  __shared__ __align__(1024) float sA[128 * 8];
  __shared__ __align__(1024) float sB[(N / 2) * 8];
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ uint32_t tslot;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(rank));
  for (int i = threadIdx.x; i < 128 * 8; i += blockDim.x) sA[i] = 1e-3f * (i & 7);
  for (int i = threadIdx.x; i < (N / 2) * 8; i += blockDim.x) sB[i] = 1e-3f * (i & 5);
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = tslot;
  if (rank == 0 && threadIdx.x == 0) {
    const uint64_t a = sdesc(smem_u32(sA)), b = sdesc(smem_u32(sB));
    constexpr uint32_t id = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(256 >> 4) << 24);
    uint32_t phase[2] = {0, 0};
    for (int it = 0; it < iters; ++it) {
#pragma unroll 8
      for (int j = 0; j < 64; ++j) {
        const uint32_t d = tmem + uint32_t((j & 1) * N);
        const uint32_t acc = (it | j) ? 1u : 0u;
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
            "l"(a), "l"(b), "r"(id), "r"(acc));
      }
      asm volatile(
          "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
              smem_u32(&bar[it & 1])), "h"((unsigned short)3) : "memory");
      if (it > 0) {
        const int pb = (it - 1) & 1;
        asm volatile(
            "{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W;\n}\n" ::"r"(
                smem_u32(&bar[pb])), "r"(phase[pb]) : "memory");
        phase[pb] ^= 1u;
      }
    }
    const int pb = (iters - 1) & 1;
    asm volatile(
        "{\n.reg .pred P1;\nW2:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W2;\n}\n" ::"r"(
            smem_u32(&bar[pb])), "r"(phase[pb]) : "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  if (warp == 0) {
    uint32_t r;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];\n" : "=r"(r) : "r"(tmem + ((threadIdx.x & 31) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
    if (__uint_as_float(r) == 12345.f) out[threadIdx.x] = __uint_as_float(r);
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

template <int N>
int run2(int sms, int iters, int reps, float *out) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const int grid = sms & ~1;
  tf32_loop_2cta<N><<<grid, 128>>>(4, out);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  double best = 0, total_fl = 0, total_ms = 0;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(e0));
    tf32_loop_2cta<N><<<grid, 128>>>(iters, out);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    const double fl = 2.0 * 256 * N * 8 * 64.0 * iters * (grid / 2);
    const double tf = fl / (ms * 1e-3) / 1e12;
    if (tf > best) best = tf;
    total_fl += fl;
    total_ms += ms;
  }
  printf("tf32 2-CTA M=256 N=%d K=8 clusters=%d : best %.1f TFLOP/s, sustained %.1f TFLOP/s over %.0f ms\n", N,
         grid / 2, best, total_fl / (total_ms * 1e-3) / 1e12, total_ms);
  return 0;
}

template <int N>
int run(int sms, int iters, int reps, float *out) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  tf32_loop<N><<<sms, 128>>>(4, out);
  CK(cudaDeviceSynchronize());
  double best = 0, total_fl = 0, total_ms = 0;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(e0));
    tf32_loop<N><<<sms, 128>>>(iters, out);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    const double fl = 2.0 * 128 * N * 8 * 64.0 * iters * sms;
    const double tf = fl / (ms * 1e-3) / 1e12;
    if (tf > best) best = tf;
    total_fl += fl;
    total_ms += ms;
  }
  printf("tf32 M=128 N=%d K=8 grid=%d : best %.1f TFLOP/s, sustained %.1f TFLOP/s over %.0f ms\n", N, sms, best,
         total_fl / (total_ms * 1e-3) / 1e12, total_ms);
  return 0;
}

int main(int argc, char **argv) {
  int dev = 0, sms = 0, clk = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
  printf("SMs=%d max_clock_khz=%d\n", sms, clk);
  float *out;
  CK(cudaMalloc(&out, 4096));
  if (run<128>(sms, 200, 10, out)) return 1;
  if (run<256>(sms, 100, 10, out)) return 1;
  if (argc > 1 && argv[1][0] == '2') {  // 2-CTA (cta_group::2) shapes only
    if (run2<128>(sms, 200, 10, out)) return 1;
    if (run2<256>(sms, 100, 10, out)) return 1;
    return 0;
  }
  if (run<256>(sms, 10000, 40, out)) return 1;  // ~2 s back to back: sustained
  return 0;
}
