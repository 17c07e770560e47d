// FP64 pipe yardsticks on sm_100a: DFMA-loop vs DMMA(m8n8k4)-loop vs a mix.
// Context measurements only; not product code.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_pipes fp64_pipes.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

constexpr int NACC = 16;

__global__ void dfma_loop(double *out, int iters, double a, double b) {
  double acc[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
#pragma unroll
      for (int i = 0; i < NACC; ++i) acc[i] = fma(acc[i], a, b);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += acc[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}

constexpr int NT = 8;  // independent accumulator tiles per warp
__global__ void dmma_loop(double *out, int iters, double a, double b) {
  double acc[NT][2];
#pragma unroll
  for (int i = 0; i < NT; ++i) { acc[i][0] = i; acc[i][1] = -i; }
  double av = a + threadIdx.x * 1e-9, bv = b;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
#pragma unroll
      for (int i = 0; i < NT; ++i) dmma(acc[i], av, bv);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NT; ++i) s += acc[i][0] + acc[i][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

// half the warps run DFMA, half DMMA: does the FP64 rate add up?
__global__ void mixed_loop(double *out, int iters_f, int iters_m, double a, double b) {
  if ((threadIdx.x / 32) & 1) {
    double acc[NT][2];
#pragma unroll
    for (int i = 0; i < NT; ++i) { acc[i][0] = i; acc[i][1] = -i; }
    for (int it = 0; it < iters_m; ++it) {
#pragma unroll
      for (int r = 0; r < 4; ++r) {
#pragma unroll
        for (int i = 0; i < NT; ++i) dmma(acc[i], a, b);
      }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < NT; ++i) s += acc[i][0] + acc[i][1];
    if (s == 12345.678) out[threadIdx.x] = s;
  } else {
    double acc[NACC];
#pragma unroll
    for (int i = 0; i < NACC; ++i) acc[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < iters_f; ++it) {
#pragma unroll
      for (int r = 0; r < 8; ++r) {
#pragma unroll
        for (int i = 0; i < NACC; ++i) acc[i] = fma(acc[i], a, b);
      }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < NACC; ++i) s += acc[i];
    if (s == 12345.678) out[threadIdx.x] = s;
  }
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
  printf("SMs=%d max_clock_khz=%d\n", sms, clk);
  double *out;
  CK(cudaMalloc(&out, 1 << 20));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int threads_list[] = {128, 256, 512, 1024};
  for (int threads : threads_list) {
    for (int blocks_per_sm : {1, 2}) {
      int grid = sms * blocks_per_sm;
      int iters = 4000;
      dfma_loop<<<grid, threads>>>(out, 10, 1.0000001, 1e-7);
      CK(cudaDeviceSynchronize());
      float best = 1e30f;
      for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        dfma_loop<<<grid, threads>>>(out, iters, 1.0000001, 1e-7);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
      }
      double flops = 2.0 * grid * threads * (double)iters * 8 * NACC;
      printf("DFMA threads=%4d grid=%4d : %.2f TFLOP/s (%.3f ms)\n", threads, grid, flops / best / 1e9, best);

      int iters_m = 2000;
      dmma_loop<<<grid, threads>>>(out, 10, 1.0000001, 1e-7);
      CK(cudaDeviceSynchronize());
      best = 1e30f;
      for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        dmma_loop<<<grid, threads>>>(out, iters_m, 1.0000001, 1e-7);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
      }
      flops = 2.0 * 256 * (grid * (threads / 32)) * (double)iters_m * 4 * NT;
      printf("DMMA threads=%4d grid=%4d : %.2f TFLOP/s (%.3f ms)\n", threads, grid, flops / best / 1e9, best);

      best = 1e30f;
      int itf = 4000, itm = 2000;
      for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        mixed_loop<<<grid, threads>>>(out, itf, itm, 1.0000001, 1e-7);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
      }
      double nw = grid * (threads / 32);
      flops = (nw / 2) * 32 * 2.0 * itf * 8 * NACC + (nw / 2) * 2.0 * 256 * itm * 4 * NT;
      printf("MIX  threads=%4d grid=%4d : %.2f TFLOP/s (%.3f ms)\n", threads, grid, flops / best / 1e9, best);
    }
  }
  // sustained: 3 s of DFMA at 256x2
  {
    int grid = sms * 2, threads = 256, iters = 40000;
    cudaEventRecord(e0);
    for (int r = 0; r < 10; ++r) dfma_loop<<<grid, threads>>>(out, iters, 1.0000001, 1e-7);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 10 * 2.0 * grid * threads * (double)iters * 8 * NACC;
    printf("DFMA sustained %.0f ms : %.2f TFLOP/s\n", ms, flops / ms / 1e9);
    int itm = 20000;
    cudaEventRecord(e0);
    for (int r = 0; r < 10; ++r) dmma_loop<<<grid, threads>>>(out, itm, 1.0000001, 1e-7);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    flops = 10 * 2.0 * 256 * (grid * (threads / 32)) * (double)itm * 4 * NT;
    printf("DMMA sustained %.0f ms : %.2f TFLOP/s\n", ms, flops / ms / 1e9);
  }
  return 0;
}
