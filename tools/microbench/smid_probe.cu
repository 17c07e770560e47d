// Which %smid values do CTAs see on this GPU, and what is %nsmid?
#include <cstdio>
#include <set>
#include <vector>
__global__ void k(unsigned *out) {
  unsigned s, n;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  asm volatile("mov.u32 %0, %%nsmid;" : "=r"(n));
  if (threadIdx.x == 0) { out[2 * blockIdx.x] = s; out[2 * blockIdx.x + 1] = n; }
}
int main() {
  const int nb = 148 * 8;
  unsigned *d; cudaMalloc(&d, nb * 2 * sizeof(unsigned));
  k<<<nb, 32>>>(d);
  std::vector<unsigned> h(nb * 2);
  cudaMemcpy(h.data(), d, h.size() * sizeof(unsigned), cudaMemcpyDeviceToHost);
  std::set<unsigned> ids; unsigned mx = 0;
  for (int i = 0; i < nb; ++i) { ids.insert(h[2 * i]); if (h[2 * i] > mx) mx = h[2 * i]; }
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  printf("{\"sm_count\": %d, \"nsmid\": %u, \"distinct_smid\": %zu, \"max_smid\": %u}\n", sms, h[1], ids.size(), mx);
  return 0;
}
