// Can two CTAs that allocate TMEM share an SM?  Occupancy API + a real launch of
// 2 x #SM CTAs that record (smid, start, end) and hold their allocation ~20 us.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/tmem_occ tools/tmem_occ_probe.cu && /tmp/tmem_occ
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#include <algorithm>
typedef unsigned int u32;
template <int COLS, bool USE_TMEM>
__global__ void __launch_bounds__(128) probe(unsigned long long* rec, int hold_ns) {
  __shared__ u32 slot;
  extern __shared__ unsigned char dyn[];
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  u32 smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  if (USE_TMEM) {
    if (threadIdx.x < 32) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"((u32)__cvta_generic_to_shared(&slot)), "r"((u32)COLS) : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    __syncthreads();
  }
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));  // hold from the allocation on
  unsigned long long t1 = t0;
  while (t1 - t0 < (unsigned long long)hold_ns) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (threadIdx.x == 0) dyn[0] = 1;
  __syncthreads();
  if (USE_TMEM && threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(slot), "r"((u32)COLS) : "memory");
  if (threadIdx.x == 0) { rec[blockIdx.x * 3] = smid; rec[blockIdx.x * 3 + 1] = t0; rec[blockIdx.x * 3 + 2] = t1; }
}
template <int COLS, bool USE_TMEM> void run(const char* name, int smem) {
  auto k = probe<COLS, USE_TMEM>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k, 128, smem);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int grid = 2 * sms;
  unsigned long long* rec; cudaMalloc(&rec, grid * 24);
  k<<<grid, 128, smem>>>(rec, 20000);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<unsigned long long> h(grid * 3);
  cudaMemcpy(h.data(), rec, grid * 24, cudaMemcpyDeviceToHost);
  unsigned long long tmin = ~0ull, tmax = 0;
  for (int i = 0; i < grid; ++i) { tmin = std::min(tmin, h[i * 3 + 1]); tmax = std::max(tmax, h[i * 3 + 2]); }
  // count SMs where two CTAs overlapped in time
  int overlapped = 0;
  for (int s = 0; s < sms; ++s) {
    std::vector<std::pair<unsigned long long, unsigned long long>> iv;
    for (int i = 0; i < grid; ++i) if ((int)h[i * 3] == s) iv.push_back({h[i * 3 + 1], h[i * 3 + 2]});
    bool ov = false;
    for (size_t a = 0; a < iv.size(); ++a) for (size_t b = a + 1; b < iv.size(); ++b)
      if (iv[a].first < iv[b].second && iv[b].first < iv[a].second) ov = true;
    overlapped += ov;
  }
  printf("%-28s smem=%6d occAPI=%d  span=%.1f us (20 us hold)  SMs with 2 overlapping CTAs: %d/%d  %s\n", name, smem, nb,
         (tmax - tmin) / 1e3, overlapped, sms, cudaGetErrorString(e));
  cudaFree(rec);
}
int main() {
  run<128, false>("no tmem", 80 * 1024);
  run<128, true>("tmem 128 cols", 80 * 1024);
  run<256, true>("tmem 256 cols", 80 * 1024);
  run<512, true>("tmem 512 cols", 80 * 1024);
  run<128, true>("tmem 128 cols, 8 KB smem", 8 * 1024);
  return 0;
}
