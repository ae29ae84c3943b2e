// Microbenchmark: TMA box streaming of a row-major bf16 matrix W[K][N] through a
// shared-memory ring (one producer lane, one consumer lane that only waits and
// releases), to find the box shape / ring depth / work split that saturate HBM
// on B200.  Build + run (on the GPU box):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/bench_tma_ring tools/bench_tma_ring.cu -lcuda
//   /tmp/bench_tma_ring
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

typedef unsigned long long u64;
typedef unsigned int u32;

__device__ __forceinline__ u32 smem_u32(const void* p) { return (u32)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(u64* b, u32 c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_wait(u64* b, u32 ph) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tLW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@P1 bra DW;\n\tbra LW;\n\tDW:\n\t}" ::"r"(
          smem_u32(b)),
      "r"(ph)
      : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(u64* b, u32 bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(u64* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* tm, int c0, int c1, u64* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"((u64)tm), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

struct Cfg {
  int box_n, box_k, slots, boxes_per_stage, split_k;  // split_k: CTAs share columns by splitting K
  int es = 2;                                         // element bytes
};

// Work: column tiles of (box_n * boxes_per_stage) columns x K rows; units = column tiles x split_k.
// CTA c processes units c, c + grid, ... (persistent); stages walk k within a unit.
__global__ void __launch_bounds__(64) ring_kernel(const __grid_constant__ CUtensorMap tm, int K, int N, Cfg cfg,
                                                  unsigned long long* sink) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ __align__(8) u64 full[16], empty[16];
  unsigned char* ring = sm + ((1024u - (smem_u32(sm) & 1023u)) & 1023u);
  const int stage_bytes = cfg.box_n * cfg.es * cfg.box_k * cfg.boxes_per_stage;
  const int tile_cols = cfg.box_n * cfg.boxes_per_stage;
  const int ntiles = N / tile_cols;
  const int units = ntiles * cfg.split_k;
  const int kper = K / cfg.split_k;
  const int nst = kper / cfg.box_k;
  if (threadIdx.x == 0) {
    for (int i = 0; i < cfg.slots; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // producer
    u32 q = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const int tile = u / cfg.split_k, ks = u % cfg.split_k;
      for (int s = 0; s < nst; ++s, ++q) {
        const u32 slot = q % cfg.slots;
        if (q >= (u32)cfg.slots) mbar_wait(&empty[slot], ((q / cfg.slots) - 1) & 1);
        mbar_expect_tx(&full[slot], stage_bytes);
        for (int b = 0; b < cfg.boxes_per_stage; ++b)
          tma2d(ring + slot * stage_bytes + b * cfg.box_n * cfg.es * cfg.box_k, &tm, tile * tile_cols + b * cfg.box_n,
                ks * kper + s * cfg.box_k, &full[slot]);
      }
    }
  } else if (threadIdx.x == 32) {  // consumer
    u32 q = 0;
    u64 acc = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x)
      for (int s = 0; s < nst; ++s, ++q) {
        const u32 slot = q % cfg.slots;
        mbar_wait(&full[slot], (q / cfg.slots) & 1);
        acc += *(volatile u32*)(ring + slot * stage_bytes);
        mbar_arrive(&empty[slot]);
      }
    if (acc == 0x12345) sink[0] = acc;
  }
}

// f32 vs bf16 box shapes at one CTA per SM, 4 x 32 KB stages (argv[1] == "dtype")
static void dtype_sweep(void* w, size_t bytes, unsigned long long* sink, int sms) {
  struct DC { const char* name; CUtensorMapDataType dt; int es; int box_n; CUtensorMapSwizzle sw; int bps; };
  const DC cs[] = {{"bf16 64x128 SW128 x2", CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, 64, CU_TENSOR_MAP_SWIZZLE_128B, 2},
                   {"f32  64x128 none   x1", CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, 64, CU_TENSOR_MAP_SWIZZLE_NONE, 1},
                   {"f32  32x128 SW128  x2", CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, 32, CU_TENSOR_MAP_SWIZZLE_128B, 2},
                   {"f32  32x128 none   x2", CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, 32, CU_TENSOR_MAP_SWIZZLE_NONE, 2}};
  for (const DC& c : cs)
    for (int cps : {1, 2}) {
      const int K = 4096;
      const int N = (int)(bytes / ((size_t)K * c.es));
      const int slots = cps == 1 ? 4 : 3;
      const int slot_bytes = cps == 1 ? 32768 : 16384;
      const int bps = cps == 1 ? c.bps : (c.bps > 1 ? c.bps / 2 : 1);
      const int box_k = slot_bytes / (bps * c.box_n * c.es);
      if (box_k > 256) continue;
      CUtensorMap tm;
      cuuint64_t gdim[2] = {(cuuint64_t)N, (cuuint64_t)K};
      cuuint64_t gstr[1] = {(cuuint64_t)N * c.es};
      cuuint32_t box[2] = {(cuuint32_t)c.box_n, (cuuint32_t)box_k};
      cuuint32_t es[2] = {1, 1};
      CUresult r = cuTensorMapEncodeTiled(&tm, c.dt, 2, w, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, c.sw,
                                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) { printf("%s encode failed %d\n", c.name, (int)r); continue; }
      Cfg cfg{c.box_n, box_k, slots, bps, 1, c.es};
      const int smem = slot_bytes * slots + 1024;
      cudaFuncSetAttribute(ring_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      const int grid = sms * cps;
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      for (int i = 0; i < 3; ++i) ring_kernel<<<grid, 64, smem>>>(tm, K, N, cfg, sink);
      cudaEventRecord(e0);
      for (int i = 0; i < 20; ++i) ring_kernel<<<grid, 64, smem>>>(tm, K, N, cfg, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("%s ctas/SM %d slots %dx%dK: %.1f us  %.0f GB/s %s\n", c.name, cps, slots, slot_bytes / 1024, ms * 50.0,
             bytes / (ms * 50.0) / 1e3, cudaGetErrorString(cudaGetLastError()));
    }
}

int main(int argc, char** argv) {
  const int K = 4096, N = 28672;  // two 4096 x 14336 bf16 weights side by side (235 MB)
  size_t bytes = (size_t)K * N * 2;
  void* w;
  cudaMalloc(&w, bytes);
  cudaMemset(w, 1, bytes);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  if (argc > 1) { dtype_sweep(w, bytes, sink, sms); return 0; }
  std::vector<Cfg> cfgs;
  for (int box_k : {32, 64, 128, 256})
    for (int slots : {4, 8, 12})
      for (int bps : {1, 2, 4})
        for (int sk : {1, 4}) {
          int sb = 64 * 2 * box_k * bps;
          if (sb * slots > 200 * 1024 || sb > 64 * 1024) continue;
          cfgs.push_back({64, box_k, slots, bps, sk});
        }
  printf("box_n box_k slots boxes/stage split_k ctas/SM  us  GB/s\n");
  for (auto c : cfgs)
    for (int cps : {1, 2}) {
      int sb = 64 * 2 * c.box_k * c.boxes_per_stage;
      int smem = sb * c.slots + 1024;
      if (cps == 2 && smem > 110 * 1024) continue;
      CUtensorMap tm;
      cuuint64_t gdim[2] = {(cuuint64_t)N, (cuuint64_t)K};
      cuuint64_t gstr[1] = {(cuuint64_t)N * 2};
      cuuint32_t box[2] = {(cuuint32_t)c.box_n, (cuuint32_t)c.box_k};
      cuuint32_t es[2] = {1, 1};
      CUresult r = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, w, gdim, gstr, box, es,
                                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); continue; }
      cudaFuncSetAttribute(ring_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      int grid = sms * cps;
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      for (int i = 0; i < 3; ++i) ring_kernel<<<grid, 64, smem>>>(tm, K, N, c, sink);
      cudaEventRecord(e0);
      const int it = 20;
      for (int i = 0; i < it; ++i) ring_kernel<<<grid, 64, smem>>>(tm, K, N, c, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      cudaError_t err = cudaGetLastError();
      double us = ms * 1000.0 / it;
      printf("%5d %5d %5d %11d %7d %7d %8.1f %6.0f %s\n", c.box_n, c.box_k, c.slots, c.boxes_per_stage, c.split_k, cps, us,
             bytes / us / 1e3, err == cudaSuccess ? "" : cudaGetErrorString(err));
    }
  return 0;
}
