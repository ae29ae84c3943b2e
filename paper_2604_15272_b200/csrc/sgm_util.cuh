// sgm_util.cuh — utility kernels of libsgm (compiled once per process by NVRTC).
// FF input generation, NaN fills, rel_err and exact comparison reductions.
#pragma once
#include "sgm_dev.cuh"

extern "C" __global__ void sgm_fill64(u64* p, i64 n, u64 v) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) p[i] = v;
}
extern "C" __global__ void sgm_fill32(u32* p, i64 n, u32 v) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) p[i] = v;
}
extern "C" __global__ void sgm_fill16(u16* p, i64 n, u16 v) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) p[i] = v;
}

// value(i) = mix64(key + i * GOLDEN) mod p   (oracle/ff_np.py:ff_uniform)
extern "C" __global__ void sgm_ff_fill(u32* dst, i64 n, u64 key) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x)
    dst[i] = sgm::modp64(sgm::mix64(key + (u64)i * 0x9E3779B97F4A7C15ULL));
}

extern "C" __global__ void sgm_cmp_u32(const u32* a, const u32* b, i64 n, u64* count) {
  u64 c = 0;
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) c += (a[i] != b[i]);
  for (int off = 16; off > 0; off >>= 1) c += __shfl_xor_sync(0xffffffffu, c, off);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, c);
}

template <class T> __device__ __forceinline__ double to_d(T v) { return (double)v; }
template <> __device__ __forceinline__ double to_d<u16>(u16 v) { return (double)__uint_as_float(((u32)v) << 16); }

// out[0] = max|a-b| (double bits), out[1] = max|b|, out[2] = #non-finite in a
template <class T, class U> __device__ void relerr_impl(const T* a, const U* b, i64 n, u64* out) {
  double md = 0.0, mb = 0.0;
  u64 bad = 0;
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
    double x = to_d(a[i]), y = to_d(b[i]);
    if (!isfinite(x)) { bad++; continue; }
    md = fmax(md, fabs(x - y));
    mb = fmax(mb, fabs(y));
  }
  for (int off = 16; off > 0; off >>= 1) {
    md = fmax(md, __shfl_xor_sync(0xffffffffu, md, off));
    mb = fmax(mb, __shfl_xor_sync(0xffffffffu, mb, off));
    bad += __shfl_xor_sync(0xffffffffu, bad, off);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax((unsigned long long*)&out[0], (unsigned long long)__double_as_longlong(md));
    atomicMax((unsigned long long*)&out[1], (unsigned long long)__double_as_longlong(mb));
    if (bad) atomicAdd((unsigned long long*)&out[2], (unsigned long long)bad);
  }
}
extern "C" __global__ void sgm_relerr_f64(const double* a, const double* b, i64 n, u64* out) { relerr_impl(a, b, n, out); }
extern "C" __global__ void sgm_relerr_f32(const float* a, const float* b, i64 n, u64* out) { relerr_impl(a, b, n, out); }
extern "C" __global__ void sgm_relerr_bf16(const u16* a, const u16* b, i64 n, u64* out) { relerr_impl(a, b, n, out); }
// deployment-dtype output `a` against an fp64 expectation `b` (the parity gate of the sweep)
extern "C" __global__ void sgm_relerr_x_f32(const float* a, const double* b, i64 n, u64* out) { relerr_impl(a, b, n, out); }
extern "C" __global__ void sgm_relerr_x_bf16(const u16* a, const double* b, i64 n, u64* out) { relerr_impl(a, b, n, out); }

// deterministic standard-normal-like values (Box-Muller on hashed counters)
template <class N> __device__ void normal_impl(typename N::S* dst, i64 n, u64 seed) {
  for (i64 i = blockIdx.x * (i64)blockDim.x + threadIdx.x; i < n; i += (i64)gridDim.x * blockDim.x) {
    u64 h1 = sgm::mix64(seed + 2 * (u64)i + 1), h2 = sgm::mix64(seed + 2 * (u64)i + 2);
    double u1 = ((h1 >> 11) + 1) * (1.0 / 9007199254740993.0);
    double u2 = (h2 >> 11) * (1.0 / 9007199254740992.0);
    double z = sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
    dst[i] = N::st((typename N::C)z);
  }
}
extern "C" __global__ void sgm_normal_f64(double* d, i64 n, u64 s) { normal_impl<sgm::NF64>(d, n, s); }
extern "C" __global__ void sgm_normal_f32(float* d, i64 n, u64 s) { normal_impl<sgm::NF32>(d, n, s); }
extern "C" __global__ void sgm_normal_bf16(u16* d, i64 n, u64 s) { normal_impl<sgm::NBF16>(d, n, s); }
