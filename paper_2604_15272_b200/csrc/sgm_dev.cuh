// sgm_dev.cuh — device building blocks for generated sGraph-candidate kernels.
//
// Every generated kernel (sgm_codegen.cpp) includes this header through NVRTC.
// A kernel executes one *logical block* of the candidate's block graph with one
// CTA, or with several CTAs: "free parts" (independent CTAs splitting an axis
// no node reduces) and "cluster parts" (CTAs of one thread-block cluster that
// split a reduced axis or the for-loop and combine partial tiles through
// distributed shared memory).  Tiles live in shared memory as dense row-major
// rank-4 arrays of the number system's compute type.
//
// Semantics follow the reference interpreter (pkg/src/symfuse/interp.py):
//   apply_op (interp.py:45-66)   -> unary/binary/sum/matmul/scale below
//   _silu    (interp.py:36-42)   -> NF64::silu (same two branches) / NF32::silu (branch-free, same function)
//   accum    (interp.py:171-176) -> plain sums (order-insensitive up to fp rounding)
// and the finite-field restatement in oracle/ff_np.py (bit-exact).
#pragma once

typedef unsigned long long u64;
typedef unsigned int u32;
typedef long long i64;
typedef unsigned short u16;

namespace sgm {

// Opaque 128-byte TMA descriptor (CUtensorMap), encoded on the host per launch.
struct __align__(64) TmaDesc {
  u64 w[16];
};

struct Args {
  const void* in[16];
  void* out[16];
  void* scratch;
  TmaDesc tm[4];
};

// Barrier among the NT compute threads only (named barrier 1).  Kernels with a
// TMA producer warp launch NT + 32 threads; the producer never joins this.
template <int NT> __device__ __forceinline__ void csync() {
  asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
}

// ---------------------------------------------------------------------------
// Finite field GF(p), p = 2^31 - 1 (Mersenne): 2^31 == 1 (mod p).

constexpr u32 P = 0x7FFFFFFFu;

__device__ __forceinline__ u32 modp64(u64 v) {
  v = (v & P) + (v >> 31);
  v = (v & P) + (v >> 31);
  u32 r = (u32)v;
  return r >= P ? r - P : r;
}
__device__ __forceinline__ u32 ff_add(u32 a, u32 b) { u32 s = a + b; return s >= P ? s - P : s; }
__device__ __forceinline__ u32 ff_mul(u32 a, u32 b) { return modp64((u64)a * b); }
// product folded below 2^32 (lazy reduction for dot products)
__device__ __forceinline__ u64 ff_mul_lazy(u32 a, u32 b) { u64 x = (u64)a * b; return (x & P) + (x >> 31); }
__device__ __forceinline__ u32 ff_inv(u32 a) {
  // a^(p-2); inv(0) := 0 (documented convention, mirrored in oracle/ff_np.py)
  u32 r = 1, b = a;
  u32 e = P - 2u;
  while (e) {
    if (e & 1u) r = ff_mul(r, b);
    b = ff_mul(b, b);
    e >>= 1;
  }
  return r;
}
__device__ __forceinline__ u64 mix64(u64 z) {
  z ^= z >> 30; z *= 0xbf58476d1ce4e5b9ULL;
  z ^= z >> 27; z *= 0x94d049bb133111ebULL;
  z ^= z >> 31;
  return z;
}
// Uninterpreted unary ops as keyed hashes: h_k(x) = mix64(x + K_k) mod p.
constexpr u64 FF_KEY_EXP = 0x9E3779B97F4A7C15ULL;
constexpr u64 FF_KEY_SILU = 0x3C6EF372FE94F82AULL;
constexpr u64 FF_KEY_SQRT = 0xDAA66D2C7DDF743FULL;
__device__ __forceinline__ u32 ff_hash(u32 x, u64 key) { return modp64(mix64((u64)x + key)); }

// ---------------------------------------------------------------------------
// Number systems.  S = storage type in HBM, C = tile (compute) type in smem,
// A = accumulator type for reductions (sum / matmul contraction).

struct NF64 {
  typedef double S; typedef double C; typedef double A;
  static constexpr int VEC = 2;  // elements per 16-byte vector
  __device__ static __forceinline__ C ld(S v) { return v; }
  __device__ static __forceinline__ S st(C v) { return v; }
  __device__ static __forceinline__ C zero() { return 0.0; }
  __device__ static __forceinline__ C nan() { return __longlong_as_double(0x7ff8000000000000LL); }
  __device__ static __forceinline__ C add(C a, C b) { return a + b; }
  __device__ static __forceinline__ C mul(C a, C b) { return a * b; }
  __device__ static __forceinline__ C div(C a, C b) { return a / b; }
  __device__ static __forceinline__ C sq(C a) { return a * a; }
  __device__ static __forceinline__ C ex(C a) { return ::exp(a); }
  __device__ static __forceinline__ C sqr(C a) { return ::sqrt(a); }
  __device__ static __forceinline__ C silu(C x) {
    if (x >= 0.0) return x / (1.0 + ::exp(-x));
    C e = ::exp(x);
    return x * e / (1.0 + e);
  }
  __device__ static __forceinline__ C scale(C x, C c) { return c * x; }
  __device__ static __forceinline__ A azero() { return 0.0; }
  __device__ static __forceinline__ void aadd(A& a, C v) { a += v; }
  __device__ static __forceinline__ void amerge(A& a, A b) { a += b; }
  __device__ static __forceinline__ void mac(A& a, C x, C y) { a = fma(x, y, a); }
  __device__ static __forceinline__ C fin(A a) { return a; }
};

struct NF32 {
  typedef float S; typedef float C; typedef float A;
  static constexpr int VEC = 4;
  __device__ static __forceinline__ C ld(S v) { return v; }
  __device__ static __forceinline__ S st(C v) { return v; }
  __device__ static __forceinline__ C zero() { return 0.0f; }
  __device__ static __forceinline__ C nan() { return __int_as_float(0x7fc00000); }
  __device__ static __forceinline__ C add(C a, C b) { return a + b; }
  __device__ static __forceinline__ C mul(C a, C b) { return a * b; }
  // Branch-free quotient: approximate reciprocal, one Newton step, one residual
  // correction (the IEEE quotient in all but extreme-exponent cases).  '/' and
  // __frcp_rn carry a slow-path call whose branch keeps the compiler from
  // overlapping consecutive elements.  0, inf and NaN cases fall back by select
  // to the plain product (a/0 = inf, a/inf = 0, 0/0 = NaN as in IEEE).
  __device__ static __forceinline__ C rcp(C b) {
    C r;
    asm("rcp.approx.f32 %0, %1;" : "=f"(r) : "f"(b));
    const C r2 = r * fmaf(-b, r, 2.0f);
    return isfinite(r2) ? r2 : r;
  }
  __device__ static __forceinline__ C div(C a, C b) {
    const C r = rcp(b);
    const C q = a * r;
    const C q2 = fmaf(r, fmaf(-b, q, a), q);
    return isfinite(q2) ? q2 : q;
  }
  __device__ static __forceinline__ C sq(C a) { return a * a; }
  __device__ static __forceinline__ C ex(C a) { return expf(a); }
  __device__ static __forceinline__ C sqr(C a) { return sqrtf(a); }
  // branchless: e = exp(-|x|) never overflows; one correctly rounded reciprocal
  // (~2 ulp overall) instead of a divergent IEEE division with its slow path
  __device__ static __forceinline__ C silu(C x) {
    const C e = expf(-fabsf(x));
    const C r = rcp(1.0f + e);  // 1 + e in [1, 2]: no special cases
    return x * (x >= 0.0f ? r : e * r);
  }
  __device__ static __forceinline__ C scale(C x, C c) { return c * x; }
  __device__ static __forceinline__ A azero() { return 0.0f; }
  __device__ static __forceinline__ void aadd(A& a, C v) { a += v; }
  __device__ static __forceinline__ void amerge(A& a, A b) { a += b; }
  __device__ static __forceinline__ void mac(A& a, C x, C y) { a = fmaf(x, y, a); }
  __device__ static __forceinline__ C fin(A a) { return a; }
};

// bf16 storage (raw bits), fp32 compute; round-to-nearest-even on store.
struct NBF16 : NF32 {
  typedef u16 S;
  static constexpr int VEC = 8;
  __device__ static __forceinline__ C ld(S v) { return __uint_as_float(((u32)v) << 16); }
  __device__ static __forceinline__ S st(C f) {
    u32 u = __float_as_uint(f);
    if ((u & 0x7fffffffu) > 0x7f800000u) return (S)0x7fc0;
    u += 0x7fffu + ((u >> 16) & 1u);
    return (S)(u >> 16);
  }
};

struct NFF {
  typedef u32 S; typedef u32 C; typedef u64 A;
  static constexpr int VEC = 4;
  __device__ static __forceinline__ C ld(S v) { return v; }
  __device__ static __forceinline__ S st(C v) { return v; }
  __device__ static __forceinline__ C zero() { return 0u; }
  __device__ static __forceinline__ C nan() { return 0xFFFFFFFFu; }  // not a residue
  __device__ static __forceinline__ C add(C a, C b) { return ff_add(a, b); }
  __device__ static __forceinline__ C mul(C a, C b) { return ff_mul(a, b); }
  __device__ static __forceinline__ C div(C a, C b) { return ff_mul(a, ff_inv(b)); }
  __device__ static __forceinline__ C sq(C a) { return ff_mul(a, a); }
  __device__ static __forceinline__ C ex(C a) { return ff_hash(a, FF_KEY_EXP); }
  __device__ static __forceinline__ C sqr(C a) { return ff_hash(a, FF_KEY_SQRT); }
  __device__ static __forceinline__ C silu(C a) { return ff_hash(a, FF_KEY_SILU); }
  __device__ static __forceinline__ C scale(C x, C c) { return ff_mul(c, x); }
  __device__ static __forceinline__ A azero() { return 0ull; }
  __device__ static __forceinline__ void aadd(A& a, C v) { a += v; }      // < 2^31 per term
  __device__ static __forceinline__ void amerge(A& a, A b) { a += b; }
  __device__ static __forceinline__ void mac(A& a, C x, C y) { a += ff_mul_lazy(x, y); }  // < 2^32 per term
  __device__ static __forceinline__ C fin(A a) { return modp64(a); }
  // streamed contractions: raw 62-bit products accumulated with one IMAD.WIDE each,
  // folded below 2^34 every FOLD products ((2^31-1)^2 * 3 + 2^34 < 2^64)
  __device__ static __forceinline__ C inv(C a) { return ff_inv(a); }
  static constexpr int FOLD = 3;
  __device__ static __forceinline__ void mac_raw(A& a, C x, C y) { a += (u64)x * y; }
  __device__ static __forceinline__ void fold(A& a) { a = (a & P) + (a >> 31); }
};
template <class N> struct has_fold { static constexpr bool v = false; };
template <> struct has_fold<NFF> { static constexpr bool v = true; };

// Storage -> compute conversion usable on either a smem tile (C) or a global view (S).
template <class X, class Y> struct same_t { static constexpr bool v = false; };
template <class X> struct same_t<X, X> { static constexpr bool v = true; };
template <class N, class T> __device__ __forceinline__ typename N::C cvs(T v) {
  if constexpr (same_t<T, typename N::C>::v) return v;
  else return N::ld(v);
}

// ---------------------------------------------------------------------------
// Warp / cluster primitives

__device__ __forceinline__ u32 atom_add_acq_rel(u32* p, u32 v) {
  u32 old;
  asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ u64 gtimer() {
  u64 t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ u32 cluster_rank() {
  u32 r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
template <class T> __device__ __forceinline__ const T* peer_ptr(const T* p, u32 rank) {
  u64 out;
  asm volatile("mapa.u64 %0, %1, %2;" : "=l"(out) : "l"((u64)p), "r"(rank));
  return (const T*)out;
}

template <class T> __device__ __forceinline__ T shfl_xor(T v, int off, u32 mask) {
  return __shfl_xor_sync(mask, v, off);
}

__device__ __forceinline__ uint4 ldg_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ uint2 ldg_stream8(const void* p) {
  uint2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  return r;
}

// ---------------------------------------------------------------------------
// Tile movement: strided rank-4 global view <-> dense smem tile.
// VEC > 1 only when the planner proved 16-byte alignment of every row start.

// Register prefetch of a small loop-body tile (at most 8 loads per thread): the
// next iteration's global loads are issued right after this iteration's tile is
// written to shared memory, so their latency hides behind the rest of the
// iteration instead of opening it (A's split-KV loops: one Kt column and one V
// row per key, two dependent round trips per iteration otherwise).
// Element e of a 16-byte vector as the storage type (selects, no local memory).
template <class S> __device__ __forceinline__ S vec_pick(const uint4& q, int e);
template <> __device__ __forceinline__ u16 vec_pick<u16>(const uint4& q, int e) {
  const u32 w = (e & 4) ? ((e & 2) ? q.w : q.z) : ((e & 2) ? q.y : q.x);
  return (u16)((e & 1) ? (w >> 16) : (w & 0xffffu));
}
template <> __device__ __forceinline__ u32 vec_pick<u32>(const uint4& q, int e) {
  return (e & 2) ? ((e & 1) ? q.w : q.z) : ((e & 1) ? q.y : q.x);
}
template <> __device__ __forceinline__ float vec_pick<float>(const uint4& q, int e) {
  return __uint_as_float(vec_pick<u32>(q, e));
}
template <> __device__ __forceinline__ double vec_pick<double>(const uint4& q, int e) {
  return e ? __hiloint2double((int)q.w, (int)q.z) : __hiloint2double((int)q.y, (int)q.x);
}

// Column strip of a loop that steps a contiguous innermost dim T elements per
// iteration (A's Kt.3.i: one key column [.., 128, 1] per iteration, every element
// in its own sector): each lane loads 16 bytes of its rows -- the next G / T
// iterations' columns, G = 16 / sizeof(S) -- once per G / T iterations, and every
// iteration writes its columns from registers.  G / T-fold fewer L1 wavefronts.
template <class N, int D0, int D1, int D2, int T, i64 S0, i64 S1, i64 S2, int NT>
struct TileStrip {
  typedef typename N::S S;
  static constexpr int ROWS = D0 * D1 * D2;
  static constexpr int IT = (ROWS + NT - 1) / NT;
  uint4 u[IT];

  __device__ __forceinline__ void load(const S* __restrict__ src) {
#pragma unroll
    for (int j = 0; j < IT; ++j) {
      const int r = threadIdx.x + j * NT;
      if (r < ROWS) {
        const int i2 = r % D2, i1 = (r / D2) % D1, i0 = r / (D2 * D1);
        u[j] = *reinterpret_cast<const uint4*>(src + i0 * S0 + i1 * S1 + i2 * S2);
      }
    }
  }
  // iteration e of the strip: its T consecutive elements of every row
  __device__ __forceinline__ void store(typename N::C* __restrict__ dst, int e) const {
#pragma unroll
    for (int j = 0; j < IT; ++j) {
      const int r = threadIdx.x + j * NT;
      if (r < ROWS) {
#pragma unroll
        for (int t = 0; t < T; ++t) dst[r * T + t] = N::ld(vec_pick<S>(u[j], e * T + t));
      }
    }
  }
};

template <class N, int D0, int D1, int D2, int D3, i64 S0, i64 S1, i64 S2, i64 S3, int VEC, int NT>
struct TilePf {
  typedef typename N::S S;
  static constexpr int ROWS = D0 * D1 * D2;
  static constexpr int V3 = VEC > 1 ? D3 / VEC : D3;
  static constexpr int TOT = ROWS * V3;
  static constexpr int IT = (TOT + NT - 1) / NT;
  union U { uint4 q; S s[VEC > 1 ? VEC : 1]; };
  U u[VEC > 1 ? IT : 1];
  S r[VEC > 1 ? 1 : IT];

  __device__ __forceinline__ void load(const S* __restrict__ src) {
#pragma unroll
    for (int j = 0; j < IT; ++j) {
      const int e = threadIdx.x + j * NT;
      if (e < TOT) {
        const int v = e % V3;
        const int rr = e / V3;
        const int i2 = rr % D2, i1 = (rr / D2) % D1, i0 = rr / (D2 * D1);
        if constexpr (VEC > 1)
          u[j].q = *reinterpret_cast<const uint4*>(src + i0 * S0 + i1 * S1 + i2 * S2 + (i64)v * VEC);
        else
          r[j] = src[i0 * S0 + i1 * S1 + i2 * S2 + (i64)v * S3];
      }
    }
  }
  __device__ __forceinline__ void store(typename N::C* __restrict__ dst) const {
#pragma unroll
    for (int j = 0; j < IT; ++j) {
      const int e = threadIdx.x + j * NT;
      if (e < TOT) {
        if constexpr (VEC > 1) {
          const int v = e % V3, rr = e / V3;
#pragma unroll
          for (int t = 0; t < VEC; ++t) dst[rr * D3 + v * VEC + t] = N::ld(u[j].s[t]);
        } else {
          dst[e] = N::ld(r[j]);
        }
      }
    }
  }
};

template <class N, int D0, int D1, int D2, int D3, i64 S0, i64 S1, i64 S2, i64 S3, int VEC, int NT>
__device__ __forceinline__ void load_tile(typename N::C* __restrict__ dst, const typename N::S* __restrict__ src) {
  typedef typename N::S S;
  constexpr int ROWS = D0 * D1 * D2;
  if constexpr (VEC > 1) {
    // batches of up to 8 independent 16-byte loads per thread in flight (a cold
    // prologue load is latency-bound, not bandwidth-bound)
    constexpr int V3 = D3 / VEC;
    constexpr int TOT = ROWS * V3;
    constexpr int IT = (TOT + NT - 1) / NT;
    constexpr int BT = IT < 8 ? IT : 8;
    for (int b = 0; b < IT; b += BT) {
      union U { uint4 q; S s[VEC]; } u[BT];
#pragma unroll
      for (int j = 0; j < BT; ++j) {
        const int e = threadIdx.x + (b + j) * NT;
        if (b + j < IT && e < TOT) {
          const int v = e % V3;
          const int r = e / V3;
          const int i2 = r % D2, i1 = (r / D2) % D1, i0 = r / (D2 * D1);
          u[j].q = *reinterpret_cast<const uint4*>(src + i0 * S0 + i1 * S1 + i2 * S2 + (i64)v * VEC);
        }
      }
#pragma unroll
      for (int j = 0; j < BT; ++j) {
        const int e = threadIdx.x + (b + j) * NT;
        if (b + j < IT && e < TOT) {
          const int v = e % V3;
          const int r = e / V3;
#pragma unroll
          for (int t = 0; t < VEC; ++t) dst[r * D3 + v * VEC + t] = N::ld(u[j].s[t]);
        }
      }
    }
  } else {
    // scalar (strided / unaligned) tiles: batches of 8 independent loads in flight
    // per thread too (a column tile of A's split-KV loop is 2048 strided elements
    // per iteration; one load at a time made each iteration ~8 round trips long)
    constexpr int TOT = ROWS * D3;
    constexpr int IT = (TOT + NT - 1) / NT;
    constexpr int BT = IT < 8 ? IT : 8;
    for (int b = 0; b < IT; b += BT) {
      S u[BT];
#pragma unroll
      for (int j = 0; j < BT; ++j) {
        const int e = threadIdx.x + (b + j) * NT;
        if (b + j < IT && e < TOT) {
          const int i3 = e % D3;
          const int r = e / D3;
          const int i2 = r % D2, i1 = (r / D2) % D1, i0 = r / (D2 * D1);
          u[j] = src[i0 * S0 + i1 * S1 + i2 * S2 + (i64)i3 * S3];
        }
      }
#pragma unroll
      for (int j = 0; j < BT; ++j) {
        const int e = threadIdx.x + (b + j) * NT;
        if (b + j < IT && e < TOT) dst[e] = N::ld(u[j]);
      }
    }
  }
}

template <class N, int D0, int D1, int D2, int D3, i64 S0, i64 S1, i64 S2, i64 S3, int VEC, int NT>
__device__ __forceinline__ void store_tile(typename N::S* __restrict__ dst, const typename N::C* __restrict__ src) {
  typedef typename N::S S;
  constexpr int ROWS = D0 * D1 * D2;
  if constexpr (VEC > 1) {
    constexpr int V3 = D3 / VEC;
    for (int e = threadIdx.x; e < ROWS * V3; e += NT) {
      const int v = e % V3;
      const int r = e / V3;
      const int i2 = r % D2, i1 = (r / D2) % D1, i0 = r / (D2 * D1);
      union { uint4 q; S s[VEC]; } u;
#pragma unroll
      for (int t = 0; t < VEC; ++t) u.s[t] = N::st(src[r * D3 + v * VEC + t]);
      *reinterpret_cast<uint4*>(dst + i0 * S0 + i1 * S1 + i2 * S2 + (i64)v * VEC) = u.q;
    }
  } else {
    for (int e = threadIdx.x; e < ROWS * D3; e += NT) {
      const int i3 = e % D3;
      const int r = e / D3;
      const int i2 = r % D2, i1 = (r / D2) % D1, i0 = r / (D2 * D1);
      dst[i0 * S0 + i1 * S1 + i2 * S2 + (i64)i3 * S3] = N::st(src[e]);
    }
  }
}

// ---------------------------------------------------------------------------
// sum over one axis (keepdims).  TPO threads cooperate on each output value.

template <int A, int B> struct cmin { static constexpr int v = A < B ? A : B; };
__host__ __device__ constexpr int pow2_floor(int x) { int p = 1; while (p * 2 <= x) p *= 2; return p; }
__host__ __device__ constexpr int pow2_ceil(int x) { int p = 1; while (p < x) p *= 2; return p; }

template <class N, int D0, int D1, int D2, int D3, int AX, int NT>
__device__ __forceinline__ void sum_axis(typename N::C* __restrict__ dst, const typename N::C* __restrict__ src) {
  typedef typename N::A Acc;
  constexpr int DIMS[4] = {D0, D1, D2, D3};
  constexpr int L = DIMS[AX];
  constexpr int INNER = (AX == 0 ? D1 * D2 * D3 : AX == 1 ? D2 * D3 : AX == 2 ? D3 : 1);
  constexpr int OUT = D0 * D1 * D2 * D3 / L;
  constexpr int TPO0 = pow2_floor(NT / OUT > 0 ? NT / OUT : 1);
  constexpr int TPO = TPO0 > pow2_ceil(L) ? pow2_ceil(L) : TPO0;  // threads per output
  constexpr int NW = NT / 32;
  const int tid = threadIdx.x;
  if constexpr (TPO <= 32) {
    constexpr int GROUPS = NT / TPO;
    const int lane = tid & 31;
    const u32 gmask = (TPO == 32) ? 0xffffffffu : (((1u << TPO) - 1u) << (lane & ~(TPO - 1)));
    for (int o = tid / TPO; o < OUT; o += GROUPS) {
      const int outer = o / INNER, inner = o % INNER;
      const typename N::C* p = src + outer * (L * INNER) + inner;
      Acc acc = N::azero();
      for (int k = tid % TPO; k < L; k += TPO) N::aadd(acc, p[k * INNER]);
#pragma unroll
      for (int off = TPO / 2; off > 0; off >>= 1) N::amerge(acc, shfl_xor(acc, off, gmask));
      if ((tid % TPO) == 0) dst[o] = N::fin(acc);
    }
  } else {
    // OUT < NW: several warps per output, combined through smem.
    constexpr int WPO = TPO / 32;
    __shared__ Acc part[NW];
    const int w = tid >> 5, lane = tid & 31;
    const int o = w / WPO;
    Acc acc = N::azero();
    if (o < OUT) {
      const int outer = o / INNER, inner = o % INNER;
      const typename N::C* p = src + outer * (L * INNER) + inner;
      for (int k = (w % WPO) * 32 + lane; k < L; k += TPO) N::aadd(acc, p[k * INNER]);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) N::amerge(acc, shfl_xor(acc, off, 0xffffffffu));
    if (lane == 0) part[w] = acc;
    csync<NT>();
    if (tid < OUT) {
      Acc t = N::azero();
      for (int q = 0; q < WPO; ++q) N::amerge(t, part[tid * WPO + q]);
      dst[tid] = N::fin(t);
    }
  }
}

// ---------------------------------------------------------------------------
// Generic batched contraction: out[b0][b1][m][n] = sum_k A(b0,b1,m,k) * B(b0,b1,k,n).
// A and B are either smem tiles (TA/TB = N::C) or global views (N::S), given by
// compile-time strides (0 for broadcast dims).  TPO lanes split k.

__host__ __device__ constexpr int pow2_divisor(int m, int cap) {
  int r = 1;
  while (r * 2 <= cap && m % (r * 2) == 0) r *= 2;
  return r;
}
__host__ __device__ constexpr int divisor_upto(int m, int cap) {
  int r = cap < m ? cap : m;
  while (m % r) --r;
  return r;
}

// Multi-value warp reduction: R (power of two) partial sums per lane in, the full
// sum of value ((lane&16)?R/2:0) + ((lane&8)?R/4:0) + ... out -- R/2 + R/4 + ...
// + the remaining single levels shuffles instead of 5 R.
template <class N, int R>
__device__ __forceinline__ typename N::A warp_reduce_multi(typename N::A (&v)[R], int lane) {
  typedef typename N::A Acc;
#pragma unroll
  for (int lvl = 0; lvl < 5; ++lvl) {
    const int off = 16 >> lvl;
    const int r = R >> lvl;
    if (r > 1) {
      const bool up = (lane & off) != 0;
#pragma unroll
      for (int i = 0; i < r / 2; ++i) {
        const Acc send = up ? v[i] : v[i + r / 2];
        Acc keep = up ? v[i + r / 2] : v[i];
        N::amerge(keep, shfl_xor(send, off, 0xffffffffu));
        v[i] = keep;
      }
    } else {
      N::amerge(v[0], shfl_xor(v[0], off, 0xffffffffu));
    }
  }
  return v[0];
}

template <class N, class TA, class TB, int B0, int B1, int M, int K, int NN,
          i64 SA0, i64 SA1, i64 SA2, i64 SA3, i64 SB0, i64 SB1, i64 SB2, i64 SB3, int NT>
__device__ __forceinline__ void mm_generic(typename N::C* __restrict__ out, const TA* __restrict__ A,
                                           const TB* __restrict__ B) {
  typedef typename N::A Acc;
  typedef typename N::C C;
  constexpr int OUT = B0 * B1 * M * NN;
  constexpr int TPO0 = pow2_floor(NT / OUT > 0 ? NT / OUT : 1);
  constexpr int TPO1 = TPO0 > 32 ? 32 : TPO0;
  // dot-product form (both operands contiguous along k): a whole warp per output,
  // lanes on consecutive k -- conflict-free shared-memory reads.  With few lanes per
  // output, lanes of different rows hit one bank (row stride a multiple of 32
  // words): A's Q @ Kt-column step took 12.7 us per loop iteration.
  constexpr bool DOT = SA3 == 1 && SB2 == 1 && K >= 32;
  // smem operands, K a multiple of 32: a warp takes R rows sharing one B column
  // (B contiguous along k) or all NB = NN columns of a row-major B tile (k stride
  // NN <= 4, e.g. A's two keys per iteration), the k values held in registers
  // (chunks of up to 8 per lane) and reused by all R rows, one multi-value
  // reduction for the R x NB sums (A's Q @ Kt-column loop step: 7.8 us as a
  // warp-per-output loop of 4 products and 5 shuffles each)
  constexpr bool ROWB = SA3 == 1 && SB3 == 1 && SB2 == NN && NN > 1 && NN <= 4 && (NN & (NN - 1)) == 0;
#ifdef SGM_NO_DOT2
  if constexpr (false) {
#else
  if constexpr ((DOT || ROWB) && K % 32 == 0 && same_t<TA, C>::v && same_t<TB, C>::v) {
#endif
    constexpr int NB = DOT ? 1 : NN;
    constexpr int R = pow2_divisor(M, 8 / NB);
    constexpr int V = R * NB;
    constexpr int KS = K / 32;
    constexpr int KC = divisor_upto(KS, 8 / NB);
    constexpr int TASKS = B0 * B1 * (NN / NB) * (M / R);
    const int tid = threadIdx.x, lane = tid & 31;
    for (int t = tid >> 5; t < TASKS; t += NT / 32) {
      int r = t;
      const int mg = r % (M / R); r /= (M / R);
      const int n0 = (r % (NN / NB)) * NB; r /= (NN / NB);
      const int b1 = r % B1, b0 = r / B1;
      const C* pa = A + b0 * SA0 + b1 * SA1 + (i64)(mg * R) * SA2 + lane;
      const C* pb = B + b0 * SB0 + b1 * SB1 + (i64)n0 * SB3 + (i64)lane * SB2;
      Acc v[V];
#pragma unroll
      for (int i = 0; i < V; ++i) v[i] = N::azero();
      for (int c = 0; c < KS; c += KC) {
        C bv[KC][NB];
#pragma unroll
        for (int s = 0; s < KC; ++s)
#pragma unroll
          for (int q = 0; q < NB; ++q) bv[s][q] = pb[(i64)(c + s) * 32 * SB2 + q];
#pragma unroll
        for (int i = 0; i < R; ++i) {
#pragma unroll
          for (int s = 0; s < KC; ++s) {
            const C av = pa[(i64)i * SA2 + (c + s) * 32];
#pragma unroll
            for (int q = 0; q < NB; ++q) {
              if constexpr (has_fold<N>::v) {
                N::mac_raw(v[i * NB + q], av, bv[s][q]);
                if (s % 3 == 2 || s == KC - 1) N::fold(v[i * NB + q]);
              } else {
                N::mac(v[i * NB + q], av, bv[s][q]);
              }
            }
          }
        }
      }
      const Acc tot = warp_reduce_multi<N, V>(v, lane);
      if ((lane & (32 / V - 1)) == 0) {
        int idx = 0;
#pragma unroll
        for (int lvl = 0; (V >> (lvl + 1)) > 0; ++lvl) idx += ((lane >> (4 - lvl)) & 1) * (V >> (lvl + 1));
        out[(((i64)b0 * B1 + b1) * M + mg * R + idx / NB) * NN + n0 + idx % NB] = N::fin(tot);
      }
    }
    return;
  }
  constexpr int TPO2 = DOT ? 32 : TPO1;
  constexpr int TPO = TPO2 > pow2_ceil(K) ? pow2_ceil(K) : TPO2;
  constexpr int GROUPS = NT / TPO;
  const int tid = threadIdx.x, lane = tid & 31;
  const u32 gmask = (TPO == 32) ? 0xffffffffu : (((1u << TPO) - 1u) << (lane & ~(TPO - 1)));
  for (int o = tid / TPO; o < OUT; o += GROUPS) {
    const int n = o % NN;
    int r = o / NN;
    const int m = r % M; r /= M;
    const int b1 = r % B1, b0 = r / B1;
    const TA* pa = A + b0 * SA0 + b1 * SA1 + (i64)m * SA2;
    const TB* pb = B + b0 * SB0 + b1 * SB1 + (i64)n * SB3;
    Acc acc = N::azero();
    int k = tid % TPO;
    if constexpr (has_fold<N>::v) {  // finite field: 3 raw products per fold
      for (; k + 2 * TPO < K; k += 3 * TPO) {
        N::mac_raw(acc, cvs<N>(pa[(i64)k * SA3]), cvs<N>(pb[(i64)k * SB2]));
        N::mac_raw(acc, cvs<N>(pa[(i64)(k + TPO) * SA3]), cvs<N>(pb[(i64)(k + TPO) * SB2]));
        N::mac_raw(acc, cvs<N>(pa[(i64)(k + 2 * TPO) * SA3]), cvs<N>(pb[(i64)(k + 2 * TPO) * SB2]));
        N::fold(acc);
      }
    }
    for (; k < K; k += TPO) N::mac(acc, cvs<N>(pa[(i64)k * SA3]), cvs<N>(pb[(i64)k * SB2]));
#pragma unroll
    for (int off = TPO / 2; off > 0; off >>= 1) N::amerge(acc, shfl_xor(acc, off, gmask));
    if ((tid % TPO) == 0) out[o] = N::fin(acc);
  }
}

// ---------------------------------------------------------------------------
// Streamed GEMV-like contraction: A small in smem ([B0][B1][M][K], strides SA*),
// B a global view streamed once (row k contiguous along n), output [B0][B1][M][NN].
// Work item = (batch, vector of VN columns); KS threads split k (interleaved),
// partials combined with warp shuffles (ks lanes inside a warp) then smem.
// `red` is a smem scratch of at least red_elems() accumulators.

template <int NV, int KS, bool SHFL> struct gemv_layout {
  // lanes: t = nv + NV*ks + NV*KS*item_hi
  static constexpr int KS_IN_WARP = (!SHFL || NV >= 32) ? 1 : ((32 / NV) < KS ? (32 / NV) : KS);
  static constexpr int KS_OUT = KS / KS_IN_WARP;
};

// A is first re-laid k-major into `at` ([A0*A1][K][M], A0/A1 = A's own batch extents)
// so each k step reads the M values of a column with 16-byte shared loads.
template <class N, class TB, int B0, int B1, int M, int K, int NN, i64 SA0, i64 SA1, i64 SA2, i64 SA3,
          i64 SB0, i64 SB1, i64 SB2, int VN, int KS, int UNR, bool SHFL, int NT>
__device__ __forceinline__ void mm_gemv(typename N::C* __restrict__ out, const typename N::C* __restrict__ A,
                                        const TB* __restrict__ B, typename N::A* __restrict__ red,
                                        typename N::C* __restrict__ at) {
  typedef typename N::A Acc;
  typedef typename N::C C;
  constexpr int NV = NN / VN;
  constexpr int ITEMS = B0 * B1 * NV;
  constexpr int WORK = ITEMS * KS;
  constexpr int A0 = SA0 ? B0 : 1, A1 = SA1 ? B1 : 1;
  typedef gemv_layout<NV, KS, SHFL> LY;
  static_assert(NN % VN == 0, "VN must divide NN");
  const int tid = threadIdx.x;
  for (int e = tid; e < A0 * A1 * K * M; e += NT) {
    const int m = e % M;
    const int k = (e / M) % K;
    const int ab = e / (M * K);
    const int a1 = ab % A1, a0 = ab / A1;
    at[e] = A[a0 * SA0 + a1 * SA1 + (i64)m * SA2 + (i64)k * SA3];
  }
  csync<NT>();
  for (int w = tid; w < WORK; w += NT) {
    const int nv = w % NV;
    const int ks = (w / NV) % KS;
    const int bi = w / (NV * KS);
    const int b1 = bi % B1, b0 = bi / B1;
    const C* pa = at + (i64)((SA0 ? b0 : 0) * A1 + (SA1 ? b1 : 0)) * K * M;
    const TB* pb = B + b0 * SB0 + b1 * SB1 + nv * VN;
    Acc acc[M][VN];
#pragma unroll
    for (int m = 0; m < M; ++m)
#pragma unroll
      for (int v = 0; v < VN; ++v) acc[m][v] = N::azero();
    constexpr int STEP = KS * UNR;
    for (int k0 = ks; k0 < K; k0 += STEP) {
      TB bv[UNR][VN];
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const int k = k0 + u * KS;
        if (K % STEP == 0 || k < K) {
          const TB* src = pb + (i64)k * SB2;
          if constexpr (sizeof(TB) * VN == 16) {
            union { uint4 q; TB s[VN]; } t; t.q = ldg_stream(src);
#pragma unroll
            for (int v = 0; v < VN; ++v) bv[u][v] = t.s[v];
          } else if constexpr (sizeof(TB) * VN == 8) {
            union { uint2 q; TB s[VN]; } t; t.q = ldg_stream8(src);
#pragma unroll
            for (int v = 0; v < VN; ++v) bv[u][v] = t.s[v];
          } else {
#pragma unroll
            for (int v = 0; v < VN; ++v) bv[u][v] = src[v];
          }
        } else {
#pragma unroll
          for (int v = 0; v < VN; ++v) bv[u][v] = TB(0);
        }
      }
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const int k = k0 + u * KS;
        if (K % STEP == 0 || k < K) {
          C bc[VN];
#pragma unroll
          for (int v = 0; v < VN; ++v) bc[v] = cvs<N>(bv[u][v]);
          C av[M];
          if constexpr ((M * sizeof(C)) % 16 == 0) {
#pragma unroll
            for (int q = 0; q < (int)(M * sizeof(C) / 16); ++q)
              *reinterpret_cast<uint4*>(&av[q * (16 / sizeof(C))]) =
                  *reinterpret_cast<const uint4*>(pa + (i64)k * M + q * (16 / sizeof(C)));
          } else {
#pragma unroll
            for (int m = 0; m < M; ++m) av[m] = pa[(i64)k * M + m];
          }
#pragma unroll
          for (int m = 0; m < M; ++m) {
#pragma unroll
            for (int v = 0; v < VN; ++v) {
              if constexpr (has_fold<N>::v) N::mac_raw(acc[m][v], av[m], bc[v]);
              else N::mac(acc[m][v], av[m], bc[v]);
            }
          }
        }
        if constexpr (has_fold<N>::v) {
          if (u % N::FOLD == N::FOLD - 1 || u == UNR - 1) {
#pragma unroll
            for (int m = 0; m < M; ++m)
#pragma unroll
              for (int v = 0; v < VN; ++v) N::fold(acc[m][v]);
          }
        }
      }
    }
    // reduce the KS_IN_WARP partials living in one warp (lanes NV apart)
    if constexpr (LY::KS_IN_WARP > 1) {
#pragma unroll
      for (int off = NV * LY::KS_IN_WARP / 2; off >= NV; off >>= 1)
#pragma unroll
        for (int m = 0; m < M; ++m)
#pragma unroll
          for (int v = 0; v < VN; ++v) N::amerge(acc[m][v], shfl_xor(acc[m][v], off, 0xffffffffu));
    }
    const int ksw = ks % LY::KS_IN_WARP;
    if constexpr (LY::KS_OUT == 1) {
      if (ksw == 0) {
#pragma unroll
        for (int m = 0; m < M; ++m)
#pragma unroll
          for (int v = 0; v < VN; ++v) out[((i64)bi * M + m) * NN + nv * VN + v] = N::fin(acc[m][v]);
      }
    } else {
      if (ksw == 0) {
        const int kso = ks / LY::KS_IN_WARP;
        const int item = bi * NV + nv;
#pragma unroll
        for (int m = 0; m < M; ++m)
#pragma unroll
          for (int v = 0; v < VN; ++v) red[(((i64)kso * ITEMS + item) * M + m) * VN + v] = acc[m][v];
      }
    }
  }
  if constexpr (LY::KS_OUT > 1) {
    csync<NT>();
    for (int e = tid; e < ITEMS * M * VN; e += NT) {
      Acc t = N::azero();
#pragma unroll 4
      for (int q = 0; q < LY::KS_OUT; ++q) N::amerge(t, red[(i64)q * ITEMS * M * VN + e]);
      const int v = e % VN;
      const int m = (e / VN) % M;
      const int item = e / (VN * M);
      const int nv = item % NV, bi = item / NV;
      out[((i64)bi * M + m) * NN + nv * VN + v] = N::fin(t);
    }
  }
}

// ---------------------------------------------------------------------------
// tcgen05 streamed GEMV (bf16 weights, fp32 accumulate in TMEM).
//   out[b][m][n] = sum_k A[b][m][k] * B[b][k][n],  M <= 16 (padded to the MMA N=16)
// Swap-AB: the weight slice is the MMA A operand (M_mma = 128 output columns,
// MN-major), A^T is the MMA B operand (N_mma = 16, K-major).  Weights stream
// through an S-stage smem ring filled by cp.async (16-byte chunks, zero-filled
// past NN) in the canonical no-swizzle UMMA layout:
//   W^T core matrix = 8 k-rows x 16 B (8 n); n-groups at SBO = 128 B,
//   k-groups at LBO = 2048 B (one 128-column tile).
//   X^T core matrix = 8 m-rows x 16 B (8 k); m-groups at SBO = 128 B,
//   k-groups at LBO = 256 B.
// One thread issues the MMAs; tcgen05.commit arrives on the stage's mbarrier,
// which gates re-filling that stage.  Descriptor / instruction-descriptor bit
// layouts follow CUTLASS cute/arch/mma_sm100_desc.hpp (SmemDescriptor, InstrDescriptor).

__device__ __forceinline__ u32 smem_u32(const void* p) { return (u32)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(u64* b, u32 cnt) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt) : "memory");
}
// Watchdog (per module): every wait on an asynchronous completion (TMA
// transaction bytes, MMA commits, remote cluster arrivals) is bounded.  A wait
// that exceeds SGM_WD_NS (2 s) sets sgm_wd_flag and gives up, so a broken candidate
// ends (with garbage) instead of hanging the GPU; the runtime reads the flag
// (sgm_plan_watchdog) and the sweep records "run: timeout" (interp.py:278-281).
#ifndef SGM_WD_NS
#define SGM_WD_NS 2000000000ull
#endif
}  // namespace sgm
extern "C" __device__ unsigned sgm_wd_flag;  // C linkage: looked up by name (cuModuleGetGlobal)
namespace sgm {
__device__ __forceinline__ u64 wd_now() {
  u64 t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __noinline__ void wd_trip() { atomicOr(&sgm_wd_flag, 1u); }
// Waits on an mbarrier phase (SGM_WD_MODE).  4 (default): one probe on the fast
// path, then probes until SGM_WD_NS (2 s) of %globaltimer elapsed, then the
// module's watchdog flag is set and the wait gives up (a probe-count bound
// tripped on legitimately long waits -- a producer waiting for ring slots while
// the consumer runs a long loop -- and corrupted the ring).  Measured vs the
// canonical unbounded loop (0): G +2.4%, L +2%, A +0.4%, R +7%; counted loops
// in the fast path cost 30%: ptxas only moves the canonical retry loop out of
// line.  Plans with hints.no_wd compile mode 0.
#ifndef SGM_WD_MODE
#define SGM_WD_MODE 4
#endif
__device__ __forceinline__ void mbar_wait(u64* b, u32 parity) {
#if defined(SGM_NO_WD) || SGM_WD_MODE == 0
  asm volatile(
      "{\n\t.reg .pred P1;\n\tLAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE;\n\tbra LAB_WAIT;\n\tDONE:\n\t}" ::"r"(smem_u32(b)), "r"(parity) : "memory");
#else
  // fast path: one probe and a branch; the slow path (out of the fall-through)
  // re-probes until %globaltimer says SGM_WD_NS elapsed, then sets the module's
  // watchdog flag and gives up; once the flag is set, later waits drain at once
  asm volatile(
      "{\n\t.reg .pred P1;\n\t.reg .u64 t0, t1;\n\t.reg .u32 f;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WD_SLOW;\n\tbra.uni WD_DONE;\n\t"
      "WD_SLOW:\n\t"
      "ld.volatile.global.u32 f, [%2];\n\tsetp.ne.u32 P1, f, 0;\n\t@P1 bra WD_DONE;\n\t"
      "mov.u64 t0, %%globaltimer;\n\t"
      "WD_LOOP:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra WD_DONE;\n\t"
      "mov.u64 t1, %%globaltimer;\n\tsub.u64 t1, t1, t0;\n\tsetp.lt.u64 P1, t1, %3;\n\t@P1 bra WD_LOOP;\n\t"
      "red.relaxed.gpu.global.or.b32 [%2], 1;\n\t"
      "WD_DONE:\n\t}" ::"r"(smem_u32(b)), "r"(parity), "l"(&sgm_wd_flag), "l"((u64)SGM_WD_NS)
      : "memory");
#endif
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void cp_async16(void* dst, const void* src, u32 bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N> __device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ u64 umma_desc(u32 saddr, u32 lbo, u32 sbo) {
  // start>>4 [0,14) | LBO>>4 [16,30) | SBO>>4 [32,46) | version 1 [46,48) | SWIZZLE_NONE [61,64)
  return (u64)((saddr >> 4) & 0x3FFFu) | ((u64)((lbo >> 4) & 0x3FFFu) << 16) |
         ((u64)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}
// kind::f16, A=B=bf16, D=f32, A MN-major, B K-major, N=16, M=128
constexpr u32 UMMA_IDESC_BF16_M128_N16 =
    (1u << 4) | (1u << 7) | (1u << 10) | (1u << 15) | ((16u >> 3) << 17) | ((128u >> 4) << 24);

__device__ __forceinline__ void umma_bf16(u32 tmem_d, u64 adesc, u64 bdesc, u32 idesc, u32 acc) {
  u32 z = 0;
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc), "r"(z), "r"(z), "r"(z), "r"(z));
}
__device__ __forceinline__ void umma_commit(u64* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld16(u32 taddr, u32* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
// TMEM allocation by warp 0 (once per kernel); the base address lands in *slot.
template <int NT> __device__ __forceinline__ u32 tmem_alloc(u32* slot, u32 ncols) {
  if ((threadIdx.x >> 5) == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)), "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  csync<NT>();
  tc_fence_after();
  return *(volatile u32*)slot;
}
template <int NT> __device__ __forceinline__ void tmem_free(u32 base, u32 ncols) {
  tc_fence_before();
  csync<NT>();
  if ((threadIdx.x >> 5) == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "r"(ncols) : "memory");
}

template <int M, int K, i64 SA2, i64 SA3, int NT>
__device__ __forceinline__ void build_xb(u16* __restrict__ xb, const float* __restrict__ Ab);

template <int NN, int K, int KC, int S> struct gemv_tc_layout {
  static constexpr int NTL = (NN + 127) / 128;     // 128-column tiles
  static constexpr int STAGE = (KC / 8) * 2048;    // one (k-chunk, tile) stage
  static constexpr int XOFF = S * STAGE;
  static constexpr int BOFF = XOFF + 32 * K;
  static constexpr int BYTES = BOFF + 8 * S;
};

// Stages are (k-chunk kc, column tile t) pairs in kc-major order; D = S-2 stages
// are in flight, and re-filling a buffer waits only on the MMAs issued two
// stages earlier.  For M <= 8 the padded MMA rows 8..15 carry the bf16 residual
// of A (A = hi + lo), so a computed fp32 operand keeps ~16 mantissa bits.
template <int B0, int B1, int M, int K, int NN, i64 SA0, i64 SA1, i64 SA2, i64 SA3, i64 SB0, i64 SB1, i64 SB2,
          int KC, int S, int NT>
__device__ __forceinline__ void mm_gemv_tc(float* __restrict__ out, const float* __restrict__ A,
                                           const u16* __restrict__ B, unsigned char* __restrict__ work, u32 tmem) {
  typedef gemv_tc_layout<NN, K, KC, S> L;
  constexpr int NTL = L::NTL;
  constexpr int NST = (K / KC) * NTL;
  constexpr int D = S - 2;
  constexpr bool SPLIT = M <= 8;
  static_assert(K % KC == 0 && KC % 16 == 0 && M <= 16 && NN % 8 == 0 && S >= 3, "tcgen05 gemv shape");
  u64* bars = reinterpret_cast<u64*>(work + L::BOFF);
  u16* xb = reinterpret_cast<u16*>(work + L::XOFF);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int bi = 0; bi < B0 * B1; ++bi) {
    const int b1 = bi % B1, b0 = bi / B1;
    const float* Ab = A + b0 * SA0 + b1 * SA1;
    const u16* Bb = B + b0 * SB0 + b1 * SB1;
    build_xb<M, K, SA2, SA3, NT>(xb, Ab);  // A^T, K-major canonical (see build_xb)
    fence_async_smem();
    if (tid == 0) {
      for (int q = 0; q < S; ++q) mbar_init(&bars[q], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    csync<NT>();
    auto issue = [&](int s) {
      const int kc = s / NTL, t = s % NTL;
      unsigned char* st = work + (s % S) * L::STAGE;
      for (int c = tid; c < KC * 16; c += NT) {
        const int kk = c & 7;
        const int n8 = (c >> 3) & 15, k8 = c >> 7;
        const int k = kc * KC + k8 * 8 + kk;
        const int col = t * 128 + n8 * 8;
        const bool in = col < NN;
        cp_async16(st + k8 * 2048 + n8 * 128 + kk * 16, Bb + (i64)k * SB2 + (in ? col : 0), in ? 16u : 0u);
      }
      cp_async_commit();
    };
#pragma unroll 1
    for (int s = 0; s < D; ++s) {
      if (s < NST) issue(s);
      else cp_async_commit();
    }
#pragma unroll 1
    for (int s = 0; s < NST; ++s) {
      const int nx = s + D;  // refill: its buffer last served stage nx - S (MMAs issued 2 stages ago)
      if (nx < NST) {
        if (nx - S >= 0) mbar_wait(&bars[nx % S], ((nx - S) / S) & 1);
        issue(nx);
      } else {
        cp_async_commit();
      }
      cp_async_wait<D>();
      fence_async_smem();
      csync<NT>();
      if (tid == 0) {
        tc_fence_after();
        const int kc = s / NTL, t = s % NTL;
        const u32 st = smem_u32(work + (s % S) * L::STAGE);
        const u32 xs = smem_u32(xb);
#pragma unroll
        for (int ks = 0; ks < KC / 16; ++ks) {
          const u64 ad = umma_desc(st + ks * 4096, 2048, 128);
          const u64 bd = umma_desc(xs + ((kc * KC + ks * 16) >> 3) * 256, 256, 128);
          umma_bf16(tmem + t * 16, ad, bd, UMMA_IDESC_BF16_M128_N16, (kc | ks) != 0);
        }
        umma_commit(&bars[s % S]);
      }
    }
    cp_async_wait<0>();
    mbar_wait(&bars[(NST - 1) % S], ((NST - 1) / S) & 1);
    tc_fence_after();
    // epilogue: warp w reads TMEM lanes 32*(w%4).. of tile t (D[n][m]) and writes out[m][n]
    for (int t = warp >> 2; t < NTL; t += NT / 128) {
      u32 v[16];
      tmem_ld16(tmem + ((u32)((warp & 3) * 32) << 16) + t * 16, v);
      const int n = t * 128 + (warp & 3) * 32 + lane;
      if (n < NN) {
#pragma unroll
        for (int m = 0; m < M; ++m)
          out[((i64)bi * M + m) * NN + n] = SPLIT ? __uint_as_float(v[m]) + __uint_as_float(v[8 + m])
                                                  : __uint_as_float(v[m]);
      }
    }
    tc_fence_before();
    csync<NT>();
  }
}

// ---------------------------------------------------------------------------
// TMA-fed streaming of the large matmul operand (warp-specialised).
//
// A producer warp (one elected lane) walks the kernel's static sequence of
// streamed boxes — every view operand of every streamed matmul, loop
// iterations included — and issues cp.async.bulk.tensor loads into a ring of
// S slots of SLOT bytes (a kernel constant, 16 or 32 KB; full[s]: 1 arrival + tx bytes; empty[s]: consumer
// release).  It runs ahead of the compute warps across node and loop
// boundaries, so HBM streaming overlaps the candidate's elementwise, reduction
// and cluster-flush phases.  Producer and consumers enumerate the same stage
// sequence, each with its own running counter.


__device__ __forceinline__ void mbar_expect_tx(u64* b, u32 bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(u64* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void tma_load_4d(void* dst, const TmaDesc* tm, int c0, int c1, int c2, int c3, u64* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];" ::"r"(smem_u32(dst)),
      "l"((u64)tm), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_prefetch_desc(const TmaDesc* tm) {
  asm volatile("prefetch.tensormap [%0];" ::"l"((u64)tm) : "memory");
}
// producer: wait until slot (q % S) is free for its (q / S)-th fill
template <int S> __device__ __forceinline__ u32 ring_acquire(u64* empty, u32 q) {
  const u32 slot = q % S;
  if (q >= (u32)S) mbar_wait(&empty[slot], ((q / S) - 1u) & 1u);
  return slot;
}
// consumer: wait until the (q / S)-th fill of slot (q % S) has landed
template <int S> __device__ __forceinline__ u32 ring_wait(u64* full, u32 q) {
  const u32 slot = q % S;
  mbar_wait(&full[slot], (q / S) & 1u);
  return slot;
}
// UMMA smem descriptor, MN-major SWIZZLE_128B (layout type 2 on sm_100):
// LBO = byte stride between 64-element MN atoms, SBO = stride between 8-row K groups.
__device__ __forceinline__ u64 umma_desc_sw128(u32 saddr, u32 lbo, u32 sbo) {
  return (u64)((saddr >> 4) & 0x3FFFu) | ((u64)((lbo >> 4) & 0x3FFFu) << 16) |
         ((u64)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | (2ull << 61);
}

// Streamed bf16 contraction on tcgen05:  out[b][m][n] = sum_k A[b][m][k] * B[b][k][n].
// Stage (kc, t) = rows kc*KC.. of the 128-column tile t of B, as up to two TMA
// boxes {64 n, KC k} (SWIZZLE_128B; box h at +h*KC*128 bytes).  Swap-AB: the B
// tile is the MMA A operand (M = 128 columns, MN-major), A^T the MMA B operand
// (N = 16, K-major, no swizzle; rows 8.. carry the bf16 residual of A when M <= 8).
// Accumulators: TMEM columns t*16 .. t*16+15.  The MMA thread releases each slot
// with tcgen05.commit on empty[slot] and signals `done` after the last stage.
// A^T of one batch as the K-major no-swizzle MMA B operand (16 rows x K, bf16):
// core matrix (k8, m) = 8 consecutive k of row m at byte (k8*16 + m)*16; rows
// 8.. hold the bf16 residual a - bf16(a) when M <= 8 (16 mantissa bits overall).
//
// Fast path (row-major A, K % 32 == 0): a warp converts 4 k8 x 8 rows per step.
// It reads with lane = (m, j) and the two 16-byte halves of each 32-byte chunk
// in an order alternating with m, so each 8-lane phase of an LDS.128 touches 8
// distinct bank groups; shuffles transpose to lane = (j, m) so each phase of the
// STS.128 writes one contiguous 128-byte core matrix (both sides conflict-free;
// a direct (k8, m) walk is an 8-way read conflict with rows K*4 bytes apart).
template <int M, int K, i64 SA2, i64 SA3, int NT>
__device__ __forceinline__ void build_xb(u16* __restrict__ xb, const float* __restrict__ Ab) {
  constexpr bool SPLIT = M <= 8;
  if constexpr (SA3 == 1 && K % 32 == 0 && M <= 16) {
    constexpr int NW = NT / 32;
    constexpr int MG = SPLIT ? 1 : 2;  // row groups of 8 read from A
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int rm = lane >> 2, rj = lane & 3, h0 = rm & 1;
    const int src_lane = ((lane & 7) << 2) | (lane >> 3);
    const int wm = lane & 7, wj = lane >> 3;
    for (int it = warp; it < K / 32; it += NW) {
#pragma unroll
      for (int g = 0; g < MG; ++g) {
        const int m = g * 8 + rm;
        float a[8];
        if (m < M) {
          const float* p = Ab + (i64)m * SA2 + (it * 4 + rj) * 8;
          const float4 x0 = *reinterpret_cast<const float4*>(p + 4 * h0);
          const float4 x1 = *reinterpret_cast<const float4*>(p + 4 * (h0 ^ 1));
          const float4 lo4 = h0 ? x1 : x0, hi4 = h0 ? x0 : x1;
          a[0] = lo4.x; a[1] = lo4.y; a[2] = lo4.z; a[3] = lo4.w; a[4] = hi4.x; a[5] = hi4.y; a[6] = hi4.z; a[7] = hi4.w;
        } else {
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) a[kk] = 0.0f;
        }
        u32 hv[4], lv[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const u16 h_0 = NBF16::st(a[2 * i]), h_1 = NBF16::st(a[2 * i + 1]);
          hv[i] = (u32)h_0 | ((u32)h_1 << 16);
          if constexpr (SPLIT) {
            const u16 l_0 = NBF16::st(a[2 * i] - NBF16::ld(h_0)), l_1 = NBF16::st(a[2 * i + 1] - NBF16::ld(h_1));
            lv[i] = (u32)l_0 | ((u32)l_1 << 16);
          }
        }
        uint4 w;
        w.x = __shfl_sync(0xffffffffu, hv[0], src_lane);
        w.y = __shfl_sync(0xffffffffu, hv[1], src_lane);
        w.z = __shfl_sync(0xffffffffu, hv[2], src_lane);
        w.w = __shfl_sync(0xffffffffu, hv[3], src_lane);
        const int k8 = it * 4 + wj;
        *reinterpret_cast<uint4*>(xb + (i64)(k8 * 16 + g * 8 + wm) * 8) = w;
        if constexpr (SPLIT) {
          w.x = __shfl_sync(0xffffffffu, lv[0], src_lane);
          w.y = __shfl_sync(0xffffffffu, lv[1], src_lane);
          w.z = __shfl_sync(0xffffffffu, lv[2], src_lane);
          w.w = __shfl_sync(0xffffffffu, lv[3], src_lane);
          *reinterpret_cast<uint4*>(xb + (i64)(k8 * 16 + 8 + wm) * 8) = w;
        }
      }
    }
  } else {
  for (int c = threadIdx.x; c < 2 * K; c += NT) {  // (k8, m) chunks of 8 elements
    const int m = c & 15, k8 = c >> 4;
    union { uint4 q; u16 h[8]; } u;
    const int src = (m < M) ? m : ((SPLIT && m >= 8 && m - 8 < M) ? m - 8 : -1);
    if (src < 0) {
      u.q = make_uint4(0u, 0u, 0u, 0u);
    } else {
      float a[8];
      if constexpr (SA3 == 1) {
        const float4 a0 = *reinterpret_cast<const float4*>(Ab + (i64)src * SA2 + k8 * 8);
        const float4 a1 = *reinterpret_cast<const float4*>(Ab + (i64)src * SA2 + k8 * 8 + 4);
        a[0] = a0.x; a[1] = a0.y; a[2] = a0.z; a[3] = a0.w; a[4] = a1.x; a[5] = a1.y; a[6] = a1.z; a[7] = a1.w;
      } else {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) a[kk] = Ab[(i64)src * SA2 + (i64)(k8 * 8 + kk) * SA3];
      }
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const u16 hi = NBF16::st(a[kk]);
        u.h[kk] = (m < M) ? hi : NBF16::st(a[kk] - NBF16::ld(hi));
      }
    }
    *reinterpret_cast<uint4*>(xb + (i64)c * 8) = u.q;
  }
  }
}

// A^T straight from a bf16 global row-major A[M][K] (row stride SA2, unit K
// stride): chunk (k8, m) is the 16 bytes at A[m][k8*8..].  bf16 is exact, so
// rows M.. (padding, and the residual rows when M <= 8) are zero.  Lane order
// m-fastest makes each store phase one contiguous 128-byte core matrix; the
// loads (up to 8 in flight per thread) mostly hit L2, A being shared by CTAs.
template <int M, int K, i64 SA2, int NT>
__device__ __forceinline__ void build_xb_g(u16* __restrict__ xb, const u16* __restrict__ A) {
  static_assert(K % 8 == 0 && M <= 16, "build_xb_g shape");
  constexpr int TOT = 2 * K;  // (k8, m) chunks, m in 0..15
  constexpr int IT = (TOT + NT - 1) / NT;
  constexpr int BT = IT < 8 ? IT : 8;
  for (int b = 0; b < IT; b += BT) {
    uint4 v[BT];
#pragma unroll
    for (int j = 0; j < BT; ++j) {
      const int c = threadIdx.x + (b + j) * NT;
      const int m = c & 15, k8 = c >> 4;
      v[j] = make_uint4(0u, 0u, 0u, 0u);
      if (b + j < IT && c < TOT && m < M) v[j] = __ldg(reinterpret_cast<const uint4*>(A + (i64)m * SA2 + k8 * 8));
    }
#pragma unroll
    for (int j = 0; j < BT; ++j) {
      const int c = threadIdx.x + (b + j) * NT;
      if (b + j < IT && c < TOT) *reinterpret_cast<uint4*>(xb + (i64)c * 8) = v[j];
    }
  }
}

// BUILD = false: the caller already built xbuf (shared A operand, or an
// item-invariant one built once per CTA); requires B0 * B1 == 1.
// ACC independent accumulators per tile (TMEM columns (t*ACC + a)*16): MMAs into
// one accumulator serialise on its read-modify-write, and with N = 16 an MMA is
// only ~8 issue cycles, so a long K chain of a single 128-column tile (attention's
// P@V) is latency-bound; consecutive MMAs rotate over the accumulators instead
// and the epilogue adds them.
// KB..KE: the k-chunk range this call consumes (a big stream may be split in two
// segments with a small, dependent chain issued in between, see sgm_codegen.cpp
// interleave); FIN = false issues the segment's MMAs only (accumulators stay in
// TMEM, no commit to `done`, no read-back).
// PRE: the first PRE accumulators of each tile already hold an earlier call's
// product (accumulate-into fusion: LoRA's T@B issued into X@W's accumulators, so
// one read-back yields X@W + T@B and the add disappears).
template <int B0, int B1, int M, int K, int NN, i64 SA0, i64 SA1, i64 SA2, i64 SA3, int KC, int S, int SLOT, int NT,
          bool BUILD = true, int ACC = 1, int KB = 0, int KE = K / KC, bool FIN = true, int PRE = 0>
__device__ __noinline__ void mm_stream_tc_core(float* __restrict__ out, const float* __restrict__ A,
                                               unsigned char* __restrict__ xbuf, u32 tmem, unsigned char* ring,
                                               u64* full, u64* empty, u64* done, u32 q, u32 dph) {
  constexpr int NTL = (NN + 127) / 128;
  constexpr int NKC = KE - KB;
  static_assert((KB == 0 && KE == K / KC && FIN && PRE == 0) ||
                    (B0 * B1 == 1 && (!BUILD || (KB == 0 && KE == K / KC)) && 0 <= KB && KB < KE && KE <= K / KC),
                "segmented / accumulate-into stream: one batch");
  constexpr bool SPLIT = M <= 8;
  constexpr u32 IDESC = UMMA_IDESC_BF16_M128_N16;
  constexpr int NMMA = K / 16;                      // MMAs per tile
  constexpr int AC = ACC < NMMA ? ACC : NMMA;        // accumulators actually written
  constexpr int AR = AC > PRE ? AC : PRE;            // accumulators read back (an earlier call's too)
  // narrow tile (NN <= 64): one 64-column box per stage; the MMA's second 64-row
  // half re-reads the first (LBO 0) and its results are discarded in the epilogue
  constexpr bool NARROW = NN <= 64;
  constexpr u32 LBO = NARROW ? 0u : (u32)(KC * 128);
  static_assert(K % KC == 0 && KC % 16 == 0 && KC * (NARROW ? 128 : 256) <= SLOT && M <= 16 &&
                    NTL * ACC * 16 <= 512,
                "mm_stream_tc shape");
  static_assert(BUILD || B0 * B1 == 1, "a prebuilt A^T covers one batch");
  u16* xb = reinterpret_cast<u16*>(xbuf);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int bi = 0; bi < B0 * B1; ++bi) {
    const int b1 = bi % B1, b0 = bi / B1;
    if constexpr (BUILD) {
      build_xb<M, K, SA2, SA3, NT>(xb, A + b0 * SA0 + b1 * SA1);
      fence_async_smem();
      csync<NT>();
    }
    const u32 q0 = q;
    q += NKC * NTL;
    if (tid == 0) {
      const u32 xs = smem_u32(xb);
#pragma unroll 1
      for (int kc = KB; kc < KE; ++kc) {
#pragma unroll 1
        for (int t = 0; t < NTL; ++t) {
          const u32 slot = ring_wait<S>(full, q0 + (u32)((kc - KB) * NTL + t));
          tc_fence_after();
          const u32 st = smem_u32(ring + slot * SLOT);
#pragma unroll
          for (int ks = 0; ks < KC / 16; ++ks) {
            const u64 ad = umma_desc_sw128(st + ks * 2048, LBO, 1024);
            const u64 bd = umma_desc(xs + ((kc * KC + ks * 16) >> 3) * 256, 256, 128);
            const int g = kc * (KC / 16) + ks;  // MMA index along K
            umma_bf16(tmem + (t * ACC + g % AC) * 16, ad, bd, IDESC, g >= AC || g < PRE);
          }
          umma_commit(&empty[slot]);
        }
      }
      if constexpr (FIN) umma_commit(done);
    }
    if constexpr (!FIN) return;
    mbar_wait(done, dph);
    dph ^= 1u;
    tc_fence_after();
    for (int t = warp >> 2; t < NTL; t += NT / 128) {
      float acc[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) acc[i] = 0.0f;
#pragma unroll
      for (int a = 0; a < AR; ++a) {
        u32 v[16];
        tmem_ld16(tmem + ((u32)((warp & 3) * 32) << 16) + (t * ACC + a) * 16, v);
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i] += __uint_as_float(v[i]);
      }
      const int n = t * 128 + (warp & 3) * 32 + lane;
      if (n < NN) {
#pragma unroll
        for (int m = 0; m < M; ++m) out[((i64)bi * M + m) * NN + n] = SPLIT ? acc[m] + acc[8 + m] : acc[m];
      }
    }
    tc_fence_before();
    csync<NT>();
  }
}

// Out of line (one copy per shape): a kernel's later calls of the same shape run
// from a warm instruction cache; the ring/phase counters advance deterministically.
template <int B0, int B1, int M, int K, int NN, i64 SA0, i64 SA1, i64 SA2, i64 SA3, int KC, int S, int SLOT, int NT,
          bool BUILD = true, int ACC = 1, int KB = 0, int KE = K / KC, bool FIN = true, int PRE = 0>
__device__ __forceinline__ void mm_stream_tc(float* __restrict__ out, const float* __restrict__ A,
                                             unsigned char* __restrict__ xbuf, u32 tmem, unsigned char* ring, u64* full,
                                             u64* empty, u64* done, u32& q, u32& dph) {
  mm_stream_tc_core<B0, B1, M, K, NN, SA0, SA1, SA2, SA3, KC, S, SLOT, NT, BUILD, ACC, KB, KE, FIN, PRE>(
      out, A, xbuf, tmem, ring, full, empty, done, q, dph);
  q += (u32)(B0 * B1 * (KE - KB) * ((NN + 127) / 128));
  if constexpr (FIN) dph ^= (u32)((B0 * B1) & 1);
}

// Streamed fp32 contraction on CUDA cores.  Stage (t, kc) = one TMA box
// {BW n, KC k} (no swizzle, row-major [KC][BW]; BW in {8,16,32,64} matches the
// slice so nothing is over-read).  Thread layout: CGN = BW/8 column groups,
// lane = cg + CGN*kq; k-lane kl = warp*(32/CGN) + kq strides the KC rows.  A
// thread owns columns cg*4.. and BW/2+cg*4.. so each quarter-warp LDS.128 phase
// reads contiguous bytes (conflict-free); per k it also reads A[k][0..M)
// (broadcast within a k-lane) and issues 8*M FMAs.  Partials reduce with
// shuffles over kq, then across warps through `red` (NW*M*64 floats); each
// warp's lane 0 releases the slot (empty count = NT/32).
template <class T> __device__ __forceinline__ T bits_as(u32 v) {
  if constexpr (same_t<T, float>::v) return __uint_as_float(v);
  else return (T)v;
}

template <class N, int B0, int B1, int M, int K, int NN, i64 SA0, i64 SA1, i64 SA2, i64 SA3, int KC, int BW, int S,
          int SLOT, int NT>
__device__ __forceinline__ void mm_stream_f32_core(typename N::C* __restrict__ out, const typename N::C* __restrict__ A,
                                                typename N::C* __restrict__ at, typename N::A* __restrict__ red,
                                                unsigned char* ring, u64* full, u64* empty, u32 q) {
  // N = NF32 (fp32 consumer) or NFF (finite-field checker: 4-byte residues stream
  // through the same ring, u64 lazy-reduced accumulators, mod p at the end)
  typedef typename N::C C;
  typedef typename N::A Acc;
  static_assert(sizeof(C) == 4, "4-byte streamed elements");
  constexpr int NTB = (NN + BW - 1) / BW;
  constexpr int NKC = K / KC;
  constexpr int NW = NT / 32;
  constexpr int CGN = BW / 8;
  constexpr int KQ = 32 / CGN;
  constexpr int KL = NW * KQ;
  constexpr int A0 = SA0 ? B0 : 1, A1 = SA1 ? B1 : 1;
  static_assert(K % KC == 0 && KC * BW * 4 <= SLOT && M <= 8 && NT % 32 == 0 && BW >= 8 && BW <= 64 &&
                (BW & (BW - 1)) == 0, "mm_stream_f32 shape");
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int cg = lane % CGN, kq = lane / CGN, kl = warp * KQ + kq;
  // DIRECT (one A batch, unit k stride): read A[m][k] in place (M scalar loads
  // per k, each a broadcast across a k-lane's column groups), saving the K*M
  // k-major copy -- shared memory the ring gets instead (more bytes in flight)
  constexpr bool DIRECT = SA3 == 1 && A0 * A1 == 1;
  if constexpr (!DIRECT) {
    // k-major copy of A: at[ab][k][m]
    for (int e = tid; e < A0 * A1 * K * M; e += NT) {
      const int m = e % M;
      const int k = (e / M) % K;
      const int ab = e / (M * K);
      const int a1 = ab % A1, a0 = ab / A1;
      at[e] = A[a0 * SA0 + a1 * SA1 + (i64)m * SA2 + (i64)k * SA3];
    }
    csync<NT>();
  }
  for (int bi = 0; bi < B0 * B1; ++bi) {
    const int b1 = bi % B1, b0 = bi / B1;
    const C* pa = DIRECT ? A : at + (i64)((SA0 ? b0 : 0) * A1 + (SA1 ? b1 : 0)) * K * M;
#pragma unroll 1
    for (int t = 0; t < NTB; ++t) {
      Acc acc[M][8];
#pragma unroll
      for (int m = 0; m < M; ++m)
#pragma unroll
        for (int v = 0; v < 8; ++v) acc[m][v] = N::azero();
#pragma unroll 1
      for (int kc = 0; kc < NKC; ++kc) {
        const u32 slot = ring_wait<S>(full, q);
        const C* st = reinterpret_cast<const C*>(ring + slot * SLOT);
        // k-rows kl, kl+KL, ... of the stage, software-pipelined one step ahead so
        // the shared-memory loads of step i+1 overlap the 8*M FMAs of step i (a
        // plain loop left the FMAs waiting on LDS: short-scoreboard stalls in ncu)
        constexpr int NI = (KC + KL - 1) / KL;
        auto load = [&](int i, uint4& w0, uint4& w1, C* av) {
          const int k = kl + i * KL;
          if (KC % KL != 0 && k >= KC) return;
          w0 = *reinterpret_cast<const uint4*>(st + k * BW + cg * 4);
          w1 = *reinterpret_cast<const uint4*>(st + k * BW + BW / 2 + cg * 4);
          if constexpr (DIRECT) {
#pragma unroll
            for (int m = 0; m < M; ++m) av[m] = pa[(i64)m * SA2 + kc * KC + k];
            return;
          }
          const C* ak = pa + (i64)(kc * KC + k) * M;
          if constexpr (M % 4 == 0) {
#pragma unroll
            for (int u = 0; u < M / 4; ++u) *reinterpret_cast<uint4*>(&av[u * 4]) = *reinterpret_cast<const uint4*>(ak + u * 4);
          } else {
#pragma unroll
            for (int m = 0; m < M; ++m) av[m] = ak[m];
          }
        };
        uint4 w0, w1;
        C av[M];
        load(0, w0, w1, av);
#pragma unroll
        for (int i = 0; i < NI; ++i) {
          uint4 n0 = w0, n1 = w1;
          C nav[M];
#pragma unroll
          for (int m = 0; m < M; ++m) nav[m] = av[m];
          if (i + 1 < NI) load(i + 1, n0, n1, nav);
          if (KC % KL == 0 || kl + i * KL < KC) {
            const C w[8] = {bits_as<C>(w0.x), bits_as<C>(w0.y), bits_as<C>(w0.z), bits_as<C>(w0.w),
                            bits_as<C>(w1.x), bits_as<C>(w1.y), bits_as<C>(w1.z), bits_as<C>(w1.w)};
#pragma unroll
            for (int m = 0; m < M; ++m)
#pragma unroll
              for (int v = 0; v < 8; ++v) {
                if constexpr (has_fold<N>::v) N::mac_raw(acc[m][v], av[m], w[v]);
                else N::mac(acc[m][v], av[m], w[v]);
              }
          }
          if constexpr (has_fold<N>::v) {
            if (i % N::FOLD == N::FOLD - 1 || i == NI - 1) {
#pragma unroll
              for (int m = 0; m < M; ++m)
#pragma unroll
                for (int v = 0; v < 8; ++v) N::fold(acc[m][v]);
            }
          }
          w0 = n0;
          w1 = n1;
#pragma unroll
          for (int m = 0; m < M; ++m) av[m] = nav[m];
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
        ++q;
      }
#pragma unroll
      for (int m = 0; m < M; ++m)
#pragma unroll
        for (int v = 0; v < 8; ++v) {
          Acc x = acc[m][v];
#pragma unroll
          for (int off = CGN; off < 32; off <<= 1) N::amerge(x, shfl_xor(x, off, 0xffffffffu));
          acc[m][v] = x;
        }
      if (kq == 0) {
#pragma unroll
        for (int m = 0; m < M; ++m)
#pragma unroll
          for (int v = 0; v < 8; ++v) red[(warp * M + m) * BW + (v >> 2) * (BW / 2) + cg * 4 + (v & 3)] = acc[m][v];
      }
      csync<NT>();
      for (int e = tid; e < M * BW; e += NT) {
        const int m = e / BW, c = e % BW;
        Acc x = N::azero();
#pragma unroll
        for (int w = 0; w < NW; ++w) N::amerge(x, red[(w * M + m) * BW + c]);
        const int n = t * BW + c;
        if (n < NN) out[((i64)bi * M + m) * NN + n] = N::fin(x);
      }
      csync<NT>();
    }
  }
}

template <class N, int B0, int B1, int M, int K, int NN, i64 SA0, i64 SA1, i64 SA2, i64 SA3, int KC, int BW, int S,
          int SLOT, int NT>
__device__ __forceinline__ void mm_stream_f32(typename N::C* __restrict__ out, const typename N::C* __restrict__ A,
                                              typename N::C* __restrict__ at, typename N::A* __restrict__ red,
                                              unsigned char* ring, u64* full, u64* empty, u32& q) {
  mm_stream_f32_core<N, B0, B1, M, K, NN, SA0, SA1, SA2, SA3, KC, BW, S, SLOT, NT>(out, A, at, red, ring, full, empty, q);
  q += (u32)(B0 * B1 * (K / KC) * ((NN + BW - 1) / BW));
}

// Staged loader tile: the producer TMA-loads the item's tile (storage type) into
// a staging buffer laid out [D3/B3][D0][D1][D2][B3] (one box per B3 columns);
// compute threads convert it into the dense compute-type tile.
template <class N, int D0, int D1, int D2, int D3, int B3, int NT>
__device__ __forceinline__ void stage_convert(typename N::C* __restrict__ dst, const typename N::S* __restrict__ stage) {
  constexpr int ROWS = D0 * D1 * D2;
  for (int e = threadIdx.x; e < ROWS * D3; e += NT) {
    const int i3 = e % D3, r = e / D3;
    dst[e] = N::ld(stage[((i64)(i3 / B3) * ROWS + r) * B3 + (i3 % B3)]);
  }
}

// Cluster barrier among compute threads only (the producer warp may be blocked
// on its ring and must not be counted): thread 0 of every CTA arrives on every
// peer's `bar` (count CL) with release.cluster and waits with acquire.cluster.
// gsplit workspace traffic in 16-byte vectors (slots are 16-byte aligned).
// gws_store: one part's partial tile -> its slot.  gws_reduce: the group's
// last item sums the GP slots in part order (fixed order: bit-identical
// results whatever the arrival order); GP independent 16-byte loads per
// thread are in flight at once instead of one scalar chain per element.
template <class N, int SZ, int NT>
__device__ __forceinline__ void gws_store(typename N::C* __restrict__ gw, const typename N::C* __restrict__ t) {
  typedef typename N::C C;
  constexpr int VW = 16 / sizeof(C);
  constexpr int NV = SZ / VW;
  for (int v = threadIdx.x; v < NV; v += NT) {
    union { uint4 q; C c[VW]; } u;
#pragma unroll
    for (int i = 0; i < VW; ++i) u.c[i] = t[v * VW + i];
    __stcg(reinterpret_cast<uint4*>(gw) + v, u.q);
  }
  for (int e = NV * VW + threadIdx.x; e < SZ; e += NT) gw[e] = t[e];
}

template <class N, int SZ, int GP, i64 STRIDE, int NT>
__device__ __forceinline__ void gws_reduce(typename N::C* __restrict__ t, const typename N::C* __restrict__ gw) {
  typedef typename N::C C;
  typedef typename N::A Acc;
  constexpr int VW = 16 / sizeof(C);
  constexpr int NV = SZ / VW;
  // partials in batches of up to 8 loads in flight per thread: all GP at once held
  // GP x 16 bytes in registers (GP = 128: 512 registers, the whole kernel spilled
  // and ran one CTA per SM for the sake of its tail)
  constexpr int QB = GP < 8 ? GP : 8;
  static_assert(GP % QB == 0, "gsplit parts are powers of two");
  for (int v = threadIdx.x; v < NV; v += NT) {
    Acc acc[VW];
#pragma unroll
    for (int i = 0; i < VW; ++i) acc[i] = N::azero();
#pragma unroll 1
    for (int q0 = 0; q0 < GP; q0 += QB) {
      union U { uint4 q; C c[VW]; } u[QB];
#pragma unroll
      for (int q = 0; q < QB; ++q) u[q].q = __ldcg(reinterpret_cast<const uint4*>(gw + (q0 + q) * STRIDE) + v);
#pragma unroll
      for (int i = 0; i < VW; ++i)
#pragma unroll
        for (int q = 0; q < QB; ++q) N::aadd(acc[i], u[q].c[i]);
    }
#pragma unroll
    for (int i = 0; i < VW; ++i) t[v * VW + i] = N::fin(acc[i]);
  }
  for (int e = NV * VW + threadIdx.x; e < SZ; e += NT) {
    Acc acc = N::azero();
    for (int q = 0; q < GP; ++q) N::aadd(acc, __ldcg(&gw[q * STRIDE + e]));
    t[e] = N::fin(acc);
  }
}

// Cluster barrier on one mbarrier per CTA (count CL): lanes 0..CL-1 each signal
// one peer with a release arrive (in parallel: one lane issuing CL dependent
// release arrives measured ~1.5 us per barrier, this ~0.9 us), thread 0 polls
// with test_wait (try_wait's suspend added latency on remote arrivals), and the
// CTA barriers on both sides order every compute thread's DSMEM traffic.
template <int NT, int CL> __device__ __noinline__ void cl_barrier_core(u64* bar, u32 phase) {
  csync<NT>();
  if (threadIdx.x < CL) {
    u32 remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(bar)), "r"((u32)threadIdx.x));
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
  }
  if (threadIdx.x == 0) {
    u32 ok = 0;
    const u64 t0 = wd_now();
    while (!ok) {
      if (wd_now() - t0 > SGM_WD_NS) { wd_trip(); break; }
      asm volatile(
          "{\n\t.reg .pred P1;\n\tmbarrier.test_wait.parity.acquire.cluster.shared::cta.b64 P1, [%1], %2;\n\t"
          "selp.u32 %0, 1, 0, P1;\n\t}"
          : "=r"(ok)
          : "r"(smem_u32(bar)), "r"(phase)
          : "memory");
    }
  }
  csync<NT>();
}
template <int NT, int CL> __device__ __forceinline__ void cl_barrier(u64* bar, u32& phase) {
  cl_barrier_core<NT, CL>(bar, phase);
  phase ^= 1u;
}

// ---------------------------------------------------------------------------
// Cluster all-reduce as reduce-scatter + all-gather over DSMEM.  The peers of
// a group are the ranks r with ((r ^ me) & KEEP) == 0.  Phase 1: each member
// sums the chunk it owns from every member (DSMEM loads) into `tmp`; phase 2
// (after a cluster barrier): it stores the summed chunk into every member's tile
// (DSMEM stores).  DSMEM traffic per CTA: SZ loads + SZ stores (vs G*SZ loads).
// Sums run in rank order so every CTA holds bit-identical values.

__host__ __device__ constexpr int cpopc(u32 x) { return x ? (int)(x & 1u) + cpopc(x >> 1) : 0; }

__device__ __forceinline__ int cl_pos(u32 me, u32 keep, int cl) {
  int pos = 0;
  for (u32 r = 0; r < (u32)cl && r < me; ++r) pos += (((r ^ me) & keep) == 0u);
  return pos;
}

template <class N, int SZ, int CL, u32 KEEP, int NT>
__device__ __noinline__ void cl_rs_phase1(const typename N::C* tile, typename N::C* tmp, u32 me) {
  typedef typename N::A Acc;
  constexpr int G = 1 << cpopc((u32)(CL - 1) & ~KEEP);
  constexpr int CH = (SZ + G - 1) / G;
  const int pos = cl_pos(me, KEEP, CL);
  const int lo = pos * CH;
  const int hi = (lo + CH < SZ) ? lo + CH : SZ;
  for (int e = lo + threadIdx.x; e < hi; e += NT) {
    Acc acc = N::azero();
#pragma unroll
    for (u32 r = 0; r < (u32)CL; ++r)
      if (((r ^ me) & KEEP) == 0u) N::aadd(acc, peer_ptr(tile, r)[e]);
    tmp[e - lo] = N::fin(acc);
  }
}

template <class N, int SZ, int CL, u32 KEEP, int NT>
__device__ __noinline__ void cl_rs_phase2(typename N::C* tile, const typename N::C* tmp, u32 me) {
  constexpr int G = 1 << cpopc((u32)(CL - 1) & ~KEEP);
  constexpr int CH = (SZ + G - 1) / G;
  const int pos = cl_pos(me, KEEP, CL);
  const int lo = pos * CH;
  const int hi = (lo + CH < SZ) ? lo + CH : SZ;
  for (int e = lo + threadIdx.x; e < hi; e += NT) {
    const typename N::C v = tmp[e - lo];
#pragma unroll
    for (u32 r = 0; r < (u32)CL; ++r)
      if (((r ^ me) & KEEP) == 0u) const_cast<typename N::C*>(peer_ptr(tile, r))[e] = v;
  }
}

// ---------------------------------------------------------------------------
// Cluster all-reduce of a small partial tile with ONE cluster barrier (push
// model): every CTA writes its partial into slot `me` of each group peer's
// receive buffer (same smem offset in every CTA), barrier, then each CTA sums
// the group's slots in rank order (its own slot read from its tile), so every
// CTA ends with the identical, fixed-order sum -- the same order as the
// reduce-scatter form.  The caller alternates two receive buffers between
// consecutive items, so a buffer is rewritten only after a later barrier.
template <class N, int SZ, int SZP, int CL, u32 KEEP, int NT>
__device__ __forceinline__ void cl_push(const typename N::C* __restrict__ tile, typename N::C* rbuf, u32 me) {
  typedef typename N::C C;
  constexpr int VW = 16 / sizeof(C);
  constexpr int NV = SZ / VW;
  for (int v = threadIdx.x; v < NV; v += NT) {
    union { uint4 q; C c[VW]; } u;
#pragma unroll
    for (int i = 0; i < VW; ++i) u.c[i] = tile[v * VW + i];
#pragma unroll
    for (u32 r = 0; r < (u32)CL; ++r)
      if (r != me && ((r ^ me) & KEEP) == 0u)
        *reinterpret_cast<uint4*>(const_cast<C*>(peer_ptr(rbuf + me * SZP + v * VW, r))) = u.q;
  }
  for (int e = NV * VW + threadIdx.x; e < SZ; e += NT)
#pragma unroll
    for (u32 r = 0; r < (u32)CL; ++r)
      if (r != me && ((r ^ me) & KEEP) == 0u) const_cast<C*>(peer_ptr(rbuf + me * SZP + e, r))[0] = tile[e];
}

template <class N, int SZ, int SZP, int CL, u32 KEEP, int NT>
__device__ __forceinline__ void cl_gather(typename N::C* __restrict__ tile, const typename N::C* rbuf, u32 me) {
  typedef typename N::A Acc;
  for (int e = threadIdx.x; e < SZ; e += NT) {
    Acc acc = N::azero();
#pragma unroll
    for (u32 r = 0; r < (u32)CL; ++r)
      if (((r ^ me) & KEEP) == 0u) N::aadd(acc, r == me ? tile[e] : rbuf[r * SZP + e]);
    tile[e] = N::fin(acc);
  }
}

// ---------------------------------------------------------------------------
// Cluster all-reduce of a partial tile (simple form, used for tiny tiles): tmp[e] = sum over peers r with
// ((r ^ me) & KEEP) == 0 of tile_r[e], in rank order (identical on every CTA).

template <class N, int SZ, int CL, u32 KEEP, int NT>
__device__ __forceinline__ void cl_reduce(const typename N::C* tile, typename N::C* tmp, u32 me) {
  typedef typename N::A Acc;
  for (int e = threadIdx.x; e < SZ; e += NT) {
    Acc acc = N::azero();
#pragma unroll
    for (u32 r = 0; r < (u32)CL; ++r)
      if (((r ^ me) & KEEP) == 0u) N::aadd(acc, peer_ptr(tile, r)[e]);
    tmp[e] = N::fin(acc);
  }
}

}  // namespace sgm
