// common.cuh -- shared device helpers for libddm (sm_100a).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ddm {

constexpr int kWarp = 32;

__host__ __device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }
constexpr unsigned kFull = 0xffffffffu;

// Order-preserving float64 -> u64 key.
// -0.0 is canonicalised to +0.0 first (IEEE -0.0 == +0.0, DESIGN reading R3);
// then non-negatives get the sign bit set and negatives are bit-inverted, so
// unsigned order on keys equals numeric order on finite doubles.
__device__ __forceinline__ uint64_t f64_key(double x) {
  uint64_t b = static_cast<uint64_t>(__double_as_longlong(x));
  if (b == 0x8000000000000000ull) b = 0;
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// inverse of f64_key (keys of finite doubles; -0 was canonicalised to +0)
__device__ __forceinline__ double key_to_f64(uint64_t k) {
  const uint64_t b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)b);
}

__device__ __forceinline__ bool f64_finite_bits(uint64_t b) {
  return (b & 0x7ff0000000000000ull) != 0x7ff0000000000000ull;
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned r;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
  return r;
}

__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_relaxed_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// ---- 1-D bulk async copies (cp.async.bulk, the TMA engine's non-tensor
// form) into shared memory, completion tracked by an mbarrier.  Addresses
// and sizes must be multiples of 16 bytes.
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t done = 0;
  while (!done)
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
}

// Streaming (read-once) loads: keep them out of L1.
template <typename T>
__device__ __forceinline__ T ldg_stream(const T* p) {
  return __ldcs(p);
}

__device__ __forceinline__ uint64_t warp_max_u64(uint64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    uint64_t w = __shfl_xor_sync(kFull, v, o);
    v = w > v ? w : v;
  }
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

// Inclusive warp scan.
template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T w = __shfl_up_sync(kFull, v, o);
    if (lane >= o) v += w;
  }
  return v;
}

// Block-wide exclusive scan for blockDim.x == NT (multiple of 32, <= 1024).
// `tmp` needs NT/32 + 1 slots.  Returns the exclusive prefix; *total = sum.
template <int NT, typename T>
__device__ __forceinline__ T block_excl_scan(T v, T* tmp, T* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T inc = warp_incl_scan(v);
  if (lane == 31) tmp[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    T w = lane < NT / 32 ? tmp[lane] : T(0);
    T wi = warp_incl_scan(w);
    if (lane < NT / 32) tmp[lane] = wi - w;
    if (lane == NT / 32 - 1) tmp[NT / 32] = wi;
  }
  __syncthreads();
  T r = tmp[warp] + inc - v;
  *total = tmp[NT / 32];
  __syncthreads();
  return r;
}

// Number of block-max levels kept over the sorted subscription upper keys
// (fan-out 32 per level: 32, 1024, 32768, 2^20, 2^25, 2^30 entries per block).
constexpr int kMaxLevels = 6;

struct MaxTree {
  const uint64_t* lvl[kMaxLevels + 1];  // lvl[0] = leaves (slo_hi), lvl[L] = max over 32^L
  int levels;                           // number of valid levels above the leaves
};

}  // namespace ddm
