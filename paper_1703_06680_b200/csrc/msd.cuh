// msd.cuh -- value-bucketed MSD sort with payload (a2 + a3 fused), sm_100a.
//
// Sorting the endpoint keys is the bulk of the path (Alg. 4 l.5).  The
// LSB onesweep sort (radix.cuh) needs 8 passes over 64-bit keys and leaves the
// subscription upper keys to a random gather (~116 DRAM bytes per 8-byte
// read).  This sort instead:
//   1. maps every value monotonically to one of NB = 2^bbits buckets by
//      linear interpolation between the array's min and max (computed during
//      validation), so buckets are balanced for the paper's uniform workloads
//      and monotone for any input;
//   2. stably multisplits the records by the bucket id in ceil(bbits/8)
//      onesweep-style passes (8-bit digits of the bucket id, LSB first).  The
//      first pass reads the float64 inputs in their original order, so the
//      payload -- the region's upper key and its id -- is read sequentially
//      and travels with the key: no gather is ever needed;
//   3. sorts each bucket (hundreds of records) in shared memory by key with
//      a stable counting sort over finer value bins plus insertion sorts.
// Equal keys keep their original (id) order at every step, so the result is
// the stable sort by key -- identical to the LSB path.  A bucket larger than
// the shared-memory capacity (only for degenerate inputs) raises a flag and
// the caller re-runs the LSB path.
#pragma once
#include "common.cuh"
#include "radix.cuh"

namespace ddm {
namespace msd {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kRadix = 256;
#ifndef DDM_MSD_ITEMS
#define DDM_MSD_ITEMS 16
#endif
constexpr int kItems = DDM_MSD_ITEMS;  // records per thread of a payload pass tile (one sort chain at a time)
constexpr int kItemsC = 8;  // ... while the three sort chains run concurrently (rank form): 80 instead of
                            // 125 registers, so every chain's pass keeps a CTA on each SM
constexpr int kItemsK = 16;  // key-only passes: bigger tiles (fewer look-backs; measured 0.83 -> 0.70 ms at c3)
constexpr int kTile = kThreads * (kItems < kItemsC ? kItems : kItemsC);  // smallest payload tile (status sizing)
#ifndef DDM_LS_SPAN
#define DDM_LS_SPAN 2048
#endif
constexpr int kSpan = DDM_LS_SPAN;  // nominal records per local-sort CTA
#ifndef DDM_LS_CAP
#define DDM_LS_CAP 2560
#endif
constexpr int kCap = DDM_LS_CAP;  // records a local-sort CTA can hold
constexpr int kCapPow2 = kCap <= 2048 ? 2048 : kCap <= 4096 ? 4096 : 8192;  // bitonic network size bound
#ifndef DDM_LS_BINBITS
#define DDM_LS_BINBITS 11
#endif
constexpr int kFineBinBits = DDM_LS_BINBITS;
#ifndef DDM_LS_MINB
#define DDM_LS_MINB 5
#endif
constexpr int kFineBins = 1 << kFineBinBits;  // value bins of the in-smem counting sort
constexpr int kMaxBinRun = 64;   // larger bins (ties, clusters) -> bitonic sort of the group
// Order inside a fine bin: DDM_LS_RANK 1 (default) ranks every record among
// its bin's members (a thread per record); 0: insertion sort per bin (round 1).
#ifndef DDM_LS_RANK
#define DDM_LS_RANK 1
#endif


// Value -> bucket map, equalised to the data.  t(x) = (x/2 - min/2) * kCoarse /
// (max/2 - min/2) places x among kCoarse equal-width coarse bins (c =
// clamp(floor(t))); coarse bin c owns the buckets [base[c], base[c+1]),
// allocated in proportion to its population (map_build_kernel), and x goes to
// base[c] + floor(frac(t) * alloc_c).  Every step (x/2, fma, floor, the clamps,
// a non-negative scale) is monotone non-decreasing in x and bin c's buckets
// all precede bin c+1's, so bucket order never contradicts key order; the
// equalisation keeps buckets near their nominal size on skewed (clustered)
// inputs.
constexpr int kCoarse = 2048;

struct MapRef {
  const uint64_t* mm;    // [min key, max key] (validation)
  const uint32_t* base;  // [kCoarse + 2]: first bucket of every coarse bin, then the "linear" flag
};

// The map is a heuristic: ANY monotone map gives the same sorted result (only
// bucket sizes change), so it is built from a sample, and when the sample
// shows no coarse bin denser than kLinearMax x the mean, the plain linear map
// round(t * NB / kCoarse) is used instead (cheaper per element).
constexpr uint32_t kSampleChunk = 32;   // the sample: runs of 32 consecutive records (one
constexpr uint32_t kSampleStride = 16;  // coalesced warp read) out of every 16 runs -- short
                                        // runs keep it representative for sorted inputs

// i-th record of the sample (i < sample_size(n))
__host__ __device__ __forceinline__ uint64_t sample_at(uint64_t i) {
  return (i / kSampleChunk) * (kSampleChunk * kSampleStride) + (i % kSampleChunk);
}
__host__ __device__ __forceinline__ uint64_t sample_size(uint64_t n) {
  const uint64_t period = (uint64_t)kSampleChunk * kSampleStride;
  return (n / period) * kSampleChunk + umin64(n % period, kSampleChunk);
}
constexpr double kLinearMax = 1.5;

#ifndef DDM_BK_ICLAMP
#define DDM_BK_ICLAMP 1
#endif
#ifndef DDM_HIST_DIRECT
#define DDM_HIST_DIRECT 1
#endif
struct Bucketer {
  double a, b;   // t = fma(x, a, b) in [0, kCoarse] over [min, max]
  double la;     // linear map: bucket = round(t * la)
  const uint32_t* base;
  uint32_t top;
  bool linear;
  __device__ __forceinline__ void init(MapRef M, int bits) {
    const double xmin = key_to_f64(M.mm[0]), xmax = key_to_f64(M.mm[1]);
    const double hmin = xmin * 0.5;
    const double range = xmax * 0.5 - hmin;
    double s = range > 0.0 ? (double)kCoarse / range : 0.0;
    if (!(s <= 1e300)) s = 1e300;
    a = 0.5 * s;
    b = -hmin * s;
    top = (1u << bits) - 1u;
    la = (double)top / (double)kCoarse;
    base = M.base;
    linear = M.base == nullptr || M.base[kCoarse + 1] != 0;
  }
  // t's coarse bin *c = clamp(floor(t), 0, kCoarse - 1) and t - *c.  The floor
  // and the clamps are taken on the integer side (the saturating float64 ->
  // int32 round-down conversion, NaN -> 0, then integer min/max: the same
  // value as fmin(fmax(floor(t), 0), kCoarse - 1) for every t, without the
  // emulated float64 min/max)
  __device__ __forceinline__ double pos_of(double x, int* c) const {
    const double t = fma(x, a, b);
#if DDM_BK_ICLAMP
    const int ci = min(max(__double2int_rd(t), 0), kCoarse - 1);
    *c = ci;
    return t - (double)ci;
#else
    const double tc = fmin(fmax(floor(t), 0.0), (double)(kCoarse - 1));
    *c = (int)tc;
    return t - tc;
#endif
  }
  __device__ __forceinline__ double pos(uint64_t key, int* c) const { return pos_of(key_to_f64(key), c); }
  __device__ __forceinline__ int coarse(uint64_t key) const {
    int c;
    pos(key, &c);
    return c;
  }
  // bucket of the key whose value is x (x = key_to_f64(key); for a float64
  // source, the input itself: key_to_f64(f64_key(x)) has x's bits, -0.0 aside,
  // and -0.0 lands in bucket 0 either way)
  __device__ __forceinline__ uint32_t of_value(double x, uint64_t key) const {
    if (linear) {  // round-to-nearest via the 1.5*2^52 magic add; clamps make it total
      const double u = fma(x, a * la, b * la);
#if DDM_BK_ICLAMP
      // fmin(fmax(u, 0.0), top) on the bit pattern (two 64-bit integer compares
      // instead of two emulated double min/max): non-negative doubles order as
      // their bits; sign set (negatives, -0.0) or NaN -> 0; >= top (+inf too) -> top
      const uint64_t ub = (uint64_t)__double_as_longlong(u);
      uint32_t r = (uint32_t)__double_as_longlong(u + 6755399441055744.0);
      r = ub >= (uint64_t)__double_as_longlong((double)top) ? top : r;
      return ub > 0x7ff0000000000000ull ? 0u : r;
#else
      const double uc = fmin(fmax(u, 0.0), (double)top);
      return (uint32_t)__double_as_longlong(uc + 6755399441055744.0);
#endif
    }
    return mapped(x);
  }
  __device__ __forceinline__ uint32_t operator()(uint64_t key) const { return of_value(key_to_f64(key), key); }
  __device__ __forceinline__ uint32_t mapped(double x) const {
    int c;
    const double f = pos_of(x, &c);
    const uint32_t b0 = __ldg(base + c), al = __ldg(base + c + 1) - b0;
    uint32_t u = 0;
#if DDM_BK_ICLAMP
    if (al) u = (uint32_t)min(max(__double2int_rd(f * (double)al), 0), (int)al - 1);  // (al <= 2^bits)
#else
    if (al) u = (uint32_t)fmin(fmax(floor(f * (double)al), 0.0), (double)(al - 1));
#endif
    const uint32_t r = b0 + u;
    return r < top ? r : top;
  }
};

constexpr int kSampleU = 8;  // sample loads in flight per thread (sampling kernels)
// The sampling kernels are launched on one CTA per SM (kSMs): fewer CTAs
// means fewer global atomics folding the per-CTA min/max and coarse counts.

// [min, max] key of the sample (runs of kSampleChunk records, one in every
// kSampleStride) into mm[0], mm[1] (initialised to [~0, 0]).  Keys outside
// the sampled range are clamped into the first / last bucket by the
// Bucketer, so the sample only shapes bucket sizes, never the result.
template <bool SRC_F64>
__global__ void __launch_bounds__(512) sample_minmax_kernel(const void* __restrict__ src, uint64_t n,
                                                            uint64_t* __restrict__ mm) {
  __shared__ uint64_t red[2][512 / 32];
  const uint64_t ns = sample_size(n);
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint64_t lo = ~0ull, hi = 0;
  // kSampleU independent loads in flight per thread (a latency-bound loop otherwise)
  for (uint64_t s0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; s0 < ns; s0 += kSampleU * stride) {
    uint64_t k[kSampleU];
#pragma unroll
    for (int u = 0; u < kSampleU; ++u) {
      const uint64_t s = s0 + u * stride;
      if (s < ns) {
        const uint64_t i = sample_at(s);
        k[u] = SRC_F64 ? f64_key(__ldcs(reinterpret_cast<const double*>(src) + i))
                       : __ldcs(reinterpret_cast<const uint64_t*>(src) + i);
      } else {
        k[u] = 0;
      }
    }
#pragma unroll
    for (int u = 0; u < kSampleU; ++u)
      if (s0 + u * stride < ns) {
        lo = k[u] < lo ? k[u] : lo;
        hi = k[u] > hi ? k[u] : hi;
      }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const uint64_t a = __shfl_xor_sync(kFull, lo, o), b = __shfl_xor_sync(kFull, hi, o);
    lo = a < lo ? a : lo;
    hi = b > hi ? b : hi;
  }
  // one atomic pair per CTA (per-warp atomics on the same two words serialise)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (lane == 0) { red[0][warp] = lo; red[1][warp] = hi; }
  __syncthreads();
  if (warp == 0) {
    lo = lane < nw ? red[0][lane] : ~0ull;
    hi = lane < nw ? red[1][lane] : 0ull;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const uint64_t a = __shfl_xor_sync(kFull, lo, o), b = __shfl_xor_sync(kFull, hi, o);
      lo = a < lo ? a : lo;
      hi = b > hi ? b : hi;
    }
    if (lane == 0) {
      if (lo != ~0ull) atomicMin((unsigned long long*)&mm[0], (unsigned long long)lo);
      if (hi != 0) atomicMax((unsigned long long*)&mm[1], (unsigned long long)hi);
    }
  }
}

// Coarse-bin population of the sample (runs of kSampleChunk records, one in
// every kSampleStride): counts[kCoarse] (zeroed), counts[kCoarse] = sample size.
template <bool SRC_F64>
__global__ void __launch_bounds__(512) coarse_hist_kernel(const void* __restrict__ src, uint64_t n, MapRef M,
                                                          uint32_t* __restrict__ counts) {
  __shared__ uint32_t sh[kCoarse];
  __shared__ uint32_t tot;
  Bucketer B;
  B.init(MapRef{M.mm, nullptr}, 1);
  for (int i = threadIdx.x; i < kCoarse; i += blockDim.x) sh[i] = 0;
  if (threadIdx.x == 0) tot = 0;
  __syncthreads();
  const uint64_t ns = sample_size(n);
  uint32_t mine = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t s0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; s0 < ns; s0 += kSampleU * stride) {
    uint64_t k[kSampleU];
#pragma unroll
    for (int u = 0; u < kSampleU; ++u) {
      const uint64_t s = s0 + u * stride;
      if (s < ns) {
        const uint64_t i = sample_at(s);
        k[u] = SRC_F64 ? f64_key(__ldcs(reinterpret_cast<const double*>(src) + i))
                       : __ldcs(reinterpret_cast<const uint64_t*>(src) + i);
      } else {
        k[u] = 0;
      }
    }
#pragma unroll
    for (int u = 0; u < kSampleU; ++u)
      if (s0 + u * stride < ns) {
        atomicAdd(&sh[B.coarse(k[u])], 1u);
        ++mine;
      }
  }
  atomicAdd(&tot, mine);
  __syncthreads();
  for (int i = threadIdx.x; i < kCoarse; i += blockDim.x)
    if (sh[i]) atomicAdd(counts + i, sh[i]);
  if (threadIdx.x == 0 && tot) atomicAdd(counts + kCoarse, tot);
}

// base[c] = floor(cum_c * NB / total) with cum_c the sampled population of
// bins < c, so base[0] = 0, base[kCoarse] = NB and every bin gets buckets in
// proportion to its population; base[kCoarse + 1] = 1 when the linear map is
// good enough (no bin above kLinearMax x the mean).  One CTA, 1024 threads.
__global__ void __launch_bounds__(1024) map_build_kernel(const uint32_t* __restrict__ counts, int bits,
                                                         uint32_t* __restrict__ base) {
  __shared__ uint64_t tmp[1024 / 32 + 1];
  __shared__ uint32_t cmax;
  const int t = threadIdx.x;
  if (t == 0) cmax = 0;
  __syncthreads();
  const uint64_t c0 = counts[2 * t], c1 = counts[2 * t + 1];
  atomicMax(&cmax, (uint32_t)(c0 > c1 ? c0 : c1));
  uint64_t total;
  const uint64_t ex = block_excl_scan<1024, uint64_t>(c0 + c1, tmp, &total);
  const uint64_t nb = 1ull << bits;
  const uint64_t nn = total ? total : 1;
  base[2 * t] = (uint32_t)(ex * nb / nn);
  base[2 * t + 1] = (uint32_t)((ex + c0) * nb / nn);
  if (t == 0) {
    base[kCoarse] = (uint32_t)nb;
    base[kCoarse + 1] = (double)cmax * kCoarse <= kLinearMax * (double)nn ? 1u : 0u;
  }
}

// Small sorts (latency-bound): sample min/max, the sample's coarse histogram
// and the bucket map in ONE launch of one CTA (sample_minmax_kernel +
// coarse_hist_kernel + map_build_kernel otherwise).  The same map: min/max
// folded into mm (atomics, as sample_minmax_kernel), coarse bins of the same
// sample, base[] by the same formula.
constexpr uint64_t kMapSmallMaxN = 1ull << 21;
template <bool SRC_F64>
__global__ void __launch_bounds__(1024) map_small_kernel(const void* __restrict__ src, uint64_t n,
                                                         uint64_t* __restrict__ mm, int bits,
                                                         uint32_t* __restrict__ base) {
  __shared__ uint32_t sh[kCoarse];
  __shared__ uint64_t red[2 * 32];
  __shared__ uint64_t tmp[1024 / 32 + 1];
  __shared__ uint32_t cmax;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const uint64_t ns = sample_size(n);
  auto key_at = [&](uint64_t s) -> uint64_t {
    const uint64_t i = sample_at(s);
    return SRC_F64 ? f64_key(__ldcs(reinterpret_cast<const double*>(src) + i))
                   : __ldcs(reinterpret_cast<const uint64_t*>(src) + i);
  };
  uint64_t lo = ~0ull, hi = 0;
  for (uint64_t s = t; s < ns; s += 1024) {
    const uint64_t k = key_at(s);
    lo = k < lo ? k : lo;
    hi = k > hi ? k : hi;
  }
  for (int i = t; i < kCoarse; i += 1024) sh[i] = 0;
  if (t == 0) cmax = 0;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const uint64_t a = __shfl_xor_sync(kFull, lo, o), b = __shfl_xor_sync(kFull, hi, o);
    lo = a < lo ? a : lo;
    hi = b > hi ? b : hi;
  }
  if (lane == 0) { red[warp] = lo; red[32 + warp] = hi; }
  __syncthreads();
  if (warp == 0) {
    lo = red[lane];
    hi = red[32 + lane];
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const uint64_t a = __shfl_xor_sync(kFull, lo, o), b = __shfl_xor_sync(kFull, hi, o);
      lo = a < lo ? a : lo;
      hi = b > hi ? b : hi;
    }
    if (lane == 0) {
      if (lo != ~0ull) atomicMin((unsigned long long*)&mm[0], (unsigned long long)lo);
      if (hi != 0) atomicMax((unsigned long long*)&mm[1], (unsigned long long)hi);
      __threadfence();
      red[0] = ld_relaxed_u64(mm);
      red[1] = ld_relaxed_u64(mm + 1);
    }
  }
  __syncthreads();
  const uint64_t mm2[2] = {red[0], red[1]};
  Bucketer B;
  B.init(MapRef{mm2, nullptr}, 1);
  for (uint64_t s = t; s < ns; s += 1024) atomicAdd(&sh[B.coarse(key_at(s))], 1u);
  __syncthreads();
  const uint64_t c0 = sh[2 * t], c1 = sh[2 * t + 1];
  atomicMax(&cmax, (uint32_t)(c0 > c1 ? c0 : c1));
  uint64_t total;
  const uint64_t ex = block_excl_scan<1024, uint64_t>(c0 + c1, tmp, &total);
  const uint64_t nb = 1ull << bits;
  const uint64_t nn = total ? total : 1;
  base[2 * t] = (uint32_t)(ex * nb / nn);
  base[2 * t + 1] = (uint32_t)((ex + c0) * nb / nn);
  if (t == 0) {
    base[kCoarse] = (uint32_t)nb;
    base[kCoarse + 1] = (double)cmax * kCoarse <= kLinearMax * (double)nn ? 1u : 0u;
  }
}

// ---------------------------------------------------------------- histograms

// Per-pass digit histograms of the bucket ids (digit p = bits [8p, 8p+8)),
// straight from the data with shared-memory counters.  out: [passes][256].
// Every counter is replicated once per lane (counter (p, digit) of lane l at
// word (p * 256 + digit) * 32 + l, bank = l): the shared atomics of a warp
// never meet in a bank, whatever the digits (with one copy, 32 random digits
// over 32 banks replay ~3.5 times per atomic).  Dynamic shared memory:
// hist_smem_bytes(passes).
#ifndef DDM_HIST_REP
#define DDM_HIST_REP 0
#endif
#ifndef DDM_HIST_U
#define DDM_HIST_U 8
#endif
#ifndef DDM_HIST_VEC
#define DDM_HIST_VEC 1
#endif
#ifndef DDM_HIST_MINB
#define DDM_HIST_MINB 2
#endif
constexpr int kHistRep = DDM_HIST_REP ? 32 : 1;
__host__ __device__ constexpr size_t hist_smem_bytes(int passes) {
  return sizeof(uint32_t) * (size_t)passes * kRadix * kHistRep;
}
template <bool SRC_F64>
__global__ void __launch_bounds__(512, DDM_HIST_MINB) msd_hist_kernel(const void* __restrict__ src, uint64_t n,
                                                       MapRef M, int bits, int passes,
                                                       uint32_t* __restrict__ out) {
  extern __shared__ uint32_t hist_sh[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t rep = kHistRep == 32 ? (uint32_t)lane : 0u;
  Bucketer B;
  B.init(M, bits);
  for (int i = threadIdx.x; i < passes * kRadix * kHistRep; i += blockDim.x) hist_sh[i] = 0;
  __syncthreads();
  // U independent loads in flight per thread, then the bucket math + counts
  constexpr int U = DDM_HIST_VEC ? DDM_HIST_U / 2 : DDM_HIST_U;
  const uint64_t* s64 = reinterpret_cast<const uint64_t*>(src);
  auto tally = [&](uint64_t rawbits) {
    uint32_t b;
    if (SRC_F64 && DDM_HIST_DIRECT) {  // straight from the input value (no key round trip)
      b = B.of_value(__longlong_as_double((long long)rawbits), 0);
    } else {
      const uint64_t k = SRC_F64 ? f64_key(__longlong_as_double((long long)rawbits)) : rawbits;
      b = B(k);
    }
    atomicAdd(&hist_sh[(b & 255) * kHistRep + rep], 1u);
    if (passes > 1) atomicAdd(&hist_sh[(kRadix + ((b >> 8) & 255)) * kHistRep + rep], 1u);
    if (passes > 2) atomicAdd(&hist_sh[(2 * kRadix + ((b >> 16) & 255)) * kHistRep + rep], 1u);
  };
#if DDM_HIST_VEC
  // 16-byte loads (two records per load; msd_hist 0.241 -> 0.216 ms per two c3
  // launches); a source not 16-byte aligned starts one record in, the records
  // left over at either end go to thread 0 of CTA 0
  const uint64_t head = (reinterpret_cast<uintptr_t>(src) & 8) && n ? 1 : 0;
  const uint64_t n2 = (n - head) / 2;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const ulonglong2* s128 = reinterpret_cast<const ulonglong2*>(s64 + head);
  for (uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < n2; i0 += U * stride) {
    ulonglong2 raw[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t i = i0 + u * stride;
      raw[u] = i < n2 ? __ldcs(s128 + i) : make_ulonglong2(0, 0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (i0 + u * stride >= n2) break;
      tally(raw[u].x);
      tally(raw[u].y);
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (head) tally(__ldcs(s64));
    if (head + 2 * n2 < n) tally(__ldcs(s64 + n - 1));
  }
#else
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < n; i0 += U * stride) {
    uint64_t raw[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t i = i0 + u * stride;
      raw[u] = i < n ? __ldcs(s64 + i) : 0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (i0 + u * stride >= n) break;
      tally(raw[u]);
    }
  }
#endif
  __syncthreads();
  if (kHistRep == 32) {  // a warp per counter: its 32 copies summed, one global atomic
    for (int i = warp; i < passes * kRadix; i += blockDim.x / 32) {
      uint32_t v = hist_sh[i * 32 + lane];
#pragma unroll
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
      if (lane == 0 && v) atomicAdd(out + i, v);
    }
  } else {
    for (int i = threadIdx.x; i < passes * kRadix; i += blockDim.x) {
      const uint32_t v = hist_sh[i];
      if (v) atomicAdd(out + i, v);
    }
  }
}

// ---------------------------------------------------------------- multisplit pass

// Ranking of the multisplit pass: per-warp digit histogram (shared atomics),
// then stable ranks from per-item peer masks (shared atomicOr).  (Round 2
// measured a ballot-only ranking -- 8 warp ballots per item, no shared
// atomics -- 8 % slower.)
// CTAs per SM the pass is compiled for: 2 for the 16-record payload tiles
// (125 registers), 3 otherwise
template <int ITEMS, bool V64>
constexpr int pass_minb() { return (V64 && ITEMS >= 16) ? 2 : 3; }

#ifndef DDM_MSD_REC
#define DDM_MSD_REC 1
#endif
#ifndef DDM_MSD_RANKFIRST
#define DDM_MSD_RANKFIRST 1
#endif
template <int ITEMS, bool V64, bool V32>
struct PassSmem {
  static constexpr int kT = kThreads * ITEMS;
  // packed records (key + one 64-bit payload) are staged as one 16-byte
  // record per position: one 16-byte store per item (4 quarter-warp phases)
  // instead of two 8-byte stores (2 x 2 half-warp phases), fewer bank-conflict
  // replays of the ranked scatter into shared memory
  static constexpr bool kRec = DDM_MSD_REC && V64 && !V32;
  alignas(16) uint64_t keys[kRec ? 2 * kT : kT];  // kRec: interleaved {key, payload}
  uint64_t v64[(V64 && !kRec) ? kT : 2];
  uint32_t v32[V32 ? kT : 4];
  uint8_t dg[kT];
  alignas(16) uint32_t wbase[kWarps][kRadix];
  uint32_t match[kWarps][kRadix];
  uint32_t digit_base[kRadix];  // (dst = digit_base + tile position, mod 2^32: n < 2^32)
  uint32_t scan_tmp[kWarps + 1];
  uint32_t tile_id;
};


// Stable multisplit of the records by digit = (bucket(key) >> shift) & 255:
// the onesweep scheme of radix.cuh (early counts, atomicOr match ranking,
// decoupled look-back) with a 64-bit and a 32-bit payload.  SRC_F64: the
// first pass, keys/v64 come from float64 arrays (encoded), v32 = index.
//
// Persistent and software-pipelined: a CTA claims tiles in increasing order
// from an atomic counter; once its current tile is ranked into shared memory
// it claims the next one and issues that tile's loads into registers, so the
// look-back wait and the scatter of the current tile overlap the next tile's
// HBM reads.  (Forward progress: the lowest unfinished tile is always some
// CTA's current tile, and it only waits on lower, finished tiles.)
constexpr uint64_t kPackSentinel = 0xffffffffull;  // packed record: upper-key delta does not fit 32 bits

template <int ITEMS, bool V64, bool V32, bool SRC_F64>
struct TileRegs {
  uint64_t key[ITEMS];
  uint64_t hv[V64 ? ITEMS : 1];
  uint32_t iv[V32 ? ITEMS : 1];
  uint32_t err = 0;  // a1 on the fly (first pass over float64 lo/hi): 1 non-finite, 2 lo > hi
  // Issue the loads only: registers receive raw bits, converted by finish()
  // when the tile is processed, so a prefetch never waits for its data.
  __device__ __forceinline__ void load(const void* __restrict__ k_in, const void* __restrict__ v64_in,
                                       const uint32_t* __restrict__ v32_in, uint64_t wb0, uint64_t n, int lane) {
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const uint64_t idx = wb0 + i * 32 + lane;
      if (idx < n) {
        key[i] = __ldcs(reinterpret_cast<const uint64_t*>(k_in) + idx);
        if (V64) hv[i] = __ldcs(reinterpret_cast<const uint64_t*>(v64_in) + idx);
        if (V32) iv[i] = SRC_F64 ? (uint32_t)idx : __ldcs(v32_in + idx);
      } else {
        key[i] = SRC_F64 ? 0x8000000000000000ull : 0;  // (encodes to key 0 below)
        if (V64) hv[i] = SRC_F64 ? 0x8000000000000000ull : 0;
        if (V32) iv[i] = 0;
      }
    }
  }
  // float64 bits -> order-preserving keys (first pass), validating lo/hi.
  // V64 && !V32 is the PACKED record: the 64-bit payload carries the id in its
  // low half and the upper key as a delta from the lower key in its high half
  // (kPackSentinel when the delta does not fit: the local sort then takes the
  // upper key from the input array) -- 16-byte records instead of 20.
  __device__ __forceinline__ void finish(uint64_t wb0, uint64_t n, int lane) {
    if constexpr (SRC_F64) {
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) {
        const uint64_t idx = wb0 + i * 32 + lane;
        const bool valid = idx < n;
        const uint64_t bx = key[i];
        if (valid && !f64_finite_bits(bx)) err |= 1u;
        key[i] = valid ? f64_key(__longlong_as_double((long long)bx)) : 0;
        if (V64) {
          const uint64_t by = hv[i];
          if (valid) {
            if (!f64_finite_bits(by)) err |= 1u;
            else if (!(__longlong_as_double((long long)bx) <= __longlong_as_double((long long)by))) err |= 2u;
          }
          const uint64_t kh = valid ? f64_key(__longlong_as_double((long long)by)) : 0;
          if constexpr (!V32) {
            const uint64_t dk = kh - key[i];
            hv[i] = ((dk < kPackSentinel ? dk : kPackSentinel) << 32) | (uint32_t)idx;
          } else {
            hv[i] = kh;
          }
        }
      }
    }
  }
};

template <int ITEMS, bool V64, bool V32, bool SRC_F64>
__global__ void __launch_bounds__(kThreads, (pass_minb<ITEMS, V64>()))
    msd_pass_kernel(const void* __restrict__ k_in, const void* __restrict__ v64_in, const uint32_t* __restrict__ v32_in,
                    uint64_t* __restrict__ k_out, uint64_t* __restrict__ v64_out, uint32_t* __restrict__ v32_out,
                    uint64_t n, MapRef M, int bits, int shift,
                    const uint32_t* __restrict__ hist, uint32_t* __restrict__ status,
                    uint32_t* __restrict__ tile_counter, uint32_t* __restrict__ err) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  using Smem = PassSmem<ITEMS, V64, V32>;
  constexpr int kT = Smem::kT;
  // (keys-only passes keep the histogram-first form: ranking first spills there)
  constexpr bool kRankFirst = DDM_MSD_RANKFIRST && V64;
  Smem& S = *reinterpret_cast<Smem*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint64_t num_tiles = (n + kT - 1) / kT;
  Bucketer BK;
  BK.init(M, bits);
  if (tid == 0) S.tile_id = atomicAdd(tile_counter, 1u);
  // this pass's global digit starts: exclusive scan of its digit histogram
  // (one digit per thread; no separate bin-start launch)
  static_assert(kThreads == kRadix, "one digit per thread");
  uint32_t ntot;
  const uint32_t bin_start = block_excl_scan<kThreads>(hist[tid], S.scan_tmp, &ntot);
  uint32_t tile = S.tile_id;
  if (tile >= num_tiles) return;
  TileRegs<ITEMS, V64, V32, SRC_F64> R;
  R.load(k_in, v64_in, v32_in, (uint64_t)tile * kT + (uint64_t)warp * (32 * ITEMS), n, lane);

  while (true) {
    const uint64_t tile_base = (uint64_t)tile * kT;
    const uint64_t wb0 = tile_base + (uint64_t)warp * (32 * ITEMS);
    const uint32_t tile_valid = (uint32_t)umin64(kT, n - tile_base);
    R.finish(wb0, n, lane);
    uint32_t* wb = S.wbase[warp];
    const unsigned lt = lanemask_lt();
    {
      uint4* z = reinterpret_cast<uint4*>(&S.wbase[0][0]);
      constexpr int kZ = 2 * kWarps * kRadix / 4;
#pragma unroll
      for (int i = tid; i < kZ; i += kThreads) z[i] = make_uint4(0, 0, 0, 0);
    }
    __syncthreads();
    uint32_t dg[ITEMS];
    if constexpr (kRankFirst) {
    // warp-private ranking first: each item's rank among its warp's items of
    // the same digit (peer masks), the warp's digit counts left in wb -- the
    // tile histogram comes out of the ranking (no separate atomicAdd pass);
    // dg[i] = digit | warp-local rank << 8
    {
      uint32_t* mmask = S.match[warp];
#pragma unroll
      for (int i = 0; i < ITEMS; ++i) {
        const bool valid = wb0 + i * 32 + lane < n;
        const uint32_t d = (BK(R.key[i]) >> shift) & 255u;
        if (valid) atomicOr(&mmask[d], 1u << lane);
        __syncwarp();
        uint32_t peers = 0, base = 0;
        if (valid) {
          peers = mmask[d];
          base = wb[d];
        }
        __syncwarp();
        const unsigned before = peers & lt;
        if (valid && before == 0) {
          wb[d] = base + __popc(peers);
          mmask[d] = 0;
        }
        dg[i] = d | ((base + __popc(before)) << 8);
        __syncwarp();
      }
    }
    } else {
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      dg[i] = (BK(R.key[i]) >> shift) & 255u;
      if (wb0 + i * 32 + lane < n) atomicAdd(&wb[dg[i]], 1u);
    }
    }
    __syncthreads();
    uint32_t total = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      const uint32_t c = S.wbase[w][tid];
      S.wbase[w][tid] = total;
      total += c;
    }
    uint32_t* my_status = status + (uint64_t)tile * kRadix + tid;
    st_relaxed_u32(my_status, (tile == 0 ? radix::kFlagPre : radix::kFlagAgg) | total);
#ifndef DDM_MSD_LB
#define DDM_MSD_LB 8
#endif
    constexpr int kLB = DDM_MSD_LB;  // predecessors read per look-back step
    uint32_t dummy;
    const uint32_t tstart = block_excl_scan<kThreads>(total, S.scan_tmp, &dummy);
#pragma unroll
    for (int w = 0; w < kWarps; ++w) S.wbase[w][tid] += tstart;
    __syncthreads();

    if constexpr (kRankFirst) {
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      if (wb0 + i * 32 + lane < n) {
        const uint32_t d = dg[i] & 255u;
        const uint32_t pos = wb[d] + (dg[i] >> 8);
        if constexpr (Smem::kRec) {
          reinterpret_cast<ulonglong2*>(S.keys)[pos] = make_ulonglong2(R.key[i], R.hv[i]);
        } else {
          S.keys[pos] = R.key[i];
          if (V64) S.v64[pos] = R.hv[i];
        }
        if (V32) S.v32[pos] = R.iv[i];
        S.dg[pos] = (uint8_t)d;
      }
    }
    } else {
    uint32_t* mmask = S.match[warp];
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const bool valid = wb0 + i * 32 + lane < n;
      const uint32_t d = dg[i];
      if (valid) atomicOr(&mmask[d], 1u << lane);
      __syncwarp();
      uint32_t peers = 0, base = 0;
      if (valid) {
        peers = mmask[d];
        base = wb[d];
      }
      __syncwarp();
      if (valid) {
        const unsigned before = peers & lt;
        if (before == 0) {
          wb[d] = base + __popc(peers);
          mmask[d] = 0;
        }
        const uint32_t pos = base + __popc(before);
        if constexpr (Smem::kRec) {
          reinterpret_cast<ulonglong2*>(S.keys)[pos] = make_ulonglong2(R.key[i], R.hv[i]);
        } else {
          S.keys[pos] = R.key[i];
          if (V64) S.v64[pos] = R.hv[i];
        }
        if (V32) S.v32[pos] = R.iv[i];
        S.dg[pos] = (uint8_t)d;
      }
      __syncwarp();
    }
    }
    // claim the next tile and start its loads (the current tile now lives in smem)
    if (tid == 0) S.tile_id = atomicAdd(tile_counter, 1u);
    __syncthreads();
    const uint32_t next = S.tile_id;
    if (next < num_tiles) R.load(k_in, v64_in, v32_in, (uint64_t)next * kT + (uint64_t)warp * (32 * ITEMS), n, lane);

    uint32_t excl = 0;
#ifdef DDM_MSD_NOLB
    if (false) {  // timing experiment only: no look-back (wrong offsets)
#else
    if (tile > 0) {
#endif
      int64_t p = (int64_t)tile - 1;
      while (true) {
        uint32_t sv[kLB];
#pragma unroll
        for (int k = 0; k < kLB; ++k)
          sv[k] = p - k >= 0 ? ld_relaxed_u32(status + (uint64_t)(p - k) * kRadix + tid) : radix::kFlagPre;
        int consumed = 0;
        bool hit_pre = false;
#pragma unroll
        for (int q = 0; q < kLB; ++q) {
          if (hit_pre || consumed != q) break;
          const uint32_t v = sv[q];
          if ((v & ~radix::kValMask) == 0) break;
          excl += v & radix::kValMask;
          consumed = q + 1;
          hit_pre = (v & radix::kFlagPre) != 0;
        }
        if (hit_pre) break;
        if (consumed == 0) __nanosleep(32);
        p -= consumed;
      }
      st_relaxed_u32(my_status, radix::kFlagPre | (excl + total));
    }
    S.digit_base[tid] = bin_start + excl - tstart;  // (mod 2^32)
    __syncthreads();

#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const uint32_t p = i * kThreads + tid;
      if (p < tile_valid) {
        uint64_t k, v = 0;
        if constexpr (Smem::kRec) {
          const ulonglong2 r = reinterpret_cast<const ulonglong2*>(S.keys)[p];
          k = r.x;
          v = r.y;
        } else {
          k = S.keys[p];
          if (V64) v = S.v64[p];
        }
        const uint32_t d = S.dg[p];
        const uint64_t dst = (uint32_t)(S.digit_base[d] + p);
        k_out[dst] = k;
        if (V64) v64_out[dst] = v;
        if (V32) v32_out[dst] = S.v32[p];
      }
    }
    if (next >= num_tiles) break;
    tile = next;  // (the next iteration's first barrier orders these reads before any smem rewrite)
  }
  if (SRC_F64 && err) {
    const uint32_t e = __reduce_or_sync(kFull, R.err);
    if (lane == 0 && e) atomicOr(err, e);
  }
}

// ---------------------------------------------------------------- local sort

// Local-sort configurations: the default, and a big one (a whole SM: 1024
// threads, groups of up to 16384 records, 2^13 fine bins) for sorts whose
// small-bucket map would need one more multisplit pass (c5: 19 bucket bits ->
// 3 passes; with ~8x larger buckets 16 bits -> 2 passes).
#ifndef DDM_LS_TARGET
#define DDM_LS_TARGET DDM_LS_CAP
#endif
struct LsSmall {
  static constexpr int T = kThreads, CAP = kCap, CAP2 = kCapPow2, BIN_BITS = kFineBinBits,
                       BINS = 1 << kFineBinBits, SPAN = kSpan, MINB = DDM_LS_MINB, TARGET = DDM_LS_TARGET;
};
#ifndef DDM_LSB_TARGET
#define DDM_LSB_TARGET 16384
#endif
struct LsBig {
  static constexpr int T = 1024, CAP = 16384, CAP2 = 16384, BIN_BITS = 13, BINS = 1 << 13, SPAN = 8192, MINB = 1,
                       TARGET = DDM_LSB_TARGET;
};

template <class C, bool V64, bool V32>
struct LocalSmem {  // keys only: payloads follow the permutation through the key buffer
  alignas(16) uint64_t keys[C::CAP + 2];  // +2: bulk copies start at a 16-byte aligned index
  uint64_t bar;                         // mbarrier of the bulk copies
  // fine-bin counts / offsets, two 16-bit fields per word (values <= C::CAP),
  // followed by perm (sorted position -> staged index); the bitonic fallback
  // uses both as one u16[C::CAP2] array (the bins are dead by then)
  uint32_t binw[C::BINS / 2 + 2];
  uint16_t perm[C::CAP];
  static_assert(sizeof(uint32_t) * (C::BINS / 2 + 2) + sizeof(uint16_t) * C::CAP >= sizeof(uint16_t) * C::CAP2,
                "the bitonic fallback's u16[C::CAP2] fits in binw + perm");
#if DDM_LS_RANK
  uint16_t perm2[C::CAP];  // final order (sorted position -> staged index)
#endif
  uint64_t red[2 * (C::T / 32) + 2];
  uint32_t flag;
  uint64_t bound[1];  // prev_boundary's reduction slot
};

// Stable sort of records [e0, e0 + c) by key inside shared memory (c <= C::CAP).
// Records arrive in (bucket, original-order) order.  Counting sort over fine
// bins of the key range of this group (integer, monotone): every record goes
// to its bin's next slot of perm, then each bin holding two or more records
// (most hold zero or one) is insertion-sorted by (key, staged index); if some
// bin is large (ties, dense clusters) the group is bitonic-sorted on (key,
// staged index) instead.  (No separate grouping array: the smaller footprint
// keeps 6 CTAs per SM; measured 1.31 -> 1.22 ms per two c3 launches.)
__device__ __forceinline__ uint32_t bin_get(const uint32_t* w, uint32_t b) {
  return (w[b >> 1] >> ((b & 1) * 16)) & 0xffffu;
}
__device__ __forceinline__ uint32_t bin_add(uint32_t* w, uint32_t b) {  // returns the old value
  return (atomicAdd(w + (b >> 1), (b & 1) ? 0x10000u : 1u) >> ((b & 1) * 16)) & 0xffffu;
}

template <class C, bool V64, bool V32>
__device__ void local_sort_group(LocalSmem<C, V64, V32>& S, const uint64_t* __restrict__ k_in,
                                 const uint64_t* __restrict__ v64_in, const uint32_t* __restrict__ v32_in,
                                 uint64_t* __restrict__ k_out, uint64_t* __restrict__ v64_out,
                                 uint32_t* __restrict__ v32_out, uint64_t e0, uint32_t c, uint32_t& phase,
                                 const double* __restrict__ hi_src) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // the group's keys arrive by one bulk async copy (16-byte aligned start;
  // reading a key past the array is safe: it is followed by another
  // workspace array)
  const uint32_t ko = (uint32_t)(e0 & 1);
  uint64_t* const K = S.keys + ko;
  if (tid == 0) {
    const uint32_t bytes = ((c + ko + 1) & ~1u) * 8;
    mbar_expect_tx(&S.bar, bytes);
    bulk_g2s(S.keys, k_in + (e0 - ko), bytes, &S.bar);
  }
  mbar_wait(&S.bar, phase);
  phase ^= 1;
  uint64_t kmin = ~0ull, kmax = 0;
  for (uint32_t i = tid; i < c; i += C::T) {
    const uint64_t k = K[i];
    kmin = k < kmin ? k : kmin;
    kmax = k > kmax ? k : kmax;
  }
  for (uint32_t b = tid; b < C::BINS / 2 + 2; b += C::T) S.binw[b] = 0;
  if (tid == 0) S.flag = 0;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const uint64_t x = __shfl_xor_sync(kFull, kmin, o), y = __shfl_xor_sync(kFull, kmax, o);
    kmin = x < kmin ? x : kmin;
    kmax = y > kmax ? y : kmax;
  }
  if (lane == 0) { S.red[warp] = kmin; S.red[(C::T / 32) + warp] = kmax; }
  __syncthreads();
  if constexpr (C::T / 32 > 8) {  // many warps: warp 0 combines, everyone reads two words
    if (warp == 0) {
      kmin = lane < C::T / 32 ? S.red[lane] : ~0ull;
      kmax = lane < C::T / 32 ? S.red[(C::T / 32) + lane] : 0ull;
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const uint64_t x = __shfl_xor_sync(kFull, kmin, o), y = __shfl_xor_sync(kFull, kmax, o);
        kmin = x < kmin ? x : kmin;
        kmax = y > kmax ? y : kmax;
      }
      if (lane == 0) { S.red[2 * (C::T / 32)] = kmin; S.red[2 * (C::T / 32) + 1] = kmax; }
    }
    __syncthreads();
    kmin = S.red[2 * (C::T / 32)];
    kmax = S.red[2 * (C::T / 32) + 1];
  } else {
    kmin = ~0ull;
    kmax = 0;
#pragma unroll
    for (int w = 0; w < (C::T / 32); ++w) {
      kmin = S.red[w] < kmin ? S.red[w] : kmin;
      kmax = S.red[(C::T / 32) + w] > kmax ? S.red[(C::T / 32) + w] : kmax;
    }
  }
  const uint64_t range = kmax - kmin;
  // smallest shift with (kmax - kmin) >> sh < C::BINS
  const int sh = range ? max(0, 64 - __clzll((long long)range) - C::BIN_BITS) : 0;
  auto fine = [&](uint64_t k) -> uint32_t { return (uint32_t)((k - kmin) >> sh); };
  for (uint32_t i = tid; i < c; i += C::T) bin_add(S.binw, fine(K[i]));
  __syncthreads();
  {  // exclusive scan over the bins (8 per thread, 4 words) + large-bin detection
    constexpr int kPer = C::BINS / C::T;
    static_assert(kPer % 2 == 0, "whole words per thread");
    uint32_t v[kPer], sum = 0;
#pragma unroll
    for (int q = 0; q < kPer; q += 2) {
      const uint32_t wv = S.binw[(tid * kPer + q) >> 1];
      v[q] = wv & 0xffffu;
      v[q + 1] = wv >> 16;
    }
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      sum += v[q];
      if (v[q] > kMaxBinRun) S.flag = 1;
    }
    __shared__ uint32_t tmp[(C::T / 32) + 1];
    uint32_t tot;
    uint32_t ex = block_excl_scan<C::T>(sum, tmp, &tot);
#pragma unroll
    for (int q = 0; q < kPer; q += 2) {
      const uint32_t e0v = ex, e1v = ex + v[q];
      ex = e1v + v[q + 1];
      S.binw[(tid * kPer + q) >> 1] = e0v | (e1v << 16);
    }
  }
  __syncthreads();
  if (S.flag == 0) {
    // place every record at its bin's next slot, straight into perm (any
    // order inside a bin; most bins hold zero or one record) ...
    for (uint32_t i = tid; i < c; i += C::T) {
      const uint32_t pos = bin_add(S.binw, fine(K[i]));
      S.perm[pos] = (uint16_t)i;
    }
    __syncthreads();
#if DDM_LS_RANK
    // ... then every record takes its rank inside its bin, (key, staged
    // index) order, from the bin's other members: one record per thread, so
    // the work is spread evenly (most bins hold one record; an insertion sort
    // per bin left a warp waiting on its longest bin); bin b spans
    // [end(b-1), end(b)), <= kMaxBinRun
    for (uint32_t x = tid; x < c; x += C::T) {
      const uint16_t v = S.perm[x];
      const uint64_t kv = K[v];
      const uint32_t b = fine(kv);
      const uint32_t lo = b ? bin_get(S.binw, b - 1) : 0, hi = bin_get(S.binw, b);
      uint32_t r = 0;
      if (hi - lo > 1)  // (most bins hold this record alone)
        for (uint32_t y = lo; y < hi; ++y) {
          const uint16_t u = S.perm[y];
          const uint64_t ku = K[u];
          r += (uint32_t)(ku < kv) | ((uint32_t)(ku == kv) & (uint32_t)(u < v));
        }
      S.perm2[lo + r] = v;
    }
  }
#else
    // ... then order each bin holding two or more records by (key, staged
    // index) with an insertion sort; bin b spans [end(b-1), end(b)), <= kMaxBinRun
    for (uint32_t b = tid; b < C::BINS; b += C::T) {
      const uint32_t lo = b ? bin_get(S.binw, b - 1) : 0, hi = bin_get(S.binw, b);
      if (hi - lo < 2) continue;
      for (uint32_t x = lo + 1; x < hi; ++x) {
        const uint16_t v = S.perm[x];
        const uint64_t kv = K[v];
        uint32_t y = x;
        while (y > lo) {
          const uint16_t u = S.perm[y - 1];
          const uint64_t ku = K[u];
          if (ku < kv || (ku == kv && u < v)) break;
          S.perm[y] = u;
          --y;
        }
        S.perm[y] = v;
      }
    }
  }
#endif
  else {
    // bitonic sort of (key, index) over the next power of two, in the
    // bins + perm storage taken as one u16 array
    uint16_t* PB = reinterpret_cast<uint16_t*>(S.binw);
    uint32_t P = 1;
    while (P < c) P <<= 1;
    for (uint32_t i = tid; i < P; i += C::T) PB[i] = (uint16_t)(i < c ? i : 0xffff);
    __syncthreads();
    for (uint32_t k = 2; k <= P; k <<= 1) {
      for (uint32_t j = k >> 1; j > 0; j >>= 1) {
        for (uint32_t i = tid; i < P; i += C::T) {
          const uint32_t l = i ^ j;
          if (l > i) {
            const uint16_t a = PB[i], b = PB[l];
            const bool a_gt_b = (a == 0xffff) ? (b != 0xffff)
                                : (b == 0xffff) ? false
                                : (K[a] > K[b] || (K[a] == K[b] && a > b));
            const bool up = (i & k) == 0;
            if (up == a_gt_b) { PB[i] = b; PB[l] = a; }
          }
        }
        __syncthreads();
      }
    }
  }
  __syncthreads();
#if DDM_LS_RANK
  const uint16_t* PERM = S.flag ? reinterpret_cast<const uint16_t*>(S.binw) : S.perm2;
#else
  const uint16_t* PERM = S.flag ? reinterpret_cast<const uint16_t*>(S.binw) : S.perm;
#endif
  if constexpr (V64 && !V32) {
    // PACKED records: sorted keys out (kept in registers), then the payload
    // (id | upper-key delta << 32) staged through the key buffer, unpacked into
    // the upper key and the id
    constexpr int kPer = (C::CAP + C::T - 1) / C::T;
    uint64_t kr[kPer];
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      const uint32_t i = tid + j * C::T;
      if (i < c) {
        kr[j] = K[PERM[i]];
        k_out[e0 + i] = kr[j];
      }
    }
    __syncthreads();  // the key buffer is free
    if (tid == 0) {
      const uint32_t bytes = ((c + ko + 1) & ~1u) * 8;
      mbar_expect_tx(&S.bar, bytes);
      bulk_g2s(S.keys, v64_in + (e0 - ko), bytes, &S.bar);
    }
    mbar_wait(&S.bar, phase);
    phase ^= 1;
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      const uint32_t i = tid + j * C::T;
      if (i < c) {
        const uint64_t P = K[PERM[i]];
        const uint32_t id = (uint32_t)P;
        const uint64_t d = P >> 32;
        v64_out[e0 + i] = d != kPackSentinel ? kr[j] + d : f64_key(__ldg(hi_src + id));
        v32_out[e0 + i] = id;
      }
    }
    __syncthreads();
    return;
  }
  for (uint32_t i = tid; i < c; i += C::T) k_out[e0 + i] = K[PERM[i]];
  // payloads: staged coalesced through the key buffer (free now), then read
  // back in permutation order -- random global gathers would cost one L1
  // request per element
  if (V64) {
    __syncthreads();  // the key buffer is free
    if (tid == 0) {
      const uint32_t bytes = ((c + ko + 1) & ~1u) * 8;
      mbar_expect_tx(&S.bar, bytes);
      bulk_g2s(S.keys, v64_in + (e0 - ko), bytes, &S.bar);
    }
    mbar_wait(&S.bar, phase);
    phase ^= 1;
    for (uint32_t i = tid; i < c; i += C::T) v64_out[e0 + i] = K[PERM[i]];
  }
  if (V32) {
    const uint32_t vo = (uint32_t)(e0 & 3);
    const uint32_t* b32 = reinterpret_cast<const uint32_t*>(S.keys) + vo;
    __syncthreads();
    if (tid == 0) {
      const uint32_t bytes = ((c + vo + 3) & ~3u) * 4;
      mbar_expect_tx(&S.bar, bytes);
      bulk_g2s(S.keys, v32_in + (e0 - vo), bytes, &S.bar);
    }
    mbar_wait(&S.bar, phase);
    phase ^= 1;
    for (uint32_t i = tid; i < c; i += C::T) v32_out[e0 + i] = b32[PERM[i]];
  }
  __syncthreads();
}

// Last bucket boundary in (lo, hi] scanning backwards; lo if none.
template <class C>
__device__ __forceinline__ uint64_t prev_boundary(const uint64_t* __restrict__ keys, uint64_t lo, uint64_t hi,
                                                  const Bucketer& BK, uint64_t* slot) {
  const int tid = threadIdx.x;
  if (tid == 0) *slot = 0;
  __syncthreads();
  for (int64_t top = (int64_t)hi; top > (int64_t)lo; top -= C::T) {
    const int64_t q = top - tid;
    const bool edge = q > (int64_t)lo && BK(keys[q]) != BK(keys[q - 1]);
    if (edge) atomicMax((unsigned long long*)slot, (unsigned long long)q);
    __syncthreads();
    const uint64_t r = *slot;
    __syncthreads();
    if (r) return r;
  }
  return lo;
}

// bounds[s] = first bucket boundary at or after s*span (s = 0..spans; n past
// the end): one thread per span.  The records are grouped by bucket in
// increasing bucket order, so the bucket id is non-decreasing along the
// positions and the boundary is an upper bound of the bucket of position
// s*span - 1: a gallop forward from s*span, then a binary search of the last
// step (O(log distance) dependent loads; the span of the big local sort is
// 8192 records with ~6000-record buckets, which a linear scan paid for).
__global__ void __launch_bounds__(256) span_bounds_kernel(const uint64_t* __restrict__ keys, uint64_t n,
                                                          MapRef M, int bits, uint32_t spans, uint32_t span,
                                                          uint64_t* __restrict__ bounds) {
  Bucketer BK;
  BK.init(M, bits);
  const uint32_t sp = blockIdx.x * blockDim.x + threadIdx.x;
  if (sp > spans) return;
  const uint64_t p = (uint64_t)sp * span;
  if (sp == 0 || p >= n) {
    bounds[sp] = sp == 0 ? 0 : n;
    return;
  }
  const uint32_t b0 = BK(__ldg(keys + p - 1));
  // first q >= p with BK(keys[q]) > b0 (n if none)
  uint64_t lo = p, hi = n, step = 1;
  while (true) {
    const uint64_t q = lo + step - 1;
    if (q >= n) break;
    if (BK(__ldg(keys + q)) > b0) { hi = q; break; }
    lo = q + 1;
    step <<= 1;
  }
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (BK(__ldg(keys + mid)) > b0) hi = mid;
    else lo = mid + 1;
  }
  bounds[sp] = lo;
}

// The same bounds when the sort took a single multisplit pass (bucket ids <
// 256): the digit starts of that pass ARE the bucket starts, so the first
// bucket boundary at or after s*span is the smallest start >= s*span -- a
// search over 256 cached values instead of a gallop over the sorted keys.
__global__ void __launch_bounds__(256) span_bounds_hist_kernel(const uint32_t* __restrict__ hist, uint32_t nb,
                                                               uint64_t n, uint32_t spans, uint32_t span,
                                                               uint64_t* __restrict__ bounds) {
  __shared__ uint32_t st[kRadix];
  __shared__ uint32_t tmp[kRadix / 32 + 1];
  {  // the digit starts: exclusive scan of the pass's digit histogram (256 threads)
    const uint32_t b = threadIdx.x;
    uint32_t tot;
    const uint32_t ex = block_excl_scan<kRadix>(b < nb ? hist[b] : 0u, tmp, &tot);
    st[b] = b < nb ? ex : (uint32_t)n;
  }
  __syncthreads();
  for (uint32_t sp = blockIdx.x * blockDim.x + threadIdx.x; sp <= spans; sp += gridDim.x * blockDim.x) {
    const uint64_t p = (uint64_t)sp * span;
    if (sp == 0 || p >= n) {
      bounds[sp] = sp == 0 ? 0 : n;
      continue;
    }
    uint32_t lo = 0, hi = kRadix;  // first bucket whose start is >= p (starts are non-decreasing)
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (st[mid] >= p) hi = mid;
      else lo = mid + 1;
    }
    bounds[sp] = lo < kRadix ? st[lo] : n;
  }
}

// CTA c sorts the whole buckets starting in [c*C::SPAN, (c+1)*C::SPAN), i.e. in
// [bounds[c], bounds[c+1]) (span_bounds_kernel), in groups of consecutive
// buckets holding <= C::CAP records in smem.  A
// single bucket larger than C::CAP sets *overflow (caller redoes with LSB).
template <class C, bool V64, bool V32>
__global__ void __launch_bounds__(C::T, C::MINB) local_sort_kernel(const uint64_t* __restrict__ k_in,
                                                              const uint64_t* __restrict__ v64_in,
                                                              const uint32_t* __restrict__ v32_in,
                                                              uint64_t* __restrict__ k_out,
                                                              uint64_t* __restrict__ v64_out,
                                                              uint32_t* __restrict__ v32_out, uint64_t n,
                                                              MapRef M, int bits,
                                                              const uint64_t* __restrict__ bounds,
                                                              uint32_t* __restrict__ overflow,
                                                              const double* __restrict__ hi_src) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  LocalSmem<C, V64, V32>& S = *reinterpret_cast<LocalSmem<C, V64, V32>*>(smem_raw);
  Bucketer BK;
  BK.init(M, bits);
  if (threadIdx.x == 0) mbar_init(&S.bar, 1);
  uint32_t phase = 0;
  uint64_t e0 = __ldg(bounds + blockIdx.x);
  const uint64_t e1 = __ldg(bounds + blockIdx.x + 1);
  __syncthreads();  // publishes the mbarrier init
  while (e0 < e1) {
    uint64_t g1 = e1;
    // groups of whole buckets, ~C::TARGET records (fewer records than fine
    // bins: most bins then hold one record), or one bucket up to C::CAP
    if (e1 - e0 > C::TARGET) {
      g1 = prev_boundary<C>(k_in, e0, e0 + C::TARGET, BK, &S.bound[0]);
      if (g1 == e0 && e1 - e0 > C::CAP) g1 = prev_boundary<C>(k_in, e0, e0 + C::CAP, BK, &S.bound[0]);
      else if (g1 == e0) g1 = e1;
      if (g1 == e0) {  // one bucket alone exceeds the capacity
        if (threadIdx.x == 0) atomicOr(overflow, 1u);
        return;
      }
    }
    local_sort_group<C, V64, V32>(S, k_in, v64_in, v32_in, k_out, v64_out, v32_out, e0, (uint32_t)(g1 - e0), phase,
                               hi_src);
    e0 = g1;
  }
}

}  // namespace msd
}  // namespace ddm
