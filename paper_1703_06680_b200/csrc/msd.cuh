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
constexpr int kItems = 8;
constexpr int kTile = kThreads * kItems;
constexpr int kSpan = 2048;      // nominal records per local-sort CTA
constexpr int kCap = 4096;       // records a local-sort CTA can hold
constexpr int kFineBins = 4096;  // value bins of the in-smem counting sort
constexpr int kMaxBinRun = 64;   // larger bins (ties, clusters) -> bitonic sort of the group

// inverse of f64_key (keys of finite doubles; -0 was canonicalised to +0)
__device__ __forceinline__ double key_to_f64(uint64_t k) {
  const uint64_t b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)b);
}

// Monotone value -> bucket map: floor((x/2 - min/2) * scale), clamped.
struct Bucketer {
  double hmin, scale;
  uint32_t last;
  __device__ __forceinline__ void init(const uint64_t* mm, int bits) {
    const double xmin = key_to_f64(mm[0]), xmax = key_to_f64(mm[1]);
    hmin = xmin * 0.5;
    const double range = xmax * 0.5 - hmin;
    const double nb = (double)(1ull << bits);
    double s = range > 0.0 ? nb / range : 0.0;
    if (!(s <= 1.7976931348623157e308)) s = 1.7976931348623157e308;
    scale = s;
    last = (uint32_t)((1ull << bits) - 1);
  }
  __device__ __forceinline__ uint32_t of_value(double x, double sc) const {
    const uint32_t b = __double2uint_rz((x * 0.5 - hmin) * sc);  // saturating; NaN -> 0
    return b;
  }
  __device__ __forceinline__ uint32_t operator()(uint64_t key) const {
    const uint32_t b = of_value(key_to_f64(key), scale);
    return b > last ? last : b;
  }
};

// ---------------------------------------------------------------- histograms

// Full bucket histogram of the keys (float64 source encoded on the fly).
template <bool SRC_F64>
__global__ void __launch_bounds__(256) bucket_hist_kernel(const void* __restrict__ src, uint64_t n,
                                                          const uint64_t* __restrict__ mm, int bits,
                                                          uint32_t* __restrict__ hist) {
  Bucketer B;
  B.init(mm, bits);
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t k = SRC_F64 ? f64_key(__ldcs(reinterpret_cast<const double*>(src) + i))
                               : __ldcs(reinterpret_cast<const uint64_t*>(src) + i);
    atomicAdd(hist + B(k), 1u);
  }
}

// Per-pass digit histograms (digit p = bits [8p, 8p+8) of the bucket id)
// from the full bucket histogram.  out: [passes][256], zeroed.
__global__ void __launch_bounds__(256) digit_hist_kernel(const uint32_t* __restrict__ hist, uint32_t nb,
                                                         int passes, uint32_t* __restrict__ out) {
  __shared__ uint32_t sh[3][kRadix];
  for (int i = threadIdx.x; i < 3 * kRadix; i += blockDim.x) (&sh[0][0])[i] = 0;
  __syncthreads();
  for (uint32_t b = blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += gridDim.x * blockDim.x) {
    const uint32_t c = hist[b];
    if (c)
      for (int p = 0; p < passes; ++p) atomicAdd(&sh[p][(b >> (8 * p)) & 255], c);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < passes * kRadix; i += blockDim.x) {
    const uint32_t v = (&sh[0][0])[i];
    if (v) atomicAdd(out + i, v);
  }
}

// exclusive scan of nb u32 counts -> starts[0..nb] (starts[nb] = n), one CTA
// per 4096 counts, decoupled look-back (u64 status words).
constexpr int kBScanItems = 16;
__global__ void __launch_bounds__(kThreads) bucket_scan_kernel(const uint32_t* __restrict__ cnt, uint32_t nb,
                                                               uint32_t* __restrict__ starts,
                                                               uint64_t* __restrict__ status) {
  __shared__ uint64_t tmp[kWarps + 1];
  __shared__ uint64_t prefix;
  const int tid = threadIdx.x;
  const uint32_t tile = blockIdx.x;
  const uint64_t base = (uint64_t)tile * kThreads * kBScanItems + (uint64_t)tid * kBScanItems;
  uint32_t v[kBScanItems];
  uint64_t local = 0;
#pragma unroll
  for (int i = 0; i < kBScanItems; ++i) {
    v[i] = base + i < nb ? cnt[base + i] : 0;
    local += v[i];
  }
  uint64_t agg;
  const uint64_t ex = block_excl_scan<kThreads>(local, tmp, &agg);
  if (tid < 32) {
    const uint64_t e = match::lookback_warp_u64(status, tile, agg);
    if (tid == 0) prefix = e;
  }
  __syncthreads();
  uint64_t run = prefix + ex;
#pragma unroll
  for (int i = 0; i < kBScanItems; ++i) {
    if (base + i < nb) starts[base + i] = (uint32_t)run;
    run += v[i];
  }
  if (tile == gridDim.x - 1 && tid == 0) starts[nb] = (uint32_t)(prefix + agg);
}

// span_lo[c] = first bucket start >= c * kSpan (c = 0..spans); whole buckets
// per local-sort CTA.
__global__ void __launch_bounds__(256) span_kernel(const uint32_t* __restrict__ starts, uint32_t nb, uint64_t n,
                                                   uint32_t spans, uint32_t* __restrict__ span_lo) {
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c > spans) return;
  const uint64_t p = umin64((uint64_t)c * kSpan, n);
  uint32_t lo = 0, hi = nb;  // first index in starts[0..nb] with starts[i] >= p
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (starts[mid] < p) lo = mid + 1;
    else hi = mid;
  }
  span_lo[c] = c == spans ? (uint32_t)n : starts[lo];
}

// ---------------------------------------------------------------- multisplit pass

template <int ITEMS, bool V64, bool V32>
struct PassSmem {
  static constexpr int kT = kThreads * ITEMS;
  uint64_t keys[kT];
  uint64_t v64[V64 ? kT : 2];
  uint32_t v32[V32 ? kT : 4];
  alignas(16) uint32_t wbase[kWarps][kRadix];
  uint32_t match[kWarps][kRadix];
  long long digit_base[kRadix];
  uint32_t scan_tmp[kWarps + 1];
  uint32_t tile_id;
};

// Stable multisplit of the records by digit = (bucket(key) >> shift) & 255:
// the onesweep scheme of radix.cuh (early counts, atomicOr match ranking,
// decoupled look-back) with a 64-bit and a 32-bit payload.  SRC_F64: the
// first pass, keys/v64 come from float64 arrays (encoded), v32 = index.
template <int ITEMS, bool V64, bool V32, bool SRC_F64>
__global__ void __launch_bounds__(kThreads, 3)
    msd_pass_kernel(const void* __restrict__ k_in, const void* __restrict__ v64_in, const uint32_t* __restrict__ v32_in,
                    uint64_t* __restrict__ k_out, uint64_t* __restrict__ v64_out, uint32_t* __restrict__ v32_out,
                    uint64_t n, const uint64_t* __restrict__ mm, int bits, int shift,
                    const uint32_t* __restrict__ bin_start, uint32_t* __restrict__ status,
                    uint32_t* __restrict__ tile_counter) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  using Smem = PassSmem<ITEMS, V64, V32>;
  constexpr int kT = Smem::kT;
  Smem& S = *reinterpret_cast<Smem*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  Bucketer BK;
  BK.init(mm, bits);
  {
    uint4* z = reinterpret_cast<uint4*>(&S.wbase[0][0]);
    constexpr int kZ = 2 * kWarps * kRadix / 4;
#pragma unroll
    for (int i = tid; i < kZ; i += kThreads) z[i] = make_uint4(0, 0, 0, 0);
  }
  if (tid == 0) S.tile_id = atomicAdd(tile_counter, 1u);
  __syncthreads();
  const uint32_t tile = S.tile_id;
  const uint64_t tile_base = (uint64_t)tile * kT;
  const uint64_t wb0 = tile_base + (uint64_t)warp * (32 * ITEMS);
  const uint32_t tile_valid = (uint32_t)umin64(kT, n - tile_base);

  uint64_t key[ITEMS], hv[ITEMS];
  uint32_t iv[ITEMS], dg[ITEMS];
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const uint64_t idx = wb0 + i * 32 + lane;
    if (idx < n) {
      if (SRC_F64) {
        key[i] = f64_key(__ldcs(reinterpret_cast<const double*>(k_in) + idx));
        if (V64) hv[i] = f64_key(__ldcs(reinterpret_cast<const double*>(v64_in) + idx));
        if (V32) iv[i] = (uint32_t)idx;
      } else {
        key[i] = __ldcs(reinterpret_cast<const uint64_t*>(k_in) + idx);
        if (V64) hv[i] = __ldcs(reinterpret_cast<const uint64_t*>(v64_in) + idx);
        if (V32) iv[i] = __ldcs(v32_in + idx);
      }
    } else {
      key[i] = 0;
      if (V64) hv[i] = 0;
      if (V32) iv[i] = 0;
    }
  }
  uint32_t* wb = S.wbase[warp];
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    dg[i] = (BK(key[i]) >> shift) & 255u;
    if (wb0 + i * 32 + lane < n) atomicAdd(&wb[dg[i]], 1u);
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
  uint32_t dummy;
  const uint32_t tstart = block_excl_scan<kThreads>(total, S.scan_tmp, &dummy);
#pragma unroll
  for (int w = 0; w < kWarps; ++w) S.wbase[w][tid] += tstart;
  __syncthreads();

  uint32_t* mmask = S.match[warp];
  const unsigned lt = lanemask_lt();
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
      S.keys[pos] = key[i];
      if (V64) S.v64[pos] = hv[i];
      if (V32) S.v32[pos] = iv[i];
    }
    __syncwarp();
  }

  uint32_t excl = 0;
  if (tile > 0) {
    constexpr int kLB = 8;
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
  S.digit_base[tid] = (long long)bin_start[tid] + (long long)excl - (long long)tstart;
  __syncthreads();

#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const uint32_t p = i * kThreads + tid;
    if (p < tile_valid) {
      const uint64_t k = S.keys[p];
      const uint32_t d = (BK(k) >> shift) & 255u;
      const uint64_t dst = (uint64_t)(S.digit_base[d] + (long long)p);
      k_out[dst] = k;
      if (V64) v64_out[dst] = S.v64[p];
      if (V32) v32_out[dst] = S.v32[p];
    }
  }
}

// ---------------------------------------------------------------- local sort

template <bool V64, bool V32>
struct LocalSmem {
  uint64_t keys[kCap];
  uint64_t v64[V64 ? kCap : 2];
  uint32_t v32[V32 ? kCap : 4];
  uint32_t bin[kFineBins + 1];
  uint16_t perm[kCap];     // sorted position -> staged index
  uint16_t binof[kCap];    // staged index -> fine bin
  uint64_t red[2 * kWarps];
  uint32_t flag;
};

// Stable sort of records [e0, e0 + c) by key inside shared memory (c <= kCap).
// Records arrive in (bucket, original-order) order.  Counting sort over fine
// value bins (monotone in the key), then a stable insertion sort by
// (key, staged index) inside each bin; if some bin is large (ties, dense
// clusters) the whole group is bitonic-sorted on (key, staged index) instead.
template <bool V64, bool V32>
__device__ void local_sort_group(LocalSmem<V64, V32>& S, const Bucketer& BK, int bits, const uint64_t* __restrict__ k_in,
                                 const uint64_t* __restrict__ v64_in, const uint32_t* __restrict__ v32_in,
                                 uint64_t* __restrict__ k_out, uint64_t* __restrict__ v64_out,
                                 uint32_t* __restrict__ v32_out, uint64_t e0, uint32_t c) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (uint32_t i = tid; i < c; i += kThreads) {
    S.keys[i] = __ldcs(k_in + e0 + i);
    if (V64) S.v64[i] = __ldcs(v64_in + e0 + i);
    if (V32) S.v32[i] = __ldcs(v32_in + e0 + i);
  }
  for (uint32_t b = tid; b <= kFineBins; b += kThreads) S.bin[b] = 0;
  if (tid == 0) S.flag = 0;
  __syncthreads();
  // fine value coordinate u = (x/2 - min/2) * scale * 2^20 (monotone); this
  // group's [umin, umax] selects the bin width
  const double fscale = BK.scale * 1048576.0;
  uint64_t umin = ~0ull, umax = 0;
  for (uint32_t i = tid; i < c; i += kThreads) {
    const double x = key_to_f64(S.keys[i]);
    const uint64_t u = (uint64_t)__double2ull_rz((x * 0.5 - BK.hmin) * fscale);
    umin = u < umin ? u : umin;
    umax = u > umax ? u : umax;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const uint64_t a = __shfl_xor_sync(kFull, umin, o), b = __shfl_xor_sync(kFull, umax, o);
    umin = a < umin ? a : umin;
    umax = b > umax ? b : umax;
  }
  if (lane == 0) { S.red[warp] = umin; S.red[kWarps + warp] = umax; }
  __syncthreads();
  umin = ~0ull;
  umax = 0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) {
    umin = S.red[w] < umin ? S.red[w] : umin;
    umax = S.red[kWarps + w] > umax ? S.red[kWarps + w] : umax;
  }
  int sh = 0;
  while (((umax - umin) >> sh) >= (uint64_t)kFineBins) ++sh;
  // histogram of fine bins
  for (uint32_t i = tid; i < c; i += kThreads) {
    const double x = key_to_f64(S.keys[i]);
    const uint64_t u = (uint64_t)__double2ull_rz((x * 0.5 - BK.hmin) * fscale);
    const uint32_t b = (uint32_t)((u - umin) >> sh);
    S.binof[i] = (uint16_t)b;
    atomicAdd(&S.bin[b], 1u);
  }
  __syncthreads();
  // exclusive scan over bins (16 per thread) + large-bin detection
  {
    constexpr int kPer = kFineBins / kThreads;
    uint32_t v[kPer], s = 0;
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      v[q] = S.bin[tid * kPer + q];
      s += v[q];
      if (v[q] > kMaxBinRun) S.flag = 1;
    }
    __shared__ uint32_t tmp[kWarps + 1];
    uint32_t tot;
    uint32_t ex = block_excl_scan<kThreads>(s, tmp, &tot);
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      S.bin[tid * kPer + q] = ex;
      ex += v[q];
    }
  }
  __syncthreads();
  const bool bitonic = S.flag != 0;
  if (!bitonic) {
    // scatter staged indices into bins (order inside a bin fixed below)
    for (uint32_t i = tid; i < c; i += kThreads) {
      const uint32_t pos = atomicAdd(&S.bin[S.binof[i]], 1u);
      S.perm[pos] = (uint16_t)i;
    }
    __syncthreads();
    // bins are [bin_end(b-1), bin_end(b)) now; insertion sort by (key, index)
    for (uint32_t b = tid; b < kFineBins; b += kThreads) {
      const uint32_t lo = b ? S.bin[b - 1] : 0, hi = S.bin[b];
      for (uint32_t x = lo + 1; x < hi; ++x) {
        const uint16_t v = S.perm[x];
        const uint64_t kv = S.keys[v];
        uint32_t y = x;
        while (y > lo) {
          const uint16_t w = S.perm[y - 1];
          const uint64_t kw = S.keys[w];
          if (kw < kv || (kw == kv && w < v)) break;
          S.perm[y] = w;
          --y;
        }
        S.perm[y] = v;
      }
    }
  } else {
    // bitonic sort of (key, index) over the next power of two
    uint32_t P = 1;
    while (P < c) P <<= 1;
    for (uint32_t i = tid; i < P; i += kThreads) S.perm[i] = (uint16_t)(i < c ? i : 0xffff);
    __syncthreads();
    for (uint32_t k = 2; k <= P; k <<= 1) {
      for (uint32_t j = k >> 1; j > 0; j >>= 1) {
        for (uint32_t i = tid; i < P; i += kThreads) {
          const uint32_t l = i ^ j;
          if (l > i) {
            const uint16_t a = S.perm[i], b = S.perm[l];
            // padding (0xffff) sorts last
            const bool a_gt_b = (a == 0xffff) ? (b != 0xffff)
                                : (b == 0xffff) ? false
                                : (S.keys[a] > S.keys[b] || (S.keys[a] == S.keys[b] && a > b));
            const bool up = (i & k) == 0;
            if (up == a_gt_b) { S.perm[i] = b; S.perm[l] = a; }
          }
        }
        __syncthreads();
      }
    }
  }
  __syncthreads();
  for (uint32_t i = tid; i < c; i += kThreads) {
    const uint16_t s = S.perm[i];
    k_out[e0 + i] = S.keys[s];
    if (V64) v64_out[e0 + i] = S.v64[s];
    if (V32) v32_out[e0 + i] = S.v32[s];
  }
  __syncthreads();
}

// One CTA per span of ~kSpan records made of whole buckets (span_lo); groups
// of consecutive buckets holding <= kCap records are sorted in smem.  A bucket
// larger than kCap sets *overflow (the caller falls back to the LSB sort).
template <bool V64, bool V32>
__global__ void __launch_bounds__(kThreads) local_sort_kernel(const uint64_t* __restrict__ k_in,
                                                              const uint64_t* __restrict__ v64_in,
                                                              const uint32_t* __restrict__ v32_in,
                                                              uint64_t* __restrict__ k_out,
                                                              uint64_t* __restrict__ v64_out,
                                                              uint32_t* __restrict__ v32_out,
                                                              const uint32_t* __restrict__ starts, uint32_t nb,
                                                              const uint32_t* __restrict__ span_lo,
                                                              const uint64_t* __restrict__ mm, int bits,
                                                              uint32_t* __restrict__ overflow) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  LocalSmem<V64, V32>& S = *reinterpret_cast<LocalSmem<V64, V32>*>(smem_raw);
  __shared__ uint64_t g_end;
  Bucketer BK;
  BK.init(mm, bits);
  uint64_t e0 = span_lo[blockIdx.x];
  const uint64_t e1 = span_lo[blockIdx.x + 1];
  while (e0 < e1) {
    uint64_t g1 = e1;
    if (e1 - e0 > kCap) {
      // largest bucket start in (e0, e0 + kCap]
      if (threadIdx.x == 0) {
        uint32_t lo = 0, hi = nb + 1;  // first index with starts[i] > e0 + kCap
        while (lo < hi) {
          const uint32_t mid = (lo + hi) >> 1;
          if (starts[mid] <= e0 + kCap) lo = mid + 1;
          else hi = mid;
        }
        const uint64_t s = lo ? starts[lo - 1] : 0;
        g_end = s > e0 ? s : ~0ull;
      }
      __syncthreads();
      g1 = g_end;
      __syncthreads();
      if (g1 == ~0ull) {  // one bucket alone exceeds the capacity
        if (threadIdx.x == 0) atomicOr(overflow, 1u);
        return;
      }
    }
    local_sort_group<V64, V32>(S, BK, bits, k_in, v64_in, v32_in, k_out, v64_out, v32_out, e0, (uint32_t)(g1 - e0));
    e0 = g1;
  }
}

}  // namespace msd
}  // namespace ddm
