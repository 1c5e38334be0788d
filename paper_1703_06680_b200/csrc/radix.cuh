// radix.cuh -- stable LSB "onesweep" radix sort for sm_100a (a2 / G2+G3).
//
// Sorts u64 keys (optionally carrying a u32 payload) by 8-bit digits.  One
// upfront kernel histograms every pass's digits in a single read of the keys;
// then each pass is ONE kernel: a CTA takes the next tile id from an atomic
// counter (forward progress for the look-back), ranks its 4096 keys with
// warp-level ballot multisplit (stable: warp-striped order), publishes its
// per-digit counts, resolves its global per-digit offsets by decoupled
// look-back over the preceding tiles' 30-bit status words, and scatters the
// keys digit-grouped from shared memory (coalesced runs).
//
// The first pass can read float64 coordinates directly and encode them into
// order-preserving keys (f64_key) with the payload = index (iota), so the
// encode step (a1) never materialises.  Paper step: "Sort T" (Alg. 4 l.5,
// P:420; Alg. 5 l.3); the paper's GNU parallel std::sort
// is prior art only.
#pragma once
#include "common.cuh"

namespace ddm {
namespace radix {

constexpr int kDigitBits = 8;
constexpr int kRadix = 1 << kDigitBits;
constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kItemsMax = 16;
constexpr int kTileMax = kThreads * kItemsMax;
// Resident CTAs per SM the pass kernel is compiled for, by items per thread.
__host__ __device__ constexpr int min_blocks_for(int items) { return items <= 8 ? 5 : items <= 12 ? 4 : 3; }
constexpr int kMaxPasses = 8;
constexpr uint32_t kFlagAgg = 1u << 30;
constexpr uint32_t kFlagPre = 2u << 30;
constexpr uint32_t kValMask = (1u << 30) - 1;

static_assert(kThreads == kRadix, "one thread per digit");

struct PassList {
  int n;
  int shift[kMaxPasses];
  uint32_t mask[kMaxPasses];
};

// ---------------------------------------------------------------- histogram

// Per-pass digit histograms of u64 keys (or of float64 values encoded on the
// fly).  hist: [n_passes][256], zeroed by the caller.
template <bool SRC_F64>
__global__ void __launch_bounds__(512) hist_kernel(const void* __restrict__ src, uint64_t n,
                                                   PassList passes, uint32_t* __restrict__ hist) {
  __shared__ uint32_t sh[kMaxPasses][kRadix];
  for (int i = threadIdx.x; i < kMaxPasses * kRadix; i += blockDim.x) (&sh[0][0])[i] = 0;
  __syncthreads();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    uint64_t k = SRC_F64 ? f64_key(__ldcs(reinterpret_cast<const double*>(src) + i))
                         : __ldcs(reinterpret_cast<const uint64_t*>(src) + i);
#pragma unroll
    for (int p = 0; p < kMaxPasses; ++p)
      if (p < passes.n) atomicAdd(&sh[p][(k >> passes.shift[p]) & passes.mask[p]], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < passes.n * kRadix; i += blockDim.x) {
    uint32_t v = (&sh[0][0])[i];
    if (v) atomicAdd(hist + i, v);
  }
}

// Exclusive scan of each pass's 256-bin histogram -> global bin starts.
// One block of 256 threads per pass.
__global__ void __launch_bounds__(kRadix) bin_start_kernel(const uint32_t* __restrict__ hist,
                                                         uint32_t* __restrict__ starts) {
  __shared__ uint32_t tmp[kRadix / 32 + 1];
  uint32_t total;
  const uint32_t v = hist[blockIdx.x * kRadix + threadIdx.x];
  starts[blockIdx.x * kRadix + threadIdx.x] = block_excl_scan<kRadix>(v, tmp, &total);
}

// ---------------------------------------------------------------- one pass

template <int ITEMS, bool HAS_VALS>
struct PassSmem {
  static constexpr int kTile = kThreads * ITEMS;
  uint64_t keys[kTile];
  uint32_t vals[HAS_VALS ? kTile : 4];
  alignas(16) uint32_t wbase[kWarps][kRadix];  // early counts -> per-warp running positions
  uint32_t match[kWarps][kRadix];  // per-warp peer masks (atomicOr match)
  long long digit_base[kRadix];
  uint32_t scan_tmp[kWarps + 1];
  uint32_t tile_id;
};

// One pass: tile = 256 threads x 16 keys.  "Early counts" ranking: the
// per-warp digit counts are taken first (order-agnostic smem atomics), so the
// tile's aggregate is published before the stable ranking runs and successor
// tiles' look-backs never wait for it.  Stable ranks within a warp come from
// a per-item peer mask (smem atomicOr match) and per-warp running bases.
template <int ITEMS, bool HAS_VALS, bool SRC_F64>
__global__ void __launch_bounds__(kThreads, min_blocks_for(ITEMS))
    onesweep_kernel(const void* __restrict__ keys_in, const uint32_t* __restrict__ vals_in,
                    uint64_t* __restrict__ keys_out, uint32_t* __restrict__ vals_out, uint64_t n,
                    int shift, uint32_t dmask, const uint32_t* __restrict__ bin_start,
                    uint32_t* __restrict__ status, uint32_t* __restrict__ tile_counter) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  using Smem = PassSmem<ITEMS, HAS_VALS>;
  constexpr int kItems = ITEMS;
  constexpr int kTile = Smem::kTile;
  Smem& S = *reinterpret_cast<Smem*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  {
    uint4* z = reinterpret_cast<uint4*>(&S.wbase[0][0]);
    constexpr int kZ = 2 * kWarps * kRadix / 4;
#pragma unroll
    for (int i = tid; i < kZ; i += kThreads) z[i] = make_uint4(0, 0, 0, 0);
  }
  if (tid == 0) S.tile_id = atomicAdd(tile_counter, 1u);
  __syncthreads();
  const uint32_t tile = S.tile_id;
  const uint64_t tile_base = (uint64_t)tile * kTile;
  const uint64_t wbase = tile_base + (uint64_t)warp * (32 * kItems);
  const uint32_t tile_valid = (uint32_t)umin64(kTile, n - tile_base);

  // load (warp-striped: element wbase + i*32 + lane), all loads in flight
  uint64_t key[kItems];
  uint32_t val[kItems];
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const uint64_t idx = wbase + i * 32 + lane;
    if (idx < n) {
      if (SRC_F64) {
        key[i] = f64_key(__ldcs(reinterpret_cast<const double*>(keys_in) + idx));
        if (HAS_VALS) val[i] = (uint32_t)idx;
      } else {
        key[i] = __ldcs(reinterpret_cast<const uint64_t*>(keys_in) + idx);
        if (HAS_VALS) val[i] = vals_in ? __ldcs(vals_in + idx) : (uint32_t)idx;
      }
    } else {
      key[i] = ~0ull;
      if (HAS_VALS) val[i] = 0;
    }
  }

  // early counts: per-warp digit histogram
  uint32_t* wb = S.wbase[warp];
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    if (wbase + i * 32 + lane < n) atomicAdd(&wb[(uint32_t)(key[i] >> shift) & dmask], 1u);
  }
  __syncthreads();

  // per digit (thread = digit): exclusive over warps, tile total; publish
  uint32_t total = 0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) {
    const uint32_t c = S.wbase[w][tid];
    S.wbase[w][tid] = total;
    total += c;
  }
  uint32_t* my_status = status + (uint64_t)tile * kRadix + tid;
  st_relaxed_u32(my_status, (tile == 0 ? kFlagPre : kFlagAgg) | total);
  uint32_t dummy;
  const uint32_t tstart = block_excl_scan<kThreads>(total, S.scan_tmp, &dummy);
#pragma unroll
  for (int w = 0; w < kWarps; ++w) S.wbase[w][tid] += tstart;
  __syncthreads();

  // stable ranking; keys go straight to their tile position in smem
  uint32_t* mm = S.match[warp];
  const unsigned lt = lanemask_lt();
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const bool valid = wbase + i * 32 + lane < n;
    const uint32_t digit = (uint32_t)(key[i] >> shift) & dmask;
    if (valid) atomicOr(&mm[digit], 1u << lane);
    __syncwarp();
    uint32_t peers = 0, base = 0;
    if (valid) {
      peers = mm[digit];
      base = wb[digit];
    }
    __syncwarp();
    if (valid) {
      const unsigned before = peers & lt;
      if (before == 0) {  // lowest lane of this digit group advances the base
        wb[digit] = base + __popc(peers);
        mm[digit] = 0;
      }
      const uint32_t pos = base + __popc(before);
      S.keys[pos] = key[i];
      if (HAS_VALS) S.vals[pos] = val[i];
    }
    __syncwarp();
  }

  // decoupled look-back for digit `tid`: read kLB predecessors per step
  uint32_t excl = 0;
  if (tile > 0) {
    constexpr int kLB = 8;
    int64_t p = (int64_t)tile - 1;
    while (true) {
      uint32_t sv[kLB];
#pragma unroll
      for (int k = 0; k < kLB; ++k)
        sv[k] = p - k >= 0 ? ld_relaxed_u32(status + (uint64_t)(p - k) * kRadix + tid) : kFlagPre;
      int consumed = 0;
      bool hit_pre = false;
#pragma unroll
      for (int q = 0; q < kLB; ++q) {
        if (hit_pre || consumed != q) break;
        const uint32_t v = sv[q];
        if ((v & ~kValMask) == 0) break;  // not published yet: re-read from here
        excl += v & kValMask;
        consumed = q + 1;
        hit_pre = (v & kFlagPre) != 0;
      }
      if (hit_pre) break;
      if (consumed == 0) __nanosleep(32);  // predecessor not published yet: back off
      p -= consumed;
    }
    st_relaxed_u32(my_status, kFlagPre | (excl + total));
  }
  S.digit_base[tid] = (long long)bin_start[tid] + (long long)excl - (long long)tstart;
  __syncthreads();

  // scatter: consecutive tile positions of one digit -> consecutive outputs
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const uint32_t p = i * kThreads + tid;
    if (p < tile_valid) {
      const uint64_t k = S.keys[p];
      const uint32_t digit = (uint32_t)(k >> shift) & dmask;
      const uint64_t dst = (uint64_t)(S.digit_base[digit] + (long long)p);
      keys_out[dst] = k;
      if (HAS_VALS) vals_out[dst] = S.vals[p];
    }
  }
}

// ---------------------------------------------------------------- host side

inline uint64_t num_tiles(uint64_t n, int items = 8) { return (n + (uint64_t)kThreads * items - 1) / ((uint64_t)kThreads * items); }

// Workspace carve for one sort of up to n keys: histograms, status words,
// tile counters, and the ping-pong key/value buffers.
struct Scratch {
  uint32_t* hist;      // [kMaxPasses][256]
  uint32_t* status;    // [tiles][256]
  uint32_t* counters;  // [kMaxPasses]
  uint64_t* alt_keys;  // [n]
  uint32_t* alt_vals;  // [n]
};

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

inline size_t scratch_bytes(uint64_t n, bool with_alt) {
  size_t b = align256(sizeof(uint32_t) * kMaxPasses * kRadix);
  b += align256(sizeof(uint32_t) * kRadix * (num_tiles(n) + 1));
  b += align256(sizeof(uint32_t) * kMaxPasses);
  if (with_alt) {
    b += align256(sizeof(uint64_t) * (n + 1));
    b += align256(sizeof(uint32_t) * (n + 1));
  }
  return b;
}

}  // namespace radix
}  // namespace ddm
