// slab.cuh -- on-device slab partition of the multi-GPU slab mode (sm_100a).
//
// SURVEY §8(e) / §8(f) #1 (fully distributed index).  Every rank starts with
// a block of the regions (its share of the input, global ids id_base + i)
// and the step redistributes them by dimension-0 coordinate slab:
//   * cut points c_1 < ... < c_{G-1}: quantiles of a sample of the update
//     lower bounds gathered from every rank (slab_sample_kernel ->
//     all_gather -> slab_cuts_kernel); slab r = [c_r, c_{r+1}), c_0 = -inf;
//   * an update goes to the rank of the slab holding its lower bound;
//   * a subscription S goes to every rank r whose slab it can reach:
//     S.hi >= c_r and S.lo <= reach_r = max U.hi over the updates of slab r
//     (all ranks, an all_reduce(MAX)).  The S with S.lo < c_r <= S.hi are the
//     stabbing set at the slab start -- Alg. 6's SubSet[p] at a segment
//     boundary, the slab's halo.  Every intersecting pair then has
//     both members on its update's rank, which finds it exactly once.
// Packing writes one row of 2d+1 words per (region, destination) --
// lo[0..d), hi[0..d), global id -- grouped by destination rank in index
// order, so one all_to_all per side moves them; unpacking restores the SoA
// arrays the matcher takes.  Regions are validated here (finite, lo <= hi in
// every dimension): a subscription that reaches no slab is still checked.
#pragma once
#include <climits>
#include "common.cuh"

namespace ddm {
namespace slab {

constexpr int kThreads = 256;
constexpr int kItems = 8;
constexpr int kTile = kThreads * kItems;
constexpr int kMaxWorld = 32;
constexpr int kMaxSample = 16384;  // gathered sample entries the cut kernel sorts in shared memory

// signed-orderable form of an order-preserving key (for MAX reductions on int64)
__device__ __forceinline__ long long key_signed(uint64_t k) { return (long long)(k ^ 0x8000000000000000ull); }

__global__ void __launch_bounds__(256) sample_kernel(const double* __restrict__ lo0, uint64_t count, uint32_t s,
                                                     double* __restrict__ out) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= s) return;
  // evenly spaced; a rank without regions contributes NaN (ignored by the cuts)
  out[i] = count ? lo0[(uint64_t)i * count / s] : __longlong_as_double(0x7ff8000000000000ll);
}

// One CTA: sort the gathered sample (non-finite entries last, ignored) and
// take cuts[r-1] = sorted[floor(r * valid / world)], r = 1..world-1.
__global__ void __launch_bounds__(1024) cuts_kernel(const double* __restrict__ sample, uint32_t s, uint32_t world,
                                                    double* __restrict__ cuts) {
  extern __shared__ double sv[];
  __shared__ uint32_t valid;
  uint32_t P = 1;
  while (P < s) P <<= 1;
  if (threadIdx.x == 0) valid = 0;
  __syncthreads();
  uint32_t mine = 0;
  for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) {
    double x = i < s ? sample[i] : __longlong_as_double(0x7ff0000000000000ll);
    const bool ok = i < s && isfinite(x);
    if (!ok) x = __longlong_as_double(0x7ff0000000000000ll);  // +inf: sorts last
    mine += ok;
    sv[i] = x;
  }
  atomicAdd(&valid, mine);
  __syncthreads();
  for (uint32_t k = 2; k <= P; k <<= 1)
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) {
        const uint32_t l = i ^ j;
        if (l > i) {
          const double a = sv[i], b = sv[l];
          if (((i & k) == 0) == (a > b)) { sv[i] = b; sv[l] = a; }
        }
      }
      __syncthreads();
    }
  const uint32_t v = valid;
  for (uint32_t r = 1 + threadIdx.x; r < world; r += blockDim.x)
    cuts[r - 1] = v ? sv[(uint32_t)min((uint64_t)r * v / world, (uint64_t)v - 1)] : 0.0;
}

struct PackArgs {
  int d;
  uint64_t count;
  const double* lo[8];
  const double* hi[8];
  uint64_t id_base;
  int side;                  // 0: subscriptions (halo rule), 1: updates (one slab)
  const double* cuts;        // world - 1
  const long long* reach;    // subscriptions: per slab max update upper key (key_signed), world
  uint32_t world;
  uint64_t tiles;
  uint64_t* tile_counts;     // [world][tiles] (count pass) -> exclusive offsets (scan)
  long long* reach_out;      // updates: per slab max upper key (key_signed), init INT64_MIN
  uint32_t* err;             // 1 non-finite, 2 inverted
  double* rows;              // scatter pass: [total][2d + 1]
};

// destination mask of region i (validating it)
__device__ __forceinline__ uint32_t dest_mask(const PackArgs& A, uint64_t i, uint32_t* err, uint64_t* hkey) {
  uint32_t e = 0;
  for (int k = 0; k < A.d; ++k) {
    const double l = A.lo[k][i], h = A.hi[k][i];
    if (!isfinite(l) || !isfinite(h)) e |= 1u;
    else if (!(l <= h)) e |= 2u;
  }
  *err |= e;
  const double l0 = A.lo[0][i], h0 = A.hi[0][i];
  *hkey = f64_key(h0);
  if (e) return 0;
  if (A.side == 1) {  // the slab holding the lower bound: #cuts <= lo
    uint32_t r = 0;
    while (r + 1 < A.world && A.cuts[r] <= l0) ++r;
    return 1u << r;
  }
  const long long lk = key_signed(f64_key(l0));
  uint32_t m = 0;
  for (uint32_t r = 0; r < A.world; ++r) {
    if (r > 0 && !(h0 >= A.cuts[r - 1])) break;  // S.hi >= c_r (a prefix of the ranks)
    if (lk <= A.reach[r]) m |= 1u << r;          // S.lo <= reach_r
  }
  return m;
}

// Count pass: per tile and destination, the rows it sends; updates also fold
// their upper keys into the per-slab maxima.
__global__ void __launch_bounds__(kThreads) count_kernel(const __grid_constant__ PackArgs A) {
  __shared__ uint32_t cnt[kMaxWorld];
  __shared__ long long rmax[kMaxWorld];
  const int tid = threadIdx.x;
  if (tid < kMaxWorld) { cnt[tid] = 0; rmax[tid] = LLONG_MIN; }
  __syncthreads();
  uint32_t err = 0;
  const uint64_t t = blockIdx.x;
  for (int k = 0; k < kItems; ++k) {
    const uint64_t i = t * kTile + (uint64_t)k * kThreads + tid;
    if (i >= A.count) break;
    uint64_t hk;
    uint32_t m = dest_mask(A, i, &err, &hk);
    if (A.side == 1 && m) atomicMax(&rmax[__ffs(m) - 1], key_signed(hk));
    while (m) {
      const int r = __ffs(m) - 1;
      m &= m - 1;
      atomicAdd(&cnt[r], 1u);
    }
  }
  err = __reduce_or_sync(kFull, err);
  if ((tid & 31) == 0 && err) atomicOr(A.err, err);
  __syncthreads();
  if (tid < (int)A.world) {
    A.tile_counts[(uint64_t)tid * A.tiles + t] = cnt[tid];
    if (A.side == 1 && rmax[tid] != LLONG_MIN) atomicMax(A.reach_out + tid, rmax[tid]);
  }
}

// Scatter pass: rows in index order within every destination, at the offsets
// the scan of tile_counts gave (destination-major: tile t's rows for rank r
// start at tile_counts[r * tiles + t]).
__global__ void __launch_bounds__(kThreads) scatter_kernel(const __grid_constant__ PackArgs A) {
  __shared__ uint32_t wcnt[kThreads / 32][kMaxWorld];
  __shared__ uint64_t wbase[kThreads / 32][kMaxWorld];
  __shared__ uint64_t run[kMaxWorld];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint64_t t = blockIdx.x;
  const int W = 2 * A.d + 1;
  const unsigned lt = lanemask_lt();
  if (tid < (int)A.world) run[tid] = A.tile_counts[(uint64_t)tid * A.tiles + t];
  uint32_t err = 0;
  for (int k = 0; k < kItems; ++k) {
    const uint64_t i = t * kTile + (uint64_t)k * kThreads + tid;
    uint64_t hk;
    const uint32_t m = i < A.count ? dest_mask(A, i, &err, &hk) : 0u;
    for (uint32_t r = 0; r < A.world; ++r) {
      const unsigned b = __ballot_sync(kFull, (m >> r) & 1u);
      if (lane == 0) wcnt[warp][r] = __popc(b);
    }
    __syncthreads();
    if (tid < (int)A.world) {  // per rank: the warps' bases in this round, then advance
      uint64_t acc = run[tid];
      for (int w = 0; w < kThreads / 32; ++w) {
        wbase[w][tid] = acc;
        acc += wcnt[w][tid];
      }
      run[tid] = acc;
    }
    __syncthreads();
    for (uint32_t r = 0; r < A.world; ++r) {
      const unsigned b = __ballot_sync(kFull, (m >> r) & 1u);
      if ((m >> r) & 1u) {
        double* row = A.rows + (wbase[warp][r] + __popc(b & lt)) * W;
        for (int q = 0; q < A.d; ++q) {
          row[q] = A.lo[q][i];
          row[A.d + q] = A.hi[q][i];
        }
        row[2 * A.d] = __longlong_as_double((long long)(A.id_base + i));
      }
    }
    __syncthreads();  // wcnt / wbase are rewritten by the next round
  }
}

// Unpack received rows into the SoA arrays of the matcher (lo[k], hi[k] of
// length count at stride `count`, ids u32).
__global__ void __launch_bounds__(256) unpack_kernel(const double* __restrict__ rows, uint64_t count, int d,
                                                     double* __restrict__ lo, double* __restrict__ hi,
                                                     uint32_t* __restrict__ ids) {
  const int W = 2 * d + 1;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
    const double* row = rows + i * W;
    for (int q = 0; q < d; ++q) {
      lo[(uint64_t)q * count + i] = row[q];
      hi[(uint64_t)q * count + i] = row[d + q];
    }
    ids[i] = (uint32_t)__double_as_longlong(row[2 * d]);
  }
}

}  // namespace slab
}  // namespace ddm
