// dyn.cuh -- dynamic DDM (the paper's future work, moving
// and resizing extents): k subscriptions of a built index take
// new coordinates, and the index is brought up to date by a MERGE instead of
// a rebuild.  The moved entries are tombstoned in the old sorted arrays, the
// k new entries are sorted on their own, and every surviving old entry and
// every new entry is scattered straight to its final position:
//   old kept entry i : pos = #kept before i + #new entries ordered before it
//   new entry j      : pos = j + #kept old entries ordered before it
// with the order (key, id) for Slo (so ties stay in id order, as a build
// sorts them) and the key alone for Shi (a multiset: equal keys are
// interchangeable).  Derived structures (block maxima, prefix maxima, d > 1
// boxes) are recomputed from the merged arrays.  The result is byte-identical
// to ddm_sub_index_build on the modified region set (tested).
#pragma once
#include "common.cuh"

namespace ddm {
namespace dyn {

constexpr int kTile = 2048;  // flag-scan tile (256 threads x 8)

// ids strictly increasing and < n; newidx[ids[j]] = j
__global__ void __launch_bounds__(256) mark_kernel(const uint32_t* __restrict__ ids, uint64_t k, uint64_t n,
                                                   uint32_t* __restrict__ newidx, uint32_t* __restrict__ bad) {
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < k; j += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t id = ids[j];
    if (id >= n || (j > 0 && ids[j - 1] >= id)) {
      atomicOr(bad, 1u);
      continue;
    }
    newidx[id] = (uint32_t)j;
  }
}

// keep[i] = slo entry i survives; the moved entries' old upper keys go to
// rhi[j] (j = the entry's index in the update)
__global__ void __launch_bounds__(256) tomb_kernel(const uint32_t* __restrict__ slo_id,
                                                   const uint64_t* __restrict__ slo_hi, uint64_t n,
                                                   const uint32_t* __restrict__ newidx, uint8_t* __restrict__ keep,
                                                   uint64_t* __restrict__ rhi) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t j = newidx[slo_id[i]];
    keep[i] = j == ~0u;
    if (j != ~0u) rhi[j] = slo_hi[i];
  }
}

// Shi tombs: the r-th removed copy of value v deletes Shi position lb(Shi, v) + r
__global__ void __launch_bounds__(256) shi_tomb_kernel(const uint64_t* __restrict__ rhi_sorted, uint64_t k,
                                                       const uint64_t* __restrict__ shi, uint64_t n,
                                                       uint8_t* __restrict__ keep_shi) {
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < k; j += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t v = rhi_sorted[j];
    uint64_t lo = 0, hi = j;  // first copy of v among the removed keys
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (rhi_sorted[mid] < v) lo = mid + 1;
      else hi = mid;
    }
    const uint64_t r = j - lo;
    uint64_t a = 0, b = n;  // lb(Shi, v)
    while (a < b) {
      const uint64_t mid = (a + b) >> 1;
      if (shi[mid] < v) a = mid + 1;
      else b = mid;
    }
    keep_shi[a + r] = 0;
  }
}

// per-tile sums of keep flags
__global__ void __launch_bounds__(256) flag_sum_kernel(const uint8_t* __restrict__ keep, uint64_t n,
                                                       uint64_t* __restrict__ tile_sum) {
  const uint64_t t0 = (uint64_t)blockIdx.x * kTile;
  uint32_t c = 0;
  for (int q = 0; q < kTile / 256; ++q) {
    const uint64_t i = t0 + (uint64_t)q * 256 + threadIdx.x;
    c += i < n ? keep[i] : 0;
  }
  c = warp_sum<uint32_t>(c);
  __shared__ uint32_t w[8];
  if ((threadIdx.x & 31) == 0) w[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t s = 0;
    for (int k = 0; k < 8; ++k) s += w[k];
    tile_sum[blockIdx.x] = s;
  }
}

// kb[i] = #kept before i, i = 0..n (tile offsets from scan_u64_kernel)
__global__ void __launch_bounds__(256) flag_scan_kernel(const uint8_t* __restrict__ keep, uint64_t n,
                                                        const uint64_t* __restrict__ tile_off,
                                                        uint32_t* __restrict__ kb) {
  __shared__ uint32_t tmp[256 / 32 + 1];
  const uint64_t t0 = (uint64_t)blockIdx.x * kTile;
  const uint64_t b0 = t0 + (uint64_t)threadIdx.x * 8;
  uint32_t v[8], s = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    v[q] = b0 + q < n ? keep[b0 + q] : 0;
    s += v[q];
  }
  uint32_t tot;
  uint32_t ex = block_excl_scan<256>(s, tmp, &tot) + (uint32_t)tile_off[blockIdx.x];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    if (b0 + q <= n) kb[b0 + q] = ex;  // (kb[n] = total kept)
    ex += v[q];
  }
}

struct SloArgs {
  // old arrays (copies) and flags
  const uint64_t* okey;
  const uint32_t* oid;
  const uint64_t* ohi;
  const double* osd;      // old sdims
  const uint8_t* keep;
  const uint32_t* kb;     // #kept before, [n + 1]
  uint64_t n;
  // new entries, sorted by (key, id)
  const uint64_t* nkey;
  const uint32_t* nidx;   // index into the update arrays
  const uint32_t* ids;    // update ids (strictly increasing)
  const double* new_lo[8];
  const double* new_hi[8];
  uint64_t k;
  int d;
  // outputs (the index)
  uint64_t* key;
  uint32_t* id;
  uint64_t* hi;
  double* sd;
};

__device__ __forceinline__ bool less_kid(uint64_t ka, uint32_t ia, uint64_t kb_, uint32_t ib) {
  return ka < kb_ || (ka == kb_ && ia < ib);
}

__global__ void __launch_bounds__(256) slo_old_kernel(const __grid_constant__ SloArgs A) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < A.n; i += (uint64_t)gridDim.x * blockDim.x) {
    if (!A.keep[i]) continue;
    const uint64_t key = A.okey[i];
    const uint32_t id = A.oid[i];
    uint64_t lo = 0, hi = A.k;  // #new entries ordered before (key, id)
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (less_kid(A.nkey[mid], A.ids[A.nidx[mid]], key, id)) lo = mid + 1;
      else hi = mid;
    }
    const uint64_t p = A.kb[i] + lo;
    A.key[p] = key;
    A.id[p] = id;
    A.hi[p] = A.ohi[i];
    for (int kk = 1; kk < A.d; ++kk) {
      A.sd[(uint64_t)(kk - 1) * 2 * A.n + p] = A.osd[(uint64_t)(kk - 1) * 2 * A.n + i];
      A.sd[(uint64_t)(kk - 1) * 2 * A.n + A.n + p] = A.osd[(uint64_t)(kk - 1) * 2 * A.n + A.n + i];
    }
  }
}

__global__ void __launch_bounds__(256) slo_new_kernel(const __grid_constant__ SloArgs A) {
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < A.k; j += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t key = A.nkey[j];
    const uint32_t x = A.nidx[j];
    const uint32_t id = A.ids[x];
    uint64_t lo = 0, hi = A.n;  // #old entries ordered before (key, id)
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (less_kid(A.okey[mid], A.oid[mid], key, id)) lo = mid + 1;
      else hi = mid;
    }
    const uint64_t p = j + A.kb[lo];
    A.key[p] = key;
    A.id[p] = id;
    A.hi[p] = f64_key(A.new_hi[0][x]);
    for (int kk = 1; kk < A.d; ++kk) {
      A.sd[(uint64_t)(kk - 1) * 2 * A.n + p] = A.new_lo[kk][x];
      A.sd[(uint64_t)(kk - 1) * 2 * A.n + A.n + p] = A.new_hi[kk][x];
    }
  }
}

// Shi: old kept value v -> kb[i] + lb(new, v); new value v (j-th) -> j + kb[ub(old, v)]
__global__ void __launch_bounds__(256) shi_merge_kernel(const uint64_t* __restrict__ oshi,
                                                        const uint8_t* __restrict__ keep,
                                                        const uint32_t* __restrict__ kb, uint64_t n,
                                                        const uint64_t* __restrict__ nhi, uint64_t k,
                                                        uint64_t* __restrict__ shi) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n + k; i += stride) {
    if (i < n) {
      if (!keep[i]) continue;
      const uint64_t v = oshi[i];
      uint64_t lo = 0, hi = k;
      while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (nhi[mid] < v) lo = mid + 1;
        else hi = mid;
      }
      shi[kb[i] + lo] = v;
    } else {
      const uint64_t j = i - n;
      const uint64_t v = nhi[j];
      uint64_t lo = 0, hi = n;
      while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (oshi[mid] <= v) lo = mid + 1;
        else hi = mid;
      }
      shi[j + kb[lo]] = v;
    }
  }
}

}  // namespace dyn
}  // namespace ddm
