// dyn.cuh -- dynamic DDM (the paper's future work, moving
// and resizing extents): k subscriptions of a built index take
// new coordinates, and the index is brought up to date by a MERGE instead of
// a rebuild.  For each sorted array (Slo in (key, id) order, Shi by key):
//  - keep[i] = 0 for the moved entries' old copies (a bitmap of moved ids
//    small enough to stay in L2 for Slo; the r-th removed copy of a value v
//    deletes Shi position lb(Shi, v) + r);
//  - the k new entries are sorted on their own, and new entry j's insertion
//    point p_j = #old entries ordered before it (p_j is non-decreasing in j);
//  - w[t] = keep[t] + #{j : p_j = t}; E = exclusive scan of w.  Then
//      old kept entry i  -> E[i] + (w[i] - keep[i])
//      new entry j       -> E[p_j] + (j - first j' with p_j' = p_j)
//    every element is written once, straight to its final position.
// Derived structures (block maxima, prefix maxima, d > 1 boxes) are then
// recomputed from the merged arrays; the result is byte-identical to
// ddm_sub_index_build on the modified region set (tested).
#pragma once
#include "common.cuh"

namespace ddm {
namespace dyn {

constexpr int kTile = 2048;  // scan tile (256 threads x 8)

// moved-id bitmap; ids must be strictly increasing and < n
__global__ void __launch_bounds__(256) mark_kernel(const uint32_t* __restrict__ ids, uint64_t k, uint64_t n,
                                                   uint32_t* __restrict__ bits, uint32_t* __restrict__ bad) {
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < k; j += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t id = ids[j];
    if (id >= n || (j > 0 && ids[j - 1] >= id)) {
      atomicOr(bad, 1u);
      continue;
    }
    atomicOr(bits + (id >> 5), 1u << (id & 31));
  }
}

__device__ __forceinline__ uint64_t lower_bound_u32(const uint32_t* a, uint64_t n, uint32_t x) {
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// Slo: w[i] = keep flag; the moved entries' old upper keys go to rhi[j]
// (j = the id's index in `ids`)
__global__ void __launch_bounds__(256) tomb_kernel(const uint32_t* __restrict__ slo_id,
                                                   const uint64_t* __restrict__ slo_hi, uint64_t n,
                                                   const uint32_t* __restrict__ bits, const uint32_t* __restrict__ ids,
                                                   uint64_t k, uint32_t* __restrict__ w, uint64_t* __restrict__ rhi) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t id = slo_id[i];
    const bool moved = (__ldg(bits + (id >> 5)) >> (id & 31)) & 1u;
    w[i] = moved ? 0u : 1u;
    if (moved) rhi[lower_bound_u32(ids, k, id)] = slo_hi[i];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) w[n] = 0;
}

__global__ void __launch_bounds__(256) fill_one_kernel(uint32_t* __restrict__ w, uint64_t n) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= n; i += (uint64_t)gridDim.x * blockDim.x)
    w[i] = i < n ? 1u : 0u;
}

// Shi: the r-th removed copy of value v clears position lb(Shi, v) + r
__global__ void __launch_bounds__(256) shi_tomb_kernel(const uint64_t* __restrict__ rhi_sorted, uint64_t k,
                                                       const uint64_t* __restrict__ shi, uint64_t n,
                                                       uint32_t* __restrict__ w, uint8_t* __restrict__ ks) {
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < k; j += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t v = rhi_sorted[j];
    uint64_t lo = 0, hi = j;
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (rhi_sorted[mid] < v) lo = mid + 1;
      else hi = mid;
    }
    uint64_t a = 0, b = n;
    while (a < b) {
      const uint64_t mid = (a + b) >> 1;
      if (shi[mid] < v) a = mid + 1;
      else b = mid;
    }
    w[a + (j - lo)] = 0;
    ks[a + (j - lo)] = 0;
  }
}

__device__ __forceinline__ bool less_kid(uint64_t ka, uint32_t ia, uint64_t kb, uint32_t ib) {
  return ka < kb || (ka == kb && ia < ib);
}

// insertion points of the new Slo entries: p_j = #old (key, id) < new (key, id)
__global__ void __launch_bounds__(256) slo_ins_kernel(const uint64_t* __restrict__ okey,
                                                      const uint32_t* __restrict__ oid, uint64_t n,
                                                      const uint64_t* __restrict__ nkey,
                                                      const uint32_t* __restrict__ nidx,
                                                      const uint32_t* __restrict__ ids, uint64_t k,
                                                      uint32_t* __restrict__ p, uint32_t* __restrict__ w) {
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < k; j += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t key = nkey[j];
    const uint32_t id = ids[nidx[j]];
    uint64_t lo = 0, hi = n;
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (less_kid(okey[mid], oid[mid], key, id)) lo = mid + 1;
      else hi = mid;
    }
    p[j] = (uint32_t)lo;
    atomicAdd(w + lo, 1u);
  }
}

// insertion points of the new Shi values: after every equal old value
__global__ void __launch_bounds__(256) shi_ins_kernel(const uint64_t* __restrict__ oshi, uint64_t n,
                                                      const uint64_t* __restrict__ nhi, uint64_t k,
                                                      uint32_t* __restrict__ p, uint32_t* __restrict__ w) {
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < k; j += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t v = nhi[j];
    uint64_t lo = 0, hi = n;
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (oshi[mid] <= v) lo = mid + 1;
      else hi = mid;
    }
    p[j] = (uint32_t)lo;
    atomicAdd(w + lo, 1u);
  }
}

// per-tile sums of w[0..len)
__global__ void __launch_bounds__(256) tile_sum_kernel(const uint32_t* __restrict__ w, uint64_t len,
                                                       uint64_t* __restrict__ tile_sum) {
  const uint64_t t0 = (uint64_t)blockIdx.x * kTile;
  uint64_t c = 0;
  for (int q = 0; q < kTile / 256; ++q) {
    const uint64_t i = t0 + (uint64_t)q * 256 + threadIdx.x;
    c += i < len ? w[i] : 0;
  }
  c = warp_sum<uint64_t>(c);
  __shared__ uint64_t s[8];
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t t = 0;
    for (int q = 0; q < 8; ++q) t += s[q];
    tile_sum[blockIdx.x] = t;
  }
}

// E[i] = sum(w[0..i)), i < len (tile offsets from scan_u64_kernel)
__global__ void __launch_bounds__(256) excl_scan_kernel(const uint32_t* __restrict__ w, uint64_t len,
                                                        const uint64_t* __restrict__ tile_off,
                                                        uint32_t* __restrict__ E) {
  __shared__ uint32_t tmp[256 / 32 + 1];
  const uint64_t b0 = (uint64_t)blockIdx.x * kTile + (uint64_t)threadIdx.x * 8;
  uint32_t v[8], s = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    v[q] = b0 + q < len ? w[b0 + q] : 0;
    s += v[q];
  }
  uint32_t tot;
  uint32_t ex = block_excl_scan<256>(s, tmp, &tot) + (uint32_t)tile_off[blockIdx.x];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    if (b0 + q < len) E[b0 + q] = ex;
    ex += v[q];
  }
}

struct SloArgs {
  // old arrays
  const uint64_t* okey;
  const uint32_t* oid;
  const uint64_t* ohi;
  const double* osd;
  const uint32_t* bits;  // moved ids
  const uint32_t* w;
  const uint32_t* E;
  uint64_t n;
  // new entries, sorted by (key, id), and their insertion points
  const uint64_t* nkey;
  const uint32_t* nidx;
  const uint32_t* ids;
  const uint32_t* p;
  const double* new_lo[8];
  const double* new_hi[8];
  uint64_t k;
  int d;
  // outputs
  uint64_t* key;
  uint32_t* id;
  uint64_t* hi;
  double* sd;
};

__global__ void __launch_bounds__(256) slo_old_kernel(const __grid_constant__ SloArgs A) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < A.n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t id = A.oid[i];
    if ((__ldg(A.bits + (id >> 5)) >> (id & 31)) & 1u) continue;
    const uint64_t q = (uint64_t)A.E[i] + (A.w[i] - 1u);
    A.key[q] = A.okey[i];
    A.id[q] = id;
    A.hi[q] = A.ohi[i];
    for (int kk = 1; kk < A.d; ++kk) {
      const uint64_t b = (uint64_t)(kk - 1) * 2 * A.n;
      A.sd[b + q] = A.osd[b + i];
      A.sd[b + A.n + q] = A.osd[b + A.n + i];
    }
  }
}

__device__ __forceinline__ uint64_t first_equal(const uint32_t* p, uint64_t j) {
  const uint32_t v = p[j];
  uint64_t lo = 0, hi = j;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (p[mid] < v) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__global__ void __launch_bounds__(256) slo_new_kernel(const __grid_constant__ SloArgs A) {
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < A.k; j += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t x = A.nidx[j];
    const uint64_t q = (uint64_t)A.E[A.p[j]] + (j - first_equal(A.p, j));
    A.key[q] = A.nkey[j];
    A.id[q] = A.ids[x];
    A.hi[q] = f64_key(A.new_hi[0][x]);
    for (int kk = 1; kk < A.d; ++kk) {
      const uint64_t b = (uint64_t)(kk - 1) * 2 * A.n;
      A.sd[b + q] = A.new_lo[kk][x];
      A.sd[b + A.n + q] = A.new_hi[kk][x];
    }
  }
}

// Shi: old kept values and new values to their final positions
__global__ void __launch_bounds__(256) shi_merge_kernel(const uint64_t* __restrict__ oshi,
                                                        const uint32_t* __restrict__ w,
                                                        const uint32_t* __restrict__ E, const uint8_t* __restrict__ ks,
                                                        uint64_t n, const uint64_t* __restrict__ nhi,
                                                        const uint32_t* __restrict__ p, uint64_t k,
                                                        uint64_t* __restrict__ shi) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n + k; i += stride) {
    if (i < n) {
      if (!ks[i]) continue;
      shi[(uint64_t)E[i] + (w[i] - 1u)] = oshi[i];
    } else {
      const uint64_t j = i - n;
      shi[(uint64_t)E[p[j]] + (j - first_equal(p, j))] = nhi[j];
    }
  }
}

}  // namespace dyn
}  // namespace ddm
