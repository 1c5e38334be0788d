// match.cuh -- validation, gathers, count+scan, and the sweep/emit kernels
// (a1, a3, a4+a5, a6+a7, a8 of DESIGN.md §2).
//
// Notation: Slo = subscription lower keys sorted ascending (stable: ties by
// sub id), slo_id the sub ids in that order, slo_hi[i] the upper key of the
// subscription at Slo position i, Shi = sorted subscription upper keys,
// Ulo/ulo_id/uhi the same for updates.  For an update U = [a, b]:
//   r_lo = #{S : S.lo <= a}   r_hi = #{S : S.hi < a}   r_b = #{S : S.lo <= b}
//   partners(U) = Stab(a) ⊔ Range(U)
//   Stab(a)  = { Slo[i] : i < r_lo, slo_hi[i] >= a },  |Stab(a)| = r_lo - r_hi
//   Range(U) = { Slo[i] : r_lo <= i < r_b }           (contiguous)
//   count(U) = r_b - r_hi                               (rank difference, I2)
// so every pair is reported exactly once, in the row of its update, which is
// the set Alg. 4 reports; rows are ordered by the sweep order of
// update lower endpoints and each row by Slo order (deterministic).
#pragma once
#include "common.cuh"

namespace ddm {
namespace match {

// ------------------------------------------------------------ validation (a1)

enum : uint32_t { kErrNonFinite = 1u, kErrInverted = 2u };

// Validate lo/hi of one dimension; optionally histogram the dim-0 keys of lo
// and/or hi for the radix sort (fused a1 + G2: one read of the inputs).
// hist_lo / hist_hi: [8][256] or nullptr.
__global__ void __launch_bounds__(512) validate_hist_kernel(const double* __restrict__ lo,
                                                            const double* __restrict__ hi,
                                                            uint64_t n, uint32_t* __restrict__ hist_lo,
                                                            uint32_t* __restrict__ hist_hi,
                                                            uint32_t* __restrict__ err) {
  __shared__ uint32_t hl[8][256];
  __shared__ uint32_t hh[8][256];
  __shared__ uint32_t serr;
  for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x) {
    (&hl[0][0])[i] = 0;
    (&hh[0][0])[i] = 0;
  }
  if (threadIdx.x == 0) serr = 0;
  __syncthreads();
  uint32_t e = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const double x = __ldcs(lo + i), y = __ldcs(hi + i);
    const uint64_t bx = (uint64_t)__double_as_longlong(x), by = (uint64_t)__double_as_longlong(y);
    if (!f64_finite_bits(bx) || !f64_finite_bits(by)) e |= kErrNonFinite;
    else if (!(x <= y)) e |= kErrInverted;
    if (hist_lo) {
      const uint64_t k = f64_key(x);
#pragma unroll
      for (int p = 0; p < 8; ++p) atomicAdd(&hl[p][(k >> (8 * p)) & 255], 1u);
    }
    if (hist_hi) {
      const uint64_t k = f64_key(y);
#pragma unroll
      for (int p = 0; p < 8; ++p) atomicAdd(&hh[p][(k >> (8 * p)) & 255], 1u);
    }
  }
  e = __reduce_or_sync(kFull, e);
  if ((threadIdx.x & 31) == 0 && e) atomicOr(&serr, e);
  __syncthreads();
  for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x) {
    if (hist_lo && (&hl[0][0])[i]) atomicAdd(hist_lo + i, (&hl[0][0])[i]);
    if (hist_hi && (&hh[0][0])[i]) atomicAdd(hist_hi + i, (&hh[0][0])[i]);
  }
  if (threadIdx.x == 0 && serr) atomicOr(err, serr);
}

// ------------------------------------------------------------ gathers (a3)

// out_key[i] = key(src[idx[i]]) and, when lvl1 != nullptr, lvl1[i/32] = max
// of the 32 keys of that aligned block (the first level of the block-max
// tree over Slo upper keys used to skip non-members in the stab scans).
__global__ void __launch_bounds__(256) gather_key_kernel(const uint32_t* __restrict__ idx,
                                                         const double* __restrict__ src, uint64_t n,
                                                         uint64_t* __restrict__ out_key,
                                                         uint64_t* __restrict__ lvl1) {
  constexpr int U = 8;  // independent gathers in flight per thread
  const uint64_t n_pad = (n + 31) & ~31ull;
  const uint64_t chunk = (uint64_t)blockDim.x * U;
  for (uint64_t base = (uint64_t)blockIdx.x * chunk; base < n_pad; base += (uint64_t)gridDim.x * chunk) {
    uint32_t id[U];
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t i = base + (uint64_t)u * blockDim.x + threadIdx.x;
      id[u] = i < n ? __ldcs(idx + i) : 0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t i = base + (uint64_t)u * blockDim.x + threadIdx.x;
      v[u] = i < n ? src[id[u]] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t i = base + (uint64_t)u * blockDim.x + threadIdx.x;
      uint64_t k = 0;
      if (i < n) {
        k = f64_key(v[u]);
        out_key[i] = k;
      }
      if (lvl1 && i < n_pad) {
        k = warp_max_u64(k);
        if ((threadIdx.x & 31) == 0) lvl1[i >> 5] = k;
      }
    }
  }
}

// lvl_out[b] = max(lvl_in[32b .. 32b+31]) (padding = 0, below every key).
__global__ void __launch_bounds__(256) block_max_kernel(const uint64_t* __restrict__ lvl_in,
                                                        uint64_t n_in, uint64_t* __restrict__ lvl_out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t n_pad = (n_in + 31) & ~31ull;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_pad; i += stride) {
    uint64_t k = i < n_in ? lvl_in[i] : 0;
    k = warp_max_u64(k);
    if ((threadIdx.x & 31) == 0) lvl_out[i >> 5] = k;
  }
}

// Other dimensions of the subscriptions, gathered into Slo order (d > 1):
// out[(k-1)*2*n + 0*n + i] = lo_k[idx[i]], out[(k-1)*2*n + n + i] = hi_k[idx[i]].
struct DimPtrs {
  const double* lo[8];
  const double* hi[8];
};

__global__ void __launch_bounds__(256) gather_dims_kernel(const uint32_t* __restrict__ idx, DimPtrs src,
                                                          int d, uint64_t n, double* __restrict__ out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint32_t s = __ldcs(idx + i);
    for (int k = 1; k < d; ++k) {
      out[(uint64_t)(k - 1) * 2 * n + i] = src.lo[k][s];
      out[(uint64_t)(k - 1) * 2 * n + n + i] = src.hi[k][s];
    }
  }
}

// ------------------------------------------------------------ searches

// first index in [lo, hi) with a[i] > x  (upper bound)
__device__ __forceinline__ uint64_t ub(const uint64_t* __restrict__ a, uint64_t lo, uint64_t hi, uint64_t x) {
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (a[mid] <= x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}
// first index in [lo, hi) with a[i] >= x  (lower bound)
__device__ __forceinline__ uint64_t lb(const uint64_t* __restrict__ a, uint64_t lo, uint64_t hi, uint64_t x) {
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}
// upper bound of x in a[0..n) knowing a[start-1] <= x: exponential probe
// forward from `start`, then binary search.
__device__ __forceinline__ uint64_t ub_gallop(const uint64_t* __restrict__ a, uint64_t n, uint64_t start,
                                              uint64_t x) {
  uint64_t lo = start, hi = n, step = 1;
  while (true) {
    const uint64_t probe = lo + step - 1;
    if (probe >= n) break;
    if (a[probe] > x) { hi = probe; break; }
    lo = probe + 1;
    step <<= 1;
  }
  return ub(a, lo, hi, x);
}

// ------------------------------------------------------------ decoupled look-back scan

constexpr uint64_t kScanAgg = 1ull << 62;
constexpr uint64_t kScanPre = 2ull << 62;
constexpr uint64_t kScanVal = (1ull << 62) - 1;

// Block-level: given this tile's aggregate, return the exclusive prefix of
// all preceding tiles (single thread, tid 0; result broadcast via smem).
__device__ __forceinline__ uint64_t lookback_u64(uint64_t* status, uint32_t tile, uint64_t agg) {
  if (tile == 0) {
    st_relaxed_u64(status, kScanPre | agg);
    return 0;
  }
  st_relaxed_u64(status + tile, kScanAgg | agg);
  uint64_t excl = 0;
  int64_t p = (int64_t)tile - 1;
  while (true) {
    const uint64_t s = ld_relaxed_u64(status + p);
    if ((s & ~kScanVal) == 0) continue;
    excl += s & kScanVal;
    if (s & kScanPre) break;
    --p;
  }
  st_relaxed_u64(status + tile, kScanPre | (excl + agg));
  return excl;
}

constexpr int kCountThreads = 256;
constexpr int kCountItems = 8;
constexpr int kCountTile = kCountThreads * kCountItems;

// a4 + a5 fused (G5 + G6): for every update j (in sorted Ulo order) compute
// r_lo, r_b and cnt = r_b - r_hi (rank difference, I2), then the exclusive
// scan off[j] = sum_{i<j} cnt[i] with a single-pass decoupled look-back;
// off[m] = K.  Each thread owns 8 consecutive updates: the first is located
// by binary search inside the tile's window, the rest by galloping forward
// (a is sorted, so r_lo and r_hi are monotone -- a merge path).
__global__ void __launch_bounds__(kCountThreads) count_scan_kernel(
    const uint64_t* __restrict__ ulo_key, const uint64_t* __restrict__ uhi, uint64_t m,
    const uint64_t* __restrict__ slo_key, const uint64_t* __restrict__ shi_key, uint64_t n,
    uint32_t* __restrict__ r_lo_out, uint32_t* __restrict__ r_b_out, uint64_t* __restrict__ off,
    uint64_t* __restrict__ status, uint32_t* __restrict__ tile_counter, uint64_t* __restrict__ k_out) {
  __shared__ uint64_t scan_tmp[kCountThreads / 32 + 1];
  __shared__ uint64_t win[4];
  __shared__ uint64_t prefix;
  __shared__ uint32_t tile_id;
  const int tid = threadIdx.x;
  if (tid == 0) tile_id = atomicAdd(tile_counter, 1u);
  __syncthreads();
  const uint32_t tile = tile_id;
  const uint64_t j0 = (uint64_t)tile * kCountTile;
  const uint64_t jn = umin64(kCountTile, m - j0);
  if (tid < 4) {
    const uint64_t a = ulo_key[(tid & 1) ? j0 + jn - 1 : j0];
    win[tid] = tid < 2 ? ub(slo_key, 0, n, a) : lb(shi_key, 0, n, a);
  }
  __syncthreads();
  const uint64_t t0 = (uint64_t)tid * kCountItems;
  uint32_t cnt[kCountItems];
  uint64_t local = 0;
  if (t0 < jn) {
    const uint64_t j = j0 + t0;
    const int ni = (int)umin64(kCountItems, jn - t0);
    uint64_t rl = ub(slo_key, win[0], win[1], ulo_key[j]);
    uint64_t rh = lb(shi_key, win[2], win[3], ulo_key[j]);
    uint64_t rb = rl, prev_b = 0;
    uint32_t ol[kCountItems], ob[kCountItems];
#pragma unroll
    for (int i = 0; i < kCountItems; ++i) {
      if (i < ni) {
        const uint64_t a = ulo_key[j + i], b = uhi[j + i];
        if (i) {
          rl = ub_gallop(slo_key, n, rl, a);
          // lb(Shi, a): gallop over entries < a
          uint64_t lo = rh, hi = n, step = 1;
          while (true) {
            const uint64_t probe = lo + step - 1;
            if (probe >= n) break;
            if (shi_key[probe] >= a) { hi = probe; break; }
            lo = probe + 1;
            step <<= 1;
          }
          rh = lb(shi_key, lo, hi, a);
        }
        const uint64_t start = (i && b >= prev_b && rb > rl) ? rb : rl;
        rb = ub_gallop(slo_key, n, start, b);
        prev_b = b;
        ol[i] = (uint32_t)rl;
        ob[i] = (uint32_t)rb;
        cnt[i] = (uint32_t)(rb > rh ? rb - rh : 0);
        local += cnt[i];
      } else {
        cnt[i] = 0;
      }
    }
#pragma unroll
    for (int i = 0; i < kCountItems; ++i)
      if (i < ni) { r_lo_out[j + i] = ol[i]; r_b_out[j + i] = ob[i]; }
  } else {
#pragma unroll
    for (int i = 0; i < kCountItems; ++i) cnt[i] = 0;
  }
  uint64_t agg;
  const uint64_t texcl = block_excl_scan<kCountThreads>(local, scan_tmp, &agg);
  if (tid == 0) prefix = lookback_u64(status, tile, agg);
  __syncthreads();
  uint64_t run = prefix + texcl;
#pragma unroll
  for (int i = 0; i < kCountItems; ++i) {
    if (t0 + i < jn) off[j0 + t0 + i] = run;
    run += cnt[i];
  }
  if (j0 + jn == m && tid == 0) {
    off[m] = prefix + agg;
    if (k_out) *k_out = prefix + agg;
  }
}

// Generic exclusive scan of u32 counts: off[j] = sum_{i<j} cnt[i], off[m] = total.
__global__ void __launch_bounds__(kCountThreads) scan_u32_kernel(const uint32_t* __restrict__ cnt, uint64_t m,
                                                                 uint64_t* __restrict__ off,
                                                                 uint64_t* __restrict__ status,
                                                                 uint32_t* __restrict__ tile_counter,
                                                                 uint64_t* __restrict__ k_out) {
  __shared__ uint64_t scan_tmp[kCountThreads / 32 + 1];
  __shared__ uint64_t prefix;
  __shared__ uint32_t tile_id;
  const int tid = threadIdx.x;
  if (tid == 0) tile_id = atomicAdd(tile_counter, 1u);
  __syncthreads();
  const uint32_t tile = tile_id;
  const uint64_t j0 = (uint64_t)tile * kCountTile;
  const uint64_t jn = umin64(kCountTile, m - j0);
  uint32_t c[kCountItems];
  uint64_t local = 0;
#pragma unroll
  for (int it = 0; it < kCountItems; ++it) {
    const uint64_t t = (uint64_t)tid * kCountItems + it;
    c[it] = t < jn ? cnt[j0 + t] : 0;
    local += c[it];
  }
  uint64_t agg;
  const uint64_t texcl = block_excl_scan<kCountThreads>(local, scan_tmp, &agg);
  if (tid == 0) prefix = lookback_u64(status, tile, agg);
  __syncthreads();
  uint64_t run = prefix + texcl;
#pragma unroll
  for (int it = 0; it < kCountItems; ++it) {
    const uint64_t t = (uint64_t)tid * kCountItems + it;
    if (t < jn) off[j0 + t] = run;
    run += c[it];
  }
  if (j0 + jn == m && tid == 0) {
    off[m] = prefix + agg;
    if (k_out) *k_out = prefix + agg;
  }
}

// ------------------------------------------------------------ sweep + emit (a6 + a7, a8)

// Stab-part scans walk Slo backwards from r_lo - 1 and stop after exactly
// |Stab(a)| = r_lo - r_hi members.  Aligned runs of 32^L positions whose
// block maximum of upper keys is < a hold no member and are skipped, so the
// cost is output-sensitive even with a few very long intervals.
__device__ __forceinline__ int skip_levels(const MaxTree& T, int64_t i, uint64_t a) {
  int L = 0;
  while (L < T.levels) {
    const int sh = 5 * (L + 1);
    if ((((uint64_t)i + 1) & ((1ull << sh) - 1)) != 0) break;
    if (T.lvl[L + 1][(uint64_t)i >> sh] >= a) break;
    ++L;
  }
  return L;
}

struct Filter {  // d > 1: dims 1..d-1 of the subs in Slo order + the query box
  int dims;      // d - 1 (0 for d == 1)
  const double* sdims;  // [(d-1)][2][n]
  uint64_t n;
};

struct UpdBox {
  double lo[8], hi[8];
};

__device__ __forceinline__ bool box_ok(const Filter& F, const UpdBox& q, uint64_t i) {
  for (int k = 0; k < F.dims; ++k) {
    const double slo = F.sdims[(uint64_t)k * 2 * F.n + i];
    const double shi = F.sdims[(uint64_t)k * 2 * F.n + F.n + i];
    if (!(slo <= q.hi[k] && q.lo[k] <= shi)) return false;  // Alg. 1 on dim k+1
  }
  return true;
}

struct EmitArgs {
  const uint64_t* ulo_key;
  const uint32_t* ulo_id;   // local update id (index into the update arrays)
  const uint32_t* upd_map;  // optional: global id of each local update
  const uint32_t* r_lo;
  const uint32_t* r_b;
  const uint64_t* off0;     // dim-0 row offsets (stab0 = cnt0 - range)
  const uint64_t* off;      // output row offsets (== off0 for d == 1)
  const uint32_t* fstab;    // d > 1 emit: filtered stab count per row
  uint32_t* cnt_out;        // d > 1 count pass: filtered row count
  uint32_t* fstab_out;      // d > 1 count pass: filtered stab count
  const uint32_t* slo_id;
  MaxTree T;
  Filter F;
  DimPtrs upd;              // d > 1: update coordinates (all dims)
  uint2* pairs;             // {sub, upd}
  uint64_t m;
  uint32_t thread_row_max;  // rows with <= this many dim-0 candidates go thread-per-row
  uint32_t force;           // 0 auto, 1 thread, 2 warp
};

enum EmitMode { kEmitD1 = 0, kCountDD = 1, kEmitDD = 2 };

constexpr int kEmitThreads = 256;

// ---- one row, one thread
template <int MODE>
__device__ __forceinline__ void row_thread(const EmitArgs& A, uint64_t j) {
  const uint64_t a = A.ulo_key[j];
  const uint32_t lid = A.ulo_id[j];
  const uint32_t uid = A.upd_map ? A.upd_map[lid] : lid;
  const uint32_t rl = A.r_lo[j], rb = A.r_b[j];
  const uint64_t c0 = A.off0[j + 1] - A.off0[j];
  const uint32_t stab0 = (uint32_t)(c0 - (rb - rl));
  UpdBox q;
  if (MODE != kEmitD1)
    for (int k = 0; k < A.F.dims; ++k) { q.lo[k] = A.upd.lo[k + 1][lid]; q.hi[k] = A.upd.hi[k + 1][lid]; }
  const uint64_t o = MODE == kCountDD ? 0 : A.off[j];
  uint32_t fst = MODE == kEmitDD ? A.fstab[j] : stab0;  // write cursor (backwards) for the stab part
  uint32_t nst = 0;                                      // filtered stab members (count pass)
  // stab part: backwards from rl-1, exactly stab0 dim-0 members
  int64_t i = (int64_t)rl - 1;
  uint32_t rem = stab0;
  while (rem) {
    if ((i & 31) == 31) {
      const int L = skip_levels(A.T, i, a);
      if (L) { i -= (int64_t)1 << (5 * L); continue; }
    }
    if (A.T.lvl[0][i] >= a) {
      --rem;
      if (MODE == kEmitD1) {
        A.pairs[o + rem] = make_uint2(A.slo_id[i], uid);
      } else if (box_ok(A.F, q, (uint64_t)i)) {
        if (MODE == kCountDD) ++nst;
        else A.pairs[o + (--fst)] = make_uint2(A.slo_id[i], uid);
      }
    }
    --i;
  }
  // range part: Slo[rl, rb)
  if (MODE == kEmitD1) {
    for (uint32_t k = rl; k < rb; ++k) A.pairs[o + stab0 + (k - rl)] = make_uint2(A.slo_id[k], uid);
  } else {
    const uint32_t base = MODE == kEmitDD ? A.fstab[j] : 0;
    uint32_t w = 0;
    for (uint32_t k = rl; k < rb; ++k) {
      if (box_ok(A.F, q, k)) {
        if (MODE == kEmitDD) A.pairs[o + base + w] = make_uint2(A.slo_id[k], uid);
        ++w;
      }
    }
    if (MODE == kCountDD) { A.cnt_out[j] = nst + w; A.fstab_out[j] = nst; }
  }
}

// ---- one row, one warp (coalesced 32-wide windows, ballot/popc compaction)
template <int MODE>
__device__ __forceinline__ void row_warp(const EmitArgs& A, uint64_t j, int lane) {
  const uint64_t a = A.ulo_key[j];
  const uint32_t lid = A.ulo_id[j];
  const uint32_t uid = A.upd_map ? A.upd_map[lid] : lid;
  const uint32_t rl = A.r_lo[j], rb = A.r_b[j];
  const uint64_t c0 = A.off0[j + 1] - A.off0[j];
  const uint32_t stab0 = (uint32_t)(c0 - (rb - rl));
  UpdBox q;
  if (MODE != kEmitD1)
    for (int k = 0; k < A.F.dims; ++k) { q.lo[k] = A.upd.lo[k + 1][lid]; q.hi[k] = A.upd.hi[k + 1][lid]; }
  const uint64_t o = MODE == kCountDD ? 0 : A.off[j];
  uint32_t fst = MODE == kEmitDD ? A.fstab[j] : stab0;
  uint32_t nst = 0;
  int64_t hi_excl = rl;
  uint32_t rem = stab0;
  while (rem) {
    const int64_t i = hi_excl - 1;
    if ((i & 31) == 31) {
      const int L = skip_levels(A.T, i, a);
      if (L) { hi_excl -= (int64_t)1 << (5 * L); continue; }
    }
    const int64_t base = i & ~31ll;
    const int64_t idx = base + lane;
    const bool member = idx < hi_excl && A.T.lvl[0][idx] >= a;
    const unsigned mm = __ballot_sync(kFull, member);
    rem -= __popc(mm);
    if (MODE == kEmitD1) {
      if (member) A.pairs[o + rem + __popc(mm & lanemask_lt())] = make_uint2(A.slo_id[idx], uid);
    } else {
      const bool keep = member && box_ok(A.F, q, (uint64_t)idx);
      const unsigned km = __ballot_sync(kFull, keep);
      if (MODE == kCountDD) nst += __popc(km);
      else {
        fst -= __popc(km);
        if (keep) A.pairs[o + fst + __popc(km & lanemask_lt())] = make_uint2(A.slo_id[idx], uid);
      }
    }
    hi_excl = base;
  }
  if (MODE == kEmitD1) {
    for (uint64_t k = (uint64_t)rl + lane; k < rb; k += 32)
      A.pairs[o + stab0 + (k - rl)] = make_uint2(A.slo_id[k], uid);
  } else {
    uint32_t w = MODE == kEmitDD ? A.fstab[j] : 0;
    for (uint64_t k0 = rl; k0 < rb; k0 += 32) {
      const uint64_t k = k0 + lane;
      const bool keep = k < rb && box_ok(A.F, q, k);
      const unsigned km = __ballot_sync(kFull, keep);
      if (MODE == kEmitDD && keep) A.pairs[o + w + __popc(km & lanemask_lt())] = make_uint2(A.slo_id[k], uid);
      w += __popc(km);
    }
    if (MODE == kCountDD && lane == 0) { A.cnt_out[j] = nst + w; A.fstab_out[j] = nst; }
  }
}

// One CTA per 256 consecutive updates (sorted order).  Rows with few dim-0
// candidates are done by their own thread; long rows are queued and taken
// by whole warps, so both sparse (alpha ~ 1: ~1 pair per row) and dense rows
// (alpha = 100: ~100 pairs per row) stream coalesced stores.
template <int MODE>
__global__ void __launch_bounds__(kEmitThreads) emit_kernel(EmitArgs A) {
  __shared__ uint32_t queue[kEmitThreads];
  __shared__ uint32_t qn;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) qn = 0;
  __syncthreads();
  const uint64_t j = (uint64_t)blockIdx.x * kEmitThreads + tid;
  if (j < A.m) {
    const uint64_t c0 = A.off0[j + 1] - A.off0[j];
    const bool thread_row = A.force == 1 || (A.force == 0 && c0 <= A.thread_row_max);
    if (thread_row) row_thread<MODE>(A, j);
    else queue[atomicAdd(&qn, 1u)] = tid;
  }
  __syncthreads();
  const uint32_t nq = qn;
  for (uint32_t q = warp; q < nq; q += kEmitThreads / 32)
    row_warp<MODE>(A, (uint64_t)blockIdx.x * kEmitThreads + queue[q], lane);
}

// ------------------------------------------------------------ pair canonical key

// 64-bit view of the pairs for the canonical sort: (upd << 32) | sub.
static_assert(sizeof(uint2) == 8, "pair layout");

}  // namespace match
}  // namespace ddm
