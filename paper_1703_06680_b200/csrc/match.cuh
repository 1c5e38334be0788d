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
//            = (r_b - r_lo) + #{i < r_lo : slo_hi[i] >= a} (walk form, R23)
// so every pair is reported exactly once, in the row of its update, which is
// the set Alg. 4 reports; rows are ordered by the sweep order of
// update lower endpoints and each row by Slo order (deterministic).
#pragma once
#include <cstddef>
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
                                                            uint32_t* __restrict__ err,
                                                            uint64_t* __restrict__ mm_lo,
                                                            uint64_t* __restrict__ mm_hi) {
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
  uint64_t lmin = ~0ull, lmax = 0, hmin = ~0ull, hmax = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const double x = __ldcs(lo + i), y = __ldcs(hi + i);
    const uint64_t bx = (uint64_t)__double_as_longlong(x), by = (uint64_t)__double_as_longlong(y);
    if (!f64_finite_bits(bx) || !f64_finite_bits(by)) e |= kErrNonFinite;
    else if (!(x <= y)) e |= kErrInverted;
    if (mm_lo) {
      const uint64_t kx = f64_key(x), ky = f64_key(y);
      lmin = kx < lmin ? kx : lmin;
      lmax = kx > lmax ? kx : lmax;
      hmin = ky < hmin ? ky : hmin;
      hmax = ky > hmax ? ky : hmax;
    }
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
  if (mm_lo) {  // min/max keys (value-bucketed MSD sort); non-finite values are rejected anyway
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      uint64_t t;
      t = __shfl_xor_sync(kFull, lmin, o); lmin = t < lmin ? t : lmin;
      t = __shfl_xor_sync(kFull, lmax, o); lmax = t > lmax ? t : lmax;
      t = __shfl_xor_sync(kFull, hmin, o); hmin = t < hmin ? t : hmin;
      t = __shfl_xor_sync(kFull, hmax, o); hmax = t > hmax ? t : hmax;
    }
    if ((threadIdx.x & 31) == 0) {
      atomicMin((unsigned long long*)&mm_lo[0], (unsigned long long)lmin);
      atomicMax((unsigned long long*)&mm_lo[1], (unsigned long long)lmax);
      if (mm_hi) {
        atomicMin((unsigned long long*)&mm_hi[0], (unsigned long long)hmin);
        atomicMax((unsigned long long*)&mm_hi[1], (unsigned long long)hmax);
      }
    }
  }
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

// Levels from .. levels of the block-max tree in one launch (instead of one
// block_max launch per level): each thread builds one level-`from` entry from
// its 32 level-(from-1) entries (16-byte loads, all in flight at once), each
// warp the level-(from+1) entry above its 32 lanes; the last CTA to finish
// (ticket, reset for the next call) builds the levels above those.
struct TreeLv {
  uint64_t* lvl[kMaxLevels + 1];
  uint64_t n[kMaxLevels + 1];
  int levels;
};
__device__ __forceinline__ uint64_t max32(const uint64_t* __restrict__ in, uint64_t n_in, uint64_t o, bool l2) {
  const uint64_t i0 = o * 32;
  uint64_t v = 0;
  if (i0 + 32 <= n_in) {
    const ulonglong2* p = reinterpret_cast<const ulonglong2*>(in + i0);
    ulonglong2 x[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) x[k] = l2 ? __ldcg(p + k) : __ldg(p + k);
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      v = x[k].x > v ? x[k].x : v;
      v = x[k].y > v ? x[k].y : v;
    }
  } else {
    for (uint64_t i = i0; i < n_in; ++i) {
      const uint64_t w = l2 ? __ldcg(in + i) : __ldg(in + i);
      v = w > v ? w : v;
    }
  }
  return v;  // (padding = 0, below every key)
}
__global__ void __launch_bounds__(256) tree_levels_kernel(const __grid_constant__ TreeLv T, int from,
                                                          uint32_t* __restrict__ ticket) {
  __shared__ bool last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint64_t o = (uint64_t)blockIdx.x * 256 + tid;
  const uint64_t v = o < T.n[from] ? max32(T.lvl[from - 1], T.n[from - 1], o, false) : 0;
  if (o < T.n[from]) T.lvl[from][o] = v;
  if (from + 1 <= T.levels) {
    const uint64_t w = warp_max_u64(v);
    const uint64_t o1 = (uint64_t)blockIdx.x * 8 + warp;
    if (lane == 0 && o1 < T.n[from + 1]) T.lvl[from + 1][o1] = w;
  }
  if (from + 2 > T.levels) return;
  __threadfence();
  __syncthreads();
  if (tid == 0) last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int L = from + 2; L <= T.levels; ++L) {  // (other CTAs' writes: read from L2)
    for (uint64_t q = tid; q < T.n[L]; q += 256) T.lvl[L][q] = max32(T.lvl[L - 1], T.n[L - 1], q, true);
    __threadfence_block();
    __syncthreads();
  }
  if (tid == 0) *ticket = 0;
}

// a3' (pairs mode): levels 1 and 2 of the block-max tree and the prefix
// maxima of the Slo upper keys, in one read of slo_hi.  With 1024-entry
// blocks, pmw[i] = max(slo_hi[1024*(i/1024) .. i]) and, after
// pmb_scan_kernel, pmb[B] = max(slo_hi[0 .. 1024*B)), so
//   max(slo_hi[0..i]) = max(pmw[i], pmb[i/1024])
// which is the stop test of the counting stab walk (count_kernel<true>):
// no position at or before i can hold a member of Stab(a) once it is < a.
// lvl1 / lvl2 may be nullptr (not kept, or the tree has fewer levels).
constexpr int kPmBlock = 1024;
__global__ void __launch_bounds__(256) tree_pm_kernel(const uint64_t* __restrict__ hi, uint64_t n,
                                                      uint64_t* __restrict__ lvl1, uint64_t n1,
                                                      uint64_t* __restrict__ lvl2, uint64_t* __restrict__ pmw,
                                                      uint64_t* __restrict__ pmb) {
  __shared__ uint64_t wt[8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t B = blockIdx.x;
  const uint64_t base = B * kPmBlock + (uint64_t)threadIdx.x * 4;
  uint64_t v[4];
  if (base + 4 <= n) {
    const ulonglong2* p = reinterpret_cast<const ulonglong2*>(hi + base);
    const ulonglong2 x = __ldcs(p), y = __ldcs(p + 1);
    v[0] = x.x; v[1] = x.y; v[2] = y.x; v[3] = y.y;
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = base + k < n ? __ldcs(hi + base + k) : 0;
  }
#pragma unroll
  for (int k = 1; k < 4; ++k) v[k] = v[k] > v[k - 1] ? v[k] : v[k - 1];  // running max
  const uint64_t t = v[3];
  uint64_t inc = t;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t w = __shfl_up_sync(kFull, inc, o);
    if (lane >= o && w > inc) inc = w;
  }
  uint64_t excl = __shfl_up_sync(kFull, inc, 1);
  if (lane == 0) excl = 0;
  if (lvl1) {  // 32 entries = 8 threads
    uint64_t g = t;
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
      const uint64_t w = __shfl_xor_sync(kFull, g, o);
      g = w > g ? w : g;
    }
    const uint64_t idx = B * (kPmBlock / 32) + (threadIdx.x >> 3);
    if ((lane & 7) == 0 && idx < n1) lvl1[idx] = g;
  }
  if (lane == 31) wt[warp] = inc;
  __syncthreads();
  uint64_t pre = excl;
  for (int w = 0; w < warp; ++w) pre = wt[w] > pre ? wt[w] : pre;
#pragma unroll
  for (int k = 0; k < 4; ++k) v[k] = v[k] > pre ? v[k] : pre;
  if (base + 4 <= n) {
    ulonglong2* q = reinterpret_cast<ulonglong2*>(pmw + base);
    q[0] = make_ulonglong2(v[0], v[1]);
    q[1] = make_ulonglong2(v[2], v[3]);
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (base + k < n) pmw[base + k] = v[k];
  }
  if (threadIdx.x == 255) {  // the block maximum (v[3] of the last thread)
    pmb[B] = v[3];
    if (lvl2) lvl2[B] = v[3];
  }
}

// Stab-density probe (pairs calls, d = 1): an estimate of the mean
// |Stab(a)| at a uniform point, n * mean(hi - lo) / (max lo - min lo) over
// 4096 evenly spaced subscriptions; +inf when a sampled value is non-finite
// (the validation reports it).  One CTA.
// Also: the fraction of sampled subscriptions (out[1]) and updates (out[2])
// whose upper key lies 2^32 - 1 or more key units above the lower key -- the
// records the packed MSD sort cannot pack (msd.cuh TileRegs): the pack
// decision of the call.
constexpr int kProbe = 4096;
__device__ __forceinline__ double unfit_fraction(const double* __restrict__ lo, const double* __restrict__ hi,
                                                 uint64_t n, int* scratch) {
  int cnt = 0;
  if (n)
    for (int k = threadIdx.x; k < kProbe; k += blockDim.x) {
      const uint64_t i = (uint64_t)((unsigned __int128)k * n / kProbe);
      const double a = lo[i], b = hi[i];
      if (!isfinite(a) || !isfinite(b) || !(a <= b)) continue;
      cnt += f64_key(b) - f64_key(a) >= 0xffffffffull;
    }
  cnt = __reduce_add_sync(kFull, cnt);
  if ((threadIdx.x & 31) == 0) atomicAdd(scratch, cnt);
  __syncthreads();
  const double f = n ? (double)*scratch / (double)kProbe : 0.0;
  __syncthreads();
  return f;
}

__global__ void __launch_bounds__(256) stab_density_kernel(const double* __restrict__ lo,
                                                           const double* __restrict__ hi, uint64_t n,
                                                           const double* __restrict__ ulo,
                                                           const double* __restrict__ uhi, uint64_t m,
                                                           double* __restrict__ out) {
  __shared__ double s_len[8], s_min[8], s_max[8];
  __shared__ int s_bad, s_cnt[2];
  if (threadIdx.x == 0) { s_bad = 0; s_cnt[0] = 0; s_cnt[1] = 0; }
  __syncthreads();
  const double fs = unfit_fraction(lo, hi, n, &s_cnt[0]);
  const double fu = unfit_fraction(ulo, uhi, m, &s_cnt[1]);
  if (threadIdx.x == 0) { out[1] = fs; out[2] = fu; }
  double len = 0.0, mn = INFINITY, mx = -INFINITY;
  int bad = 0;
  for (int k = threadIdx.x; k < kProbe; k += blockDim.x) {
    const uint64_t i = (uint64_t)((unsigned __int128)k * n / kProbe);
    const double a = lo[i], b = hi[i];
    if (!isfinite(a) || !isfinite(b)) { bad = 1; continue; }
    len += b > a ? b - a : 0.0;
    mn = fmin(mn, a);
    mx = fmax(mx, a);
  }
  for (int o = 16; o; o >>= 1) {
    len += __shfl_xor_sync(kFull, len, o);
    mn = fmin(mn, __shfl_xor_sync(kFull, mn, o));
    mx = fmax(mx, __shfl_xor_sync(kFull, mx, o));
  }
  if (bad) s_bad = 1;
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) { s_len[w] = len; s_min[w] = mn; s_max[w] = mx; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < 8; ++k) { len += s_len[k]; mn = fmin(mn, s_min[k]); mx = fmax(mx, s_max[k]); }
    const double span = mx - mn;
    const double mean = len / (double)kProbe;
    out[0] = (s_bad || !(span > 0.0)) ? INFINITY : (double)n * mean / span;
  }
}

// Sweep-dimension probe (d > 1; SURVEY §8(a) a8 "k* = argmin_k K_k"): per
// dimension k an estimate of the dim-k candidate pairs K_k up to the common
// factor n*m -- (mean S length + mean U length) / (max lo - min lo) over 4096
// evenly spaced regions of each kind (uniformly placed intervals overlap with
// that probability).  out[k]; +inf when the span is empty or a sampled value is
// non-finite (the validation reports it).  One CTA per dimension.
struct ProbeDims {
  const double* sub_lo[8];
  const double* sub_hi[8];
  const double* upd_lo[8];
  const double* upd_hi[8];
};
__global__ void __launch_bounds__(256) dim_probe_kernel(const __grid_constant__ ProbeDims P, uint64_t n, uint64_t m,
                                                        double* __restrict__ out) {
  __shared__ double s_v[4][8];
  __shared__ int s_bad;
  const int k = blockIdx.x;
  if (threadIdx.x == 0) s_bad = 0;
  __syncthreads();
  double ls = 0.0, lu = 0.0, mn = INFINITY, mx = -INFINITY;
  int bad = 0;
  for (int t = threadIdx.x; t < kProbe; t += blockDim.x) {
    const uint64_t i = (uint64_t)((unsigned __int128)t * n / kProbe), j = (uint64_t)((unsigned __int128)t * m / kProbe);
    const double a = P.sub_lo[k][i], b = P.sub_hi[k][i], c = P.upd_lo[k][j], e = P.upd_hi[k][j];
    if (!isfinite(a) || !isfinite(b) || !isfinite(c) || !isfinite(e)) { bad = 1; continue; }
    ls += b > a ? b - a : 0.0;
    lu += e > c ? e - c : 0.0;
    mn = fmin(mn, fmin(a, c));
    mx = fmax(mx, fmax(a, c));
  }
  for (int o = 16; o; o >>= 1) {
    ls += __shfl_xor_sync(kFull, ls, o);
    lu += __shfl_xor_sync(kFull, lu, o);
    mn = fmin(mn, __shfl_xor_sync(kFull, mn, o));
    mx = fmax(mx, __shfl_xor_sync(kFull, mx, o));
  }
  if (bad) s_bad = 1;
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) { s_v[0][w] = ls; s_v[1][w] = lu; s_v[2][w] = mn; s_v[3][w] = mx; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int q = 1; q < 8; ++q) { ls += s_v[0][q]; lu += s_v[1][q]; mn = fmin(mn, s_v[2][q]); mx = fmax(mx, s_v[3][q]); }
    const double span = mx - mn;
    out[k] = (s_bad || !(span > 0.0)) ? INFINITY : (ls + lu) / (double)kProbe / span;
  }
}

// Exclusive max-scan of the nb block maxima, in place: chunks of
// kPmChunk = 8192 blocks; pmb_chunk_kernel writes each chunk's maximum,
// pmb_scan_kernel scans a chunk after taking the maximum of the chunks
// before it (at most nb / 8192 values).
constexpr int kPmChunk = 8192;
__global__ void __launch_bounds__(1024) pmb_chunk_kernel(const uint64_t* __restrict__ pmb, uint64_t nb,
                                                         uint64_t* __restrict__ cmax) {
  __shared__ uint64_t wt[32];
  const uint64_t c0 = (uint64_t)blockIdx.x * kPmChunk;
  uint64_t mx = 0;
#pragma unroll
  for (int k = 0; k < kPmChunk / 1024; ++k) {
    const uint64_t i = c0 + (uint64_t)k * 1024 + threadIdx.x;
    const uint64_t x = i < nb ? pmb[i] : 0;
    mx = x > mx ? x : mx;
  }
  mx = warp_max_u64(mx);
  if ((threadIdx.x & 31) == 0) wt[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x < 32) {
    mx = warp_max_u64(wt[threadIdx.x]);
    if (threadIdx.x == 0) cmax[blockIdx.x] = mx;
  }
}

__global__ void __launch_bounds__(1024) pmb_scan_kernel(uint64_t* __restrict__ pmb, uint64_t nb,
                                                        const uint64_t* __restrict__ cmax) {
  __shared__ uint64_t wt[33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t c0 = (uint64_t)blockIdx.x * kPmChunk;
  constexpr int E = kPmChunk / 1024;  // 8 consecutive blocks per thread
  const uint64_t b0 = c0 + (uint64_t)threadIdx.x * E;
  uint64_t v[E];
#pragma unroll
  for (int k = 0; k < E; ++k) v[k] = b0 + k < nb ? pmb[b0 + k] : 0;
  uint64_t pre = 0;  // maximum of the chunks before this one
  if (warp == 0) {
    for (uint32_t c = lane; c < blockIdx.x; c += 32) pre = cmax[c] > pre ? cmax[c] : pre;
    pre = warp_max_u64(pre);
    if (lane == 0) wt[32] = pre;
  }
  uint64_t mx = 0;
#pragma unroll
  for (int k = 0; k < E; ++k) mx = v[k] > mx ? v[k] : mx;
  uint64_t inc = mx;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t w = __shfl_up_sync(kFull, inc, o);
    if (lane >= o && w > inc) inc = w;
  }
  uint64_t excl = __shfl_up_sync(kFull, inc, 1);
  if (lane == 0) excl = 0;
  if (lane == 31) wt[warp] = inc;
  __syncthreads();
  excl = wt[32] > excl ? wt[32] : excl;
  for (int w = 0; w < warp; ++w) excl = wt[w] > excl ? wt[w] : excl;
#pragma unroll
  for (int k = 0; k < E; ++k) {
    if (b0 + k < nb) pmb[b0 + k] = excl;
    excl = v[k] > excl ? v[k] : excl;
  }
}

// Other dimensions of the subscriptions, gathered into Slo order (d > 1):
// out[(k-1)*2*n + 0*n + i] = lo_k[idx[i]], out[(k-1)*2*n + n + i] = hi_k[idx[i]].
struct DimPtrs {
  const double* lo[8];
  const double* hi[8];
};

__global__ void __launch_bounds__(256) gather_dims_kernel(const uint32_t* __restrict__ idx, const __grid_constant__ DimPtrs src,
                                                          int d, uint64_t n, double* __restrict__ out,
                                                          const uint32_t* __restrict__ abort_flag) {
  if (abort_flag && *abort_flag) return;  // MSD bucket overflow: idx is not a permutation, attempt discarded
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

// lower bound of x in a[0..n) knowing a[start-1] < x: exponential probe.
__device__ __forceinline__ uint64_t gallop_lb(const uint64_t* __restrict__ a, uint64_t n, uint64_t start,
                                              uint64_t x) {
  uint64_t lo = start, hi = n, step = 1;
  while (true) {
    const uint64_t probe = lo + step - 1;
    if (probe >= n) break;
    if (a[probe] >= x) { hi = probe; break; }
    lo = probe + 1;
    step <<= 1;
  }
  return lb(a, lo, hi, x);
}

// ------------------------------------------------------------ decoupled look-back scan

constexpr uint64_t kScanAgg = 1ull << 62;
constexpr uint64_t kScanPre = 2ull << 62;
constexpr uint64_t kScanVal = (1ull << 62) - 1;

// Decoupled look-back by one whole warp: 32 predecessors are examined per
// step (lane k reads tile - 1 - k), so the walk over tiles that have
// published only their aggregate costs one round trip per 32 tiles.
// Call with all 32 lanes of one warp; returns the exclusive prefix.
__device__ __forceinline__ uint64_t lookback_warp_u64(uint64_t* status, uint32_t tile, uint64_t agg) {
  const int lane = threadIdx.x & 31;
  if (tile == 0) {
    if (lane == 0) st_relaxed_u64(status, kScanPre | agg);
    return 0;
  }
  if (lane == 0) st_relaxed_u64(status + tile, kScanAgg | agg);
  uint64_t excl = 0;
  int64_t base = (int64_t)tile - 1;
  while (true) {
    const int64_t p = base - lane;
    const uint64_t s = p >= 0 ? ld_relaxed_u64(status + p) : kScanPre;
    const unsigned pre = __ballot_sync(kFull, (s & kScanPre) != 0);
    const unsigned unpub = __ballot_sync(kFull, (s & ~kScanVal) == 0);
    const int first = pre ? __ffs(pre) - 1 : 31;
    const unsigned need = first == 31 ? kFull : ((2u << first) - 1u);
    if (unpub & need) {  // some needed predecessor not published yet: back off
      __nanosleep(64);
      continue;
    }
    excl += warp_sum<uint64_t>(lane <= first && p >= 0 ? (s & kScanVal) : 0);
    if (pre) break;
    base -= 32;
  }
  if (lane == 0) st_relaxed_u64(status + tile, kScanPre | (excl + agg));
  return excl;
}

#ifndef DDM_ADV_BF
#define DDM_ADV_BF 1
#endif
constexpr int kCountThreads = 512;
constexpr int kCountItems = 4;  // rows per thread (short dependent merge chains, more warps)
constexpr int kCountTile = kCountThreads * kCountItems;
#ifndef DDM_COUNT_WIN
#define DDM_COUNT_WIN 2560
#endif
#ifndef DDM_COUNT_EXT
#define DDM_COUNT_EXT 256
#endif
constexpr int kCountWin = DDM_COUNT_WIN;  // smem window (keys) per sorted array
constexpr int kCountExt = DDM_COUNT_EXT;  // Slo window extension past r_lo(a_last) for the r_b searches
constexpr int kRowTile = 256;    // rows per emit CTA == granularity of the row-offset scan
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

static_assert(kCountTile % kRowTile == 0, "count tile holds whole row tiles");

// Rank of x in the sorted a[0, n) by one group of 8 lanes (lanes 8g .. 8g+7
// of the warp, g = lane / 8): #{a[i] <= x} (upper) or #{a[i] < x}.  An 8-ary
// search: the 8 lanes probe 8 evenly spaced positions of the current interval
// and the group's ballot narrows it ~9x per step (log9 n dependent rounds
// instead of log2 n -- these searches run on latency, with L2 flushed between
// small calls every round trip is a DRAM miss).  All 32 lanes must call it.
__device__ __forceinline__ uint64_t group8_rank(const uint64_t* __restrict__ a, uint64_t n, uint64_t x, bool upper,
                                                int lane) {
  const int g = lane & 7, sh = lane & ~7;
  uint64_t lo = 0, hi = n;  // the rank lies in [lo, hi]
  while (__any_sync(kFull, hi - lo > 8)) {
    const bool act = hi - lo > 8;
    const uint64_t p = lo + ((uint64_t)(g + 1) * (hi - lo)) / 9;
    const bool pr = act && (upper ? a[p] <= x : a[p] < x);
    const uint32_t c = __popc((__ballot_sync(kFull, pr) >> sh) & 0xffu);  // probes with rank > p
    if (act) {
      const uint64_t plo = c ? lo + ((uint64_t)c * (hi - lo)) / 9 + 1 : lo;
      const uint64_t phi = c < 8 ? lo + ((uint64_t)(c + 1) * (hi - lo)) / 9 : hi;
      lo = plo;
      hi = phi;
    }
  }
  const uint64_t p = lo + g;
  const bool pr = p < hi && (upper ? a[p] <= x : a[p] < x);
  return lo + __popc((__ballot_sync(kFull, pr) >> sh) & 0xffu);
}

// Per count tile: r_lo(a_first), r_lo(a_last), r_hi(a_first), r_hi(a_last)
// (merge-path partition of the sorted updates against Slo and Shi).
// Few tiles (small calls, latency-bound): one warp per tile, the four
// searches side by side in groups of 8 lanes (count_partition_kernel);
// many tiles: one thread per tile, binary searches (count_partition1_kernel,
// fewer loads in total: c3 25 vs 33 us).
constexpr uint64_t kPartWarpMaxTiles = 2048;
__global__ void __launch_bounds__(256) count_partition1_kernel(const uint64_t* __restrict__ ulo_key, uint64_t m,
                                                               const uint64_t* __restrict__ slo_key,
                                                               const uint64_t* __restrict__ shi_key, uint64_t n,
                                                               uint64_t* __restrict__ part) {
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t tiles = (m + kCountTile - 1) / kCountTile;
  if (t >= tiles) return;
  const uint64_t j0 = t * kCountTile, j1 = umin64(m, j0 + kCountTile) - 1;
  const uint64_t af = ulo_key[j0], al = ulo_key[j1];
  part[4 * t + 0] = ub(slo_key, 0, n, af);
  part[4 * t + 1] = ub(slo_key, 0, n, al);
  part[4 * t + 2] = shi_key ? lb(shi_key, 0, n, af) : 0;  // (walk form: no Shi)
  part[4 * t + 3] = shi_key ? lb(shi_key, 0, n, al) : 0;
}
__global__ void __launch_bounds__(256) count_partition_kernel(const uint64_t* __restrict__ ulo_key, uint64_t m,
                                                              const uint64_t* __restrict__ slo_key,
                                                              const uint64_t* __restrict__ shi_key, uint64_t n,
                                                              uint64_t* __restrict__ part) {
  const uint64_t t = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31, q = lane >> 3;
  const uint64_t tiles = (m + kCountTile - 1) / kCountTile;
  if (t >= tiles) return;  // (warp-uniform)
  const uint64_t j0 = t * kCountTile, j1 = umin64(m, j0 + kCountTile) - 1;
  const uint64_t x = ulo_key[(q & 1) ? j1 : j0];
  // groups 0, 1: ub(Slo, a_first / a_last); 2, 3: lb(Shi, ...) (0 without Shi: walk form)
  const bool up = q < 2;
  const uint64_t r = group8_rank(up || !shi_key ? slo_key : shi_key, up || shi_key ? n : 0, x, up, lane);
  if ((lane & 7) == 0) part[4 * t + q] = r;
}

constexpr int kWalkPad = 256;  // walk form: slo_hi / pmw windows start this far before r_lo(a_first)
struct CountSmem {
  uint64_t bar;
  uint64_t pad_;
  uint64_t pbw[8];                   // walk form: pmb of the 1024-blocks the windows touch
  uint64_t tsum[kCountTile / kRowTile];  // per 256-row tile count sums
  alignas(16) uint64_t ws[kCountWin + 2];  // Slo window; +2: the bulk copies start at an even (16-byte) index
  alignas(16) uint64_t wh[kCountWin + 2];  // Shi window (rank form) / slo_hi window (walk form)
  alignas(16) uint64_t wp[kCountWin + 2];  // pmw window (walk form only)
};
// dynamic shared memory of count_kernel<WALK>
constexpr size_t count_smem_bytes(bool walk) { return walk ? sizeof(CountSmem) : offsetof(CountSmem, wp); }

// First window position at or after k whose entry is "after" x (> x for
// UPPER, >= x otherwise), given every entry before k is not: gallop forward
// from the cursor (1, 2, 4, ... steps), then binary search the last gap; len
// when the window holds no such entry.  Cursors of consecutive sorted
// queries move by a few positions, so this is O(1) probes per query.
template <bool UPPER>
__device__ __forceinline__ uint32_t wseek(const uint64_t* W, uint32_t k, uint32_t len, uint64_t x) {
  uint32_t lo = k, hi = len, step = 1;
  while (lo < len) {
    const uint32_t probe = min(lo + step - 1, len - 1);
    const uint64_t v = W[probe];
    if (UPPER ? v > x : v >= x) { hi = probe; break; }
    lo = probe + 1;
    step <<= 1;
  }
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    const uint64_t v = W[mid];
    if (UPPER ? v > x : v >= x) hi = mid;
    else lo = mid + 1;
  }
  return lo;
}

// First index of the sorted window W[0, len) whose key is > x (len if none),
// starting from an interpolated guess and galloping towards the answer: the
// first row of a count thread lands within a few entries of its guess on
// near-uniform keys (a plain binary search over the window took 12 steps).
__device__ __forceinline__ uint32_t ub_interp(const uint64_t* W, uint32_t len, uint64_t x) {
  if (len == 0) return 0;
  const uint64_t w0 = W[0], w1 = W[len - 1];
  if (x < w0) return 0;
  if (x >= w1) return len;
  uint32_t g = (uint32_t)((double)(x - w0) / (double)(w1 - w0) * (double)(len - 1));
  g = min(g, len - 1);
  uint32_t lo, hi;  // the answer lies in [lo, hi]
  if (W[g] <= x) {
    lo = g + 1;
    for (uint32_t step = 1;; step <<= 1) {
      const uint32_t p = lo + step - 1;
      if (p >= len) { hi = len; break; }
      if (W[p] > x) { hi = p; break; }
      lo = p + 1;
    }
  } else {
    hi = g;
    for (uint32_t step = 1;; step <<= 1) {
      if (hi < step) { lo = 0; break; }
      const uint32_t p = hi - step;
      if (W[p] <= x) { lo = p + 1; break; }
      hi = p;
    }
  }
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (W[mid] > x) hi = mid;
    else lo = mid + 1;
  }
  return lo;
}

// Advance a merge cursor: pos is an absolute index into the sorted array g
// with every entry before pos "before" x; returns the first index whose entry
// is "after" x.  The slice [base, base+len) is staged in W (shared memory);
// past it (rare) a gallop in global memory.
template <bool UPPER>
__device__ __forceinline__ uint64_t advance(const uint64_t* W, uint64_t base, uint32_t len, const uint64_t* g,
                                            uint64_t n, uint64_t pos, uint64_t x) {
  uint32_t k = pos >= base ? (uint32_t)umin64(pos - base, len) : 0;
  // cursors of consecutive sorted queries usually move by 0..2 entries: a
  // short linear scan first, the gallop only for longer moves
  uint32_t r = len;
#if DDM_ADV_BF
  if (k + 3 <= len) {  // branch-free: W is sorted, so the entries "before" x among the next 3 are a prefix
    const uint64_t v0 = W[k], v1 = W[k + 1], v2 = W[k + 2];
    const uint32_t c = (uint32_t)(UPPER ? v0 <= x : v0 < x) + (uint32_t)(UPPER ? v1 <= x : v1 < x) +
                       (uint32_t)(UPPER ? v2 <= x : v2 < x);
    if (c < 3) return base + k + c;
    k += 3;
  } else {
#pragma unroll
    for (int t = 0; t < 3; ++t) {
      if (k >= len) break;
      const uint64_t v = W[k];
      if (UPPER ? v > x : v >= x) { r = k; break; }
      ++k;
    }
  }
#else
#pragma unroll
  for (int t = 0; t < 3; ++t) {
    if (k >= len) break;
    const uint64_t v = W[k];
    if (UPPER ? v > x : v >= x) { r = k; break; }
    ++k;
  }
#endif
  if (r == len && k < len) r = wseek<UPPER>(W, k, len, x);
  if (r < len) return base + r;
  if (base + len >= n) return n;
  return UPPER ? ub_gallop(g, n, base + len, x) : gallop_lb(g, n, base + len, x);
}

// a4 (G5): for every update j (sorted Ulo order) r_lo = #{S.lo <= a},
// r_b = #{S.lo <= b} and cnt = |Stab(a)| + (r_b - r_lo).  b_j =
// key(upd_hi[ulo_id[j]]) is gathered here on the LSB path (a3).
//  - rank form (WALK = false; count-only calls, the paper's K-independent
//    count mode): |Stab(a)| = r_lo - r_hi with r_hi = #{S.hi < a} from the
//    sorted Shi (the rank difference of I2);
//  - walk form (WALK = true; pairs calls, whose emission is O(K) anyway):
//    |Stab(a)| counted by walking Slo backwards from r_lo - 1 until the
//    prefix maximum of slo_hi drops below a (tree_pm_kernel), skipping
//    aligned blocks whose maximum is < a -- so no Shi sort is needed.
// Each thread owns 8 consecutive updates: a binary search locates its first
// one in the tile's staged windows, then the cursors only move forward (a is
// sorted: a merge path).  Also writes the count sum of every 256-row tile
// (for the row-offset scan, a5).
struct CountWalk {  // walk form inputs
  const uint64_t* slo_hi;
  const uint64_t* pmw;
  const uint64_t* pmb;
  uint64_t nb;  // entries of pmb
  MaxTree T;
};

// One step of the counting stab walk of a row at position i (walking down):
// returns false once max(slo_hi[0..i]) < a (nothing at or before i can be a
// member), else counts i, or skips an aligned block whose maximum is < a.
// WP holds pmw over the staged slice [q0, q0 + lq) and PB the pmb of the
// blocks it touches; outside it, pmw and pmb from global memory.
__device__ __forceinline__ bool walk_step(const uint64_t* WH, const uint64_t* WP, const uint64_t* PB, uint64_t q0,
                                          uint32_t lq, const CountWalk& C, int64_t& i, uint64_t a, uint32_t& s) {
  if (i < 0) return false;
  const uint64_t u = (uint64_t)i;
  const bool in = u - q0 < lq;  // (wraps for u < q0)
  uint64_t p, h;
  if (in) {
    p = WP[u - q0];
    const uint64_t pb = PB[(u >> 10) - (q0 >> 10)];
    p = pb > p ? pb : p;
    h = WH[u - q0];
  } else {
    p = __ldg(C.pmw + u);
    const uint64_t pb = __ldg(C.pmb + (u >> 10));
    p = pb > p ? pb : p;
    h = __ldg(C.slo_hi + u);
  }
  if (p < a) return false;
  if (h >= a) ++s;
  else if (((u + 1) & 31) == 0) {  // (a member's own block cannot be skipped)
    const int L = skip_levels(C.T, i, a);
    if (L) { i -= (int64_t)1 << (5 * L); return true; }
  }
  --i;
  return true;
}

template <bool WALK>
#ifndef DDM_COUNT_MINB
#define DDM_COUNT_MINB 3
#endif
__global__ void __launch_bounds__(kCountThreads, DDM_COUNT_MINB) count_kernel(
    const uint64_t* __restrict__ ulo_key, const uint32_t* __restrict__ ulo_id, const double* __restrict__ upd_hi,
    const uint64_t* __restrict__ uhi, uint64_t m, const uint64_t* __restrict__ slo_key, const uint64_t* __restrict__ shi_key, uint64_t n,
    const uint64_t* __restrict__ part, uint32_t* __restrict__ r_lo_out, uint32_t* __restrict__ r_b_out,
    uint32_t* __restrict__ cnt_out, uint64_t* __restrict__ row_tile_sum, const __grid_constant__ CountWalk C) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  CountSmem& S = *reinterpret_cast<CountSmem*>(smem_raw);  // wp unused by the rank form
  const int tid = threadIdx.x;
  const uint32_t tile = blockIdx.x;
  const uint64_t j0 = (uint64_t)tile * kCountTile;
  const uint64_t jn = umin64(kCountTile, m - j0);
  const uint64_t p0 = part[4 * tile + 0], p1 = part[4 * tile + 1], h0 = part[4 * tile + 2], h1 = part[4 * tile + 3];
  const uint64_t t0 = (uint64_t)tid * kCountItems;
  const int ni = t0 < jn ? (int)umin64(kCountItems, jn - t0) : 0;
  const uint64_t j = j0 + t0;
  // issue this thread's loads first (the random upd_hi gather overlaps the
  // window staging below)
  uint64_t a[kCountItems], b[kCountItems];
  if (uhi && ni == kCountItems) {  // upper keys already in sorted order (MSD sort payload)
    // 16-byte loads through L1: a thread's 8 consecutive keys share lines with
    // its neighbours', so later loads hit L1 instead of refetching from L2
    const ulonglong2* pa = reinterpret_cast<const ulonglong2*>(ulo_key + j);
    const ulonglong2* pb = reinterpret_cast<const ulonglong2*>(uhi + j);
#pragma unroll
    for (int i = 0; i < kCountItems / 2; ++i) {
      const ulonglong2 va = __ldg(pa + i), vb = __ldg(pb + i);
      a[2 * i] = va.x; a[2 * i + 1] = va.y;
      b[2 * i] = vb.x; b[2 * i + 1] = vb.y;
    }
  } else if (uhi) {
#pragma unroll
    for (int i = 0; i < kCountItems; ++i) {
      a[i] = i < ni ? __ldg(ulo_key + j + i) : 0;
      b[i] = i < ni ? __ldg(uhi + j + i) : 0;
    }
  } else {  // gather them (LSB sort path)
    uint32_t id[kCountItems];
#pragma unroll
    for (int i = 0; i < kCountItems; ++i) id[i] = i < ni ? __ldcs(ulo_id + j + i) : 0;
    double hv[kCountItems];
#pragma unroll
    for (int i = 0; i < kCountItems; ++i) hv[i] = i < ni ? upd_hi[id[i]] : 0.0;
#pragma unroll
    for (int i = 0; i < kCountItems; ++i) a[i] = i < ni ? __ldcs(ulo_key + j + i) : 0;
#pragma unroll
    for (int i = 0; i < kCountItems; ++i) b[i] = f64_key(hv[i]);
  }
  const uint32_t ls = (uint32_t)umin64(umin64(kCountWin, p1 - p0 + kCountExt), n - p0);
  // rank form: the Shi window from r_hi(a_first); walk form: the slo_hi and
  // pmw windows from kWalkPad entries before r_lo(a_first)
  const uint64_t q0 = WALK ? (p0 > kWalkPad ? p0 - kWalkPad : 0) : h0;
  const uint32_t lh = WALK ? (uint32_t)umin64(kCountWin, n - q0)
                           : (uint32_t)umin64(kCountWin, umin64(h1 - h0 + 1, n - h0));
  // the windows arrive by bulk async copies (TMA engine) from 16-byte
  // aligned starts, tracked by one mbarrier; the threads' own loads of a and
  // b above are in flight meanwhile.  Reading up to one key past the array is
  // safe: every sorted key array is followed by another workspace array.
  const uint32_t os = (uint32_t)(p0 & 1), oh = (uint32_t)(q0 & 1);
  const uint64_t* W0 = S.ws + os;
  const uint64_t* H0 = S.wh + oh;
  const uint64_t* P0 = S.wp + oh;
  if (tid < kCountTile / kRowTile) S.tsum[tid] = 0;
  if (WALK && tid < 8) {
    const uint64_t bb = (q0 >> 10) + tid;
    if (bb < C.nb) S.pbw[tid] = __ldg(C.pmb + bb);
  }
  if (tid == 0) {
    mbar_init(&S.bar, 1);
    const uint32_t bs = ((ls + os + 1) & ~1u) * 8, bh = ((lh + oh + 1) & ~1u) * 8;
    mbar_expect_tx(&S.bar, bs + (WALK ? 2 : 1) * bh);
    if (bs) bulk_g2s(S.ws, slo_key + (p0 - os), bs, &S.bar);
    if (bh) bulk_g2s(S.wh, (WALK ? C.slo_hi : shi_key) + (q0 - oh), bh, &S.bar);
    if (WALK && bh) bulk_g2s(S.wp, C.pmw + (q0 - oh), bh, &S.bar);
  }
  __syncthreads();  // the barrier is initialised before anyone waits on it
  mbar_wait(&S.bar, 0);

  uint32_t cnt[kCountItems];
#pragma unroll
  for (int i = 0; i < kCountItems; ++i) cnt[i] = 0;
  if (ni > 0) {
    // first update: binary search inside the windows (falls back to global)
    uint64_t rl = advance<true>(W0, p0, ls, slo_key, n, p0 + ub_interp(W0, ls, a[0]), a[0]);
    uint64_t rh = 0;
    if (!WALK)
      rh = advance<false>(H0, h0, lh, shi_key, n, h0 + ((lh && H0[lh - 1] >= a[0]) ? lb(H0, 0, lh, a[0]) : lh), a[0]);
    uint64_t rb = rl;
    uint32_t ol[kCountItems], ob[kCountItems];
#pragma unroll
    for (int i = 0; i < kCountItems; ++i) {
      if (i < ni) {
        if (i) {
          rl = advance<true>(W0, p0, ls, slo_key, n, rl, a[i]);
          if (!WALK) rh = advance<false>(H0, h0, lh, shi_key, n, rh, a[i]);
        }
        const uint64_t start = (i && b[i] >= b[i - 1] && rb > rl) ? rb : rl;
        rb = advance<true>(W0, p0, ls, slo_key, n, start, b[i]);
        ol[i] = (uint32_t)rl;
        ob[i] = (uint32_t)rb;
        if (WALK) cnt[i] = (uint32_t)(rb - rl);
        else cnt[i] = (uint32_t)(rb > rh ? rb - rh : 0);
      }
    }
    if (WALK) {  // the rows' stab walks, interleaved (independent loads in flight)
      int64_t pos[kCountItems];
      unsigned act = 0;
#pragma unroll
      for (int i = 0; i < kCountItems; ++i) {
        pos[i] = (int64_t)ol[i] - 1;
        if (i < ni) act |= 1u << i;
      }
      while (act) {
#pragma unroll
        for (int i = 0; i < kCountItems; ++i)
          if ((act >> i) & 1u)
            if (!walk_step(H0, P0, S.pbw, q0, lh, C, pos[i], a[i], cnt[i])) act &= ~(1u << i);
      }
    }
    if (!r_lo_out) {
      // (count-only call: the tile sums below are all that is needed)
    } else if (ni == kCountItems) {
      uint4* dl = reinterpret_cast<uint4*>(r_lo_out + j);
      uint4* db = reinterpret_cast<uint4*>(r_b_out + j);
      uint4* dc = reinterpret_cast<uint4*>(cnt_out + j);
#pragma unroll
      for (int h = 0; h < kCountItems / 4; ++h) {
        dl[h] = make_uint4(ol[4 * h], ol[4 * h + 1], ol[4 * h + 2], ol[4 * h + 3]);
        db[h] = make_uint4(ob[4 * h], ob[4 * h + 1], ob[4 * h + 2], ob[4 * h + 3]);
        dc[h] = make_uint4(cnt[4 * h], cnt[4 * h + 1], cnt[4 * h + 2], cnt[4 * h + 3]);
      }
    } else {
#pragma unroll
      for (int i = 0; i < kCountItems; ++i)
        if (i < ni) { r_lo_out[j + i] = ol[i]; r_b_out[j + i] = ob[i]; cnt_out[j + i] = cnt[i]; }
    }
  }
  // per 256-row tile sums (a row tile = kRowTile / kCountItems consecutive threads)
  uint64_t local = 0;
#pragma unroll
  for (int i = 0; i < kCountItems; ++i) local += cnt[i];
  local = warp_sum<uint64_t>(local);
  if ((tid & 31) == 0) atomicAdd((unsigned long long*)&S.tsum[(tid * kCountItems) / kRowTile], (unsigned long long)local);
  __syncthreads();
  if (tid < kCountTile / kRowTile) {
    const uint64_t rt = j0 + (uint64_t)tid * kRowTile;
    if (rt < m) row_tile_sum[rt / kRowTile] = S.tsum[tid];
  }
}

// Sum of the counts of each 256-row tile (used after the d > 1 count pass).
__global__ void __launch_bounds__(kRowTile) row_tile_sum_kernel(const uint32_t* __restrict__ cnt, uint64_t m,
                                                                uint64_t* __restrict__ row_tile_sum) {
  __shared__ uint64_t tmp[kRowTile / 32 + 1];
  const uint64_t j = (uint64_t)blockIdx.x * kRowTile + threadIdx.x;
  uint64_t total;
  block_excl_scan<kRowTile>((uint64_t)(j < m ? cnt[j] : 0), tmp, &total);
  if (threadIdx.x == 0) row_tile_sum[blockIdx.x] = total;
}

// a5: exclusive scan of the row-tile sums (T = ceil(m/256) values) -> the
// output offset of each tile's first row; total K.  One CTA per 4096 sums,
// chained by decoupled look-back (a few CTAs even at m = 1e9).
// status: gridDim.x + 1 zeroed words; the last one is the tile counter: a CTA
// works on the tile it claims from it, not on blockIdx.x, so every tile whose
// predecessors it waits on was claimed (is running or done) before it --
// forward progress does not depend on the order CTAs are scheduled in.
constexpr int kScanThreads = 512;
constexpr int kScanItems = 8;
__global__ void __launch_bounds__(kScanThreads) scan_u64_kernel(const uint64_t* __restrict__ in, uint64_t T,
                                                                uint64_t* __restrict__ out,
                                                                uint64_t* __restrict__ status,
                                                                uint64_t* __restrict__ k_out) {
  __shared__ uint64_t scan_tmp[kScanThreads / 32 + 1];
  __shared__ uint64_t prefix;
  __shared__ uint32_t claimed;
  const int tid = threadIdx.x;
  if (tid == 0) claimed = (uint32_t)atomicAdd((unsigned long long*)(status + gridDim.x), 1ull);
  __syncthreads();
  const uint32_t tile = claimed;
  const uint64_t base = (uint64_t)tile * kScanThreads * kScanItems + (uint64_t)tid * kScanItems;
  uint64_t v[kScanItems];
  uint64_t local = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    v[i] = base + i < T ? in[base + i] : 0;
    local += v[i];
  }
  uint64_t agg;
  const uint64_t texcl = block_excl_scan<kScanThreads>(local, scan_tmp, &agg);
  if (tid < 32) {
    const uint64_t e = lookback_warp_u64(status, tile, agg);
    if (tid == 0) prefix = e;
  }
  __syncthreads();
  uint64_t run = prefix + texcl;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    if (base + i < T) out[base + i] = run;
    run += v[i];
  }
  if (tile == gridDim.x - 1 && tid == 0 && k_out) *k_out = prefix + agg;
}

// ------------------------------------------------------------ sweep + emit (a6 + a7, a8)

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

// Output id of a subscription: its global id when a map is given (slab-
// partitioned multi-GPU matching, dist.py), else the local array index.
__device__ __forceinline__ uint32_t sub_out(const uint32_t* map, uint32_t s) { return map ? __ldg(map + s) : s; }

struct EmitArgs {
  const uint64_t* ulo_key;
  const uint32_t* ulo_id;   // local update id (index into the update arrays)
  const uint32_t* upd_map;  // optional: global id of each local update
  const uint32_t* sub_map;  // optional: global id of each local subscription
  const uint32_t* r_lo;
  const uint32_t* r_b;
  const uint32_t* cnt0;     // dim-0 candidate count per row (stab0 = cnt0 - range)
  const uint32_t* cnt;      // output pairs per row (== cnt0 for d == 1)
  const uint64_t* tile_off; // output offset of each 256-row tile
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
  uint32_t force;           // 0 auto, 1 thread, 2 warp, 3 chunk (staged) for every tile
  const uint32_t* abort_flag;  // MSD bucket overflow: the sorted arrays are not valid, do nothing
};

enum EmitMode { kEmitD1 = 0, kCountDD = 1, kEmitDD = 2 };

// Row offsets of one 256-row tile: ro[t] = tile_off + exclusive scan of cnt.
struct RowSmem {
  uint64_t ro[kRowTile + 1];
  uint64_t tmp[kRowTile / 32 + 1];
  uint32_t queue[kRowTile];
  uint32_t qn;
};

template <int MODE>
__device__ __forceinline__ void row_offsets(const EmitArgs& A, RowSmem& R, uint64_t j0) {
  const uint64_t j = j0 + threadIdx.x;
  if (MODE == kCountDD) {
    if (threadIdx.x == 0) R.qn = 0;
    __syncthreads();
    return;
  }
  uint64_t total;
  const uint64_t e = block_excl_scan<kRowTile>((uint64_t)(j < A.m ? A.cnt[j] : 0), R.tmp, &total);
  const uint64_t base = A.tile_off[j0 / kRowTile];
  R.ro[threadIdx.x] = base + e;
  if (threadIdx.x == 0) {
    R.ro[kRowTile] = base + total;
    R.qn = 0;
  }
  __syncthreads();
}

// ---- one row, one thread
template <int MODE>
__device__ __forceinline__ void row_thread(const EmitArgs& A, uint64_t j, uint64_t o) {
  const uint64_t a = A.ulo_key[j];
  const uint32_t lid = A.ulo_id[j];
  const uint32_t uid = A.upd_map ? A.upd_map[lid] : lid;
  const uint32_t rl = A.r_lo[j], rb = A.r_b[j];
  const uint32_t stab0 = A.cnt0[j] - (rb - rl);
  UpdBox q;
  if (MODE != kEmitD1)
    for (int k = 0; k < A.F.dims; ++k) { q.lo[k] = A.upd.lo[k + 1][lid]; q.hi[k] = A.upd.hi[k + 1][lid]; }
  uint32_t fst = MODE == kEmitDD ? A.fstab[j] : stab0;  // write cursor (backwards) for the stab part
  uint32_t nst = 0;                                      // filtered stab members (count pass)
  int64_t i = (int64_t)rl - 1;
  uint32_t rem = stab0;
  if (MODE == kEmitD1) {
    // 4 positions of one aligned 32-block per step, loaded together (the walk
    // is otherwise a chain of dependent global loads)
    while (rem) {
      if ((i & 31) == 31) {
        const int L = skip_levels(A.T, i, a);
        if (L) { i -= (int64_t)1 << (5 * L); continue; }
      }
      const int c = (int)min((int64_t)4, (i & 31) + 1);
      uint64_t h[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) h[u] = u < c ? A.T.lvl[0][i - u] : 0;
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (u < c && rem && h[u] >= a) {
          --rem;
          A.pairs[o + rem] = make_uint2(sub_out(A.sub_map, A.slo_id[i - u]), uid);
        }
      i -= c;
    }
  }
  while (rem) {
    if ((i & 31) == 31) {
      const int L = skip_levels(A.T, i, a);
      if (L) { i -= (int64_t)1 << (5 * L); continue; }
    }
    if (A.T.lvl[0][i] >= a) {
      --rem;
      if (MODE == kEmitD1) {
        A.pairs[o + rem] = make_uint2(sub_out(A.sub_map, A.slo_id[i]), uid);
      } else if (box_ok(A.F, q, (uint64_t)i)) {
        if (MODE == kCountDD) ++nst;
        else A.pairs[o + (--fst)] = make_uint2(sub_out(A.sub_map, A.slo_id[i]), uid);
      }
    }
    --i;
  }
  if (MODE == kEmitD1) {
    for (uint32_t k = rl; k < rb; ++k) A.pairs[o + stab0 + (k - rl)] = make_uint2(sub_out(A.sub_map, A.slo_id[k]), uid);
  } else {
    const uint32_t base = MODE == kEmitDD ? A.fstab[j] : 0;
    uint32_t w = 0;
    for (uint32_t k = rl; k < rb; ++k) {
      if (box_ok(A.F, q, k)) {
        if (MODE == kEmitDD) A.pairs[o + base + w] = make_uint2(sub_out(A.sub_map, A.slo_id[k]), uid);
        ++w;
      }
    }
    if (MODE == kCountDD) { A.cnt_out[j] = nst + w; A.fstab_out[j] = nst; }
  }
}

// ---- one row, one warp (coalesced 32-wide windows, ballot/popc compaction)
template <int MODE>
__device__ __forceinline__ void row_warp(const EmitArgs& A, uint64_t j, uint64_t o, int lane) {
  const uint64_t a = A.ulo_key[j];
  const uint32_t lid = A.ulo_id[j];
  const uint32_t uid = A.upd_map ? A.upd_map[lid] : lid;
  const uint32_t rl = A.r_lo[j], rb = A.r_b[j];
  const uint32_t stab0 = A.cnt0[j] - (rb - rl);
  UpdBox q;
  if (MODE != kEmitD1)
    for (int k = 0; k < A.F.dims; ++k) { q.lo[k] = A.upd.lo[k + 1][lid]; q.hi[k] = A.upd.hi[k + 1][lid]; }
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
      if (member) A.pairs[o + rem + __popc(mm & lanemask_lt())] = make_uint2(sub_out(A.sub_map, A.slo_id[idx]), uid);
    } else {
      const bool keep = member && box_ok(A.F, q, (uint64_t)idx);
      const unsigned km = __ballot_sync(kFull, keep);
      if (MODE == kCountDD) nst += __popc(km);
      else {
        fst -= __popc(km);
        if (keep) A.pairs[o + fst + __popc(km & lanemask_lt())] = make_uint2(sub_out(A.sub_map, A.slo_id[idx]), uid);
      }
    }
    hi_excl = base;
  }
  if (MODE == kEmitD1) {
    for (uint64_t k = (uint64_t)rl + lane; k < rb; k += 32)
      A.pairs[o + stab0 + (k - rl)] = make_uint2(sub_out(A.sub_map, A.slo_id[k]), uid);
  } else {
    uint32_t w = MODE == kEmitDD ? A.fstab[j] : 0;
    for (uint64_t k0 = rl; k0 < rb; k0 += 32) {
      const uint64_t k = k0 + lane;
      const bool keep = k < rb && box_ok(A.F, q, k);
      const unsigned km = __ballot_sync(kFull, keep);
      if (MODE == kEmitDD && keep) A.pairs[o + w + __popc(km & lanemask_lt())] = make_uint2(sub_out(A.sub_map, A.slo_id[k]), uid);
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
__global__ void __launch_bounds__(kRowTile) emit_kernel(const __grid_constant__ EmitArgs A) {
  if (A.abort_flag && *A.abort_flag) return;  // (the pre-sync d > 1 count runs before the host sees it)
  __shared__ RowSmem R;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint64_t j0 = (uint64_t)blockIdx.x * kRowTile;
  row_offsets<MODE>(A, R, j0);
  const uint64_t j = j0 + tid;
  if (j < A.m) {
    const uint32_t c0 = A.cnt0[j];
    const bool thread_row = A.force == 1 || (A.force == 0 && c0 <= A.thread_row_max);
    if (thread_row) row_thread<MODE>(A, j, MODE == kCountDD ? 0 : R.ro[tid]);
    else if (c0) R.queue[atomicAdd(&R.qn, 1u)] = tid;
  }
  __syncthreads();
  const uint32_t nq = R.qn;
  for (uint32_t q = warp; q < nq; q += kRowTile / 32) {
    const uint32_t t = R.queue[q];
    row_warp<MODE>(A, j0 + t, MODE == kCountDD ? 0 : R.ro[t], lane);
  }
}

// ------------------------------------------------------------ tiled sparse emit (a7, d = 1)
//
// Sparse outputs (a few pairs per row, alpha ~ 1): the per-row walks of
// emit_kernel are chains of dependent global loads.  Here a CTA takes 2048
// consecutive rows (8 per thread, the count pass's tiling), the Slo window
// their stab and range parts live in -- [r_lo(first) - kEmitPad, max r_b) --
// arrives by bulk async copies (upper keys and ids), and every thread walks
// its rows inside shared memory; positions outside the window (long
// intervals) fall back to global memory with the block-max skips.  Row
// offsets: each warp's 256 rows are one offset-scan tile.  Output identical
// to the other d = 1 paths.
#ifndef DDM_EMIT_ITEMS
#define DDM_EMIT_ITEMS 8
#endif
constexpr int kEmitItems = DDM_EMIT_ITEMS;                 // rows per thread
constexpr int kEmitThreads = 2048 / kEmitItems;            // 2048-row tiles
constexpr int kEmitTile = kEmitThreads * kEmitItems;
constexpr int kEmitWarpsPerRowTile = kRowTile / (32 * kEmitItems);  // warps sharing one 256-row offset tile
constexpr int kEmitWin = 4096;                     // window entries
constexpr int kEmitPad = 512;                      // window entries before r_lo(first row)

struct EmitTileSmem {
  alignas(16) uint64_t wh[kEmitWin + 2];
  alignas(16) uint32_t wi[kEmitWin + 4];
  uint64_t bar;
  uint32_t rbmax;
  uint64_t wsum[32];
};

#ifndef DDM_EMIT_MINB
#define DDM_EMIT_MINB 3
#endif
__global__ void __launch_bounds__(kEmitThreads, DDM_EMIT_MINB) emit_tile_kernel(const __grid_constant__ EmitArgs A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  EmitTileSmem& S = *reinterpret_cast<EmitTileSmem*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint64_t j0 = (uint64_t)blockIdx.x * kEmitTile;
  const uint64_t jt = j0 + (uint64_t)tid * kEmitItems;  // this thread's first row
  const int ni = jt < A.m ? (int)umin64(kEmitItems, A.m - jt) : 0;
  uint32_t rl[kEmitItems], rb[kEmitItems], c0[kEmitItems];
  if (ni == kEmitItems) {
    const uint4* pl = reinterpret_cast<const uint4*>(A.r_lo + jt);
    const uint4* pb = reinterpret_cast<const uint4*>(A.r_b + jt);
    const uint4* pc = reinterpret_cast<const uint4*>(A.cnt0 + jt);
#pragma unroll
    for (int h = 0; h < kEmitItems / 4; ++h) {
      const uint4 x = __ldg(pl + h), y = __ldg(pb + h), z = __ldg(pc + h);
      rl[4 * h] = x.x; rl[4 * h + 1] = x.y; rl[4 * h + 2] = x.z; rl[4 * h + 3] = x.w;
      rb[4 * h] = y.x; rb[4 * h + 1] = y.y; rb[4 * h + 2] = y.z; rb[4 * h + 3] = y.w;
      c0[4 * h] = z.x; c0[4 * h + 1] = z.y; c0[4 * h + 2] = z.z; c0[4 * h + 3] = z.w;
    }
  } else {
#pragma unroll
    for (int i = 0; i < kEmitItems; ++i) {
      rl[i] = i < ni ? A.r_lo[jt + i] : 0;
      rb[i] = i < ni ? A.r_b[jt + i] : 0;
      c0[i] = i < ni ? A.cnt0[jt + i] : 0;
    }
  }
  // window [w0, w0 + wlen) of Slo positions, staged by bulk copies
  uint32_t mx = 0;
#pragma unroll
  for (int i = 0; i < kEmitItems; ++i) mx = i < ni && rb[i] > mx ? rb[i] : mx;
  mx = __reduce_max_sync(kFull, mx);
  if (tid == 0) S.rbmax = 0;
  __syncthreads();
  if (lane == 0) atomicMax(&S.rbmax, mx);
  __syncthreads();
  const uint64_t rl_first = A.r_lo[j0];
  const uint64_t w0 = rl_first > (uint64_t)kEmitPad ? rl_first - kEmitPad : 0;
  const uint64_t wend = S.rbmax > w0 ? (uint64_t)S.rbmax : w0;
  const uint32_t wlen = (uint32_t)umin64(kEmitWin, wend - w0);
  const uint32_t oh = (uint32_t)(w0 & 1), oi = (uint32_t)(w0 & 3);
  const uint64_t* WH = S.wh + oh;
  const uint32_t* WI = S.wi + oi;
  if (tid == 0) {
    mbar_init(&S.bar, 1);
    const uint32_t bh = ((wlen + oh + 1) & ~1u) * 8, bi = ((wlen + oi + 3) & ~3u) * 4;
    mbar_expect_tx(&S.bar, bh + bi);
    if (wlen) {
      bulk_g2s(S.wh, A.T.lvl[0] + (w0 - oh), bh, &S.bar);
      bulk_g2s(S.wi, A.slo_id + (w0 - oi), bi, &S.bar);
    }
  }
  // row keys / ids meanwhile
  uint64_t a[kEmitItems];
  uint32_t lid[kEmitItems];
  if (ni == kEmitItems) {
    const ulonglong2* pa = reinterpret_cast<const ulonglong2*>(A.ulo_key + jt);
    const uint4* pi = reinterpret_cast<const uint4*>(A.ulo_id + jt);
#pragma unroll
    for (int h = 0; h < kEmitItems / 2; ++h) {
      const ulonglong2 x = __ldg(pa + h);
      a[2 * h] = x.x; a[2 * h + 1] = x.y;
    }
#pragma unroll
    for (int h = 0; h < kEmitItems / 4; ++h) {
      const uint4 x = __ldg(pi + h);
      lid[4 * h] = x.x; lid[4 * h + 1] = x.y; lid[4 * h + 2] = x.z; lid[4 * h + 3] = x.w;
    }
  } else {
#pragma unroll
    for (int i = 0; i < kEmitItems; ++i) {
      a[i] = i < ni ? A.ulo_key[jt + i] : 0;
      lid[i] = i < ni ? A.ulo_id[jt + i] : 0;
    }
  }
  // row offsets: the warps of one 256-row offset tile (j0 >> 8) + w / kEmitWarpsPerRowTile
  uint64_t mine = 0;
#pragma unroll
  for (int i = 0; i < kEmitItems; ++i) mine += c0[i];
  uint64_t incl = warp_incl_scan<uint64_t>(mine);
  uint64_t wpre = 0;
  if (kEmitWarpsPerRowTile > 1) {  // sums of the earlier warps of the same row tile
    if (lane == 31) S.wsum[warp] = incl;
    __syncthreads();
    for (int v = warp - warp % kEmitWarpsPerRowTile; v < warp; ++v) wpre += S.wsum[v];
  }
  uint64_t o = (ni > 0 ? A.tile_off[(j0 >> 8) + warp / kEmitWarpsPerRowTile] : 0) + wpre + incl - mine;
  __syncthreads();  // the barrier is initialised before anyone waits on it
  mbar_wait(&S.bar, 0);
  auto hi_at = [&](uint64_t i) -> uint64_t {
    const uint64_t k = i - w0;
    return (i >= w0 && k < wlen) ? WH[k] : A.T.lvl[0][i];
  };
  auto id_at = [&](uint64_t i) -> uint32_t {
    const uint64_t k = i - w0;
    return sub_out(A.sub_map, (i >= w0 && k < wlen) ? WI[k] : A.slo_id[i]);
  };
#pragma unroll
  for (int r = 0; r < kEmitItems; ++r) {
    if (r >= ni) break;
    const uint32_t uid = A.upd_map ? A.upd_map[lid[r]] : lid[r];
    const uint32_t stab = c0[r] - (rb[r] - rl[r]);
    uint2* row = A.pairs + o;
    // stab part: walk Slo backwards from r_lo - 1, exactly `stab` members
    uint32_t rem = stab;
    int64_t i = (int64_t)rl[r] - 1;
    while (rem) {
      if ((uint64_t)i < w0 && (i & 31) == 31) {  // outside the window: block-max skips
        const int L = skip_levels(A.T, i, a[r]);
        if (L) { i -= (int64_t)1 << (5 * L); continue; }
      }
      if (hi_at((uint64_t)i) >= a[r]) row[--rem] = make_uint2(id_at((uint64_t)i), uid);
      --i;
    }
    // range part [r_lo, r_b)
    for (uint32_t k = rl[r]; k < rb[r]; ++k) row[stab + (k - rl[r])] = make_uint2(id_at(k), uid);
    o += c0[r];
  }
}

// ------------------------------------------------------------ few dense rows (d = 1)
//
// When a d = 1 output has few rows with very many pairs each (few updates
// against many subscriptions), one CTA per 256-row tile would leave the GPU
// idle.  Here a warp takes one (row, segment) task: segment s writes pairs
// [s*4096, (s+1)*4096) of the row's range part (the last one the rest),
// segment 0 also the row's stab part (the backward walk of row_warp).  The
// row's output offset is its tile's offset plus the counts of the tile's
// earlier rows.  Output is byte-identical to the other emission paths.
constexpr int kSplitSeg = 64;
constexpr uint32_t kSplitLen = 4096;

__global__ void __launch_bounds__(256) emit_split_kernel(const __grid_constant__ EmitArgs A) {
  const int lane = threadIdx.x & 31;
  const uint64_t wid = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t task = wid; task < A.m * kSplitSeg; task += nw) {
    const uint64_t j = task / kSplitSeg;
    const uint32_t s = (uint32_t)(task % kSplitSeg);
    const uint32_t rl = A.r_lo[j], rb = A.r_b[j];
    const uint32_t nr = rb - rl;
    const uint64_t seg0 = (uint64_t)s * kSplitLen;
    if (s > 0 && seg0 >= nr) continue;  // no such segment
    const uint64_t jt = j & ~(uint64_t)(kRowTile - 1);
    uint64_t pre = 0;
    for (uint64_t r = jt + lane; r < j; r += 32) pre += A.cnt[r];
    pre = warp_sum<uint64_t>(pre);
    const uint64_t o = A.tile_off[j / kRowTile] + pre;
    const uint64_t a = A.ulo_key[j];
    const uint32_t lid = A.ulo_id[j];
    const uint32_t uid = A.upd_map ? A.upd_map[lid] : lid;
    const uint32_t stab = A.cnt[j] - nr;
    if (s == 0) {  // the stab part: walk Slo backwards from r_lo - 1 (row_warp)
      int64_t hi_excl = rl;
      uint32_t rem = stab;
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
        if (member) A.pairs[o + rem + __popc(mm & lanemask_lt())] = make_uint2(sub_out(A.sub_map, A.slo_id[idx]), uid);
        hi_excl = base;
      }
    }
    const uint64_t seg_end = s == kSplitSeg - 1 ? nr : umin64(nr, seg0 + kSplitLen);
    uint2* const rng = A.pairs + o + stab;
    for (uint64_t k = seg0 + lane; k < seg_end; k += 32)
      rng[k] = make_uint2(sub_out(A.sub_map, __ldg(A.slo_id + rl + k)), uid);
  }
}

// ------------------------------------------------------------ chunked sweep (a6 + a7)
//
// One CTA per tile of kRowTile consecutive updates (sorted order), the
// GPU form of Alg. 5's segments with Alg. 6's initial set
// at the tile's first query point x_t = a_{j0}:
//   A_t = Stab(x_t) = { S : S.lo <= x_t <= S.hi }  -- the chunk-start set,
// found by one warp walking Slo backwards from r_lo(x_t) with the block-max
// skips, and known to hold exactly r_lo - r_hi members (I4).  Every stab
// member of a later row j (a_j >= x_t) is either in A_t or in the Slo slice
// [r_lo(x_t), r_lo(a_j)), and every range member is in [r_lo(a_j), r_b(a_j)),
// so the tile stages A_t and the contiguous Slo slice (ids + upper keys) in
// shared memory once and all its rows are swept from there: short rows by one
// thread, long rows by one warp (ballot/popc compaction).  Output is
// byte-identical to the per-row paths.

constexpr int kChunkSlice = 1280;
constexpr int kChunkAct = 512;

struct ChunkRow {  // one row's data, loaded once per tile (coalesced) for the warp rows
  uint64_t a;
  uint32_t rl, rb, cnt, uid;
};

struct ChunkSmem {
  uint64_t shi[kChunkSlice];
  uint64_t ahi[kChunkAct];
  uint32_t sid[kChunkSlice];
  uint32_t aid[kChunkAct];
  ChunkRow row[kRowTile];
  RowSmem R;
  uint32_t nact;
  uint32_t slen;
};

// (id, upper key) of Slo position i: from the staged slice when inside it.
__device__ __forceinline__ uint64_t c_hi(const ChunkSmem& S, const EmitArgs& A, uint64_t rl0, uint64_t i) {
  const uint64_t k = i - rl0;
  return k < S.slen ? S.shi[k] : A.T.lvl[0][i];
}
__device__ __forceinline__ uint32_t c_id(const ChunkSmem& S, const EmitArgs& A, uint64_t rl0, uint64_t i) {
  const uint64_t k = i - rl0;
  return k < S.slen ? S.sid[k] : sub_out(A.sub_map, A.slo_id[i]);
}

__device__ __forceinline__ void chunk_row_thread(const ChunkSmem& S, const EmitArgs& A, const ChunkRow& R, uint64_t o,
                                                 uint64_t rl0) {
  const uint64_t a = R.a;
  const uint32_t uid = R.uid;
  const uint64_t rl = R.rl, rb = R.rb;
  const uint32_t stab = (uint32_t)(R.cnt - (rb - rl));
  // members of A_t still alive at a (ascending Slo order)
  uint32_t w = 0;
  for (uint32_t k = 0; k < S.nact && w < stab; ++k)
    if (S.ahi[k] >= a) A.pairs[o + (w++)] = make_uint2(S.aid[k], uid);
  // the rest of the stab part lies in the slice [rl0, rl): walk it backwards
  uint32_t need = stab - w;
  for (uint64_t i = rl; need;) {
    --i;
    if (c_hi(S, A, rl0, i) >= a) A.pairs[o + w + (--need)] = make_uint2(c_id(S, A, rl0, i), uid);
  }
  for (uint64_t i = rl; i < rb; ++i) A.pairs[o + stab + (i - rl)] = make_uint2(c_id(S, A, rl0, i), uid);
}

__device__ __forceinline__ void chunk_row_warp(const ChunkSmem& S, const EmitArgs& A, const ChunkRow& R, uint64_t o,
                                               uint64_t rl0, int lane) {
  const uint64_t a = R.a;
  const uint32_t uid = R.uid;
  const uint64_t rl = R.rl, rb = R.rb;
  const uint32_t stab = (uint32_t)(R.cnt - (rb - rl));
  uint2* const row = A.pairs + o;  // this row's output
  uint32_t w = 0;
  const uint32_t nact = S.nact;
  for (uint32_t k0 = 0; k0 < nact && w < stab; k0 += 32) {
    const uint32_t k = k0 + lane;
    const bool alive = k < nact && S.ahi[k] >= a;
    const unsigned mm = __ballot_sync(kFull, alive);
    if (alive) row[w + __popc(mm & lanemask_lt())] = make_uint2(S.aid[k], uid);
    w += __popc(mm);
  }
  // the rest of the stab part lies in the slice [rl0, rl): 32-wide windows
  // walking backwards, window-relative 32-bit indices (rl - rl0 <= slen here
  // unless the row's stab walk leaves the staged slice)
  uint32_t need = stab - w;
  int32_t hi_excl = (int32_t)(rl - rl0);
  const int32_t slen = (int32_t)S.slen;
  while (need) {
    const int32_t base = hi_excl - 32;
    const int32_t k = base + lane;
    bool member = false;
    uint32_t id = 0;
    if (k >= 0) {
      if (k < slen) {
        member = S.shi[k] >= a;
        if (member) id = S.sid[k];
      } else {
        member = A.T.lvl[0][rl0 + k] >= a;
        if (member) id = sub_out(A.sub_map, A.slo_id[rl0 + k]);
      }
    }
    const unsigned mm = __ballot_sync(kFull, member);
    need -= __popc(mm);
    if (member) row[w + need + __popc(mm & lanemask_lt())] = make_uint2(id, uid);
    hi_excl = base;
  }
  // the range part [rl, rb): staged slice first, then global memory
  uint2* const rng = row + stab;
  const uint32_t nr = (uint32_t)(rb - rl);
  const uint32_t k0 = (uint32_t)(rl - rl0);
  const uint32_t in_slice = k0 < (uint32_t)slen ? min(nr, (uint32_t)slen - k0) : 0u;
  for (uint32_t t = lane; t < in_slice; t += 32) rng[t] = make_uint2(S.sid[k0 + t], uid);
  for (uint32_t t = in_slice + lane; t < nr; t += 32) rng[t] = make_uint2(sub_out(A.sub_map, A.slo_id[rl + t]), uid);
}

// a6: the chunk-start set A_t = Stab(x_t) = {i < r_lo(x_t) : slo_hi[i] >= x_t}
// (Alg. 6 SubSet[p] at a boundary placed before the tile's first update, App.
// A I6), |A_t| = nact known exactly from the counts.  One warp walks Slo
// backwards from r_lo(x_t) with block-max skips and hands every member to
// sink(pos, upper key, output id), pos = its rank in Slo order (0..nact).
template <typename Sink>
__device__ __forceinline__ void walk_chunk_start(const EmitArgs& A, int64_t rl0, uint64_t x, uint32_t nact, int lane,
                                                 Sink&& sink) {
  int64_t hi_excl = rl0;
  uint32_t rem = nact;
  while (rem) {
    const int64_t i = hi_excl - 1;
    if ((i & 31) == 31) {
      const int L = skip_levels(A.T, i, x);
      if (L) { hi_excl -= (int64_t)1 << (5 * L); continue; }
    }
    const int64_t base = i & ~31ll;
    const int64_t idx = base + lane;
    uint64_t h = 0;
    const bool member = idx < hi_excl && (h = A.T.lvl[0][idx]) >= x;
    const unsigned mm = __ballot_sync(kFull, member);
    rem -= __popc(mm);
    if (member) sink(rem + __popc(mm & lanemask_lt()), h, sub_out(A.sub_map, A.slo_id[idx]));
    hi_excl = base;
  }
}

// ddm_chunk_start_sets (exported for tests): |A_t| of every kRowTile-row tile
// of emit_chunk_kernel, then the members through the same walk.
__global__ void __launch_bounds__(256) chunk_set_sizes_kernel(const __grid_constant__ EmitArgs A, uint64_t tiles,
                                                              uint64_t* __restrict__ sizes,
                                                              uint32_t* __restrict__ first_upd) {
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= tiles) return;
  const uint64_t j0 = t * kRowTile;
  sizes[t] = A.cnt[j0] - (A.r_b[j0] - A.r_lo[j0]);
  first_upd[t] = A.upd_map ? A.upd_map[A.ulo_id[j0]] : A.ulo_id[j0];
}
__global__ void __launch_bounds__(32) chunk_set_ids_kernel(const __grid_constant__ EmitArgs A,
                                                          const uint64_t* __restrict__ off,
                                                          uint32_t* __restrict__ ids) {
  const uint64_t t = blockIdx.x, j0 = t * kRowTile;
  const uint32_t nact = (uint32_t)(off[t + 1] - off[t]);
  uint32_t* out = ids + off[t];
  walk_chunk_start(A, (int64_t)A.r_lo[j0], A.ulo_key[j0], nact, threadIdx.x & 31,
                   [&](uint32_t pos, uint64_t, uint32_t id) { out[pos] = id; });
}

__global__ void __launch_bounds__(kRowTile) emit_chunk_kernel(const __grid_constant__ EmitArgs A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  ChunkSmem& S = *reinterpret_cast<ChunkSmem*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint64_t j0 = (uint64_t)blockIdx.x * kRowTile;
  const uint64_t jn = umin64(kRowTile, A.m - j0);
  const uint64_t rl0 = A.r_lo[j0];
  // slice [rl0, rl0 + slen): covers the stab candidates of every row (up to
  // r_lo of the last row) and, when room allows, the range parts; entries past
  // the slice are read from global memory.
  const uint32_t slen = (uint32_t)umin64(kChunkSlice, A.r_b[j0 + jn - 1] - rl0);
  // a6: the chunk-start set A_t = Stab(x_t), |A_t| = stab(j0) known exactly
  const uint64_t x = A.ulo_key[j0];
  const uint32_t nact = A.cnt[j0] - (A.r_b[j0] - (uint32_t)rl0);
  row_offsets<kEmitD1>(A, S.R, j0);
  // sparse tiles (a few pairs per row) gain nothing from staging: rows go
  // straight to the per-row walks; so do tiles whose A_t exceeds smem
  const bool sparse = A.force == 0 && S.R.ro[kRowTile] - S.R.ro[0] <= 4ull * kRowTile;
  const bool fits = nact <= kChunkAct && !sparse;
  if (tid == 0) {
    S.slen = slen;
    S.nact = nact;
  }
  const uint64_t j = j0 + tid;
  ChunkRow mine{};
  if (fits && j < A.m) {  // every row's data once, coalesced (the warp rows read it from smem)
    mine.a = A.ulo_key[j];
    const uint32_t lid = A.ulo_id[j];
    mine.uid = A.upd_map ? A.upd_map[lid] : lid;
    mine.rl = A.r_lo[j];
    mine.rb = A.r_b[j];
    mine.cnt = A.cnt[j];
  }
  if (warp == 0) {
    if (fits)  // warp 0 walks Slo backwards from r_lo(x_t) with block-max skips
      walk_chunk_start(A, (int64_t)rl0, x, nact, lane, [&](uint32_t pos, uint64_t h, uint32_t id) {
        S.ahi[pos] = h;
        S.aid[pos] = id;
      });
  } else if (fits) {  // the other warps stage the Slo slice meanwhile
    for (uint32_t k = tid - 32; k < slen; k += kRowTile - 32) {
      S.shi[k] = __ldcs(A.T.lvl[0] + rl0 + k);
      S.sid[k] = sub_out(A.sub_map, __ldcs(A.slo_id + rl0 + k));
    }
  }
  if (fits && j < A.m) S.row[tid] = mine;
  __syncthreads();
  if (!fits) {  // chunk-start set too large for shared memory: per-row global walks
    if (j < A.m) {
      const uint32_t c0 = A.cnt0[j];
      if (c0 <= A.thread_row_max) row_thread<kEmitD1>(A, j, S.R.ro[tid]);
      else if (c0) S.R.queue[atomicAdd(&S.R.qn, 1u)] = tid;
    }
    __syncthreads();
    for (uint32_t q = warp; q < S.R.qn; q += kRowTile / 32)
      row_warp<kEmitD1>(A, j0 + S.R.queue[q], S.R.ro[S.R.queue[q]], lane);
    return;
  }
  if (j < A.m) {
    const uint32_t c = mine.cnt;
    if (c <= A.thread_row_max && nact <= 32) chunk_row_thread(S, A, mine, S.R.ro[tid], rl0);
    else if (c) S.R.queue[atomicAdd(&S.R.qn, 1u)] = tid;
  }
  __syncthreads();
  const uint32_t nq = S.R.qn;
  for (uint32_t q = warp; q < nq; q += kRowTile / 32) {
    const uint32_t t = S.R.queue[q];
    chunk_row_warp(S, A, S.row[t], S.R.ro[t], rl0, lane);
  }
}

// ------------------------------------------------------------ literal d > 1 (G10)
//
// The paper's literal reading of d > 1: the pair set of every
// dimension separately, intersected.  ddm_match_pairs_literal sorts each
// dimension's pairs into canonical u64 words (upd << 32) | sub and
// intersects the running result A with the next dimension's B: a word of A
// survives iff a binary search finds it in B; survivors are compacted (in
// order) by an exclusive scan of the flags.  Small inputs only: each
// per-dimension set is materialised.
__global__ void __launch_bounds__(256) intersect_flags_kernel(const uint64_t* __restrict__ A, uint64_t na,
                                                              const uint64_t* __restrict__ B, uint64_t nb,
                                                              uint64_t* __restrict__ flag) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < na; i += stride) {
    const uint64_t x = A[i];
    uint64_t lo = 0, hi = nb;
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (B[mid] < x) lo = mid + 1;
      else hi = mid;
    }
    flag[i] = lo < nb && B[lo] == x;
  }
}
__global__ void __launch_bounds__(256) compact_kernel(const uint64_t* __restrict__ A, uint64_t na,
                                                      const uint64_t* __restrict__ flag,
                                                      const uint64_t* __restrict__ off, uint64_t* __restrict__ out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < na; i += stride)
    if (flag[i]) out[off[i]] = A[i];
}

// ------------------------------------------------------------ pair canonical key

// 64-bit view of the pairs for the canonical sort: (upd << 32) | sub.
static_assert(sizeof(uint2) == 8, "pair layout");

}  // namespace match
}  // namespace ddm
