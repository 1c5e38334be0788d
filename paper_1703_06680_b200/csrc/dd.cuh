// dd.cuh -- d > 1 matching (a8): tiled dim-0 sweep + exact filter on the
// other dimensions, with an in-shared-memory bin index over dimension 1.
//
// two d-rectangles intersect iff their projections
// intersect on every dimension, so the d-dim result is the intersection of
// the d per-dimension pair sets.  Materialising those sets is infeasible at
// c4 (~2.3e11 pairs per dimension, R16); the same set is obtained by
// sweeping dimension 0 and keeping a dim-0 candidate iff Alg. 1 holds on every
// other dimension.
//
// One CTA owns a tile of T = 256*R consecutive updates in Ulo (sweep) order,
// the GPU form of an Alg. 5 segment.  Every dim-0 candidate of every row of
// the tile lies in
//   C_t = A_t  ⊔  Slo[r_lo(x_t), max_j r_b(j))
// where A_t = Stab(x_t) = {S : S.lo <= x_t <= S.hi} is the chunk-start set at
// the tile's first query x_t (Alg. 6 SubSet[p], exactly r_lo - r_hi members,
// SURVEY App. A I4/I6).  C_t is streamed through shared memory in chunks of
// kCap candidates.
//
// Filter.  Each subscription carries a float32 box on dims 0..2 with the lower
// bounds rounded down and the upper bounds rounded up (built once with the
// index); each update row gets the same widened box.  Widening only enlarges
// intervals, so a pair that overlaps exactly also overlaps in float32: the
// float test never rejects a true pair, and every pair that passes it is
// re-tested exactly (float64 coordinates / order-preserving keys, Alg. 1 on
// every dimension) before it is counted or written.
//
// Bins.  Each chunk is counting-sorted (stably, deterministically) into kBins
// bins of its float32 dim-1 lower bounds; a row only scans the bins whose
// lower bounds can pass its float test on dim 1:
//   lo1(U) <= hi1(S) <= lo1(S) + maxlen  =>  lo1(S) >= rd(lo1(U) - maxlen)
// with maxlen the chunk's largest float32 dim-1 length rounded up and a
// monotone bucketer, so [bin(rd(lo1(U) - maxlen)), bin(hi1(U))] covers them.
// Two passes run the identical enumeration: a count pass (row counts + 256-row
// tile sums for the offset scan) and an emit pass writing each row at its
// offset, so the output is deterministic.
#pragma once
#include "common.cuh"
#include "match.cuh"

namespace ddm {
namespace dd {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kBins = 128;
constexpr int kWin = 1024;  // A_t walk window (positions per step), 4 per thread
constexpr int kCap = 1024;  // candidates per shared-memory chunk
constexpr int kRounds = kCap / kThreads;
static_assert(kCap >= kWin, "a whole walk window must fit one chunk");

// ------------------------------------------------------------ index boxes

// Widened float32 boxes of the subscriptions in Slo order (dims 0..2; a
// missing dim 2 is (-inf, +inf)): box12[i] = (lo1, hi1, lo2, hi2),
// box0[i] = (lo0, hi0), lower bounds rounded down, upper bounds rounded up.
__global__ void __launch_bounds__(256) box_kernel(const uint64_t* __restrict__ slo_key,
                                                  const uint64_t* __restrict__ slo_hi,
                                                  const double* __restrict__ sdims, int d, uint64_t n,
                                                  float4* __restrict__ box12, float2* __restrict__ box0,
                                                  const uint32_t* __restrict__ abort_flag) {
  if (abort_flag && *abort_flag) return;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    box0[i] = make_float2(__double2float_rd(key_to_f64(slo_key[i])), __double2float_ru(key_to_f64(slo_hi[i])));
    float4 b;
    b.x = __double2float_rd(sdims[i]);
    b.y = __double2float_ru(sdims[n + i]);
    if (d > 2) {
      b.z = __double2float_rd(sdims[2 * n + i]);
      b.w = __double2float_ru(sdims[3 * n + i]);
    } else {
      b.z = -__int_as_float(0x7f800000);
      b.w = __int_as_float(0x7f800000);
    }
    box12[i] = b;
  }
}

// ------------------------------------------------------------ tile kernel

struct Args {
  const uint64_t* ulo_key;   // sorted update lower keys (dim 0)
  const uint32_t* ulo_id;    // local update ids in that order
  const uint32_t* upd_map;   // optional global ids
  const uint32_t* r_lo;      // dim-0 ranks (count pass a4)
  const uint32_t* r_b;
  const uint32_t* cnt0;      // dim-0 counts
  const uint64_t* slo_key;   // index: Slo keys, ids, upper keys (lvl[0]), block maxima
  const uint32_t* slo_id;
  match::DimPtrs upd;        // update coordinates, all dims
  MaxTree T;
  const double* sdims;       // [(d-1)][2][n] other dims of the subs in Slo order
  const float4* box12;       // widened float32 boxes (box_kernel)
  const float2* box0;
  uint64_t n, m;
  int d;
  const uint32_t* abort_flag;  // non-zero: an MSD bucket overflowed, inputs are not sorted -> no-op
  // count pass
  uint32_t* cnt_out;
  uint64_t* tile_sum;        // per 256-row tile
  // emit pass
  const uint32_t* cnt;
  const uint64_t* tile_off;
  uint2* pairs;
};

template <int R>
struct Smem {
  static constexpr int kRows = kThreads * R;
  float4 c12[kCap];     // chunk boxes in bin order
  float2 c0[kCap];
  uint32_t cpos[kCap];  // Slo position of each binned slot
  uint32_t fpos[kCap];  // Slo positions in fill order
  uint64_t ra[kRows];   // row exact data: lower key, upper key, offset, local id, output id
  uint64_t rb[kRows];
  uint64_t roff[kRows];
  uint32_t rlid[kRows];
  uint32_t ruid[kRows];
  uint16_t wc[kRounds * kWarps * kBins];  // per (round, warp, bin) counts -> prefixes
  uint32_t bstart[kBins + 1];
  float red[3 * kWarps];
  uint64_t scan64[kWarps + 1];
  uint32_t scan32[kWarps + 1];
  uint32_t rbmax;
};

// Monotone float bucketer over one chunk's dim-1 lower bounds.
struct Bins {
  float mn, scale;
  __device__ __forceinline__ int operator()(float x) const {
    float u = floorf((x - mn) * scale);
    u = fminf(fmaxf(u, 0.0f), (float)(kBins - 1));  // fmaxf(NaN, 0) = 0
    return (int)u;
  }
};

template <int R>
struct Rows {  // widened float32 row boxes (dims 0..2) + hit counters
  float lo0[R], hi0[R], lo1[R], hi1[R], lo2[R], hi2[R];
  uint32_t hits[R];
  bool valid[R];
};

// Exact Alg. 1 test on every dimension for the sub at Slo position p and row r.
template <int R>
__device__ __forceinline__ bool exact_hit(const Args& A, const Smem<R>& S, uint32_t p, int r) {
  if (!(A.slo_key[p] <= S.rb[r] && A.T.lvl[0][p] >= S.ra[r])) return false;  // dim 0 (keys)
  const uint32_t lid = S.rlid[r];
  for (int k = 1; k < A.d; ++k) {
    const double slo = A.sdims[(uint64_t)(k - 1) * 2 * A.n + p];
    const double shi = A.sdims[(uint64_t)(k - 1) * 2 * A.n + A.n + p];
    if (!(slo <= A.upd.hi[k][lid] && A.upd.lo[k][lid] <= shi)) return false;
  }
  return true;
}

template <int R, bool EMIT>
__device__ void process_chunk(const Args& A, Smem<R>& S, Rows<R>& rw, uint32_t fill) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // 1. float boxes of the staged candidates; chunk min/max lo1, max length
  float4 b12[kRounds];
  float2 b0[kRounds];
  float mn = __int_as_float(0x7f800000), mx = -mn, ml = 0.0f;
#pragma unroll
  for (int r = 0; r < kRounds; ++r) {
    const uint32_t s = r * kThreads + tid;
    if (s < fill) {
      const uint32_t p = S.fpos[s];
      b12[r] = A.box12[p];
      b0[r] = A.box0[p];
      mn = fminf(mn, b12[r].x);
      mx = fmaxf(mx, b12[r].x);
      ml = fmaxf(ml, __fsub_ru(b12[r].y, b12[r].x));
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    mn = fminf(mn, __shfl_xor_sync(kFull, mn, o));
    mx = fmaxf(mx, __shfl_xor_sync(kFull, mx, o));
    ml = fmaxf(ml, __shfl_xor_sync(kFull, ml, o));
  }
  if (lane == 0) { S.red[warp] = mn; S.red[kWarps + warp] = mx; S.red[2 * kWarps + warp] = ml; }
  for (int i = tid; i < kRounds * kWarps * kBins / 2; i += kThreads) reinterpret_cast<uint32_t*>(S.wc)[i] = 0;
  __syncthreads();
#pragma unroll
  for (int w = 0; w < kWarps; ++w) {
    mn = fminf(mn, S.red[w]);
    mx = fmaxf(mx, S.red[kWarps + w]);
    ml = fmaxf(ml, S.red[2 * kWarps + w]);
  }
  Bins B;
  B.mn = mn;
  {
    float sc = mx > mn ? (float)kBins / (mx - mn) : 0.0f;
    if (!(sc <= 1e30f)) sc = 1e30f;
    B.scale = sc;
  }
  // 2. stable ranking by bin: counts per (round, warp, bin)
  int bn[kRounds];
  uint32_t rk[kRounds];
#pragma unroll
  for (int r = 0; r < kRounds; ++r) {
    const uint32_t s = r * kThreads + tid;
    const bool v = s < fill;
    bn[r] = v ? B(b12[r].x) : kBins;  // kBins = "no bin"
    const unsigned peers = __match_any_sync(kFull, bn[r]);
    rk[r] = __popc(peers & lanemask_lt());
    if (v && rk[r] == 0) S.wc[(r * kWarps + warp) * kBins + bn[r]] = (uint16_t)__popc(peers);
  }
  __syncthreads();
  uint32_t tot = 0;  // per bin: total, and exclusive prefix over (round, warp) in place
  if (tid < kBins) {
#pragma unroll 8
    for (int q = 0; q < kRounds * kWarps; ++q) {
      const uint32_t c = S.wc[q * kBins + tid];
      S.wc[q * kBins + tid] = (uint16_t)tot;
      tot += c;
    }
  }
  {
    uint32_t total;
    const uint32_t ex = block_excl_scan<kThreads, uint32_t>(tid < kBins ? tot : 0u, S.scan32, &total);
    if (tid < kBins) S.bstart[tid] = ex;
    if (tid == 0) S.bstart[kBins] = total;
  }
  __syncthreads();
  // 3. place every candidate at its binned slot
#pragma unroll
  for (int r = 0; r < kRounds; ++r) {
    const uint32_t s = r * kThreads + tid;
    if (s < fill) {
      const uint32_t q = S.bstart[bn[r]] + S.wc[(r * kWarps + warp) * kBins + bn[r]] + rk[r];
      S.c12[q] = b12[r];
      S.c0[q] = b0[r];
      S.cpos[q] = S.fpos[s];
    }
  }
  __syncthreads();
  // 4. every row scans the bins that can pass its dim-1 float test
#pragma unroll
  for (int q = 0; q < R; ++q) {
    if (!rw.valid[q]) continue;
    const int bl = B(__fsub_rd(rw.lo1[q], ml));
    const int bh = B(rw.hi1[q]);
    const uint32_t k1 = S.bstart[bh + 1];
    for (uint32_t k = S.bstart[bl]; k < k1; ++k) {
      const float4 f = S.c12[k];
      if (!(f.x <= rw.hi1[q] && rw.lo1[q] <= f.y && f.z <= rw.hi2[q] && rw.lo2[q] <= f.w)) continue;
      const float2 g = S.c0[k];
      if (!(g.x <= rw.hi0[q] && rw.lo0[q] <= g.y)) continue;
      const int row = q * kThreads + tid;
      const uint32_t p = S.cpos[k];
      if (!exact_hit<R>(A, S, p, row)) continue;
      if (EMIT) A.pairs[S.roff[row] + rw.hits[q]] = make_uint2(A.slo_id[p], S.ruid[row]);
      ++rw.hits[q];
    }
  }
  __syncthreads();
}

template <int R, bool EMIT>
__global__ void __launch_bounds__(kThreads, 3) dd_tile_kernel(Args A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem<R>& S = *reinterpret_cast<Smem<R>*>(smem_raw);
  constexpr int kRows = kThreads * R;
  const int tid = threadIdx.x;
  const uint64_t j0 = (uint64_t)blockIdx.x * kRows;
  if (A.abort_flag && *A.abort_flag) return;  // this attempt is discarded (ddm.cu retries with LSB)
  const float kInf = __int_as_float(0x7f800000);
  if (tid == 0) S.rbmax = 0;
  __syncthreads();
  Rows<R> rw;
  uint32_t rbmax = 0;
#pragma unroll
  for (int q = 0; q < R; ++q) {
    const uint64_t j = j0 + (uint64_t)q * kThreads + tid;
    const int row = q * kThreads + tid;
    rw.valid[q] = j < A.m;
    rw.hits[q] = 0;
    if (rw.valid[q]) {
      const uint32_t lid = A.ulo_id[j];
      const uint64_t a = A.ulo_key[j];
      const double hi0 = A.upd.hi[0][lid];
      S.ra[row] = a;
      S.rb[row] = f64_key(hi0);
      S.rlid[row] = lid;
      S.ruid[row] = A.upd_map ? A.upd_map[lid] : lid;
      rw.lo0[q] = __double2float_rd(key_to_f64(a));
      rw.hi0[q] = __double2float_ru(hi0);
      rw.lo1[q] = __double2float_rd(A.upd.lo[1][lid]);
      rw.hi1[q] = __double2float_ru(A.upd.hi[1][lid]);
      rw.lo2[q] = A.d > 2 ? __double2float_rd(A.upd.lo[2][lid]) : -kInf;
      rw.hi2[q] = A.d > 2 ? __double2float_ru(A.upd.hi[2][lid]) : kInf;
      const uint32_t rb = A.r_b[j];
      rbmax = rb > rbmax ? rb : rbmax;
    }
  }
  if (EMIT) {  // row offsets: tile_off of each 256-row tile + exclusive scan of the counts
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const uint64_t j = j0 + (uint64_t)q * kThreads + tid;
      uint64_t total;
      const uint64_t e = block_excl_scan<kThreads, uint64_t>(rw.valid[q] ? (uint64_t)A.cnt[j] : 0ull, S.scan64, &total);
      if (rw.valid[q]) S.roff[q * kThreads + tid] = A.tile_off[(j0 >> 8) + q] + e;
    }
  }
  rbmax = __reduce_max_sync(kFull, rbmax);
  if ((tid & 31) == 0) atomicMax(&S.rbmax, rbmax);
  __syncthreads();
  rbmax = S.rbmax;
  const uint64_t rl0 = A.r_lo[j0];
  const uint64_t x = A.ulo_key[j0];
  const uint32_t nact = A.cnt0[j0] - (A.r_b[j0] - (uint32_t)rl0);  // |A_t| = stab(x_t) (I4)

  uint32_t fill = 0;
  // a6: A_t by a CTA-wide backward walk over Slo (windows of kWin positions,
  // aligned runs of 32^L positions with block max < x_t skipped).  hi_excl > 0
  // bounds the walk even on inconsistent inputs.
  int64_t hi_excl = (int64_t)rl0;
  uint32_t rem = nact;
  while (rem && hi_excl > 0) {
    const int64_t i = hi_excl - 1;
    if (((i + 1) & (kWin - 1)) == 0) {
      const int L = match::skip_levels(A.T, i, x);
      if (L >= 2) { hi_excl -= (int64_t)1 << (5 * L); continue; }
    }
    const int64_t base = i & ~(int64_t)(kWin - 1);
    bool mem[4];
    uint32_t c = 0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t p = base + tid * 4 + u;
      mem[u] = p < hi_excl && A.T.lvl[0][p] >= x;
      c += mem[u];
    }
    uint32_t total;
    const uint32_t ex = block_excl_scan<kThreads, uint32_t>(c, S.scan32, &total);
    if (fill + total > (uint32_t)kCap) {  // uniform
      process_chunk<R, EMIT>(A, S, rw, fill);
      fill = 0;
    }
    uint32_t o = fill + ex;
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (mem[u]) S.fpos[o++] = (uint32_t)(base + tid * 4 + u);
    fill += total;
    rem = total < rem ? rem - total : 0;
    hi_excl = base;
    __syncthreads();
  }
  // the contiguous Slo slice [rl0, rbmax)
  for (uint64_t p = rl0; p < rbmax;) {
    const uint32_t take = (uint32_t)umin64(kCap - fill, rbmax - p);
    for (uint32_t t = tid; t < take; t += kThreads) S.fpos[fill + t] = (uint32_t)(p + t);
    fill += take;
    p += take;
    __syncthreads();
    if (fill == (uint32_t)kCap) {
      process_chunk<R, EMIT>(A, S, rw, fill);
      fill = 0;
    }
  }
  if (fill) process_chunk<R, EMIT>(A, S, rw, fill);

  if (!EMIT) {
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const uint64_t j = j0 + (uint64_t)q * kThreads + tid;
      if (rw.valid[q]) A.cnt_out[j] = rw.hits[q];
      uint64_t total;
      block_excl_scan<kThreads, uint64_t>(rw.valid[q] ? (uint64_t)rw.hits[q] : 0ull, S.scan64, &total);
      if (tid == 0 && j0 + (uint64_t)q * kThreads < A.m) A.tile_sum[(j0 >> 8) + q] = total;
    }
  }
}

}  // namespace dd
}  // namespace ddm
