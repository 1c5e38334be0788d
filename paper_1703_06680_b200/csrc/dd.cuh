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
// Cells.  Each chunk is counting-sorted (stably, deterministically) into a
// kG1 x kG2 grid of cells over its float32 (dim-1, dim-2) lower bounds; a row
// only scans the cells whose lower bounds can pass its float test on both:
//   lo_k(U) <= hi_k(S) <= lo_k(S) + maxlen_k  =>  lo_k(S) >= rd(lo_k(U) - maxlen_k)
// with maxlen_k the chunk's largest float32 length on dim k rounded up and a
// monotone bucketer per dimension, so the cell rectangle
// [bin(rd(lo_k(U) - maxlen_k)), bin(hi_k(U))] (k = 1, 2) covers them.  With
// d = 2 every dim-2 value is -inf/+inf and all cells share one dim-2 bin.
// Cells are stored dim-2 major, so each dim-2 bin of the rectangle is one
// contiguous run of slots.
// Output (one enumeration).  The stage pass enumerates every tile once,
// writing the row counts, the 256-row tile sums and each hit as (row, its
// index within the row, sub id) into the tile's global staging slot.  After
// the offset scan (and the host's capacity check) the place pass groups each
// tile's staged hits by row and orders every row by sub id: deterministic
// output (rows in sweep order, each row by ascending output sub id) without a
// second enumeration, so the stage pass may place candidates into cells with
// plain atomic cursors.  Only a tile whose hits overflowed its staging slot
// enumerates again in the place pass (stable cell ranking, enumeration
// order), writing directly at its known offsets.  The count-only entry point
// runs the enumeration without staging.
#pragma once
#include <cstddef>
#include "common.cuh"
#include "match.cuh"

namespace ddm {
namespace dd {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
#ifndef DDM_DD_G1
#define DDM_DD_G1 32
#endif
#ifndef DDM_DD_G2
#define DDM_DD_G2 48
#endif
constexpr int kG1 = DDM_DD_G1;      // cells along dim 1
constexpr int kG2 = DDM_DD_G2;      // cells along dim 2
constexpr int kCells = kG1 * kG2;
constexpr int kCPT = kCells / 256;  // cells per thread in the cell scans
constexpr int kWin = 1024;          // A_t walk window (positions per step), 4 per thread
#ifndef DDM_DD_CAP
#define DDM_DD_CAP 1024
#endif
constexpr int kCap = DDM_DD_CAP;    // candidates per shared-memory chunk
constexpr int kRounds = kCap / kThreads;
constexpr int kList = 4;            // queued float passes per lane before an exact batch
static_assert(kCap >= kWin, "a whole walk window must fit one chunk");
static_assert(kCells == kThreads * kCPT, "whole cells per thread in the cell scans");

// ------------------------------------------------------------ index boxes

// Widened float32 boxes of the subscriptions on dims 1 and 2, in Slo order
// (a missing dim 2 is (-inf, +inf)): box12[i] = (lo1, hi1, lo2, hi2), lower
// bounds rounded down, upper bounds rounded up; box0[i] = the same for dim 0.
__global__ void __launch_bounds__(256) box_kernel(const double* __restrict__ sdims, int d, uint64_t n,
                                                  float4* __restrict__ box12,
                                                  const uint32_t* __restrict__ abort_flag,
                                                  const uint64_t* __restrict__ slo_key,
                                                  const uint64_t* __restrict__ slo_hi, float2* __restrict__ box0,
                                                  const float4* __restrict__ box_in, const uint32_t* __restrict__ slo_id) {
  if (abort_flag && *abort_flag) return;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    float4 b;
    if (box_in) {  // gathered from the input-order boxes (one 16-byte read)
      b = __ldg(box_in + slo_id[i]);
    } else {
      b.x = __double2float_rd(sdims[i]);
      b.y = __double2float_ru(sdims[n + i]);
      if (d > 2) {
        b.z = __double2float_rd(sdims[2 * n + i]);
        b.w = __double2float_ru(sdims[3 * n + i]);
      } else {
        b.z = -__int_as_float(0x7f800000);
        b.w = __int_as_float(0x7f800000);
      }
    }
    box12[i] = b;
    // dim 0 (the sweep dimension) from the sorted keys: [rd(lo), ru(hi)]
    box0[i] = make_float2(__double2float_rd(key_to_f64(slo_key[i])), __double2float_ru(key_to_f64(slo_hi[i])));
  }
}

// Widened dims-1/2 boxes in INPUT order (coalesced reads of the coordinates):
// the row-indexed calls gather these 16-byte boxes by id instead of gathering
// 2 (d - 1) float64 coordinates per region into sweep order.  The same read
// validates dims 1 and 2 (a1: finite, lo <= hi) into *err, so those dims need
// no separate validation launch.
__device__ __forceinline__ uint32_t box_check(double x, double y) {
  const uint64_t bx = (uint64_t)__double_as_longlong(x), by = (uint64_t)__double_as_longlong(y);
  if (!f64_finite_bits(bx) || !f64_finite_bits(by)) return match::kErrNonFinite;
  return x <= y ? 0u : match::kErrInverted;
}
__global__ void __launch_bounds__(256) box_in_kernel(const __grid_constant__ match::DimPtrs src, int d, uint64_t n,
                                                     float4* __restrict__ out, uint32_t* __restrict__ err) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const float kInf = __int_as_float(0x7f800000);
  uint32_t e = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    float4 b;
    const double l1 = __ldcs(src.lo[1] + i), h1 = __ldcs(src.hi[1] + i);
    e |= box_check(l1, h1);
    b.x = __double2float_rd(l1);
    b.y = __double2float_ru(h1);
    if (d > 2) {
      const double l2 = __ldcs(src.lo[2] + i), h2 = __ldcs(src.hi[2] + i);
      e |= box_check(l2, h2);
      b.z = __double2float_rd(l2);
      b.w = __double2float_ru(h2);
    } else {
      b.z = -kInf;
      b.w = kInf;
    }
    out[i] = b;
  }
  e = __reduce_or_sync(kFull, e);
  if (err && e && (threadIdx.x & 31) == 0) atomicOr(err, e);
}

// ------------------------------------------------------------ tile kernel

struct Args {
  const uint64_t* ulo_key;   // sorted update lower keys (dim 0)
  const uint32_t* ulo_id;    // local update ids in that order
  const uint32_t* upd_map;   // optional global ids
  const uint32_t* sub_map;   // optional global ids of the subscriptions
  const uint32_t* r_lo;      // dim-0 ranks (count pass a4)
  const uint32_t* r_b;
  const uint32_t* cnt0;      // dim-0 counts
  const uint64_t* slo_key;   // index: Slo keys, ids, upper keys (lvl[0]), block maxima
  const uint32_t* slo_id;
  match::DimPtrs upd;        // update coordinates, all dims
  MaxTree T;
  const double* sdims;       // [(d-1)][2][n] other dims of the subs in Slo order
  const double* udims;       // [(d-1)][2][m] other dims of the updates in Ulo order
  const uint64_t* uhi;       // dim-0 upper keys in Ulo order (nullptr: from upd.hi[0])
  const float4* box12;       // widened float32 boxes (box_kernel)
  const float2* box0;        // widened float32 dim-0 boxes in Slo order (box_kernel)
  match::DimPtrs sub;        // subscription coordinates, all dims (exact tests when sdims is null)
  const float4* ubox;        // widened dims-1/2 boxes of the updates in INPUT order (box_in_kernel), or null
  const uint32_t* tile_rk;   // row-indexed tiles: {r_lo(x_t), r_b(max b)} per tile (tile_ranks_kernel), or null
  const uint64_t* pmw;       //   with the prefix maxima of slo_hi (the A_t walk stops where they drop below x_t)
  const uint64_t* pmb;
  uint64_t n, m;
  int d;
  const uint32_t* abort_flag;  // non-zero: an MSD bucket overflowed, inputs are not sorted -> no-op
  // count pass
  uint32_t* cnt_out;
  uint64_t* tile_sum;        // per 256-row tile
  // stage / place passes
  uint2* stage;               // [tiles][kStageCap] staged hits: {sub id, (row << 16) | index in row}
  uint32_t* stage_n;          // [tiles] staged hits per tile, or ~0u when the slot overflowed
  const uint32_t* cnt;        // place: row counts (stage pass output)
  const uint64_t* tile_off;   // place: exclusive scan of the 256-row tile sums
  uint2* pairs;
  uint64_t capacity;          // pairs at or past capacity are never written
  uint32_t* ovf_any;          // rows_kernel stage pass: set when some tile's staging slot overflowed
};

constexpr uint32_t kTileSkip = 0xfffffffeu;  // stage_n: the tile is placed by rows_place_kernel
constexpr uint32_t kStageCap = 8192;  // staged hits per tile (c4 averages ~4100 per 1024-row tile)
enum { kEmCount = 0, kEmDirect = 1, kEmStage = 2 };

template <int R>
struct Smem {
  static constexpr int kRows = kThreads * R;
  float4 c12[kCap];          // chunk boxes in cell order
  float4 rbox[kRows];        // widened row boxes (lo1, hi1, lo2, hi2)
  uint32_t cpos[kCap];       // Slo position of each slot (cell order)
  uint32_t fpos[kCap];       // Slo positions in fill order
  uint16_t lst[kList * kThreads];  // per-lane queues of float passes: (row q << 12) | slot
  uint32_t cstart[kCells + 1];
  uint32_t run[kCells];      // slots already assigned per cell (earlier rounds)
  float red[6 * kWarps];
  uint64_t scan64[kWarps + 1];
  uint32_t scan32[kWarps + 1];
  uint32_t rbmax;
  uint32_t nout;     // staged hits of this tile
  uint32_t ovf;      // staging overflowed -> re-enumerate in the place pass
  uint32_t tile;
  // last: per (warp, cell) counts of one stable ranking round -> prefixes;
  // only the place pass's direct enumeration uses them, the count / stage
  // passes are launched without this tail (smem_bytes)
  uint16_t wc[kWarps * kCells];
};


// Monotone float bucketer over one chunk's lower bounds on one dimension
// (G bins).
template <int G>
struct Bins {
  float mn, scale;
  __device__ __forceinline__ int operator()(float x) const {
    float u = floorf((x - mn) * scale);
    u = fminf(fmaxf(u, 0.0f), (float)(G - 1));  // fmaxf(NaN, 0) = 0
    return (int)u;
  }
  __device__ __forceinline__ void init(float lo, float hi) {
    mn = lo;
    float sc = hi > lo ? (float)G / (hi - lo) : 0.0f;
    if (!(sc <= 1e30f)) sc = 1e30f;
    scale = sc;
  }
};

template <int R>
struct Rows {
  uint32_t hits[R];
  uint64_t off[R];
  bool valid[R];
};

// Exact Alg. 1 test on every dimension for the sub at Slo position p and the
// update at sorted position j (only float passes get here).  Both sides are
// read in sweep order (sdims / udims), so these reads stay local; without
// them (row-indexed calls: only float boxes were built) from the input arrays
// through the ids.
__device__ __forceinline__ bool exact_hit(const Args& A, uint32_t p, uint64_t j, uint32_t lid) {
  const uint64_t b = A.uhi ? A.uhi[j] : f64_key(A.upd.hi[0][lid]);
  if (!(A.slo_key[p] <= b && A.T.lvl[0][p] >= A.ulo_key[j])) return false;  // dim 0 (keys)
  if (A.sdims) {
    for (int k = 1; k < A.d; ++k) {
      const double slo = A.sdims[(uint64_t)(k - 1) * 2 * A.n + p];
      const double shi = A.sdims[(uint64_t)(k - 1) * 2 * A.n + A.n + p];
      const double ulo = A.udims[(uint64_t)(k - 1) * 2 * A.m + j];
      const double uhi = A.udims[(uint64_t)(k - 1) * 2 * A.m + A.m + j];
      if (!(slo <= uhi && ulo <= shi)) return false;
    }
    return true;
  }
  const uint32_t sid = A.slo_id[p], uid = A.ulo_id[j];
  for (int k = 1; k < A.d; ++k)
    if (!(A.sub.lo[k][sid] <= A.upd.hi[k][uid] && A.upd.lo[k][uid] <= A.sub.hi[k][sid])) return false;
  return true;
}

// Widened dims-1/2 box of the update at sorted position j.
__device__ __forceinline__ float4 row_box(const Args& A, uint64_t j) {
  if (A.ubox) return __ldg(A.ubox + A.ulo_id[j]);
  const float kInf = __int_as_float(0x7f800000);
  float4 u;
  u.x = __double2float_rd(A.udims[j]);
  u.y = __double2float_ru(A.udims[A.m + j]);
  u.z = A.d > 2 ? __double2float_rd(A.udims[2 * A.m + j]) : -kInf;
  u.w = A.d > 2 ? __double2float_ru(A.udims[3 * A.m + j]) : kInf;
  return u;
}

// Exact re-test of this lane's queued float passes, in queue order.
template <int R, int EM>
__device__ __forceinline__ void flush_list(const Args& A, Smem<R>& S, Rows<R>& rw, uint32_t nl, uint64_t j0) {
  const int tid = threadIdx.x;
  for (uint32_t e = 0; e < nl; ++e) {
    const uint32_t v = S.lst[e * kThreads + tid];
    const int q = (int)(v >> 12);
    const uint32_t p = S.cpos[v & 4095u];
    const uint64_t j = j0 + (uint64_t)q * kThreads + tid;
    const uint32_t lid = A.ulo_id[j];
    if (!exact_hit(A, p, j, lid)) continue;
#pragma unroll
    for (int qq = 0; qq < R; ++qq)
      if (qq == q) {
        const uint32_t seq = rw.hits[qq];
        if (EM == kEmDirect) {
          const uint64_t pos = rw.off[qq] + seq;
          if (pos < A.capacity)
            A.pairs[pos] = make_uint2(match::sub_out(A.sub_map, A.slo_id[p]), A.upd_map ? A.upd_map[lid] : lid);
        } else if (EM == kEmStage) {
          const uint32_t slot = atomicAdd(&S.nout, 1u);
          if (slot < kStageCap && seq < 65536u)
            A.stage[(uint64_t)S.tile * kStageCap + slot] =
                make_uint2(match::sub_out(A.sub_map, A.slo_id[p]), ((uint32_t)(q * kThreads + tid) << 16) | seq);
          else
            S.ovf = 1;
        }
        ++rw.hits[qq];
      }
  }
}

template <int R, int EM>
__device__ void process_chunk(const Args& A, Smem<R>& S, Rows<R>& rw, uint32_t fill, uint64_t j0) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // 1. chunk min/max lower bound and max length (rounded up) on dims 1, 2
  float mn1 = __int_as_float(0x7f800000), mx1 = -mn1, ml1 = 0.0f;
  float mn2 = mn1, mx2 = -mn1, ml2 = 0.0f;
  int cell[kRounds];
#pragma unroll
  for (int r = 0; r < kRounds; ++r) {
    const uint32_t s = r * kThreads + tid;
    if (s < fill) {
      const float4 b = A.box12[S.fpos[s]];
      mn1 = fminf(mn1, b.x);
      mx1 = fmaxf(mx1, b.x);
      ml1 = fmaxf(ml1, __fsub_ru(b.y, b.x));
      mn2 = fminf(mn2, b.z);
      mx2 = fmaxf(mx2, b.z);
      ml2 = fmaxf(ml2, __fsub_ru(b.w, b.z));
      S.c12[s] = b;  // fill-order staging (re-placed in step 3)
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    mn1 = fminf(mn1, __shfl_xor_sync(kFull, mn1, o));
    mx1 = fmaxf(mx1, __shfl_xor_sync(kFull, mx1, o));
    ml1 = fmaxf(ml1, __shfl_xor_sync(kFull, ml1, o));
    mn2 = fminf(mn2, __shfl_xor_sync(kFull, mn2, o));
    mx2 = fmaxf(mx2, __shfl_xor_sync(kFull, mx2, o));
    ml2 = fmaxf(ml2, __shfl_xor_sync(kFull, ml2, o));
  }
  if (lane == 0) {
    S.red[warp] = mn1; S.red[kWarps + warp] = mx1; S.red[2 * kWarps + warp] = ml1;
    S.red[3 * kWarps + warp] = mn2; S.red[4 * kWarps + warp] = mx2; S.red[5 * kWarps + warp] = ml2;
  }
#pragma unroll
  for (int c = 0; c < kCPT; ++c) S.run[tid * kCPT + c] = 0;
  __syncthreads();
#pragma unroll
  for (int w = 0; w < kWarps; ++w) {
    mn1 = fminf(mn1, S.red[w]);
    mx1 = fmaxf(mx1, S.red[kWarps + w]);
    ml1 = fmaxf(ml1, S.red[2 * kWarps + w]);
    mn2 = fminf(mn2, S.red[3 * kWarps + w]);
    mx2 = fmaxf(mx2, S.red[4 * kWarps + w]);
    ml2 = fmaxf(ml2, S.red[5 * kWarps + w]);
  }
  Bins<kG1> B1;
  Bins<kG2> B2;
  B1.init(mn1, mx1);
  B2.init(mn2, mx2);
  // 2. cells, totals per cell (order-free), then the cell starts
#pragma unroll
  for (int r = 0; r < kRounds; ++r) {
    const uint32_t s = r * kThreads + tid;
    if (s < fill) {
      const float4 b = S.c12[s];
      cell[r] = B2(b.z) * kG1 + B1(b.x);
      atomicAdd(&S.run[cell[r]], 1u);
    } else {
      cell[r] = kCells;  // "no cell"
    }
  }
  __syncthreads();
  {
    uint32_t v[kCPT], sum = 0;
#pragma unroll
    for (int c = 0; c < kCPT; ++c) { v[c] = S.run[tid * kCPT + c]; sum += v[c]; }
    uint32_t total;
    uint32_t ex = block_excl_scan<kThreads, uint32_t>(sum, S.scan32, &total);
#pragma unroll
    for (int c = 0; c < kCPT; ++c) {
      S.cstart[tid * kCPT + c] = ex;
      S.run[tid * kCPT + c] = ex;  // running slot cursor per cell
      ex += v[c];
    }
    if (tid == 0) S.cstart[kCells] = total;
  }
  __syncthreads();
  // 3. placement into cell order.  The stage and count passes place with one
  // atomic cursor per cell (the order inside a cell does not matter: the
  // place pass orders every row by sub id); the direct pass of an overflowed
  // tile ranks stably (per-round warp counts + match_any) so that its
  // enumeration order, which is its output order, is deterministic.
  float4 keep[kRounds];
  uint32_t kpos[kRounds];
#pragma unroll
  for (int r = 0; r < kRounds; ++r) {
    const uint32_t s = r * kThreads + tid;
    if (s < fill) { keep[r] = S.c12[s]; kpos[r] = S.fpos[s]; }
  }
  __syncthreads();  // c12 is rewritten in cell order below
  if (EM != kEmDirect) {
#pragma unroll
    for (int r = 0; r < kRounds; ++r)
      if (cell[r] < kCells) {
        const uint32_t q = atomicAdd(&S.run[cell[r]], 1u);
        S.c12[q] = keep[r];
        S.cpos[q] = kpos[r];
      }
  } else {
#pragma unroll
    for (int r = 0; r < kRounds; ++r) {
      for (int i = tid; i < kWarps * kCells / 2; i += kThreads) reinterpret_cast<uint32_t*>(S.wc)[i] = 0;
      __syncthreads();
      const unsigned peers = __match_any_sync(kFull, cell[r]);
      const uint32_t rk = __popc(peers & lanemask_lt());
      if (cell[r] < kCells && rk == 0) S.wc[warp * kCells + cell[r]] = (uint16_t)__popc(peers);
      __syncthreads();
#pragma unroll
      for (int cc = 0; cc < kCPT; ++cc) {  // per cell: exclusive prefix over warps, advance the cursor
        const int cl = tid * kCPT + cc;
        uint32_t acc = S.run[cl];
        const uint32_t c0 = S.cstart[cl];
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
          const uint32_t c = S.wc[w * kCells + cl];
          S.wc[w * kCells + cl] = (uint16_t)(acc - c0);
          acc += c;
        }
        S.run[cl] = acc;
      }
      __syncthreads();
      if (cell[r] < kCells) {
        const uint32_t q = S.cstart[cell[r]] + S.wc[warp * kCells + cell[r]] + rk;
        S.c12[q] = keep[r];
        S.cpos[q] = kpos[r];
      }
      __syncthreads();  // wc is zeroed again by the next round
    }
  }
  __syncthreads();
  // 4. every row scans the cells that can pass its float test on dims 1, 2
  // (one contiguous run per dim-2 bin).  Float passes are queued per lane and
  // re-tested exactly in batches (the exact test reads global memory;
  // batching keeps one lane's rare pass from stalling its warp every time).
  uint32_t nl = 0;
#pragma unroll
  for (int q = 0; q < R; ++q) {
    if (!rw.valid[q]) continue;
    const float4 u = S.rbox[q * kThreads + tid];
    const int b1l = B1(__fsub_rd(u.x, ml1)), b1h = B1(u.y);
    const int b2l = B2(__fsub_rd(u.z, ml2)), b2h = B2(u.w);
    for (int b2 = b2l; b2 <= b2h; ++b2) {
      const uint32_t k1 = S.cstart[b2 * kG1 + b1h + 1];
      for (uint32_t k = S.cstart[b2 * kG1 + b1l]; k < k1; ++k) {
        const float4 f = S.c12[k];
        if (!(f.x <= u.y && u.x <= f.y && f.z <= u.w && u.z <= f.w)) continue;
        if (nl == kList) {
          flush_list<R, EM>(A, S, rw, nl, j0);
          nl = 0;
        }
        S.lst[nl * kThreads + tid] = (uint16_t)((q << 12) | k);
        ++nl;
      }
    }
  }
  flush_list<R, EM>(A, S, rw, nl, j0);
  __syncthreads();
}

// Every dim-0 candidate of the tile's rows (A_t by a CTA-wide backward walk
// over Slo in windows of kWin positions with aligned runs of 32^L positions
// whose block max < x_t skipped, then the Slo slice [rl0, rbmax)), pushed
// through process_chunk.  hi_excl > 0 bounds the walk on inconsistent inputs.
template <int R, int EM>
__device__ void enumerate(const Args& A, Smem<R>& S, Rows<R>& rw, uint64_t j0, uint32_t rbmax) {
  const int tid = threadIdx.x;
  const uint64_t rl0 = A.r_lo[j0];
  const uint64_t x = A.ulo_key[j0];
  const uint32_t nact = A.cnt0[j0] - (A.r_b[j0] - (uint32_t)rl0);  // |A_t| = stab(x_t) (I4)
  uint32_t fill = 0;
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
      process_chunk<R, EM>(A, S, rw, fill, j0);
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
  for (uint64_t p = rl0; p < rbmax;) {
    const uint32_t take = (uint32_t)umin64(kCap - fill, rbmax - p);
    for (uint32_t t = tid; t < take; t += kThreads) S.fpos[fill + t] = (uint32_t)(p + t);
    fill += take;
    p += take;
    __syncthreads();
    if (fill == (uint32_t)kCap) {
      process_chunk<R, EM>(A, S, rw, fill, j0);
      fill = 0;
    }
  }
  if (fill) process_chunk<R, EM>(A, S, rw, fill, j0);
}

enum { kModeCount = 0, kModeStage = 1, kModePlace = 2 };
template <int R>
constexpr size_t smem_bytes(int mode) {
  return mode == kModePlace ? sizeof(Smem<R>) : (offsetof(Smem<R>, wc) + 15) / 16 * 16;
}

// kModeCount: row counts + 256-row tile sums.  kModeStage: the same plus the
// staged hits.  kModePlace: staged hits -> pairs (or, for a tile whose slot
// overflowed, a second enumeration writing directly).
template <int R, int MODE>
#ifndef DDM_DD_MINB
#define DDM_DD_MINB 4
#endif
__global__ void __launch_bounds__(kThreads, DDM_DD_MINB) dd_tile_kernel(const __grid_constant__ Args A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem<R>& S = *reinterpret_cast<Smem<R>*>(smem_raw);
  constexpr int kRows = kThreads * R;
  const int tid = threadIdx.x;
  if (A.abort_flag && *A.abort_flag) return;  // this attempt is discarded (ddm.cu retries with LSB)
  const uint32_t tile = blockIdx.x;
  const uint64_t j0 = (uint64_t)tile * kRows;
  if (tid == 0) {
    S.rbmax = 0;
    S.nout = 0;
    S.ovf = 0;
    S.tile = tile;
  }
  __syncthreads();
  Rows<R> rw;
#pragma unroll
  for (int q = 0; q < R; ++q) {
    rw.valid[q] = j0 + (uint64_t)q * kThreads + tid < A.m;
    rw.hits[q] = 0;
    rw.off[q] = 0;
  }
  if (MODE == kModePlace) {
    // row offsets = 256-row tile offset + exclusive scan of the row counts
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const uint64_t j = j0 + (uint64_t)q * kThreads + tid;
      uint64_t total;
      const uint64_t e = block_excl_scan<kThreads, uint64_t>(rw.valid[q] ? (uint64_t)A.cnt[j] : 0ull, S.scan64, &total);
      if (rw.valid[q]) rw.off[q] = A.tile_off[(j0 >> 8) + q] + e;
    }
    __syncthreads();
    const uint32_t nst = A.stage_n[tile];
    if (nst == kTileSkip) return;  // placed by rows_place_kernel
    if (nst != ~0u) {
      // the tile's staged hits, grouped by row (counting sort on the row
      // prefix) and each row ordered by sub id: output order = rows in sweep
      // order, each row by ascending sub id, whatever the staging order was.
      // Shared memory: sub ids over the chunk-box + row-box areas, row
      // cursors over cpos (all contiguous, unused by a placing tile).
      static_assert(sizeof(float4) * (kCap + kThreads * R) >= sizeof(uint32_t) * kStageCap, "staged ids fit");
      static_assert(sizeof(uint32_t) * kCap >= sizeof(uint32_t) * kThreads * R, "row cursors fit");
      uint32_t* sid = reinterpret_cast<uint32_t*>(S.c12);
      uint32_t* cur = S.cpos;
      const uint64_t t0 = A.tile_off[j0 >> 8];
      __syncthreads();
#pragma unroll
      for (int q = 0; q < R; ++q) cur[q * kThreads + tid] = (uint32_t)(rw.off[q] - t0);
      __syncthreads();
      for (uint32_t e = tid; e < nst; e += kThreads) {
        const uint2 h = A.stage[(uint64_t)tile * kStageCap + e];
        sid[atomicAdd(&cur[h.y >> 16], 1u)] = h.x;
      }
      __syncthreads();
#pragma unroll
      for (int q = 0; q < R; ++q) {  // each thread sorts and writes its rows (a few hits each)
        if (!rw.valid[q]) continue;
        const uint32_t lo = (uint32_t)(rw.off[q] - t0), hi = cur[q * kThreads + tid];
        for (uint32_t x = lo + 1; x < hi; ++x) {
          const uint32_t v = sid[x];
          uint32_t y = x;
          while (y > lo && sid[y - 1] > v) { sid[y] = sid[y - 1]; --y; }
          sid[y] = v;
        }
        if (hi > lo) {
          const uint32_t lid = A.ulo_id[j0 + (uint64_t)q * kThreads + tid];
          const uint32_t uid = A.upd_map ? A.upd_map[lid] : lid;
          for (uint32_t x = lo; x < hi; ++x)
            if (t0 + x < A.capacity) A.pairs[t0 + x] = make_uint2(sid[x], uid);
        }
      }
      return;
    }
    // overflowed tile: fall through to a direct enumeration (block-uniform)
    __syncthreads();
  }
  const float kInf = __int_as_float(0x7f800000);
  uint32_t rbmax = 0;
#pragma unroll
  for (int q = 0; q < R; ++q) {
    const uint64_t j = j0 + (uint64_t)q * kThreads + tid;
    if (rw.valid[q]) {
      S.rbox[q * kThreads + tid] = row_box(A, j);
      const uint32_t rb = A.r_b[j];
      rbmax = rb > rbmax ? rb : rbmax;
    }
  }
  rbmax = __reduce_max_sync(kFull, rbmax);
  if ((tid & 31) == 0) atomicMax(&S.rbmax, rbmax);
  __syncthreads();
  rbmax = S.rbmax;
  if (MODE == kModePlace) {
    enumerate<R, kEmDirect>(A, S, rw, j0, rbmax);
    return;
  }
  if (MODE == kModeStage) enumerate<R, kEmStage>(A, S, rw, j0, rbmax);
  else enumerate<R, kEmCount>(A, S, rw, j0, rbmax);
#pragma unroll
  for (int q = 0; q < R; ++q) {
    const uint64_t j = j0 + (uint64_t)q * kThreads + tid;
    if (rw.valid[q]) A.cnt_out[j] = rw.hits[q];
    uint64_t total;
    block_excl_scan<kThreads, uint64_t>(rw.valid[q] ? (uint64_t)rw.hits[q] : 0ull, S.scan64, &total);
    if (tid == 0 && j0 + (uint64_t)q * kThreads < A.m) A.tile_sum[(j0 >> 8) + q] = total;
  }
  if (MODE == kModeStage && tid == 0) A.stage_n[tile] = S.ovf ? ~0u : S.nout;
}


// ------------------------------------------------------------ row-indexed tiles
//
// The same tile and candidate set as dd_tile_kernel -- T consecutive updates
// in sweep order against C_t = A_t ⊔ Slo[r_lo(x_t), max_j r_b(j)) (Alg. 6
// SubSet[p] + the segment's inserted subscriptions) -- with the loop turned
// around.  dd_tile_kernel streams C_t through shared memory in chunks,
// cell-sorts every chunk and lets each ROW scan the cells it can reach: every
// row pays for every chunk (c4: 1024 rows x ~46 chunks per tile).  Here the
// tile's rows are binned ONCE into a G1 x G2 cell grid over their float32
// (dim-1, dim-2) lower bounds (counting sort of row indices in shared memory),
// and every CANDIDATE -- one per lane, read straight from the Slo-ordered box
// arrays, no staging -- scans the row cells its widened box can reach:
//   lo_k(S) <= hi_k(U) and lo_k(U) <= hi_k(S) <= lo_k(S) + len_k(S)
//   =>  lo_k(U) in [rd(lo_k(S) - maxlen_k(rows)), hi_k(S)]      (k = 1, 2)
// with maxlen_k the largest widened row length.
//
// Decision per (candidate, row) in the cells, on dims 0..2 (float32 boxes of
// the subscriptions: box12 + box0; of the rows: built here):
//  - the widened ("outer") boxes do not overlap on some dimension: no pair
//    (widening only enlarges intervals, so a true pair always overlaps);
//  - both inequalities of every dimension hold with a margin of more than the
//    float rounding of both endpoints (sure_le): a pair, decided without
//    touching the float64 data (d <= 3);
//  - otherwise (endpoints within rounding of each other, or d > 3): queued and
//    re-tested exactly on every dimension (exact_hit, Alg. 1), a warp at a time.
// Hits are counted per row with shared-memory atomics; the stage pass stages
// (sub, row) per tile, the place pass (rows_place_kernel) orders each row by
// sub id.  A tile whose staging slot overflows marks its 1024-row
// dd_tile_kernel tiles for that kernel's direct (deterministic) place pass.

#ifndef DDM_DDR_THREADS
#define DDM_DDR_THREADS 1024
#endif
constexpr int kRT = DDM_DDR_THREADS;  // threads of a row-indexed CTA
constexpr int kRW = kRT / 32;
constexpr int kRowFpos = 4 * kWin;    // A_t positions staged per batch

struct RBins {  // monotone float bucketer, runtime bin count
  float mn, scale;
  int top;
  __device__ __forceinline__ int operator()(float x) const {
    float u = floorf((x - mn) * scale);
    u = fminf(fmaxf(u, 0.0f), (float)top);  // fmaxf(NaN, 0) = 0
    return (int)u;
  }
  __device__ __forceinline__ void init(float lo, float hi, int g) {
    mn = lo;
    top = g - 1;
    float sc = hi > lo ? (float)g / (hi - lo) : 0.0f;
    if (!(sc <= 1e30f)) sc = 1e30f;
    scale = sc;
  }
};

// x <= y certainly holds for the float64 values behind a = rd(x) and b = ru(y):
// x < next(a) <= a + |a| 2^-23 + 2^-149 and y > prev(b) >= b - |b| 2^-23 -
// 2^-149, so a + (|a| + |b|) 2^-22 + 2^-148 <= b suffices; every operation of
// the test rounds up (a larger left side only makes it stricter), and
// 2.4e-7f >= 2^-22, 1e-44f >= 2^-148.  b = +inf (y beyond the float range:
// rd / ru saturate, a may be FLT_MAX for any larger x) never passes; a = -inf
// gives NaN, which fails.
__device__ __forceinline__ bool sure_le(float a, float b) {
  const float m = __fadd_ru(fabsf(a), fabsf(b));
  return __fadd_ru(__fmaf_ru(m, 2.4e-7f, a), 1e-44f) <= b && b < __int_as_float(0x7f800000);
}

template <int R>
struct RowSmem {
  static constexpr int kRows = kRT * R;
  float4 cbox[kRows];          // widened row boxes (lo1, hi1, lo2, hi2) in CELL order (slot k holds row rrow[k]):
                               // the candidates' cell scans read them without the rrow indirection
  float2 rbox0[kRows];         // widened dim-0 row boxes (lo0, hi0), tile-row order
  uint16_t rrow[kRows];        // tile row of each cell slot (cell order)
  uint16_t cstart[kRows + 2];  // G1 x G2 = kRows cells (d = 2: kRows x 1)
  uint32_t rcnt[kRows];        // hits per row; cell counts / cursors while binning
  uint32_t fpos[kRowFpos];     // A_t members of a batch of walk windows
  unsigned long long lst[kList * kRT];  // queued uncertain passes, per warp: [warp][e][lane] = (cell slot << 32) | Slo position
  float red[6 * kRW];
  uint32_t scan32[kRW + 1];
  uint64_t scan64[kRW + 1];
  uint32_t rbmax;
  uint32_t nout;
  uint32_t ovf;
};

template <int R>
constexpr uint32_t rows_stage_cap() { return 8u * kRT * R; }  // staged hits per tile (c4: ~4.1 per row)

// Decision for a queued (row r, Slo position p) whose dims-1/2 boxes overlap:
// the dim-0 boxes, then the certain test (float margins, d <= 3), else the
// exact test (Alg. 1 on every dimension, float64 / keys).
template <int R>
__device__ __forceinline__ bool rows_decide(const Args& A, const RowSmem<R>& S, unsigned long long v, uint64_t j0,
                                            bool sure_ok, uint32_t& r) {
  const uint32_t k = (uint32_t)(v >> 32), p = (uint32_t)v;
  r = S.rrow[k];
  const float2 f0 = __ldg(A.box0 + p);
  const float2 u0 = S.rbox0[r];
  if (!(f0.x <= u0.y && u0.x <= f0.y)) return false;
  if (sure_ok && sure_le(f0.x, u0.y) && sure_le(u0.x, f0.y)) {
    const float4 f = __ldg(A.box12 + p);
    const float4 u = S.cbox[k];
    if (sure_le(f.x, u.y) && sure_le(u.x, f.y) && (A.d == 2 || (sure_le(f.z, u.w) && sure_le(u.z, f.w))))
      return true;
  }
  const uint64_t j = j0 + r;
  return exact_hit(A, p, j, A.uhi ? 0u : A.ulo_id[j]);
}

// A pair of the tile (row r, Slo position p): counted, and staged by the
// stage pass (slot from the per-tile counter; `slot` precomputed by a
// warp-aggregated reservation, or ~0u to reserve one here).
template <int R, int MODE>
__device__ __forceinline__ void rows_hit(const Args& A, RowSmem<R>& S, uint32_t r, uint32_t p, uint32_t tile,
                                         uint32_t slot) {
  const uint32_t seq = atomicAdd(&S.rcnt[r], 1u);
  if (MODE == kModeStage) {
    if (slot == ~0u) slot = atomicAdd(&S.nout, 1u);
    if (slot < rows_stage_cap<R>())
      A.stage[(uint64_t)tile * rows_stage_cap<R>() + slot] =
          make_uint2(match::sub_out(A.sub_map, A.slo_id[p]), (r << 16) | (seq & 0xffffu));
    else
      S.ovf = 1;
  }
}

// Queued passes live per warp: lst[warp][e][lane].  A lane whose queue fills
// inside a candidate decides it alone (rare); otherwise the warp decides
// together at converged points: entry x of the warp's queues (in lane-major
// order) is taken by lane x % 32, its owner found by a binary search over the
// lanes' queue prefixes, so the decisions and hits run with full warps.
__device__ __forceinline__ unsigned long long* rows_lane_q(unsigned long long* lst, int tid) {
  return lst + (tid >> 5) * (kList * 32) + (tid & 31);
}
template <int R, int MODE>
__device__ __forceinline__ void rows_flush_lane(const Args& A, RowSmem<R>& S, uint32_t nl, uint64_t j0,
                                                uint32_t tile, bool sure_ok) {
  const unsigned long long* q = rows_lane_q(S.lst, threadIdx.x);
  for (uint32_t e = 0; e < nl; ++e) {
    const unsigned long long v = q[e * 32];
    uint32_t r;
    if (rows_decide<R>(A, S, v, j0, sure_ok, r)) rows_hit<R, MODE>(A, S, r, (uint32_t)v, tile, ~0u);
  }
}
template <int R, int MODE>
__device__ __forceinline__ void rows_flush_warp(const Args& A, RowSmem<R>& S, uint32_t& nl, uint64_t j0,
                                                uint32_t tile, bool sure_ok, bool force) {
  const int tid = threadIdx.x, lane = tid & 31;
  const uint32_t tot = __reduce_add_sync(kFull, nl);
  if (tot == 0 || (!force && tot < 32 && !__any_sync(kFull, nl + 1 >= (uint32_t)kList))) return;
  uint32_t pre = nl;  // inclusive prefix over the lanes
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(kFull, pre, o);
    if (lane >= o) pre += t;
  }
  pre -= nl;  // exclusive
  const unsigned long long* w = S.lst + (tid >> 5) * (kList * 32);
  for (uint32_t base = 0; base < tot; base += 32) {
    const uint32_t x = base + lane;
    // owner: the largest lane L with pre_L <= x (lanes with empty queues share
    // the next lane's prefix, so the largest one owns x)
    int L = 0;
#pragma unroll
    for (int step = 16; step; step >>= 1) {
      const uint32_t pv = __shfl_sync(kFull, pre, L + step);
      if (pv <= x) L += step;
    }
    const uint32_t pl = __shfl_sync(kFull, pre, L);
    bool hit = false;
    unsigned long long v = 0;
    uint32_t r = 0;
    if (x < tot) {
      v = w[(x - pl) * 32 + L];
      hit = rows_decide<R>(A, S, v, j0, sure_ok, r);
    }
    uint32_t slot = ~0u;
    if (MODE == kModeStage) {  // one slot reservation per warp
      const unsigned hm = __ballot_sync(kFull, hit);
      uint32_t b = 0;
      if (lane == 0 && hm) b = atomicAdd(&S.nout, (uint32_t)__popc(hm));
      b = __shfl_sync(kFull, b, 0);
      slot = b + __popc(hm & lanemask_lt());
    }
    if (hit) rows_hit<R, MODE>(A, S, r, (uint32_t)v, tile, slot);
  }
  __syncwarp();
  nl = 0;
}

// One candidate (Slo position p) against the binned rows: rows whose widened
// dims-1/2 boxes overlap the candidate's are queued for rows_decide.
template <int R, int MODE>
__device__ __forceinline__ void rows_candidate(const Args& A, RowSmem<R>& S, const RBins& B1, const RBins& B2, int g1,
                                               float ml1, float ml2, bool sure_ok, uint32_t p, uint32_t& nl,
                                               uint64_t j0, uint32_t tile) {
  const float4 f = __ldg(A.box12 + p);
  const int c1l = B1(__fsub_rd(f.x, ml1)), c1h = B1(f.y);
  const int c2l = B2(__fsub_rd(f.z, ml2)), c2h = B2(f.w);
  unsigned long long* q = rows_lane_q(S.lst, threadIdx.x);
  for (int c2 = c2l; c2 <= c2h; ++c2) {
    const uint32_t k1 = S.cstart[c2 * g1 + c1h + 1];
    for (uint32_t k = S.cstart[c2 * g1 + c1l]; k < k1; ++k) {
      const float4 u = S.cbox[k];
      if (!(f.x <= u.y && u.x <= f.y && f.z <= u.w && u.z <= f.w)) continue;
      if (nl == kList) {
        rows_flush_lane<R, MODE>(A, S, nl, j0, tile, sure_ok);
        nl = 0;
      }
      q[nl * 32] = ((unsigned long long)k << 32) | p;
      ++nl;
    }
  }
}

// Per row-indexed tile: rk[2t] = r_lo(x_t) = #{S.lo <= x_t} (x_t = the tile's
// first update lower key) and rk[2t+1] = #{S.lo <= max_j b_j} (the end of the
// tile's candidate slice), by binary search over Slo -- what the row-indexed
// pass needs from the a4 count pass, without running it (nor sorting Shi).
// One warp per tile: the lanes reduce the tile's upper keys, lane 0 searches.
template <int R>
__global__ void __launch_bounds__(256) tile_ranks_kernel(const __grid_constant__ Args A, uint32_t* __restrict__ rk) {
  constexpr int kRows = kRT * R;
  const uint32_t t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const uint64_t tiles = (A.m + kRows - 1) / kRows;
  if (t >= tiles) return;
  if (A.abort_flag && *A.abort_flag) return;
  const uint64_t j0 = (uint64_t)t * kRows, j1 = umin64(A.m, j0 + kRows);
  uint64_t bmax = 0;
  for (uint64_t j = j0 + lane; j < j1; j += 32) {
    const uint64_t b = A.uhi ? A.uhi[j] : f64_key(A.upd.hi[0][A.ulo_id[j]]);
    bmax = b > bmax ? b : bmax;
  }
  bmax = warp_max_u64(bmax);
  if (lane == 0) {
    rk[2 * t] = (uint32_t)match::ub(A.slo_key, 0, A.n, A.ulo_key[j0]);
    rk[2 * t + 1] = (uint32_t)match::ub(A.slo_key, 0, A.n, bmax);
  }
}

// kModeCount: row counts + 256-row tile sums.  kModeStage: the same plus the
// staged hits; stage_n[tile] = their number or ~0u (overflow), and the
// 1024-row dd_tile_kernel tiles inside it (old_n) are marked kTileSkip or ~0u.
template <int R, int MODE>
__global__ void __launch_bounds__(kRT, 1024 / kRT) rows_kernel(const __grid_constant__ Args A, uint32_t* __restrict__ old_n) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  RowSmem<R>& S = *reinterpret_cast<RowSmem<R>*>(smem_raw);
  constexpr int kRows = kRT * R;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (A.abort_flag && *A.abort_flag) return;  // this attempt is discarded (ddm.cu retries with LSB)
  const uint32_t tile = blockIdx.x;
  const uint64_t j0 = (uint64_t)tile * kRows;
  const uint32_t nrows = (uint32_t)umin64(kRows, A.m - j0);
  if (tid == 0) {
    S.rbmax = 0;
    S.nout = 0;
    S.ovf = 0;
  }
  // 1. widened row boxes (tile-row order), their dims-1/2 bounds and max lengths
  const float kInf = __int_as_float(0x7f800000);
  float mn1 = kInf, mx1 = -kInf, ml1 = 0.0f, mn2 = kInf, mx2 = -kInf, ml2 = 0.0f;
  uint32_t rbmax = 0;
  float4 ub[R];  // this thread's rows r = tid + i kRT, binned below
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const uint32_t r = tid + i * kRT;
    S.rcnt[r] = 0;
    ub[i] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
    if (r >= nrows) continue;
    const uint64_t j = j0 + r;
    const float4 u = row_box(A, j);
    ub[i] = u;
    const double a0 = key_to_f64(A.ulo_key[j]);
    const double b0 = A.uhi ? key_to_f64(A.uhi[j]) : A.upd.hi[0][A.ulo_id[j]];
    S.rbox0[r] = make_float2(__double2float_rd(a0), __double2float_ru(b0));
    mn1 = fminf(mn1, u.x); mx1 = fmaxf(mx1, u.x); ml1 = fmaxf(ml1, __fsub_ru(u.y, u.x));
    mn2 = fminf(mn2, u.z); mx2 = fmaxf(mx2, u.z); ml2 = fmaxf(ml2, __fsub_ru(u.w, u.z));
    if (!A.tile_rk) {
      const uint32_t rb = A.r_b[j];
      rbmax = rb > rbmax ? rb : rbmax;
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    mn1 = fminf(mn1, __shfl_xor_sync(kFull, mn1, o));
    mx1 = fmaxf(mx1, __shfl_xor_sync(kFull, mx1, o));
    ml1 = fmaxf(ml1, __shfl_xor_sync(kFull, ml1, o));
    mn2 = fminf(mn2, __shfl_xor_sync(kFull, mn2, o));
    mx2 = fmaxf(mx2, __shfl_xor_sync(kFull, mx2, o));
    ml2 = fmaxf(ml2, __shfl_xor_sync(kFull, ml2, o));
  }
  rbmax = __reduce_max_sync(kFull, rbmax);
  if (lane == 0) {
    S.red[warp] = mn1; S.red[kRW + warp] = mx1; S.red[2 * kRW + warp] = ml1;
    S.red[3 * kRW + warp] = mn2; S.red[4 * kRW + warp] = mx2; S.red[5 * kRW + warp] = ml2;
  }
  __syncthreads();
  if (lane == 0) atomicMax(&S.rbmax, A.tile_rk ? A.tile_rk[2 * tile + 1] : rbmax);
  for (int w = 0; w < kRW; ++w) {
    mn1 = fminf(mn1, S.red[w]);
    mx1 = fmaxf(mx1, S.red[kRW + w]);
    ml1 = fmaxf(ml1, S.red[2 * kRW + w]);
    mn2 = fminf(mn2, S.red[3 * kRW + w]);
    mx2 = fmaxf(mx2, S.red[4 * kRW + w]);
    ml2 = fmaxf(ml2, S.red[5 * kRW + w]);
  }
  // 2. cells of the rows: G1 x G2 = kRows (d = 2: one dim-2 bin); counting
  // sort of the row indices by cell (the order inside a cell is irrelevant:
  // counts do not depend on it and the place pass orders every row)
  int g1 = kRows, g2 = 1;
  if (A.d > 2) {
    g1 = 1;
    while (g1 * g1 < kRows) g1 <<= 1;
    g2 = kRows / g1;
  }
  RBins B1, B2;
  B1.init(mn1, mx1, g1);
  B2.init(mn2, mx2, g2);
  int cell[R];
#pragma unroll
  for (int i = 0; i < R; ++i) {
    cell[i] = B2(ub[i].z) * g1 + B1(ub[i].x);
    if (tid + i * kRT < nrows) atomicAdd(&S.rcnt[cell[i]], 1u);
  }
  __syncthreads();
  {
    constexpr int kPer = kRows / kRT;  // = R cells per thread
    uint32_t v[kPer], sum = 0;
#pragma unroll
    for (int c = 0; c < kPer; ++c) { v[c] = S.rcnt[tid * kPer + c]; sum += v[c]; }
    uint32_t total;
    uint32_t ex = block_excl_scan<kRT, uint32_t>(sum, S.scan32, &total);
#pragma unroll
    for (int c = 0; c < kPer; ++c) {
      S.cstart[tid * kPer + c] = (uint16_t)ex;
      S.rcnt[tid * kPer + c] = ex;
      ex += v[c];
    }
    if (tid == 0) S.cstart[kRows] = (uint16_t)total;
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const uint32_t r = tid + i * kRT;
    if (r >= nrows) continue;
    const uint32_t k = atomicAdd(&S.rcnt[cell[i]], 1u);
    S.rrow[k] = (uint16_t)r;
    S.cbox[k] = ub[i];
  }
  __syncthreads();
  for (uint32_t r = tid; r < (uint32_t)kRows; r += kRT) S.rcnt[r] = 0;
  __syncthreads();
  const uint32_t rbm = S.rbmax;
  const bool sure_ok = A.d <= 3;  // dims beyond 2 have no float boxes: always the exact test
  // 3. candidates: A_t (CTA-wide backward walk over Slo, windows of kWin
  // positions, runs of 32^L positions whose block max < x_t skipped), then the
  // Slo slice [rl0, rbmax) straight from global memory
  uint32_t nl = 0;
  const uint64_t x = A.ulo_key[j0];
  const uint64_t rl0 = A.tile_rk ? A.tile_rk[2 * tile] : A.r_lo[j0];
  // the walk ends after |A_t| = stab(x_t) members (I4, from the count pass),
  // or -- row-indexed calls without a count pass -- where the prefix maximum
  // of slo_hi drops below x_t (nothing earlier can be a member)
  uint32_t rem = A.tile_rk ? ~0u : A.cnt0[j0] - (A.r_b[j0] - (uint32_t)rl0);
  int64_t hi_excl = (int64_t)rl0;
  uint32_t fill = 0;  // A_t members staged in fpos (a few walk windows per batch)
  static_assert(kWin % kRT == 0, "whole walk window positions per thread");
  while (rem && hi_excl > 0) {
    const int64_t i = hi_excl - 1;
    if (A.tile_rk) {  // max(slo_hi[0..i]) < x: no member at or before i
      const uint64_t pw = __ldg(A.pmw + i), pb = __ldg(A.pmb + (i >> 10));
      if ((pw > pb ? pw : pb) < x) break;
    }
    if (((i + 1) & (kWin - 1)) == 0) {
      const int L = match::skip_levels(A.T, i, x);
      if (L >= 2) { hi_excl -= (int64_t)1 << (5 * L); continue; }
    }
    const int64_t base = i & ~(int64_t)(kWin - 1);
    constexpr int kPW = kWin / kRT;  // window positions per thread
    bool mem[kPW];
    uint32_t c = 0;
#pragma unroll
    for (int u = 0; u < kPW; ++u) {
      const int64_t pp = base + tid * kPW + u;
      mem[u] = pp < hi_excl && A.T.lvl[0][pp] >= x;
      c += mem[u];
    }
    uint32_t total;
    uint32_t o = fill + block_excl_scan<kRT, uint32_t>(c, S.scan32, &total);
#pragma unroll
    for (int u = 0; u < kPW; ++u)
      if (mem[u]) S.fpos[o++] = (uint32_t)(base + tid * kPW + u);
    fill += total;
    rem = total < rem ? rem - total : 0;
    hi_excl = base;
    if (fill + kWin > (uint32_t)kRowFpos || !(rem && hi_excl > 0)) {  // (block-uniform) a batch of windows
      __syncthreads();
      for (uint32_t s0 = 0; s0 < fill; s0 += kRT) {  // (warp-uniform trip count)
        if (s0 + tid < fill)
          rows_candidate<R, MODE>(A, S, B1, B2, g1, ml1, ml2, sure_ok, S.fpos[s0 + tid], nl, j0, tile);
        rows_flush_warp<R, MODE>(A, S, nl, j0, tile, sure_ok, false);
      }
      fill = 0;
      __syncthreads();  // fpos is rewritten by the next windows
    }
  }
  if (fill) {  // (the walk ended on a skip with members still staged)
    __syncthreads();
    for (uint32_t s0 = 0; s0 < fill; s0 += kRT) {
      if (s0 + tid < fill)
        rows_candidate<R, MODE>(A, S, B1, B2, g1, ml1, ml2, sure_ok, S.fpos[s0 + tid], nl, j0, tile);
      rows_flush_warp<R, MODE>(A, S, nl, j0, tile, sure_ok, false);
    }
  }
  for (uint64_t p0 = rl0; p0 < rbm; p0 += kRT) {  // (warp-uniform trip count)
    if (p0 + tid < rbm)
      rows_candidate<R, MODE>(A, S, B1, B2, g1, ml1, ml2, sure_ok, (uint32_t)(p0 + tid), nl, j0, tile);
    rows_flush_warp<R, MODE>(A, S, nl, j0, tile, sure_ok, false);
  }
  rows_flush_warp<R, MODE>(A, S, nl, j0, tile, sure_ok, true);
  __syncthreads();
  // 4. row counts, 256-row tile sums, staging state
  for (uint32_t r = tid; r < nrows; r += kRT) A.cnt_out[j0 + r] = S.rcnt[r];
  for (uint32_t t = warp; t * 256 < nrows; t += kRW) {  // a warp per 256-row tile
    uint32_t sum = 0;
    for (uint32_t r = t * 256 + lane; r < t * 256 + 256 && r < nrows; r += 32) sum += S.rcnt[r];
    sum = __reduce_add_sync(kFull, sum);
    if (lane == 0) A.tile_sum[(j0 >> 8) + t] = sum;
  }
  if (MODE == kModeStage && tid == 0) {
    A.stage_n[tile] = S.ovf ? ~0u : S.nout;
    if (S.ovf && A.ovf_any) atomicOr(A.ovf_any, 1u);
    constexpr int kOld = kRows / (kThreads * 4);  // dd_tile_kernel<4> tiles per row tile
    for (int t = 0; t < kOld; ++t)
      if ((j0 >> 10) + t < (A.m + 1023) / 1024) old_n[(j0 >> 10) + t] = S.ovf ? ~0u : kTileSkip;
  }
}

// Place pass of rows_kernel's stage pass: each tile's staged hits grouped by
// row (counting sort on the row index), every row ordered by sub id, written
// at its offset.  Overflowed tiles (stage_n == ~0u) are left to the direct
// place pass of dd_tile_kernel.
template <int R>
__global__ void __launch_bounds__(kRT, 1) rows_place_kernel(const __grid_constant__ Args A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int kRows = kRT * R;
  constexpr uint32_t kCapT = rows_stage_cap<R>();
  uint32_t* sid = reinterpret_cast<uint32_t*>(smem_raw);  // [kCapT]
  uint32_t* cur = sid + kCapT;                            // [kRows]
  __shared__ uint64_t scan64[kRW + 1];
  const int tid = threadIdx.x;
  if (A.abort_flag && *A.abort_flag) return;
  const uint32_t tile = blockIdx.x;
  const uint32_t nst = A.stage_n[tile];
  if (nst == ~0u) return;
  const uint64_t j0 = (uint64_t)tile * kRows;
  const uint64_t t0 = A.tile_off[j0 >> 8];
  uint64_t off[R];
#pragma unroll
  for (int q = 0; q < R; ++q) {  // row q*kRT + tid (256-row tiles never straddle: kRT % 256 == 0)
    const uint64_t j = j0 + (uint64_t)q * kRT + tid;
    const bool valid = j < A.m;
    const uint32_t c = valid ? A.cnt[j] : 0u;
    uint64_t e = c;  // exclusive scan inside the 256-row tile: warp scan + the tile's earlier warps
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t t = __shfl_up_sync(kFull, e, o);
      if ((tid & 31) >= o) e += t;
    }
    if ((tid & 31) == 31) scan64[tid >> 5] = e;
    e -= c;
    __syncthreads();
    for (int w = (tid >> 5) & ~7; w < (tid >> 5); ++w) e += scan64[w];
    __syncthreads();
    off[q] = valid ? A.tile_off[j >> 8] + e : 0;
    cur[q * kRT + tid] = (uint32_t)(off[q] - t0);
  }
  __syncthreads();
  for (uint32_t e = tid; e < nst; e += kRT) {
    const uint2 h = A.stage[(uint64_t)tile * kCapT + e];
    sid[atomicAdd(&cur[h.y >> 16], 1u)] = h.x;
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < R; ++q) {
    const uint64_t j = j0 + (uint64_t)q * kRT + tid;
    if (j >= A.m) continue;
    const uint32_t lo = (uint32_t)(off[q] - t0), hi = cur[q * kRT + tid];
    for (uint32_t x = lo + 1; x < hi; ++x) {
      const uint32_t v = sid[x];
      uint32_t y = x;
      while (y > lo && sid[y - 1] > v) { sid[y] = sid[y - 1]; --y; }
      sid[y] = v;
    }
    if (hi > lo) {
      const uint32_t lid = A.ulo_id[j];
      const uint32_t uid = A.upd_map ? A.upd_map[lid] : lid;
      for (uint32_t x = lo; x < hi; ++x)
        if (t0 + x < A.capacity) A.pairs[t0 + x] = make_uint2(sid[x], uid);
    }
  }
}
template <int R>
constexpr size_t rows_place_smem() { return sizeof(uint32_t) * (rows_stage_cap<R>() + kRT * R); }

}  // namespace dd
}  // namespace ddm
