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
// bounds rounded down, upper bounds rounded up.
__global__ void __launch_bounds__(256) box_kernel(const double* __restrict__ sdims, int d, uint64_t n,
                                                  float4* __restrict__ box12,
                                                  const uint32_t* __restrict__ abort_flag) {
  if (abort_flag && *abort_flag) return;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
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
};

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
// read in sweep order (sdims / udims), so these reads stay local.
__device__ __forceinline__ bool exact_hit(const Args& A, uint32_t p, uint64_t j, uint32_t lid) {
  const uint64_t b = A.uhi ? A.uhi[j] : f64_key(A.upd.hi[0][lid]);
  if (!(A.slo_key[p] <= b && A.T.lvl[0][p] >= A.ulo_key[j])) return false;  // dim 0 (keys)
  for (int k = 1; k < A.d; ++k) {
    const double slo = A.sdims[(uint64_t)(k - 1) * 2 * A.n + p];
    const double shi = A.sdims[(uint64_t)(k - 1) * 2 * A.n + A.n + p];
    const double ulo = A.udims[(uint64_t)(k - 1) * 2 * A.m + j];
    const double uhi = A.udims[(uint64_t)(k - 1) * 2 * A.m + A.m + j];
    if (!(slo <= uhi && ulo <= shi)) return false;
  }
  return true;
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
      float4 u;
      u.x = __double2float_rd(A.udims[j]);
      u.y = __double2float_ru(A.udims[A.m + j]);
      u.z = A.d > 2 ? __double2float_rd(A.udims[2 * A.m + j]) : -kInf;
      u.w = A.d > 2 ? __double2float_ru(A.udims[3 * A.m + j]) : kInf;
      S.rbox[q * kThreads + tid] = u;
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

}  // namespace dd
}  // namespace ddm
