// events.cuh -- the event-order variant of the sweep: the
// GPU analogue of the paper's own parallel algorithm, Alg. 5 + 6
// (P:501-737), kept as an independent cross-check of the rank-difference
// path (match.cuh).  Semantics are Alg. 4's: every pair is reported once, at
// the EARLIER of its two upper endpoints, by the owner of that endpoint.
//
//  T  = all 2(n+m) endpoints sorted by (coord, is_upper, kind, id) -- one
//       stable sort of [S lowers | U lowers | S uppers | U uppers] on the
//       coordinate key (SURVEY App. A "stable-layout trick"; R1 tie order).
//  code[t] = is_upper << 31 | kind << 30 | id   (kind 0 = subscription)
//  hp[t]   = for a lower endpoint, the position in T of its upper endpoint;
//            0 for an upper endpoint.  x (lower at t) is active at s iff
//            t < s < hp[t].
//  Segments T_p of kSeg endpoints (Alg. 5 l.6).  SubSet[p] / UpdSet[p], the
//  sets the sequential sweep holds at the start of T_p (Alg. 6), have the
//  combined size |SubSet[p]| + |UpdSet[p]| = #lowers before start_p -
//  #uppers before start_p: Alg. 6's combine in counting form, an exclusive
//  scan of the per-segment upper-endpoint counts.  Their members -- the
//  lowers before start_p with hp >= start_p -- are collected by a backward
//  walk over T with block-max skips on hp that stops after exactly that many
//  members (the set-valued prefix of Alg. 6, materialised per segment on
//  demand instead of by a serial master).
//  Within T_p every upper endpoint u (position t) of kind k emits (Alg. 5
//  l.14-16 / l.22-24) its pairs with the other kind's active set at t:
//  members of the initial sets with hp > t, and lowers at s in [start_p, t)
//  with hp[s] > t (a backward scan stopped by the in-segment prefix maximum
//  of hp).  d > 1: a candidate is kept iff the 1-D test holds on every other
//  dimension.  Output: "Atomic L <- L u {...}":
//  per-thread batches appended by atomics, so the order is unspecified
//  (ddm_sort_pairs canonicalises); a count pass gives K first.
#pragma once
#include "common.cuh"

namespace ddm {
namespace ev {

constexpr int kThreads = 256;
constexpr int kItems = 8;
constexpr int kSeg = kThreads * kItems;  // endpoints per segment (one CTA)
constexpr int kInitCap = 2048;           // initial-set members staged per chunk
constexpr uint32_t kUpper = 1u << 31, kKindU = 1u << 30, kIdMask = (1u << 30) - 1;

struct Coords {  // all dimensions of both sides (d > 1 filter)
  const double* sub_lo[8];
  const double* sub_hi[8];
  const double* upd_lo[8];
  const double* upd_hi[8];
  int d;
};

// keys / codes of the 2(n+m) endpoints in the stable-layout order
__global__ void __launch_bounds__(256) build_kernel(const double* __restrict__ sl, const double* __restrict__ sh,
                                                    const double* __restrict__ ul, const double* __restrict__ uh,
                                                    uint64_t n, uint64_t m, uint64_t* __restrict__ key,
                                                    uint32_t* __restrict__ code) {
  const uint64_t N2 = 2 * (n + m);
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N2; i += (uint64_t)gridDim.x * blockDim.x) {
    double x;
    uint32_t c;
    if (i < n) { x = sl[i]; c = (uint32_t)i; }
    else if (i < n + m) { x = ul[i - n]; c = kKindU | (uint32_t)(i - n); }
    else if (i < 2 * n + m) { x = sh[i - n - m]; c = kUpper | (uint32_t)(i - n - m); }
    else { x = uh[i - 2 * n - m]; c = kUpper | kKindU | (uint32_t)(i - 2 * n - m); }
    key[i] = f64_key(x);
    code[i] = c;
  }
}

// posH[kind][id] = position of the upper endpoint; per-segment upper counts
__global__ void __launch_bounds__(256) pos_kernel(const uint32_t* __restrict__ code, uint64_t N2, uint64_t n,
                                                  uint32_t* __restrict__ posH, uint64_t* __restrict__ seg_uppers) {
  __shared__ uint32_t cnt;
  if (threadIdx.x == 0) cnt = 0;
  __syncthreads();
  // one CTA per segment
  const uint64_t t0 = (uint64_t)blockIdx.x * kSeg;
  uint32_t mine = 0;
  for (int k = 0; k < kItems; ++k) {
    const uint64_t t = t0 + (uint64_t)k * kThreads + threadIdx.x;
    if (t < N2) {
      const uint32_t c = code[t];
      if (c & kUpper) {
        posH[((c & kKindU) ? n : 0) + (c & kIdMask)] = (uint32_t)t;
        ++mine;
      }
    }
  }
  mine = warp_sum<uint32_t>(mine);
  if ((threadIdx.x & 31) == 0) atomicAdd(&cnt, mine);
  __syncthreads();
  if (threadIdx.x == 0) seg_uppers[blockIdx.x] = cnt;
}

// hp[t] for every position (lowers: partner upper position, uppers: 0) and
// level 1 of its block-max tree
__global__ void __launch_bounds__(256) hp_kernel(const uint32_t* __restrict__ code, uint64_t N2, uint64_t n,
                                                 const uint32_t* __restrict__ posH, uint64_t* __restrict__ hp,
                                                 uint64_t* __restrict__ lvl1) {
  const uint64_t N2p = (N2 + 31) & ~31ull;
  for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < N2p; t += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t h = 0;
    if (t < N2) {
      const uint32_t c = code[t];
      if (!(c & kUpper)) h = posH[((c & kKindU) ? n : 0) + (c & kIdMask)];
      hp[t] = h;
    }
    h = warp_max_u64(h);
    if (lvl1 && (threadIdx.x & 31) == 0) lvl1[t >> 5] = h;
  }
}

struct Args {
  const uint32_t* code;  // T
  const uint64_t* hp;
  MaxTree T;             // block maxima of hp
  const uint64_t* ub;    // #upper endpoints before each segment (exclusive scan)
  uint64_t N2;
  Coords X;
  uint2* pairs;          // emit pass: {sub, upd}
  uint64_t capacity;
  unsigned long long* cursor;  // emit: next free output slot; count: K
};

struct Smem {
  uint32_t code[kSeg];
  uint64_t hp[kSeg];
  uint64_t pmx[kSeg];  // inclusive prefix max of hp within the segment
  uint32_t icode[kInitCap];
  uint64_t ihp[kInitCap];
  uint32_t icnt;       // members in the current chunk
  int64_t walk_pos;    // the initial-set walk's next position
  uint32_t red[kThreads / 32];
};

__device__ __forceinline__ bool other_dims(const Coords& X, uint32_t s, uint32_t u) {
  for (int k = 1; k < X.d; ++k)
    if (!(X.sub_lo[k][s] <= X.upd_hi[k][u] && X.upd_lo[k][u] <= X.sub_hi[k][s])) return false;
  return true;
}

// the pair of the upper endpoint `cu` with the active lower endpoint `cx`
template <bool EMIT>
__device__ __forceinline__ void report(const Args& A, uint32_t cu, uint32_t cx, uint32_t& cnt, uint64_t* buf,
                                       int& nb) {
  const bool u_is_sub = !(cu & kKindU);
  const uint32_t s = u_is_sub ? (cu & kIdMask) : (cx & kIdMask);
  const uint32_t u = u_is_sub ? (cx & kIdMask) : (cu & kIdMask);
  if (A.X.d > 1 && !other_dims(A.X, s, u)) return;
  ++cnt;
  if (EMIT) buf[nb++] = ((uint64_t)u << 32) | s;
}

// append the thread's buffered pairs (one atomic per flush)
__device__ __forceinline__ void flush(const Args& A, uint64_t* buf, int& nb) {
  if (nb == 0) return;
  uint64_t o = atomicAdd(A.cursor, (unsigned long long)nb);
  for (int i = 0; i < nb; ++i, ++o)
    if (o < A.capacity) A.pairs[o] = make_uint2((uint32_t)buf[i], (uint32_t)(buf[i] >> 32));
  nb = 0;
}

template <bool EMIT>
__global__ void __launch_bounds__(kThreads) segment_kernel(const __grid_constant__ Args A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem& S = *reinterpret_cast<Smem*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint64_t start = (uint64_t)blockIdx.x * kSeg;
  const uint32_t len = (uint32_t)umin64(kSeg, A.N2 - start);
  for (uint32_t k = tid; k < kSeg; k += kThreads) {
    S.code[k] = k < len ? A.code[start + k] : kUpper;  // (padding: uppers never active)
    S.hp[k] = k < len ? A.hp[start + k] : 0;
  }
  __syncthreads();
  // in-segment inclusive prefix max of hp (thread-contiguous runs + warp scans)
  {
    uint64_t run[kItems];
    uint64_t mx = 0;
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
      const uint64_t h = S.hp[tid * kItems + i];
      mx = h > mx ? h : mx;
      run[i] = mx;
    }
    uint64_t inc = mx;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(kFull, inc, o);
      if (lane >= o && y > inc) inc = y;
    }
    uint64_t ex = __shfl_up_sync(kFull, inc, 1);
    if (lane == 0) ex = 0;
    __shared__ uint64_t wmax[kThreads / 32];
    if (lane == 31) wmax[warp] = inc;
    __syncthreads();
    for (int w = 0; w < warp; ++w) ex = wmax[w] > ex ? wmax[w] : ex;
#pragma unroll
    for (int i = 0; i < kItems; ++i) S.pmx[tid * kItems + i] = run[i] > ex ? run[i] : ex;
  }
  __syncthreads();  // pmx complete before any scan reads it
  uint32_t cnt = 0;
  uint64_t buf[8];
  int nb = 0;
  // (1) pairs with the initial sets SubSet[p] u UpdSet[p], chunk by chunk
  // |SubSet[p]| + |UpdSet[p]| = #lowers before start - #uppers before start
  const uint64_t total = start - 2 * A.ub[blockIdx.x];
  uint64_t done = 0;
  if (tid == 0) S.walk_pos = (int64_t)start - 1;
  while (done < total) {
    __syncthreads();
    if (warp == 0) {  // collect up to kInitCap members: lowers before start with hp >= start
      uint32_t got = 0;
      int64_t i = S.walk_pos;  // next position to examine (walking down)
      const uint32_t want = (uint32_t)umin64(kInitCap, total - done);
      while (got < want && i >= 0) {
        int L = 0;  // aligned runs of 32^L positions whose max hp < start hold no member
        while (L < A.T.levels) {
          const int sh = 5 * (L + 1);
          if ((((uint64_t)i + 1) & ((1ull << sh) - 1)) != 0) break;
          if (A.T.lvl[L + 1][(uint64_t)i >> sh] >= start) break;
          ++L;
        }
        if (L) { i -= (int64_t)1 << (5 * L); continue; }
        const int64_t q = i - lane;  // 32 positions i-31 .. i
        bool mem = false;
        uint32_t c = 0;
        uint64_t h = 0;
        if (q >= 0) {
          h = A.hp[q];
          c = A.code[q];
          mem = !(c & kUpper) && h >= start;
        }
        const unsigned bal = __ballot_sync(kFull, mem);
        const uint32_t room = want - got;
        unsigned keep = bal;
        int64_t next = i - 32;
        if ((uint32_t)__popc(bal) > room) {  // keep the first `room` (highest positions)
          unsigned b = bal;
          for (uint32_t r = 0; r < room; ++r) b &= b - 1;
          keep = bal & ~b;
          next = i - (__ffs(b) - 1);  // resume at the first member not kept
        }
        if ((keep >> lane) & 1u) {
          const uint32_t slot = got + __popc(keep & lanemask_lt());
          S.icode[slot] = c;
          S.ihp[slot] = h;
        }
        got += __popc(keep);
        i = next;
      }
      if (lane == 0) {
        S.icnt = got;
        S.walk_pos = i;
      }
    }
    __syncthreads();
    const uint32_t ic = S.icnt;
    if (ic == 0) break;  // (cannot happen when the counts are consistent)
#pragma unroll
    for (int it = 0; it < kItems; ++it) {
      const uint32_t k = tid * kItems + it;
      const uint32_t cu = S.code[k];
      if (k >= len || !(cu & kUpper)) continue;
      const uint64_t t = start + k;
      for (uint32_t x = 0; x < ic; ++x) {
        const uint32_t cx = S.icode[x];
        if (((cx ^ cu) & kKindU) && S.ihp[x] > t) {
          report<EMIT>(A, cu, cx, cnt, buf, nb);
          if (EMIT && nb == 8) flush(A, buf, nb);
        }
      }
    }
    done += ic;
  }
  // (2) pairs with lowers inside the segment before the upper endpoint
#pragma unroll
  for (int it = 0; it < kItems; ++it) {
    const uint32_t k = tid * kItems + it;
    const uint32_t cu = S.code[k];
    if (k >= len || !(cu & kUpper)) continue;
    const uint64_t t = start + k;
    for (int32_t s = (int32_t)k - 1; s >= 0 && S.pmx[s] > t; --s) {
      const uint32_t cx = S.code[s];
      if (!(cx & kUpper) && ((cx ^ cu) & kKindU) && S.hp[s] > t) {
        report<EMIT>(A, cu, cx, cnt, buf, nb);
        if (EMIT && nb == 8) flush(A, buf, nb);
      }
    }
  }
  if (EMIT) {
    flush(A, buf, nb);
  } else {
    cnt = warp_sum<uint32_t>(cnt);
    if (lane == 0 && cnt) atomicAdd(A.cursor, (unsigned long long)cnt);
  }
}

}  // namespace ev
}  // namespace ddm
