// ddm.cu -- host side of libddm: the C ABI of include/ddm.h and the launch
// orchestration of the sort-based matching pipeline on the caller's stream.
//
// Pipeline for d = 1:
//   validate_hist(subs)  -> onesweep x8 (Slo: key+id, from float64)
//                        -> onesweep x8 (Shi: keys)     -> gather slo_hi + block maxima
//   validate_hist(upds)  -> onesweep x8 (Ulo: key+id)
//   count (rank differences, b gathered in-kernel) -> scan of the 256-row tile sums
//   one 16-byte D2H {K, error word}; capacity check
//   emit (stab part from the sweep state + contiguous range part)
// The subscription half forms the byte-copyable "index" (multi-GPU: built by
// one rank and broadcast).
#include <atomic>
#include <cmath>
#include <memory>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "../../include/ddm.h"
#include "common.cuh"
#include "match.cuh"
#include "radix.cuh"
#include "msd.cuh"
#include "dd.cuh"
#include "events.cuh"
#include "dyn.cuh"
#include "slab.cuh"

using namespace ddm;

namespace {

std::atomic<uint64_t> g_launches{0};
std::atomic<int> g_last_cuda{0};

// Optional per-launch timing with CUDA events on the launching stream
// (ddm_profile_enable / ddm_profile_read): bench.py uses it to measure the
// dominant kernel's average duration live inside its timed region.
struct ProfRec {
  const char* name;
  double bytes;
  int e0, e1;
};
struct Prof {
  bool on = false;
  std::vector<cudaEvent_t> ev;
  std::vector<ProfRec> recs;
  int next = 0;
  int take() {
    if (next >= (int)ev.size()) {
      cudaEvent_t e;
      if (cudaEventCreate(&e) != cudaSuccess) return -1;
      ev.push_back(e);
    }
    return next++;
  }
} g_prof;
std::mutex g_prof_mu;

bool serial_env() {
  static const bool serial = getenv("DDM_SERIAL") != nullptr;
  return serial;
}
// DDM_CHAINS=1: the sort chains share the call's stream (graphs stay on)
bool one_chain_env() {
  static const bool one = [] {
    const char* e = getenv("DDM_CHAINS");
    return e && atoi(e) == 1;
  }();
  return one;
}
// Set for the duration of a walk-form call: with only two sort chains left
// (Slo, Ulo) one stream and full-occupancy persistent passes beat running
// them side by side (measured c3: 6.07 vs 6.47 ms; c5: 71.8 vs 80.0 ms).
thread_local bool t_one_chain = false;
struct OneChain {
  bool prev;
  explicit OneChain(bool on) : prev(t_one_chain) { t_one_chain = on; }
  ~OneChain() { t_one_chain = prev; }
};
// the sort chains run on side streams (not profiling, not DDM_SERIAL)
bool chains_concurrent() { return !(serial_env() || g_prof.on || one_chain_env() || t_one_chain); }

inline int prof_begin(cudaStream_t st) {
  if (!g_prof.on) return -1;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  const int e = g_prof.take();
  if (e >= 0) cudaEventRecord(g_prof.ev[e], st);
  return e;
}
inline void prof_end(const char* name, double bytes, cudaStream_t st, int e0) {
  if (e0 < 0) return;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  const int e1 = g_prof.take();
  if (e1 < 0) return;
  cudaEventRecord(g_prof.ev[e1], st);
  g_prof.recs.push_back({name, bytes, e0, e1});
}

// NAME: kernel class; BYTES: algorithmic DRAM bytes of this launch
thread_local const char* t_last_launch = "";  // (DDM_DEBUG: named in launch errors)
#define DDM_LAUNCH(NAME, BYTES, ST, ...)                  \
  do {                                                    \
    t_last_launch = NAME;                                 \
    const int e0_ = prof_begin(ST);                       \
    __VA_ARGS__;                                          \
    prof_end(NAME, (double)(BYTES), ST, e0_);             \
    g_launches.fetch_add(1, std::memory_order_relaxed);   \
  } while (0)

#define DDM_CUDA(call)                                                                   \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess) {                                                             \
      g_last_cuda.store((int)e_);                                                        \
      if (getenv("DDM_DEBUG")) fprintf(stderr, "libddm: %s at ddm.cu:%d (%s)\n", cudaGetErrorString(e_), \
                                       __LINE__, #call);                                 \
      return DDM_ERR_CUDA;                                                               \
    }                                                                                    \
  } while (0)

#define DDM_CUDA_RET(call) DDM_CUDA(call)

inline ddm_status check_launch() {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    if (getenv("DDM_DEBUG")) fprintf(stderr, "libddm: launch error %s (last launch: %s)\n", cudaGetErrorString(e), t_last_launch);
    g_last_cuda.store((int)e);
    return DDM_ERR_CUDA;
  }
  return DDM_OK;
}

#define DDM_TRY(x)                \
  do {                            \
    ddm_status s_ = (x);          \
    if (s_ != DDM_OK) return s_;  \
  } while (0)

// Payload records of the MSD sort: packed to 16 bytes (key + id | upper-key
// delta << 32, msd.cuh) for sorts of at least kPackMinN records, where the
// sort streams through HBM (c3: 5.55 -> 5.24 ms, c5: 66.3 -> 60.4 ms);
// smaller (L2-resident) sorts keep 20-byte records, since a delta that does
// not fit 32 bits costs a re-read of the upper bound (DDM_MSD_PACK=0/1 forces).
#ifndef DDM_MSD_PACK
#define DDM_MSD_PACK 2
#endif
constexpr uint64_t kPackMinN = 1ull << 22;
constexpr double kPackMaxUnfit = 0.15;  // no packing when more sampled deltas than this do not fit 32 bits (c3: 2 %; alpha = 100: all)
// Per-call pack decision of the subscription / update sorts (match_full's
// probe; -1: by size only), set for the duration of a call like OneChain.
struct PackHint {
  int sub = -1, upd = -1;
};
thread_local PackHint t_pack;
struct PackScope {
  PackHint prev;
  PackScope(int s, int u) : prev(t_pack) { t_pack = PackHint{s, u}; }
  ~PackScope() { t_pack = prev; }
};
inline bool pack_records(uint64_t n, int hint) {
  if (DDM_MSD_PACK != 2) return DDM_MSD_PACK != 0;
  return n >= kPackMinN && hint != 0;
}

#ifndef DDM_LS_BIG
#define DDM_LS_BIG 1
#endif
constexpr int kSMs = 148;
#ifndef DDM_DD_ROWS
#define DDM_DD_ROWS 4
#endif
constexpr int kDDRows = DDM_DD_ROWS;  // rows per thread of the d > 1 tile kernel (1024-row tiles)
#ifndef DDM_DDR_ROWS
#define DDM_DDR_ROWS 4
#endif
constexpr int kDDRRows = DDM_DDR_ROWS;  // rows per thread of the row-indexed d > 1 kernel (1024 threads: 4096-row tiles)

inline size_t a256(size_t x) { return (x + 255) & ~size_t(255); }

// A bump allocator that either measures (base == nullptr) or carves.
struct Carver {
  uint8_t* base;
  size_t used = 0;
  explicit Carver(void* b) : base(static_cast<uint8_t*>(b)) {}
  template <typename T>
  T* take(uint64_t count) {
    T* p = base ? reinterpret_cast<T*>(base + used) : nullptr;
    used += a256(sizeof(T) * (count ? count : 1));
    return p;
  }
};

// ------------------------------------------------------------ index layout

struct Index {
  uint32_t d = 1;
  uint64_t n = 0;
  int levels = 0;
  uint64_t lvl_n[kMaxLevels + 1] = {};
  uint64_t* slo_key = nullptr;
  uint32_t* slo_id = nullptr;
  uint64_t* slo_hi = nullptr;
  uint64_t* lvl[kMaxLevels + 1] = {};
  uint64_t* shi_key = nullptr;
  uint64_t* pmw = nullptr;  // prefix maxima of slo_hi within 1024-entry blocks (match.cuh tree_pm_kernel)
  uint64_t* pmb = nullptr;  // prefix maxima of slo_hi before each 1024-entry block
  uint64_t* pmc = nullptr;  // maxima of 8192-block chunks (scratch of the pmb scan)
  uint64_t nb = 0;          // number of 1024-entry blocks
  double* sdims = nullptr;
  float4* box12 = nullptr;  // d > 1: widened float32 boxes (dims 1, 2) in Slo order (dd.cuh)
  float2* box0 = nullptr;   // d > 1: widened float32 dim-0 boxes in Slo order (dd.cuh)
  uint32_t* tick = nullptr;  // ticket of match::tree_levels_kernel (scratch)
  size_t bytes = 0;
};

Index index_layout(uint32_t d, uint64_t n, void* base) {
  Index I;
  I.d = d;
  I.n = n;
  Carver c(base);
  I.slo_key = c.take<uint64_t>(n);
  I.slo_id = c.take<uint32_t>(n);
  I.slo_hi = c.take<uint64_t>(n);
  I.lvl[0] = I.slo_hi;
  I.lvl_n[0] = n;
  uint64_t sz = n;
  while (sz > 1 && I.levels < kMaxLevels) {
    sz = (sz + 31) / 32;
    ++I.levels;
    I.lvl_n[I.levels] = sz;
    I.lvl[I.levels] = c.take<uint64_t>(sz);
  }
  I.shi_key = c.take<uint64_t>(n);
  I.nb = (n + match::kPmBlock - 1) / match::kPmBlock;
  I.pmw = c.take<uint64_t>(n);
  I.pmb = c.take<uint64_t>(I.nb);
  I.pmc = c.take<uint64_t>(I.nb / match::kPmChunk + 1);
  I.sdims = c.take<double>((uint64_t)2 * (d - 1) * n);
  if (d > 1) {
    I.box12 = c.take<float4>(n);
    I.box0 = c.take<float2>(n);
  }
  I.tick = c.take<uint32_t>(1);
  I.bytes = c.used;
  return I;
}

MaxTree tree_of(const Index& I) {
  MaxTree T{};
  for (int L = 0; L <= I.levels; ++L) T.lvl[L] = I.lvl[L];
  T.levels = I.levels;
  return T;
}

// ------------------------------------------------------------ sort scratch

// bucket bits of the MSD sort: ~768 records per bucket on average
int bits_for_bucket(uint64_t n, double per_bucket) {
  if (n <= per_bucket) return 1;
  const double b = std::log2((double)n / per_bucket);
  int r = (int)std::lround(b);
  return r < 1 ? 1 : r > 24 ? 24 : r;
}
// The big local sort (msd::LsBig, ~6000 records per bucket) is used when it
// saves a multisplit pass over the default (~768 per bucket): c5's 5e8
// records need 19 bucket bits (3 passes) with small buckets, 16 (2) with big.
bool msd_big(uint64_t n) {
  const int small = bits_for_bucket(n, 768.0), big = bits_for_bucket(n, 6000.0);
  return DDM_LS_BIG && (big + 7) / 8 < (small + 7) / 8;
}
int msd_bits(uint64_t n) { return bits_for_bucket(n, msd_big(n) ? 6000.0 : 768.0); }


// LSB onesweep scratch (the fallback path and the exported primitives).  The
// alternate key/value buffers are set per use (they alias an MSD chain's).
struct SortScratch {
  uint32_t* hist[3];   // [8][256] each: Slo, Shi, Ulo (or generic)
  uint32_t* starts;    // [8][256] global bin starts of the sort in flight
  uint32_t* status;    // [tiles][256]
  uint32_t* counters;  // [8]
  uint64_t* alt_keys;
  uint32_t* alt_vals;
};

SortScratch sort_scratch(Carver& c, uint64_t cap, bool own_alt) {
  SortScratch s{};
  for (int i = 0; i < 3; ++i) s.hist[i] = c.take<uint32_t>(radix::kMaxPasses * radix::kRadix);
  s.starts = c.take<uint32_t>(radix::kMaxPasses * radix::kRadix);
  s.status = c.take<uint32_t>((radix::num_tiles(cap) + 1) * radix::kRadix);
  s.counters = c.take<uint32_t>(radix::kMaxPasses);
  if (own_alt) {
    s.alt_keys = c.take<uint64_t>(cap);
    s.alt_vals = c.take<uint32_t>(cap);
  }
  return s;
}

// Scratch of one MSD sort chain: its own buffers, so the Slo, Shi and Ulo
// sorts can run concurrently on separate streams.
struct MsdScratch {
  uint32_t* dh;        // [3][256] digit histograms of the bucket id
  uint32_t* starts;    // [3][256] global digit starts
  uint32_t* status;    // [tiles][256] look-back words
  uint32_t* counters;  // [8] tile counters
  uint32_t* ccount;    // [kCoarse + 1] sampled coarse-bin population
  uint32_t* cbase;     // [kCoarse + 2] bucket map
  uint64_t* bounds;    // [spans + 1] group boundaries of the local sort
  uint64_t* k[2];      // ping-pong record buffers
  uint64_t* v64[2];
  uint32_t* v32[2];
};

MsdScratch msd_scratch(Carver& c, uint64_t cap, bool kv) {
  MsdScratch s{};
  s.dh = c.take<uint32_t>(3 * 256);
  s.starts = c.take<uint32_t>(3 * 256);
  s.status = c.take<uint32_t>(((cap + msd::kTile - 1) / msd::kTile + 1) * radix::kRadix);
  s.counters = c.take<uint32_t>(radix::kMaxPasses);
  s.ccount = c.take<uint32_t>(msd::kCoarse + 1);
  s.cbase = c.take<uint32_t>(msd::kCoarse + 2);
  s.bounds = c.take<uint64_t>(cap / msd::kSpan + 3);
  for (int i = 0; i < 2; ++i) {
    s.k[i] = c.take<uint64_t>(cap);
    if (kv) {
      s.v64[i] = c.take<uint64_t>(cap);
      s.v32[i] = c.take<uint32_t>(cap);
    }
  }
  return s;
}

// Side streams for the concurrent sort chains: per calling thread and device
// (created on first use), so concurrent callers -- and a graph capture on one
// thread -- never share a side stream with another thread's eager launches.
struct SideStreams {
  cudaStream_t s[2] = {nullptr, nullptr};
};
struct ThreadStreams {
  SideStreams side[64];
  cudaStream_t cap[64] = {};  // capture streams (run_cached)
  ~ThreadStreams() {
    for (auto& d : side)
      for (cudaStream_t x : d.s)
        if (x) cudaStreamDestroy(x);
    for (cudaStream_t x : cap)
      if (x) cudaStreamDestroy(x);
  }
};
thread_local ThreadStreams t_streams;

ddm_status side_streams(cudaStream_t out[2], cudaStream_t st) {
  // one stream while profiling (per-kernel event intervals must not overlap)
  // or when DDM_SERIAL is set (debugging)
  if (!chains_concurrent()) {
    out[0] = out[1] = st;
    return DDM_OK;
  }
  int dev = 0;
  DDM_CUDA_RET(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) return DDM_ERR_CUDA;
  SideStreams& S = t_streams.side[dev];
  for (int i = 0; i < 2; ++i) {
    if (!S.s[i]) DDM_CUDA_RET(cudaStreamCreateWithFlags(&S.s[i], cudaStreamNonBlocking));
    out[i] = S.s[i];
  }
  return DDM_OK;
}

// A side stream even in walk-form (one-chain) calls: only profiling and
// DDM_SERIAL keep everything on `st`.
ddm_status side_stream_any(cudaStream_t* out, cudaStream_t st) {
  if (serial_env() || g_prof.on) {
    *out = st;
    return DDM_OK;
  }
  int dev = 0;
  DDM_CUDA_RET(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) return DDM_ERR_CUDA;
  SideStreams& S = t_streams.side[dev];
  if (!S.s[1]) DDM_CUDA_RET(cudaStreamCreateWithFlags(&S.s[1], cudaStreamNonBlocking));
  *out = S.s[1];
  return DDM_OK;
}

// `to` waits for everything enqueued on `from` so far.
ddm_status stream_join(cudaStream_t to, cudaStream_t from) {
  if (to == from) return DDM_OK;
  cudaEvent_t e;
  DDM_CUDA_RET(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  const cudaError_t r1 = cudaEventRecord(e, from);
  const cudaError_t r2 = r1 == cudaSuccess ? cudaStreamWaitEvent(to, e, 0) : r1;
  cudaEventDestroy(e);  // released once the recorded work completes
  DDM_CUDA_RET(r2);
  return DDM_OK;
}

struct Misc {  // device-side results read back with one copy
  uint64_t K;
  uint32_t err;
  uint32_t overflow;  // an MSD bucket exceeded shared memory: redo with the LSB sort
  uint32_t dd_ovf;    // d > 1 row-indexed stage pass: some tile's staging slot overflowed
  uint32_t pad_;
};

constexpr ddm_status kRetryLSB = (ddm_status)100;  // internal



struct MatchWs {
  uint64_t* ulo_key;
  uint64_t* uhi;       // upper keys in Ulo order (MSD path)
  uint32_t* ulo_id;
  uint32_t* r_lo;
  uint32_t* r_b;
  uint32_t* cnt0;      // dim-0 counts (rank differences)
  uint32_t* cnt;       // d > 1: filtered counts
  uint32_t* fstab;     // d > 1: filtered stab counts
  uint64_t* tile_sum;  // per 256-row tile count sums
  uint64_t* tile_off;  // their exclusive scan: output offset of each row tile
  uint64_t* scan_status;
  uint64_t* part;
  uint2* dd_stage;      // d > 1 stage pass: per-tile staged hits
  double* udims;        // d > 1: dims 1..d-1 of the updates in Ulo order
  uint32_t* dd_stage_n; // their number per tile (~0u: overflowed)
  uint32_t* dd_stage_n2; // the same per row-indexed tile (dd::rows_kernel)
  Misc* misc;
  uint64_t* mm;        // [3][2] min/max keys (Slo, Shi, Ulo)
  double* probe;       // stab-density estimate (count-form choice)
  MsdScratch slo, shi, ulo;  // MSD chains (slo/shi only with the index scratch)
  SortScratch sort;    // LSB fallback
  size_t bytes;
};

MatchWs match_layout(uint32_t d, uint64_t n_sub, uint64_t m, void* base, bool index_scratch) {
  Carver c(base);
  MatchWs W{};
  const uint64_t rtiles = m / match::kRowTile + 2;
  W.misc = c.take<Misc>(1);
  W.mm = c.take<uint64_t>(6);
  W.probe = c.take<double>(DDM_MAX_DIMS);
  W.scan_status = c.take<uint64_t>(rtiles / (match::kScanThreads * match::kScanItems) + 2);
  W.part = c.take<uint64_t>(4 * (m / match::kCountTile + 2));
  W.tile_sum = c.take<uint64_t>(rtiles);
  W.tile_off = c.take<uint64_t>(rtiles);
  W.ulo_key = c.take<uint64_t>(m);
  W.uhi = c.take<uint64_t>(m);
  W.ulo_id = c.take<uint32_t>(m);
  W.r_lo = c.take<uint32_t>(m);
  W.r_b = c.take<uint32_t>(m);
  W.cnt0 = c.take<uint32_t>(m);
  if (d > 1) {
    W.cnt = c.take<uint32_t>(m);
    W.fstab = c.take<uint32_t>(m);
    const uint64_t dtiles = m / (dd::kThreads * kDDRows) + 1;
    const uint64_t rtiles2 = m / (dd::kRT * kDDRRows) + 1;
    const uint64_t st_old = dtiles * dd::kStageCap, st_new = rtiles2 * dd::rows_stage_cap<kDDRRows>();
    W.dd_stage = c.take<uint2>(st_old > st_new ? st_old : st_new);
    W.udims = c.take<double>((uint64_t)2 * (d - 1) * m);
    W.dd_stage_n = c.take<uint32_t>(dtiles);
    W.dd_stage_n2 = c.take<uint32_t>(rtiles2);
  }
  W.ulo = msd_scratch(c, m, true);
  if (index_scratch) {
    W.slo = msd_scratch(c, n_sub, true);
    W.shi = msd_scratch(c, n_sub, false);
  }
  W.sort = sort_scratch(c, index_scratch && n_sub > m ? n_sub : m, false);
  W.bytes = c.used;
  return W;
}

// LSB scratch whose alternate buffers alias an MSD chain's first record buffer.
SortScratch lsb_with(const SortScratch& s, const MsdScratch& m) {
  SortScratch r = s;
  r.alt_keys = m.k[0];
  r.alt_vals = m.v32[0];
  return r;
}

// ------------------------------------------------------------ radix sort driver

int g_radix_items = 0;  // items per thread of the onesweep pass (env DDM_RADIX_ITEMS)

int radix_items() {
  if (!g_radix_items) {
    const char* e = getenv("DDM_RADIX_ITEMS");
    int v = e ? atoi(e) : 0;
    g_radix_items = (v == 8 || v == 12 || v == 16) ? v : 8;
  }
  return g_radix_items;
}

template <int ITEMS, bool KV, bool F64>
void set_attr() {
  cudaFuncSetAttribute(radix::onesweep_kernel<ITEMS, KV, F64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)sizeof(radix::PassSmem<ITEMS, KV>));
}

template <int ITEMS>
void set_attrs_items() {
  set_attr<ITEMS, true, true>();
  set_attr<ITEMS, true, false>();
  set_attr<ITEMS, false, true>();
  set_attr<ITEMS, false, false>();
}

void init_attrs_once() {
  static bool done = false;
  if (done) return;
  set_attrs_items<8>();
  set_attrs_items<12>();
  set_attrs_items<16>();
  cudaFuncSetAttribute(match::count_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)match::count_smem_bytes(false));
  cudaFuncSetAttribute(match::count_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)match::count_smem_bytes(true));
  cudaFuncSetAttribute(ev::segment_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(ev::Smem));
  cudaFuncSetAttribute(ev::segment_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(ev::Smem));
  cudaFuncSetAttribute(match::emit_chunk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)sizeof(match::ChunkSmem));
  cudaFuncSetAttribute(match::emit_tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)sizeof(match::EmitTileSmem));
  cudaFuncSetAttribute(msd::msd_hist_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)msd::hist_smem_bytes(3));
  for (auto f : {(const void*)msd::msd_pass_kernel<msd::kItemsC, true, true, true>,
                 (const void*)msd::msd_pass_kernel<msd::kItemsC, true, true, false>})
    cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(msd::PassSmem<msd::kItemsC, true, true>));
  for (auto f : {(const void*)msd::msd_pass_kernel<msd::kItemsC, true, false, true>,
                 (const void*)msd::msd_pass_kernel<msd::kItemsC, true, false, false>})
    cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(msd::PassSmem<msd::kItemsC, true, false>));
  cudaFuncSetAttribute(msd::msd_pass_kernel<msd::kItems, true, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)sizeof(msd::PassSmem<msd::kItems, true, true>));
  cudaFuncSetAttribute(msd::msd_pass_kernel<msd::kItems, true, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)sizeof(msd::PassSmem<msd::kItems, true, true>));
  cudaFuncSetAttribute(msd::msd_pass_kernel<msd::kItems, true, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)sizeof(msd::PassSmem<msd::kItems, true, false>));
  cudaFuncSetAttribute(msd::msd_pass_kernel<msd::kItems, true, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)sizeof(msd::PassSmem<msd::kItems, true, false>));
  cudaFuncSetAttribute(msd::msd_pass_kernel<msd::kItemsK, false, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)sizeof(msd::PassSmem<msd::kItemsK, false, false>));
  cudaFuncSetAttribute(msd::msd_pass_kernel<msd::kItemsK, false, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)sizeof(msd::PassSmem<msd::kItemsK, false, false>));
#define DDM_LOCAL_ATTR(C, V64, V32)                                                                  \
  cudaFuncSetAttribute(msd::local_sort_kernel<C, V64, V32>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                       (int)sizeof(msd::LocalSmem<C, V64, V32>))
  DDM_LOCAL_ATTR(msd::LsSmall, true, true);
  DDM_LOCAL_ATTR(msd::LsSmall, true, false);
  DDM_LOCAL_ATTR(msd::LsSmall, false, false);
  DDM_LOCAL_ATTR(msd::LsBig, true, true);
  DDM_LOCAL_ATTR(msd::LsBig, true, false);
  DDM_LOCAL_ATTR(msd::LsBig, false, false);
#undef DDM_LOCAL_ATTR
  cudaFuncSetAttribute(dd::dd_tile_kernel<kDDRows, dd::kModeCount>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(dd::Smem<kDDRows>));
  cudaFuncSetAttribute(dd::dd_tile_kernel<kDDRows, dd::kModeStage>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(dd::Smem<kDDRows>));
  cudaFuncSetAttribute(dd::dd_tile_kernel<kDDRows, dd::kModePlace>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(dd::Smem<kDDRows>));
  cudaFuncSetAttribute(dd::rows_kernel<kDDRRows, dd::kModeCount>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(dd::RowSmem<kDDRRows>));
  cudaFuncSetAttribute(dd::rows_kernel<kDDRRows, dd::kModeStage>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(dd::RowSmem<kDDRRows>));
  cudaFuncSetAttribute(dd::rows_place_kernel<kDDRRows>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dd::rows_place_smem<kDDRRows>());
  if (const char* e = getenv("DDM_L2_FETCH")) cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)atoi(e));
  done = true;
}

template <int ITEMS>
void launch_pass(bool kv, bool f64, uint64_t tiles, cudaStream_t st, const void* ki, const uint32_t* vi,
                 uint64_t* ko, uint32_t* vo, uint64_t n, int shift, uint32_t mask, const uint32_t* starts,
                 uint32_t* status, uint32_t* counter) {
  dim3 g((unsigned)tiles);
  if (kv && f64)
    radix::onesweep_kernel<ITEMS, true, true><<<g, radix::kThreads, sizeof(radix::PassSmem<ITEMS, true>), st>>>(
        ki, vi, ko, vo, n, shift, mask, starts, status, counter);
  else if (kv)
    radix::onesweep_kernel<ITEMS, true, false><<<g, radix::kThreads, sizeof(radix::PassSmem<ITEMS, true>), st>>>(
        ki, vi, ko, vo, n, shift, mask, starts, status, counter);
  else if (f64)
    radix::onesweep_kernel<ITEMS, false, true><<<g, radix::kThreads, sizeof(radix::PassSmem<ITEMS, false>), st>>>(
        ki, vi, ko, vo, n, shift, mask, starts, status, counter);
  else
    radix::onesweep_kernel<ITEMS, false, false><<<g, radix::kThreads, sizeof(radix::PassSmem<ITEMS, false>), st>>>(
        ki, vi, ko, vo, n, shift, mask, starts, status, counter);
}

// Resident CTAs of a kernel for a persistent grid: occupancy x SM count.
unsigned persistent_grid(const void* fn, int threads, size_t smem, uint64_t work_tiles) {
  int dev = 0, sms = kSMs, per = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, threads, smem) != cudaSuccess || per < 1) per = 1;
  // While the three sort chains run concurrently, a persistent pass keeps one
  // CTA per SM and leaves the other slots to the other chains' kernels
  // (measured: 7.7 vs 7.9 ms per c3 step); DDM_PASS_CTAS_PER_SM overrides.
  static const int env_cap = [] {
    const char* e = getenv("DDM_PASS_CTAS_PER_SM");
    return e ? atoi(e) : 0;
  }();
  const int cap = env_cap > 0 ? env_cap : (chains_concurrent() ? 1 : 0);
  if (cap > 0 && per > cap) per = cap;
  const uint64_t g = (uint64_t)sms * per;
  return (unsigned)(work_tiles < g ? (work_tiles ? work_tiles : 1) : g);
}

inline unsigned grid_for(uint64_t n, int threads, int per_sm) {
  uint64_t g = (n + threads - 1) / threads;
  uint64_t cap = (uint64_t)kSMs * per_sm;
  if (g > cap) g = cap;
  return (unsigned)(g ? g : 1);
}

radix::PassList full_passes() {
  radix::PassList P{};
  P.n = 8;
  for (int p = 0; p < 8; ++p) { P.shift[p] = 8 * p; P.mask[p] = 255; }
  return P;
}

// Sort n keys (float64 encoded on the fly when src_f64) into keys_out (and
// vals_out when non-null).  `hist` must hold the per-pass histograms already
// when hist_ready; otherwise it is computed here.
ddm_status radix_sort(const void* src, bool src_f64, const uint32_t* vals_in, uint64_t* keys_out,
                      uint32_t* vals_out, uint64_t n, const radix::PassList& P, uint32_t* hist,
                      bool hist_ready, SortScratch& s, cudaStream_t st) {
  if (n == 0) return DDM_OK;
  if (P.n == 0) return DDM_ERR_INVALID_ARGUMENT;
  // the look-back words carry 30-bit per-digit prefixes (radix.cuh): larger
  // sorts would overflow into the flag bits
  if (n > radix::kValMask) return DDM_ERR_INVALID_ARGUMENT;
  init_attrs_once();
  if (!hist_ready) {
    DDM_CUDA(cudaMemsetAsync(hist, 0, sizeof(uint32_t) * radix::kMaxPasses * radix::kRadix, st));
    if (src_f64)
      DDM_LAUNCH("radix_hist", 8.0 * n, st, radix::hist_kernel<true><<<grid_for(n, 512, 4), 512, 0, st>>>(src, n, P, hist));
    else
      DDM_LAUNCH("radix_hist", 8.0 * n, st, radix::hist_kernel<false><<<grid_for(n, 512, 4), 512, 0, st>>>(src, n, P, hist));
    DDM_TRY(check_launch());
  }
  DDM_LAUNCH("radix_bin_start", 0, st, radix::bin_start_kernel<<<P.n, radix::kRadix, 0, st>>>(hist, s.starts));
  DDM_TRY(check_launch());
  const uint64_t tiles = radix::num_tiles(n, radix_items());
  const bool kv = vals_out != nullptr;
  const void* cur_k = src;
  const uint32_t* cur_v = vals_in;
  bool cur_f64 = src_f64;
  // in-place request with an odd pass count: move the input out of the way
  if (!src_f64 && cur_k == keys_out && (P.n & 1)) {
    DDM_CUDA(cudaMemcpyAsync(s.alt_keys, cur_k, n * 8, cudaMemcpyDeviceToDevice, st));
    cur_k = s.alt_keys;
    if (kv && vals_in == vals_out && vals_in) {
      DDM_CUDA(cudaMemcpyAsync(s.alt_vals, vals_in, n * 4, cudaMemcpyDeviceToDevice, st));
      cur_v = s.alt_vals;
    }
  }
  DDM_CUDA(cudaMemsetAsync(s.counters, 0, sizeof(uint32_t) * radix::kMaxPasses, st));
  const int items = radix_items();
  for (int p = 0; p < P.n; ++p) {
    const bool to_out = ((P.n - 1 - p) % 2) == 0;
    uint64_t* dk = to_out ? keys_out : s.alt_keys;
    uint32_t* dv = kv ? (to_out ? vals_out : s.alt_vals) : nullptr;
    DDM_CUDA(cudaMemsetAsync(s.status, 0, sizeof(uint32_t) * radix::kRadix * tiles, st));
    const uint32_t* ph = s.starts + p * radix::kRadix;
    const char* pname = kv ? (cur_f64 ? "onesweep_kv_f64" : "onesweep_kv") : (cur_f64 ? "onesweep_k_f64" : "onesweep_k");
    const double pbytes = (double)n * ((cur_f64 ? 8.0 : 8.0 + (kv && cur_v ? 4.0 : 0.0)) + 8.0 + (kv ? 4.0 : 0.0));
    if (items == 16)
      DDM_LAUNCH(pname, pbytes, st, launch_pass<16>(kv, cur_f64, tiles, st, cur_k, cur_v, dk, dv, n, P.shift[p], P.mask[p], ph,
                                                    s.status, s.counters + p));
    else if (items == 12)
      DDM_LAUNCH(pname, pbytes, st, launch_pass<12>(kv, cur_f64, tiles, st, cur_k, cur_v, dk, dv, n, P.shift[p], P.mask[p], ph,
                                                    s.status, s.counters + p));
    else
      DDM_LAUNCH(pname, pbytes, st, launch_pass<8>(kv, cur_f64, tiles, st, cur_k, cur_v, dk, dv, n, P.shift[p], P.mask[p], ph,
                                                   s.status, s.counters + p));
    DDM_TRY(check_launch());
    cur_k = dk;
    cur_v = dv;
    cur_f64 = false;
  }
  return DDM_OK;
}

// Value-bucketed MSD sort (msd.cuh) of n float64 keys `src` with optional
// payload: the upper coordinate `v64_src` (encoded to keys) and the index.
// mm = the keys' [min, max] (from validation).  Sets *overflow on a bucket
// too large for shared memory (caller falls back to radix_sort + gather).
// stages of msd_sort_t: the latency-bound preparation (sample, bucket map,
// digit histograms) and the record passes + local sort; a walk-form call
// overlaps one chain's preparation with the other chain's passes
enum : int { kMsdPrep = 1, kMsdRun = 2, kMsdAll = 3 };

template <bool PAY>
ddm_status msd_sort_t(const double* src, const double* v64_src, uint64_t n, uint64_t* mm, uint64_t* out_key,
                      uint64_t* out_v64, uint32_t* out_v32, MsdScratch& s, uint32_t* overflow, uint32_t* err,
                      cudaStream_t st, int stage = kMsdAll, int pack_hint = -1) {
  const int bits = msd_bits(n);
  const uint32_t nb = 1u << bits;
  const int passes = (bits + 7) / 8;
  const msd::MapRef M{mm, s.cbase};
  if (stage & kMsdPrep) {
  // bucket map equalised to the data (coarse population -> bucket allocation)
  if (n <= msd::kMapSmallMaxN) {  // small sorts: one latency-bound launch instead of three
    DDM_LAUNCH("msd_map", 16.0 * n / msd::kSampleStride, st,
               msd::map_small_kernel<true><<<1, 1024, 0, st>>>(src, n, mm, bits, s.cbase));
    DDM_TRY(check_launch());
  } else {
    DDM_CUDA(cudaMemsetAsync(s.ccount, 0, sizeof(uint32_t) * (msd::kCoarse + 1), st));
    const unsigned sgrid = grid_for((n + msd::kSampleStride - 1) / msd::kSampleStride, 512, 1);
    DDM_LAUNCH("msd_sample", 8.0 * n / msd::kSampleStride, st,
               msd::sample_minmax_kernel<true><<<sgrid, 512, 0, st>>>(src, n, mm));
    DDM_TRY(check_launch());
    DDM_LAUNCH("msd_coarse", 8.0 * n / msd::kSampleStride, st,
               msd::coarse_hist_kernel<true><<<sgrid, 512, 0, st>>>(
                   src, n, M, s.ccount));
    DDM_TRY(check_launch());
    DDM_LAUNCH("msd_map", 0, st, msd::map_build_kernel<<<1, 1024, 0, st>>>(s.ccount, bits, s.cbase));
    DDM_TRY(check_launch());
  }
  // digit histograms of every pass (their exclusive scans -- the digit
  // starts -- are taken inside the passes and the span-bounds kernel)
  DDM_CUDA(cudaMemsetAsync(s.dh, 0, sizeof(uint32_t) * 3 * 256, st));
  {  // lane-replicated counters: 32 KB of shared memory per pass, as many 512-thread CTAs per SM as fit
    const size_t hsm = msd::hist_smem_bytes(passes);
    const int per_sm = hsm > 64 * 1024 ? 2 : hsm > 48 * 1024 ? 3 : 4;
    DDM_LAUNCH("msd_hist", 8.0 * n, st, msd::msd_hist_kernel<true><<<grid_for(n, 512, per_sm), 512, hsm, st>>>(src, n, M, bits, passes, s.dh));
  }
  DDM_TRY(check_launch());
  }
  if (!(stage & kMsdRun)) return DDM_OK;
  const bool big = msd_big(n);
  const uint32_t span = big ? msd::LsBig::SPAN : msd::LsSmall::SPAN;
  const uint32_t spans = (uint32_t)((n + span - 1) / span);
  uint64_t* bk[2] = {s.k[0], s.k[1]};
  uint64_t* bv[2] = {s.v64[0], s.v64[1]};
  uint32_t* bi[2] = {s.v32[0], s.v32[1]};
  // payload passes: 16-record tiles when this chain runs alone, 8-record tiles
  // (fewer registers) while the rank form's three chains share the SMs
  const bool conc = chains_concurrent();
  const int items = PAY ? (conc ? msd::kItemsC : msd::kItems) : msd::kItemsK;
  const uint64_t tiles = (n + (uint64_t)msd::kThreads * items - 1) / ((uint64_t)msd::kThreads * items);
  DDM_CUDA(cudaMemsetAsync(s.counters, 0, sizeof(uint32_t) * radix::kMaxPasses, st));
  for (int p = 0; p < passes; ++p) {
    DDM_CUDA(cudaMemsetAsync(s.status, 0, sizeof(uint32_t) * radix::kRadix * tiles, st));
    const int o = p & 1, q = (p - 1) & 1;
    // PAY: packed 16-byte records (key + id | upper-key delta << 32, msd.cuh
    // TileRegs) unless DDM_MSD_PACK=0 (20-byte key + upper key + id)
    const bool pk = pack_records(n, pack_hint);
    const double rec = pk ? 16.0 : 20.0;
    const double bytes = (double)n * (PAY ? (p == 0 ? 16.0 + rec : 2.0 * rec) : 16.0);
#define DDM_PASS_KERNEL msd::msd_pass_kernel
#define DDM_MSD_PASS(ITEMS, V64, V32, F64, NAME, KI, VI, II)                                                       \
  DDM_LAUNCH(NAME, bytes, st,                                                                                     \
             (DDM_PASS_KERNEL<ITEMS, V64, V32, F64>                                                                \
              <<<persistent_grid((const void*)DDM_PASS_KERNEL<ITEMS, V64, V32, F64>, msd::kThreads,             \
                                 sizeof(msd::PassSmem<ITEMS, V64, V32>), tiles),                                  \
                 msd::kThreads, sizeof(msd::PassSmem<ITEMS, V64, V32>), st>>>(                                \
                  KI, VI, II, bk[o], V64 ? bv[o] : nullptr, V32 ? bi[o] : nullptr, n, M, bits, 8 * p,              \
                  s.dh + p * 256, s.status, s.counters + p, err)))
    if (p == 0) {
      if (PAY && pk && conc) DDM_MSD_PASS(msd::kItemsC, true, false, true, "msd_pass_pay", src, v64_src, nullptr);
      else if (PAY && pk) DDM_MSD_PASS(msd::kItems, true, false, true, "msd_pass_pay", src, v64_src, nullptr);
      else if (PAY && conc) DDM_MSD_PASS(msd::kItemsC, true, true, true, "msd_pass_pay", src, v64_src, nullptr);
      else if (PAY) DDM_MSD_PASS(msd::kItems, true, true, true, "msd_pass_pay", src, v64_src, nullptr);
      else DDM_MSD_PASS(msd::kItemsK, false, false, true, "msd_pass", src, nullptr, nullptr);
    } else {
      if (PAY && pk && conc) DDM_MSD_PASS(msd::kItemsC, true, false, false, "msd_pass_pay", bk[q], bv[q], nullptr);
      else if (PAY && pk) DDM_MSD_PASS(msd::kItems, true, false, false, "msd_pass_pay", bk[q], bv[q], nullptr);
      else if (PAY && conc) DDM_MSD_PASS(msd::kItemsC, true, true, false, "msd_pass_pay", bk[q], bv[q], bi[q]);
      else if (PAY) DDM_MSD_PASS(msd::kItems, true, true, false, "msd_pass_pay", bk[q], bv[q], bi[q]);
      else DDM_MSD_PASS(msd::kItemsK, false, false, false, "msd_pass", bk[q], nullptr, nullptr);
    }
#undef DDM_MSD_PASS
#undef DDM_PASS_KERNEL
    DDM_TRY(check_launch());
  }
  const int l = (passes - 1) & 1;
  if (passes == 1)  // bucket starts = the pass's digit starts
    DDM_LAUNCH("msd_bounds", 0, st, msd::span_bounds_hist_kernel<<<(spans + 256) / 256, 256, 0, st>>>(
        s.dh, nb, n, spans, span, s.bounds));
  else
    DDM_LAUNCH("msd_bounds", 0, st, msd::span_bounds_kernel<<<(spans + 256) / 256, 256, 0, st>>>(bk[l], n, M, bits, spans,
                                                                                               span, s.bounds));
  DDM_TRY(check_launch());
#define DDM_LOCAL(C, V64, V32, NAME, BYTES, VI, II, HI)                                                         \
  DDM_LAUNCH(NAME, BYTES, st,                                                                                  \
             (msd::local_sort_kernel<C, V64, V32><<<spans, C::T, sizeof(msd::LocalSmem<C, V64, V32>), st>>>(   \
                 bk[l], VI, II, out_key, V64 ? out_v64 : nullptr, V32 || V64 ? out_v32 : nullptr, n, M, bits,    \
                 s.bounds, overflow, HI)))
  if (PAY && pack_records(n, pack_hint)) {
    if (big) DDM_LOCAL(msd::LsBig, true, false, "msd_local_pay", 36.0 * n, bv[l], nullptr, v64_src);
    else DDM_LOCAL(msd::LsSmall, true, false, "msd_local_pay", 36.0 * n, bv[l], nullptr, v64_src);
  } else if (PAY) {
    if (big) DDM_LOCAL(msd::LsBig, true, true, "msd_local_pay", 40.0 * n, bv[l], bi[l], nullptr);
    else DDM_LOCAL(msd::LsSmall, true, true, "msd_local_pay", 40.0 * n, bv[l], bi[l], nullptr);
  } else {
    if (big) DDM_LOCAL(msd::LsBig, false, false, "msd_local", 16.0 * n, nullptr, nullptr, nullptr);
    else DDM_LOCAL(msd::LsSmall, false, false, "msd_local", 16.0 * n, nullptr, nullptr, nullptr);
  }
#undef DDM_LOCAL
  return check_launch();
}

ddm_status init_minmax(uint64_t* mm, cudaStream_t st) {  // [min, max] x 3 = [~0, 0] x 3
  DDM_CUDA(cudaMemsetAsync(mm, 0xff, 6 * sizeof(uint64_t), st));
  for (int k = 0; k < 3; ++k) DDM_CUDA(cudaMemsetAsync(mm + 2 * k + 1, 0, sizeof(uint64_t), st));
  return DDM_OK;
}

// ------------------------------------------------------------ argument checks

bool aligned(const void* p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

ddm_status check_side(uint32_t d, uint64_t cnt, const double* const* lo, const double* const* hi) {
  if (cnt > DDM_MAX_REGIONS) return DDM_ERR_INVALID_ARGUMENT;
  if (cnt == 0) return DDM_OK;
  for (uint32_t k = 0; k < d; ++k)
    if (!lo[k] || !hi[k] || !aligned(lo[k], 8) || !aligned(hi[k], 8)) return DDM_ERR_INVALID_ARGUMENT;
  return DDM_OK;
}

ddm_status check_regions(const ddm_regions* R, bool need_sub, bool need_upd) {
  if (!R || R->d == 0 || R->d > DDM_MAX_DIMS) return DDM_ERR_INVALID_ARGUMENT;
  if (need_sub) DDM_TRY(check_side(R->d, R->n_sub, R->sub_lo, R->sub_hi));
  if (need_upd) DDM_TRY(check_side(R->d, R->n_upd, R->upd_lo, R->upd_hi));
  return DDM_OK;
}

ddm_status err_status(uint32_t e) {
  if (e & match::kErrNonFinite) return DDM_ERR_NONFINITE;
  if (e & match::kErrInverted) return DDM_ERR_INVERTED_INTERVAL;
  return DDM_OK;
}

// validate all dims of one side; histogram dim 0 into hist_lo / hist_hi
ddm_status validate_side(uint32_t d, uint64_t cnt, const double* const* lo, const double* const* hi,
                         uint32_t* hist_lo, uint32_t* hist_hi, uint32_t* err, cudaStream_t st,
                         uint64_t* mm_lo = nullptr, uint64_t* mm_hi = nullptr, uint32_t k_begin = 0) {
  if (cnt == 0) return DDM_OK;
  for (uint32_t k = k_begin; k < d; ++k) {
    DDM_LAUNCH("validate_hist", 16.0 * cnt, st, match::validate_hist_kernel<<<grid_for(cnt, 512, 4), 512, 0, st>>>(
        lo[k], hi[k], cnt, k == 0 ? hist_lo : nullptr, k == 0 ? hist_hi : nullptr, err, k == 0 ? mm_lo : nullptr,
        k == 0 ? mm_hi : nullptr));
    DDM_TRY(check_launch());
  }
  return DDM_OK;
}

// ------------------------------------------------------------ index build (async)

// Subscription half: validate, sort Slo (key + upper key + id) and Shi (keys),
// block maxima, other dimensions in Slo order.  MSD path: the Shi chain runs
// on a side stream concurrently with the Slo chain; `st` has joined it on
// return.  mm[0..3] must hold the [min, max] initial values (init_minmax).
// What the index keeps: Shi for the rank-form counts (count-only calls), the
// slo_hi prefix maxima for the walk-form counts (pairs calls); ddm_sub_index_build
// keeps both.
enum : int { kNeedShi = 1, kNeedPm = 2, kNeedKeysOnly = 4 };  // kNeedKeysOnly: d = 1 count-only calls
constexpr uint64_t kWalkMinN = 1ull << 20;  // below: rank form (the Shi chain hides on a side stream)
constexpr double kWalkMaxStab = 4.0;        // walk form while the estimated mean |Stab(a)| is at most this

// levels >= 1 of the block-max tree (+ the prefix maxima when kNeedPm); on
// the LSB path level 1 was written by gather_key_kernel
ddm_status tree_async(const Index& I, int need, bool have_lvl1, cudaStream_t st) {
  const uint64_t n = I.n;
  int from = have_lvl1 ? 2 : 1;
  if (need & kNeedPm) {
    DDM_LAUNCH("tree_pm", 16.0 * n, st, match::tree_pm_kernel<<<(unsigned)I.nb, 256, 0, st>>>(
        I.slo_hi, n, (!have_lvl1 && I.levels >= 1) ? I.lvl[1] : nullptr, I.levels >= 1 ? I.lvl_n[1] : 0,
        I.levels >= 2 ? I.lvl[2] : nullptr, I.pmw, I.pmb));
    DDM_TRY(check_launch());
    const unsigned chunks = (unsigned)((I.nb + match::kPmChunk - 1) / match::kPmChunk);
    DDM_LAUNCH("pmb_scan", 8.0 * I.nb, st, match::pmb_chunk_kernel<<<chunks, 1024, 0, st>>>(I.pmb, I.nb, I.pmc));
    DDM_TRY(check_launch());
    DDM_LAUNCH("pmb_scan", 16.0 * I.nb, st, match::pmb_scan_kernel<<<chunks, 1024, 0, st>>>(I.pmb, I.nb, I.pmc));
    DDM_TRY(check_launch());
    from = 3;
  }
  if (from <= I.levels) {  // the remaining levels in one launch
    match::TreeLv T{};
    for (int L = 0; L <= I.levels; ++L) { T.lvl[L] = I.lvl[L]; T.n[L] = I.lvl_n[L]; }
    T.levels = I.levels;
    DDM_CUDA(cudaMemsetAsync(I.tick, 0, sizeof(uint32_t), st));
    DDM_LAUNCH("block_max", 8.0 * I.lvl_n[from - 1], st, match::tree_levels_kernel<<<(unsigned)((I.lvl_n[from] + 255) / 256), 256, 0, st>>>(
        T, from, I.tick));
    DDM_TRY(check_launch());
  }
  return DDM_OK;
}

ddm_status build_index_async(const ddm_regions* R, const Index& I, MsdScratch& slo, MsdScratch& shi,
                             const SortScratch& lsb, uint64_t* mm, Misc* misc, bool use_msd, cudaStream_t st,
                             int need = kNeedShi | kNeedPm, bool boxes_only = false) {
  init_attrs_once();
  const uint64_t n = R->n_sub;
  if (n == 0) return DDM_OK;
  if (use_msd) {
    // a1 for dims 1..d-1 here; dim 0 is validated inside the first Slo pass,
    // which reads lo and hi anyway (the sort's key range comes from a sample)
    // (dim 0 is validated by the first multisplit pass; row-indexed d > 1
    // calls validate dims 1-2 in box_in_kernel)
    // d = 1 count-only calls (rank form: K = sum r_b - r_hi, App. A I2) need
    // the sorted lower keys alone: Slo is sorted keys-only (8-byte records, no
    // upper keys / ids / block maxima), and dim 0 is validated here because no
    // pass reads both of its bounds
    const bool keys_only = (need & kNeedKeysOnly) != 0 && R->d == 1;
    DDM_TRY(validate_side(R->d, n, R->sub_lo, R->sub_hi, nullptr, nullptr, &misc->err, st, nullptr, nullptr,
                          keys_only ? 0 : boxes_only ? 3 : 1));
    cudaStream_t side[2];
    const bool with_shi = (need & kNeedShi) != 0;
    if (with_shi) {
      DDM_TRY(side_streams(side, st));
      DDM_TRY(stream_join(side[0], st));
      // a2: Shi keys on a side stream, concurrent with the Slo chain
      DDM_TRY(msd_sort_t<false>(R->sub_hi[0], nullptr, n, mm + 2, I.shi_key, nullptr, nullptr, shi, &misc->overflow,
                                nullptr, side[0]));
    }
    if (keys_only) {
      DDM_TRY(msd_sort_t<false>(R->sub_lo[0], nullptr, n, mm + 0, I.slo_key, nullptr, nullptr, slo, &misc->overflow,
                                nullptr, st));
    } else {
      // a2 + a3: Slo with the upper key and the id as payload
      DDM_TRY(msd_sort_t<true>(R->sub_lo[0], R->sub_hi[0], n, mm + 0, I.slo_key, I.slo_hi, I.slo_id, slo,
                               &misc->overflow, &misc->err, st, kMsdAll, t_pack.sub));
      DDM_TRY(tree_async(I, need, false, st));
    }
    if (with_shi) DDM_TRY(stream_join(st, side[0]));
  } else {
    SortScratch s = lsb_with(lsb, slo);
    DDM_CUDA(cudaMemsetAsync(s.hist[0], 0, sizeof(uint32_t) * 8 * 256, st));
    DDM_CUDA(cudaMemsetAsync(s.hist[1], 0, sizeof(uint32_t) * 8 * 256, st));
    DDM_TRY(validate_side(R->d, n, R->sub_lo, R->sub_hi, s.hist[0], s.hist[1], &misc->err, st));
    const radix::PassList P = full_passes();
    // a2: Slo (key + sub id, encoded from float64 in pass 1), Shi (keys)
    DDM_TRY(radix_sort(R->sub_lo[0], true, nullptr, I.slo_key, I.slo_id, n, P, s.hist[0], true, s, st));
    if (need & kNeedShi)
      DDM_TRY(radix_sort(R->sub_hi[0], true, nullptr, I.shi_key, nullptr, n, P, s.hist[1], true, s, st));
    // a3: slo_hi[i] = key(sub_hi[slo_id[i]]) + block maxima
    DDM_LAUNCH("gather_slo_hi", 20.0 * n, st, match::gather_key_kernel<<<grid_for(n, 256, 8), 256, 0, st>>>(I.slo_id, R->sub_hi[0], n,
                                                                               I.slo_hi, I.levels ? I.lvl[1] : nullptr));
    DDM_TRY(check_launch());
    DDM_TRY(tree_async(I, need, true, st));
  }
  if (R->d > 1) {
    match::DimPtrs D{};
    for (uint32_t k = 0; k < R->d; ++k) { D.lo[k] = R->sub_lo[k]; D.hi[k] = R->sub_hi[k]; }
    if (boxes_only) {
      // row-indexed d > 1 calls: dims-1/2 float boxes in input order (over the
      // sdims storage), gathered by id into Slo order; exact tests read the
      // input arrays through the ids
      float4* bin = reinterpret_cast<float4*>(I.sdims);
      DDM_LAUNCH("dd_boxes", 32.0 * n, st, dd::box_in_kernel<<<grid_for(n, 256, 8), 256, 0, st>>>(D, (int)R->d, n, bin, &misc->err));
      DDM_TRY(check_launch());
      DDM_LAUNCH("dd_boxes", 56.0 * n, st,
                 dd::box_kernel<<<grid_for(n, 256, 8), 256, 0, st>>>(nullptr, (int)R->d, n, I.box12,
                                                                     use_msd ? &misc->overflow : nullptr, I.slo_key,
                                                                     I.slo_hi, I.box0, bin, I.slo_id));
      DDM_TRY(check_launch());
      return DDM_OK;
    }
    DDM_LAUNCH("gather_dims", 36.0 * (R->d - 1) * n, st, match::gather_dims_kernel<<<grid_for(n, 256, 8), 256, 0, st>>>(I.slo_id, D, (int)R->d, n, I.sdims,
                                                                                   use_msd ? &misc->overflow : nullptr));
    DDM_TRY(check_launch());
    DDM_LAUNCH("dd_boxes", 16.0 * (R->d > 2 ? 2 : 1) * n + 16.0 * n, st,
               dd::box_kernel<<<grid_for(n, 256, 8), 256, 0, st>>>(I.sdims, (int)R->d, n, I.box12,
                                                                   use_msd ? &misc->overflow : nullptr, I.slo_key,
                                                                   I.slo_hi, I.box0, nullptr, nullptr));
    DDM_TRY(check_launch());
  }
  return DDM_OK;
}

// ------------------------------------------------------------ d > 1 tiled filter (dd.cuh)


// Row-indexed d > 1 passes (dd::rows_kernel): the default when their
// 4096-row tiles fill the GPU; DDM_DD_CHUNKS=1 keeps the chunk-indexed
// dd_tile_kernel (A/B and cross-check).
bool dd_rows_enabled(uint64_t m, uint32_t flags) {
  static const bool off = [] {
    const char* e = getenv("DDM_DD_CHUNKS");
    return e && atoi(e) == 1;
  }();
  if (flags & DDM_DD_FORCE_ROWS) return true;
  if (flags & DDM_DD_FORCE_CHUNKS) return false;
  constexpr uint64_t kRowsT = dd::kRT * kDDRRows;
  return !off && (m + kRowsT - 1) / kRowsT >= (uint64_t)kSMs;
}

void launch_dd_rows(int mode, const dd::Args& a, uint32_t* old_n, cudaStream_t st) {
  constexpr int kRows = dd::kRT * kDDRRows;
  const unsigned grid = (unsigned)((a.m + kRows - 1) / kRows);
  if (mode == dd::kModeCount)
    dd::rows_kernel<kDDRRows, dd::kModeCount><<<grid, dd::kRT, sizeof(dd::RowSmem<kDDRRows>), st>>>(a, old_n);
  else if (mode == dd::kModeStage)
    dd::rows_kernel<kDDRRows, dd::kModeStage><<<grid, dd::kRT, sizeof(dd::RowSmem<kDDRRows>), st>>>(a, old_n);
  else
    dd::rows_place_kernel<kDDRRows><<<grid, dd::kRT, dd::rows_place_smem<kDDRRows>(), st>>>(a);
}

void launch_dd(int mode, const dd::Args& a, cudaStream_t st) {
  constexpr int kRows = dd::kThreads * kDDRows;
  const unsigned grid = (unsigned)((a.m + kRows - 1) / kRows);
  const size_t sm = dd::smem_bytes<kDDRows>(mode);
  if (mode == dd::kModeCount) dd::dd_tile_kernel<kDDRows, dd::kModeCount><<<grid, dd::kThreads, sm, st>>>(a);
  else if (mode == dd::kModeStage) dd::dd_tile_kernel<kDDRows, dd::kModeStage><<<grid, dd::kThreads, sm, st>>>(a);
  else dd::dd_tile_kernel<kDDRows, dd::kModePlace><<<grid, dd::kThreads, sm, st>>>(a);
}

// ------------------------------------------------------------ match against an index

// ddm_chunk_start_sets: export A_t of every emit tile instead of emitting
struct ChunkExport {
  uint32_t* first_upd;
  uint64_t* off;
  uint32_t* ids;
  uint64_t cap;
  uint64_t* total_out;
};

struct MatchReq {
  const Index* I;
  const ddm_regions* R;       // update side (d, n_upd, upd_lo/hi)
  const uint32_t* upd_map;    // optional global ids of the updates
  ddm_pair* pairs;            // nullptr = count only
  uint64_t capacity;
  uint32_t flags;
  const uint32_t* sub_map = nullptr;  // optional global ids of the subscriptions
  bool walk = false;                  // walk-form counts (index holds the slo_hi prefix maxima, not Shi)
  bool boxes_only = false;            // d > 1 row-indexed call: the index holds float boxes, no sdims
  const ChunkExport* chunk = nullptr;  // export the chunk-start sets (d = 1) instead of the pairs
};

// Update side, a1 + a2 (+ a3): validate every dimension, sort Ulo with the
// upper key and the id as payload (MSD) or key + id (LSB fallback).  With
// n_sub == 0 only the validation runs.  mm[4..5] must hold init values.
ddm_status upd_sort_async(const ddm_regions* R, MatchWs& W, uint64_t n_sub, bool use_msd, cudaStream_t st,
                          int stage = kMsdAll, uint32_t v_begin = 1) {
  const uint64_t m = R->n_upd;
  const uint32_t d = R->d;
  if (m == 0) return DDM_OK;
  init_attrs_once();
  if (n_sub == 0) return (stage & kMsdPrep) ? validate_side(d, m, R->upd_lo, R->upd_hi, nullptr, nullptr, &W.misc->err, st)
                                            : DDM_OK;
  if (use_msd) {
    if (stage & kMsdPrep)
      DDM_TRY(validate_side(d, m, R->upd_lo, R->upd_hi, nullptr, nullptr, &W.misc->err, st, nullptr, nullptr, v_begin));
    return msd_sort_t<true>(R->upd_lo[0], R->upd_hi[0], m, W.mm + 4, W.ulo_key, W.uhi, W.ulo_id, W.ulo,
                            &W.misc->overflow, &W.misc->err, st, stage, t_pack.upd);
  }
  if (!(stage & kMsdRun)) return DDM_OK;  // (the LSB path has no separate preparation)
  SortScratch s = lsb_with(W.sort, W.ulo);
  DDM_CUDA(cudaMemsetAsync(s.hist[2], 0, sizeof(uint32_t) * 8 * 256, st));
  DDM_TRY(validate_side(d, m, R->upd_lo, R->upd_hi, s.hist[2], nullptr, &W.misc->err, st));
  return radix_sort(R->upd_lo[0], true, nullptr, W.ulo_key, W.ulo_id, m, full_passes(), s.hist[2], true, s, st);
}

// a4..a8 against a built index, with the updates already sorted on `st`:
// counts, scan, one D2H of {K, error, overflow}, then the emission.
// a4..a8 against a built index with the updates already sorted on `st`.
// Phase PRE enqueues the counts and the offset scan (everything before the
// host needs K: capturable in a CUDA graph); phase POST reads {K, error,
// overflow} back (the call's one sync) and enqueues the emission.
enum MatchPhase { kPhasePre = 1, kPhasePost = 2, kPhaseAll = 3 };

ddm_status match_sorted(const MatchReq& q, MatchWs& W, uint64_t* count_out, bool use_msd, cudaStream_t st,
                        int phase = kPhaseAll) {
  const Index& I = *q.I;
  const ddm_regions* R = q.R;
  const uint64_t m = R->n_upd, n = I.n;
  const uint32_t d = R->d;
  if (m == 0 || n == 0) {  // nothing can match; the non-empty side(s) were validated
    if (!(phase & kPhasePost)) return DDM_OK;
    Misc h{};
    DDM_CUDA(cudaMemcpyAsync(&h, W.misc, sizeof(Misc), cudaMemcpyDeviceToHost, st));
    DDM_CUDA(cudaStreamSynchronize(st));
    *count_out = 0;
    return err_status(h.err);
  }
  const bool pre = (phase & kPhasePre) != 0;
  // a4: counts by rank difference (+ the row-tile sums); a5: exclusive scan
  // of the row-tile sums -> output offset of every 256-row tile, K
  const uint64_t ctiles = (m + match::kCountTile - 1) / match::kCountTile;
  const uint64_t rtiles = (m + match::kRowTile - 1) / match::kRowTile;
  const unsigned stiles = (unsigned)((rtiles + match::kScanThreads * match::kScanItems - 1) /
                                     (match::kScanThreads * match::kScanItems));
  // a4 for the row-indexed d > 1 filter: only r_lo of each tile's first
  // query and the end of its candidate slice (tile_ranks_kernel); the count
  // pass runs only if a tile overflows its staging slot (its fallback needs
  // the per-row ranks)
  const match::CountWalk CW{I.slo_hi, I.pmw, I.pmb, I.nb, tree_of(I)};
  auto count_pass = [&](cudaStream_t cs) -> ddm_status {
    if (ctiles <= match::kPartWarpMaxTiles)
      DDM_LAUNCH("count_partition", 0, cs, match::count_partition_kernel<<<(unsigned)((ctiles * 32 + 255) / 256), 256, 0, cs>>>(
          W.ulo_key, m, I.slo_key, q.walk ? nullptr : I.shi_key, n, W.part));
    else
      DDM_LAUNCH("count_partition", 0, cs, match::count_partition1_kernel<<<(unsigned)((ctiles + 255) / 256), 256, 0, cs>>>(
          W.ulo_key, m, I.slo_key, q.walk ? nullptr : I.shi_key, n, W.part));
    DDM_TRY(check_launch());
    // d = 1 count-only calls keep only the 256-row tile sums (no per-row r_lo / r_b / cnt)
    const bool rows = !(d == 1 && !q.pairs && !q.chunk);
    uint32_t* const o_lo = rows ? W.r_lo : nullptr;
    uint32_t* const o_b = rows ? W.r_b : nullptr;
    uint32_t* const o_c = rows ? W.cnt0 : nullptr;
    const double cbytes = (use_msd ? (rows ? 28.0 : 16.0) : 48.0) * m + (q.walk ? 24.0 : 16.0) * n;
    if (q.walk)
      DDM_LAUNCH("count", cbytes, cs, match::count_kernel<true><<<(unsigned)ctiles, match::kCountThreads, match::count_smem_bytes(true), cs>>>(
          W.ulo_key, W.ulo_id, R->upd_hi[0], use_msd ? W.uhi : nullptr, m, I.slo_key, nullptr, n, W.part, o_lo, o_b,
          o_c, W.tile_sum, CW));
    else
      DDM_LAUNCH("count", cbytes, cs, match::count_kernel<false><<<(unsigned)ctiles, match::kCountThreads, match::count_smem_bytes(false), cs>>>(
          W.ulo_key, W.ulo_id, R->upd_hi[0], use_msd ? W.uhi : nullptr, m, I.slo_key, I.shi_key, n, W.part, o_lo, o_b,
          o_c, W.tile_sum, CW));
    return check_launch();
  };
  if (pre && !q.boxes_only) DDM_TRY(count_pass(st));
  if (pre && d == 1) {
    DDM_CUDA(cudaMemsetAsync(W.scan_status, 0, sizeof(uint64_t) * (stiles + 1), st));
    DDM_LAUNCH("scan", 16.0 * rtiles, st, match::scan_u64_kernel<<<stiles, match::kScanThreads, 0, st>>>(
        W.tile_sum, rtiles, W.tile_off, W.scan_status, &W.misc->K));
    DDM_TRY(check_launch());
  }

  match::EmitArgs A{};
  A.ulo_key = W.ulo_key;
  A.ulo_id = W.ulo_id;
  A.upd_map = q.upd_map;
  A.sub_map = q.sub_map;
  A.r_lo = W.r_lo;
  A.r_b = W.r_b;
  A.cnt0 = W.cnt0;
  A.cnt = W.cnt0;
  A.tile_off = W.tile_off;
  A.slo_id = I.slo_id;
  A.T = tree_of(I);
  A.F.dims = (int)d - 1;
  A.F.sdims = I.sdims;
  A.F.n = n;
  for (uint32_t k = 0; k < d; ++k) { A.upd.lo[k] = R->upd_lo[k]; A.upd.hi[k] = R->upd_hi[k]; }
  A.m = m;
  A.abort_flag = use_msd ? &W.misc->overflow : nullptr;
  A.thread_row_max = 16;
  A.force = (q.flags & DDM_EMIT_FORCE_THREAD) ? 1 : (q.flags & DDM_EMIT_FORCE_WARP) ? 2
            : (q.flags & DDM_EMIT_FORCE_CHUNK) ? 3 : 0;
  const unsigned egrid = (unsigned)rtiles;

  // per-row d > 1 filter: forced by the emit flags, or chosen when the update
  // tiles of the tiled filter could not fill the GPU (fewer tiles than SMs,
  // e.g. few updates against many subscriptions: 35 ms instead of 1.4 s at
  // n = 4e6, m = 2e3); each row then gets a thread or a warp
  const bool per_row = (q.flags & (DDM_EMIT_FORCE_THREAD | DDM_EMIT_FORCE_WARP)) != 0 ||
                       (d > 1 && !(q.flags & (DDM_DD_FORCE_ROWS | DDM_DD_FORCE_CHUNKS)) &&
                        (m + dd::kThreads * kDDRows - 1) / (dd::kThreads * kDDRows) < (uint64_t)kSMs);
  dd::Args D{};
  const bool dd_rows = d > 1 && !per_row && dd_rows_enabled(m, q.flags);
  if (d > 1 && !per_row) {
    // a8: tiled dim-0 sweep with the exact filter on dims 1..d-1 (dd.cuh):
    // count pass -> 256-row tile sums -> scan; the emit pass runs after the sync
    D.ulo_key = W.ulo_key;
    D.ulo_id = W.ulo_id;
    D.upd_map = q.upd_map;
    D.sub_map = q.sub_map;
    D.r_lo = W.r_lo;
    D.r_b = W.r_b;
    D.cnt0 = W.cnt0;
    D.slo_key = I.slo_key;
    D.slo_id = I.slo_id;
    for (uint32_t k = 0; k < d; ++k) { D.upd.lo[k] = R->upd_lo[k]; D.upd.hi[k] = R->upd_hi[k]; }
    D.T = tree_of(I);
    D.sdims = q.boxes_only ? nullptr : I.sdims;
    D.udims = q.boxes_only ? nullptr : W.udims;
    D.ubox = q.boxes_only ? reinterpret_cast<const float4*>(W.udims) : nullptr;
    for (uint32_t k = 0; k < d && q.boxes_only; ++k) { D.sub.lo[k] = R->sub_lo[k]; D.sub.hi[k] = R->sub_hi[k]; }
    D.uhi = use_msd ? W.uhi : nullptr;
    D.box12 = I.box12;
    D.box0 = I.box0;
    if (pre) {
      match::DimPtrs U{};
      for (uint32_t k = 0; k < d; ++k) { U.lo[k] = R->upd_lo[k]; U.hi[k] = R->upd_hi[k]; }
      if (q.boxes_only)  // dims-1/2 float boxes in input order (over the udims storage), read by id
        DDM_LAUNCH("dd_boxes", 48.0 * m, st, dd::box_in_kernel<<<grid_for(m, 256, 8), 256, 0, st>>>(
            U, (int)d, m, reinterpret_cast<float4*>(W.udims), &W.misc->err));
      else  // dims 1..d-1 of the updates gathered into sweep order (exact re-tests stay local)
        DDM_LAUNCH("gather_dims", 36.0 * (d - 1) * m, st, match::gather_dims_kernel<<<grid_for(m, 256, 8), 256, 0, st>>>(
            W.ulo_id, U, (int)d, m, W.udims, &W.misc->overflow));
      DDM_TRY(check_launch());
    }
    D.n = n;
    D.m = m;
    D.d = (int)d;
    D.abort_flag = &W.misc->overflow;
    D.cnt_out = W.cnt;
    D.tile_sum = W.tile_sum;
    D.stage = W.dd_stage;
    D.stage_n = W.dd_stage_n;
    D.cnt = W.cnt;
    D.tile_off = W.tile_off;
    D.ovf_any = &W.misc->dd_ovf;
    if (q.boxes_only) {
      D.tile_rk = reinterpret_cast<const uint32_t*>(W.part);
      D.pmw = I.pmw;
      D.pmb = I.pmb;
    }
    // one enumeration: counts (+ staged hits when pairs are wanted) -> scan;
    // the place pass runs after the sync and the capacity check
    if (pre) {
      if (dd_rows) {
        dd::Args D2 = D;
        D2.stage_n = W.dd_stage_n2;
        if (q.boxes_only) {
          constexpr uint64_t kRowsT = dd::kRT * kDDRRows;
          const uint64_t rt = (m + kRowsT - 1) / kRowsT;
          DDM_LAUNCH("tile_ranks", 8.0 * m, st, dd::tile_ranks_kernel<kDDRRows><<<(unsigned)((rt * 32 + 255) / 256), 256, 0, st>>>(
              D, reinterpret_cast<uint32_t*>(W.part)));
          DDM_TRY(check_launch());
        }
        if (q.pairs) DDM_LAUNCH("dd_stage", 24.0 * m, st, launch_dd_rows(dd::kModeStage, D2, W.dd_stage_n, st));
        else DDM_LAUNCH("dd_count", 24.0 * m, st, launch_dd_rows(dd::kModeCount, D2, W.dd_stage_n, st));
      } else if (q.pairs) {
        DDM_LAUNCH("dd_stage", 24.0 * m, st, launch_dd(dd::kModeStage, D, st));
      } else {
        DDM_LAUNCH("dd_count", 24.0 * m, st, launch_dd(dd::kModeCount, D, st));
      }
      DDM_TRY(check_launch());
      DDM_CUDA(cudaMemsetAsync(W.scan_status, 0, sizeof(uint64_t) * (stiles + 1), st));
      DDM_LAUNCH("scan", 16.0 * rtiles, st, match::scan_u64_kernel<<<stiles, match::kScanThreads, 0, st>>>(
          W.tile_sum, rtiles, W.tile_off, W.scan_status, &W.misc->K));
      DDM_TRY(check_launch());
    }
  } else if (d > 1 && pre) {
    // a8, per-row form (forced by the emit-path flags; cross-check of the tiled form)
    A.cnt_out = W.cnt;
    A.fstab_out = W.fstab;
    DDM_LAUNCH("count_dd", 44.0 * m, st, match::emit_kernel<match::kCountDD><<<egrid, match::kRowTile, 0, st>>>(A));
    DDM_TRY(check_launch());
    DDM_LAUNCH("row_tile_sum", 4.0 * m, st, match::row_tile_sum_kernel<<<egrid, match::kRowTile, 0, st>>>(W.cnt, m, W.tile_sum));
    DDM_TRY(check_launch());
    DDM_CUDA(cudaMemsetAsync(W.scan_status, 0, sizeof(uint64_t) * (stiles + 1), st));
    DDM_LAUNCH("scan", 16.0 * rtiles, st, match::scan_u64_kernel<<<stiles, match::kScanThreads, 0, st>>>(
        W.tile_sum, rtiles, W.tile_off, W.scan_status, &W.misc->K));
    DDM_TRY(check_launch());
  }
  if (d > 1 && per_row) {
    A.cnt = W.cnt;
    A.fstab = W.fstab;
  }
  if (!(phase & kPhasePost)) return DDM_OK;
  Misc h{};
  DDM_CUDA(cudaMemcpyAsync(&h, W.misc, sizeof(Misc), cudaMemcpyDeviceToHost, st));
  DDM_CUDA(cudaStreamSynchronize(st));
  *count_out = h.K;
  DDM_TRY(err_status(h.err));
  if (h.overflow) return kRetryLSB;  // degenerate bucket: nothing written yet, redo with the LSB sort
  if (q.chunk) {
    // a6 exported: |A_t| per emit tile -> offsets (scan) -> members by the
    // emit_chunk_kernel walk
    const ChunkExport& C = *q.chunk;
    DDM_LAUNCH("chunk_sets", 12.0 * rtiles, st, match::chunk_set_sizes_kernel<<<(unsigned)((rtiles + 255) / 256), 256, 0, st>>>(
        A, rtiles, W.tile_sum, C.first_upd));
    DDM_TRY(check_launch());
    DDM_CUDA(cudaMemsetAsync(W.scan_status, 0, sizeof(uint64_t) * (stiles + 1), st));
    DDM_LAUNCH("scan", 16.0 * rtiles, st, match::scan_u64_kernel<<<stiles, match::kScanThreads, 0, st>>>(
        W.tile_sum, rtiles, C.off, W.scan_status, C.off + rtiles));
    DDM_TRY(check_launch());
    uint64_t total = 0;
    DDM_CUDA(cudaMemcpyAsync(&total, C.off + rtiles, sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
    DDM_CUDA(cudaStreamSynchronize(st));
    *C.total_out = total;
    if (total > C.cap) return DDM_ERR_CAPACITY;
    DDM_LAUNCH("chunk_sets", 4.0 * total, st, match::chunk_set_ids_kernel<<<(unsigned)rtiles, 32, 0, st>>>(
        A, C.off, C.ids));
    return check_launch();
  }
  if (!q.pairs) return DDM_OK;
  if (h.K > q.capacity) return DDM_ERR_CAPACITY;
  if (h.K == 0) return DDM_OK;
  A.pairs = reinterpret_cast<uint2*>(q.pairs);
  if (d > 1 && !per_row) {
    D.pairs = A.pairs;
    D.capacity = q.capacity;
    if (dd_rows) {
      dd::Args D2 = D;
      D2.stage_n = W.dd_stage_n2;
      DDM_LAUNCH("dd_place", 16.0 * h.K + 8.0 * h.K, st, launch_dd_rows(dd::kModePlace, D2, nullptr, st));
      DDM_TRY(check_launch());
      if (!h.dd_ovf) return DDM_OK;
      // tiles whose staging slot overflowed: the direct (deterministic) place
      // pass of the chunk-indexed kernel, on its 1024-row tiles marked ~0u
      // (it needs the per-row ranks of the count pass)
      if (q.boxes_only) DDM_TRY(count_pass(st));
    }
    DDM_LAUNCH("dd_place", 16.0 * h.K + 8.0 * h.K, st, launch_dd(dd::kModePlace, D, st));
    return check_launch();
  }
  // sparse outputs (a few pairs per row on average, e.g. alpha ~ 1) gain
  // nothing from staging chunk-start sets: the light per-row kernel (higher
  // occupancy) is used unless the chunk path is forced
  if (d == 1 && !per_row && !(q.flags & DDM_EMIT_FORCE_CHUNK) && h.K > 4ull * m && egrid < (unsigned)kSMs) {
    // few dense rows: (row, segment) tasks spread over every SM
    const uint64_t warps = m * match::kSplitSeg;
    const unsigned sgrid = (unsigned)umin64((warps * 32 + 255) / 256, (uint64_t)kSMs * 8);
    DDM_LAUNCH("emit", 24.0 * m + 8.0 * h.K + 12.0 * n, st, match::emit_split_kernel<<<sgrid, 256, 0, st>>>(A));
  } else if (d == 1 && !per_row && (h.K > 4ull * m || (q.flags & DDM_EMIT_FORCE_CHUNK)))
    DDM_LAUNCH("emit", 24.0 * m + 8.0 * h.K + 12.0 * n, st,
               match::emit_chunk_kernel<<<egrid, match::kRowTile, sizeof(match::ChunkSmem), st>>>(A));
  else if (d == 1 && !per_row)  // sparse: tiles of 2048 rows walking a staged Slo window
    DDM_LAUNCH("emit", 24.0 * m + 8.0 * h.K + 12.0 * n, st,
               match::emit_tile_kernel<<<(unsigned)((m + match::kEmitTile - 1) / match::kEmitTile), match::kEmitThreads,
                                         sizeof(match::EmitTileSmem), st>>>(A));
  else if (d == 1)  // forced per-row paths (cross-checks)
    DDM_LAUNCH("emit", 24.0 * m + 8.0 * h.K + 12.0 * n, st, match::emit_kernel<match::kEmitD1><<<egrid, match::kRowTile, 0, st>>>(A));
  else
    DDM_LAUNCH("emit_dd", 44.0 * m + 8.0 * h.K, st, match::emit_kernel<match::kEmitDD><<<egrid, match::kRowTile, 0, st>>>(A));
  DDM_TRY(check_launch());
  return DDM_OK;
}

__global__ void encode_kernel(const double* __restrict__ x, uint64_t* __restrict__ k, uint64_t n) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) k[i] = f64_key(x[i]);
}

int bits_for(uint64_t v) {  // bits needed to represent v (0 -> 0)
  int b = 0;
  while (v) { ++b; v >>= 1; }
  return b;
}

// ------------------------------------------------------------ CUDA graphs
//
// The pre-sync half of a full match (validation, the three concurrent sort
// chains, counts, offset scan: ~35 launches and memsets over three streams)
// is captured into a CUDA graph the second time an identical call (same
// sizes, pointers, workspace, flags, stream) is made, and replayed from then
// on: one launch instead of dozens, which matters when the kernels are short
// (c1, c2).  Disabled while profiling or with DDM_GRAPHS=0 / DDM_SERIAL.

struct GraphEntry {
  cudaGraphExec_t exec = nullptr;
  int hits = 0;
  bool capturing = false;  // some thread is capturing this key right now
  bool failed = false;     // capture or instantiation failed: stay eager
  uint64_t launches = 0;   // kernels in the graph (for ddm_kernel_launch_count)
  uint64_t last_use = 0;
  ~GraphEntry() {
    // an in-flight executable graph is released once it completes
    if (exec) cudaGraphExecDestroy(exec);
  }
};
std::mutex g_graph_mu;
std::unordered_map<std::string, std::shared_ptr<GraphEntry>> g_graphs;
uint64_t g_graph_tick = 0;
constexpr size_t kMaxGraphs = 64;      // instantiated graphs kept (least recently used evicted)
constexpr size_t kMaxGraphKeys = 1024; // call sites tracked

bool graphs_enabled() {
  static const bool off = [] {
    const char* e = getenv("DDM_GRAPHS");
    return e && atoi(e) == 0;
  }();
  return !off && !serial_env() && !g_prof.on;
}

template <typename T>
void key_put(std::string& k, const T& v) { k.append(reinterpret_cast<const char*>(&v), sizeof(T)); }

std::string graph_key(const ddm_regions* R, const void* ws, size_t ws_bytes, uint32_t flags, bool want_pairs,
                      const uint32_t* sub_map, const uint32_t* upd_map, cudaStream_t st) {
  std::string k;
  int dev = 0;
  cudaGetDevice(&dev);
  key_put(k, dev);
  key_put(k, st);
  key_put(k, R->d);
  key_put(k, R->n_sub);
  key_put(k, R->n_upd);
  for (uint32_t i = 0; i < R->d; ++i) {
    key_put(k, R->sub_lo[i]);
    key_put(k, R->sub_hi[i]);
    key_put(k, R->upd_lo[i]);
    key_put(k, R->upd_hi[i]);
  }
  key_put(k, ws);
  key_put(k, ws_bytes);
  key_put(k, flags);
  key_put(k, want_pairs);
  key_put(k, sub_map);
  key_put(k, upd_map);
  return k;
}

// Bound the cache (g_graph_mu held): drop call sites never captured, then the
// least recently used instantiated graphs.  Entries are shared_ptrs, so a
// thread still using an evicted entry keeps it alive until it is done.
void graph_evict_locked() {
  if (g_graphs.size() > kMaxGraphKeys)
    for (auto it = g_graphs.begin(); it != g_graphs.end();)
      it = (!it->second->exec && !it->second->capturing) ? g_graphs.erase(it) : std::next(it);
  size_t live = 0;
  for (auto& kv : g_graphs) live += kv.second->exec != nullptr;
  while (live > kMaxGraphs) {
    auto victim = g_graphs.end();
    for (auto it = g_graphs.begin(); it != g_graphs.end(); ++it)
      if (it->second->exec && (victim == g_graphs.end() || it->second->last_use < victim->second->last_use))
        victim = it;
    if (victim == g_graphs.end()) break;
    g_graphs.erase(victim);
    --live;
  }
}

// Run pre(stream) -- enqueue-only work on `stream` and side streams joined
// back into it -- through the graph cache.  Capture happens on the calling
// thread's own capture stream (the caller's may be the legacy default stream,
// which cannot capture) with the thread's own side streams; the instantiated
// graph is then launched on the caller's stream.
template <typename F>
ddm_status run_cached(const std::string& key, F&& pre, cudaStream_t st) {
  std::shared_ptr<GraphEntry> e;
  bool capture = false;
  {
    std::lock_guard<std::mutex> lk(g_graph_mu);
    graph_evict_locked();
    std::shared_ptr<GraphEntry>& slot = g_graphs[key];
    if (!slot) slot = std::make_shared<GraphEntry>();
    slot->last_use = ++g_graph_tick;
    if (!slot->exec) {
      if (slot->failed || slot->capturing || ++slot->hits < 2) return pre(st);  // eager
      slot->capturing = capture = true;
    }
    e = slot;
  }
  if (capture) {
    auto give_up = [&]() {
      std::lock_guard<std::mutex> lk(g_graph_mu);
      e->capturing = false;
      e->failed = true;
    };
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) {
      give_up();
      return pre(st);
    }
    cudaStream_t& cs = t_streams.cap[dev];
    if (!cs && cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) != cudaSuccess) {
      cs = nullptr;
      give_up();
      return pre(st);
    }
    cudaStream_t side[2];
    if (side_streams(side, cs) != DDM_OK || side_stream_any(&side[1], cs) != DDM_OK) {  // created outside the capture
      give_up();
      return pre(st);
    }
    const uint64_t l0 = g_launches.load();
    if (cudaStreamBeginCapture(cs, cudaStreamCaptureModeRelaxed) != cudaSuccess) {
      cudaGetLastError();
      give_up();
      return pre(st);
    }
    const ddm_status r = pre(cs);
    cudaGraph_t g = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(cs, &g);
    const uint64_t nl = g_launches.load() - l0;
    g_launches.fetch_sub(nl);  // counted on every replay below instead
    cudaGraphExec_t x = nullptr;
    const bool ok = r == DDM_OK && ce == cudaSuccess && g && cudaGraphInstantiate(&x, g, 0) == cudaSuccess;
    if (g) cudaGraphDestroy(g);
    if (!ok) {
      cudaGetLastError();
      if (getenv("DDM_DEBUG")) fprintf(stderr, "libddm: graph capture failed (%d, %s)\n", (int)r, cudaGetErrorString(ce));
      give_up();
      return pre(st);  // plain launches
    }
    std::lock_guard<std::mutex> lk(g_graph_mu);
    e->exec = x;
    e->launches = nl;
    e->capturing = false;
  }
  DDM_CUDA(cudaGraphLaunch(e->exec, st));
  g_launches.fetch_add(e->launches);
  return DDM_OK;
}

}  // namespace

// ============================================================ C ABI

extern "C" {

size_t ddm_sub_index_bytes(uint32_t d, uint64_t n_sub) {
  if (d == 0 || d > DDM_MAX_DIMS) return 0;
  return index_layout(d, n_sub, nullptr).bytes;
}

// index build workspace: Misc, mm, the Slo / Shi MSD chains, LSB scratch
struct BuildWs {
  Misc* misc;
  uint64_t* mm;
  MsdScratch slo, shi;
  SortScratch lsb;
  size_t bytes;
};
static BuildWs build_layout(uint64_t n_sub, void* base) {
  Carver c(base);
  BuildWs B{};
  B.misc = c.take<Misc>(1);
  B.mm = c.take<uint64_t>(6);
  B.slo = msd_scratch(c, n_sub, true);
  B.shi = msd_scratch(c, n_sub, false);
  B.lsb = sort_scratch(c, n_sub, false);
  B.bytes = c.used;
  return B;
}

size_t ddm_index_build_workspace_bytes(uint32_t d, uint64_t n_sub) {
  if (d == 0 || d > DDM_MAX_DIMS) return 0;
  return build_layout(n_sub, nullptr).bytes;
}

size_t ddm_indexed_workspace_bytes(uint32_t d, uint64_t n_sub, uint64_t n_upd) {
  if (d == 0 || d > DDM_MAX_DIMS) return 0;
  return match_layout(d, n_sub, n_upd, nullptr, false).bytes;
}

size_t ddm_workspace_bytes(uint32_t d, uint64_t n_sub, uint64_t n_upd, int want_pairs) {
  (void)want_pairs;
  if (d == 0 || d > DDM_MAX_DIMS) return 0;
  return a256(index_layout(d, n_sub, nullptr).bytes) + match_layout(d, n_sub, n_upd, nullptr, true).bytes;
}

struct Probe {
  bool walk = false;
  bool pack_s = true, pack_u = true;
};
std::mutex g_probe_mu;
std::unordered_map<std::string, Probe> g_probe;  // count-form and packing decisions per call site

// k* for d > 1: the dimension with the fewest estimated
// candidate pairs (match::dim_probe_kernel), dimension 0 unless another one
// is estimated at least 10 % smaller.  Any choice gives the same pair set
// (the other dimensions are filtered exactly); it changes the work and the
// row order, so it is decided from the data on every call (one small
// device->host read) -- a decision cached per call site could be stale when
// new data arrives in the same buffers and would change the order.
static ddm_status sweep_dim(const ddm_regions* R, double* probe, cudaStream_t st, int* kout) {
  *kout = 0;
  match::ProbeDims P{};
  for (uint32_t k = 0; k < R->d; ++k) {
    P.sub_lo[k] = R->sub_lo[k]; P.sub_hi[k] = R->sub_hi[k]; P.upd_lo[k] = R->upd_lo[k]; P.upd_hi[k] = R->upd_hi[k];
  }
  DDM_LAUNCH("dim_probe", 0, st, match::dim_probe_kernel<<<R->d, 256, 0, st>>>(P, R->n_sub, R->n_upd, probe));
  DDM_TRY(check_launch());
  double est[DDM_MAX_DIMS];
  DDM_CUDA(cudaMemcpyAsync(est, probe, sizeof(double) * R->d, cudaMemcpyDeviceToHost, st));
  DDM_CUDA(cudaStreamSynchronize(st));
  int best = 0;
  for (uint32_t k = 1; k < R->d; ++k)
    if (est[k] < est[best]) best = (int)k;
  if (!(est[best] < 0.9 * est[0])) best = 0;
  if (getenv("DDM_DEBUG")) {
    fprintf(stderr, "libddm: sweep-dimension estimates");
    for (uint32_t k = 0; k < R->d; ++k) fprintf(stderr, " %g", est[k]);
    fprintf(stderr, " -> k* = %d\n", best);
  }
  *kout = best;
  return DDM_OK;
}

static ddm_status match_full_dim(const ddm_regions* R, ddm_pair* pairs, uint64_t capacity, uint64_t* count_out,
                                 uint32_t flags, void* ws, size_t ws_bytes, cudaStream_t st,
                                 const uint32_t* sub_map, const uint32_t* upd_map);

static ddm_status match_full(const ddm_regions* R, ddm_pair* pairs, uint64_t capacity, uint64_t* count_out,
                             uint32_t flags, void* ws, size_t ws_bytes, cudaStream_t st,
                             const uint32_t* sub_map = nullptr, const uint32_t* upd_map = nullptr) {
  DDM_TRY(check_regions(R, true, true));
  if (R->d > 1 && !(flags & DDM_SWEEP_DIM0) && R->n_sub > 0 && R->n_upd > 0 && ws &&
      ws_bytes >= ddm_workspace_bytes(R->d, R->n_sub, R->n_upd, pairs != nullptr)) {
    // the sweep dimension k*: swap it into position 0 (a view; the filter
    // tests every other dimension exactly, so the pair set is unchanged)
    MatchWs W = match_layout(R->d, R->n_sub, R->n_upd,
                             static_cast<uint8_t*>(ws) + a256(index_layout(R->d, R->n_sub, nullptr).bytes), true);
    int k = 0;
    DDM_TRY(sweep_dim(R, W.probe, st, &k));
    if (k != 0) {
      ddm_regions V = *R;
      std::swap(V.sub_lo[0], V.sub_lo[k]);
      std::swap(V.sub_hi[0], V.sub_hi[k]);
      std::swap(V.upd_lo[0], V.upd_lo[k]);
      std::swap(V.upd_hi[0], V.upd_hi[k]);
      return match_full_dim(&V, pairs, capacity, count_out, flags, ws, ws_bytes, st, sub_map, upd_map);
    }
  }
  return match_full_dim(R, pairs, capacity, count_out, flags, ws, ws_bytes, st, sub_map, upd_map);
}

static ddm_status match_full_dim(const ddm_regions* R, ddm_pair* pairs, uint64_t capacity, uint64_t* count_out,
                                 uint32_t flags, void* ws, size_t ws_bytes, cudaStream_t st,
                                 const uint32_t* sub_map, const uint32_t* upd_map) {
  if (!count_out || (!ws && ws_bytes) || !aligned(ws, 256)) return DDM_ERR_INVALID_ARGUMENT;
  if (pairs && !aligned(pairs, 8)) return DDM_ERR_INVALID_ARGUMENT;
  if (ws_bytes < ddm_workspace_bytes(R->d, R->n_sub, R->n_upd, pairs != nullptr)) return DDM_ERR_WORKSPACE;
  uint8_t* base = static_cast<uint8_t*>(ws);
  Index I = index_layout(R->d, R->n_sub, base);
  MatchWs W = match_layout(R->d, R->n_sub, R->n_upd, base + a256(I.bytes), true);
  MatchReq q{&I, R, upd_map, pairs, capacity, flags, sub_map};
  // d > 1 with the row-indexed filter: only float boxes are built (no float64
  // coordinates gathered into sweep order; exact tests read them by id)
  q.boxes_only = R->d > 1 && R->n_sub > 0 && R->n_upd > 0 &&
                 !(flags & (DDM_EMIT_FORCE_THREAD | DDM_EMIT_FORCE_WARP)) && dd_rows_enabled(R->n_upd, flags);
  const bool lsb_only = (flags & DDM_SORT_LSB) != 0;
  // count form (ddm.h DDM_COUNT_RANKS / DDM_COUNT_WALK): d > 1 always ranks
  // (its dim-0 candidates outnumber the pairs); d = 1 pairs calls walk when
  // forced, or when the probe finds sparse stab sets on a big input (the
  // walk replaces the Shi sort, ~1/3 of the sort traffic)
  // One probe of 4096 sampled regions per kind decides, per call site, the
  // count form of d = 1 pairs calls (mean stab size) and whether the big
  // sorts pack their records (sampled upper-key deltas that fit 32 bits).
  // The decisions are kept per call site (regions, workspace, flags, stream):
  // repeated calls -- graph replays -- skip the probe and its host read; every
  // choice gives the same output, so a stale decision costs time only.
  const bool walk_open = pairs && R->d == 1 && !(flags & (DDM_COUNT_RANKS | DDM_COUNT_WALK)) &&
                         R->n_sub >= kWalkMinN && R->n_upd > 0;
  const bool pack_open = DDM_MSD_PACK == 2 && (R->n_sub >= kPackMinN || R->n_upd >= kPackMinN) && R->n_sub > 0 &&
                         R->n_upd > 0;
  bool walk = pairs && R->d == 1 && (flags & DDM_COUNT_WALK) && !(flags & DDM_COUNT_RANKS);
  int pack_s = -1, pack_u = -1;
  if (walk_open || pack_open) {
    const std::string pk = graph_key(R, ws, ws_bytes, flags, pairs != nullptr, sub_map, upd_map, st);
    Probe pr{};
    bool known = false;
    {
      std::lock_guard<std::mutex> lk(g_probe_mu);
      const auto it = g_probe.find(pk);
      if (it != g_probe.end()) {
        pr = it->second;
        known = true;
      }
    }
    if (!known) {
      double est[3] = {INFINITY, 0.0, 0.0};
      DDM_LAUNCH("stab_probe", 0, st, match::stab_density_kernel<<<1, 256, 0, st>>>(
          R->sub_lo[0], R->sub_hi[0], R->n_sub, R->upd_lo[0], R->upd_hi[0], R->n_upd, W.probe));
      DDM_TRY(check_launch());
      DDM_CUDA(cudaMemcpyAsync(est, W.probe, 3 * sizeof(double), cudaMemcpyDeviceToHost, st));
      DDM_CUDA(cudaStreamSynchronize(st));
      pr.walk = est[0] <= kWalkMaxStab;
      pr.pack_s = est[1] <= kPackMaxUnfit;
      pr.pack_u = est[2] <= kPackMaxUnfit;
      std::lock_guard<std::mutex> lk(g_probe_mu);
      if (g_probe.size() > 4096) g_probe.clear();
      g_probe[pk] = pr;
    }
    if (walk_open) walk = pr.walk;
    if (pack_open) {
      pack_s = pr.pack_s;
      pack_u = pr.pack_u;
    }
  }
  const PackScope pack_scope(pack_s, pack_u);
  const uint32_t key_flags = (flags & ~(uint32_t)(DDM_COUNT_RANKS | DDM_COUNT_WALK)) |
                             (walk ? DDM_COUNT_WALK : DDM_COUNT_RANKS);
  const OneChain one_chain(walk);
  for (int attempt = lsb_only ? 1 : 0; attempt < 2; ++attempt) {
    const bool use_msd = attempt == 0;
    const int need = (walk || q.boxes_only) ? kNeedPm : (pairs || R->d != 1) ? kNeedShi : (kNeedShi | kNeedKeysOnly);
    q.walk = need == kNeedPm;
    auto pre = [&](cudaStream_t s) -> ddm_status {
      DDM_CUDA(cudaMemsetAsync(W.misc, 0, sizeof(Misc), s));
      DDM_TRY(init_minmax(W.mm, s));
      if (use_msd && walk) {
        // walk form: the two record chains run one after the other at full
        // occupancy; the update chain's latency-bound preparation (sample,
        // bucket map, histograms) overlaps the Slo chain on a side stream
        cudaStream_t s1;
        DDM_TRY(side_stream_any(&s1, s));
        DDM_TRY(stream_join(s1, s));
        DDM_TRY(upd_sort_async(R, W, R->n_sub, true, s1, kMsdPrep));
        DDM_TRY(build_index_async(R, I, W.slo, W.shi, W.sort, W.mm, W.misc, true, s, need, q.boxes_only));
        DDM_TRY(stream_join(s, s1));
        DDM_TRY(upd_sort_async(R, W, R->n_sub, true, s, kMsdRun));
      } else if (use_msd) {
        // the update chain (side stream 1) runs concurrently with the index
        // build (Slo on s, Shi on side stream 0); s joins both before a4
        cudaStream_t side[2];
        DDM_TRY(side_streams(side, s));
        DDM_TRY(stream_join(side[1], s));
        DDM_TRY(upd_sort_async(R, W, R->n_sub, true, side[1], kMsdAll, q.boxes_only ? 3u : 1u));
        DDM_TRY(build_index_async(R, I, W.slo, W.shi, W.sort, W.mm, W.misc, true, s, need, q.boxes_only));
        DDM_TRY(stream_join(s, side[1]));
      } else {
        DDM_TRY(build_index_async(R, I, W.slo, W.shi, W.sort, W.mm, W.misc, false, s, need, q.boxes_only));
        DDM_TRY(upd_sort_async(R, W, R->n_sub, false, s));
      }
      return match_sorted(q, W, count_out, use_msd, s, kPhasePre);
    };
    init_attrs_once();
    if (use_msd && graphs_enabled())
      DDM_TRY(run_cached(graph_key(R, ws, ws_bytes, key_flags, pairs != nullptr, sub_map, upd_map, st), pre, st));
    else
      DDM_TRY(pre(st));
    const ddm_status r = match_sorted(q, W, count_out, use_msd, st, kPhasePost);
    if (r != kRetryLSB) return r;
  }
  return DDM_ERR_CUDA;
}

ddm_status ddm_chunk_start_sets(const ddm_regions* R, uint32_t* first_upd, uint64_t* set_off, uint32_t* set_ids,
                                uint64_t capacity, uint64_t* total_out, void* ws, size_t ws_bytes,
                                cudaStream_t st) {
  DDM_TRY(check_regions(R, true, true));
  if (R->d != 1 || !total_out || !aligned(ws, 256)) return DDM_ERR_INVALID_ARGUMENT;
  if (R->n_upd && (!first_upd || !set_off || (capacity && !set_ids))) return DDM_ERR_INVALID_ARGUMENT;
  if (ws_bytes < ddm_workspace_bytes(R->d, R->n_sub, R->n_upd, 1)) return DDM_ERR_WORKSPACE;
  *total_out = 0;
  if (R->n_upd == 0 || R->n_sub == 0) {
    const uint64_t tiles = (R->n_upd + match::kRowTile - 1) / match::kRowTile;
    if (tiles) DDM_CUDA(cudaMemsetAsync(set_off, 0, sizeof(uint64_t) * (tiles + 1), st));
    // (first_upd of an empty-index tile still names its first update: not needed by callers)
    uint64_t k = 0;
    ddm_pair dummy;
    ddm_status r = match_full(R, &dummy, 0, &k, DDM_COUNT_RANKS, ws, ws_bytes, st);  // validation only
    return r == DDM_ERR_CAPACITY ? DDM_OK : r;
  }
  init_attrs_once();
  uint8_t* base = static_cast<uint8_t*>(ws);
  Index I = index_layout(R->d, R->n_sub, base);
  MatchWs W = match_layout(R->d, R->n_sub, R->n_upd, base + a256(I.bytes), true);
  ChunkExport C{first_upd, set_off, set_ids, capacity, total_out};
  ddm_pair dummy;
  MatchReq q{&I, R, nullptr, &dummy, 0, DDM_COUNT_RANKS};
  q.chunk = &C;
  uint64_t K = 0;
  for (int attempt = 0; attempt < 2; ++attempt) {
    const bool use_msd = attempt == 0;
    DDM_CUDA(cudaMemsetAsync(W.misc, 0, sizeof(Misc), st));
    DDM_TRY(init_minmax(W.mm, st));
    DDM_TRY(build_index_async(R, I, W.slo, W.shi, W.sort, W.mm, W.misc, use_msd, st, kNeedShi));
    DDM_TRY(upd_sort_async(R, W, R->n_sub, use_msd, st));
    DDM_TRY(match_sorted(q, W, &K, use_msd, st, kPhasePre));
    const ddm_status r = match_sorted(q, W, &K, use_msd, st, kPhasePost);
    if (r != kRetryLSB) return r;
  }
  return DDM_ERR_CUDA;
}

ddm_status ddm_match_count(const ddm_regions* regions, uint64_t* count_out, void* ws, size_t ws_bytes,
                           cudaStream_t stream) {
  return match_full(regions, nullptr, 0, count_out, 0, ws, ws_bytes, stream);
}

ddm_status ddm_match_pairs(const ddm_regions* regions, ddm_pair* pairs, uint64_t capacity,
                           uint64_t* count_out, uint32_t flags, void* ws, size_t ws_bytes,
                           cudaStream_t stream) {
  if (!pairs && capacity) return DDM_ERR_INVALID_ARGUMENT;
  ddm_pair dummy;
  return match_full(regions, pairs ? pairs : &dummy, pairs ? capacity : 0, count_out, flags, ws, ws_bytes,
                    stream);
}

ddm_status ddm_match_pairs_mapped(const ddm_regions* regions, const uint32_t* sub_ids, const uint32_t* upd_ids,
                                  ddm_pair* pairs, uint64_t capacity, uint64_t* count_out, uint32_t flags,
                                  void* ws, size_t ws_bytes, cudaStream_t stream) {
  if (!pairs && capacity) return DDM_ERR_INVALID_ARGUMENT;
  ddm_pair dummy;
  return match_full(regions, pairs ? pairs : &dummy, pairs ? capacity : 0, count_out, flags, ws, ws_bytes, stream,
                    sub_ids, upd_ids);
}

ddm_status ddm_sub_index_build(const ddm_regions* subs, void* index, size_t index_bytes, void* ws,
                               size_t ws_bytes, cudaStream_t stream) {
  DDM_TRY(check_regions(subs, true, false));
  if (!index || !aligned(index, 256) || !aligned(ws, 256)) return DDM_ERR_INVALID_ARGUMENT;
  if (index_bytes < ddm_sub_index_bytes(subs->d, subs->n_sub)) return DDM_ERR_WORKSPACE;
  if (ws_bytes < ddm_index_build_workspace_bytes(subs->d, subs->n_sub)) return DDM_ERR_WORKSPACE;
  Index I = index_layout(subs->d, subs->n_sub, index);
  BuildWs B = build_layout(subs->n_sub, ws);
  Misc h{};
  for (int attempt = 0; attempt < 2; ++attempt) {
    const bool use_msd = attempt == 0;
    DDM_CUDA(cudaMemsetAsync(B.misc, 0, sizeof(Misc), stream));
    DDM_TRY(init_minmax(B.mm, stream));
    DDM_TRY(build_index_async(subs, I, B.slo, B.shi, B.lsb, B.mm, B.misc, use_msd, stream));
    DDM_CUDA(cudaMemcpyAsync(&h, B.misc, sizeof(Misc), cudaMemcpyDeviceToHost, stream));
    DDM_CUDA(cudaStreamSynchronize(stream));
    if (h.err || !h.overflow) break;
  }
  return err_status(h.err);
}

static ddm_status indexed_common(const void* index, const ddm_regions* upds, const uint32_t* upd_ids,
                                 ddm_pair* pairs, uint64_t capacity, uint64_t* count_out, uint32_t flags,
                                 void* ws, size_t ws_bytes, cudaStream_t st) {
  DDM_TRY(check_regions(upds, false, true));
  if (!index || !count_out || !aligned(index, 256) || !aligned(ws, 256)) return DDM_ERR_INVALID_ARGUMENT;
  if (upds->n_sub > DDM_MAX_REGIONS) return DDM_ERR_INVALID_ARGUMENT;
  if (ws_bytes < ddm_indexed_workspace_bytes(upds->d, upds->n_sub, upds->n_upd)) return DDM_ERR_WORKSPACE;
  Index I = index_layout(upds->d, upds->n_sub, const_cast<void*>(index));
  MatchWs W = match_layout(upds->d, upds->n_sub, upds->n_upd, ws, false);
  MatchReq q{&I, upds, upd_ids, pairs, capacity, flags};
  // the index keeps both Shi and the prefix maxima; ranks are cheaper here
  q.walk = pairs && upds->d == 1 && (flags & DDM_COUNT_WALK) && !(flags & DDM_COUNT_RANKS);
  for (int attempt = (flags & DDM_SORT_LSB) ? 1 : 0; attempt < 2; ++attempt) {
    const bool use_msd = attempt == 0;
    DDM_CUDA(cudaMemsetAsync(W.misc, 0, sizeof(Misc), st));
    DDM_TRY(init_minmax(W.mm, st));
    DDM_TRY(upd_sort_async(upds, W, upds->n_sub, use_msd, st));
    const ddm_status r = match_sorted(q, W, count_out, use_msd, st);
    if (r != kRetryLSB) return r;
  }
  return DDM_ERR_CUDA;
}

ddm_status ddm_match_pairs_indexed(const void* index, const ddm_regions* upds, const uint32_t* upd_ids,
                                   ddm_pair* pairs, uint64_t capacity, uint64_t* count_out, uint32_t flags,
                                   void* ws, size_t ws_bytes, cudaStream_t stream) {
  if (!pairs && capacity) return DDM_ERR_INVALID_ARGUMENT;
  ddm_pair dummy;
  return indexed_common(index, upds, upd_ids, pairs ? pairs : &dummy, pairs ? capacity : 0, count_out, flags,
                        ws, ws_bytes, stream);
}

ddm_status ddm_match_count_indexed(const void* index, const ddm_regions* upds, uint64_t* count_out, void* ws,
                                   size_t ws_bytes, cudaStream_t stream) {
  return indexed_common(index, upds, nullptr, nullptr, 0, count_out, 0, ws, ws_bytes, stream);
}

// ------------------------------------------------------------ dynamic DDM (dyn.cuh)

struct DynWs {
  uint32_t* bad;
  uint32_t* bits;   // moved-id bitmap
  uint32_t* w;      // Slo: keep + insertion histogram, [n + 1]
  uint32_t* E;      // its exclusive scan
  uint32_t* wsh;     // Shi: the same
  uint32_t* Es;
  uint8_t* ks;      // Shi keep flags
  uint64_t* tsum;
  uint64_t* toff;
  uint64_t* scan_status;
  uint64_t* rhi;
  uint64_t* rhi_sorted;
  uint64_t* nkey;
  uint32_t* nidx;
  uint64_t* nhi;
  uint32_t* p;      // Slo insertion points
  uint32_t* ps;     // Shi insertion points
  SortScratch sort;
  uint8_t* copy;    // in-place updates: a copy of the old index
  size_t bytes;
};

static DynWs dyn_layout(uint32_t d, uint64_t n, uint64_t k, bool in_place, void* base) {
  Carver c(base);
  DynWs W{};
  const uint64_t tiles = (n + 1) / dyn::kTile + 2;
  W.bad = c.take<uint32_t>(4);
  W.bits = c.take<uint32_t>(n / 32 + 1);
  W.w = c.take<uint32_t>(n + 1);
  W.E = c.take<uint32_t>(n + 1);
  W.wsh = c.take<uint32_t>(n + 1);
  W.Es = c.take<uint32_t>(n + 1);
  W.ks = c.take<uint8_t>(n);
  W.tsum = c.take<uint64_t>(tiles);
  W.toff = c.take<uint64_t>(tiles);
  W.scan_status = c.take<uint64_t>(tiles / (match::kScanThreads * match::kScanItems) + 2);
  W.rhi = c.take<uint64_t>(k);
  W.rhi_sorted = c.take<uint64_t>(k);
  W.nkey = c.take<uint64_t>(k);
  W.nidx = c.take<uint32_t>(k);
  W.nhi = c.take<uint64_t>(k);
  W.p = c.take<uint32_t>(k);
  W.ps = c.take<uint32_t>(k);
  W.sort = sort_scratch(c, k, true);
  W.copy = in_place ? c.take<uint8_t>(index_layout(d, n, nullptr).bytes) : nullptr;
  W.bytes = c.used;
  return W;
}

// E[i] = sum(w[0..i)), i = 0..len-1
static ddm_status excl_scan_u32(const uint32_t* w, uint64_t len, uint32_t* E, DynWs& W, cudaStream_t st) {
  const uint64_t tiles = (len + dyn::kTile - 1) / dyn::kTile;
  DDM_LAUNCH("dyn_scan", 4.0 * len, st, dyn::tile_sum_kernel<<<(unsigned)tiles, 256, 0, st>>>(w, len, W.tsum));
  DDM_TRY(check_launch());
  const unsigned stiles = (unsigned)((tiles + match::kScanThreads * match::kScanItems - 1) /
                                     (match::kScanThreads * match::kScanItems));
  DDM_CUDA(cudaMemsetAsync(W.scan_status, 0, sizeof(uint64_t) * (stiles + 1), st));
  DDM_LAUNCH("scan", 16.0 * tiles, st, match::scan_u64_kernel<<<stiles, match::kScanThreads, 0, st>>>(
      W.tsum, tiles, W.toff, W.scan_status, nullptr));
  DDM_TRY(check_launch());
  DDM_LAUNCH("dyn_scan", 8.0 * len, st, dyn::excl_scan_kernel<<<(unsigned)tiles, 256, 0, st>>>(w, len, W.toff, E));
  return check_launch();
}

extern "C" size_t ddm_sub_index_update_workspace_bytes(uint32_t d, uint64_t n_sub, uint64_t k, int in_place) {
  if (d == 0 || d > DDM_MAX_DIMS) return 0;
  return dyn_layout(d, n_sub, k, in_place != 0, nullptr).bytes;
}

extern "C" ddm_status ddm_sub_index_update(const void* index_in, void* index_out, size_t index_bytes, uint64_t n_sub,
                                           const ddm_regions* moved, const uint32_t* ids, void* ws, size_t ws_bytes,
                                           cudaStream_t st) {
  DDM_TRY(check_regions(moved, true, false));
  const uint32_t d = moved->d;
  const uint64_t n = n_sub, k = moved->n_sub;
  const bool in_place = index_in == index_out;
  if (!index_in || !index_out || !aligned(index_in, 256) || !aligned(index_out, 256) || !aligned(ws, 256) ||
      (k && !ids) || k > n)
    return DDM_ERR_INVALID_ARGUMENT;
  const size_t ib = ddm_sub_index_bytes(d, n);
  if (index_bytes < ib) return DDM_ERR_WORKSPACE;
  if (ws_bytes < ddm_sub_index_update_workspace_bytes(d, n, k, in_place ? 1 : 0)) return DDM_ERR_WORKSPACE;
  init_attrs_once();
  DynWs W = dyn_layout(d, n, k, in_place, ws);
  DDM_CUDA(cudaMemsetAsync(W.bad, 0, 4 * sizeof(uint32_t), st));
  // errors are reported before anything is written
  DDM_TRY(validate_side(d, k, moved->sub_lo, moved->sub_hi, nullptr, nullptr, W.bad + 1, st));
  DDM_CUDA(cudaMemsetAsync(W.bits, 0, sizeof(uint32_t) * (n / 32 + 1), st));
  if (k) {
    DDM_LAUNCH("dyn_mark", 0, st, dyn::mark_kernel<<<grid_for(k, 256, 8), 256, 0, st>>>(ids, k, n, W.bits, W.bad));
    DDM_TRY(check_launch());
  }
  {
    uint32_t h[2] = {0, 0};
    DDM_CUDA(cudaMemcpyAsync(h, W.bad, sizeof(h), cudaMemcpyDeviceToHost, st));
    DDM_CUDA(cudaStreamSynchronize(st));
    if (h[0]) return DDM_ERR_INVALID_ARGUMENT;  // ids not strictly increasing or out of range
    DDM_TRY(err_status(h[1]));
  }
  if (k == 0) {
    if (!in_place) DDM_CUDA(cudaMemcpyAsync(index_out, index_in, ib, cudaMemcpyDeviceToDevice, st));
    return DDM_OK;
  }
  const void* src = index_in;
  if (in_place) {
    DDM_CUDA(cudaMemcpyAsync(W.copy, index_in, ib, cudaMemcpyDeviceToDevice, st));
    src = W.copy;
  }
  const Index O = index_layout(d, n, const_cast<void*>(src));
  Index I = index_layout(d, n, index_out);
  // Slo: keep flags + the moved entries' old upper keys
  DDM_LAUNCH("dyn_tomb", 16.0 * n, st, dyn::tomb_kernel<<<grid_for(n, 256, 8), 256, 0, st>>>(
      O.slo_id, O.slo_hi, n, W.bits, ids, k, W.w, W.rhi));
  DDM_TRY(check_launch());
  // Shi: keep flags from the sorted removed keys
  const radix::PassList P = full_passes();
  DDM_TRY(radix_sort(W.rhi, false, nullptr, W.rhi_sorted, nullptr, k, P, W.sort.hist[0], false, W.sort, st));
  DDM_LAUNCH("dyn_fill", 4.0 * n, st, dyn::fill_one_kernel<<<grid_for(n + 1, 256, 8), 256, 0, st>>>(W.wsh, n));
  DDM_TRY(check_launch());
  DDM_CUDA(cudaMemsetAsync(W.ks, 1, n, st));
  DDM_LAUNCH("dyn_tomb", 0, st, dyn::shi_tomb_kernel<<<grid_for(k, 256, 8), 256, 0, st>>>(W.rhi_sorted, k, O.shi_key, n,
                                                                                          W.wsh, W.ks));
  DDM_TRY(check_launch());
  // the new entries sorted on their own -- (lower key, input index), which is
  // (key, id) order as the ids increase -- and their insertion points
  DDM_TRY(radix_sort(moved->sub_lo[0], true, nullptr, W.nkey, W.nidx, k, P, W.sort.hist[0], false, W.sort, st));
  DDM_TRY(radix_sort(moved->sub_hi[0], true, nullptr, W.nhi, nullptr, k, P, W.sort.hist[0], false, W.sort, st));
  DDM_LAUNCH("dyn_ins", 0, st, dyn::slo_ins_kernel<<<grid_for(k, 256, 8), 256, 0, st>>>(O.slo_key, O.slo_id, n, W.nkey,
                                                                                         W.nidx, ids, k, W.p, W.w));
  DDM_TRY(check_launch());
  DDM_LAUNCH("dyn_ins", 0, st, dyn::shi_ins_kernel<<<grid_for(k, 256, 8), 256, 0, st>>>(O.shi_key, n, W.nhi, k, W.ps,
                                                                                         W.wsh));
  DDM_TRY(check_launch());
  DDM_TRY(excl_scan_u32(W.w, n + 1, W.E, W, st));
  DDM_TRY(excl_scan_u32(W.wsh, n + 1, W.Es, W, st));
  // merge: every element written once to its final position
  dyn::SloArgs A{};
  A.okey = O.slo_key;
  A.oid = O.slo_id;
  A.ohi = O.slo_hi;
  A.osd = O.sdims;
  A.bits = W.bits;
  A.w = W.w;
  A.E = W.E;
  A.n = n;
  A.nkey = W.nkey;
  A.nidx = W.nidx;
  A.ids = ids;
  A.p = W.p;
  for (uint32_t kk = 0; kk < d; ++kk) {
    A.new_lo[kk] = moved->sub_lo[kk];
    A.new_hi[kk] = moved->sub_hi[kk];
  }
  A.k = k;
  A.d = (int)d;
  A.key = I.slo_key;
  A.id = I.slo_id;
  A.hi = I.slo_hi;
  A.sd = I.sdims;
  DDM_LAUNCH("dyn_merge", (28.0 + 32.0 * (d - 1)) * n, st, dyn::slo_old_kernel<<<grid_for(n, 256, 8), 256, 0, st>>>(A));
  DDM_TRY(check_launch());
  DDM_LAUNCH("dyn_merge", 0, st, dyn::slo_new_kernel<<<grid_for(k, 256, 8), 256, 0, st>>>(A));
  DDM_TRY(check_launch());
  DDM_LAUNCH("dyn_merge", 25.0 * n, st, dyn::shi_merge_kernel<<<grid_for(n + k, 256, 8), 256, 0, st>>>(
      O.shi_key, W.wsh, W.Es, W.ks, n, W.nhi, W.ps, k, I.shi_key));
  DDM_TRY(check_launch());
  // derived structures, as the build computes them
  DDM_TRY(tree_async(I, kNeedShi | kNeedPm, false, st));
  if (d > 1) {
    DDM_LAUNCH("dd_boxes", 32.0 * n, st, dd::box_kernel<<<grid_for(n, 256, 8), 256, 0, st>>>(I.sdims, (int)d, n, I.box12,
                                                                                              nullptr, I.slo_key, I.slo_hi, I.box0, nullptr, nullptr));
    DDM_TRY(check_launch());
  }
  return check_launch();
}

// ------------------------------------------------------------ event-order variant (events.cuh)

struct EvWs {
  uint64_t N2 = 0, P = 0;
  uint64_t* key0;
  uint32_t* code0;
  uint64_t* tkey;
  uint32_t* tcode;
  SortScratch sort;
  uint32_t* posH;
  uint64_t* hp;
  int levels = 0;
  uint64_t lvl_n[kMaxLevels + 1] = {};
  uint64_t* lvl[kMaxLevels + 1] = {};
  uint64_t* seg_uppers;
  uint64_t* ub;  // uppers before each segment (exclusive scan)
  uint64_t* scan_status;
  uint64_t* misc;  // [0] cursor / K, [1] error word
  size_t bytes = 0;
};

static EvWs ev_layout(uint64_t n, uint64_t m, void* base) {
  Carver c(base);
  EvWs E;
  E.N2 = 2 * (n + m);
  E.P = (E.N2 + ev::kSeg - 1) / ev::kSeg;
  E.misc = c.take<uint64_t>(2);
  E.key0 = c.take<uint64_t>(E.N2);
  E.code0 = c.take<uint32_t>(E.N2);
  E.tkey = c.take<uint64_t>(E.N2);
  E.tcode = c.take<uint32_t>(E.N2);
  E.sort = sort_scratch(c, E.N2, true);
  E.posH = c.take<uint32_t>(n + m);
  E.hp = c.take<uint64_t>(E.N2);
  E.lvl[0] = E.hp;
  E.lvl_n[0] = E.N2;
  uint64_t sz = E.N2;
  while (sz > 1 && E.levels < kMaxLevels) {
    sz = (sz + 31) / 32;
    ++E.levels;
    E.lvl_n[E.levels] = sz;
    E.lvl[E.levels] = c.take<uint64_t>(sz);
  }
  E.seg_uppers = c.take<uint64_t>(E.P + 1);
  E.ub = c.take<uint64_t>(E.P + 1);
  E.scan_status = c.take<uint64_t>(E.P / (match::kScanThreads * match::kScanItems) + 2);
  E.bytes = c.used;
  return E;
}

extern "C" size_t ddm_events_workspace_bytes(uint32_t d, uint64_t n_sub, uint64_t n_upd) {
  if (d == 0 || d > DDM_MAX_DIMS) return 0;
  return ev_layout(n_sub, n_upd, nullptr).bytes;
}

extern "C" ddm_status ddm_match_pairs_events(const ddm_regions* R, ddm_pair* pairs, uint64_t capacity,
                                             uint64_t* count_out, void* ws, size_t ws_bytes, cudaStream_t st) {
  DDM_TRY(check_regions(R, true, true));
  if (!count_out || !aligned(ws, 256) || (pairs && !aligned(pairs, 8))) return DDM_ERR_INVALID_ARGUMENT;
  if (2 * (R->n_sub + R->n_upd) > DDM_MAX_SORT_KEYS) return DDM_ERR_INVALID_ARGUMENT;  // one endpoint sort
  if (ws_bytes < ddm_events_workspace_bytes(R->d, R->n_sub, R->n_upd)) return DDM_ERR_WORKSPACE;
  init_attrs_once();
  const uint64_t n = R->n_sub, m = R->n_upd;
  EvWs E = ev_layout(n, m, ws);
  uint32_t* err = reinterpret_cast<uint32_t*>(E.misc + 1);
  DDM_CUDA(cudaMemsetAsync(E.misc, 0, 2 * sizeof(uint64_t), st));
  // a1 on every dimension of both sides
  DDM_TRY(validate_side(R->d, n, R->sub_lo, R->sub_hi, nullptr, nullptr, err, st));
  DDM_TRY(validate_side(R->d, m, R->upd_lo, R->upd_hi, nullptr, nullptr, err, st));
  uint64_t h[2] = {0, 0};
  if (n && m) {
    // T: one stable sort of [S lowers | U lowers | S uppers | U uppers] (8 LSB passes)
    DDM_LAUNCH("ev_build", 16.0 * E.N2, st, ev::build_kernel<<<grid_for(E.N2, 256, 8), 256, 0, st>>>(
        R->sub_lo[0], R->sub_hi[0], R->upd_lo[0], R->upd_hi[0], n, m, E.key0, E.code0));
    DDM_TRY(check_launch());
    DDM_TRY(radix_sort(E.key0, false, E.code0, E.tkey, E.tcode, E.N2, full_passes(), E.sort.hist[0], false, E.sort, st));
    DDM_LAUNCH("ev_pos", 8.0 * E.N2, st, ev::pos_kernel<<<(unsigned)E.P, 256, 0, st>>>(E.tcode, E.N2, n, E.posH,
                                                                                       E.seg_uppers));
    DDM_TRY(check_launch());
    DDM_LAUNCH("ev_hp", 16.0 * E.N2, st, ev::hp_kernel<<<grid_for(E.N2, 256, 8), 256, 0, st>>>(
        E.tcode, E.N2, n, E.posH, E.hp, E.levels ? E.lvl[1] : nullptr));
    DDM_TRY(check_launch());
    for (int L = 2; L <= E.levels; ++L) {
      DDM_LAUNCH("block_max", 8.0 * E.lvl_n[L - 1], st, match::block_max_kernel<<<grid_for(E.lvl_n[L - 1], 256, 8), 256, 0, st>>>(
          E.lvl[L - 1], E.lvl_n[L - 1], E.lvl[L]));
      DDM_TRY(check_launch());
    }
    // Alg. 6's combine in counting form: uppers before each segment
    const unsigned stiles = (unsigned)((E.P + match::kScanThreads * match::kScanItems - 1) /
                                       (match::kScanThreads * match::kScanItems));
    DDM_CUDA(cudaMemsetAsync(E.scan_status, 0, sizeof(uint64_t) * (stiles + 1), st));
    DDM_LAUNCH("scan", 16.0 * E.P, st, match::scan_u64_kernel<<<stiles, match::kScanThreads, 0, st>>>(
        E.seg_uppers, E.P, E.ub, E.scan_status, nullptr));
    DDM_TRY(check_launch());
    ev::Args A{};
    A.code = E.tcode;
    A.hp = E.hp;
    for (int L = 0; L <= E.levels; ++L) A.T.lvl[L] = E.lvl[L];
    A.T.levels = E.levels;
    A.ub = E.ub;
    A.N2 = E.N2;
    A.X.d = (int)R->d;
    for (uint32_t k = 0; k < R->d; ++k) {
      A.X.sub_lo[k] = R->sub_lo[k];
      A.X.sub_hi[k] = R->sub_hi[k];
      A.X.upd_lo[k] = R->upd_lo[k];
      A.X.upd_hi[k] = R->upd_hi[k];
    }
    A.cursor = reinterpret_cast<unsigned long long*>(E.misc);
    DDM_LAUNCH("ev_count", 0, st, ev::segment_kernel<false><<<(unsigned)E.P, ev::kThreads, sizeof(ev::Smem), st>>>(A));
    DDM_TRY(check_launch());
    DDM_CUDA(cudaMemcpyAsync(h, E.misc, sizeof(h), cudaMemcpyDeviceToHost, st));
    DDM_CUDA(cudaStreamSynchronize(st));
    *count_out = h[0];
    DDM_TRY(err_status((uint32_t)h[1]));
    if (!pairs || h[0] == 0) return DDM_OK;
    if (h[0] > capacity) return DDM_ERR_CAPACITY;
    DDM_CUDA(cudaMemsetAsync(E.misc, 0, sizeof(uint64_t), st));
    A.pairs = reinterpret_cast<uint2*>(pairs);
    A.capacity = capacity;
    DDM_LAUNCH("ev_emit", 8.0 * h[0], st, ev::segment_kernel<true><<<(unsigned)E.P, ev::kThreads, sizeof(ev::Smem), st>>>(A));
    return check_launch();
  }
  DDM_CUDA(cudaMemcpyAsync(h, E.misc, sizeof(h), cudaMemcpyDeviceToHost, st));
  DDM_CUDA(cudaStreamSynchronize(st));
  *count_out = 0;
  return err_status((uint32_t)h[1]);
}

// ------------------------------------------------------------ multi-GPU slab partition (slab.cuh)

namespace {
struct SlabWs {
  uint64_t tiles = 0;
  uint64_t* cnt;       // [world][tiles]
  uint64_t* off;       // [world * tiles + 1]
  uint64_t* status;
  uint64_t* misc;      // [world + 1] segment starts + total, then the error word
  size_t bytes;
};
SlabWs slab_layout(uint64_t count, uint32_t world, void* base) {
  Carver c(base);
  SlabWs W;
  W.tiles = (count + slab::kTile - 1) / slab::kTile;
  const uint64_t T = W.tiles * world;
  W.cnt = c.take<uint64_t>(T + 1);
  W.off = c.take<uint64_t>(T + 1);
  W.status = c.take<uint64_t>(T / (match::kScanThreads * match::kScanItems) + 2);
  W.misc = c.take<uint64_t>(world + 2);
  W.bytes = c.used;
  return W;
}
__global__ void slab_seg_starts_kernel(const uint64_t* __restrict__ off, uint64_t tiles, uint32_t world,
                                       uint64_t* __restrict__ misc) {
  const uint32_t r = threadIdx.x;
  if (r <= world) misc[r] = off[(uint64_t)r * tiles];  // off[world * tiles] = total
}
}  // namespace

ddm_status ddm_slab_sample(const double* lo0, uint64_t count, double* sample, uint32_t s, cudaStream_t st) {
  if (!sample || s == 0 || (count && !lo0)) return DDM_ERR_INVALID_ARGUMENT;
  DDM_LAUNCH("slab_sample", 8.0 * s, st, slab::sample_kernel<<<(s + 255) / 256, 256, 0, st>>>(lo0, count, s, sample));
  return check_launch();
}

ddm_status ddm_slab_cuts(const double* sample, uint32_t s, uint32_t world, double* cuts, cudaStream_t st) {
  if (world < 1 || world > slab::kMaxWorld || s == 0 || s > (uint32_t)slab::kMaxSample || !sample)
    return DDM_ERR_INVALID_ARGUMENT;
  if (world == 1) return DDM_OK;
  if (!cuts) return DDM_ERR_INVALID_ARGUMENT;
  uint32_t P = 1;
  while (P < s) P <<= 1;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(slab::cuts_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, slab::kMaxSample * 8);
    attr = true;
  }
  DDM_LAUNCH("slab_cuts", 8.0 * s, st, slab::cuts_kernel<<<1, 1024, P * sizeof(double), st>>>(sample, s, world, cuts));
  return check_launch();
}

size_t ddm_slab_pack_workspace_bytes(uint64_t count, uint32_t world) {
  if (world < 1 || world > slab::kMaxWorld) return 0;
  return slab_layout(count, world, nullptr).bytes;
}

ddm_status ddm_slab_pack(const ddm_regions* R, int side, uint64_t id_base, const double* cuts, uint32_t world,
                         const int64_t* reach_in, int64_t* reach_out, uint64_t* send_counts, double* rows,
                         uint64_t rows_cap, uint64_t* total_out, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (!R || R->d == 0 || R->d > DDM_MAX_DIMS || (side != 0 && side != 1) || world < 1 ||
      world > slab::kMaxWorld || !send_counts || !total_out || !aligned(ws, 256))
    return DDM_ERR_INVALID_ARGUMENT;
  const uint64_t count = side == 0 ? R->n_sub : R->n_upd;
  DDM_TRY(side == 0 ? check_side(R->d, count, R->sub_lo, R->sub_hi) : check_side(R->d, count, R->upd_lo, R->upd_hi));
  if (world > 1 && !cuts) return DDM_ERR_INVALID_ARGUMENT;
  if (side == 0 && !reach_in) return DDM_ERR_INVALID_ARGUMENT;
  if (side == 1 && !reach_out) return DDM_ERR_INVALID_ARGUMENT;
  if (id_base + count > (1ull << 32)) return DDM_ERR_INVALID_ARGUMENT;  // global ids are uint32
  if (ws_bytes < ddm_slab_pack_workspace_bytes(count, world)) return DDM_ERR_WORKSPACE;
  init_attrs_once();
  SlabWs W = slab_layout(count, world, ws);
  slab::PackArgs A{};
  A.d = (int)R->d;
  A.count = count;
  for (uint32_t k = 0; k < R->d; ++k) {
    A.lo[k] = side == 0 ? R->sub_lo[k] : R->upd_lo[k];
    A.hi[k] = side == 0 ? R->sub_hi[k] : R->upd_hi[k];
  }
  A.id_base = id_base;
  A.side = side;
  A.cuts = cuts;
  A.reach = reinterpret_cast<const long long*>(reach_in);
  A.world = world;
  A.tiles = W.tiles;
  A.tile_counts = W.cnt;
  A.reach_out = reinterpret_cast<long long*>(reach_out);
  A.err = reinterpret_cast<uint32_t*>(W.misc + world + 1);
  A.rows = rows;
  DDM_CUDA(cudaMemsetAsync(W.misc, 0, sizeof(uint64_t) * (world + 2), st));
  if (side == 1) {  // INT64_MIN = no update in the slab
    std::vector<int64_t> init(world, INT64_MIN);
    DDM_CUDA(cudaMemcpyAsync(reach_out, init.data(), sizeof(int64_t) * world, cudaMemcpyHostToDevice, st));
  }
  const uint64_t T = W.tiles * world;
  if (W.tiles) {
    DDM_LAUNCH("slab_pack", 16.0 * R->d * count, st, slab::count_kernel<<<(unsigned)W.tiles, slab::kThreads, 0, st>>>(A));
    DDM_TRY(check_launch());
    const unsigned stiles = (unsigned)((T + match::kScanThreads * match::kScanItems - 1) /
                                       (match::kScanThreads * match::kScanItems));
    DDM_CUDA(cudaMemsetAsync(W.status, 0, sizeof(uint64_t) * (stiles + 1), st));
    DDM_LAUNCH("scan", 16.0 * T, st, match::scan_u64_kernel<<<stiles, match::kScanThreads, 0, st>>>(
        W.cnt, T, W.off, W.status, W.off + T));
    DDM_TRY(check_launch());
    DDM_LAUNCH("slab_pack", 0, st, slab_seg_starts_kernel<<<1, 64, 0, st>>>(W.off, W.tiles, world, W.misc));
    DDM_TRY(check_launch());
  }
  std::vector<uint64_t> h(world + 2, 0);
  DDM_CUDA(cudaMemcpyAsync(h.data(), W.misc, sizeof(uint64_t) * (world + 2), cudaMemcpyDeviceToHost, st));
  DDM_CUDA(cudaStreamSynchronize(st));
  DDM_TRY(err_status((uint32_t)h[world + 1]));
  const uint64_t total = W.tiles ? h[world] : 0;
  for (uint32_t r = 0; r < world; ++r) send_counts[r] = W.tiles ? h[r + 1] - h[r] : 0;
  *total_out = total;
  if (total > rows_cap) return DDM_ERR_CAPACITY;
  if (total == 0) return DDM_OK;
  if (!rows) return DDM_ERR_INVALID_ARGUMENT;
  A.tile_counts = W.off;  // exclusive offsets
  DDM_LAUNCH("slab_pack", 16.0 * R->d * count + (16.0 * R->d + 8.0) * total, st,
             slab::scatter_kernel<<<(unsigned)W.tiles, slab::kThreads, 0, st>>>(A));
  return check_launch();
}

ddm_status ddm_slab_unpack(const double* rows, uint64_t count, uint32_t d, double* lo, double* hi, uint32_t* ids,
                           cudaStream_t st) {
  if (d == 0 || d > DDM_MAX_DIMS) return DDM_ERR_INVALID_ARGUMENT;
  if (count == 0) return DDM_OK;
  if (!rows || !lo || !hi || !ids) return DDM_ERR_INVALID_ARGUMENT;
  DDM_LAUNCH("slab_unpack", (32.0 * d + 12.0) * count, st,
             slab::unpack_kernel<<<grid_for(count, 256, 8), 256, 0, st>>>(rows, count, (int)d, lo, hi, ids));
  return check_launch();
}

// ------------------------------------------------------------ literal d > 1 (G10)

namespace {
struct LitWs {
  uint8_t* match_ws;
  size_t match_bytes;
  uint64_t* a;     // running intersection (canonical words)
  uint64_t* b;     // this dimension's pairs
  uint64_t* c;     // compaction target
  uint64_t* off;   // [cap + 1] flags -> offsets
  uint64_t* flag;
  uint64_t* status;
  uint8_t* sort_ws;
  size_t sort_bytes;
  size_t bytes;
};
LitWs lit_layout(uint64_t n_sub, uint64_t n_upd, uint64_t cap, void* base) {
  Carver c(base);
  LitWs L{};
  L.match_bytes = ddm_workspace_bytes(1, n_sub, n_upd, 1);
  L.match_ws = c.take<uint8_t>(L.match_bytes);
  L.a = c.take<uint64_t>(cap + 1);
  L.b = c.take<uint64_t>(cap + 1);
  L.c = c.take<uint64_t>(cap + 1);
  L.flag = c.take<uint64_t>(cap + 1);
  L.off = c.take<uint64_t>(cap + 1);
  L.status = c.take<uint64_t>(cap / (match::kScanThreads * match::kScanItems) + 2);
  L.sort_bytes = ddm_sort_pairs_workspace_bytes(cap);
  L.sort_ws = c.take<uint8_t>(L.sort_bytes);
  L.bytes = c.used;
  return L;
}
}  // namespace

size_t ddm_literal_workspace_bytes(uint32_t d, uint64_t n_sub, uint64_t n_upd, uint64_t dim_capacity) {
  if (d == 0 || d > DDM_MAX_DIMS) return 0;
  return lit_layout(n_sub, n_upd, dim_capacity, nullptr).bytes;
}

ddm_status ddm_match_pairs_literal(const ddm_regions* R, ddm_pair* pairs, uint64_t capacity, uint64_t* count_out,
                                   uint64_t dim_capacity, uint64_t* dim_count_out, void* ws, size_t ws_bytes,
                                   cudaStream_t st) {
  DDM_TRY(check_regions(R, true, true));
  if (!count_out || !dim_count_out || !aligned(ws, 256) || (capacity && !pairs)) return DDM_ERR_INVALID_ARGUMENT;
  if (dim_capacity > DDM_MAX_SORT_KEYS) return DDM_ERR_INVALID_ARGUMENT;
  if (ws_bytes < ddm_literal_workspace_bytes(R->d, R->n_sub, R->n_upd, dim_capacity)) return DDM_ERR_WORKSPACE;
  init_attrs_once();
  LitWs L = lit_layout(R->n_sub, R->n_upd, dim_capacity, ws);
  *count_out = 0;
  *dim_count_out = 0;
  uint64_t na = 0;
  for (uint32_t k = 0; k < R->d; ++k) {
    // this dimension alone (a 1-D instance): its pairs, canonical order
    ddm_regions V{};
    V.d = 1;
    V.n_sub = R->n_sub;
    V.n_upd = R->n_upd;
    V.sub_lo[0] = R->sub_lo[k]; V.sub_hi[0] = R->sub_hi[k];
    V.upd_lo[0] = R->upd_lo[k]; V.upd_hi[0] = R->upd_hi[k];
    uint64_t* dst = k == 0 ? L.a : L.b;
    uint64_t kk = 0;
    const ddm_status r = match_full(&V, reinterpret_cast<ddm_pair*>(dst), dim_capacity, &kk, 0, L.match_ws,
                                    L.match_bytes, st);
    if (kk > *dim_count_out) *dim_count_out = kk;
    if (r == DDM_ERR_CAPACITY) return r;  // *dim_count_out = a K_k above dim_capacity
    DDM_TRY(r);
    DDM_TRY(ddm_sort_pairs(reinterpret_cast<ddm_pair*>(dst), kk, R->n_sub, R->n_upd, L.sort_ws, L.sort_bytes, st));
    if (k == 0) {
      na = kk;
      continue;
    }
    // A <- A ∩ B by sort-merge (binary search of each A word in B), compacted in order
    if (na) {
      DDM_LAUNCH("lit_intersect", 8.0 * na + 8.0 * kk, st, match::intersect_flags_kernel<<<grid_for(na, 256, 8), 256, 0, st>>>(
          L.a, na, L.b, kk, L.flag));
      DDM_TRY(check_launch());
      const unsigned stiles = (unsigned)((na + match::kScanThreads * match::kScanItems - 1) /
                                         (match::kScanThreads * match::kScanItems));
      DDM_CUDA(cudaMemsetAsync(L.status, 0, sizeof(uint64_t) * (stiles + 1), st));
      DDM_LAUNCH("scan", 16.0 * na, st, match::scan_u64_kernel<<<stiles, match::kScanThreads, 0, st>>>(
          L.flag, na, L.off, L.status, L.off + na));
      DDM_TRY(check_launch());
      DDM_LAUNCH("lit_intersect", 24.0 * na, st, match::compact_kernel<<<grid_for(na, 256, 8), 256, 0, st>>>(
          L.a, na, L.flag, L.off, L.c));
      DDM_TRY(check_launch());
      DDM_CUDA(cudaMemcpyAsync(&na, L.off + na, sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
      DDM_CUDA(cudaStreamSynchronize(st));
      std::swap(L.a, L.c);
    }
  }
  *count_out = na;
  if (na > capacity) return DDM_ERR_CAPACITY;
  if (na) DDM_CUDA(cudaMemcpyAsync(pairs, L.a, na * sizeof(uint64_t), cudaMemcpyDeviceToDevice, st));
  DDM_CUDA(cudaStreamSynchronize(st));
  return DDM_OK;
}

size_t ddm_sort_pairs_workspace_bytes(uint64_t k) {
  Carver c(nullptr);
  sort_scratch(c, k, true);
  return c.used;
}

ddm_status ddm_sort_pairs(ddm_pair* pairs, uint64_t k, uint64_t n_sub, uint64_t n_upd, void* ws,
                          size_t ws_bytes, cudaStream_t stream) {
  if (k == 0) return DDM_OK;
  if (!pairs || !aligned(pairs, 8) || !aligned(ws, 256)) return DDM_ERR_INVALID_ARGUMENT;
  if (k > DDM_MAX_SORT_KEYS) return DDM_ERR_INVALID_ARGUMENT;  // 30-bit look-back prefixes
  if (ws_bytes < ddm_sort_pairs_workspace_bytes(k)) return DDM_ERR_WORKSPACE;
  Carver c(ws);
  SortScratch s = sort_scratch(c, k, true);
  // canonical key (upd << 32) | sub: only the digits that can be non-zero
  radix::PassList P{};
  const int nb = bits_for(n_sub ? n_sub - 1 : 0), mb = bits_for(n_upd ? n_upd - 1 : 0);
  for (int b = 0; b < nb; b += 8) { P.shift[P.n] = b; P.mask[P.n] = 255; ++P.n; }
  for (int b = 32; b < 32 + mb; b += 8) { P.shift[P.n] = b; P.mask[P.n] = 255; ++P.n; }
  if (P.n == 0) return DDM_OK;
  uint64_t* keys = reinterpret_cast<uint64_t*>(pairs);
  return radix_sort(keys, false, nullptr, keys, nullptr, k, P, s.hist[0], false, s, stream);
}

size_t ddm_radix_sort_workspace_bytes(uint64_t n) {
  Carver c(nullptr);
  sort_scratch(c, n, true);
  return c.used;
}

ddm_status ddm_radix_sort_u64(const uint64_t* keys_in, const uint32_t* vals_in, uint64_t* keys_out,
                              uint32_t* vals_out, uint64_t n, int begin_bit, int end_bit, void* ws,
                              size_t ws_bytes, cudaStream_t stream) {
  if (n == 0) return DDM_OK;
  if (n > DDM_MAX_REGIONS || !keys_in || !keys_out || begin_bit < 0 || end_bit > 64 || begin_bit >= end_bit)
    return DDM_ERR_INVALID_ARGUMENT;
  if ((end_bit - begin_bit + 7) / 8 > radix::kMaxPasses) return DDM_ERR_INVALID_ARGUMENT;
  if (keys_in == keys_out || (vals_in && vals_in == vals_out)) return DDM_ERR_INVALID_ARGUMENT;
  if (!aligned(ws, 256) || ws_bytes < ddm_radix_sort_workspace_bytes(n)) return DDM_ERR_WORKSPACE;
  Carver c(ws);
  SortScratch s = sort_scratch(c, n, true);
  radix::PassList P{};
  for (int b = begin_bit; b < end_bit; b += 8) {
    const int w = end_bit - b < 8 ? end_bit - b : 8;
    P.shift[P.n] = b;
    P.mask[P.n] = (1u << w) - 1;
    ++P.n;
  }
  return radix_sort(keys_in, false, vals_in, keys_out, vals_out, n, P, s.hist[0], false, s, stream);
}

ddm_status ddm_encode_keys(const double* x, uint64_t* keys, uint64_t n, cudaStream_t stream) {
  if (n == 0) return DDM_OK;
  if (!x || !keys) return DDM_ERR_INVALID_ARGUMENT;
  DDM_LAUNCH("encode", 16.0 * n, stream, encode_kernel<<<grid_for(n, 256, 8), 256, 0, stream>>>(x, keys, n));
  return check_launch();
}

const char* ddm_status_string(ddm_status s) {
  switch (s) {
    case DDM_OK: return "DDM_OK";
    case DDM_ERR_INVALID_ARGUMENT: return "DDM_ERR_INVALID_ARGUMENT";
    case DDM_ERR_NONFINITE: return "DDM_ERR_NONFINITE";
    case DDM_ERR_INVERTED_INTERVAL: return "DDM_ERR_INVERTED_INTERVAL";
    case DDM_ERR_CAPACITY: return "DDM_ERR_CAPACITY";
    case DDM_ERR_WORKSPACE: return "DDM_ERR_WORKSPACE";
    case DDM_ERR_CUDA: return "DDM_ERR_CUDA";
  }
  return "DDM_ERR_UNKNOWN";
}

int ddm_last_cuda_error(void) { return g_last_cuda.load(); }

uint64_t ddm_kernel_launch_count(void) { return g_launches.load(); }

void ddm_profile_enable(int on) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  g_prof.on = on != 0;
  g_prof.recs.clear();
  g_prof.next = 0;
}

int ddm_profile_read(ddm_kernel_stat* out, int cap) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  std::vector<ddm_kernel_stat> agg;
  for (const ProfRec& r : g_prof.recs) {
    float ms = 0.f;
    if (cudaEventSynchronize(g_prof.ev[r.e1]) != cudaSuccess) return -1;
    if (cudaEventElapsedTime(&ms, g_prof.ev[r.e0], g_prof.ev[r.e1]) != cudaSuccess) return -1;
    ddm_kernel_stat* hit = nullptr;
    for (auto& a : agg)
      if (strncmp(a.name, r.name, sizeof(a.name)) == 0) hit = &a;
    if (!hit) {
      agg.push_back(ddm_kernel_stat{});
      hit = &agg.back();
      strncpy(hit->name, r.name, sizeof(hit->name) - 1);
    }
    hit->launches += 1;
    hit->total_ms += ms;
    hit->bytes += r.bytes;
  }
  const int k = (int)agg.size() < cap ? (int)agg.size() : cap;
  for (int i = 0; i < k; ++i) out[i] = agg[i];
  return (int)agg.size();
}

const char* ddm_build_info(void) {
  return "libddm sm_100a sort(value-bucketed MSD: 8-bit multisplit passes + smem local sort; LSB onesweep fallback) "
         "count(merge path 2048/tile; rank form | stab walk over slo_hi prefix maxima) scan(decoupled look-back) "
         "emit(tile window | chunk-start sets | per-row) d>1(k* sweep dim; row-indexed tiles: rows binned by dims 1-2, "
         "candidates streamed, float-certain decisions, exact f64 re-test of the rest)";
}

}  // extern "C"
