/*
 * ddm.h -- C ABI of libddm: B200-native sort-based DDM region matching.
 *
 * Operation (§3, P:190-197 and Alg. 1, d-dim P:237-247):
 * given n subscription extents S_i and m update extents U_j, each a
 * d-dimensional axis-parallel box of CLOSED intervals [lo, hi], report every
 * pair (S_i, U_j) with S_i ∩ U_j ≠ ∅, i.e. for every dimension k
 *        sub_lo[k][i] <= upd_hi[k][j]  &&  upd_lo[k][j] <= sub_hi[k][i].
 * The result is computed by the paper's sort-based matching (Alg. 4/5,
 * P:413-557) re-designed for sm_100a: order-preserving u64 endpoint keys, a
 * value-bucketed MSD sort (stable 8-bit multisplit passes over the bucket id,
 * then an in-shared-memory sort of every bucket; a stable LSB onesweep radix
 * sort is the fallback for buckets too large for shared memory and the
 * DDM_SORT_LSB path), a rank-difference count pass, an exclusive scan of the
 * counts, and a chunked sweep that emits every pair exactly once.
 *
 * Conventions shared by every entry point
 *  - Coordinates: IEEE float64, compared exactly (no epsilon).  -0.0 equals
 *    +0.0.  NaN/±inf are rejected (DDM_ERR_NONFINITE).  lo > hi in
 *    any dimension is rejected (DDM_ERR_INVERTED_INTERVAL); lo == hi is
 *    a legal point interval.  Duplicates are distinct regions.
 *  - Ids are the array indices 0..n-1 / 0..m-1.
 *  - Pointers marked (device) must be CUDA device pointers (cudaMalloc /
 *    torch CUDA tensors) on the current device; (host) are host pointers.
 *  - Ownership: the caller owns every buffer (inputs, outputs, workspace,
 *    index).  The library allocates no device memory.  It keeps two internal
 *    side streams and one capture stream per calling thread and device (the
 *    sort chains run concurrently on them, joined back into `stream` by
 *    events) and a process-wide cache of CUDA graphs: from the second
 *    identical full-match call (same sizes, pointers, workspace, flags and
 *    stream) the pre-sync half is replayed as one graph launch (DDM_GRAPHS=0
 *    disables); at most 64 instantiated graphs are kept, least recently used
 *    evicted.  Graphs read the buffers' current contents.  Calls are
 *    reentrant (thread-safe) given distinct workspaces and output buffers.
 *  - Streams: all device work is stream-ordered on `stream`.  Entry points
 *    that return a count block on one small device->host read of it.
 *  - Alignment: workspace and index must be 256-byte aligned; region arrays
 *    8-byte aligned; the pair buffer 8-byte aligned.
 *  - Sizes: 0 <= n_sub, n_upd <= DDM_MAX_REGIONS; counts K are uint64.
 *  - Errors never write past `capacity` pairs; on any error the contents of
 *    the pair buffer are unspecified.
 */
#ifndef DDM_H
#define DDM_H

#include <stddef.h>
#include <stdint.h>
#include <cuda_runtime_api.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DDM_MAX_DIMS 8
/* Per-kind region limit: the sorts' decoupled look-back words hold 30-bit
 * per-digit prefixes (2^30 - 1; SURVEY §8(b) proposed UINT32_MAX -- the
 * narrower limit still holds every BASELINE config, c5 has 5e8 per kind). */
#define DDM_MAX_REGIONS 1073741823ull
/* Largest key count of one radix sort (ddm_sort_pairs' k, the event-order
 * variant's 2(n_sub + n_upd) endpoints, ddm_radix_sort_u64's n): the same
 * 30-bit bound.  Larger requests return DDM_ERR_INVALID_ARGUMENT. */
#define DDM_MAX_SORT_KEYS 1073741823ull

typedef enum {
    DDM_OK = 0,
    DDM_ERR_INVALID_ARGUMENT = 1,  /* null pointer, d == 0 or d > DDM_MAX_DIMS,
                                      n > DDM_MAX_REGIONS, misalignment */
    DDM_ERR_NONFINITE = 2,         /* a NaN or ±inf coordinate */
    DDM_ERR_INVERTED_INTERVAL = 3, /* lo > hi in some dimension */
    DDM_ERR_CAPACITY = 4,          /* capacity < K; *count_out = K, no pair written */
    DDM_ERR_WORKSPACE = 5,         /* ws_bytes (or index_bytes) too small */
    DDM_ERR_CUDA = 6               /* CUDA launch/runtime failure; see ddm_last_cuda_error() */
} ddm_status;

/* Regions of one problem instance, structure-of-arrays per dimension.
 * sub_lo[k] / sub_hi[k] (device) have n_sub float64 entries for k < d;
 * upd_lo[k] / upd_hi[k] (device) have n_upd entries.  Unused slots ignored. */
typedef struct {
    uint32_t d;
    uint64_t n_sub;
    uint64_t n_upd;
    const double *sub_lo[DDM_MAX_DIMS];
    const double *sub_hi[DDM_MAX_DIMS];
    const double *upd_lo[DDM_MAX_DIMS];
    const double *upd_hi[DDM_MAX_DIMS];
} ddm_regions;

/* One reported intersection, paper order (S_i, U_j).  Read as a
 * little-endian uint64 it equals (upd << 32) | sub -- the canonical key. */
typedef struct {
    uint32_t sub;
    uint32_t upd;
} ddm_pair;

/* Flags for ddm_match_pairs / ddm_match_pairs_indexed.  The pair SET never
 * depends on flags, and the output ORDER is deterministic for given inputs,
 * sizes and flags: rows by (upd lower bound, upd id) on the sweep dimension
 * (0 for d = 1; see DDM_SWEEP_DIM0 for d > 1).  Within a row: d = 1,
 * subscriptions by (sub lower bound, sub id) -- every emission path writes
 * byte-identical output; d > 1, the tiled filter writes ascending sub id
 * (a tile whose hits overflow its staging slot: its enumeration order) and the
 * per-row paths (FORCE_THREAD / FORCE_WARP, or few updates) Slo order -- the
 * order inside a d > 1 row is unspecified; canonicalise with ddm_sort_pairs.
 * The emit-path flags only force one of the emission paths (for tests). */
#define DDM_EMIT_AUTO 0u
#define DDM_EMIT_FORCE_THREAD (1u << 8) /* one thread per update row */
#define DDM_EMIT_FORCE_WARP (1u << 9)   /* one warp per update row, global scan */
#define DDM_EMIT_FORCE_CHUNK (1u << 10) /* chunk-start sets staged in smem */
/* Sort selection: by default the value-bucketed MSD sort (payload carried,
 * no gathers) runs and falls back to the LSB radix sort + gathers if some
 * bucket exceeds shared memory; this flag forces the LSB path.  Output is
 * identical either way. */
#define DDM_SORT_LSB (1u << 12)
/* Count form of the pairs calls (the count half of the two-pass emission).
 * Rank form: |Stab(a)| = r_lo - r_hi from a sorted array of the upper bounds
 * (Shi) -- what ddm_match_count always uses, independent of K.  Walk form:
 * |Stab(a)| counted by walking the sorted lower bounds backwards from r_lo,
 * stopped by the prefix maximum of their upper bounds -- O(K) like the
 * emission itself, and no Shi sort.  Default for ddm_match_pairs (d = 1,
 * n_sub >= 2^20): one small probe kernel estimates the mean stab size
 * n_sub * mean(hi - lo) / (max lo - min lo) over 4096 sampled subscriptions
 * (one extra 24-byte device->host read, on the first call with given
 * regions / workspace / flags / stream; repeated calls reuse the decision)
 * and picks the walk form when it is <= 4; otherwise, and for every indexed
 * match, the rank form.  These flags force one form.  Output is identical
 * either way.  The same probe (also run for count calls with a side of at
 * least 2^22 regions) decides per side whether the sort packs its records to
 * 16 bytes (upper key as a 32-bit delta from the lower key): not when more
 * than 15 % of the sampled deltas need more bits -- a performance choice only. */
#define DDM_COUNT_RANKS (1u << 13)
#define DDM_COUNT_WALK (1u << 14)
/* Sweep dimension (d > 1, ddm_match_pairs / ddm_match_count /
 * ddm_match_pairs_mapped): by default the pipeline sweeps the dimension k*
 * with the fewest estimated candidate pairs (k* = argmin_k
 * K_k; P:237-247 leaves the choice open) -- a probe of 4096 sampled regions
 * per kind estimates K_k / (n m) = (mean S length + mean U length) / span of
 * the lower bounds, and k* replaces dimension 0 when its estimate is at least
 * 10 % smaller (one small device->host read per call: the choice follows
 * the data).  The pair set is the same for every sweep dimension; the row order
 * then follows dimension k*.  This flag sweeps dimension 0 always.  The
 * subscription index (ddm_sub_index_build) always sweeps dimension 0. */
#define DDM_SWEEP_DIM0 (1u << 15)
/* d > 1 filter form (cross-checks and tests; the pair SET is the same).
 * Default: the row-indexed tiles (4096 updates per tile, binned once by their
 * dims-1/2 lower bounds; every candidate subscription scans the row cells it
 * can reach) when they fill the GPU, else the chunk-indexed tiles (1024
 * updates; candidates streamed through shared memory and binned per chunk),
 * else one thread / warp per update row when there are fewer tiles than SMs.
 * FORCE_ROWS / FORCE_CHUNKS select a tiled form whatever the sizes. */
#define DDM_DD_FORCE_ROWS (1u << 16)
#define DDM_DD_FORCE_CHUNKS (1u << 17)

/* Workspace bytes needed by ddm_match_count (want_pairs = 0) or
 * ddm_match_pairs (want_pairs != 0) for these sizes.  Independent of K. */
size_t ddm_workspace_bytes(uint32_t d, uint64_t n_sub, uint64_t n_upd, int want_pairs);

/* K = number of intersecting pairs (SPEC S:41-46 count mode, the paper's
 * experimental mode P:915-918).  count_out (host) receives K. */
ddm_status ddm_match_count(const ddm_regions *regions, uint64_t *count_out, void *ws,
                           size_t ws_bytes, cudaStream_t stream);

/* List mode: writes the K pairs to pairs[0..K) (device) and K to *count_out
 * (host).  If capacity < K returns DDM_ERR_CAPACITY with *count_out = K and
 * writes no pair (call with capacity 0 to size the buffer).  Validation
 * errors are reported before any pair is written. */
ddm_status ddm_match_pairs(const ddm_regions *regions, ddm_pair *pairs, uint64_t capacity,
                           uint64_t *count_out, uint32_t flags, void *ws, size_t ws_bytes,
                           cudaStream_t stream);

/* ddm_match_pairs with id maps: the pair written for local subscription s and
 * local update u is {sub_ids[s], upd_ids[u]} (device arrays of n_sub / n_upd
 * uint32; either may be NULL = the local index).  Used by the slab-partitioned
 * multi-GPU mode, where every rank matches its own slab of updates against the
 * subscriptions that can reach it and reports global ids.  Same workspace,
 * errors and output order as ddm_match_pairs. */
ddm_status ddm_match_pairs_mapped(const ddm_regions *regions, const uint32_t *sub_ids, const uint32_t *upd_ids,
                                  ddm_pair *pairs, uint64_t capacity, uint64_t *count_out, uint32_t flags,
                                  void *ws, size_t ws_bytes, cudaStream_t stream);

/* Sort pairs[0..k) (device) in place into canonical order: ascending
 * (upd << 32) | sub.  ids must satisfy sub < n_sub and upd < n_upd;
 * k <= DDM_MAX_SORT_KEYS (else DDM_ERR_INVALID_ARGUMENT).  This replaces the
 * DDM_SORTED flag SURVEY §8(b) proposed: the result is a set and
 * ddm_match_pairs' own order is already deterministic, so canonical order is
 * a separate call whose workspace is sized by the K the caller knows. */
size_t ddm_sort_pairs_workspace_bytes(uint64_t k);
ddm_status ddm_sort_pairs(ddm_pair *pairs, uint64_t k, uint64_t n_sub, uint64_t n_upd,
                          void *ws, size_t ws_bytes, cudaStream_t stream);

/* --- Subscription index: the subscription half of the pipeline, built once
 * (sorted dim-0 lower/upper keys, ids, gathered upper keys, block maxima and
 * the other dimensions in sweep order) and byte-copyable, so one rank can
 * build it and broadcast it to the others (multi-GPU split). */
size_t ddm_sub_index_bytes(uint32_t d, uint64_t n_sub);
size_t ddm_index_build_workspace_bytes(uint32_t d, uint64_t n_sub);
ddm_status ddm_sub_index_build(const ddm_regions *subs /* n_upd ignored */, void *index,
                               size_t index_bytes, void *ws, size_t ws_bytes,
                               cudaStream_t stream);

/* Dynamic DDM (moving / resizing extents):
 * subscriptions ids[0..k) of a built index (n_sub regions) take the new
 * coordinates moved->sub_lo/sub_hi[dim][0..k) (moved->d = the index's d,
 * moved->n_sub = k; device arrays).  ids: device, strictly increasing, < n_sub.
 * The updated index is written to index_out by a merge (tombstone the old
 * entries, sort the k new ones, scatter every entry once to its final
 * position, recompute the block / prefix maxima and d > 1 boxes): O(n + k log
 * k) work instead of a rebuild's sort, and the result is byte-identical to
 * ddm_sub_index_build on the modified region set.  index_out == index_in
 * updates in place through a copy in the workspace (in_place = 1 sizes it);
 * distinct buffers (ping-pong) avoid the copy.  Errors (bad ids, non-finite
 * or inverted new coordinates) are reported before anything is written.
 * Stream-ordered; blocks on one small device->host read.  ws: 256-byte
 * aligned, >= ddm_sub_index_update_workspace_bytes(d, n_sub, k, in_place). */
size_t ddm_sub_index_update_workspace_bytes(uint32_t d, uint64_t n_sub, uint64_t k, int in_place);
ddm_status ddm_sub_index_update(const void *index_in, void *index_out, size_t index_bytes, uint64_t n_sub,
                                const ddm_regions *moved, const uint32_t *ids, void *ws, size_t ws_bytes,
                                cudaStream_t stream);

/* Match updates against a built index.  upds->n_sub must equal the indexed
 * n_sub and upds->d its d.  upd_ids (device, may be NULL): global id of each
 * local update, written into ddm_pair.upd (NULL = local index).  Workspace
 * from ddm_indexed_workspace_bytes. */
size_t ddm_indexed_workspace_bytes(uint32_t d, uint64_t n_sub, uint64_t n_upd);
ddm_status ddm_match_pairs_indexed(const void *index, const ddm_regions *upds,
                                   const uint32_t *upd_ids, ddm_pair *pairs, uint64_t capacity,
                                   uint64_t *count_out, uint32_t flags, void *ws,
                                   size_t ws_bytes, cudaStream_t stream);
ddm_status ddm_match_count_indexed(const void *index, const ddm_regions *upds,
                                   uint64_t *count_out, void *ws, size_t ws_bytes,
                                   cudaStream_t stream);

/* --- Literal d-dimensional reading (SURVEY §8(a) a8 "literal",
 * G10): the pair set of every dimension separately (the 1-D pipeline on
 * dimension k), each sorted into canonical u64 words (upd << 32) | sub, then
 * intersected by sort-merge (binary search of the running result's words in
 * the next dimension's sorted list, survivors compacted in order).  The same
 * set as ddm_match_pairs, written in canonical order -- an independent
 * cross-check of the filtered sweep, for SMALL inputs: every per-dimension
 * set is materialised (up to dim_capacity pairs each; a larger one returns
 * DDM_ERR_CAPACITY with *dim_count_out = its size).  *count_out (host) = K;
 * capacity < K -> DDM_ERR_CAPACITY.  ws >= ddm_literal_workspace_bytes(d,
 * n_sub, n_upd, dim_capacity), 256-byte aligned; dim_capacity <=
 * DDM_MAX_SORT_KEYS.  Blocks on small device->host reads. */
size_t ddm_literal_workspace_bytes(uint32_t d, uint64_t n_sub, uint64_t n_upd, uint64_t dim_capacity);
ddm_status ddm_match_pairs_literal(const ddm_regions *regions, ddm_pair *pairs, uint64_t capacity,
                                   uint64_t *count_out, uint64_t dim_capacity, uint64_t *dim_count_out,
                                   void *ws, size_t ws_bytes, cudaStream_t stream);

/* --- Multi-GPU slab partition: the
 * device half of the slab mode's data redistribution.  Every rank holds a
 * block of the regions (global ids id_base + i) and sends each region to the
 * ranks of the dimension-0 slabs it can take part in: an update to the slab
 * holding its lower bound; a subscription S to every slab r with
 * S.hi >= c_r and S.lo <= reach_r (max upper bound of slab r's updates) --
 * the slab plus its halo, the stabbing set at the slab start (Alg. 6's
 * SubSet[p] at a segment boundary).  Then every intersecting pair
 * has both members on its update's rank.  The caller moves the packed rows
 * with all_to_all (torch.distributed / NCCL) and matches with
 * ddm_match_pairs_mapped.  All pointers device unless marked (host).
 *
 * ddm_slab_sample: sample[i] = lo0[floor(i * count / s)], i < s (NaN when
 *   count == 0).  ddm_slab_cuts: cut points c_1..c_{world-1} (cuts, world-1
 *   doubles) = quantiles floor(r * v / world) of the v finite entries of the
 *   gathered sample (s <= 16384, world <= 32); slab r = [c_r, c_{r+1}).
 * ddm_slab_pack: side 0 = subscriptions (regions->sub_*, n_sub), 1 = updates.
 *   Validates every region (finite, lo <= hi in every dimension: errors as
 *   ddm_match_pairs, nothing written).  Updates: reach_out (world int64)
 *   receives the local per-slab maxima of the upper bounds as order-preserving
 *   signed keys (INT64_MIN = none) -- all_reduce(MAX) it and pass it as the
 *   subscriptions' reach_in.  send_counts (host, world) = rows per
 *   destination; *total_out (host) = their sum; rows ([total][2d+1] words:
 *   lo[0..d), hi[0..d), global id as a uint64 bit pattern) grouped by
 *   destination, index order within each; rows_cap < total ->
 *   DDM_ERR_CAPACITY (counts returned, rows not written).  id_base + count
 *   <= 2^32.  One small device->host read.
 * ddm_slab_unpack: rows [count][2d+1] -> lo[k][count], hi[k][count] (k < d,
 *   contiguous [d][count]) and ids (uint32). */
ddm_status ddm_slab_sample(const double *lo0, uint64_t count, double *sample, uint32_t s, cudaStream_t stream);
ddm_status ddm_slab_cuts(const double *sample, uint32_t s, uint32_t world, double *cuts, cudaStream_t stream);
size_t ddm_slab_pack_workspace_bytes(uint64_t count, uint32_t world);
ddm_status ddm_slab_pack(const ddm_regions *regions, int side, uint64_t id_base, const double *cuts,
                         uint32_t world, const int64_t *reach_in, int64_t *reach_out, uint64_t *send_counts,
                         double *rows, uint64_t rows_cap, uint64_t *total_out, void *ws, size_t ws_bytes,
                         cudaStream_t stream);
ddm_status ddm_slab_unpack(const double *rows, uint64_t count, uint32_t d, double *lo, double *hi,
                           uint32_t *ids, cudaStream_t stream);

/* --- Event-order variant: the paper's own parallel
 * algorithm, Alg. 5 + 6, on the GPU -- an independent
 * cross-check of ddm_match_pairs, not the fast path.  All 2(n_sub+n_upd)
 * endpoints of dimension 0 are sorted into one list T by (coord, is_upper,
 * kind, id) (R1), T is cut into segments of 2048 endpoints (one CTA each);
 * each segment's initial SubSet / UpdSet (Alg. 6) has its size from an
 * exclusive scan of per-segment upper-endpoint counts (Alg. 6's combine in
 * counting form) and its members from a backward walk over T; then every
 * upper endpoint in the segment reports its pairs with the other kind's
 * active set (Alg. 5 l.14-16, l.22-24) -- each pair once, at its earlier
 * upper endpoint.  d > 1: candidates filtered exactly on dims 1..d-1.
 * Output order: unspecified (atomic appends; canonicalise with
 * ddm_sort_pairs).  Two passes (count, then emit); *count_out = K; capacity
 * and validation errors as ddm_match_pairs (nothing written on either).
 * Regions: device float64 SoA as ddm_match_pairs; ws: 256-byte aligned,
 * >= ddm_events_workspace_bytes(d, n_sub, n_upd) (~ 60 B per region). */
size_t ddm_events_workspace_bytes(uint32_t d, uint64_t n_sub, uint64_t n_upd);
ddm_status ddm_match_pairs_events(const ddm_regions *regions, ddm_pair *pairs, uint64_t capacity,
                                  uint64_t *count_out, void *ws, size_t ws_bytes, cudaStream_t stream);

/* --- a6 exported for tests: the chunk-start sets.  ddm_match_pairs' dense
 * emission processes the sorted updates in tiles of DDM_CHUNK_ROWS rows; tile
 * t starts at the update x_t with the (lower key, id)-rank t*DDM_CHUNK_ROWS,
 * and its chunk-start set is A_t = Stab(x_t.lo) = {S : S.lo <= x_t.lo <=
 * S.hi} on dimension 0 -- Alg. 6's SubSet[p] for a segment boundary placed
 * right before x_t's lower endpoint.
 * This runs the a1-a5 pipeline and then the same backward walk with
 * block-max skips that emit_chunk_kernel stages into shared memory, writing:
 * first_upd[t] (device, tiles = ceil(n_upd / DDM_CHUNK_ROWS)) = x_t's id;
 * set_off[0..tiles] (device, uint64) = offsets; set_ids[set_off[t] ..
 * set_off[t+1]) (device) = A_t's subscription ids in (lower key, id) order.
 * *total_out (host) = sum |A_t|; capacity < total -> DDM_ERR_CAPACITY (ids
 * not written; first_upd and set_off are).  d must be 1.  n_sub == 0: every
 * set is empty (set_off zeroed, first_upd not written).  Workspace as
 * ddm_match_pairs.  Validation errors as ddm_match_pairs. */
#define DDM_CHUNK_ROWS 256
ddm_status ddm_chunk_start_sets(const ddm_regions *regions, uint32_t *first_upd, uint64_t *set_off,
                                uint32_t *set_ids, uint64_t capacity, uint64_t *total_out, void *ws,
                                size_t ws_bytes, cudaStream_t stream);

/* --- Primitive exported for tests: stable LSB onesweep radix sort of u64
 * keys (device) with optional u32 values, over bits [begin_bit, end_bit).
 * keys_out/vals_out (device) receive the result; inputs are not modified. */
size_t ddm_radix_sort_workspace_bytes(uint64_t n);
ddm_status ddm_radix_sort_u64(const uint64_t *keys_in, const uint32_t *vals_in,
                              uint64_t *keys_out, uint32_t *vals_out, uint64_t n,
                              int begin_bit, int end_bit, void *ws, size_t ws_bytes,
                              cudaStream_t stream);

/* Order-preserving float64 -> u64 key used by the sort:
 * canonicalise -0.0 to +0.0, then flip the sign bit of non-negatives and all
 * bits of negatives.  Device arrays of length n. */
ddm_status ddm_encode_keys(const double *x, uint64_t *keys, uint64_t n, cudaStream_t stream);

/* Per-kernel-class timing with CUDA events recorded on the launching stream
 * around every library launch while enabled (enable(1) also resets).  While
 * enabled, the sort chains that normally run concurrently on internal side
 * streams all run on the caller's stream, so the recorded intervals of
 * different kernels never overlap.
 * ddm_profile_read synchronises the recorded events and fills up to cap
 * entries; returns the number of kernel classes (or -1 on a CUDA error).
 * bytes = the algorithmic DRAM bytes of those launches. */
typedef struct {
    char name[32];
    uint64_t launches;
    double total_ms;
    double bytes;
} ddm_kernel_stat;
void ddm_profile_enable(int on);
int ddm_profile_read(ddm_kernel_stat *out, int cap);

const char *ddm_status_string(ddm_status s);
int ddm_last_cuda_error(void);          /* last cudaError_t seen by the library */
uint64_t ddm_kernel_launch_count(void); /* kernels launched by this process so far */
const char *ddm_build_info(void);

#ifdef __cplusplus
}
#endif
#endif /* DDM_H */
