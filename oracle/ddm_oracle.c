/*
 * oracle/ddm_oracle.c -- CPU ORACLE for DDM region matching (arXiv 1703.06680).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_1703_06680_b200/, libddm.so) never calls it and
 * shares no code, header, table or helper with it.
 *
 * Plain, slow, obviously-correct C.  Coordinates are compared as IEEE doubles
 * (no key encoding), exactly as Alg. 1 states the predicate.  Every function
 * cites the passage of /root/reference/PAPER.md (P:line) it follows.
 *
 *   orc_bf_*        Alg. 2  BruteForce-1D with the d-dim
 *                   conjunction of P:237-240.            [pinned: see tests]
 *   orc_sbm_seq     Alg. 4  Sort-Based-Matching-1D; d>1 filters
 *                   every emitted candidate on dims 1..d-1 (P:237-247,
 *                   SPEC S:181-189).                       [pinned]
 *   orc_sbm_dd_literal  per-dimension pair sets + sort-merge intersection
 *                   (the BASELINE c4 reading).  [pinned]
 *   orc_par_sbm     Alg. 5 + Alg. 6 Parallel-SBM-1D with OpenMP,
 *                   master combine with p-1 indices (Alg. 6 l.25-28, P:658-662;
 *                   DESIGN.md reading R8).                  [pinned]
 *   orc_sbm_boundary_states / orc_par_sbm_states
 *                   SubSet[p]/UpdSet[p] from the sequential sweep
 *                   and from Alg. 6 -- the boundary-state oracle.
 *   orc_sbm_states_at  the same sequential snapshots taken right before
 *                   chosen update lower endpoints (GPU chunk-start sets).  [pinned]
 *
 * Endpoint order (reading R1): T is sorted by
 * (coordinate, lower-before-upper, subscription-before-update, id).  The paper
 * never states the tie rule; closed intervals (Alg. 1 uses <=) require lower
 * endpoints to be swept before upper endpoints at equal coordinates.
 *
 * Pair encoding: canonical u64 (upd << 32) | sub; a result list is the set of
 * such words sorted ascending (orc_canonicalize).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_OK 0
#define ORC_ERR_ALLOC (-1)
#define ORC_ERR_SETS_NOT_EMPTY (-2)
#define ORC_ERR_ARG (-3)

/* ---------------------------------------------------------------- predicate */

/* Alg. 1 Intersect-1D: x.low <= y.high AND y.low <= x.high. */
int orc_intersect_1d(double xlo, double xhi, double ylo, double yhi) {
    return xlo <= yhi && ylo <= xhi;
}

/* d-rectangles overlap iff all d projections overlap.
 * Arrays are SoA blocks [d][count]; element (k, i) is at k*count + i. */
static int overlap_dims(int k0, int d, const double *sl, const double *sh, int64_t n, int64_t i,
                        const double *ul, const double *uh, int64_t m, int64_t j) {
    for (int k = k0; k < d; ++k)
        if (!orc_intersect_1d(sl[k * n + i], sh[k * n + i], ul[k * m + j], uh[k * m + j])) return 0;
    return 1;
}

static uint64_t pair_word(int64_t sub, int64_t upd) {
    return ((uint64_t)upd << 32) | (uint64_t)(uint32_t)sub;
}

static int cmp_u64(const void *a, const void *b) {
    uint64_t x = *(const uint64_t *)a, y = *(const uint64_t *)b;
    return (x > y) - (x < y);
}

/* Sort a pair list into canonical order (the result is a set). */
void orc_canonicalize(uint64_t *pairs, int64_t k) {
    if (k > 1) qsort(pairs, (size_t)k, sizeof(uint64_t), cmp_u64);
}

/* ------------------------------------------------------------- brute force */

/* Alg. 2, loop over j outermost so each update's row is formed
 * independently (the loop iterations are independent).
 * Rows are written in update order, subscriptions ascending => the output is
 * already in canonical order.  Returns K; pairs written only when K <= cap. */
int64_t orc_bf_pairs(int d, int64_t n, int64_t m, const double *sl, const double *sh,
                     const double *ul, const double *uh, uint64_t *out, int64_t cap) {
    int64_t *cnt = (int64_t *)calloc((size_t)(m + 1), sizeof(int64_t));
    if (!cnt) return ORC_ERR_ALLOC;
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t j = 0; j < m; ++j) {
        int64_t c = 0;
        for (int64_t i = 0; i < n; ++i) c += overlap_dims(0, d, sl, sh, n, i, ul, uh, m, j);
        cnt[j + 1] = c;
    }
    for (int64_t j = 0; j < m; ++j) cnt[j + 1] += cnt[j];
    int64_t K = cnt[m];
    if (out && K <= cap) {
#pragma omp parallel for schedule(dynamic, 64)
        for (int64_t j = 0; j < m; ++j) {
            int64_t w = cnt[j];
            for (int64_t i = 0; i < n; ++i)
                if (overlap_dims(0, d, sl, sh, n, i, ul, uh, m, j)) out[w++] = pair_word(i, j);
        }
    }
    free(cnt);
    return K;
}

/* Alg. 2 restricted to the update ids in rows[0..nrows) (sampled-row parity
 * at sizes where the full n*m loop is too slow).  Output: rows in the given
 * order, subscriptions ascending.  Returns total pairs. */
int64_t orc_bf_rows(int d, int64_t n, int64_t m, const double *sl, const double *sh,
                    const double *ul, const double *uh, const int64_t *rows, int64_t nrows,
                    uint64_t *out, int64_t cap, int64_t *row_counts) {
    int64_t *cnt = (int64_t *)calloc((size_t)(nrows + 1), sizeof(int64_t));
    if (!cnt) return ORC_ERR_ALLOC;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t r = 0; r < nrows; ++r) {
        int64_t j = rows[r], c = 0;
        for (int64_t i = 0; i < n; ++i) c += overlap_dims(0, d, sl, sh, n, i, ul, uh, m, j);
        cnt[r + 1] = c;
    }
    if (row_counts)
        for (int64_t r = 0; r < nrows; ++r) row_counts[r] = cnt[r + 1];
    for (int64_t r = 0; r < nrows; ++r) cnt[r + 1] += cnt[r];
    int64_t K = cnt[nrows];
    if (out && K <= cap) {
#pragma omp parallel for schedule(dynamic, 1)
        for (int64_t r = 0; r < nrows; ++r) {
            int64_t j = rows[r], w = cnt[r];
            for (int64_t i = 0; i < n; ++i)
                if (overlap_dims(0, d, sl, sh, n, i, ul, uh, m, j)) out[w++] = pair_word(i, j);
        }
    }
    free(cnt);
    return K;
}

/* -------------------------------------------------------- endpoint list T */

/* One element of T (Alg. 4 l.1-4): coordinate, lower/upper flag,
 * owner kind (0 = subscription S, 1 = update U) and owner id. */
typedef struct {
    double x;
    uint32_t id;
    uint8_t is_upper;
    uint8_t kind;
} endpoint;

/* Strict total order (coord, is_upper, kind, id) -- DESIGN.md reading R1/R2. */
static int cmp_endpoint(const void *a, const void *b) {
    const endpoint *p = (const endpoint *)a, *q = (const endpoint *)b;
    if (p->x < q->x) return -1;
    if (p->x > q->x) return 1;
    if (p->is_upper != q->is_upper) return (int)p->is_upper - (int)q->is_upper;
    if (p->kind != q->kind) return (int)p->kind - (int)q->kind;
    return (p->id > q->id) - (p->id < q->id);
}

/* Alg. 4 l.2-4: insert x.lower and x.upper of every extent into T (dim k). */
static endpoint *build_T(int k, int64_t n, int64_t m, const double *sl, const double *sh,
                         const double *ul, const double *uh) {
    int64_t N2 = 2 * (n + m);
    endpoint *T = (endpoint *)malloc((size_t)(N2 > 0 ? N2 : 1) * sizeof(endpoint));
    if (!T) return NULL;
#pragma omp parallel for
    for (int64_t i = 0; i < n; ++i) {
        T[2 * i] = (endpoint){sl[k * n + i], (uint32_t)i, 0, 0};
        T[2 * i + 1] = (endpoint){sh[k * n + i], (uint32_t)i, 1, 0};
    }
#pragma omp parallel for
    for (int64_t j = 0; j < m; ++j) {
        T[2 * n + 2 * j] = (endpoint){ul[k * m + j], (uint32_t)j, 0, 1};
        T[2 * n + 2 * j + 1] = (endpoint){uh[k * m + j], (uint32_t)j, 1, 1};
    }
    return T;
}

/* ------------------------------------------------------------------ id set */

/* A set over dense ids 0..cap-1 with O(1) insert / erase / membership and
 * iteration over the members (the paper tried bit vectors and std::set,
 * P:819-834; any representation with these operations is valid). */
typedef struct {
    uint32_t *members;
    int64_t *pos; /* pos[id] = index in members, or -1 */
    int64_t size;
} idset;

static int idset_init(idset *s, int64_t cap) {
    s->members = (uint32_t *)malloc((size_t)(cap > 0 ? cap : 1) * sizeof(uint32_t));
    s->pos = (int64_t *)malloc((size_t)(cap > 0 ? cap : 1) * sizeof(int64_t));
    s->size = 0;
    if (!s->members || !s->pos) return ORC_ERR_ALLOC;
    for (int64_t i = 0; i < cap; ++i) s->pos[i] = -1;
    return ORC_OK;
}
static void idset_free(idset *s) {
    free(s->members);
    free(s->pos);
}
static int idset_has(const idset *s, uint32_t id) { return s->pos[id] >= 0; }
static void idset_insert(idset *s, uint32_t id) {
    if (s->pos[id] >= 0) return;
    s->pos[id] = s->size;
    s->members[s->size++] = id;
}
static void idset_erase(idset *s, uint32_t id) {
    int64_t p = s->pos[id];
    if (p < 0) return;
    uint32_t last = s->members[--s->size];
    s->members[p] = last;
    s->pos[last] = p;
    s->pos[id] = -1;
}

/* Growable pair buffer. */
typedef struct {
    uint64_t *v;
    int64_t size, cap;
    int64_t count; /* total emitted, including those not stored */
    int store;
} pairbuf;

static void pb_push(pairbuf *b, uint64_t w) {
    b->count++;
    if (!b->store) return;
    if (b->size == b->cap) {
        int64_t nc = b->cap ? 2 * b->cap : 1024;
        uint64_t *nv = (uint64_t *)realloc(b->v, (size_t)nc * sizeof(uint64_t));
        if (!nv) { b->store = 0; return; }
        b->v = nv;
        b->cap = nc;
    }
    b->v[b->size++] = w;
}

/* ---------------------------------------------------- sequential SBM (O2) */

/* Process one endpoint t as in Alg. 4 lines 6-21, emitting into
 * `pb` (or adding cardinalities in count mode, SPEC S:174 -- d == 1 only). */
static void sbm_step(const endpoint *t, idset *SubSet, idset *UpdSet, pairbuf *pb, int count_only,
                     int d, const double *sl, const double *sh, int64_t n, const double *ul,
                     const double *uh, int64_t m) {
    if (t->kind == 0) {                 /* t belongs to subscription extent S_i */
        if (!t->is_upper) {
            idset_insert(SubSet, t->id);  /* SubSet <- SubSet U {S_i} */
        } else {
            idset_erase(SubSet, t->id);   /* SubSet <- SubSet \ {S_i} */
            if (count_only && d == 1) { pb->count += UpdSet->size; return; }
            for (int64_t q = 0; q < UpdSet->size; ++q) { /* forall x in UpdSet: L <- L U {(S_i, x)} */
                uint32_t x = UpdSet->members[q];
                if (d == 1 || overlap_dims(1, d, sl, sh, n, t->id, ul, uh, m, x)) {
                    if (count_only) pb->count++; else pb_push(pb, pair_word(t->id, x));
                }
            }
        }
    } else {                            /* t belongs to update extent U_j */
        if (!t->is_upper) {
            idset_insert(UpdSet, t->id);
        } else {
            idset_erase(UpdSet, t->id);
            if (count_only && d == 1) { pb->count += SubSet->size; return; }
            for (int64_t q = 0; q < SubSet->size; ++q) { /* forall x in SubSet: L <- L U {(x, U_j)} */
                uint32_t x = SubSet->members[q];
                if (d == 1 || overlap_dims(1, d, sl, sh, n, x, ul, uh, m, t->id)) {
                    if (count_only) pb->count++; else pb_push(pb, pair_word(x, t->id));
                }
            }
        }
    }
}

/* Alg. 4 Sort-Based-Matching-1D on dimension 0; for d > 1 each
 * emitted candidate is kept iff the 1-D test holds on dims 1..d-1.
 * Returns K (or a negative ORC_ERR_*).  Pairs (emission order, NOT
 * canonical) are copied to out[0..K) when K <= cap. */
int64_t orc_sbm_seq(int d, int64_t n, int64_t m, const double *sl, const double *sh,
                    const double *ul, const double *uh, int count_only, uint64_t *out,
                    int64_t cap) {
    int64_t N2 = 2 * (n + m);
    endpoint *T = build_T(0, n, m, sl, sh, ul, uh);   /* l.1-4 */
    if (!T) return ORC_ERR_ALLOC;
    qsort(T, (size_t)N2, sizeof(endpoint), cmp_endpoint); /* l.5: sort T non-decreasing */
    idset SubSet, UpdSet;                                 /* l.6 */
    if (idset_init(&SubSet, n) || idset_init(&UpdSet, m)) { free(T); return ORC_ERR_ALLOC; }
    pairbuf pb = {0};
    pb.store = !count_only && out != NULL;
    for (int64_t q = 0; q < N2; ++q)                      /* l.7-22 */
        sbm_step(&T[q], &SubSet, &UpdSet, &pb, count_only, d, sl, sh, n, ul, uh, m);
    int64_t K = pb.count;
    int empty = SubSet.size == 0 && UpdSet.size == 0;     /* S:194 invariant */
    if (pb.store && K <= cap && pb.size == K) memcpy(out, pb.v, (size_t)K * sizeof(uint64_t));
    free(pb.v);
    idset_free(&SubSet);
    idset_free(&UpdSet);
    free(T);
    return empty ? K : ORC_ERR_SETS_NOT_EMPTY;
}

/* Literal d-dimensional reading: run Alg. 4 on every dimension
 * separately, canonicalise each per-dimension pair set and intersect them by
 * sort-merge.  Only for small inputs (per-dimension sets can be huge). */
int64_t orc_sbm_dd_literal(int d, int64_t n, int64_t m, const double *sl, const double *sh,
                           const double *ul, const double *uh, uint64_t *out, int64_t cap) {
    uint64_t *acc = NULL;
    int64_t acc_n = 0;
    for (int k = 0; k < d; ++k) {
        /* 1-D instance of dimension k */
        int64_t K = orc_sbm_seq(1, n, m, sl + k * n, sh + k * n, ul + k * m, uh + k * m, 1, NULL, 0);
        if (K < 0) { free(acc); return K; }
        uint64_t *cur = (uint64_t *)malloc((size_t)(K > 0 ? K : 1) * sizeof(uint64_t));
        if (!cur) { free(acc); return ORC_ERR_ALLOC; }
        int64_t K2 = orc_sbm_seq(1, n, m, sl + k * n, sh + k * n, ul + k * m, uh + k * m, 0, cur, K);
        if (K2 != K) { free(cur); free(acc); return ORC_ERR_ARG; }
        orc_canonicalize(cur, K);
        if (k == 0) { acc = cur; acc_n = K; continue; }
        int64_t a = 0, b = 0, w = 0; /* sort-merge intersection, in place into acc */
        while (a < acc_n && b < K) {
            if (acc[a] < cur[b]) a++;
            else if (acc[a] > cur[b]) b++;
            else { acc[w++] = acc[a]; a++; b++; }
        }
        acc_n = w;
        free(cur);
    }
    if (out && acc_n <= cap) memcpy(out, acc, (size_t)acc_n * sizeof(uint64_t));
    free(acc);
    return acc_n;
}

/* ------------------------------------------- segments and boundary states */

/* SPEC S:240-247 plan: the first (len mod P) segments hold ceil(len/P)
 * records, the rest floor(len/P).  bounds has P+1 entries. */
static void plan_segments(int64_t len, int P, int64_t *bounds) {
    int64_t base = len / P, rem = len % P;
    bounds[0] = 0;
    for (int p = 0; p < P; ++p) bounds[p + 1] = bounds[p] + base + (p < rem ? 1 : 0);
}

/* Sequential-sweep snapshots: SubSet and UpdSet right after the last endpoint
 * of T_{p-1} for p = 0..P-1, ids sorted ascending.
 * Outputs are flat arrays with offsets (sub_off/upd_off have P+1 entries);
 * returns the total number of ids written, or a negative error if the
 * capacities are too small. */
static int64_t states_flatten(idset *S, uint32_t *ids, int64_t *w, int64_t cap) {
    if (*w + S->size > cap) return ORC_ERR_ARG;
    for (int64_t q = 0; q < S->size; ++q) ids[*w + q] = S->members[q];
    /* ascending ids for comparison */
    for (int64_t a = 1; a < S->size; ++a) {
        uint32_t v = ids[*w + a];
        int64_t b = a - 1;
        while (b >= 0 && ids[*w + b] > v) { ids[*w + b + 1] = ids[*w + b]; --b; }
        ids[*w + b + 1] = v;
    }
    *w += S->size;
    return ORC_OK;
}

int64_t orc_sbm_boundary_states(int64_t n, int64_t m, const double *sl, const double *sh,
                                const double *ul, const double *uh, int P, uint32_t *sub_ids,
                                int64_t *sub_off, int64_t sub_cap, uint32_t *upd_ids,
                                int64_t *upd_off, int64_t upd_cap) {
    if (P < 1) return ORC_ERR_ARG;
    int64_t N2 = 2 * (n + m);
    endpoint *T = build_T(0, n, m, sl, sh, ul, uh);
    if (!T) return ORC_ERR_ALLOC;
    qsort(T, (size_t)N2, sizeof(endpoint), cmp_endpoint);
    int64_t *bounds = (int64_t *)malloc(sizeof(int64_t) * (size_t)(P + 1));
    idset SubSet, UpdSet;
    if (!bounds || idset_init(&SubSet, n) || idset_init(&UpdSet, m)) { free(T); free(bounds); return ORC_ERR_ALLOC; }
    plan_segments(N2, P, bounds);
    pairbuf pb = {0};
    int64_t ws = 0, wu = 0, q = 0, rc = ORC_OK;
    for (int p = 0; p < P && rc == ORC_OK; ++p) {
        for (; q < bounds[p]; ++q)
            sbm_step(&T[q], &SubSet, &UpdSet, &pb, 1, 1, sl, sh, n, ul, uh, m);
        sub_off[p] = ws;
        upd_off[p] = wu;
        rc = states_flatten(&SubSet, sub_ids, &ws, sub_cap);
        if (rc == ORC_OK) rc = states_flatten(&UpdSet, upd_ids, &wu, upd_cap);
    }
    sub_off[P] = ws;
    upd_off[P] = wu;
    idset_free(&SubSet);
    idset_free(&UpdSet);
    free(bounds);
    free(T);
    return rc == ORC_OK ? ws + wu : rc;
}

/* Sequential-sweep snapshots at chosen update lower endpoints: SubSet right
 * before the lower endpoint of update q[r] is processed (the same snapshot as
 * P:552-557, taken at a segment boundary placed just before that endpoint),
 * for r = 0..nq-1, ids sorted ascending.  This is the chunk-start set of a
 * GPU tile whose first update is q[r].
 * sub_off has nq+1 entries; returns the number of ids (sub_ids == NULL: only
 * sizes them and fills sub_off), or a negative error (capacity, duplicate /
 * out-of-range query ids). */
int64_t orc_sbm_states_at(int64_t n, int64_t m, const double *sl, const double *sh,
                          const double *ul, const double *uh, const int64_t *q, int64_t nq,
                          uint32_t *sub_ids, int64_t *sub_off, int64_t sub_cap) {
    int64_t N2 = 2 * (n + m);
    int64_t *slot = (int64_t *)malloc(sizeof(int64_t) * (size_t)(m > 0 ? m : 1));
    int64_t *cnt = (int64_t *)calloc((size_t)(nq + 1), sizeof(int64_t));
    if (!slot || !cnt) { free(slot); free(cnt); return ORC_ERR_ALLOC; }
    for (int64_t j = 0; j < m; ++j) slot[j] = -1;
    for (int64_t r = 0; r < nq; ++r) {
        if (q[r] < 0 || q[r] >= m || slot[q[r]] >= 0) { free(slot); free(cnt); return ORC_ERR_ARG; }
        slot[q[r]] = r;
    }
    endpoint *T = build_T(0, n, m, sl, sh, ul, uh);
    if (!T) { free(slot); free(cnt); return ORC_ERR_ALLOC; }
    qsort(T, (size_t)N2, sizeof(endpoint), cmp_endpoint);
    idset SubSet, UpdSet;
    if (idset_init(&SubSet, n) || idset_init(&UpdSet, m)) { free(T); free(slot); free(cnt); return ORC_ERR_ALLOC; }
    /* pass 1: snapshot sizes; pass 2: the members, at offsets from pass 1 */
    pairbuf pb = {0};
    for (int pass = 0; pass < 2; ++pass) {
        if (pass == 1) {
            sub_off[0] = 0;
            for (int64_t r = 0; r < nq; ++r) sub_off[r + 1] = sub_off[r] + cnt[r];
            if (!sub_ids || sub_off[nq] > sub_cap) break;  /* size query / too small */
            SubSet.size = 0;
            UpdSet.size = 0;
            for (int64_t i = 0; i < n; ++i) SubSet.pos[i] = -1;
            for (int64_t j = 0; j < m; ++j) UpdSet.pos[j] = -1;
        }
        for (int64_t t = 0; t < N2; ++t) {
            if (T[t].kind == 1 && !T[t].is_upper && slot[T[t].id] >= 0) {
                const int64_t r = slot[T[t].id];
                if (pass == 0) cnt[r] = SubSet.size;
                else {
                    int64_t w = sub_off[r];
                    states_flatten(&SubSet, sub_ids, &w, sub_off[r] + SubSet.size);
                }
            }
            sbm_step(&T[t], &SubSet, &UpdSet, &pb, 1, 1, sl, sh, n, ul, uh, m);
        }
    }
    int64_t total = 0;
    for (int64_t r = 0; r < nq; ++r) total += cnt[r];
    idset_free(&SubSet);
    idset_free(&UpdSet);
    free(T);
    free(slot);
    free(cnt);
    return (sub_ids && total > sub_cap) ? ORC_ERR_ARG : total;
}

/* ------------------------------------------------ Parallel SBM (Alg. 5+6) */

/* Parallel sort of T (Alg. 5 l.3): P chunks sorted concurrently, then
 * pairwise merge rounds (the paper used GNU parallel std::sort). */
static int parallel_sort_T(endpoint *T, int64_t len, int P) {
    if (len < 2) return ORC_OK;
    endpoint *tmp = (endpoint *)malloc((size_t)len * sizeof(endpoint));
    if (!tmp) return ORC_ERR_ALLOC;
    int64_t *b = (int64_t *)malloc(sizeof(int64_t) * (size_t)(P + 1));
    if (!b) { free(tmp); return ORC_ERR_ALLOC; }
    plan_segments(len, P, b);
#pragma omp parallel for schedule(static, 1)
    for (int p = 0; p < P; ++p)
        qsort(T + b[p], (size_t)(b[p + 1] - b[p]), sizeof(endpoint), cmp_endpoint);
    endpoint *src = T, *dst = tmp;
    for (int width = 1; width < P; width *= 2) {
#pragma omp parallel for schedule(static, 1)
        for (int p = 0; p < P; p += 2 * width) {
            int64_t lo = b[p], mid = b[p + width < P ? p + width : P], hi = b[p + 2 * width < P ? p + 2 * width : P];
            int64_t x = lo, y = mid, w = lo;
            while (x < mid && y < hi) dst[w++] = cmp_endpoint(&src[y], &src[x]) < 0 ? src[y++] : src[x++];
            while (x < mid) dst[w++] = src[x++];
            while (y < hi) dst[w++] = src[y++];
        }
        endpoint *t = src; src = dst; dst = t;
    }
    if (src != T) memcpy(T, src, (size_t)len * sizeof(endpoint));
    free(tmp);
    free(b);
    return ORC_OK;
}

typedef struct {
    idset Sadd, Sdel, Uadd, Udel;
} deltas;

/* Alg. 6 lines 1-24: local delta scan of segment T_p. */
static void local_delta_scan(const endpoint *T, int64_t lo, int64_t hi, deltas *D) {
    for (int64_t q = lo; q < hi; ++q) {
        const endpoint *t = &T[q];
        idset *add = t->kind == 0 ? &D->Sadd : &D->Uadd;
        idset *del = t->kind == 0 ? &D->Sdel : &D->Udel;
        if (!t->is_upper) idset_insert(add, t->id);        /* lower bound: add */
        else if (idset_has(add, t->id)) idset_erase(add, t->id); /* ElsIf in add: remove */
        else idset_insert(del, t->id);                     /* Else: del */
    }
}

typedef struct {
    uint32_t *ids;
    int64_t size;
} idlist;

static int snapshot(const idset *s, idlist *l) {
    l->size = s->size;
    l->ids = (uint32_t *)malloc((size_t)(s->size > 0 ? s->size : 1) * sizeof(uint32_t));
    if (!l->ids) return ORC_ERR_ALLOC;
    memcpy(l->ids, s->members, (size_t)s->size * sizeof(uint32_t));
    return ORC_OK;
}

/* Shared driver of Alg. 5 + Alg. 6.  If `states_only`, stops after the master
 * combine and returns SubSet[p]/UpdSet[p] via the flat outputs. */
static int64_t par_sbm_impl(int64_t n, int64_t m, const double *sl, const double *sh,
                            const double *ul, const double *uh, int P, int count_only,
                            uint64_t *out, int64_t cap, int states_only, uint32_t *sub_ids,
                            int64_t *sub_off, int64_t sub_cap, uint32_t *upd_ids, int64_t *upd_off,
                            int64_t upd_cap) {
    if (P < 1) return ORC_ERR_ARG;
    int64_t N2 = 2 * (n + m);
    /* Alg. 5 l.2-4: parallel fill of T; l.5: parallel sort. */
    endpoint *T = build_T(0, n, m, sl, sh, ul, uh);
    if (!T) return ORC_ERR_ALLOC;
    if (parallel_sort_T(T, N2, P)) { free(T); return ORC_ERR_ALLOC; }
    /* Alg. 5 l.6: split T into P segments. */
    int64_t *b = (int64_t *)malloc(sizeof(int64_t) * (size_t)(P + 1));
    deltas *D = (deltas *)calloc((size_t)P, sizeof(deltas));
    idlist *SubSet0 = (idlist *)calloc((size_t)P, sizeof(idlist));
    idlist *UpdSet0 = (idlist *)calloc((size_t)P, sizeof(idlist));
    if (!b || !D || !SubSet0 || !UpdSet0) { free(T); free(b); free(D); free(SubSet0); free(UpdSet0); return ORC_ERR_ALLOC; }
    plan_segments(N2, P, b);
    int err = 0;
    /* Alg. 6 l.1-24, executed by all cores in parallel. */
#pragma omp parallel for schedule(static, 1) reduction(| : err)
    for (int p = 0; p < P; ++p) {
        if (idset_init(&D[p].Sadd, n) || idset_init(&D[p].Sdel, n) || idset_init(&D[p].Uadd, m) ||
            idset_init(&D[p].Udel, m)) { err |= 1; continue; }
        local_delta_scan(T, b[p], b[p + 1], &D[p]);
    }
    /* Alg. 6 l.25-28, executed by the master only:
     *   SubSet[0] = UpdSet[0] = {};  SubSet[p] = SubSet[p-1] U Sadd[p-1] \ Sdel[p-1]. */
    idset curS = {0}, curU = {0};
    if (err || idset_init(&curS, n) || idset_init(&curU, m)) err = 1;
    for (int p = 0; p < P && !err; ++p) {
        if (p > 0) {
            for (int64_t q = 0; q < D[p - 1].Sadd.size; ++q) idset_insert(&curS, D[p - 1].Sadd.members[q]);
            for (int64_t q = 0; q < D[p - 1].Sdel.size; ++q) idset_erase(&curS, D[p - 1].Sdel.members[q]);
            for (int64_t q = 0; q < D[p - 1].Uadd.size; ++q) idset_insert(&curU, D[p - 1].Uadd.members[q]);
            for (int64_t q = 0; q < D[p - 1].Udel.size; ++q) idset_erase(&curU, D[p - 1].Udel.members[q]);
        }
        if (snapshot(&curS, &SubSet0[p]) || snapshot(&curU, &UpdSet0[p])) err = 1;
    }
    int64_t result = 0;
    if (!err && states_only) {
        int64_t ws = 0, wu = 0;
        for (int p = 0; p < P && result == 0; ++p) {
            sub_off[p] = ws;
            upd_off[p] = wu;
            if (ws + SubSet0[p].size > sub_cap) { result = ORC_ERR_ARG; break; }
            memcpy(sub_ids + ws, SubSet0[p].ids, (size_t)SubSet0[p].size * sizeof(uint32_t));
            ws += SubSet0[p].size;
            if (wu + UpdSet0[p].size > upd_cap) { result = ORC_ERR_ARG; break; }
            memcpy(upd_ids + wu, UpdSet0[p].ids, (size_t)UpdSet0[p].size * sizeof(uint32_t));
            wu += UpdSet0[p].size;
        }
        if (result == 0) {
            sub_off[P] = ws;
            upd_off[P] = wu;
            result = ws + wu;
        }
    } else if (!err) {
        /* Alg. 5 l.7-33: final local scans in parallel from the initial sets;
         * "Atomic L <- L U ..." realised as private buffers concatenated in
         * segment order (reading R9). */
        pairbuf *pb = (pairbuf *)calloc((size_t)P, sizeof(pairbuf));
        int64_t *left = (int64_t *)calloc((size_t)P, sizeof(int64_t));
        if (!pb || !left) err = 1;
#pragma omp parallel for schedule(static, 1) reduction(| : err)
        for (int p = 0; p < P; ++p) {
            if (err) continue;
            idset SubSet, UpdSet;
            if (idset_init(&SubSet, n) || idset_init(&UpdSet, m)) { err |= 1; continue; }
            for (int64_t q = 0; q < SubSet0[p].size; ++q) idset_insert(&SubSet, SubSet0[p].ids[q]);
            for (int64_t q = 0; q < UpdSet0[p].size; ++q) idset_insert(&UpdSet, UpdSet0[p].ids[q]);
            pb[p].store = !count_only && out != NULL;
            for (int64_t q = b[p]; q < b[p + 1]; ++q)
                sbm_step(&T[q], &SubSet, &UpdSet, &pb[p], count_only, 1, sl, sh, n, ul, uh, m);
            left[p] = SubSet.size + UpdSet.size;
            idset_free(&SubSet);
            idset_free(&UpdSet);
        }
        if (!err) {
            int64_t K = 0;
            for (int p = 0; p < P; ++p) K += pb[p].count;
            int stored = 1;
            for (int p = 0; p < P; ++p) stored &= pb[p].store ? pb[p].size == pb[p].count : 0;
            if (!count_only && out && K <= cap && stored) {
                int64_t w = 0;
                for (int p = 0; p < P; ++p) { memcpy(out + w, pb[p].v, (size_t)pb[p].size * sizeof(uint64_t)); w += pb[p].size; }
            }
            /* the last segment must end with empty sets */
            result = left[P - 1] == 0 ? K : ORC_ERR_SETS_NOT_EMPTY;
        }
        if (pb) for (int p = 0; p < P; ++p) free(pb[p].v);
        free(pb);
        free(left);
    }
    if (err) result = ORC_ERR_ALLOC;
    for (int p = 0; p < P; ++p) {
        if (D[p].Sadd.members) { idset_free(&D[p].Sadd); idset_free(&D[p].Sdel); idset_free(&D[p].Uadd); idset_free(&D[p].Udel); }
        free(SubSet0[p].ids);
        free(UpdSet0[p].ids);
    }
    if (curS.members) idset_free(&curS);
    if (curU.members) idset_free(&curU);
    free(D);
    free(SubSet0);
    free(UpdSet0);
    free(b);
    free(T);
    return result;
}

/* Alg. 5 Parallel-SBM-1D with Alg. 6 initialisation, P segments/threads. */
int64_t orc_par_sbm(int64_t n, int64_t m, const double *sl, const double *sh, const double *ul,
                    const double *uh, int P, int count_only, uint64_t *out, int64_t cap) {
#ifdef _OPENMP
    int saved = omp_get_max_threads();
    omp_set_num_threads(P);
#endif
    int64_t r = par_sbm_impl(n, m, sl, sh, ul, uh, P, count_only, out, cap, 0, NULL, NULL, 0, NULL, NULL, 0);
#ifdef _OPENMP
    omp_set_num_threads(saved);
#endif
    return r;
}

/* SubSet[p] / UpdSet[p] as computed by Alg. 6 (unsorted ids per segment). */
int64_t orc_par_sbm_states(int64_t n, int64_t m, const double *sl, const double *sh,
                           const double *ul, const double *uh, int P, uint32_t *sub_ids,
                           int64_t *sub_off, int64_t sub_cap, uint32_t *upd_ids, int64_t *upd_off,
                           int64_t upd_cap) {
    return par_sbm_impl(n, m, sl, sh, ul, uh, P, 1, NULL, 0, 1, sub_ids, sub_off, sub_cap, upd_ids,
                        upd_off, upd_cap);
}

int orc_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
