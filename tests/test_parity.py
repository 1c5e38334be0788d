"""GPU parity: libddm (through the C ABI) vs the CPU oracle, bit-exact.

Endpoints are compared exactly on both sides, so there is no tolerance: the
GPU pair count must equal the oracle's and the GPU pair list, canonicalised
as ascending (upd << 32) | sub, must be byte-equal to the oracle's
(SURVEY §8(c) parity rule).  All inputs are seeded and synthetic.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_1703_06680_b200 import ddm
from paper_1703_06680_b200 import workload as wl
from tests.helpers import arrays, cuda, gpu_args, oracle_list_by_cells, raw_words, words_of

EMIT_FLAGS = [ddm.DDM_EMIT_AUTO, ddm.DDM_EMIT_FORCE_THREAD, ddm.DDM_EMIT_FORCE_WARP, ddm.DDM_EMIT_FORCE_CHUNK,
              ddm.DDM_SORT_LSB, ddm.DDM_SORT_LSB | ddm.DDM_EMIT_FORCE_CHUNK,
              ddm.DDM_COUNT_WALK, ddm.DDM_COUNT_WALK | ddm.DDM_EMIT_FORCE_CHUNK,
              ddm.DDM_COUNT_WALK | ddm.DDM_SORT_LSB, ddm.DDM_COUNT_RANKS]
# d > 1: both tiled filter forms at any size (row-indexed 4096-row tiles,
# chunk-indexed 1024-row tiles), with the MSD and the LSB sorts
DD_FLAGS = [ddm.DDM_DD_FORCE_ROWS, ddm.DDM_DD_FORCE_CHUNKS, ddm.DDM_DD_FORCE_ROWS | ddm.DDM_SORT_LSB]


@pytest.fixture(scope="module", autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA GPU")
    ddm.load()


def check_against(orc, sl, sh, ul, uh, flags=(0,), ref=None):
    a = [np.ascontiguousarray(np.asarray(x, dtype=np.float64)) for x in (sl, sh, ul, uh)]
    a = [x if x.ndim == 2 else x[None] for x in a]
    if ref is None:
        ref = orc.sbm_seq(*a)
    g = [cuda(x) for x in a]
    assert ddm.match_count(*g) == ref.size
    first = {}
    per_row = ddm.DDM_EMIT_FORCE_THREAD | ddm.DDM_EMIT_FORCE_WARP
    for f in flags:
        p = ddm.match_pairs(*g, flags=f)
        assert p.shape[0] == ref.size
        got = words_of(p)
        assert np.array_equal(got, ref), f"flags={f}"
        # d = 1: every emission path writes byte-identical output (rows by
        # sweep order, each row in Slo order).  d > 1: the tiled filter and
        # the per-row filter each write a deterministic order of their own.
        # (d > 1: one family per forced filter form; the default form depends
        # on the sizes)
        fam = f & (per_row | ddm.DDM_DD_FORCE_ROWS | ddm.DDM_DD_FORCE_CHUNKS) if a[0].shape[0] > 1 else 0
        if fam not in first:
            first[fam] = raw_words(p)
        else:
            assert np.array_equal(raw_words(p), first[fam]), f"flags={f}"
    return ref


# ------------------------------------------------------------ key encoding and sort

def test_encode_keys_order_preserving():
    vals = np.array([-np.finfo(np.float64).max, -1e300, -2.5, -1.0, -5e-324, -0.0, 0.0, 5e-324,
                     2.2250738585072014e-308, 1.0, 1.0000000000000002, 3.0, 1e300,
                     np.finfo(np.float64).max])
    k = ddm.encode_keys(cuda(vals)).cpu().numpy().view(np.uint64)
    assert k[5] == k[6]                       # -0.0 and +0.0 encode equally
    assert np.all(np.diff(k[6:].astype(object)) > 0) and np.all(np.diff(k[:6].astype(object)) > 0)
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.normal(0, 1e3, 5000), rng.uniform(-1, 1, 5000) * 1e-310, [0.0, -0.0] * 10])
    kx = ddm.encode_keys(cuda(x)).cpu().numpy().view(np.uint64)
    order_k = np.argsort(kx, kind="stable")
    order_x = np.argsort(x + 0.0, kind="stable")
    assert np.array_equal(x[order_k], x[order_x])


@pytest.mark.parametrize("n", [1, 31, 4095, 4096, 4097, 12289, 100_003, 1_000_000])
@pytest.mark.parametrize("spread", ["full", "dups"])
def test_radix_sort_matches_stable_sort(n, spread):
    rng = np.random.default_rng(n)
    if spread == "full":
        keys = rng.integers(0, 2**63, n, dtype=np.int64).view(np.uint64) * np.uint64(2) + rng.integers(0, 2, n).astype(np.uint64)
    else:
        keys = rng.integers(0, 7, n).astype(np.uint64) << np.uint64(40)
    kt = torch.from_numpy(keys.view(np.int64)).cuda()
    ko, vo = ddm.radix_sort_u64(kt)
    ref = np.argsort(keys, kind="stable")
    assert np.array_equal(ko.cpu().numpy().view(np.uint64), keys[ref])
    assert np.array_equal(vo.cpu().numpy(), ref.astype(np.int32))


@pytest.mark.parametrize("bits", [(0, 20), (8, 40), (32, 61)])
def test_radix_sort_bit_ranges(bits):
    rng = np.random.default_rng(bits[0])
    keys = rng.integers(0, 2**62, 50_000, dtype=np.int64).view(np.uint64)
    vals = rng.integers(0, 2**31, 50_000).astype(np.int32)
    ko, vo = ddm.radix_sort_u64(torch.from_numpy(keys.view(np.int64)).cuda(), torch.from_numpy(vals).cuda(),
                                bits[0], bits[1])
    sub = (keys >> np.uint64(bits[0])) & np.uint64((1 << (bits[1] - bits[0])) - 1)
    ref = np.argsort(sub, kind="stable")
    assert np.array_equal(ko.cpu().numpy().view(np.uint64), keys[ref])
    assert np.array_equal(vo.cpu().numpy(), vals[ref])


# ------------------------------------------------------------ worked examples and edge cases

@pytest.mark.parametrize("S,U,K", [
    ([(0, 10)], [(2, 3)], 1),          # S:178 nested
    ([(1, 2)], [(1, 2)], 1),           # S:129 identical
    ([(5, 10)], [(10, 12)], 1),        # S:56 touching
    ([(5, 5)], [(5, 9)], 1),           # S:77 point interval
    ([(0, 1)], [(2, 3)], 0),           # S:55 disjoint
    ([(-1, -0.0)], [(0.0, 1)], 1),     # -0.0 vs +0.0 (DESIGN reading R3)
    ([(0.0, 0.0)], [(-0.0, -0.0)], 1),
])
def test_small_cases(orc, S, U, K):
    sl, sh = [s[0] for s in S], [s[1] for s in S]
    ul, uh = [u[0] for u in U], [u[1] for u in U]
    ref = check_against(orc, sl, sh, ul, uh, flags=EMIT_FLAGS)
    assert ref.size == K


def test_fig1_instance(orc):
    import json, os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "fig1_instance.json")))
    sl = np.array([[s[k][0] for s in g["sub"]] for k in range(2)])
    sh = np.array([[s[k][1] for s in g["sub"]] for k in range(2)])
    ul = np.array([[u[k][0] for u in g["upd"]] for k in range(2)])
    uh = np.array([[u[k][1] for u in g["upd"]] for k in range(2)])
    expect = np.array(sorted(((u - 1) << 32) | (s - 1) for s, u in g["expected_pairs_1based"]), dtype=np.uint64)
    check_against(orc, sl, sh, ul, uh, flags=EMIT_FLAGS, ref=expect)


def test_tie_storms(orc):
    """Random instances with integer endpoints in {0..4} (every kind of tie)."""
    rng = np.random.default_rng(7)
    for _ in range(120):
        n, m = rng.integers(1, 40, 2)
        s = np.sort(rng.integers(0, 5, (2, n)), axis=0).astype(np.float64)
        u = np.sort(rng.integers(0, 5, (2, m)), axis=0).astype(np.float64)
        ref = orc.bf_pairs(s[0:1], s[1:2], u[0:1], u[1:2])
        check_against(orc, s[0:1], s[1:2], u[0:1], u[1:2], flags=EMIT_FLAGS, ref=ref)


def test_random_mixtures_fuzz(orc):
    """Seeded fuzz over sizes spanning several sort/count/emit tiles and
    mixtures of distributions: uniform, clustered spikes (bucket-map
    equalisation), duplicates, long intervals, negative and mixed-magnitude
    coordinates, point intervals; d = 1..3.  Every case against brute force."""
    rng = np.random.default_rng(2024)
    for case in range(24):
        d = int(rng.integers(1, 4))
        n, m = (int(x) for x in rng.integers(1, 9000, 2))
        def side(cnt):
            kind = rng.integers(0, 5)
            if kind == 0:
                lo = rng.uniform(-1e3, 1e3, (d, cnt))
            elif kind == 1:  # a few dense spikes
                c = rng.uniform(-1e6, 1e6, 4)
                lo = c[rng.integers(0, 4, (d, cnt))] + rng.normal(0, 1e-3, (d, cnt))
            elif kind == 2:  # heavy duplicates
                lo = rng.integers(-5, 5, (d, cnt)).astype(np.float64)
            elif kind == 3:  # mixed magnitudes
                lo = rng.choice([-1.0, 1.0], (d, cnt)) * 10.0 ** rng.uniform(-300, 300, (d, cnt))
            else:
                lo = rng.uniform(0, 1e5, (d, cnt))
            ln = np.abs(rng.normal(0, 50.0, (d, cnt)))
            ln[rng.random((d, cnt)) < 0.02] = 1e6   # long intervals
            ln[rng.random((d, cnt)) < 0.05] = 0.0   # points
            return lo, lo + ln
        sl, sh = side(n)
        ul, uh = side(m)
        ok = np.all(np.isfinite(sh)) and np.all(np.isfinite(uh))
        if not ok:
            continue
        ref = orc.bf_pairs(sl, sh, ul, uh)
        flags = EMIT_FLAGS if case % 4 == 0 else (0, ddm.DDM_COUNT_WALK)
        check_against(orc, sl, sh, ul, uh, flags=flags, ref=ref)


def test_extreme_magnitudes(orc):
    rng = np.random.default_rng(3)
    v = np.concatenate([rng.uniform(-1, 1, 300) * 1e308, rng.uniform(-1, 1, 300) * 5e-324 * 1000,
                        [-5e-324, 5e-324, 0.0, -0.0, 1e308, -1e308]])
    lo = rng.choice(v, 800)
    ln = rng.choice([0.0, 5e-324, 1e-310, 1.0, 1e300], 800)
    hi = np.where(lo + ln >= lo, lo + ln, lo)
    hi = np.where(np.isfinite(hi), hi, lo)
    ref = orc.bf_pairs(lo[None, :400], hi[None, :400], lo[None, 400:], hi[None, 400:])
    check_against(orc, lo[:400], hi[:400], lo[400:], hi[400:], flags=EMIT_FLAGS, ref=ref)


def test_duplicates_all_overlap(orc):
    n = 2000
    z = np.zeros(n)
    o = np.ones(n)
    g = [cuda(x) for x in (z, o, z, o)]
    assert ddm.match_count(*g) == n * n
    p = ddm.match_pairs(*g)
    w = words_of(p)
    assert w.size == n * n and np.array_equal(w, orc.bf_pairs(z[None], o[None], z[None], o[None]))


def test_asymmetric(orc):
    rng = np.random.default_rng(11)
    lo = rng.uniform(0, 1e6, 1_000_000)
    hi = lo + 10.0
    one_lo, one_hi = np.array([5e5]), np.array([5e5 + 3e3])
    check_against(orc, one_lo, one_hi, lo, hi, ref=orc.bf_pairs(one_lo[None], one_hi[None], lo[None], hi[None]))
    check_against(orc, lo, hi, one_lo, one_hi, ref=orc.bf_pairs(lo[None], hi[None], one_lo[None], one_hi[None]))


def test_empty_sides():
    e = cuda(np.zeros(0))
    x = cuda(np.array([1.0, 2.0]))
    assert ddm.match_count(e, e, x, x) == 0
    assert ddm.match_count(x, x, e, e) == 0
    assert ddm.match_pairs(x, x, e, e).shape[0] == 0


def test_long_intervals(orc):
    """1% of subscriptions span the whole domain (exercises the block-max skips)."""
    rng = np.random.default_rng(21)
    w = wl.uniform(20_000, 20_000, 1e6, 50.0, 1, seed=5)
    sl, sh = w.sub_lo.copy(), w.sub_hi.copy()
    idx = rng.choice(w.n, w.n // 100, replace=False)
    sl[0, idx] = 0.0
    sh[0, idx] = 1e6
    check_against(orc, sl, sh, w.upd_lo, w.upd_hi, flags=EMIT_FLAGS)
    # a single long interval at the very start, rest short
    sl2, sh2 = w.sub_lo.copy(), w.sub_hi.copy()
    sl2[0, 0], sh2[0, 0] = -1.0, 2e6
    check_against(orc, sl2, sh2, w.upd_lo, w.upd_hi, flags=EMIT_FLAGS)


@pytest.mark.parametrize("n", [1, 31, 32, 33, 1023, 1024, 1025, 2049, 40_000])
def test_stab_walk_prefix_max_blocks(orc, n):
    """Walk-form counts (pairs calls): the stop test max(pmw[i], pmb[i/1024])
    < a and the block skips across 32- and 1024-entry boundaries, with long
    intervals placed just before / after block edges and dense stab sets;
    against brute force, forced walk vs rank forms (EMIT_FLAGS)."""
    rng = np.random.default_rng(n)
    m = max(1, n // 2)
    sl = np.sort(rng.uniform(0, 1e4, n))[None].copy()
    sh = sl + rng.exponential(3.0, n)[None]
    for pos in (0, 31, 32, 1023, 1024, n // 2, n - 1):
        if pos < n:
            sh[0, pos] = sl[0, pos] + rng.uniform(100, 5e3)
    perm = rng.permutation(n)
    sl, sh = sl[:, perm], sh[:, perm]
    ul = rng.uniform(-10, 1.1e4, m)[None]
    uh = ul + rng.exponential(2.0, m)[None]
    ref = orc.bf_pairs(sl, sh, ul, uh)
    check_against(orc, sl, sh, ul, uh, flags=EMIT_FLAGS, ref=ref)


def test_clamped_mixture_ties(orc):
    """c5-style clustered lower bounds with clamping -> point masses (ties)."""
    rng = np.random.default_rng(4)
    L, l = 1e6, 5.0
    c = rng.uniform(0, L, 8)
    lo = np.clip(rng.normal(c[rng.integers(0, 8, 60_000)], 3e4), 0, L - l)
    hi = lo + rng.uniform(0.5 * l, 1.5 * l, lo.size)
    check_against(orc, lo[:30_000], hi[:30_000], lo[30_000:], hi[30_000:], flags=EMIT_FLAGS)


# ------------------------------------------------------------ BASELINE configs

def test_c1_full(orc):
    w = wl.make("c1")
    ref = orc.bf_pairs(w.sub_lo, w.sub_hi, w.upd_lo, w.upd_hi)
    assert np.array_equal(orc.sbm_seq(w.sub_lo, w.sub_hi, w.upd_lo, w.upd_hi), ref)
    check_against(orc, w.sub_lo, w.sub_hi, w.upd_lo, w.upd_hi, flags=EMIT_FLAGS, ref=ref)


@pytest.mark.parametrize("alpha", [0.01, 1.0, 100.0])
def test_ragged_sizes(orc, alpha):
    """Sizes that span several sort/count/emit tiles and leave ragged tails."""
    for n, m in [(4097, 12289), (9000, 2049), (33_333, 30_001)]:
        N = n + m
        w = wl.uniform(n, m, 1e6, wl.side_length(N, 1e6, alpha, 1), 1, seed=n + m)
        check_against(orc, w.sub_lo, w.sub_hi, w.upd_lo, w.upd_hi, flags=EMIT_FLAGS)


def test_c2_full(orc):
    w = wl.make("c2")
    g = gpu_args(w)
    K = ddm.match_count(*g)
    assert K == orc.rank_count(w.sub_lo, w.sub_hi, w.upd_lo, w.upd_hi)
    ref = orc.sbm_seq(w.sub_lo, w.sub_hi, w.upd_lo, w.upd_hi)
    assert ref.size == K
    for f in EMIT_FLAGS:
        p = ddm.match_pairs(*g, flags=f)
        assert np.array_equal(words_of(p), ref)


def _check_sampled_rows(orc, w, p, n_rows=400, seed=0):
    """Rows of the GPU list for random update ids == brute force rows."""
    rng = np.random.default_rng(seed)
    rows = np.sort(rng.choice(w.m, size=min(n_rows, w.m), replace=False))
    ref, counts = orc.bf_rows(w.sub_lo, w.sub_hi, w.upd_lo, w.upd_hi, rows)
    pw = words_of(p)
    upd = (pw >> np.uint64(32)).astype(np.int64)
    lo = np.searchsorted(upd, rows, side="left")
    hi = np.searchsorted(upd, rows, side="right")
    got = np.concatenate([pw[a:b] for a, b in zip(lo, hi)]) if rows.size else pw[:0]
    assert np.array_equal(hi - lo, counts)
    assert np.array_equal(got, ref)


def test_c3_full_sampled(orc):
    """c3 at full size (N = 1e8), the bench configuration: K against the
    rank identity over numpy sorts, sampled rows against brute force, and
    list invariants (no duplicate, every pair overlaps)."""
    w = wl.make("c3")
    g = gpu_args(w)
    p = ddm.match_pairs(*g)
    K = p.shape[0]
    assert K == orc.rank_count(w.sub_lo, w.sub_hi, w.upd_lo, w.upd_hi)
    # invariants on the device
    s, u = p[:, 0].long(), p[:, 1].long()
    assert bool(((g[0][0][s] <= g[3][0][u]) & (g[2][0][u] <= g[1][0][s])).all())
    wds = torch.sort((u << 32) | s).values
    assert bool((wds[1:] > wds[:-1]).all())
    _check_sampled_rows(orc, w, p)
    # the default picks the walk-form counts here (sparse stab sets); the
    # rank form writes byte-identical output
    del s, u, wds
    p2 = ddm.match_pairs(*g, flags=ddm.DDM_COUNT_RANKS)
    assert torch.equal(p, p2)


def test_c4_scaled(orc):
    """d = 3 (c4 recipe) at a size the oracle finishes quickly."""
    w = wl.uniform(20_000, 20_000, 1e4, wl.side_length(40_000, 1e4, 1.0, 3) * 3.0, 3, seed=3)
    ref = orc.sbm_seq(w.sub_lo, w.sub_hi, w.upd_lo, w.upd_hi)
    assert np.array_equal(ref, orc.bf_pairs(w.sub_lo, w.sub_hi, w.upd_lo, w.upd_hi))
    check_against(orc, w.sub_lo, w.sub_hi, w.upd_lo, w.upd_hi, flags=EMIT_FLAGS + DD_FLAGS, ref=ref)


@pytest.mark.parametrize("d", [2, 3, 4, 5, 8])
def test_dd_tie_storms(orc, d):
    rng = np.random.default_rng(d)
    for _ in range(40):
        n, m = rng.integers(1, 30, 2)
        s = np.sort(rng.integers(0, 4, (2, d, n)), axis=0).astype(np.float64)
        u = np.sort(rng.integers(0, 4, (2, d, m)), axis=0).astype(np.float64)
        ref = orc.bf_pairs(s[0], s[1], u[0], u[1])
        assert np.array_equal(orc.sbm_dd_literal(s[0], s[1], u[0], u[1]), ref)
        check_against(orc, s[0], s[1], u[0], u[1], flags=EMIT_FLAGS + DD_FLAGS, ref=ref)


def test_c4_full_exact(orc):
    """c4 at full size (d = 3, N = 1e7): the whole GPU pair list is
    byte-identical to the oracle's (serial SBM, Alg. 4 + filter, assembled
    over 3-D cells of side 500 -- every pair of the instance, no sampling),
    and the count entry point agrees (BASELINE north star: bit-exact K and
    list on every config)."""
    w = wl.make("c4")
    g = gpu_args(w)
    p = ddm.match_pairs(*g)
    K = p.shape[0]
    assert ddm.match_count(*g) == K
    got = words_of(p)
    del p, g
    torch.cuda.empty_cache()
    ref = oracle_list_by_cells(orc, w, 500.0)
    assert ref.size == K
    assert np.array_equal(got, ref)


def test_sweep_dim_choice_skewed(orc):
    """k* = argmin_k K_k: with long dim-0 extents and short
    dim-1 extents the pipeline sweeps dimension 1 (its rows then follow the
    dim-1 lower bounds); the pair set equals the oracle's and the forced
    dim-0 sweep's (DDM_SWEEP_DIM0), for pairs and count."""
    rng = np.random.default_rng(81)
    for d in (2, 3):
        n, m = 30_000, 25_000
        sl = rng.uniform(0, 1e4, (d, n))
        ul = rng.uniform(0, 1e4, (d, m))
        ls = np.full((d, 1), 60.0)
        ls[0] = 900.0  # dim 0: long (dense); dim 1 shortest, so k* = 1
        ls[1] = 3.0
        sh, uh = sl + ls, ul + ls
        ref = orc.sbm_seq(sl, sh, ul, uh)
        g = [cuda(x) for x in (sl, sh, ul, uh)]
        p = ddm.match_pairs(*g)
        assert np.array_equal(words_of(p), ref)
        # rows follow the lower bounds of the swept dimension 1
        rows_lo = ul[1][p[:, 1].cpu().numpy().astype(np.int64)]
        assert np.all(np.diff(rows_lo) >= 0)
        p0 = ddm.match_pairs(*g, flags=ddm.DDM_SWEEP_DIM0)
        assert np.array_equal(words_of(p0), ref)
        assert np.all(np.diff(ul[0][p0[:, 1].cpu().numpy().astype(np.int64)]) >= 0)
        assert ddm.match_count(*g) == ref.size
        for f in (ddm.DDM_EMIT_FORCE_THREAD, ddm.DDM_EMIT_FORCE_WARP, ddm.DDM_SORT_LSB):
            assert np.array_equal(words_of(ddm.match_pairs(*g, flags=f)), ref)


def test_literal_intersection_equals_sweep(orc):
    """G10, the literal reading of P:237-247: per-dimension pair sets sorted
    and intersected by sort-merge on the GPU equal the oracle's literal form
    (sbm_dd_literal), brute force and the filtered sweep; canonical order."""
    rng = np.random.default_rng(82)
    for d in (1, 2, 3, 5):
        for trial in range(3):
            n, m = int(rng.integers(1, 3000)), int(rng.integers(1, 3000))
            sl = np.floor(rng.uniform(0, 60, (d, n)))
            ul = np.floor(rng.uniform(0, 60, (d, m)))
            sh = sl + np.floor(rng.uniform(0, 12, (d, n)))
            uh = ul + np.floor(rng.uniform(0, 12, (d, m)))
            ref = orc.sbm_dd_literal(sl, sh, ul, uh)
            assert np.array_equal(ref, orc.bf_pairs(sl, sh, ul, uh))
            g = [cuda(x) for x in (sl, sh, ul, uh)]
            lit = ddm.match_pairs_literal(*g)
            assert np.array_equal(raw_words(lit), ref)  # already canonical
            assert np.array_equal(words_of(ddm.match_pairs(*g)), ref)
    # a per-dimension set larger than dim_capacity is refused, not truncated
    with pytest.raises(ddm.DDMError) as e:
        ddm.match_pairs_literal(*g, dim_capacity=1)
    assert e.value.status == 4


def test_dd_chunks_and_long_intervals(orc):
    """d = 2 and 3 with tiles whose candidate sets span many shared-memory
    chunks, long intervals in every dimension (A_t walk skips, dim-1 bin
    ranges covering all bins), negative coordinates and point extents."""
    rng = np.random.default_rng(33)
    for d in (2, 3):
        n, m = 6000, 7000
        sl = rng.uniform(-500.0, 500.0, (d, n))
        ul = rng.uniform(-500.0, 500.0, (d, m))
        sh = sl + rng.uniform(0.0, 120.0, (d, n))
        uh = ul + rng.uniform(0.0, 120.0, (d, m))
        big = rng.choice(n, 40, replace=False)
        sl[:, big[:20]] = -1e4
        sh[:, big[:20]] = 1e4
        sh[1, big[20:]] = sl[1, big[20:]] + 900.0
        pts = rng.choice(m, 50, replace=False)
        uh[:, pts] = ul[:, pts]
        ref = orc.bf_pairs(sl, sh, ul, uh)
        assert np.array_equal(orc.sbm_seq(sl, sh, ul, uh), ref)
        check_against(orc, sl, sh, ul, uh, flags=EMIT_FLAGS + DD_FLAGS, ref=ref)


def test_dd_degenerate_dim1(orc):
    """All dim-1 coordinates equal (zero-width bin range) and all dim-0
    coordinates equal (every sub a candidate of every row)."""
    rng = np.random.default_rng(34)
    n, m = 1500, 1300
    sl = np.stack([rng.uniform(0, 100, n), np.full(n, 7.0)])
    ul = np.stack([rng.uniform(0, 100, m), np.full(m, 7.0)])
    check_against(orc, sl, sl + 3.0, ul, ul + 3.0, flags=EMIT_FLAGS + DD_FLAGS)
    sl = np.stack([np.full(n, 1.0), rng.uniform(0, 100, n)])
    ul = np.stack([np.full(m, 1.0), rng.uniform(0, 100, m)])
    check_against(orc, sl, sl + 0.5, ul, ul + 0.5, flags=EMIT_FLAGS + DD_FLAGS)


def test_dd_staging_overflow(orc):
    """d > 1 tiles whose hits exceed the per-tile staging slot (8192) or a row
    with more than 65535 hits: the place pass re-enumerates them directly."""
    rng = np.random.default_rng(35)
    # dense tile: every region of both kinds overlaps every other (K = n*m)
    sl = rng.uniform(0.0, 0.5, (2, 300))
    ul = rng.uniform(0.0, 0.5, (2, 400))
    check_against(orc, sl, sl + 1.0, ul, ul + 1.0, flags=(0,) + tuple(DD_FLAGS))
    # one row with 70000 partners
    sl = rng.uniform(0.0, 0.5, (2, 70_000))
    ul = np.array([[0.2, 5.0], [0.3, 5.0]])
    check_against(orc, sl, sl + 1.0, ul, ul + 0.5, flags=(0,) + tuple(DD_FLAGS))


def test_dd_float_boundaries(orc):
    """d = 2, 3: the row-indexed filter decides most pairs on float32 boxes
    ("certain" when both inequalities hold with more than the rounding
    margin); endpoints one float64 ulp apart inside one float32 ulp, values
    beyond the float32 range (rd/ru saturate), subnormals and signed zeros
    must all fall to the exact test.  Brute force decides."""
    rng = np.random.default_rng(36)
    mags = np.array([0.0, 1e-310, 1e-40, 1.0, 3.0e38, 3.4028234663852886e38, 1e39, 1e300])
    for d in (2, 3):
        for trial in range(6):
            n, m = 700, 600
            def side(cnt):
                lo = rng.choice(mags, (d, cnt)) * rng.choice([-1.0, 1.0], (d, cnt))
                lo = lo * (1.0 + rng.integers(-2, 3, (d, cnt)) * 2.0 ** -52)
                ln = np.abs(lo) * rng.choice([0.0, 2.0 ** -52, 2.0 ** -30, 1e-7, 0.5], (d, cnt))
                return lo, lo + ln
            sl, sh = side(n)
            ul, uh = side(m)
            # partners that touch: some update bounds equal a sub bound (or one
            # double ulp away from it)
            k = rng.choice(m, 100, replace=False)
            j = rng.choice(n, 100)
            ul[:, k] = np.nextafter(sh[:, j], rng.choice([-np.inf, np.inf], (d, 100)))
            uh[:, k] = np.maximum(uh[:, k], ul[:, k])
            ref = orc.bf_pairs(sl, sh, ul, uh)
            check_against(orc, sl, sh, ul, uh, flags=(0,) + tuple(DD_FLAGS), ref=ref)


def test_dd_deterministic_output():
    w = wl.make("c4", scale=0.02)
    g = gpu_args(w)
    a = ddm.match_pairs(*g)
    b = ddm.match_pairs(*g)
    assert torch.equal(a, b)


def test_c5_full_windows(orc):
    """c5 at full size (N = 1e9, clustered, the bench configuration): K equal
    to the oracle's rank-identity count, the list invariants on the device
    (together: the list is the exact result set), count == list length, sampled rows against
    brute force over all 5e8 subscriptions, and three exact slices: every
    update whose lower bound lies in a window, matched by the oracle's
    Parallel-SBM against every subscription that can reach the window (lower
    bound within the longest subscription length of it), must have exactly
    the GPU's rows."""
    w = wl.make("c5")
    g = gpu_args(w)
    p = ddm.match_pairs(*g)
    K = p.shape[0]
    assert ddm.match_count(*g) == K
    # the oracle's count over all 1e9 regions (I2 rank identity, O3): with the
    # device checks below (every listed pair overlaps, no duplicates) this
    # proves the GPU list IS the result set -- a subset of the right size
    assert K == orc.rank_count(w.sub_lo, w.sub_hi, w.upd_lo, w.upd_hi)
    s, u = p[:, 0].long(), p[:, 1].long()
    assert bool(((g[0][0][s] <= g[3][0][u]) & (g[2][0][u] <= g[1][0][s])).all())
    wds = torch.sort((u << 32) | s).values
    assert bool((wds[1:] > wds[:-1]).all())
    del s, wds
    _check_sampled_rows(orc, w, p, n_rows=120)
    gpu_u = u.cpu().numpy()
    words = raw_words(p)
    del p, g, u
    torch.cuda.empty_cache()
    # a sub overlapping an update of [x0, x1) has x0 - len(S) <= S.lo <= U.hi < x1 + len(U)
    margin = max(float(np.max(w.sub_hi[0] - w.sub_lo[0])), float(np.max(w.upd_hi[0] - w.upd_lo[0]))) + 1.0
    for q in (0.25, 0.5, 0.75):
        x0 = float(np.quantile(w.upd_lo[0][::97], q))
        x1 = x0 + 2e6
        ui = np.nonzero((w.upd_lo[0] >= x0) & (w.upd_lo[0] < x1))[0]
        si = np.nonzero((w.sub_lo[0] >= x0 - margin) & (w.sub_lo[0] < x1 + margin))[0]
        loc = orc.par_sbm(w.sub_lo[:, si], w.sub_hi[:, si], w.upd_lo[:, ui], w.upd_hi[:, ui], canonicalize=False)
        ref = np.sort((ui[(loc >> np.uint64(32)).astype(np.int64)].astype(np.uint64) << np.uint64(32))
                      | si[(loc & np.uint64(0xffffffff)).astype(np.int64)].astype(np.uint64))
        inwin = np.zeros(w.m, dtype=bool)
        inwin[ui] = True
        got = np.sort(words[inwin[gpu_u]])
        assert ui.size > 1000 and np.array_equal(got, ref), f"window at quantile {q}"


def test_c5_scaled(orc):
    w = wl.clustered(400_000, 400_000, 1e9, 0.01 * 2500, seed=4)
    check_against(orc, w.sub_lo, w.sub_hi, w.upd_lo, w.upd_hi, flags=EMIT_FLAGS)


# ------------------------------------------------------------ errors and contract

def test_validation_errors():
    x = np.linspace(0, 10, 100)
    for bad, code in [(np.nan, 2), (np.inf, 2), (-np.inf, 2)]:
        y = x.copy()
        y[37] = bad
        with pytest.raises(ddm.DDMError) as e:
            ddm.match_pairs(cuda(y), cuda(x + 1), cuda(x), cuda(x + 1))
        assert e.value.status == code
        with pytest.raises(ddm.DDMError) as e:
            ddm.match_count(cuda(x), cuda(x + 1), cuda(x), cuda(np.where(np.arange(100) == 5, bad, x + 1)))
        assert e.value.status == code
    inv = x + 1
    inv[50] = x[50] - 1
    with pytest.raises(ddm.DDMError) as e:
        ddm.match_pairs(cuda(x), cuda(inv), cuda(x), cuda(x + 1))
    assert e.value.status == 3
    # other dimensions are validated too (d = 2)
    lo2 = np.stack([x, x])
    hi2 = np.stack([x + 1, inv])
    with pytest.raises(ddm.DDMError) as e:
        ddm.match_count(cuda(lo2), cuda(hi2), cuda(lo2), cuda(lo2 + 1))
    assert e.value.status == 3


def test_validation_errors_row_indexed_dd():
    """Row-indexed d > 1 calls validate dims 1-2 inside the float-box kernel
    (no separate validation launch): a non-finite or inverted coordinate on
    dim 1 or 2 of either side is still reported, dim 3 too."""
    rng = np.random.default_rng(5)
    lo = rng.uniform(0, 100, (4, 6000))
    hi = lo + 2.0
    for side, k, bad, code in [(0, 1, np.nan, 2), (1, 2, np.inf, 2), (0, 2, "inv", 3), (1, 1, "inv", 3),
                               (1, 3, np.nan, 2), (0, 3, "inv", 3)]:
        a = [lo.copy(), hi.copy(), lo.copy(), hi.copy()]
        if bad == "inv":
            a[2 * side + 1][k, 4321] = a[2 * side][k, 4321] - 1.0
        else:
            a[2 * side][k, 4321] = bad
        for f in (ddm.DDM_DD_FORCE_ROWS, ddm.DDM_DD_FORCE_CHUNKS):
            with pytest.raises(ddm.DDMError) as e:
                ddm.match_pairs(*[cuda(x) for x in a], flags=f)
            assert e.value.status == code, (side, k, bad, f)


def test_capacity_and_workspace():
    import ctypes
    L = ddm.load()
    x = cuda(np.zeros(100))
    y = cuda(np.ones(100))
    r, keep = ddm.regions(x, y, x, y)
    ws = torch.empty(L.ddm_workspace_bytes(1, 100, 100, 1), dtype=torch.uint8, device="cuda")
    K = ctypes.c_uint64(0)
    out = torch.empty((50, 2), dtype=torch.int32, device="cuda")
    st = L.ddm_match_pairs(ctypes.byref(r), out.data_ptr(), 50, ctypes.byref(K), 0, ws.data_ptr(), ws.numel(),
                           torch.cuda.current_stream().cuda_stream)
    assert st == 4 and K.value == 10_000
    st = L.ddm_match_pairs(ctypes.byref(r), out.data_ptr(), 50, ctypes.byref(K), 0, ws.data_ptr(), 1024,
                           torch.cuda.current_stream().cuda_stream)
    assert st == 5
    r.d = 0
    assert L.ddm_match_count(ctypes.byref(r), ctypes.byref(K), ws.data_ptr(), ws.numel(), None) == 1
    r.d = 9
    assert L.ddm_match_count(ctypes.byref(r), ctypes.byref(K), ws.data_ptr(), ws.numel(), None) == 1
    r.d = 1
    r.n_sub = 2**31
    assert L.ddm_match_count(ctypes.byref(r), ctypes.byref(K), ws.data_ptr(), ws.numel(), None) == 1
    r.n_sub = 100
    r.sub_lo[0] = None
    assert L.ddm_match_count(ctypes.byref(r), ctypes.byref(K), ws.data_ptr(), ws.numel(), None) == 1


def test_walk_capacity_and_graph_replay(orc):
    """Walk-form pairs calls: with capacity < K DDM_ERR_CAPACITY and K,
    nothing written past capacity; with enough room the output is exact, also
    on graph replays (second and third identical calls)."""
    import ctypes
    L = ddm.load()
    w = wl.uniform(30_000, 30_000, 1e5, 1.0, 1, seed=3)
    ref = orc.sbm_seq(w.sub_lo, w.sub_hi, w.upd_lo, w.upd_hi)
    K0 = ref.size
    g = gpu_args(w)
    r, keep = ddm.regions(*g)
    ws = torch.empty(L.ddm_workspace_bytes(1, w.n, w.m, 1), dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    K = ctypes.c_uint64(0)
    out = torch.empty((K0 + 64, 2), dtype=torch.int32, device="cuda")
    for cap in (K0 // 2, K0 // 2, K0 // 2):  # eager, capture, replay
        out.fill_(-7)
        s_ = L.ddm_match_pairs(ctypes.byref(r), out.data_ptr(), cap, ctypes.byref(K), ddm.DDM_COUNT_WALK,
                               ws.data_ptr(), ws.numel(), st)
        torch.cuda.synchronize()
        assert s_ == 4 and K.value == K0
        assert bool((out[cap:] == -7).all())
    for _ in range(3):
        out.fill_(-7)
        s_ = L.ddm_match_pairs(ctypes.byref(r), out.data_ptr(), K0, ctypes.byref(K), ddm.DDM_COUNT_WALK,
                               ws.data_ptr(), ws.numel(), st)
        torch.cuda.synchronize()
        assert s_ == 0 and K.value == K0
        assert np.array_equal(words_of(out[:K0]), ref)
        assert bool((out[K0:] == -7).all())


def test_capacity_dd_never_writes_past_capacity(orc):
    """d > 1 (single fused pass): capacity < K reports DDM_ERR_CAPACITY with the
    exact K and writes nothing at or past `capacity`; then the full call works."""
    import ctypes
    L = ddm.load()
    w = wl.uniform(3000, 3000, 100.0, 20.0, 2, seed=7)
    g = gpu_args(w)
    ref = orc.sbm_seq(w.sub_lo, w.sub_hi, w.upd_lo, w.upd_hi)
    r, keep = ddm.regions(*g)
    ws = torch.empty(L.ddm_workspace_bytes(2, w.n, w.m, 1), dtype=torch.uint8, device="cuda")
    K = ctypes.c_uint64(0)
    cap = ref.size // 3
    out = torch.full((ref.size, 2), -7, dtype=torch.int32, device="cuda")
    st = L.ddm_match_pairs(ctypes.byref(r), out.data_ptr(), cap, ctypes.byref(K), 0, ws.data_ptr(), ws.numel(),
                           torch.cuda.current_stream().cuda_stream)
    assert st == 4 and K.value == ref.size
    assert bool((out[cap:] == -7).all())
    st = L.ddm_match_pairs(ctypes.byref(r), out.data_ptr(), ref.size, ctypes.byref(K), 0, ws.data_ptr(),
                           ws.numel(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert st == 0 and np.array_equal(words_of(out), ref)


def test_graph_replay_reads_current_inputs(orc):
    """Identical repeated calls run the pre-sync half as a captured CUDA graph
    (from the 2nd call on): results stay exact when the input contents change
    in place between calls, and validation errors are still reported."""
    w = wl.make("c2", scale=0.05)
    g = [cuda(x) for x in (w.sub_lo, w.sub_hi, w.upd_lo, w.upd_hi)]
    M = ddm.Matcher(1, w.n, w.m)
    ref = orc.sbm_seq(w.sub_lo, w.sub_hi, w.upd_lo, w.upd_hi)
    out = torch.empty((ref.size * 2 + 16, 2), dtype=torch.int32, device="cuda")
    for _ in range(4):  # eager, capture, replay, replay
        k = M.pairs_into(out, *g)
        assert k == ref.size and np.array_equal(words_of(out[:k]), ref)
        assert M.count(*g) == ref.size
    rng = np.random.default_rng(5)
    for _ in range(2):  # new contents, same buffers
        sl = rng.uniform(0.0, w.L - w.l, w.n)
        ul = rng.uniform(0.0, w.L - w.l, w.m)
        for t, a in zip(g, (sl, sl + w.l, ul, ul + w.l)):
            t.copy_(torch.from_numpy(a[None]))
        ref2 = orc.sbm_seq(sl[None], (sl + w.l)[None], ul[None], (ul + w.l)[None])
        assert ref2.size < out.shape[0]
        k = M.pairs_into(out, *g)
        assert k == ref2.size and np.array_equal(words_of(out[:k]), ref2)
    g[0][0, 3] = float("nan")
    with pytest.raises(ddm.DDMError) as e:
        M.pairs_into(out, *g)
    assert e.value.status == 2


def test_pipelined_matcher_batches(orc):
    """PipelinedMatcher: a stream of host batches with overlapped copies; each
    batch's pairs (copied back into its own pinned buffer) equal the oracle's."""
    n = 20_000
    rng = np.random.default_rng(41)
    batches, refs = [], []
    for b in range(5):
        sl = rng.uniform(0, 1e6, (1, n))
        ul = rng.uniform(0, 1e6, (1, n))
        ln = 50.0 * (1 + b)
        host = [torch.from_numpy(np.ascontiguousarray(x)).pin_memory() for x in (sl, sl + ln, ul, ul + ln)]
        refs.append(orc.sbm_seq(sl, sl + ln, ul, ul + ln))
        batches.append(host)
    cap = max(r.size for r in refs)
    outs = [torch.empty((cap, 2), dtype=torch.int32).pin_memory() for _ in batches]
    pm = ddm.PipelinedMatcher(1, n, n, cap)
    got = list(pm.run(zip(batches, outs)))
    for (k, hout), ref in zip(got, refs):
        assert k == ref.size and np.array_equal(words_of(hout[:k]), ref)


def test_more_than_2_pow_32_pairs():
    """64-bit counts and offsets: 65537 point subscriptions inside [0, 1) and
    65537 updates covering [-1, 2] give K = 4,295,098,369 > 2^32 pairs (34 GB
    of output).  The count is exact; on the device every row is one update
    repeated n times, the rows are a permutation of the update ids, and
    sampled rows hold every subscription once."""
    n = 65537
    rng = np.random.default_rng(44)
    lo = rng.uniform(0.0, 1.0, n)
    ul = np.full(n, -1.0) - rng.uniform(0.0, 0.5, n)
    g = [cuda(lo), cuda(lo), cuda(ul), cuda(np.full(n, 2.0))]
    K = ddm.match_count(*g)
    assert K == n * n and K > 2 ** 32
    free, _ = torch.cuda.mem_get_info()
    if free < K * 8 + (8 << 30):
        pytest.skip("not enough device memory for the 34 GB pair list")
    p = ddm.match_pairs(*g, capacity=K)
    assert p.shape[0] == K
    u = p[:, 1].view(n, n)
    first = u[:, 0]
    assert bool((u == first[:, None]).all())
    assert bool((torch.sort(first.long()).values == torch.arange(n, device=u.device)).all())
    for r in (0, 1, n // 2, n - 2, n - 1):
        row = p[r * n:(r + 1) * n, 0].long()
        assert bool((torch.sort(row).values == torch.arange(n, device=row.device)).all())


def test_deterministic_output():
    w = wl.make("c2", scale=0.1)
    g = gpu_args(w)
    a = ddm.match_pairs(*g)
    b = ddm.match_pairs(*g)
    assert torch.equal(a, b)


def test_sort_pairs_canonical(orc):
    w = wl.make("c2", scale=0.2)
    g = gpu_args(w)
    p = ddm.match_pairs(*g, sort=True)
    got = raw_words(p)
    assert np.all(np.diff(got.astype(np.int64)) > 0)
    assert np.array_equal(got, orc.sbm_seq(w.sub_lo, w.sub_hi, w.upd_lo, w.upd_hi))


# ------------------------------------------------------------ index / shards (multi-GPU analogue)

@pytest.mark.parametrize("d", [1, 3])
def test_indexed_shards_equal_single(orc, d):
    """G-invariance: partition updates by coordinate slab, match each slab
    against the broadcastable subscription index with global ids, and the
    concatenation equals the single-call list; d = 3 runs the
    tiled filter against the index's boxes and other dimensions."""
    w = wl.make("c2", scale=0.2) if d == 1 else wl.make("c4", scale=0.01)
    g = gpu_args(w)
    ref = words_of(ddm.match_pairs(*g))
    assert np.array_equal(ref, orc.sbm_seq(w.sub_lo, w.sub_hi, w.upd_lo, w.upd_hi))
    idx = ddm.sub_index_build(g[0], g[1])
    for G in (1, 2, 3, 8):
        cuts = np.quantile(w.sub_lo[0], np.arange(1, G) / G)
        slab = np.searchsorted(cuts, w.upd_lo[0], side="right")
        parts = []
        total = 0
        for r in range(G):
            ids = np.nonzero(slab == r)[0]
            ul, uh = cuda(w.upd_lo[:, ids]), cuda(w.upd_hi[:, ids])
            idt = torch.from_numpy(ids.astype(np.int32)).cuda()
            p = ddm.match_pairs_indexed(idx, w.n, ul, uh, upd_ids=idt)
            if d == 1:  # the walk-form counts over the index's prefix maxima give the same list
                pw = ddm.match_pairs_indexed(idx, w.n, ul, uh, upd_ids=idt, flags=ddm.DDM_COUNT_WALK)
                assert torch.equal(p, pw)
            total += ddm.match_count_indexed(idx, w.n, ul, uh)
            parts.append(words_of(p))
        got = np.sort(np.concatenate(parts))
        assert total == ref.size
        assert np.array_equal(got, ref), G


def test_slab_device_ops_equal_numpy_rules(orc):
    """ddm_slab_sample / _cuts / _pack / _unpack (the slab mode's on-device
    partition) against tests/dist_workers.NumpyOps, which states the rules of
    include/ddm.h in numpy: identical samples, cut points, per-slab reach,
    send counts and rows (byte for byte), round trip through unpack; invalid
    regions (NaN, inverted) are reported even when they reach no slab."""
    from paper_1703_06680_b200 import dist as ddist
    from tests.dist_workers import NumpyOps
    for d, G in ((1, 3), (2, 5), (3, 1)):
        w = wl.uniform(3000, 3300, 1e4, 80.0, d, seed=50 + d)
        sl, sh = w.sub_lo.copy(), w.sub_hi.copy()
        sl[0, :5], sh[0, :5] = -3.0, 3e4
        D, N = ddist.DeviceOps(d, "cuda"), NumpyOps(d)
        T = lambda a: torch.from_numpy(np.ascontiguousarray(a))  # noqa: E731
        samp = D.sample(cuda(w.upd_lo[0]), 700)
        assert np.array_equal(samp.cpu().numpy(), N.sample(T(w.upd_lo[0]), 700).numpy())
        big = torch.cat([samp, cuda(np.array([np.nan] * 9)), cuda(w.sub_lo[0][:300])])
        cuts = D.cuts(big, G)
        assert np.array_equal(cuts.cpu().numpy(), N.cuts_np(big.cpu().numpy(), G))
        ur, uc, reach = D.pack(1, cuda(w.upd_lo), cuda(w.upd_hi), 1000, cuts, G)
        nur, nuc, nreach = N.pack(1, T(w.upd_lo), T(w.upd_hi), 1000, cuts.cpu(), G)
        assert uc == nuc and np.array_equal(reach.cpu().numpy(), nreach.numpy())
        assert np.array_equal(ur.cpu().numpy().view(np.uint64), nur.numpy().view(np.uint64))
        sr, sc, _ = D.pack(0, cuda(sl), cuda(sh), 7, cuts, G, reach=reach)
        nsr, nsc, _ = N.pack(0, T(sl), T(sh), 7, cuts.cpu(), G, reach=nreach)
        assert sc == nsc and np.array_equal(sr.cpu().numpy().view(np.uint64), nsr.numpy().view(np.uint64))
        lo, hi, ids = D.unpack(sr)
        nlo, nhi, nids = N.unpack(nsr)
        assert np.array_equal(lo.cpu().numpy(), nlo.numpy()) and np.array_equal(hi.cpu().numpy(), nhi.numpy())
        assert np.array_equal(ids.cpu().numpy().astype(np.int64), nids.numpy())
    bad = w.sub_hi.copy()
    bad[0, 17] = np.nan
    with pytest.raises(ddm.DDMError) as e:
        D.pack(0, cuda(w.sub_lo), cuda(bad), 0, cuts, 1, reach=reach[:1])
    assert e.value.status == 2
    bad = w.sub_hi.copy()
    bad[-1, 3] = w.sub_lo[-1, 3] - 1.0
    with pytest.raises(ddm.DDMError) as e:
        D.pack(0, cuda(w.sub_lo), cuda(bad), 0, cuts, 1, reach=reach[:1])
    assert e.value.status == 3


@pytest.mark.parametrize("world", [2, 3])
def test_slab_matcher_processes_one_gpu(orc, tmp_path, world):
    """dist.SlabMatcher.step with the libddm ops, `world` processes sharing
    cuda:0 over gloo: on-device cuts, partition with halos, all_to_all
    exchange, mapped match, K all-reduce.  The union of the rank lists equals
    the oracle list, each pair once; every rank's K is the total."""
    import torch.multiprocessing as mp
    from tests import dist_workers as dw
    mp.spawn(dw.slab_worker_gpu, args=(world, dw.free_port(), str(tmp_path), "gpu"), nprocs=world, join=True)
    w = dw.instance("gpu")
    ref = orc.sbm_seq(w.sub_lo, w.sub_hi, w.upd_lo, w.upd_hi)
    parts = [np.load(tmp_path / f"g_pairs_{r}.npy") for r in range(world)]
    got = np.concatenate(parts)
    assert got.size == ref.size and np.array_equal(np.sort(got), ref)
    assert all(int(np.load(tmp_path / f"g_k_{r}.npy")[0]) == ref.size for r in range(world))
    assert all(p.size for p in parts)


def test_broadcast_matcher_processes_one_gpu(orc, tmp_path):
    """dist.ShardedMatcher.step (index built on rank 0, broadcast, indexed
    match per update block, K all-reduce) with two processes on cuda:0."""
    import torch.multiprocessing as mp
    from tests import dist_workers as dw
    mp.spawn(dw.broadcast_worker_gpu, args=(2, dw.free_port(), str(tmp_path), "gpu"), nprocs=2, join=True)
    w = dw.instance("gpu")
    ref = orc.sbm_seq(w.sub_lo, w.sub_hi, w.upd_lo, w.upd_hi)
    got = np.sort(np.concatenate([np.load(tmp_path / f"gb_pairs_{r}.npy") for r in range(2)]))
    assert np.array_equal(got, ref)
    assert all(int(np.load(tmp_path / f"gb_k_{r}.npy")[0]) == ref.size for r in range(2))


def _check_chunk_sets(orc, sl, sh, ul, uh):
    """GPU chunk-start sets A_t (a6, the emit_chunk_kernel walk) equal the
    oracle's sequential-sweep SubSet snapshot before each tile's first update
    (oracle.states_at), member for member, in Slo order."""
    sl, sh, ul, uh = arrays(sl, sh, ul, uh)
    first, off, ids = ddm.chunk_start_sets(cuda(sl), cuda(sh), cuda(ul), cuda(uh))
    first, off, ids = first.cpu().numpy(), off.cpu().numpy(), ids.cpu().numpy().astype(np.int64)
    # the tiles start at every DDM_CHUNK_ROWS-th update in (lower bound, id) order
    order = np.lexsort((np.arange(ul.shape[1]), ul[0]))
    assert np.array_equal(first, order[::ddm.DDM_CHUNK_ROWS])
    ref = orc.states_at(sl, sh, ul, uh, first)
    for t in range(first.size):
        got = ids[off[t]:off[t + 1]]
        assert np.array_equal(np.sort(got), ref[t].astype(np.int64)), f"tile {t}"
        # Slo order: (lower bound, id) ascending
        assert np.all(np.lexsort((got, sl[0, got])) == np.arange(got.size))
    return int(off[-1])


def test_chunk_start_sets_equal_sweep_states(orc):
    rng = np.random.default_rng(71)
    total = 0
    # dense overlaps (c2 recipe scaled), ties on a grid, long intervals
    w = wl.uniform(60_000, 50_000, 1e5, wl.side_length(110_000, 1e5, 100.0, 1), 1, seed=71)
    total += _check_chunk_sets(orc, w.sub_lo, w.sub_hi, w.upd_lo, w.upd_hi)
    sl = np.floor(rng.uniform(0, 3000, 20_000))
    ul = np.floor(rng.uniform(0, 3000, 30_000))
    total += _check_chunk_sets(orc, sl, sl + np.floor(rng.uniform(0, 40, sl.size)), ul, ul + 3.0)
    sl = rng.uniform(0, 1e6, 40_000)
    sh = sl + 5.0
    sh[:30] = 1e6 + 1.0  # spans everything: members of every A_t, reached past block-max skips
    ul = rng.uniform(0, 1e6, 20_000)
    total += _check_chunk_sets(orc, sl, sh, ul, ul + 5.0)
    assert total > 10_000


def test_chunk_start_sets_c2_full(orc):
    w = wl.make("c2")
    assert _check_chunk_sets(orc, w.sub_lo, w.sub_hi, w.upd_lo, w.upd_hi) > 50_000


def test_msd_overflow_falls_back_to_lsb(orc):
    """A bucket larger than shared memory (here: 12000 equal lower bounds plus a
    spread) makes the MSD sort hand over to the LSB sort: same result."""
    rng = np.random.default_rng(9)
    lo = np.concatenate([np.full(12000, 5.0), rng.uniform(0, 100, 3000)])
    hi = lo + rng.uniform(0, 2, lo.size)
    ul = rng.uniform(0, 100, 5000)
    uh = ul + 1.0
    ref = orc.sbm_seq(lo[None], hi[None], ul[None], uh[None])
    check_against(orc, lo, hi, ul, uh, flags=(0, ddm.DDM_SORT_LSB), ref=ref)
    # and the same on the update side
    ref2 = orc.sbm_seq(ul[None], uh[None], lo[None], hi[None])
    check_against(orc, ul, uh, lo, hi, flags=(0, ddm.DDM_SORT_LSB), ref=ref2)
    # d = 2 with few updates (the per-row filter, which runs before the host
    # learns of the overflow and must then do nothing), count-only first
    lo2 = np.stack([lo, rng.uniform(0, 100, lo.size)])
    hi2 = lo2 + rng.uniform(0, 2, lo2.shape)
    ul2 = np.stack([ul, rng.uniform(0, 100, ul.size)])
    uh2 = ul2 + 1.0
    for _ in range(3):
        check_against(orc, lo2, hi2, ul2, uh2, flags=(0,), ref=orc.sbm_seq(lo2, hi2, ul2, uh2))
        check_against(orc, ul2, uh2, lo2, hi2, flags=(0,), ref=orc.sbm_seq(ul2, uh2, lo2, hi2))


def test_packed_records_with_unfit_deltas(orc):
    """Sorts of >= 2^22 records carry 16-byte packed records (id | upper-key
    delta << 32); an upper key whose delta from the lower key needs more than
    32 bits (long intervals, small magnitudes) is re-read from the input.  Half
    the subscriptions and updates here take that path: the pair count equals
    the oracle's rank identity, every pair overlaps, none repeats, and the list
    equals the (unpacked) LSB path's."""
    rng = np.random.default_rng(61)
    n = m = 4_300_000
    sl = rng.uniform(0.0, 1e6, n)
    ul = rng.uniform(0.0, 1e6, m)
    sh = sl + np.where(rng.random(n) < 0.5, 1e-3, 1.0)     # 1.0 at ~5e5: delta > 2^32 key units
    uh = ul + np.where(rng.random(m) < 0.5, 1e-3, 1.0)
    g = [cuda(x[None]) for x in (sl, sh, ul, uh)]
    p = ddm.match_pairs(*g)
    K = p.shape[0]
    assert K == orc.rank_count(sl[None], sh[None], ul[None], uh[None]) and K > 100_000
    s_, u_ = p[:, 0].long(), p[:, 1].long()
    assert bool(((g[0][0][s_] <= g[3][0][u_]) & (g[2][0][u_] <= g[1][0][s_])).all())
    wds = torch.sort((u_ << 32) | s_).values
    assert bool((wds[1:] > wds[:-1]).all())
    q = ddm.match_pairs(*g, flags=ddm.DDM_SORT_LSB)
    assert torch.equal(p, q)  # same rows, same order: the packing changes no byte


def test_big_local_sort_range(orc):
    """7.5e7 subscriptions: with ~768 records per bucket the MSD sort would
    need 17 bucket bits (3 multisplit passes); the big local sort (groups of up
    to 16384 records per SM) takes ~6000 per bucket, 14 bits, 2 passes.  K
    equals the oracle's rank identity; the list is valid, unique, and equal to
    the LSB path's."""
    rng = np.random.default_rng(62)
    n, m = 75_000_000, 1_000_000
    sl = rng.uniform(0.0, 1e8, n)
    ul = rng.uniform(0.0, 1e8, m)
    sh, uh = sl + 1.5, ul + 1.5
    g = [cuda(x[None]) for x in (sl, sh, ul, uh)]
    p = ddm.match_pairs(*g)
    K = p.shape[0]
    assert K == orc.rank_count(sl[None], sh[None], ul[None], uh[None]) and K > 1_000_000
    s_, u_ = p[:, 0].long(), p[:, 1].long()
    assert bool(((g[0][0][s_] <= g[3][0][u_]) & (g[2][0][u_] <= g[1][0][s_])).all())
    wds = torch.sort((u_ << 32) | s_).values
    assert bool((wds[1:] > wds[:-1]).all())
    del s_, u_, wds
    q = ddm.match_pairs(*g, flags=ddm.DDM_SORT_LSB)
    assert torch.equal(p, q)


@pytest.mark.parametrize("n", [1, 700, 769, 5000, 70_000, 300_000])
def test_msd_sizes(orc, n):
    """Bucket-bit choices from 1 to ~9 bits, ragged spans and tails."""
    w = wl.uniform(n, max(1, n // 2), 1e5, 3.0, 1, seed=n)
    check_against(orc, w.sub_lo, w.sub_hi, w.upd_lo, w.upd_hi, flags=(0, ddm.DDM_SORT_LSB))


def test_msd_negative_and_wide_ranges(orc):
    rng = np.random.default_rng(2)
    lo = np.concatenate([rng.uniform(-1e300, 1e300, 2000), rng.normal(0, 1, 20000), [-0.0, 0.0] * 50])
    hi = lo + np.abs(rng.normal(0, 0.5, lo.size))
    ul = rng.normal(0, 1, 8000)
    uh = ul + 0.1
    check_against(orc, lo, hi, ul, uh, flags=(0, ddm.DDM_SORT_LSB))


# ------------------------------------------------------------ event-order variant

@pytest.mark.parametrize("S,U,K", [
    ([[0.0, 1.0]], [[1.0, 2.0]], 1),     # touching endpoints (closed, R1)
    ([[0.0, 0.0]], [[0.0, 0.0]], 1),     # points
    ([[-1.0, -0.0]], [[0.0, 1.0]], 1),   # -0.0 == +0.0 (R3)
    ([[0.0, 1.0]], [[1.5, 2.0]], 0),
])
def test_events_small_cases(orc, S, U, K):
    sl, sh = np.array([[s[0] for s in S]]), np.array([[s[1] for s in S]])
    ul, uh = np.array([[u[0] for u in U]]), np.array([[u[1] for u in U]])
    p = ddm.match_pairs_events(*[cuda(x) for x in (sl, sh, ul, uh)])
    assert p.shape[0] == K
    assert np.array_equal(words_of(p), orc.bf_pairs(sl, sh, ul, uh))


def test_events_fuzz_against_oracle(orc):
    """Alg. 5 + 6 on the GPU against brute force: ties, duplicates, points,
    long intervals crossing many segments (initial sets from the backward
    walk, chunked past 2048 members), d = 1..3, sizes across several
    segments with ragged tails, and one empty side."""
    rng = np.random.default_rng(77)
    for case in range(16):
        d = int(rng.integers(1, 4))
        n, m = (int(x) for x in rng.integers(1, 7000, 2))
        def side(cnt):
            kind = rng.integers(0, 3)
            if kind == 0:
                lo = rng.uniform(0, 1e4, (d, cnt))
            elif kind == 1:
                lo = rng.integers(0, 30, (d, cnt)).astype(np.float64)
            else:
                lo = rng.normal(5e3, 50.0, (d, cnt))
            ln = np.abs(rng.normal(0, 20.0, (d, cnt)))
            ln[rng.random((d, cnt)) < 0.03] = 1e5   # long intervals
            ln[rng.random((d, cnt)) < 0.05] = 0.0   # points
            return lo, lo + ln
        sl, sh = side(n)
        ul, uh = side(m)
        ref = orc.bf_pairs(sl, sh, ul, uh)
        p = ddm.match_pairs_events(*[cuda(x) for x in (sl, sh, ul, uh)])
        assert np.array_equal(words_of(p), ref), f"case {case} d={d} n={n} m={m}"
    e = np.zeros((1, 0))
    x = rng.uniform(0, 1, (1, 50))
    assert ddm.match_pairs_events(cuda(e), cuda(e), cuda(x), cuda(x + 1)).shape[0] == 0


def test_events_dense_initial_sets(orc):
    """Every region spans the whole domain: each segment's initial sets hold
    thousands of members (several 2048-member chunks)."""
    rng = np.random.default_rng(5)
    n, m = 6000, 3000
    sl = rng.uniform(0, 1, (1, n)); sh = sl + 10.0
    ul = rng.uniform(0, 1, (1, m)); uh = ul + 10.0
    p = ddm.match_pairs_events(*[cuda(x) for x in (sl, sh, ul, uh)])
    assert p.shape[0] == n * m
    assert np.array_equal(words_of(p), orc.bf_pairs(sl, sh, ul, uh))


def test_events_equal_main_path_c2_c4(orc):
    """Full-size c2 and a scaled c4: the event-order list, canonicalised,
    equals the main path's canonicalised list (two independent GPU
    algorithms: rank differences + tile sweep vs. Alg. 5 + 6)."""
    for cfg, scale in (("c2", 1.0), ("c4", 0.02)):
        w = wl.make(cfg, scale)
        g = gpu_args(w)
        a = ddm.match_pairs(*g, sort=True)
        b = ddm.match_pairs_events(*g)
        assert torch.equal(a, b), cfg


def test_events_validation():
    x = cuda(np.array([[0.0, 1.0]]))
    bad = cuda(np.array([[np.nan, 1.0]]))
    with pytest.raises(ddm.DDMError) as e:
        ddm.match_pairs_events(bad, x, x, x + 1)
    assert e.value.status == 2
    with pytest.raises(ddm.DDMError) as e:
        ddm.match_pairs_events(x + 5, x, x, x + 1)
    assert e.value.status == 3


def test_events_c3_full_equals_main_path():
    """c3 at full size (1e8 regions, 2e8 endpoints, ~1e5 segments): the
    event-order variant's canonical list equals the main path's."""
    w = wl.make("c3")
    g = gpu_args(w)
    a = ddm.match_pairs(*g, sort=True)
    b = ddm.match_pairs_events(*g)
    assert a.shape == b.shape and torch.equal(a, b)


# ------------------------------------------------------------ dynamic DDM

def _index_zeroed(L, sl, sh):
    import ctypes
    r, keep = ddm.regions(sl, sh)
    idx = torch.zeros(L.ddm_sub_index_bytes(r.d, r.n_sub), dtype=torch.uint8, device="cuda")
    ws = torch.empty(L.ddm_index_build_workspace_bytes(r.d, r.n_sub), dtype=torch.uint8, device="cuda")
    assert L.ddm_sub_index_build(ctypes.byref(r), idx.data_ptr(), idx.numel(), ws.data_ptr(), ws.numel(),
                                 torch.cuda.current_stream().cuda_stream) == 0
    return idx


@pytest.mark.parametrize("d,n,k", [(1, 1, 1), (1, 5000, 1), (1, 20_000, 700), (1, 20_000, 20_000),
                                   (2, 9000, 400), (3, 4097, 4097)])
def test_index_update_equals_rebuild(orc, d, n, k):
    """Moving / resizing k subscriptions by merge gives the byte-identical
    index of a rebuild on the modified set (ties, duplicates, long intervals,
    moves onto other entries' exact coordinates), and matches through it
    equal brute force."""
    L = ddm.load()
    rng = np.random.default_rng(n + k + d)
    sl = rng.integers(0, 300, (d, n)).astype(np.float64)
    sh = sl + rng.integers(0, 5, (d, n))
    sh[:, rng.random(n) < 0.02] += 1e4
    ids = np.sort(rng.choice(n, k, replace=False)).astype(np.int32)
    nl = rng.integers(0, 300, (d, k)).astype(np.float64)
    nh = nl + rng.integers(0, 5, (d, k))
    copy = rng.random(k) < 0.3  # some moves land exactly on other entries' coordinates
    src = rng.integers(0, n, k)
    nl[:, copy], nh[:, copy] = sl[:, src[copy]], sh[:, src[copy]]
    idx = _index_zeroed(L, cuda(sl), cuda(sh))
    out = torch.zeros_like(idx)
    tid = torch.from_numpy(ids).cuda()
    ddm.sub_index_update(idx, n, tid, cuda(nl), cuda(nh), out=out)  # ping-pong
    sl2, sh2 = sl.copy(), sh.copy()
    sl2[:, ids], sh2[:, ids] = nl, nh
    ref_idx = _index_zeroed(L, cuda(sl2), cuda(sh2))
    assert torch.equal(out, ref_idx)
    ddm.sub_index_update(idx, n, tid, cuda(nl), cuda(nh))  # in place
    assert torch.equal(idx, ref_idx)
    m = 3000
    ul = rng.integers(0, 300, (d, m)).astype(np.float64)
    uh = ul + rng.integers(0, 5, (d, m))
    p = ddm.match_pairs_indexed(idx, n, cuda(ul), cuda(uh))
    assert np.array_equal(words_of(p), orc.bf_pairs(sl2, sh2, ul, uh))


def test_index_update_errors_leave_index_untouched():
    L = ddm.load()
    sl = cuda(np.arange(10.0)[None]); sh = sl + 1
    idx = _index_zeroed(L, sl, sh)
    before = idx.clone()
    for ids, nl, nh, st in (([3, 3], [[0.0, 1.0]], [[1.0, 2.0]], 1),      # not strictly increasing
                            ([2, 10], [[0.0, 1.0]], [[1.0, 2.0]], 1),     # out of range
                            ([1, 2], [[np.nan, 1.0]], [[1.0, 2.0]], 2),   # non-finite
                            ([1, 2], [[5.0, 1.0]], [[1.0, 2.0]], 3)):     # inverted
        with pytest.raises(ddm.DDMError) as e:
            ddm.sub_index_update(idx, 10, torch.tensor(ids, dtype=torch.int32), cuda(np.array(nl)), cuda(np.array(nh)))
        assert e.value.status == st
        assert torch.equal(idx, before)


def test_msd_sample_unbiased_on_sorted_input(orc):
    """The bucket map's sample takes short runs spread over the whole array,
    so already-sorted (or reverse-sorted) inputs get balanced buckets and stay
    on the MSD path (no LSB fallback launches), with exact results."""
    rng = np.random.default_rng(12)
    n = 1_000_000
    lo = np.sort(rng.uniform(-1.0, 1.0, n))
    sl, sh = lo[None], (lo + 1e-7)[None]
    ul, uh = lo[::-1].copy()[None], (lo[::-1] + 1e-7)[None]
    g = [cuda(x) for x in (sl, sh, ul, uh)]
    ddm.profile_enable(True)
    p = ddm.match_pairs(*g)
    torch.cuda.synchronize()
    prof = ddm.profile_read()
    ddm.profile_enable(False)
    assert not any(k.startswith("onesweep") for k in prof), sorted(prof)
    assert p.shape[0] == orc.rank_count(sl, sh, ul, uh)


def test_few_dense_rows_split_emission(orc):
    """Few updates with very many partners each (few row tiles, K > 4m): the
    (row, segment) split emission, including rows longer than 64 segments and
    long-interval stab parts, is byte-identical to every other path and exact
    against brute force."""
    rng = np.random.default_rng(31)
    n, m = 300_000, 40
    sl = rng.uniform(0, 1e6, n)[None]
    sh = sl + rng.exponential(20.0, n)[None]
    sh[0, rng.choice(n, 30, replace=False)] += 5e5  # long subscriptions in the stab parts
    ul = rng.uniform(0, 6e5, m)[None]
    uh = ul + rng.uniform(1e3, 4e5, m)[None]        # up to ~1.2e5 range pairs per row
    check_against(orc, sl, sh, ul, uh, flags=EMIT_FLAGS, ref=orc.bf_pairs(sl, sh, ul, uh))
