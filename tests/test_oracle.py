"""Pins for the CPU oracle (oracle/) against what the paper and mathematics fix.

Every oracle function is pinned by something other than itself:
  * SPEC/PAPER worked examples (intersect_1d examples S:55-58, Fig. 1
    via tests/golden/fig1_instance.json, nested S:178, identical S:129,
    empty S:128, touching/point-interval ties S:56);
  * a set-theoretic brute force on tiny integer grids (does a sampled point lie
    in both closed boxes?) -- independent of the Alg. 1 formula;
  * agreement of independent implementations (Alg. 2 vs Alg. 4 vs Alg. 5+6 vs
    the literal per-dimension intersection vs the App. A rank identity);
  * the boundary-state oracle for Alg. 6;
  * the generator's closed-form E[K] and the paper's l formula.
"""
import itertools
import json
import os

import numpy as np
import pytest

from paper_1703_06680_b200 import workload as wl

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ------------------------------------------------------------ helpers

def setdef_pairs(S, U):
    """Set-theoretic definition on a half-integer grid: (i, j) is a pair iff
    some sampled point lies in both closed boxes.  Boxes have integer (or
    half-integer) corners, so sampling at step 1/2 is exact."""
    out = []
    for j, u in enumerate(U):
        for i, s in enumerate(S):
            axes = []
            for (slo, shi), (ulo, uhi) in zip(s, u):
                ps = {x / 2 for x in range(int(2 * slo), int(2 * shi) + 1)}
                pu = {x / 2 for x in range(int(2 * ulo), int(2 * uhi) + 1)}
                axes.append(sorted(ps & pu))
            if all(axes) and any(True for _ in itertools.product(*axes)):
                out.append((j << 32) | i)
    return np.array(sorted(out), dtype=np.uint64)


def to_arrays(S, U, d):
    n, m = len(S), len(U)
    sl = np.array([[S[i][k][0] for i in range(n)] for k in range(d)], dtype=np.float64).reshape(d, n)
    sh = np.array([[S[i][k][1] for i in range(n)] for k in range(d)], dtype=np.float64).reshape(d, n)
    ul = np.array([[U[j][k][0] for j in range(m)] for k in range(d)], dtype=np.float64).reshape(d, m)
    uh = np.array([[U[j][k][1] for j in range(m)] for k in range(d)], dtype=np.float64).reshape(d, m)
    return sl, sh, ul, uh


def rand_int_boxes(rng, count, d, hi=4):
    out = []
    for _ in range(count):
        box = []
        for _ in range(d):
            a, b = sorted(rng.integers(0, hi + 1, 2))
            box.append((float(a), float(b)))
        out.append(box)
    return out


def all_1d_methods(orc, sl, sh, ul, uh):
    """Every 1-D oracle path, canonical u64 words."""
    res = {"bf": orc.bf_pairs(sl, sh, ul, uh), "sbm": orc.sbm_seq(sl, sh, ul, uh)}
    for P in (1, 2, 3, 4, 7, 8):
        res[f"par{P}"] = orc.par_sbm(sl, sh, ul, uh, P=P)
    return res


def words(pairs_1based):
    return np.array(sorted(((u - 1) << 32) | (s - 1) for s, u in pairs_1based), dtype=np.uint64)


# ------------------------------------------------------------ worked examples

@pytest.mark.parametrize("x,y,expect", [
    ((0, 1), (2, 3), False),   # S:55 disjoint
    ((5, 10), (10, 12), True),  # S:56 touching (closed, Alg. 1 uses <=)
    ((3, 3), (1, 5), True),     # S:57 point interval inside
    ((1, 4), (2, 3), True),     # S:58 containment
])
def test_intersect_1d_spec_examples(orc, x, y, expect):
    assert orc.intersect_1d(*x, *y) is expect
    assert orc.intersect_1d(*y, *x) is expect  # symmetry


def test_fig1_instance_four_pairs(orc):
    g = json.load(open(os.path.join(GOLDEN, "fig1_instance.json")))
    S, U, d = g["sub"], g["upd"], g["d"]
    sl, sh, ul, uh = to_arrays(S, U, d)
    expect = words(g["expected_pairs_1based"])
    # the constructed coordinates realise the paper's topology (set definition)
    assert np.array_equal(setdef_pairs(S, U), expect)
    assert np.array_equal(orc.bf_pairs(sl, sh, ul, uh), expect)
    assert np.array_equal(orc.sbm_seq(sl, sh, ul, uh), expect)
    assert np.array_equal(orc.sbm_dd_literal(sl, sh, ul, uh), expect)
    assert orc.bf_count(sl, sh, ul, uh) == 4 and orc.sbm_count(sl, sh, ul, uh) == 4
    # dimension 0 alone also yields (S2, U1): the d>1 filter is what removes it
    s2u1 = words([g["dim0_only_extra_pair_1based"]])
    d0 = orc.sbm_seq(sl[:1], sh[:1], ul[:1], uh[:1])
    assert d0.size == 5 and s2u1[0] in d0
    for P in (1, 2, 4):  # SPEC S:287 Fig. 1 topology for every P (1-D projection)
        assert np.array_equal(orc.par_sbm(sl[:1], sh[:1], ul[:1], uh[:1], P=P), d0)


@pytest.mark.parametrize("S,U,K", [
    ([[(0, 10)]], [[(2, 3)]], 1),          # S:178 nested: reported once
    ([[(1, 2)]], [[(1, 2)]], 1),           # S:129 identical extents
    ([[(5, 10)]], [[(10, 12)]], 1),        # S:56 touching
    ([[(5, 5)]], [[(5, 9)]], 1),           # S:77 point interval, tie at 5
    ([[(0, 1)]], [[(2, 3)]], 0),           # S:55 disjoint
    ([[(-1, -0.0)]], [[(0.0, 1)]], 1),     # -0.0 == +0.0 (reading R3)
    ([[(3, 3)]], [[(3, 3)]], 1),           # two degenerate points at the same place
])
def test_small_cases(orc, S, U, K):
    sl, sh, ul, uh = to_arrays(S, U, 1)
    for name, got in all_1d_methods(orc, sl, sh, ul, uh).items():
        assert got.size == K, name
    assert orc.rank_count(sl, sh, ul, uh) == K


def test_empty_inputs(orc):
    e = np.zeros((1, 0))
    one = np.array([[0.0]]), np.array([[1.0]])
    assert orc.bf_count(e, e, *one) == 0
    assert orc.sbm_count(*one, e, e) == 0
    assert orc.par_sbm(e, e, e, e, P=4, count_only=True) == 0
    assert orc.rank_count(*one, e, e) == 0


# ------------------------------------------------------------ exhaustive / random tiny grids

INTERVALS = [(float(a), float(b)) for a in range(5) for b in range(a, 5)]


def test_exhaustive_single_pairs(orc):
    """All 15 x 15 closed integer intervals in {0..4}: oracle == set definition."""
    S = [[iv] for iv in INTERVALS]
    U = [[iv] for iv in INTERVALS]
    sl, sh, ul, uh = to_arrays(S, U, 1)
    expect = setdef_pairs(S, U)
    for name, got in all_1d_methods(orc, sl, sh, ul, uh).items():
        assert np.array_equal(got, expect), name
    assert orc.rank_count(sl, sh, ul, uh) == expect.size


def test_random_tie_storms_1d(orc):
    rng = np.random.default_rng(1234)
    for _ in range(300):
        n, m = rng.integers(0, 13, 2)
        S, U = rand_int_boxes(rng, n, 1), rand_int_boxes(rng, m, 1)
        sl, sh, ul, uh = to_arrays(S, U, 1)
        expect = setdef_pairs(S, U)
        for name, got in all_1d_methods(orc, sl, sh, ul, uh).items():
            assert np.array_equal(got, expect), name
        assert orc.rank_count(sl, sh, ul, uh) == expect.size
        assert orc.sbm_count(sl, sh, ul, uh) == expect.size
        assert orc.par_sbm(sl, sh, ul, uh, P=3, count_only=True) == expect.size


@pytest.mark.parametrize("d", [2, 3])
def test_random_tie_storms_dd(orc, d):
    rng = np.random.default_rng(99 + d)
    for _ in range(150):
        n, m = rng.integers(0, 9, 2)
        S, U = rand_int_boxes(rng, n, d, hi=3), rand_int_boxes(rng, m, d, hi=3)
        sl, sh, ul, uh = to_arrays(S, U, d)
        expect = setdef_pairs(S, U)
        assert np.array_equal(orc.bf_pairs(sl, sh, ul, uh), expect)
        assert np.array_equal(orc.sbm_seq(sl, sh, ul, uh), expect)
        assert np.array_equal(orc.sbm_dd_literal(sl, sh, ul, uh), expect)
        assert orc.sbm_count(sl, sh, ul, uh) == expect.size


@pytest.mark.parametrize("alpha", [0.01, 1.0, 100.0])
def test_random_float_agreement(orc, alpha):
    """SPEC S:448 (N=1e3..1e4, alpha in {0.01,1,100}): all paths agree with
    brute force; the list is duplicate-free and every pair satisfies Alg. 1."""
    N = 4000
    w = wl.uniform(N // 2, N // 2, 1e6, wl.side_length(N, 1e6, alpha, 1), 1, seed=int(alpha * 100))
    a = (w.sub_lo, w.sub_hi, w.upd_lo, w.upd_hi)
    res = all_1d_methods(orc, *a)
    ref = res["bf"]
    for name, got in res.items():
        assert np.array_equal(got, ref), name
    assert orc.rank_count(*a) == ref.size
    assert np.all(np.diff(ref.astype(np.int64)) > 0) if ref.size > 1 else True
    sub = (ref & np.uint64(0xFFFFFFFF)).astype(np.int64)
    upd = (ref >> np.uint64(32)).astype(np.int64)
    assert np.all(w.sub_lo[0, sub] <= w.upd_hi[0, upd]) and np.all(w.upd_lo[0, upd] <= w.sub_hi[0, sub])


def test_duplicates_and_asymmetric(orc):
    rng = np.random.default_rng(5)
    lo = rng.uniform(0, 100, 50)
    sl = np.concatenate([lo, lo])[None]  # every region duplicated
    sh = sl + 3.0
    ul = rng.uniform(0, 100, 1000)[None]
    uh = ul + 1.0
    ref = orc.bf_pairs(sl, sh, ul, uh)
    assert ref.size % 2 == 0 and ref.size > 0
    assert np.array_equal(orc.sbm_seq(sl, sh, ul, uh), ref)
    assert np.array_equal(orc.par_sbm(sl, sh, ul, uh, P=5), ref)
    # asymmetric n=1
    assert np.array_equal(orc.sbm_seq(sl[:, :1], sh[:, :1], ul, uh), orc.bf_pairs(sl[:, :1], sh[:, :1], ul, uh))
    assert np.array_equal(orc.par_sbm(ul, uh, sl[:, :1], sh[:, :1], P=4), orc.bf_pairs(ul, uh, sl[:, :1], sh[:, :1]))


def test_bf_rows_matches_full(orc):
    w = wl.uniform(700, 900, 1e4, 30.0, 1, seed=7)
    a = (w.sub_lo, w.sub_hi, w.upd_lo, w.upd_hi)
    full = orc.bf_pairs(*a)
    rows = np.array([0, 5, 17, 899, 450])
    got, counts = orc.bf_rows(*a, rows)
    upd = full >> np.uint64(32)
    expect = np.concatenate([full[upd == r] for r in rows])
    assert np.array_equal(got, expect)
    assert counts.tolist() == [int((upd == r).sum()) for r in rows]


# ------------------------------------------------------------ Alg. 6 boundary states

@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_alg6_states_equal_sequential_snapshots(orc, P):
    """combine_deltas output == the sequential sweep's snapshot at
    every segment boundary (the equivalence condition of P:549-557)."""
    rng = np.random.default_rng(P)
    for trial in range(25):
        if trial % 2:
            S, U = rand_int_boxes(rng, rng.integers(0, 20), 1), rand_int_boxes(rng, rng.integers(0, 20), 1)
            a = to_arrays(S, U, 1)
        else:
            w = wl.uniform(int(rng.integers(1, 300)), int(rng.integers(1, 300)), 1e3, 25.0, 1, seed=trial)
            a = (w.sub_lo, w.sub_hi, w.upd_lo, w.upd_hi)
        seq_s, seq_u = orc.boundary_states(*a, P)
        par_s, par_u = orc.par_states(*a, P)
        assert len(seq_s) == P and not seq_s[0].size and not seq_u[0].size  # SubSet[0] = {}
        for p in range(P):
            assert np.array_equal(seq_s[p], par_s[p]), (trial, p)
            assert np.array_equal(seq_u[p], par_u[p]), (trial, p)


def test_alg6_inline_formula_index_shift_is_wrong(orc):
    """DESIGN.md reading R8: the inline recurrence of P:717-726 uses Sadd[p],
    Alg. 6 uses Sadd[p-1]; only the latter reproduces the sequential sweep.
    Demonstrated on a hand case: S0=[0,1] alone, P=2 (T = lo0 | hi0)."""
    a = to_arrays([[(0.0, 1.0)]], [], 1)
    a = (a[0], a[1], np.zeros((1, 0)), np.zeros((1, 0)))
    seq_s, _ = orc.boundary_states(*a, 2)
    par_s, _ = orc.par_states(*a, 2)
    # after T_0 = {lo(S0)} the sweep holds {S0}; Sadd[0] = {S0}, Sadd[1] = {}
    assert seq_s[1].tolist() == [0] and par_s[1].tolist() == [0]


def _endpoint_order(sl, sh, ul, uh):
    """Positions of the sorted endpoint list T by (coord, is_upper, kind, id)
    (reading R1/R2), as records (kind, is_upper, id) -- test-side only."""
    n, m = sl.shape[1], ul.shape[1]
    x = np.concatenate([sl[0], sh[0], ul[0], uh[0]])
    up = np.concatenate([np.zeros(n), np.ones(n), np.zeros(m), np.ones(m)]).astype(np.int64)
    kind = np.concatenate([np.zeros(2 * n), np.ones(2 * m)]).astype(np.int64)
    ids = np.concatenate([np.arange(n), np.arange(n), np.arange(m), np.arange(m)])
    o = np.lexsort((ids, kind, up, x))
    return kind[o], up[o], ids[o]


def test_states_at_equals_boundary_states_and_stab_definition(orc):
    """states_at (snapshot right before chosen update lower endpoints) is
    pinned two ways: (a) where a segment of the SPEC S:240-247 plan starts at
    an update lower endpoint, it equals boundary_states' SubSet[p];
    (b) it equals the stabbing-set definition {S : S.lo <= a <= S.hi} (I6 with
    lowers before uppers at ties, reading R1) evaluated by brute force."""
    rng = np.random.default_rng(91)
    checked_a = 0
    for trial in range(40):
        if trial % 2:
            S, U = rand_int_boxes(rng, rng.integers(1, 25), 1), rand_int_boxes(rng, rng.integers(1, 25), 1)
            sl, sh, ul, uh = to_arrays(S, U, 1)
        else:
            w = wl.uniform(int(rng.integers(1, 200)), int(rng.integers(1, 200)), 1e3, 40.0, 1, seed=100 + trial)
            sl, sh, ul, uh = w.sub_lo, w.sub_hi, w.upd_lo, w.upd_hi
        m = ul.shape[1]
        q = rng.permutation(m)[: max(1, m // 2)]
        got = orc.states_at(sl, sh, ul, uh, q)
        for r, j in enumerate(q):  # (b) definition
            a = ul[0, j]
            assert np.array_equal(got[r], np.nonzero((sl[0] <= a) & (a <= sh[0]))[0]), (trial, j)
        # (a) segment starts that are update lower endpoints
        kind, up, ids = _endpoint_order(sl, sh, ul, uh)
        N2 = kind.size
        for P in (2, 3, 5, 8):
            base, rem = divmod(N2, P)
            starts = np.cumsum([0] + [base + (1 if p < rem else 0) for p in range(P - 1)])
            seq_s, _ = orc.boundary_states(sl, sh, ul, uh, P)
            for p, t in enumerate(starts):
                if t < N2 and kind[t] == 1 and up[t] == 0:
                    (snap,) = orc.states_at(sl, sh, ul, uh, [ids[t]])
                    assert np.array_equal(snap, seq_s[p]), (trial, P, p)
                    checked_a += 1
    assert checked_a > 20


def test_states_at_errors(orc):
    a = to_arrays([[(0.0, 1.0)]], [[(0.5, 0.7)]], 1)
    with pytest.raises(RuntimeError):
        orc.states_at(*a, [0, 0])  # duplicate query
    with pytest.raises(RuntimeError):
        orc.states_at(*a, [1])  # out of range


def test_oracle_by_cells_equals_whole(orc):
    """tests.helpers.oracle_list_by_cells (the full-size c4 parity check
    assembles the oracle's list over 3-D cells) returns the oracle's
    whole-instance list (d = 1..3, side lengths up to the cell size, ties on
    cell edges)."""
    from tests.helpers import oracle_list_by_cells
    rng = np.random.default_rng(5)
    for d in (1, 2, 3):
        n, m = 3000, 2500
        sl = np.floor(rng.uniform(0, 200, (d, n)))
        ul = np.floor(rng.uniform(0, 200, (d, m)))
        sh = sl + np.floor(rng.uniform(0, 20, (d, n)))
        uh = ul + np.floor(rng.uniform(0, 20, (d, m)))
        w = wl.Workload("t", d, 200.0, 20.0, 0, sl, sh, ul, uh)
        got = oracle_list_by_cells(orc, w, 20.0)
        assert got.size > 1000 and np.array_equal(got, orc.sbm_seq(sl, sh, ul, uh))


# ------------------------------------------------------------ generator

def test_generator_length_formula():
    # P:907-908 l = alpha L / N; SPEC S:345-346 examples
    assert wl.side_length(10**6, 1e6, 100.0, 1) == 100.0
    assert abs(wl.side_length(10**6, 1e6, 0.01, 1) - 0.01) < 1e-15
    assert abs(wl.side_length(10**7, 1e4, 1.0, 3) - 46.4158883361278) < 1e-9


def test_generator_determinism_and_bounds():
    a = wl.make("c1")
    b = wl.make("c1")
    assert np.array_equal(a.sub_lo, b.sub_lo) and np.array_equal(a.upd_hi, b.upd_hi)
    assert a.n == a.m == 5000 and a.l == 100.0
    assert a.sub_lo.min() >= 0 and a.sub_hi.max() <= a.L
    assert np.array_equal(a.sub_hi, a.sub_lo + a.l)


def test_generator_expected_pairs_c1(orc):
    """c1 count from brute force within 5 sigma of n*m*(2r - r^2)."""
    w = wl.make("c1")
    K = orc.bf_count(w.sub_lo, w.sub_hi, w.upd_lo, w.upd_hi)
    E = wl.expected_pairs_uniform(w.n, w.m, w.L, w.l)
    assert abs(E - 5000.25) < 0.01
    assert abs(K - E) <= 5 * np.sqrt(E)


def test_generator_expected_pairs_mean_many_seeds(orc):
    """mean K over many seeds within 3 sigma of the expectation."""
    Ks = []
    for s in range(60):
        w = wl.uniform(500, 500, 1e4, 20.0, 1, seed=1000 + s)
        Ks.append(orc.rank_count(w.sub_lo, w.sub_hi, w.upd_lo, w.upd_hi))
    E = wl.expected_pairs_uniform(500, 500, 1e4, 20.0)
    assert abs(np.mean(Ks) - E) <= 3 * np.std(Ks) / np.sqrt(len(Ks)) + 1e-9


def test_clustered_generator_in_domain():
    w = wl.clustered(20000, 20000, 1e9, 0.01, seed=4)
    assert w.sub_lo.min() >= 0 and w.sub_hi.max() < 1e9
    ln = w.sub_hi - w.sub_lo
    assert ln.min() >= 0.005 - 1e-9 and ln.max() < 0.015 + 1e-9


def test_window_sample():
    w = wl.make("c2", scale=0.01)
    s = wl.window_sample(w, 0.25)
    width = np.ptp(np.concatenate([s.sub_lo[0], s.upd_lo[0]]))
    assert 0 < s.n < w.n and 0 < s.m < w.m and width < 0.25 * w.L
    c = wl.clustered(20_000, 20_000, 1e9, 0.01 * 2500, seed=4)
    assert wl.window_sample(c, 0.01).n > 0  # the window sits where the clusters are
