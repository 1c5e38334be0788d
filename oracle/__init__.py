"""CPU oracle for DDM region matching (arXiv 1703.06680) -- TEST INFRASTRUCTURE.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline /
`--impl reference` legs may import this package.  The product path
(`paper_1703_06680_b200`, `libddm.so`) never imports or links it, and the two
share no code.

Functions (each follows a PAPER.md passage, see oracle/ddm_oracle.c):

  bf_pairs / bf_count / bf_rows   Alg. 2 brute force + d-dim conjunction
  sbm_seq                         Alg. 4 sequential SBM, d>1 filter
  sbm_dd_literal                  per-dim pair sets + sort-merge intersection
  par_sbm                         Alg. 5 + Alg. 6 parallel SBM
  boundary_states / par_states    SubSet[p]/UpdSet[p] snapshots vs Alg. 6
  states_at                       SubSet snapshots before chosen update lower endpoints
  rank_count                      App. A identity I2 (numpy; O3)

All pins live in tests/test_oracle.py; none of these functions is "parity
unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ddm_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

ORC_ERR = {-1: "allocation failed", -2: "sweep sets not empty at the end (S:194)", -3: "bad argument"}


def build(force: bool = False) -> str:
    """Compile the oracle with plain gcc (-O2 -fopenmp)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               "-o", _LIB, _SRC])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        i64, i32, dp, u64p, u32p, i64p = (ctypes.c_int64, ctypes.c_int, ctypes.c_void_p,
                                          ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p)
        L.orc_intersect_1d.argtypes = [ctypes.c_double] * 4
        L.orc_intersect_1d.restype = i32
        L.orc_bf_pairs.argtypes = [i32, i64, i64, dp, dp, dp, dp, u64p, i64]
        L.orc_bf_pairs.restype = i64
        L.orc_bf_rows.argtypes = [i32, i64, i64, dp, dp, dp, dp, i64p, i64, u64p, i64, i64p]
        L.orc_bf_rows.restype = i64
        L.orc_sbm_seq.argtypes = [i32, i64, i64, dp, dp, dp, dp, i32, u64p, i64]
        L.orc_sbm_seq.restype = i64
        L.orc_sbm_dd_literal.argtypes = [i32, i64, i64, dp, dp, dp, dp, u64p, i64]
        L.orc_sbm_dd_literal.restype = i64
        L.orc_par_sbm.argtypes = [i64, i64, dp, dp, dp, dp, i32, i32, u64p, i64]
        L.orc_par_sbm.restype = i64
        L.orc_sbm_boundary_states.argtypes = [i64, i64, dp, dp, dp, dp, i32, u32p, i64p, i64, u32p, i64p, i64]
        L.orc_sbm_boundary_states.restype = i64
        L.orc_par_sbm_states.argtypes = [i64, i64, dp, dp, dp, dp, i32, u32p, i64p, i64, u32p, i64p, i64]
        L.orc_par_sbm_states.restype = i64
        L.orc_sbm_states_at.argtypes = [i64, i64, dp, dp, dp, dp, i64p, i64, u32p, i64p, i64]
        L.orc_sbm_states_at.restype = i64
        L.orc_canonicalize.argtypes = [u64p, i64]
        L.orc_canonicalize.restype = None
        L.orc_max_threads.argtypes = []
        L.orc_max_threads.restype = i32
        _lib = L
    return _lib


def _arr(a) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    if a.ndim == 1:
        a = a[None, :]
    return a


def _args(sub_lo, sub_hi, upd_lo, upd_hi):
    sl, sh, ul, uh = (_arr(x) for x in (sub_lo, sub_hi, upd_lo, upd_hi))
    d = sl.shape[0]
    if not (sh.shape == sl.shape and ul.shape[0] == d and uh.shape == ul.shape):
        raise ValueError("inconsistent region arrays")
    return d, sl.shape[1], ul.shape[1], (sl, sh, ul, uh)


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def _check(k: int) -> int:
    if k < 0:
        raise RuntimeError(f"oracle error {k}: {ORC_ERR.get(k, '?')}")
    return k


def intersect_1d(xlo, xhi, ylo, yhi) -> bool:
    """Alg. 1."""
    return bool(lib().orc_intersect_1d(xlo, xhi, ylo, yhi))


def canonical(pairs: np.ndarray) -> np.ndarray:
    """Sort u64 pair words ((upd << 32) | sub) ascending."""
    p = np.ascontiguousarray(pairs, dtype=np.uint64).copy()
    lib().orc_canonicalize(_ptr(p), p.size)
    return p


def bf_count(sub_lo, sub_hi, upd_lo, upd_hi) -> int:
    d, n, m, a = _args(sub_lo, sub_hi, upd_lo, upd_hi)
    return _check(lib().orc_bf_pairs(d, n, m, *map(_ptr, a), None, 0))


def bf_pairs(sub_lo, sub_hi, upd_lo, upd_hi) -> np.ndarray:
    """Alg. 2; returns canonical u64 pair words."""
    d, n, m, a = _args(sub_lo, sub_hi, upd_lo, upd_hi)
    K = bf_count(*a)
    out = np.empty(max(K, 1), dtype=np.uint64)
    K2 = _check(lib().orc_bf_pairs(d, n, m, *map(_ptr, a), _ptr(out), K))
    assert K2 == K
    return out[:K]


def bf_rows(sub_lo, sub_hi, upd_lo, upd_hi, rows) -> tuple[np.ndarray, np.ndarray]:
    """Alg. 2 for the update ids `rows` only -> (pairs in row order, per-row counts)."""
    d, n, m, a = _args(sub_lo, sub_hi, upd_lo, upd_hi)
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    counts = np.zeros(rows.size, dtype=np.int64)
    K = _check(lib().orc_bf_rows(d, n, m, *map(_ptr, a), _ptr(rows), rows.size, None, 0, _ptr(counts)))
    out = np.empty(max(K, 1), dtype=np.uint64)
    _check(lib().orc_bf_rows(d, n, m, *map(_ptr, a), _ptr(rows), rows.size, _ptr(out), K, _ptr(counts)))
    return out[:K], counts


def sbm_count(sub_lo, sub_hi, upd_lo, upd_hi) -> int:
    d, n, m, a = _args(sub_lo, sub_hi, upd_lo, upd_hi)
    return _check(lib().orc_sbm_seq(d, n, m, *map(_ptr, a), 1, None, 0))


def sbm_seq(sub_lo, sub_hi, upd_lo, upd_hi, canonicalize: bool = True) -> np.ndarray:
    """Alg. 4 (sweep dim 0, filter dims 1..d-1); canonical u64 pair words."""
    d, n, m, a = _args(sub_lo, sub_hi, upd_lo, upd_hi)
    K = sbm_count(*a)
    out = np.empty(max(K, 1), dtype=np.uint64)
    K2 = _check(lib().orc_sbm_seq(d, n, m, *map(_ptr, a), 0, _ptr(out), K))
    assert K2 == K
    out = out[:K]
    return canonical(out) if canonicalize else out


def sbm_dd_literal(sub_lo, sub_hi, upd_lo, upd_hi) -> np.ndarray:
    d, n, m, a = _args(sub_lo, sub_hi, upd_lo, upd_hi)
    K = _check(lib().orc_sbm_dd_literal(d, n, m, *map(_ptr, a), None, 0))
    out = np.empty(max(K, 1), dtype=np.uint64)
    _check(lib().orc_sbm_dd_literal(d, n, m, *map(_ptr, a), _ptr(out), K))
    return out[:K]


def par_sbm(sub_lo, sub_hi, upd_lo, upd_hi, P: int | None = None, count_only: bool = False,
            canonicalize: bool = True):
    """Alg. 5 + 6 on P OpenMP threads (d = 1 only, as in the paper)."""
    d, n, m, a = _args(sub_lo, sub_hi, upd_lo, upd_hi)
    if d != 1:
        raise ValueError("Parallel-SBM-1D is one-dimensional (P:481-557)")
    P = P or max_threads()
    K = _check(lib().orc_par_sbm(n, m, *map(_ptr, a), P, 1, None, 0))
    if count_only:
        return K
    out = np.empty(max(K, 1), dtype=np.uint64)
    K2 = _check(lib().orc_par_sbm(n, m, *map(_ptr, a), P, 0, _ptr(out), K))
    assert K2 == K
    out = out[:K]
    return canonical(out) if canonicalize else out


def _states(fn, sub_lo, sub_hi, upd_lo, upd_hi, P):
    d, n, m, a = _args(sub_lo, sub_hi, upd_lo, upd_hi)
    cap_s, cap_u = max(1, n * P), max(1, m * P)
    sid = np.empty(cap_s, dtype=np.uint32)
    uid = np.empty(cap_u, dtype=np.uint32)
    soff = np.zeros(P + 1, dtype=np.int64)
    uoff = np.zeros(P + 1, dtype=np.int64)
    _check(fn(n, m, *map(_ptr, a), P, _ptr(sid), _ptr(soff), cap_s, _ptr(uid), _ptr(uoff), cap_u))
    subs = [np.sort(sid[soff[p]:soff[p + 1]]) for p in range(P)]
    upds = [np.sort(uid[uoff[p]:uoff[p + 1]]) for p in range(P)]
    return subs, upds


def boundary_states(sub_lo, sub_hi, upd_lo, upd_hi, P: int):
    """Sequential-sweep snapshots SubSet/UpdSet at the start of each T_p."""
    return _states(lib().orc_sbm_boundary_states, sub_lo, sub_hi, upd_lo, upd_hi, P)


def par_states(sub_lo, sub_hi, upd_lo, upd_hi, P: int):
    """SubSet[p]/UpdSet[p] computed by Alg. 6 (delta scan + master combine)."""
    return _states(lib().orc_par_sbm_states, sub_lo, sub_hi, upd_lo, upd_hi, P)


def states_at(sub_lo, sub_hi, upd_lo, upd_hi, upd_ids) -> list:
    """Sequential-sweep SubSet snapshot right before the lower endpoint of
    each update in `upd_ids` (d = 1; sorted id arrays, one per query)."""
    d, n, m, a = _args(sub_lo, sub_hi, upd_lo, upd_hi)
    if d != 1:
        raise ValueError("one sweep dimension")
    q = np.ascontiguousarray(upd_ids, dtype=np.int64)
    off = np.zeros(q.size + 1, dtype=np.int64)
    total = _check(lib().orc_sbm_states_at(n, m, *map(_ptr, a), _ptr(q), q.size, None, _ptr(off), 0))
    ids = np.empty(max(total, 1), dtype=np.uint32)
    _check(lib().orc_sbm_states_at(n, m, *map(_ptr, a), _ptr(q), q.size, _ptr(ids), _ptr(off), total))
    return [ids[off[r]:off[r + 1]].copy() for r in range(q.size)]


def max_threads() -> int:
    return int(lib().orc_max_threads())


def rank_count(sub_lo, sub_hi, upd_lo, upd_hi) -> int:
    """App. A identity I2 (O3): K = sum_u #{S.lo <= U.hi} - #{S.hi < U.lo},
    using np.sort / np.searchsorted as library primitives.  d = 1."""
    d, n, m, (sl, sh, ul, uh) = _args(sub_lo, sub_hi, upd_lo, upd_hi)
    if d != 1:
        raise ValueError("rank identity is per dimension")
    slo = np.sort(sl[0])
    shi = np.sort(sh[0])
    # the sums do not depend on the order of the queries: searching them in
    # ascending order keeps the binary searches cache-resident (c5: 5e8
    # queries in under a minute instead of a quarter of an hour)
    a = np.searchsorted(slo, np.sort(uh[0]), side="right").astype(np.int64).sum()
    b = np.searchsorted(shi, np.sort(ul[0]), side="left").astype(np.int64).sum()
    return int(a - b)
