"""Shared helpers for the GPU parity tests (host-side marshalling only)."""
import numpy as np


def cuda(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float64))).cuda()


def gpu_args(w):
    return cuda(w.sub_lo), cuda(w.sub_hi), cuda(w.upd_lo), cuda(w.upd_hi)


def words_of(pairs) -> np.ndarray:
    """[K,2] int32 (sub, upd) -> canonical u64 words, sorted."""
    p = pairs.cpu().numpy().astype(np.uint32)
    if p.size == 0:
        return np.zeros(0, dtype=np.uint64)
    w = (p[:, 1].astype(np.uint64) << np.uint64(32)) | p[:, 0].astype(np.uint64)
    return np.sort(w)


def raw_words(pairs) -> np.ndarray:
    p = pairs.cpu().numpy().astype(np.uint32)
    if p.size == 0:
        return np.zeros(0, dtype=np.uint64)
    return (p[:, 1].astype(np.uint64) << np.uint64(32)) | p[:, 0].astype(np.uint64)


def arrays(sl, sh, ul, uh):
    f = lambda x: np.ascontiguousarray(np.asarray(x, dtype=np.float64).reshape(len(x) if np.ndim(x) > 1 else 1, -1))
    return f(sl), f(sh), f(ul), f(uh)


def oracle_list_by_cells(orc, w, cell: float) -> np.ndarray:
    """The full canonical pair list of a d-dim instance from the oracle's
    serial SBM (Alg. 4 + filter), run cell by cell.  Space is cut
    into cubes of side `cell`; a pair (S, U) is owned by the cube holding the
    lower corner of S ∩ U, x_k = max(S.lo_k, U.lo_k) -- exactly one cube.
    Both boxes meet that cube (S.lo_k <= x_k and S.hi_k >= x_k, likewise U),
    so running the oracle on the regions meeting each cube and keeping the
    pairs whose corner lies in it yields every pair exactly once."""
    d = w.d
    lo_b = np.concatenate([np.floor(w.sub_lo / cell), np.floor(w.upd_lo / cell)], axis=1).astype(np.int64)
    hi_b = np.concatenate([np.floor(w.sub_hi / cell), np.floor(w.upd_hi / cell)], axis=1).astype(np.int64)
    span = hi_b - lo_b
    assert span.min() >= 0 and span.max() <= 1, "cells must exceed every side length"
    nc = int(max(hi_b.max(), 0)) + 2
    n = w.n
    # every (region, cube met) pair: at most 2^d cubes per region
    regs, cubes = [], []
    for corner in range(1 << d):
        off = np.array([(corner >> k) & 1 for k in range(d)], dtype=np.int64)[:, None]
        ok = np.all(off <= span, axis=0)
        c = lo_b[:, ok] + off
        key = np.zeros(c.shape[1], dtype=np.int64)
        for k in range(d):
            key = key * nc + c[k]
        regs.append(np.nonzero(ok)[0])
        cubes.append(key)
    regs, cubes = np.concatenate(regs), np.concatenate(cubes)
    o = np.lexsort((regs, cubes))
    regs, cubes = regs[o], cubes[o]
    bounds = np.flatnonzero(np.diff(cubes)) + 1
    starts, ends = np.concatenate([[0], bounds]), np.concatenate([bounds, [cubes.size]])
    out = []
    for a, b in zip(starts, ends):
        r = regs[a:b]
        si, ui = r[r < n], r[r >= n] - n
        if si.size == 0 or ui.size == 0:
            continue
        loc = orc.sbm_seq(w.sub_lo[:, si], w.sub_hi[:, si], w.upd_lo[:, ui], w.upd_hi[:, ui], canonicalize=False)
        if loc.size == 0:
            continue
        ls, lu = (loc & np.uint64(0xFFFFFFFF)).astype(np.int64), (loc >> np.uint64(32)).astype(np.int64)
        gs, gu = si[ls], ui[lu]
        key = np.zeros(gs.size, dtype=np.int64)
        for k in range(d):
            key = key * nc + np.floor(np.maximum(w.sub_lo[k, gs], w.upd_lo[k, gu]) / cell).astype(np.int64)
        mine = key == cubes[a]
        out.append((gu[mine].astype(np.uint64) << np.uint64(32)) | gs[mine].astype(np.uint64))
    return np.sort(np.concatenate(out)) if out else np.zeros(0, dtype=np.uint64)
