"""Multi-GPU matching: one process per GPU.

The update set is partitioned across ranks by coordinate slab (dim-0 lower
bound at equal-count quantiles).  Two modes:

  * "slab" (default, fully distributed index): rank r holds its updates
    (lo in [c_r, c_{r+1})) and exactly the subscriptions that can reach them,
    {S : S.hi >= c_r and S.lo <= max hi of its updates} -- its slab plus the
    halo of intervals crossing c_r (the stabbing set at the slab start,
    Alg. 6's SubSet[p] at a segment boundary) and the few starting
    past c_{r+1} that the slab's last updates reach.  Every rank runs the
    whole pipeline on its partition (ddm_match_pairs_mapped, global ids) and
    the pair counts are all-reduced: no data-path collective, each pair found
    once (on its update's rank), per-rank work ~1/G.
  * "broadcast" (the north star's literal split): rank 0 builds the
    byte-copyable subscription index once and broadcasts it over NVLink with
    NCCL; every rank matches its own updates against it.  Its index build is
    a serial term that does not shrink with G.

Each rank keeps its pair list local (global ids).

Host logic (slab cut points, id bookkeeping, the collective sequence) is
backend-agnostic so it is covered by world-size-2 gloo tests on CPU with a
stand-in matcher (tests/test_dist.py); the device work goes through libddm.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from . import ddm


def slab_cuts(values: np.ndarray, world: int) -> np.ndarray:
    """world-1 cut points at equal-count quantiles of `values` (dim-0 lower
    bounds): slab r holds lo in [cut[r-1], cut[r])."""
    if world <= 1 or values.size == 0:
        return np.zeros(0, dtype=np.float64)
    q = np.arange(1, world, dtype=np.float64) / world
    return np.quantile(values, q, method="inverted_cdf").astype(np.float64)


def slab_of(lo0: np.ndarray, cuts: np.ndarray) -> np.ndarray:
    return np.searchsorted(cuts, lo0, side="right")


def local_updates(upd_lo: np.ndarray, upd_hi: np.ndarray, rank: int, world: int, cuts=None):
    """This rank's updates (arrays [d, m_r]) and their global ids (int32)."""
    if cuts is None:
        cuts = slab_cuts(upd_lo[0], world)
    ids = np.nonzero(slab_of(upd_lo[0], cuts) == rank)[0]
    return (np.ascontiguousarray(upd_lo[:, ids]), np.ascontiguousarray(upd_hi[:, ids]),
            ids.astype(np.int32))


def reach_bounds(upd_lo: np.ndarray, upd_hi: np.ndarray, cuts: np.ndarray, world: int):
    """Per slab r: (c_r, max upper bound of its updates) -- a subscription can
    meet an update of slab r only if S.hi >= c_r and S.lo <= that maximum."""
    slab = slab_of(upd_lo[0], cuts)
    lo = np.concatenate([[-np.inf], cuts])
    hi = np.full(world, -np.inf)
    np.maximum.at(hi, slab, upd_hi[0])
    return lo, hi


def local_subscriptions(sub_lo: np.ndarray, sub_hi: np.ndarray, rank: int, c_lo: float, reach_hi: float):
    """Rank r's subscriptions for the slab mode and their global ids: the
    slab's own plus the halo (intervals crossing c_r from below, and those
    starting past the slab that its updates still reach)."""
    ids = np.nonzero((sub_hi[0] >= c_lo) & (sub_lo[0] <= reach_hi))[0]
    return (np.ascontiguousarray(sub_lo[:, ids]), np.ascontiguousarray(sub_hi[:, ids]),
            ids.astype(np.int32))


def slab_partition(w, rank: int, world: int):
    """(sub_lo, sub_hi, sub_ids, upd_lo, upd_hi, upd_ids) of rank r in slab mode."""
    cuts = slab_cuts(w.upd_lo[0], world)
    ul, uh, uids = local_updates(w.upd_lo, w.upd_hi, rank, world, cuts)
    lo, hi = reach_bounds(w.upd_lo, w.upd_hi, cuts, world)
    sl, sh, sids = local_subscriptions(w.sub_lo, w.sub_hi, rank, lo[rank], hi[rank])
    return sl, sh, sids, ul, uh, uids


class SlabMatcher:
    """Slab mode (fully distributed index): the whole pipeline on this rank's
    partition with global ids, then all_reduce(K).  Preallocated for bench.py."""

    def __init__(self, d: int, n_sub_local: int, m_local: int, capacity: int, device, group=None):
        self.M = ddm.Matcher(d, n_sub_local, m_local, device)
        self.device = torch.device(device)
        self.group = group
        self.out = torch.empty((max(capacity, 1), 2), dtype=torch.int32, device=self.device)
        self.k_buf = torch.zeros(1, dtype=torch.int64, device=self.device)

    def step(self, sub_lo, sub_hi, sub_ids, upd_lo, upd_hi, upd_ids, flags: int = 0) -> "DistResult":
        k_local = self.M.pairs_mapped_into(self.out, sub_lo, sub_hi, upd_lo, upd_hi, sub_ids, upd_ids, flags)
        self.k_buf.fill_(k_local)
        dist.all_reduce(self.k_buf, op=dist.ReduceOp.SUM, group=self.group)  # C2: the only collective
        return DistResult(k_local, int(self.k_buf.item()))


@dataclass
class DistResult:
    k_local: int
    k_total: int


class ShardedMatcher:
    """Preallocated multi-GPU matcher for a fixed problem (used by bench.py).

    step(): rank 0 builds the subscription index, broadcast(index) to all
    ranks, each rank matches its local updates into `out`, all_reduce(K)."""

    def __init__(self, d: int, n_sub: int, m_local: int, capacity: int, device, group=None):
        L = ddm.load()
        self.d, self.n_sub, self.m_local = d, n_sub, m_local
        self.device = torch.device(device)
        self.group = group
        self.index = torch.empty(max(L.ddm_sub_index_bytes(d, n_sub), 256), dtype=torch.uint8, device=self.device)
        self.ws_build = torch.empty(max(L.ddm_index_build_workspace_bytes(d, n_sub), 256), dtype=torch.uint8,
                                    device=self.device)
        self.ws = torch.empty(max(L.ddm_indexed_workspace_bytes(d, n_sub, m_local), 256), dtype=torch.uint8,
                              device=self.device)
        self.out = torch.empty((max(capacity, 1), 2), dtype=torch.int32, device=self.device)
        self.k_buf = torch.zeros(1, dtype=torch.int64, device=self.device)

    def build_index(self, sub_lo, sub_hi):
        L = ddm.load()
        r, keep = ddm.regions(sub_lo, sub_hi)
        ddm._check(L.ddm_sub_index_build(ctypes.byref(r), self.index.data_ptr(), self.index.numel(),
                                         self.ws_build.data_ptr(), self.ws_build.numel(),
                                         ddm._stream(self.device)), "ddm_sub_index_build")

    def match_local(self, upd_lo, upd_hi, upd_ids, flags: int = 0) -> int:
        L = ddm.load()
        r, keep = ddm.regions(upd_lo=upd_lo, upd_hi=upd_hi, n_sub=self.n_sub)
        K = ctypes.c_uint64(0)
        ddm._check(L.ddm_match_pairs_indexed(self.index.data_ptr(), ctypes.byref(r), upd_ids.data_ptr(),
                                             self.out.data_ptr(), self.out.shape[0], ctypes.byref(K), flags,
                                             self.ws.data_ptr(), self.ws.numel(), ddm._stream(self.device)),
                   "ddm_match_pairs_indexed")
        return int(K.value)

    def step(self, sub_lo, sub_hi, upd_lo, upd_hi, upd_ids, flags: int = 0) -> DistResult:
        rank = dist.get_rank(self.group)
        if rank == 0:
            self.build_index(sub_lo, sub_hi)
        dist.broadcast(self.index, src=0, group=self.group)   # C1: index over NVLink
        k_local = self.match_local(upd_lo, upd_hi, upd_ids, flags)
        self.k_buf.fill_(k_local)
        dist.all_reduce(self.k_buf, op=dist.ReduceOp.SUM, group=self.group)  # C2
        return DistResult(k_local, int(self.k_buf.item()))


def run_sharded(step_build, step_match, rank: int, world: int, index_nbytes: int, device="cpu", group=None):
    """Backend-agnostic collective sequence of one multi-GPU step, used by
    the CPU (gloo) tests with stand-in build/match callables:
       index = build() on rank 0; broadcast(index); k = match(index); all_reduce(k)."""
    index = torch.empty(index_nbytes, dtype=torch.uint8, device=device)
    if rank == 0:
        index.copy_(step_build())
    dist.broadcast(index, src=0, group=group)
    pairs, k_local = step_match(index)
    k = torch.tensor([k_local], dtype=torch.int64, device=device)
    dist.all_reduce(k, op=dist.ReduceOp.SUM, group=group)
    return pairs, int(k.item())
