"""Multi-GPU matching: one process per GPU.

The update set is partitioned across ranks by coordinate slab (dim-0 lower
bound); rank 0 builds the byte-copyable subscription index (sorted Slo/Shi,
ids, gathered upper keys, block maxima) once and broadcasts it over NVLink
with NCCL; every rank matches its own updates against the index in its own
kernels and keeps its pair list local (global update ids); the pair counts are
all-reduced.  The only exchange steps are the index broadcast and the 8-byte
count all-reduce.

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
