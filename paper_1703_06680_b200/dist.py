"""Multi-GPU matching: one process per GPU.

Two modes, both with every rank's pair list kept local (global ids):

  * "slab" (default, fully distributed index).  Every rank starts with a
    block of the regions -- global ids [base, base + count) of each kind --
    in its own HBM.  One step:
      1. sample its update lower bounds (ddm_slab_sample), all_gather the
         samples, cut points at their quantiles (ddm_slab_cuts);
      2. pack its updates by destination slab (ddm_slab_pack, side 1), which
         also yields the per-slab maximum update upper bound -> all_reduce(MAX);
      3. pack its subscriptions to every slab they can reach (side 0): the
         slab's own plus the halo of intervals crossing the slab start -- the
         stabbing set at a segment boundary, Alg. 6's SubSet[p];
      4. all_to_all of the per-destination counts, then of the packed rows
         (C5, the exchange step), unpack (ddm_slab_unpack);
      5. match the received regions (ddm_match_pairs_mapped, global ids):
         every pair is found exactly once, on its update's rank;
      6. all_reduce(K) (C2).
    Every step of the partition runs in libddm kernels; the host only moves
    counts (split sizes for the all_to_all).  Per-rank work ~1/G plus the
    halo; nothing serial remains.
  * "broadcast" (the north star's literal split): rank 0 builds the
    byte-copyable subscription index once and broadcasts it (NCCL over
    NVLink); every rank matches its own updates against it.  Its index build
    is a serial term that does not shrink with G.

The orchestration (SlabMatcher.step, ShardedMatcher.step) is backend-agnostic:
collectives go through `Coll`, which stages tensors through host memory when
the backend cannot take device tensors (gloo), and the device work goes
through an `ops` object -- `DeviceOps` (libddm) here; the CPU tests plug a
numpy stand-in into the same step over gloo (tests/test_dist.py).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import torch
import torch.distributed as dist

from . import ddm

SAMPLE_PER_RANK = 2048  # update lower bounds each rank contributes to the cut points


class Coll:
    """The collectives of the multi-GPU step over one process group.  NCCL
    takes device tensors directly; any other backend (gloo: the CPU tests, and
    several ranks sharing one GPU in tests) gets host copies."""

    def __init__(self, group=None):
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.stage = dist.get_backend(group) != "nccl"

    def _h(self, t):
        return t.cpu() if self.stage else t

    def all_gather(self, t: torch.Tensor) -> torch.Tensor:
        src = self._h(t.contiguous())
        parts = [torch.empty_like(src) for _ in range(self.world)]
        dist.all_gather(parts, src, group=self.group)
        return torch.cat(parts).to(t.device)

    def all_reduce_(self, t: torch.Tensor, op) -> torch.Tensor:
        if self.stage and t.device.type != "cpu":
            h = t.cpu()
            dist.all_reduce(h, op=op, group=self.group)
            t.copy_(h)
        else:
            dist.all_reduce(t, op=op, group=self.group)
        return t

    def all_to_all(self, inp: torch.Tensor, in_splits: list, out_splits: list) -> torch.Tensor:
        """First-dimension splits; returns the received tensor."""
        out = torch.empty((sum(out_splits),) + tuple(inp.shape[1:]), dtype=inp.dtype,
                          device="cpu" if self.stage else inp.device)
        dist.all_to_all_single(out, self._h(inp.contiguous()), output_split_sizes=out_splits,
                               input_split_sizes=in_splits, group=self.group)
        return out.to(inp.device)

    def broadcast_(self, t: torch.Tensor, src: int = 0) -> torch.Tensor:
        if self.stage and t.device.type != "cpu":
            h = t.cpu()
            dist.broadcast(h, src=src, group=self.group)
            t.copy_(h)
        else:
            dist.broadcast(t, src=src, group=self.group)
        return t


class DeviceOps:
    """The slab mode's device work through libddm (float64 [d, count] CUDA
    tensors; global ids int32 bit patterns of uint32)."""

    def __init__(self, d: int, device):
        self.d = d
        self.device = torch.device(device)
        self.M = None  # Matcher, grown with the received sizes
        self.out = torch.empty((1, 2), dtype=torch.int32, device=self.device)

    def sample(self, lo0: torch.Tensor, s: int) -> torch.Tensor:
        L = ddm.load()
        out = torch.empty(s, dtype=torch.float64, device=self.device)
        ddm._check(L.ddm_slab_sample(lo0.data_ptr() if lo0.numel() else None, lo0.numel(), out.data_ptr(), s,
                                     ddm._stream(self.device)), "ddm_slab_sample")
        return out

    def cuts(self, samples: torch.Tensor, world: int) -> torch.Tensor:
        L = ddm.load()
        cuts = torch.zeros(max(world - 1, 1), dtype=torch.float64, device=self.device)
        ddm._check(L.ddm_slab_cuts(samples.data_ptr(), samples.numel(), world, cuts.data_ptr(),
                                   ddm._stream(self.device)), "ddm_slab_cuts")
        return cuts[: world - 1]

    def pack(self, side: int, lo, hi, id_base: int, cuts, world: int, reach=None):
        """-> (rows [total, 2d+1] float64, send counts (list), reach_out (updates) or None)."""
        L = ddm.load()
        if side == 0:
            r, keep = ddm.regions(sub_lo=lo, sub_hi=hi)
        else:
            r, keep = ddm.regions(upd_lo=lo, upd_hi=hi, d=self.d)
        count = lo.shape[-1]
        ws = ddm._workspace(L.ddm_slab_pack_workspace_bytes(count, world), self.device)
        reach_out = torch.empty(world, dtype=torch.int64, device=self.device) if side == 1 else None
        counts = (ctypes.c_uint64 * world)()
        total = ctypes.c_uint64(0)
        cp = cuts.data_ptr() if world > 1 else None
        rp = reach.data_ptr() if reach is not None else None
        op = reach_out.data_ptr() if reach_out is not None else None
        st = ddm._stream(self.device)
        cnt_p = ctypes.cast(counts, ctypes.c_void_p)
        s = L.ddm_slab_pack(ctypes.byref(r), side, id_base, cp, world, rp, op, cnt_p, None, 0, ctypes.byref(total),
                            ws.data_ptr(), ws.numel(), st)
        if s not in (0, 4):
            ddm._check(s, "ddm_slab_pack(size)")
        rows = torch.empty((int(total.value), 2 * self.d + 1), dtype=torch.float64, device=self.device)
        if rows.shape[0]:
            ddm._check(L.ddm_slab_pack(ctypes.byref(r), side, id_base, cp, world, rp, op, cnt_p, rows.data_ptr(),
                                       rows.shape[0], ctypes.byref(total), ws.data_ptr(), ws.numel(), st),
                       "ddm_slab_pack")
        return rows, [int(c) for c in counts], reach_out

    def unpack(self, rows: torch.Tensor):
        L = ddm.load()
        c = rows.shape[0]
        lo = torch.empty((self.d, c), dtype=torch.float64, device=self.device)
        hi = torch.empty_like(lo)
        ids = torch.empty(c, dtype=torch.int32, device=self.device)
        if c:
            ddm._check(L.ddm_slab_unpack(rows.data_ptr(), c, self.d, lo.data_ptr(), hi.data_ptr(), ids.data_ptr(),
                                         ddm._stream(self.device)), "ddm_slab_unpack")
        return lo, hi, ids

    def match(self, sub_lo, sub_hi, sub_ids, upd_lo, upd_hi, upd_ids, flags: int = 0):
        """ddm_match_pairs_mapped into a buffer grown on demand -> (pairs view, K)."""
        n, m = sub_lo.shape[1], upd_lo.shape[1]
        if self.M is None or self.M.n_sub < n or self.M.n_upd < m:
            self.M = ddm.Matcher(self.d, int(n * 1.05) + 1, int(m * 1.05) + 1, self.device)
        try:
            k = self.M.pairs_mapped_into(self.out, sub_lo, sub_hi, upd_lo, upd_hi, sub_ids, upd_ids, flags)
        except ddm.DDMError as e:
            if e.status != 4:  # DDM_ERR_CAPACITY: grow and redo (first steps only)
                raise
            k = self.M.count(sub_lo, sub_hi, upd_lo, upd_hi)
            self.out = torch.empty((int(k * 1.05) + 1, 2), dtype=torch.int32, device=self.device)
            k = self.M.pairs_mapped_into(self.out, sub_lo, sub_hi, upd_lo, upd_hi, sub_ids, upd_ids, flags)
        return self.out[:k], k


@dataclass
class DistResult:
    k_local: int
    k_total: int
    pairs: torch.Tensor | None = None  # this rank's pairs (global ids), a view valid until the next step
    marks: dict = field(default_factory=dict)  # CUDA events between the phases (device runs)


class SlabMatcher:
    """Slab mode (fully distributed index), see the module docstring.
    step() takes this rank's block of subscriptions and updates ([d, count]
    tensors, global ids sub_base + i / upd_base + i) and returns its pairs and
    the all-reduced K."""

    def __init__(self, d: int, device, group=None, ops=None):
        self.d = d
        self.device = torch.device(device)
        self.coll = Coll(group)
        self.ops = ops if ops is not None else DeviceOps(d, self.device)
        self.timed = self.device.type == "cuda"

    def _mark(self, marks, name):
        if self.timed:
            e = torch.cuda.Event(enable_timing=True)
            e.record(torch.cuda.current_stream(self.device))
            marks[name] = e

    def step(self, sub_lo, sub_hi, sub_base: int, upd_lo, upd_hi, upd_base: int, flags: int = 0) -> DistResult:
        C, ops, G = self.coll, self.ops, self.coll.world
        marks: dict = {}
        self._mark(marks, "start")
        # 1. cut points from a gathered sample of update lower bounds
        cuts = ops.cuts(C.all_gather(ops.sample(upd_lo[0], SAMPLE_PER_RANK)), G)
        # 2. updates by slab; per-slab reach of their upper bounds
        u_rows, u_cnt, reach = ops.pack(1, upd_lo, upd_hi, upd_base, cuts, G)
        C.all_reduce_(reach, dist.ReduceOp.MAX)
        # 3. subscriptions to every slab they reach (slab + halo)
        s_rows, s_cnt, _ = ops.pack(0, sub_lo, sub_hi, sub_base, cuts, G, reach=reach)
        # 4. exchange (C5): counts, then the rows
        cnt = torch.tensor(u_cnt + s_cnt, dtype=torch.int64).reshape(2, G).t().contiguous()  # [G][2]
        got = C.all_to_all(cnt.to(self.device) if not C.stage else cnt, [1] * G, [1] * G).cpu()  # [G][2]
        u_in, s_in = [int(x) for x in got[:, 0]], [int(x) for x in got[:, 1]]
        ul, uh, uids = ops.unpack(C.all_to_all(u_rows, u_cnt, u_in))
        sl, sh, sids = ops.unpack(C.all_to_all(s_rows, s_cnt, s_in))
        self._mark(marks, "partitioned")
        # 5. match the slab (global ids); 6. K over all ranks
        pairs, k_local = ops.match(sl, sh, sids, ul, uh, uids, flags)
        self._mark(marks, "matched")
        k = torch.tensor([k_local], dtype=torch.int64, device=self.device)
        C.all_reduce_(k, dist.ReduceOp.SUM)
        self._mark(marks, "end")
        return DistResult(k_local, int(k.item()), pairs, marks)


class ShardedMatcher:
    """Broadcast mode: rank 0 builds the subscription index, broadcast(index)
    to all ranks, each rank matches its local updates into `out`,
    all_reduce(K).  Preallocated for a fixed problem (bench.py)."""

    def __init__(self, d: int, n_sub: int, m_local: int, capacity: int, device, group=None):
        L = ddm.load()
        self.d, self.n_sub, self.m_local = d, n_sub, m_local
        self.device = torch.device(device)
        self.coll = Coll(group)
        self.index = torch.empty(max(L.ddm_sub_index_bytes(d, n_sub), 256), dtype=torch.uint8, device=self.device)
        self.ws_build = torch.empty(max(L.ddm_index_build_workspace_bytes(d, n_sub), 256), dtype=torch.uint8,
                                    device=self.device)
        self.ws = torch.empty(max(L.ddm_indexed_workspace_bytes(d, n_sub, m_local), 256), dtype=torch.uint8,
                              device=self.device)
        self.out = torch.empty((max(capacity, 1), 2), dtype=torch.int32, device=self.device)

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
        marks: dict = {}
        stream = torch.cuda.current_stream(self.device)

        def mark(name):
            e = torch.cuda.Event(enable_timing=True)
            e.record(stream)
            marks[name] = e

        mark("start")
        if self.coll.rank == 0:
            self.build_index(sub_lo, sub_hi)
        self.coll.broadcast_(self.index, src=0)   # C1: index over NVLink
        mark("indexed")
        k_local = self.match_local(upd_lo, upd_hi, upd_ids, flags)
        mark("matched")
        k = torch.tensor([k_local], dtype=torch.int64, device=self.device)
        self.coll.all_reduce_(k, dist.ReduceOp.SUM)  # C2
        mark("end")
        return DistResult(k_local, int(k.item()), self.out[:k_local], marks)


def block_of(count: int, rank: int, world: int) -> tuple[int, int]:
    """[begin, end) of rank's contiguous block of `count` items (the initial
    distribution of the regions over the ranks: input order)."""
    b = count * rank // world
    return b, count * (rank + 1) // world


def slab_of_updates(upd_lo0, cuts):
    """Host reference of the update rule (tests): slab = #cuts <= lo."""
    import numpy as np
    return np.searchsorted(np.asarray(cuts), np.asarray(upd_lo0), side="right")
