"""Thin Python binding of libddm (include/ddm.h) -- argument marshalling only.

Every step of the matching path runs in libddm's CUDA kernels; this module
only converts torch CUDA tensors into the C ABI's pointers, sizes and the
current CUDA stream, and allocates the caller-owned workspace / outputs with
torch.  There is no CPU fallback: without the built library or a CUDA device
every entry point raises.

Names follow the C ABI: match_count, match_pairs, sort_pairs, sub_index_build,
match_pairs_indexed, match_count_indexed, radix_sort_u64, encode_keys.
"""
from __future__ import annotations

import ctypes
import os

import torch

from . import _build

DDM_MAX_DIMS = 8
DDM_MAX_REGIONS = (1 << 30) - 1
DDM_EMIT_AUTO = 0
DDM_EMIT_FORCE_THREAD = 1 << 8
DDM_EMIT_FORCE_WARP = 1 << 9
DDM_EMIT_FORCE_CHUNK = 1 << 10
DDM_SORT_LSB = 1 << 12
DDM_COUNT_RANKS = 1 << 13
DDM_COUNT_WALK = 1 << 14
DDM_SWEEP_DIM0 = 1 << 15
DDM_DD_FORCE_ROWS = 1 << 16
DDM_DD_FORCE_CHUNKS = 1 << 17

STATUS = {0: "DDM_OK", 1: "DDM_ERR_INVALID_ARGUMENT", 2: "DDM_ERR_NONFINITE",
          3: "DDM_ERR_INVERTED_INTERVAL", 4: "DDM_ERR_CAPACITY", 5: "DDM_ERR_WORKSPACE",
          6: "DDM_ERR_CUDA"}


class DDMError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        name = STATUS.get(status, f"status {status}")
        extra = ""
        if status == 6 and _lib is not None:
            extra = f" (cudaError {_lib.ddm_last_cuda_error()})"
        super().__init__(f"{where}: {name}{extra}")


class _KernelStat(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char * 32), ("launches", ctypes.c_uint64), ("total_ms", ctypes.c_double),
                ("bytes", ctypes.c_double)]


class _Regions(ctypes.Structure):
    _fields_ = [("d", ctypes.c_uint32), ("n_sub", ctypes.c_uint64), ("n_upd", ctypes.c_uint64),
                ("sub_lo", ctypes.c_void_p * DDM_MAX_DIMS), ("sub_hi", ctypes.c_void_p * DDM_MAX_DIMS),
                ("upd_lo", ctypes.c_void_p * DDM_MAX_DIMS), ("upd_hi", ctypes.c_void_p * DDM_MAX_DIMS)]


_lib = None


def lib_path() -> str:
    return _build.LIB


def load() -> ctypes.CDLL:
    """Load the in-tree libddm.so; raise loudly if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_build.LIB):
        raise RuntimeError(f"libddm.so not built ({_build.LIB}); run __graft_entry__.build()")
    L = ctypes.CDLL(_build.LIB)
    vp, u64, u32, i32, sz = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int, ctypes.c_size_t
    R = ctypes.POINTER(_Regions)
    sig = {
        "ddm_workspace_bytes": ([u32, u64, u64, i32], sz),
        "ddm_match_count": ([R, ctypes.POINTER(u64), vp, sz, vp], i32),
        "ddm_match_pairs": ([R, vp, u64, ctypes.POINTER(u64), u32, vp, sz, vp], i32),
        "ddm_match_pairs_mapped": ([R, vp, vp, vp, u64, ctypes.POINTER(u64), u32, vp, sz, vp], i32),
        "ddm_sort_pairs_workspace_bytes": ([u64], sz),
        "ddm_sort_pairs": ([vp, u64, u64, u64, vp, sz, vp], i32),
        "ddm_sub_index_bytes": ([u32, u64], sz),
        "ddm_index_build_workspace_bytes": ([u32, u64], sz),
        "ddm_sub_index_build": ([R, vp, sz, vp, sz, vp], i32),
        "ddm_indexed_workspace_bytes": ([u32, u64, u64], sz),
        "ddm_match_pairs_indexed": ([vp, R, vp, vp, u64, ctypes.POINTER(u64), u32, vp, sz, vp], i32),
        "ddm_events_workspace_bytes": ([u32, u64, u64], sz),
        "ddm_sub_index_update_workspace_bytes": ([u32, u64, u64, i32], sz),
        "ddm_sub_index_update": ([vp, vp, sz, u64, R, vp, vp, sz, vp], i32),
        "ddm_match_pairs_events": ([R, vp, u64, ctypes.POINTER(u64), vp, sz, vp], i32),
        "ddm_match_count_indexed": ([vp, R, ctypes.POINTER(u64), vp, sz, vp], i32),
        "ddm_chunk_start_sets": ([R, vp, vp, vp, u64, ctypes.POINTER(u64), vp, sz, vp], i32),
        "ddm_slab_sample": ([vp, u64, vp, u32, vp], i32),
        "ddm_literal_workspace_bytes": ([u32, u64, u64, u64], sz),
        "ddm_match_pairs_literal": ([R, vp, u64, ctypes.POINTER(u64), u64, ctypes.POINTER(u64), vp, sz, vp], i32),
        "ddm_slab_cuts": ([vp, u32, u32, vp, vp], i32),
        "ddm_slab_pack_workspace_bytes": ([u64, u32], sz),
        "ddm_slab_pack": ([R, i32, u64, vp, u32, vp, vp, vp, vp, u64, ctypes.POINTER(u64), vp, sz, vp], i32),
        "ddm_slab_unpack": ([vp, u64, u32, vp, vp, vp, vp], i32),
        "ddm_radix_sort_workspace_bytes": ([u64], sz),
        "ddm_radix_sort_u64": ([vp, vp, vp, vp, u64, i32, i32, vp, sz, vp], i32),
        "ddm_encode_keys": ([vp, vp, u64, vp], i32),
        "ddm_status_string": ([i32], ctypes.c_char_p),
        "ddm_last_cuda_error": ([], i32),
        "ddm_kernel_launch_count": ([], u64),
        "ddm_build_info": ([], ctypes.c_char_p),
        "ddm_profile_enable": ([i32], None),
        "ddm_profile_read": ([ctypes.POINTER(_KernelStat), i32], i32),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _lib = L
    return L


EXPORTED = ["ddm_workspace_bytes", "ddm_match_count", "ddm_match_pairs", "ddm_match_pairs_mapped",
            "ddm_sort_pairs_workspace_bytes",
            "ddm_sort_pairs", "ddm_sub_index_bytes", "ddm_index_build_workspace_bytes", "ddm_sub_index_build",
            "ddm_indexed_workspace_bytes", "ddm_match_pairs_indexed", "ddm_match_count_indexed",
            "ddm_events_workspace_bytes", "ddm_match_pairs_events",
            "ddm_sub_index_update_workspace_bytes", "ddm_sub_index_update",
            "ddm_chunk_start_sets", "ddm_literal_workspace_bytes", "ddm_match_pairs_literal", "ddm_slab_sample", "ddm_slab_cuts", "ddm_slab_pack_workspace_bytes",
            "ddm_slab_pack", "ddm_slab_unpack",
            "ddm_radix_sort_workspace_bytes", "ddm_radix_sort_u64", "ddm_encode_keys", "ddm_status_string",
            "ddm_last_cuda_error", "ddm_kernel_launch_count", "ddm_build_info", "ddm_profile_enable",
            "ddm_profile_read"]


def _check(st: int, where: str):
    if st != 0:
        raise DDMError(st, where)


def _stream(device=None) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _as_2d(x: torch.Tensor, name: str) -> torch.Tensor:
    if not isinstance(x, torch.Tensor) or not x.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if x.dtype != torch.float64:
        raise TypeError(f"{name} must be float64")
    if x.dim() == 1:
        x = x.unsqueeze(0)
    if x.dim() != 2:
        raise ValueError(f"{name} must have shape [d, count]")
    return x.contiguous()


def regions(sub_lo=None, sub_hi=None, upd_lo=None, upd_hi=None, d=None, n_sub=0):
    """Build the C `ddm_regions` struct from [d, count] float64 CUDA tensors.
    Returns (struct, keepalive) -- keep the tensors alive during the call."""
    r = _Regions()
    keep = []
    dims = d
    if sub_lo is not None:
        sl, sh = _as_2d(sub_lo, "sub_lo"), _as_2d(sub_hi, "sub_hi")
        if sl.shape != sh.shape:
            raise ValueError("sub_lo/sub_hi shape mismatch")
        dims = sl.shape[0]
        r.n_sub = sl.shape[1]
        keep += [sl, sh]
        for k in range(dims):
            r.sub_lo[k] = sl[k].data_ptr()
            r.sub_hi[k] = sh[k].data_ptr()
    else:
        r.n_sub = n_sub
    if upd_lo is not None:
        ul, uh = _as_2d(upd_lo, "upd_lo"), _as_2d(upd_hi, "upd_hi")
        if ul.shape != uh.shape or (dims is not None and ul.shape[0] != dims):
            raise ValueError("update arrays inconsistent with subscriptions")
        dims = ul.shape[0]
        r.n_upd = ul.shape[1]
        keep += [ul, uh]
        for k in range(dims):
            r.upd_lo[k] = ul[k].data_ptr()
            r.upd_hi[k] = uh[k].data_ptr()
    if dims is None or dims < 1 or dims > DDM_MAX_DIMS:
        raise ValueError("d must be in 1..8")
    r.d = dims
    return r, keep


def _workspace(nbytes: int, device) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)


class Matcher:
    """Reusable workspace for repeated matches of one problem size (the
    hot loop in bench.py): no allocation inside match calls."""

    def __init__(self, d: int, n_sub: int, n_upd: int, device="cuda"):
        L = load()
        self.d, self.n_sub, self.n_upd = d, n_sub, n_upd
        self.device = torch.device(device)
        self.ws = _workspace(L.ddm_workspace_bytes(d, n_sub, n_upd, 1), self.device)

    def count(self, sub_lo, sub_hi, upd_lo, upd_hi) -> int:
        L = load()
        r, keep = regions(sub_lo, sub_hi, upd_lo, upd_hi)
        K = ctypes.c_uint64(0)
        _check(L.ddm_match_count(ctypes.byref(r), ctypes.byref(K), self.ws.data_ptr(), self.ws.numel(),
                                 _stream(self.device)), "ddm_match_count")
        return int(K.value)

    def pairs_into(self, out: torch.Tensor, sub_lo, sub_hi, upd_lo, upd_hi, flags: int = 0) -> int:
        """Write pairs into `out` (int32/uint32 CUDA tensor [cap, 2]); returns K."""
        L = load()
        r, keep = regions(sub_lo, sub_hi, upd_lo, upd_hi)
        K = ctypes.c_uint64(0)
        st = L.ddm_match_pairs(ctypes.byref(r), out.data_ptr() if out.numel() else None, out.shape[0],
                               ctypes.byref(K), flags, self.ws.data_ptr(), self.ws.numel(),
                               _stream(self.device))
        _check(st, "ddm_match_pairs")
        return int(K.value)


    def pairs_mapped_into(self, out: torch.Tensor, sub_lo, sub_hi, upd_lo, upd_hi, sub_ids=None, upd_ids=None,
                          flags: int = 0) -> int:
        """pairs_into with global id maps (uint32/int32 CUDA tensors or None):
        writes {sub_ids[s], upd_ids[u]} (ddm_match_pairs_mapped)."""
        L = load()
        r, keep = regions(sub_lo, sub_hi, upd_lo, upd_hi)
        K = ctypes.c_uint64(0)
        st = L.ddm_match_pairs_mapped(ctypes.byref(r), sub_ids.data_ptr() if sub_ids is not None else None,
                                      upd_ids.data_ptr() if upd_ids is not None else None,
                                      out.data_ptr() if out.numel() else None, out.shape[0], ctypes.byref(K), flags,
                                      self.ws.data_ptr(), self.ws.numel(), _stream(self.device))
        _check(st, "ddm_match_pairs_mapped")
        return int(K.value)


class PipelinedMatcher:
    """Matching of a stream of host-resident batches (the serving case: a new
    batch of regions every step) with the transfers overlapped: batch i+1's
    host->device copy (copy stream) is enqueued before batch i is matched
    (compute stream), and batch i's pairs travel device->host on a third
    stream while batch i+1 is matched (the link is full duplex).  Device
    inputs and outputs are double-buffered; one workspace serves every match
    (they are ordered on the compute stream).  Host buffers should be pinned.

        for k, host_out in pm.run((host_in, host_out) for ...):  ...

    yields (K, host_out) per batch once its copy-back is enqueued; the pairs
    are in host_out[:K] after the next batch's match returns or after run()
    finishes (it synchronises at the end)."""

    def __init__(self, d: int, n_sub: int, n_upd: int, capacity: int, device="cuda"):
        self.dev = torch.device(device)
        self.M = Matcher(d, n_sub, n_upd, self.dev)
        mk = lambda cnt: torch.empty((d, cnt), dtype=torch.float64, device=self.dev)  # noqa: E731
        self.inp = [[mk(n_sub), mk(n_sub), mk(n_upd), mk(n_upd)] for _ in range(2)]
        self.out = [torch.empty((max(capacity, 1), 2), dtype=torch.int32, device=self.dev) for _ in range(2)]
        self.s_h2d = torch.cuda.Stream(self.dev)
        self.s_cmp = torch.cuda.Stream(self.dev)
        self.s_d2h = torch.cuda.Stream(self.dev)
        self.ev_in = [torch.cuda.Event() for _ in range(2)]    # inputs of a slot copied in
        self.ev_used = [torch.cuda.Event() for _ in range(2)]  # a slot's inputs consumed by its match
        self.ev_out = [torch.cuda.Event() for _ in range(2)]   # a slot's pairs copied out

    def _h2d(self, slot, host):
        with torch.cuda.stream(self.s_h2d):
            self.s_h2d.wait_event(self.ev_used[slot])
            for dst, src in zip(self.inp[slot], host):
                dst.copy_(src, non_blocking=True)
            self.ev_in[slot].record(self.s_h2d)

    def run(self, batches):
        it = iter(batches)
        nxt = next(it, None)
        slot = 0
        if nxt is not None:
            self._h2d(slot, nxt[0])
        while nxt is not None:
            host_in, host_out = nxt
            nxt = next(it, None)
            if nxt is not None:
                self._h2d(slot ^ 1, nxt[0])  # next batch's copy overlaps this match
            with torch.cuda.stream(self.s_cmp):
                self.s_cmp.wait_event(self.ev_in[slot])
                self.s_cmp.wait_event(self.ev_out[slot])  # the slot's previous pairs have left
                k = self.M.pairs_into(self.out[slot], *self.inp[slot])  # one sync of s_cmp (K)
                self.ev_used[slot].record(self.s_cmp)
            with torch.cuda.stream(self.s_d2h):
                self.s_d2h.wait_stream(self.s_cmp)
                host_out[:k].copy_(self.out[slot][:k], non_blocking=True)
                self.ev_out[slot].record(self.s_d2h)
            yield k, host_out
            slot ^= 1
        torch.cuda.synchronize(self.dev)


def match_count(sub_lo, sub_hi, upd_lo, upd_hi) -> int:
    """K = number of intersecting (subscription, update) pairs."""
    L = load()
    r, keep = regions(sub_lo, sub_hi, upd_lo, upd_hi)
    dev = keep[0].device if keep else torch.device("cuda")
    ws = _workspace(L.ddm_workspace_bytes(r.d, r.n_sub, r.n_upd, 0), dev)
    K = ctypes.c_uint64(0)
    _check(L.ddm_match_count(ctypes.byref(r), ctypes.byref(K), ws.data_ptr(), ws.numel(), _stream(dev)),
           "ddm_match_count")
    return int(K.value)


def match_pairs(sub_lo, sub_hi, upd_lo, upd_hi, flags: int = 0, sort: bool = False,
                capacity: int | None = None) -> torch.Tensor:
    """All intersecting pairs as an int32 CUDA tensor [K, 2] of (sub, upd)
    (bit pattern of uint32).  Two-call pattern: sizes with capacity 0 first
    unless `capacity` is given.  sort=True returns canonical order."""
    L = load()
    r, keep = regions(sub_lo, sub_hi, upd_lo, upd_hi)
    dev = keep[0].device if keep else torch.device("cuda")
    ws = _workspace(L.ddm_workspace_bytes(r.d, r.n_sub, r.n_upd, 1), dev)
    K = ctypes.c_uint64(0)
    st = _stream(dev)
    if capacity is None:
        s = L.ddm_match_pairs(ctypes.byref(r), None, 0, ctypes.byref(K), flags, ws.data_ptr(), ws.numel(), st)
        if s not in (0, 4):
            _check(s, "ddm_match_pairs(size)")
        capacity = int(K.value)
    out = torch.empty((max(capacity, 1), 2), dtype=torch.int32, device=dev)
    _check(L.ddm_match_pairs(ctypes.byref(r), out.data_ptr(), capacity, ctypes.byref(K), flags, ws.data_ptr(),
                             ws.numel(), st), "ddm_match_pairs")
    out = out[: int(K.value)]
    if sort:
        sort_pairs(out, r.n_sub, r.n_upd)
    return out


DDM_CHUNK_ROWS = 256


def chunk_start_sets(sub_lo, sub_hi, upd_lo, upd_hi):
    """a6 exported (ddm_chunk_start_sets, d = 1): for every tile of
    DDM_CHUNK_ROWS sorted updates, (first update id x_t, A_t = Stab(x_t.lo) as
    subscription ids in Slo order).  Returns (first_upd [tiles] int32,
    offsets [tiles+1] int64, ids [total] int32) CUDA tensors."""
    L = load()
    r, keep = regions(sub_lo, sub_hi, upd_lo, upd_hi)
    dev = keep[0].device if keep else torch.device("cuda")
    ws = _workspace(L.ddm_workspace_bytes(r.d, r.n_sub, r.n_upd, 1), dev)
    tiles = (r.n_upd + DDM_CHUNK_ROWS - 1) // DDM_CHUNK_ROWS
    first = torch.empty(max(tiles, 1), dtype=torch.int32, device=dev)
    off = torch.zeros(tiles + 1, dtype=torch.int64, device=dev)
    T = ctypes.c_uint64(0)
    st = _stream(dev)
    s = L.ddm_chunk_start_sets(ctypes.byref(r), first.data_ptr(), off.data_ptr(), None, 0, ctypes.byref(T),
                               ws.data_ptr(), ws.numel(), st)
    if s not in (0, 4):
        _check(s, "ddm_chunk_start_sets(size)")
    ids = torch.empty(max(int(T.value), 1), dtype=torch.int32, device=dev)
    _check(L.ddm_chunk_start_sets(ctypes.byref(r), first.data_ptr(), off.data_ptr(), ids.data_ptr(), ids.numel(),
                                  ctypes.byref(T), ws.data_ptr(), ws.numel(), st), "ddm_chunk_start_sets")
    return first[:tiles], off, ids[: int(T.value)]


def match_pairs_literal(sub_lo, sub_hi, upd_lo, upd_hi, dim_capacity: int | None = None) -> torch.Tensor:
    """The literal d-dim reading (ddm_match_pairs_literal: per-dimension pair
    sets intersected by sort-merge), canonical order.  dim_capacity defaults
    to the largest per-dimension count (found by a first call)."""
    L = load()
    r, keep = regions(sub_lo, sub_hi, upd_lo, upd_hi)
    dev = keep[0].device if keep else torch.device("cuda")
    st = _stream(dev)
    K, Kd = ctypes.c_uint64(0), ctypes.c_uint64(0)
    if dim_capacity is None:
        dim_capacity = max(match_count(sub_lo[k:k + 1], sub_hi[k:k + 1], upd_lo[k:k + 1], upd_hi[k:k + 1])
                           for k in range(r.d))
    ws = _workspace(L.ddm_literal_workspace_bytes(r.d, r.n_sub, r.n_upd, dim_capacity), dev)
    out = torch.empty((max(dim_capacity, 1), 2), dtype=torch.int32, device=dev)
    _check(L.ddm_match_pairs_literal(ctypes.byref(r), out.data_ptr(), out.shape[0], ctypes.byref(K), dim_capacity,
                                     ctypes.byref(Kd), ws.data_ptr(), ws.numel(), st), "ddm_match_pairs_literal")
    return out[: int(K.value)]


def match_pairs_events(sub_lo, sub_hi, upd_lo, upd_hi, sort: bool = True) -> torch.Tensor:
    """The event-order variant (ddm_match_pairs_events: the paper's Alg. 5 + 6
    on the GPU, a cross-check of match_pairs).  Its own order is unspecified;
    sort=True (default) returns canonical order."""
    L = load()
    r, keep = regions(sub_lo, sub_hi, upd_lo, upd_hi)
    dev = keep[0].device if keep else torch.device("cuda")
    ws = _workspace(L.ddm_events_workspace_bytes(r.d, r.n_sub, r.n_upd), dev)
    K = ctypes.c_uint64(0)
    st = _stream(dev)
    _check(L.ddm_match_pairs_events(ctypes.byref(r), None, 0, ctypes.byref(K), ws.data_ptr(), ws.numel(), st),
           "ddm_match_pairs_events(count)")
    cap = int(K.value)
    out = torch.empty((max(cap, 1), 2), dtype=torch.int32, device=dev)
    _check(L.ddm_match_pairs_events(ctypes.byref(r), out.data_ptr(), cap, ctypes.byref(K), ws.data_ptr(), ws.numel(),
                                    st), "ddm_match_pairs_events")
    out = out[: int(K.value)]
    if sort:
        sort_pairs(out, r.n_sub, r.n_upd)
    return out


def sort_pairs(pairs: torch.Tensor, n_sub: int, n_upd: int) -> torch.Tensor:
    """In-place canonical order: ascending (upd << 32) | sub."""
    L = load()
    k = pairs.shape[0]
    if k == 0:
        return pairs
    ws = _workspace(L.ddm_sort_pairs_workspace_bytes(k), pairs.device)
    _check(L.ddm_sort_pairs(pairs.data_ptr(), k, n_sub, n_upd, ws.data_ptr(), ws.numel(), _stream(pairs.device)),
           "ddm_sort_pairs")
    return pairs


def pair_words(pairs: torch.Tensor) -> torch.Tensor:
    """View [K,2] int32 (sub, upd) as int64 words (upd << 32) | sub."""
    return pairs.contiguous().view(torch.int64).view(-1)


def sub_index_build(sub_lo, sub_hi) -> torch.Tensor:
    """Build the byte-copyable subscription index (uint8 CUDA tensor)."""
    L = load()
    r, keep = regions(sub_lo, sub_hi)
    dev = keep[0].device
    idx = _workspace(L.ddm_sub_index_bytes(r.d, r.n_sub), dev)
    ws = _workspace(L.ddm_index_build_workspace_bytes(r.d, r.n_sub), dev)
    _check(L.ddm_sub_index_build(ctypes.byref(r), idx.data_ptr(), idx.numel(), ws.data_ptr(), ws.numel(),
                                 _stream(dev)), "ddm_sub_index_build")
    return idx


def sub_index_update(index: torch.Tensor, n_sub: int, ids: torch.Tensor, new_lo, new_hi,
                     out: torch.Tensor | None = None) -> torch.Tensor:
    """Dynamic DDM: subscriptions `ids` (int32 CUDA, strictly increasing) of a
    built index take the coordinates new_lo/new_hi ([d, k] float64 CUDA).  The
    merged index goes to `out` (a second index buffer: ping-pong, no copy) or,
    by default, back into `index`; returns it (ddm_sub_index_update)."""
    L = load()
    r, keep = regions(new_lo, new_hi)
    dev = keep[0].device
    ids = ids.to(device=dev, dtype=torch.int32).contiguous()
    dst = index if out is None else out
    in_place = 1 if dst.data_ptr() == index.data_ptr() else 0
    ws = _workspace(L.ddm_sub_index_update_workspace_bytes(r.d, n_sub, r.n_sub, in_place), dev)
    _check(L.ddm_sub_index_update(index.data_ptr(), dst.data_ptr(), dst.numel(), n_sub, ctypes.byref(r),
                                  ids.data_ptr(), ws.data_ptr(), ws.numel(), _stream(dev)), "ddm_sub_index_update")
    return dst


def match_pairs_indexed(index: torch.Tensor, n_sub: int, upd_lo, upd_hi, upd_ids: torch.Tensor | None = None,
                        flags: int = 0, capacity: int | None = None) -> torch.Tensor:
    L = load()
    r, keep = regions(upd_lo=upd_lo, upd_hi=upd_hi, n_sub=n_sub)
    dev = keep[0].device
    ws = _workspace(L.ddm_indexed_workspace_bytes(r.d, n_sub, r.n_upd), dev)
    K = ctypes.c_uint64(0)
    st = _stream(dev)
    ids = upd_ids.data_ptr() if upd_ids is not None else None
    if capacity is None:
        s = L.ddm_match_pairs_indexed(index.data_ptr(), ctypes.byref(r), ids, None, 0, ctypes.byref(K), flags,
                                      ws.data_ptr(), ws.numel(), st)
        if s not in (0, 4):
            _check(s, "ddm_match_pairs_indexed(size)")
        capacity = int(K.value)
    out = torch.empty((max(capacity, 1), 2), dtype=torch.int32, device=dev)
    _check(L.ddm_match_pairs_indexed(index.data_ptr(), ctypes.byref(r), ids, out.data_ptr(), capacity,
                                     ctypes.byref(K), flags, ws.data_ptr(), ws.numel(), st),
           "ddm_match_pairs_indexed")
    return out[: int(K.value)]


def match_count_indexed(index: torch.Tensor, n_sub: int, upd_lo, upd_hi) -> int:
    L = load()
    r, keep = regions(upd_lo=upd_lo, upd_hi=upd_hi, n_sub=n_sub)
    dev = keep[0].device
    ws = _workspace(L.ddm_indexed_workspace_bytes(r.d, n_sub, r.n_upd), dev)
    K = ctypes.c_uint64(0)
    _check(L.ddm_match_count_indexed(index.data_ptr(), ctypes.byref(r), ctypes.byref(K), ws.data_ptr(),
                                     ws.numel(), _stream(dev)), "ddm_match_count_indexed")
    return int(K.value)


def radix_sort_u64(keys: torch.Tensor, vals: torch.Tensor | None = None, begin_bit: int = 0, end_bit: int = 64,
                   want_vals: bool = True):
    """Stable LSB radix sort of int64 (bit pattern u64) keys with optional
    int32 payload (payload = index when vals is None and want_vals)."""
    L = load()
    n = keys.numel()
    ko = torch.empty_like(keys)
    vo = torch.empty(n, dtype=torch.int32, device=keys.device) if (want_vals or vals is not None) else None
    if n == 0:
        return ko, vo
    ws = _workspace(L.ddm_radix_sort_workspace_bytes(n), keys.device)
    _check(L.ddm_radix_sort_u64(keys.data_ptr(), vals.data_ptr() if vals is not None else None, ko.data_ptr(),
                                vo.data_ptr() if vo is not None else None, n, begin_bit, end_bit, ws.data_ptr(),
                                ws.numel(), _stream(keys.device)), "ddm_radix_sort_u64")
    return ko, vo


def encode_keys(x: torch.Tensor) -> torch.Tensor:
    L = load()
    out = torch.empty(x.numel(), dtype=torch.int64, device=x.device)
    _check(L.ddm_encode_keys(x.data_ptr(), out.data_ptr(), x.numel(), _stream(x.device)), "ddm_encode_keys")
    return out


def launch_count() -> int:
    return int(load().ddm_kernel_launch_count())


def build_info() -> str:
    return load().ddm_build_info().decode()


def profile_enable(on: bool = True) -> None:
    """Record CUDA events around every library launch (resets the record)."""
    load().ddm_profile_enable(1 if on else 0)


def profile_read() -> dict:
    """{kernel class: {"launches", "total_ms", "bytes"}} of the recorded launches."""
    L = load()
    buf = (_KernelStat * 64)()
    k = L.ddm_profile_read(buf, 64)
    if k < 0:
        raise DDMError(6, "ddm_profile_read")
    return {buf[i].name.decode(): {"launches": int(buf[i].launches), "total_ms": float(buf[i].total_ms),
                                   "bytes": float(buf[i].bytes)} for i in range(min(k, 64))}
