"""Process entry points and stand-ins for the multi-process dist tests.

NumpyOps implements the slab mode's device operations (ddm_slab_sample,
ddm_slab_cuts, ddm_slab_pack, ddm_slab_unpack, the match) in numpy with the
CPU oracle as the matcher, following the rules stated in include/ddm.h, so
SlabMatcher.step's collective sequence can run over gloo on CPU.  Test
infrastructure only.
"""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist

from paper_1703_06680_b200 import workload as wl


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def instance(kind: str):
    if kind == "clustered":
        return wl.clustered(3000, 3500, 1e6, 2000.0, seed=19)
    if kind == "long_d2":
        w = wl.uniform(2500, 2700, 1e4, 90.0, 2, seed=23)
        sl, sh, ul, uh = w.sub_lo.copy(), w.sub_hi.copy(), w.upd_lo.copy(), w.upd_hi.copy()
        sl[0, :9], sh[0, :9] = -5.0, 2e4   # cross every cut
        uh[:, :40] = ul[:, :40]            # point extents
        return wl.Workload("long_d2", 2, w.L, w.l, 0, sl, sh, ul, uh)
    if kind == "gpu":
        w = wl.clustered(60_000, 70_000, 1e7, 4000.0, seed=41)
        sl, sh = w.sub_lo.copy(), w.sub_hi.copy()
        sl[0, :11], sh[0, :11] = -1.0, 2e7
        return wl.Workload("gpu", 1, w.L, w.l, 0, sl, sh, w.upd_lo, w.upd_hi)
    raise ValueError(kind)


def block(count, rank, world):
    return count * rank // world, count * (rank + 1) // world


class NumpyOps:
    """numpy stand-in of dist.DeviceOps (CPU float64 tensors)."""

    def __init__(self, d):
        self.d = d

    def sample(self, lo0, s):
        x = lo0.numpy()
        if x.size == 0:
            return torch.full((s,), float("nan"), dtype=torch.float64)
        return torch.from_numpy(x[(np.arange(s, dtype=np.int64) * x.size) // s].copy())

    @staticmethod
    def cuts_np(samples, world):
        v = np.sort(samples[np.isfinite(samples)])
        if world <= 1:
            return np.zeros(0)
        if v.size == 0:
            return np.zeros(world - 1)
        return np.array([v[min(r * v.size // world, v.size - 1)] for r in range(1, world)])

    def cuts(self, samples, world):
        return torch.from_numpy(self.cuts_np(samples.numpy(), world))

    @staticmethod
    def _key_signed(x):
        b = np.asarray(x, dtype=np.float64).copy()
        b[b == 0] = 0.0
        u = b.view(np.uint64)
        k = np.where(u >> np.uint64(63), ~u, u | np.uint64(1 << 63))
        return (k ^ np.uint64(1 << 63)).view(np.int64)

    def pack(self, side, lo, hi, id_base, cuts, world, reach=None):
        lo, hi, c = lo.numpy(), hi.numpy(), cuts.numpy()
        n = lo.shape[1]
        dests = []
        reach_out = np.full(world, np.iinfo(np.int64).min, dtype=np.int64)
        for i in range(n):
            if side == 1:
                r = int(np.searchsorted(c, lo[0, i], side="right"))
                dests.append([r])
                reach_out[r] = max(reach_out[r], self._key_signed([hi[0, i]])[0])
            else:
                lk = self._key_signed([lo[0, i]])[0]
                ds = [r for r in range(world) if (r == 0 or hi[0, i] >= c[r - 1]) and lk <= int(reach[r])]
                dests.append(ds)
        rows, counts = [], []
        for r in range(world):
            idx = [i for i in range(n) if r in dests[i]]
            counts.append(len(idx))
            for i in idx:
                rows.append(np.concatenate([lo[:, i], hi[:, i], [np.uint64(id_base + i).view(np.float64)]]))
        arr = np.array(rows, dtype=np.float64).reshape(-1, 2 * self.d + 1)
        return torch.from_numpy(arr), counts, (torch.from_numpy(reach_out) if side == 1 else None)

    def unpack(self, rows):
        a = rows.numpy()
        lo = np.ascontiguousarray(a[:, : self.d].T)
        hi = np.ascontiguousarray(a[:, self.d: 2 * self.d].T)
        ids = a[:, 2 * self.d].copy().view(np.uint64).astype(np.int64)
        return torch.from_numpy(lo), torch.from_numpy(hi), torch.from_numpy(ids)

    def match(self, sl, sh, sids, ul, uh, uids, flags=0):
        import oracle
        p = oracle.bf_pairs(sl.numpy(), sh.numpy(), ul.numpy(), uh.numpy())
        s = sids.numpy()[(p & np.uint64(0xFFFFFFFF)).astype(np.int64)].astype(np.uint64)
        u = uids.numpy()[(p >> np.uint64(32)).astype(np.int64)].astype(np.uint64)
        words = (u << np.uint64(32)) | s
        return torch.from_numpy(words.view(np.int64)), int(p.size)


def _init(rank, world, port, backend="gloo"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group(backend, rank=rank, world_size=world)


def slab_worker_cpu(rank, world, port, out_dir, kind):
    from paper_1703_06680_b200 import dist as ddist
    _init(rank, world, port)
    w = instance(kind)
    s0, s1 = block(w.n, rank, world)
    u0, u1 = block(w.m, rank, world)
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a))  # noqa: E731
    SM = ddist.SlabMatcher(w.d, "cpu", ops=NumpyOps(w.d))
    res = SM.step(T(w.sub_lo[:, s0:s1]), T(w.sub_hi[:, s0:s1]), s0, T(w.upd_lo[:, u0:u1]), T(w.upd_hi[:, u0:u1]), u0)
    np.save(os.path.join(out_dir, f"slab_pairs_{rank}.npy"), res.pairs.numpy().view(np.uint64))
    np.save(os.path.join(out_dir, f"slab_k_{rank}.npy"), np.array([res.k_total]))
    dist.destroy_process_group()


def broadcast_worker_cpu(rank, world, port, out_dir):
    """ShardedMatcher.step's sequence with a stand-in index and matcher."""
    import oracle
    from paper_1703_06680_b200 import dist as ddist
    _init(rank, world, port)
    w = instance("clustered")
    u0, u1 = block(w.m, rank, world)
    C = ddist.Coll()
    index = torch.zeros(2 * w.n, dtype=torch.float64)
    if rank == 0:
        index.copy_(torch.from_numpy(np.concatenate([w.sub_lo[0], w.sub_hi[0]])))
    C.broadcast_(index, src=0)
    arr = index.numpy()
    p = oracle.bf_pairs(arr[: w.n][None], arr[w.n:][None], w.upd_lo[:, u0:u1], w.upd_hi[:, u0:u1])
    glob = (((p >> np.uint64(32)) + np.uint64(u0)) << np.uint64(32)) | (p & np.uint64(0xFFFFFFFF))
    k = torch.tensor([p.size], dtype=torch.int64)
    C.all_reduce_(k, dist.ReduceOp.SUM)
    np.save(os.path.join(out_dir, f"bc_pairs_{rank}.npy"), glob)
    np.save(os.path.join(out_dir, f"bc_k_{rank}.npy"), np.array([int(k.item())]))
    dist.destroy_process_group()


def slab_worker_gpu(rank, world, port, out_dir, kind):
    """The real slab step (libddm DeviceOps) with `world` processes sharing
    cuda:0 over gloo (Coll stages the collectives through host memory)."""
    from paper_1703_06680_b200 import dist as ddist
    _init(rank, world, port)
    torch.cuda.set_device(0)
    w = instance(kind)
    s0, s1 = block(w.n, rank, world)
    u0, u1 = block(w.m, rank, world)
    C = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    SM = ddist.SlabMatcher(w.d, "cuda:0")
    for _ in range(2):  # a second step reuses the grown buffers
        res = SM.step(C(w.sub_lo[:, s0:s1]), C(w.sub_hi[:, s0:s1]), s0, C(w.upd_lo[:, u0:u1]),
                      C(w.upd_hi[:, u0:u1]), u0)
    p = res.pairs.cpu().numpy().astype(np.uint32)
    words = (p[:, 1].astype(np.uint64) << np.uint64(32)) | p[:, 0].astype(np.uint64)
    np.save(os.path.join(out_dir, f"g_pairs_{rank}.npy"), words)
    np.save(os.path.join(out_dir, f"g_k_{rank}.npy"), np.array([res.k_total]))
    dist.destroy_process_group()


def broadcast_worker_gpu(rank, world, port, out_dir, kind):
    """The real broadcast step (libddm index build + indexed match)."""
    from paper_1703_06680_b200 import ddm
    from paper_1703_06680_b200 import dist as ddist
    _init(rank, world, port)
    torch.cuda.set_device(0)
    w = instance(kind)
    u0, u1 = block(w.m, rank, world)
    C = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    sub = [C(w.sub_lo), C(w.sub_hi)]
    ul, uh = C(w.upd_lo[:, u0:u1]), C(w.upd_hi[:, u0:u1])
    uid = torch.arange(u0, u1, dtype=torch.int32, device="cuda")
    cap = ddm.match_count(sub[0], sub[1], ul, uh)
    SM = ddist.ShardedMatcher(w.d, w.n, u1 - u0, cap, "cuda:0")
    res = SM.step(sub[0], sub[1], ul, uh, uid)
    p = res.pairs.cpu().numpy().astype(np.uint32)
    words = (p[:, 1].astype(np.uint64) << np.uint64(32)) | p[:, 0].astype(np.uint64)
    np.save(os.path.join(out_dir, f"gb_pairs_{rank}.npy"), words)
    np.save(os.path.join(out_dir, f"gb_k_{rank}.npy"), np.array([res.k_total]))
    dist.destroy_process_group()
