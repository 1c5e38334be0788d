"""Multi-GPU host logic on CPU: world_size 2, gloo backend.

The device kernels are not exercised here (no GPU); a stand-in "index" (the
sorted subscription arrays serialised to bytes) and a stand-in matcher (the
CPU oracle on the rank's slab) drive the same collective sequence and slab
bookkeeping as paper_1703_06680_b200.dist, and the union of the per-rank
lists must equal the single-process oracle list (G-invariance).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1703_06680_b200 import dist as ddist
from paper_1703_06680_b200 import workload as wl


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    import oracle
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w = wl.uniform(3000, 4000, 1e5, 40.0, 1, seed=17)
    ul, uh, ids = ddist.local_updates(w.upd_lo, w.upd_hi, rank, world)
    nbytes = w.n * 16

    def build():
        return torch.from_numpy(np.concatenate([w.sub_lo[0], w.sub_hi[0]]).view(np.uint8).copy())

    def match(index):
        arr = index.numpy().view(np.float64)
        sl, sh = arr[: w.n][None], arr[w.n:][None]
        p = oracle.bf_pairs(sl, sh, ul, uh)
        upd_local = (p >> np.uint64(32)).astype(np.int64)
        sub = p & np.uint64(0xFFFFFFFF)
        glob = (ids[upd_local].astype(np.uint64) << np.uint64(32)) | sub  # global update ids
        return glob, int(p.size)

    pairs, k_total = ddist.run_sharded(build, match, rank, world, nbytes)
    np.save(os.path.join(out_dir, f"pairs_{rank}.npy"), pairs)
    np.save(os.path.join(out_dir, f"k_{rank}.npy"), np.array([k_total]))
    dist.destroy_process_group()


def test_sharded_two_ranks_equal_single(tmp_path):
    import oracle
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    w = wl.uniform(3000, 4000, 1e5, 40.0, 1, seed=17)
    ref = oracle.bf_pairs(w.sub_lo, w.sub_hi, w.upd_lo, w.upd_hi)
    parts = [np.load(tmp_path / f"pairs_{r}.npy") for r in range(world)]
    got = np.sort(np.concatenate(parts))
    assert np.array_equal(got, ref)
    for r in range(world):
        assert int(np.load(tmp_path / f"k_{r}.npy")[0]) == ref.size   # all-reduced count on every rank
    assert all(p.size > 0 for p in parts)  # both slabs did work


def test_slab_cuts_balance_and_cover():
    rng = np.random.default_rng(0)
    lo = rng.uniform(0, 1e6, 100_000)
    for world in (1, 2, 3, 8):
        cuts = ddist.slab_cuts(lo, world)
        assert cuts.size == max(world - 1, 0) and np.all(np.diff(cuts) >= 0)
        s = ddist.slab_of(lo, cuts)
        counts = np.bincount(s, minlength=world)
        assert counts.sum() == lo.size and counts.size == world
        assert counts.max() - counts.min() <= 2
    # every update lands in exactly one slab, ids preserved
    lo2 = lo[None]
    hi2 = lo2 + 1
    seen = np.concatenate([ddist.local_updates(lo2, hi2, r, 3)[2] for r in range(3)])
    assert np.array_equal(np.sort(seen), np.arange(lo.size))


def test_slab_cuts_with_ties():
    lo = np.repeat(np.arange(10.0), 1000)  # heavy ties: slabs may be unequal but must partition
    cuts = ddist.slab_cuts(lo, 4)
    s = ddist.slab_of(lo, cuts)
    assert np.bincount(s, minlength=4).sum() == lo.size


def _slab_worker(rank, world, port, out_dir):
    import oracle
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w = wl.clustered(3000, 3500, 1e6, 2000.0, seed=19)
    sl, sh, sids, ul, uh, uids = ddist.slab_partition(w, rank, world)
    p = oracle.bf_pairs(sl, sh, ul, uh)   # stand-in for ddm_match_pairs_mapped on this rank's partition
    glob = (uids[(p >> np.uint64(32)).astype(np.int64)].astype(np.uint64) << np.uint64(32)) | \
        sids[(p & np.uint64(0xFFFFFFFF)).astype(np.int64)].astype(np.uint64)
    k = torch.tensor([p.size], dtype=torch.int64)
    dist.all_reduce(k, op=dist.ReduceOp.SUM)   # the slab mode's only collective
    np.save(os.path.join(out_dir, f"slab_pairs_{rank}.npy"), glob)
    np.save(os.path.join(out_dir, f"slab_k_{rank}.npy"), np.array([int(k.item())]))
    dist.destroy_process_group()


def test_slab_mode_two_ranks_equal_single(tmp_path):
    """Slab mode (fully distributed index): each rank holds its updates and the
    subscriptions that can reach them (halo); the union of the per-rank lists
    is the single-process list, with no pair reported twice."""
    import oracle
    world = 2
    mp.spawn(_slab_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    w = wl.clustered(3000, 3500, 1e6, 2000.0, seed=19)
    ref = oracle.bf_pairs(w.sub_lo, w.sub_hi, w.upd_lo, w.upd_hi)
    parts = [np.load(os.path.join(tmp_path, f"slab_pairs_{r}.npy")) for r in range(world)]
    got = np.sort(np.concatenate(parts))
    assert np.array_equal(got, ref)
    for r in range(world):
        assert int(np.load(os.path.join(tmp_path, f"slab_k_{r}.npy"))[0]) == ref.size


def test_slab_partition_covers_every_pair():
    """Host logic only: for G slabs the partitions' subscription sets contain
    every partner of every update of the slab (brute-force check)."""
    import oracle
    w = wl.uniform(1500, 1700, 1e4, 60.0, 1, seed=23)
    sl, sh = w.sub_lo.copy(), w.sub_hi.copy()
    sl[0, :5], sh[0, :5] = 0.0, 1e4  # long intervals cross every cut
    w2 = wl.Workload("t", 1, w.L, w.l, 0, sl, sh, w.upd_lo, w.upd_hi)
    ref = oracle.bf_pairs(sl, sh, w.upd_lo, w.upd_hi)
    for G in (1, 3, 5):
        allp = []
        for r in range(G):
            psl, psh, sids, ul, uh, uids = ddist.slab_partition(w2, r, G)
            p = oracle.bf_pairs(psl, psh, ul, uh)
            allp.append((uids[(p >> np.uint64(32)).astype(np.int64)].astype(np.uint64) << np.uint64(32))
                        | sids[(p & np.uint64(0xFFFFFFFF)).astype(np.int64)].astype(np.uint64))
        assert np.array_equal(np.sort(np.concatenate(allp)), ref), f"G={G}"
