"""Multi-GPU orchestration on CPU: world_size 2 and 3, gloo backend.

The REAL SlabMatcher.step / ShardedMatcher.step collective sequences of
paper_1703_06680_b200.dist run here over gloo.  The device work of the slab
mode is swapped for `NumpyOps` (tests/dist_workers.py): a numpy stand-in of
ddm_slab_sample / _cuts / _pack / _unpack with the oracle as the matcher, so
these tests pin the host logic -- sampling, cut points, reach all-reduce,
count and row all_to_all, id bookkeeping, the K all-reduce.  The union of the
per-rank lists must equal the single-process oracle list with no pair twice
(G-invariance).  The same step with the libddm ops runs on the
GPU in tests/test_parity.py::test_slab_matcher_two_processes_one_gpu.
"""
import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1703_06680_b200 import workload as wl
from tests import dist_workers as dw


def _run(world, fn, *args):
    port = dw.free_port()
    mp.spawn(fn, args=(world, port) + args, nprocs=world, join=True)


@pytest.mark.parametrize("world", [2, 3])
def test_slab_step_equal_single(tmp_path, world):
    """Slab mode (fully distributed index) over gloo with the numpy ops: each
    rank starts with an index block of both kinds; the partition, halo and
    exchange give every pair exactly once, on its update's rank."""
    import oracle
    _run(world, dw.slab_worker_cpu, str(tmp_path), "clustered")
    w = dw.instance("clustered")
    ref = oracle.bf_pairs(w.sub_lo, w.sub_hi, w.upd_lo, w.upd_hi)
    parts = [np.load(tmp_path / f"slab_pairs_{r}.npy") for r in range(world)]
    got = np.concatenate(parts)
    assert got.size == ref.size and np.array_equal(np.sort(got), ref)
    for r in range(world):
        assert int(np.load(tmp_path / f"slab_k_{r}.npy")[0]) == ref.size   # all-reduced count
    assert all(p.size > 0 for p in parts)  # every slab did work


def test_slab_step_long_intervals_and_d2(tmp_path):
    """Subscriptions spanning every cut (halos on every rank), point extents
    and d = 2."""
    import oracle
    _run(2, dw.slab_worker_cpu, str(tmp_path), "long_d2")
    w = dw.instance("long_d2")
    ref = oracle.bf_pairs(w.sub_lo, w.sub_hi, w.upd_lo, w.upd_hi)
    got = np.sort(np.concatenate([np.load(tmp_path / f"slab_pairs_{r}.npy") for r in range(2)]))
    assert np.array_equal(got, ref)


def test_broadcast_step_equal_single(tmp_path):
    """Broadcast mode over gloo: rank 0's index (stand-in: the serialised
    subscription arrays) is broadcast, every rank matches its update block."""
    import oracle
    _run(2, dw.broadcast_worker_cpu, str(tmp_path))
    w = dw.instance("clustered")
    ref = oracle.bf_pairs(w.sub_lo, w.sub_hi, w.upd_lo, w.upd_hi)
    got = np.sort(np.concatenate([np.load(tmp_path / f"bc_pairs_{r}.npy") for r in range(2)]))
    assert np.array_equal(got, ref)
    for r in range(2):
        assert int(np.load(tmp_path / f"bc_k_{r}.npy")[0]) == ref.size


def test_numpy_cuts_balance_and_ties():
    """The cut rule (quantiles of the finite gathered samples): balanced on
    distinct values, a partition under heavy ties, NaN samples ignored."""
    ops = dw.NumpyOps(1)
    rng = np.random.default_rng(0)
    lo = rng.uniform(0, 1e6, 100_000)
    for world in (1, 2, 3, 8):
        cuts = ops.cuts_np(np.sort(lo), world)
        assert cuts.size == world - 1 and np.all(np.diff(cuts) >= 0)
        counts = np.bincount(np.searchsorted(cuts, lo, side="right"), minlength=world)
        assert counts.sum() == lo.size and counts.max() - counts.min() <= 2
    ties = np.repeat(np.arange(10.0), 1000)
    cuts = ops.cuts_np(np.concatenate([ties, [np.nan] * 50]), 4)
    assert np.bincount(np.searchsorted(cuts, ties, side="right"), minlength=4).sum() == ties.size
