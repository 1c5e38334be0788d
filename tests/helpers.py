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
