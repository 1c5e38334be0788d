"""Seeded synthetic DDM workloads (the paper's generator, §5).

This module holds *only* random draws and the stored `hi = lo + l` add; it
contains none of the matching arithmetic, so both the CUDA path and the CPU
oracle (`oracle/`) may consume its arrays (DESIGN.md §3 "input recipe").

Recipe (BASELINE.json configs):
  * n = m = N/2 regions per kind; equal length l = alpha*L/N
    (P:903-908); lower bound uniform in [0, L-l) so every extent lies inside
    the routing space.
  * d > 1 (config c4): independent per-dimension placement with the side
    l = L*(alpha/N)^(1/d) (volume overlap degree, reading R15).
  * c5: 64-component Gaussian mixture (sigma = 1e6) of lower bounds with
    lengths ~ U[0.5 l, 1.5 l); out-of-domain draws are resampled.
  * numpy PCG64 (`numpy.random.default_rng(seed)`), float64 throughout; draw
    order: subscriptions then updates, within each dim 0..d-1.

Arrays are returned as float64 numpy arrays of shape [d, count] (SoA per
dimension), the layout the C ABI takes (include/ddm.h, `ddm_regions`).
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

__all__ = ["Workload", "CONFIGS", "make", "uniform", "clustered", "window_sample",
           "expected_pairs_uniform"]


@dataclasses.dataclass
class Workload:
    name: str
    d: int
    L: float
    l: float
    seed: int
    sub_lo: np.ndarray  # [d, n] float64
    sub_hi: np.ndarray  # [d, n]
    upd_lo: np.ndarray  # [d, m]
    upd_hi: np.ndarray  # [d, m]

    @property
    def n(self) -> int:
        return int(self.sub_lo.shape[1])

    @property
    def m(self) -> int:
        return int(self.upd_lo.shape[1])

    def describe(self) -> dict:
        return {"workload": self.name, "d": self.d, "n_sub": self.n, "n_upd": self.m,
                "L": self.L, "l": self.l, "seed": self.seed, "rng": "numpy PCG64 " + np.__version__}


# BASELINE.json configs[0..4].
CONFIGS = {
    "c1": dict(kind="uniform", d=1, n=5_000, L=1e6, alpha=1.0, seed=0),
    "c2": dict(kind="uniform", d=1, n=500_000, L=1e6, alpha=100.0, seed=1),
    "c3": dict(kind="uniform", d=1, n=50_000_000, L=1e8, alpha=1.0, seed=2),
    "c4": dict(kind="uniform", d=3, n=5_000_000, L=1e4, alpha=1.0, seed=3),
    "c5": dict(kind="clustered", d=1, n=500_000_000, L=1e9, alpha=0.01, seed=4),
}


def side_length(N: int, L: float, alpha: float, d: int) -> float:
    """l = alpha*L/N for d=1; l = L*(alpha/N)^(1/d) for d>1."""
    if d == 1:
        return alpha * L / N
    return L * (alpha / N) ** (1.0 / d)


def uniform(n: int, m: int, L: float, l: float, d: int = 1, seed: int = 0,
            name: str = "uniform") -> Workload:
    """Paper §5 generator: equal lengths, uniformly placed inside [0, L)."""
    if not (0.0 < l < L):
        raise ValueError("extent length must satisfy 0 < l < L (SPEC S:343)")
    rng = np.random.default_rng(seed)
    out = {}
    for kind, cnt in (("sub", n), ("upd", m)):
        lo = np.empty((d, cnt), dtype=np.float64)
        for k in range(d):
            lo[k] = rng.uniform(0.0, L - l, cnt)
        out[kind] = (lo, lo + l)  # one IEEE add, stored (reading R13)
    return Workload(name, d, float(L), float(l), seed, out["sub"][0], out["sub"][1],
                    out["upd"][0], out["upd"][1])


_C5_CHUNK = 1 << 24


def clustered(n: int, m: int, L: float, l: float, seed: int, n_centres: int = 64,
              sigma: float = 1e6, name: str = "clustered") -> Workload:
    """c5 recipe: Gaussian-mixture lower bounds, lengths ~ U[0.5l, 1.5l),
    out-of-domain draws resampled in ascending index order."""
    rng = np.random.default_rng(seed)
    centres = rng.uniform(0.0, L, n_centres)
    out = {}
    for kind, cnt in (("sub", n), ("upd", m)):
        lo_all = np.empty((1, cnt), dtype=np.float64)
        hi_all = np.empty((1, cnt), dtype=np.float64)
        for start in range(0, cnt, _C5_CHUNK):
            c = min(_C5_CHUNK, cnt - start)
            comp = rng.integers(0, n_centres, c)
            lo = rng.normal(centres[comp], sigma)
            ln = rng.uniform(0.5 * l, 1.5 * l, c)
            bad = np.nonzero((lo < 0.0) | (lo + ln >= L))[0]
            while bad.size:
                comp_b = rng.integers(0, n_centres, bad.size)
                lo[bad] = rng.normal(centres[comp_b], sigma)
                ln[bad] = rng.uniform(0.5 * l, 1.5 * l, bad.size)
                bad = bad[(lo[bad] < 0.0) | (lo[bad] + ln[bad] >= L)]
            lo_all[0, start:start + c] = lo
            hi_all[0, start:start + c] = lo + ln
        out[kind] = (lo_all, hi_all)
    return Workload(name, 1, float(L), float(l), seed, out["sub"][0], out["sub"][1],
                    out["upd"][0], out["upd"][1])


def make(name: str, scale: float = 1.0, alpha: float | None = None) -> Workload:
    """Build BASELINE config `name` (c1..c5).  `scale` < 1 shrinks n and m while
    keeping L, alpha and the seed's recipe (used only by tests and samples);
    `alpha` replaces the config's overlap degree (the paper's K-independence
    sweep of count mode)."""
    cfg = CONFIGS[name]
    n = max(1, int(round(cfg["n"] * scale)))
    N = 2 * cfg["n"]
    a = cfg["alpha"] if alpha is None else float(alpha)
    l = side_length(N, cfg["L"], a, cfg["d"])
    tag = name if scale == 1.0 else f"{name}@{scale:g}"
    if alpha is not None:
        tag += f"[alpha={a:g}]"
    if cfg["kind"] == "uniform":
        return uniform(n, n, cfg["L"], l, cfg["d"], cfg["seed"], name=tag)
    return clustered(n, n, cfg["L"], l, cfg["seed"], name=tag)


def window_sample(w: Workload, frac: float) -> Workload:
    """The regions whose dim-0 lower bound lies in a window of width frac*L
    centred on the median subscription lower bound: same local density and
    alpha, a bounded slice of the workload (the CPU-baseline sample).  For the
    uniform configs that is ~frac of the regions; for the clustered c5 the
    window sits inside the populated part of the domain."""
    x0 = float(np.median(w.sub_lo[0])) - 0.5 * frac * w.L if w.n else 0.0
    x1 = x0 + frac * w.L
    s = (w.sub_lo[0] >= x0) & (w.sub_lo[0] < x1)
    u = (w.upd_lo[0] >= x0) & (w.upd_lo[0] < x1)
    return Workload(f"{w.name}[{x0:.6g}<=lo<{x1:.6g}]", w.d, w.L, w.l, w.seed,
                    np.ascontiguousarray(w.sub_lo[:, s]), np.ascontiguousarray(w.sub_hi[:, s]),
                    np.ascontiguousarray(w.upd_lo[:, u]), np.ascontiguousarray(w.upd_hi[:, u]))


def expected_pairs_uniform(n: int, m: int, L: float, l: float, d: int = 1) -> float:
    """E[K] for equal lengths l placed uniformly in [0, L-l): two such
    intervals overlap iff |lo_s - lo_u| <= l, probability p = 2r - r^2 with
    r = l/(L-l); dimensions independent (SURVEY §8(c) closed form)."""
    r = l / (L - l)
    p = 2.0 * r - r * r
    return n * m * p ** d


def stddev_bound(mean: float) -> float:
    return math.sqrt(max(mean, 1.0))
