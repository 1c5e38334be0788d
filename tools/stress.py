"""Adversarial inputs at ~1e7 regions (dev tool): counts against the oracle's
rank identity, pairs K and invariants, both count forms, LSB fallback."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1703_06680_b200 import ddm
import oracle as orc

rng = np.random.default_rng(11)
N = 5_000_000
def case(name, sl, sh, ul, uh):
    g = [torch.from_numpy(np.ascontiguousarray(x[None])).cuda() for x in (sl, sh, ul, uh)]
    t0 = time.time()
    ref = orc.rank_count(sl[None], sh[None], ul[None], uh[None])
    K = ddm.match_count(*g)
    ok = K == ref
    msg = f"{name}: K={K} ref={ref} {'OK' if ok else 'MISMATCH'}"
    if ok and K <= 3e8:
        for f in (0, ddm.DDM_COUNT_WALK, ddm.DDM_COUNT_RANKS):
            p = ddm.match_pairs(*g, flags=f)
            s, u = p[:, 0].long(), p[:, 1].long()
            good = p.shape[0] == K and bool(((g[0][0][s] <= g[3][0][u]) & (g[2][0][u] <= g[1][0][s])).all())
            msg += f" pairs[{f:#x}]={'OK' if good else 'BAD'}"
            del p, s, u
    print(msg, f"{time.time() - t0:.1f}s", flush=True)
    torch.cuda.empty_cache()

x = rng.uniform(0, 1e6, N)
case("all identical points", np.full(N, 5.0), np.full(N, 5.0), np.full(N // 100, 5.0), np.full(N // 100, 5.0))
case("few distinct values", rng.integers(0, 7, N).astype(float), rng.integers(7, 9, N).astype(float),
     rng.integers(0, 9, N // 50).astype(float), rng.integers(9, 12, N // 50).astype(float))
case("one long + sparse", np.r_[0.0, x[1:]], np.r_[2e6, x[1:] + 0.01], x, x + 0.01)
mm = np.sign(x - 5e5) * 10.0 ** rng.uniform(-300, 300, N)
um = np.sign(rng.uniform(-1, 1, N // 10)) * 10.0 ** rng.uniform(-300, 300, N // 10)
case("mixed magnitudes", mm, mm + np.abs(mm) * 1e-3, um, um + np.abs(um) * 1e-3)
lo = np.sort(rng.uniform(-1, 1, N)); case("sorted input, tiny lengths", lo, lo + 1e-9, lo[::-1].copy(), lo[::-1] + 1e-9)
c = rng.normal(0, 1e-3, N); case("single dense cluster", c, c + 1e-6, c[:N // 10].copy(), c[:N // 10] + 1e-6)
# asymmetric sizes and timing of the pairs path
def timed(name, sl, sh, ul, uh):
    g = [torch.from_numpy(np.ascontiguousarray(x if x.ndim == 2 else x[None])).cuda() for x in (sl, sh, ul, uh)]
    K = ddm.match_count(*g)
    ref = orc.rank_count(*(x if x.ndim == 2 else x[None] for x in (sl, sh, ul, uh))) if sl.ndim == 1 else K
    for _ in range(2):
        torch.cuda.synchronize(); t = time.time(); p = ddm.match_pairs(*g); torch.cuda.synchronize(); dt = time.time() - t
    print(f"{name}: K={K} ref={ref} pairs={p.shape[0]} {'OK' if p.shape[0] == K == ref else 'MISMATCH'} {dt*1e3:.1f} ms", flush=True)
    del p; torch.cuda.empty_cache()
a = rng.uniform(0, 1e6, 10_000_000); b = rng.uniform(0, 1e6, 1000)
timed("n >> m (1e7 vs 1e3)", a, a + 0.5, b, b + 0.5)
timed("n << m (1e3 vs 1e7)", b, b + 0.5, a, a + 0.5)
timed("n >> m, long updates", a, a + 0.5, b, b + 5e3)
A = rng.uniform(0, 1e4, (2, 4_000_000)); B = rng.uniform(0, 1e4, (2, 2000))
timed("d=2 n >> m", A, A + 20.0, B, B + 20.0)
timed("d=2 n << m", B, B + 20.0, A, A + 20.0)
s = np.sort(rng.normal(0, 1e6, 10_000_000)); timed("sorted clustered", s, s + 0.01, s[::-1].copy(), s[::-1] + 0.01)
