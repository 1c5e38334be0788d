"""More adversarial inputs (dev tool): exact K vs the oracle's rank identity / brute force, no CUDA errors."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1703_06680_b200 import ddm
import oracle as orc
rng = np.random.default_rng(5)
def run(name, sl, sh, ul, uh, bf=False):
    a = [np.ascontiguousarray(x if x.ndim == 2 else x[None]) for x in (sl, sh, ul, uh)]
    g = [torch.from_numpy(x).cuda() for x in a]
    t = time.time()
    try:
        K = ddm.match_count(*g)
        ref = orc.bf_count(*a) if bf else (orc.rank_count(*a) if a[0].shape[0] == 1 else K)
        res = []
        for f in (0, ddm.DDM_SORT_LSB, ddm.DDM_COUNT_WALK):
            p = ddm.match_pairs(*g, flags=f)
            res.append(p.shape[0] == K)
            del p
        idx = ddm.sub_index_build(g[0], g[1])
        ki = ddm.match_count_indexed(idx, a[0].shape[1], g[2], g[3])
        ev = ddm.match_pairs_events(*g).shape[0] if K < 5e7 else K
        ok = K == ref and all(res) and ki == K and ev == K
        print(f"{name}: K={K} ref={ref} idx={ki} ev={ev} {'OK' if ok else 'MISMATCH ' + str(res)} {time.time()-t:.1f}s", flush=True)
    except Exception as e:  # noqa: BLE001
        print(f"{name}: ERROR {e}", flush=True)
    torch.cuda.empty_cache()
d3 = lambda cnt: rng.integers(-5, 5, (3, cnt)).astype(float)
A = d3(20000); B = d3(300)
run("d=3 heavy ties, few updates", A, A + 1, B, B + 1, bf=True)
run("d=3 heavy ties, few subs", B, B + 1, A, A + 1, bf=True)
x = rng.uniform(0, 1e6, 2_000_000)
run("n=1 vs 2e6", np.array([0.0]), np.array([1e6]), x, x + 1)
run("2e6 vs m=1", x, x + 1, np.array([5e5]), np.array([5e5 + 100]))
s = np.zeros(100_000); run("all subs identical long, 1e3 updates", s, s + 1e6, x[:1000], x[:1000] + 1)
L = rng.uniform(0, 1e4, (2, 1_000_000)); run("d=2 long tails", L, L + np.where(rng.random((2, 1_000_000)) < 0.001, 5e3, 5.0), L[:, ::-1].copy(), L[:, ::-1] + 5.0)
e = np.empty(0); run("empty subs", e, e, x[:10], x[:10] + 1)
run("empty upds", x[:10], x[:10] + 1, e, e)
