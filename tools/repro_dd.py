import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_1703_06680_b200 import ddm
from tests.helpers import cuda
rng = np.random.default_rng(33)
for d in (2, 3):
    n, m = 6000, 7000
    sl = rng.uniform(-500.0, 500.0, (d, n)); ul = rng.uniform(-500.0, 500.0, (d, m))
    sh = sl + rng.uniform(0.0, 120.0, (d, n)); uh = ul + rng.uniform(0.0, 120.0, (d, m))
    big = rng.choice(n, 40, replace=False)
    sl[:, big[:20]] = -1e4; sh[:, big[:20]] = 1e4
    sh[1, big[20:]] = sl[1, big[20:]] + 900.0
    pts = rng.choice(m, 50, replace=False); uh[:, pts] = ul[:, pts]
    for variant in range(4):
        a = [sl, sh, ul, uh]
        if variant == 1: a = [np.where(np.arange(n) < 0, 0, sl), sh, ul, uh]
        try:
            K = ddm.match_count(*[cuda(x) for x in a]); print(d, variant, "K", K, flush=True)
        except Exception as e:
            print(d, variant, "ERR", e, flush=True); raise
