"""d=2, n >> m: tiled filter vs per-row paths (dev tool)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1703_06680_b200 import ddm
rng = np.random.default_rng(3)
for n, m in ((4_000_000, 2000), (4_000_000, 50_000), (4_000_000, 200_000), (1_000_000, 1_000_000)):
    A = rng.uniform(0, 1e4, (2, n)); B = rng.uniform(0, 1e4, (2, m))
    g = [torch.from_numpy(x).cuda() for x in (A, A + 20.0, B, B + 20.0)]
    for f in (0, ddm.DDM_EMIT_FORCE_WARP, ddm.DDM_EMIT_FORCE_THREAD):
        for _ in range(2):
            torch.cuda.synchronize(); t = time.time(); p = ddm.match_pairs(*g, flags=f); torch.cuda.synchronize(); dt = time.time() - t
        print(f"n={n} m={m} flags={f:#x}: K={p.shape[0]} {dt*1e3:.1f} ms", flush=True)
