import sys, time; sys.path.insert(0, '.')
import numpy as np, torch
from paper_1703_06680_b200 import ddm
rng = np.random.default_rng(11); N = 5_000_000
lo = np.sort(rng.uniform(-1, 1, N))
for nm, (sl, sh, ul, uh) in {"sorted": (lo, lo + 1e-9, lo[::-1].copy(), lo[::-1] + 1e-9),
                             "random": (rng.permutation(lo), None, None, None)}.items():
    if sh is None:
        sl = sl; sh = sl + 1e-9; ul = rng.permutation(lo); uh = ul + 1e-9
    g = [torch.from_numpy(np.ascontiguousarray(x[None])).cuda() for x in (sl, sh, ul, uh)]
    for f in (0, ddm.DDM_COUNT_WALK, ddm.DDM_COUNT_RANKS, ddm.DDM_SORT_LSB):
        for rep in range(3):
            torch.cuda.synchronize(); t = time.time(); p = ddm.match_pairs(*g, flags=f); torch.cuda.synchronize(); dt = time.time() - t
        ddm.profile_enable(True); p = ddm.match_pairs(*g, flags=f); torch.cuda.synchronize(); pr = ddm.profile_read(); ddm.profile_enable(False)
        top = sorted(pr.items(), key=lambda kv: -kv[1]["total_ms"])[:3]
        print(nm, hex(f), f"{dt*1e3:.1f} ms", [(k, round(v["total_ms"], 2)) for k, v in top], flush=True)
