"""Dynamic DDM timing (dev tool): ddm_sub_index_update of k moved subscriptions vs a full ddm_sub_index_build."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1703_06680_b200 import ddm, workload as wl
cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
w = wl.make(cfg, 1.0)
sl, sh = torch.from_numpy(w.sub_lo).cuda(), torch.from_numpy(w.sub_hi).cuda()
def t(f, reps=3):
    ts = []
    for _ in range(reps + 1):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); f(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    return float(np.median(ts[1:]))
idx = ddm.sub_index_build(sl, sh)
tb = t(lambda: ddm.sub_index_build(sl, sh))
print(f"{cfg} n={w.n}: full index build {tb:.3f} ms", flush=True)
rng = np.random.default_rng(0)
for frac in (0.0001, 0.001, 0.01, 0.1):
    k = max(1, int(w.n * frac))
    ids = torch.from_numpy(np.sort(rng.choice(w.n, k, replace=False)).astype(np.int32)).cuda()
    nl = sl[:, ids.long()] + 0.5
    nh = sh[:, ids.long()] + 0.5
    out = torch.empty_like(idx)
    tu = t(lambda: ddm.sub_index_update(idx, w.n, ids, nl, nh, out=out))
    ti = t(lambda: ddm.sub_index_update(idx, w.n, ids, nl, nh))
    print(f"  update k={k} ({frac:.2%}): ping-pong {tu:.3f} ms ({tb / tu:.1f}x faster than a rebuild), "
          f"in place {ti:.3f} ms", flush=True)
    del out
k = int(w.n * 0.001)
ids = torch.from_numpy(np.sort(rng.choice(w.n, k, replace=False)).astype(np.int32)).cuda()
nl = sl[:, ids.long()] + 0.5
nh = sh[:, ids.long()] + 0.5
ddm.profile_enable(True)
out = torch.empty_like(idx)
ddm.sub_index_update(idx, w.n, ids, nl, nh, out=out)
torch.cuda.synchronize()
prof = ddm.profile_read(); ddm.profile_enable(False)
for kk, v in sorted(prof.items(), key=lambda kv: -kv[1]["total_ms"]):
    print(f"   {kk:20s} {v['total_ms']:8.3f} ms x{v['launches']}", flush=True)
