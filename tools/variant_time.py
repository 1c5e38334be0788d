"""A/B timing of libddm builds (dev tool).  Run once per variant (DDM_LIB
selects the build): official-style step time (concurrent chains, graphs) of
match_pairs on a config, the per-kernel profile of one serialised step, and a
checksum of the pair list (must agree across variants).  Prints one JSON line."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1703_06680_b200 import ddm, workload as wl

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
mode = sys.argv[3] if len(sys.argv) > 3 else "pairs"
w = wl.make(cfg)
g = [torch.from_numpy(a).cuda() for a in (w.sub_lo, w.sub_hi, w.upd_lo, w.upd_hi)]
M = ddm.Matcher(w.d, w.n, w.m)
K = M.count(*g)
out = torch.zeros((max(K, 1), 2), dtype=torch.int32, device="cuda")
step = (lambda: M.pairs_into(out, *g)) if mode == "pairs" else (lambda: M.count(*g))
for _ in range(3):
    step()
torch.cuda.synchronize()
ts = []
for _ in range(reps):
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); step(); b.record(); torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
ddm.profile_enable(True)
step()
prof = ddm.profile_read()
ddm.profile_enable(False)
wd = out[:K].view(torch.int64)
chk = int((wd * 0x9E3779B97F4A7C15).sum().item()) if mode == "pairs" else K
print(json.dumps({"lib": os.environ.get("DDM_LIB", "default"), "cfg": cfg, "mode": mode, "K": K,
                  "median_ms": round(float(np.median(ts)), 4), "min_ms": round(float(np.min(ts)), 4),
                  "checksum": chk,
                  "prof": {k: [round(v["total_ms"], 4), v["launches"], round(v["bytes"] / max(v["total_ms"], 1e-9) / 1e6, 1)]
                           for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["total_ms"])}}), flush=True)
