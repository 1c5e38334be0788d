"""Quick timing of match_pairs on a BASELINE config (dev tool)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1703_06680_b200 import ddm, workload as wl

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
t0 = time.time()
w = wl.make(cfg, scale)
print(f"gen {cfg}@{scale}: {time.time()-t0:.1f}s n={w.n}", flush=True)
g = [torch.from_numpy(a).cuda() for a in (w.sub_lo, w.sub_hi, w.upd_lo, w.upd_hi)]
M = ddm.Matcher(w.d, w.n, w.m)
K = M.count(*g)
out = torch.empty((K, 2), dtype=torch.int32, device="cuda")
for flags in (0, ddm.DDM_EMIT_FORCE_CHUNK, ddm.DDM_EMIT_FORCE_THREAD, ddm.DDM_EMIT_FORCE_WARP):
    for i in range(3):
        M.pairs_into(out, *g, flags=flags)
    torch.cuda.synchronize()
    ts = []
    for i in range(5):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); M.pairs_into(out, *g, flags=flags); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    t = np.median(ts)
    ddm.profile_enable(True)
    M.pairs_into(out, *g, flags=flags)
    pr = ddm.profile_read()
    ddm.profile_enable(False)
    print("   emit ms:", round(pr.get("emit", {}).get("total_ms", 0.0), 3))
    print(f"{cfg} flags={flags} K={K} pairs: {t:.3f} ms  regions/s={(w.n+w.m)/t*1e3:.3e} pairs/s={K/t*1e3:.3e}", flush=True)
ts = []
for i in range(5):
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); M.count(*g); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
print(f"{cfg} count: {np.median(ts):.3f} ms", flush=True)
