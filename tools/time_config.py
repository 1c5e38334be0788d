"""Time one BASELINE config through the C ABI (dev tool): count + pairs, median of reps."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1703_06680_b200 import ddm, workload as wl

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
scale = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
t0 = time.time()
w = wl.make(cfg, scale)
print(f"gen {cfg}@{scale}: {time.time()-t0:.1f}s n={w.n} m={w.m} d={w.d}", flush=True)
g = [torch.from_numpy(a).cuda() for a in (w.sub_lo, w.sub_hi, w.upd_lo, w.upd_hi)]
M = ddm.Matcher(w.d, w.n, w.m)
t0 = time.time()
K = M.count(*g)
torch.cuda.synchronize()
print(f"first count K={K} in {time.time()-t0:.2f}s", flush=True)
out = torch.empty((max(K, 1), 2), dtype=torch.int32, device="cuda")
ddm.profile_enable(True)
ts = []
for i in range(reps):
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); M.pairs_into(out, *g); b.record(); torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
prof = ddm.profile_read()
ddm.profile_enable(False)
t = float(np.median(ts))
print(f"{cfg} K={K} pairs: median {t:.3f} ms over {reps} (all {['%.2f' % x for x in ts]}) "
      f"regions/s={(w.n + w.m) / t * 1e3:.3e} pairs/s={K / t * 1e3:.3e}", flush=True)
for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["total_ms"]):
    print(f"   {k:24s} {v['total_ms']/reps:9.3f} ms/step  x{v['launches']/reps:.0f}", flush=True)
