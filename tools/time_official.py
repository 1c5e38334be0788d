"""Official-style timing (no profiling, concurrent chains) of match_pairs on a config (dev tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1703_06680_b200 import ddm, workload as wl
cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
w = wl.make(cfg)
g = [torch.from_numpy(a).cuda() for a in (w.sub_lo, w.sub_hi, w.upd_lo, w.upd_hi)]
M = ddm.Matcher(w.d, w.n, w.m)
K = M.count(*g)
out = torch.empty((max(K, 1), 2), dtype=torch.int32, device="cuda")
for _ in range(3):
    M.pairs_into(out, *g)
torch.cuda.synchronize()
a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(reps):
    M.pairs_into(out, *g)
b.record(); torch.cuda.synchronize()
print(f"{cfg} env={os.environ.get('DDM_PASS_CTAS_PER_SM', '-')} serial={os.environ.get('DDM_SERIAL', '-')}: "
      f"{a.elapsed_time(b) / reps:.3f} ms/step K={K}", flush=True)
