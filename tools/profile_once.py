"""One warm-up + one timed match on a config (for ncu launch lists)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1703_06680_b200 import ddm, workload as wl
cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
w = wl.make(cfg, scale)
g = [torch.from_numpy(a).cuda() for a in (w.sub_lo, w.sub_hi, w.upd_lo, w.upd_hi)]
M = ddm.Matcher(w.d, w.n, w.m)
K = M.count(*g)
out = torch.empty((max(K, 1), 2), dtype=torch.int32, device="cuda")
M.pairs_into(out, *g)
torch.cuda.synchronize()
print("launches before timed call:", ddm.launch_count())
M.pairs_into(out, *g)
torch.cuda.synchronize()
print("K", K, "launches total:", ddm.launch_count())
