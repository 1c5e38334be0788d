"""Time dense-overlap workloads (large alpha: big chunk-start sets) (dev tool)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1703_06680_b200 import ddm, workload as wl
for n, alpha in [(500_000, 100.0), (500_000, 400.0), (250_000, 2000.0), (100_000, 8000.0)]:
    N = 2 * n
    w = wl.uniform(n, n, 1e6, wl.side_length(N, 1e6, alpha, 1), 1, seed=1)
    g = [torch.from_numpy(a).cuda() for a in (w.sub_lo, w.sub_hi, w.upd_lo, w.upd_hi)]
    M = ddm.Matcher(1, n, n)
    K = M.count(*g)
    out = torch.empty((K, 2), dtype=torch.int32, device="cuda")
    for _ in range(2):
        M.pairs_into(out, *g)
    ddm.profile_enable(True)
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); M.pairs_into(out, *g); b.record(); torch.cuda.synchronize()
    pr = ddm.profile_read(); ddm.profile_enable(False)
    t = a.elapsed_time(b)
    print(f"n={n} alpha={alpha} K={K:.3e} step {t:.3f} ms  emit {pr['emit']['total_ms']:.3f} ms  pairs/s {K/t*1e3:.3e}", flush=True)
