"""A/B timing of pairs calls under two flag sets (dev tool): median device time, no profiling.
usage: ab_flags.py cfg[,cfg...] reps flagsA flagsB"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1703_06680_b200 import ddm, workload as wl

cfgs = sys.argv[1].split(",")
reps = int(sys.argv[2])
fl = [int(eval(x, {"ddm": ddm})) for x in sys.argv[3:]] or [0]
for cfg in cfgs:
    w = wl.make(cfg, 1.0)
    g = [torch.from_numpy(a).cuda() for a in (w.sub_lo, w.sub_hi, w.upd_lo, w.upd_hi)]
    M = ddm.Matcher(w.d, w.n, w.m)
    K = M.count(*g)
    out = torch.empty((max(K, 1), 2), dtype=torch.int32, device="cuda")
    res = {}
    for f in fl:
        for _ in range(3):
            M.pairs_into(out, *g, flags=f)
        ts = []
        for _ in range(reps):
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(); M.pairs_into(out, *g, flags=f); b.record(); torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        res[f] = float(np.median(ts))
    print(cfg, f"K={K}", "  ".join(f"flags={f:#x}: {t:.3f} ms" for f, t in res.items()), flush=True)
    del M, out, g
    torch.cuda.empty_cache()
