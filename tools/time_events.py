"""Time the event-order variant (ddm_match_pairs_events, Alg. 5 + 6) against the main path (dev tool)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1703_06680_b200 import ddm, workload as wl
for cfg in (sys.argv[1] if len(sys.argv) > 1 else "c2,c3").split(","):
    w = wl.make(cfg, 1.0)
    g = [torch.from_numpy(a).cuda() for a in (w.sub_lo, w.sub_hi, w.upd_lo, w.upd_hi)]
    L = ddm.load()
    r, keep = ddm.regions(*g)
    ws = torch.empty(L.ddm_events_workspace_bytes(r.d, r.n_sub, r.n_upd), dtype=torch.uint8, device="cuda")
    K = ctypes.c_uint64(0)
    st = torch.cuda.current_stream().cuda_stream
    s0 = L.ddm_match_pairs_events(ctypes.byref(r), None, 0, ctypes.byref(K), ws.data_ptr(), ws.numel(), st)
    print(cfg, "count status", s0, "K", K.value, "cuda", L.ddm_last_cuda_error(), flush=True)
    out = torch.empty((K.value, 2), dtype=torch.int32, device="cuda")
    ts = []
    for i in range(4):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record()
        s = L.ddm_match_pairs_events(ctypes.byref(r), out.data_ptr(), K.value, ctypes.byref(K), ws.data_ptr(), ws.numel(), st)
        b.record(); torch.cuda.synchronize()
        assert s == 0, (s, L.ddm_last_cuda_error(), K.value)
        ts.append(a.elapsed_time(b))
    ddm.profile_enable(True)
    L.ddm_match_pairs_events(ctypes.byref(r), out.data_ptr(), K.value, ctypes.byref(K), ws.data_ptr(), ws.numel(), st)
    torch.cuda.synchronize()
    prof = ddm.profile_read(); ddm.profile_enable(False)
    t = float(np.median(ts[1:]))
    print(f"{cfg} events K={K.value}: {t:.3f} ms  regions/s={(w.n + w.m) / t * 1e3:.3e}  ws={ws.numel()/1e9:.2f} GB", flush=True)
    for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["total_ms"])[:8]:
        print(f"   {k:20s} {v['total_ms']:8.3f} ms x{v['launches']}", flush=True)
    del out, ws, g
    torch.cuda.empty_cache()
