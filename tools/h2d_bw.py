import torch, time
N = 400_000_000 // 8
hs = [torch.empty(N, dtype=torch.float64).pin_memory() for _ in range(4)]
ds = [torch.empty(N, dtype=torch.float64, device="cuda") for _ in range(4)]
for nst in (1, 2, 4):
    sts = [torch.cuda.Stream() for _ in range(nst)]
    for rep in range(3):
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record()
        for s in sts: s.wait_stream(torch.cuda.current_stream())
        for i in range(4):
            with torch.cuda.stream(sts[i % nst]):
                ds[i].copy_(hs[i], non_blocking=True)
        for s in sts: torch.cuda.current_stream().wait_stream(s)
        b.record(); torch.cuda.synchronize()
        t = a.elapsed_time(b)
    print(f"H2D {nst} streams: {1.6e9 / (t * 1e-3) / 1e9:.1f} GB/s ({t:.2f} ms)", flush=True)
# D2H concurrently with H2D
d2 = torch.empty(N, dtype=torch.float64, device="cuda"); h2 = torch.empty(N, dtype=torch.float64).pin_memory()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize(); t0 = time.time()
with torch.cuda.stream(s1):
    for i in range(4): ds[i].copy_(hs[i], non_blocking=True)
with torch.cuda.stream(s2):
    h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize(); print(f"H2D 1.6GB + D2H 0.4GB concurrently: {(time.time()-t0)*1e3:.2f} ms", flush=True)
