#!/usr/bin/env python
"""bench.py -- B200 DDM sort-based matching benchmark (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ddm|reference] [--config c3]

A step is one pass of the whole hot path (validate +
encode, sort Slo/Shi/Ulo, gathers, rank-difference counts, scan, chunked
sweep + pair emission) over one synthetic BASELINE workload already resident
in HBM, through the C ABI (`ddm_match_pairs`), with the pair list written to a
preallocated device buffer.  Default workload: BASELINE configs[2] = c3
(d=1, n=m=5e7, N=1e8), the configuration the north star's roofline target is
quoted on.  Rank 0 prints one JSON line.

N > 1 (one process per GPU, NCCL; `--gpus N` without a launcher starts its
own N ranks through torch.distributed.run): default slab mode -- every rank
starts with an index block of the regions in HBM, and each step computes the
slab cut points, partitions (slab + halo) and exchanges the regions on the
device (all_to_all), matches its slab and all-reduces K; `--dist broadcast`
builds the subscription index on rank 0 and broadcasts it instead
(DESIGN.md §7).  Total work is fixed -> "scaling": "strong".

--impl reference: the CPU oracle (oracle/, Alg. 5+6 Parallel-SBM on all host
cores) on a bounded window sample of the same workload (the reference arm of
this tier; rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "regions matched/sec and pairs emitted/sec per GPU; % of HBM roofline, 1/2/4/8 B200"
FALLBACK_HBM_GBS = 6650.0
CPU_SAMPLE_FRAC = {"c1": 1.0, "c2": 0.5, "c3": 0.5, "c4": 0.006, "c5": 0.01}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ddm", choices=["ddm", "reference"])
    ap.add_argument("--config", default="c3", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--alpha", type=float, default=None,
                    help="replace the config's overlap degree alpha (count-mode K-independence sweep, P:960-963)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--mode", default="pairs", choices=["pairs", "count"],
                    help="pairs: the list (default); count: K only (ddm_match_count, the paper's experimental "
                         "mode P:915-918), single GPU")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="N>1 process group; gloo stages collectives through host memory and lets ranks share a "
                         "GPU (tests of the multi-GPU path on one GPU; not a performance configuration)")
    ap.add_argument("--dist", default="slab", choices=["slab", "broadcast"],
                    help="N>1: slab = fully distributed index (each rank its slab + halo, "
                         "only the count all-reduce); broadcast = rank 0 builds the sub index, NCCL broadcast")
    return ap.parse_args()


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


_SAMPLER = r"""
import sys, time, pynvml
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(int(sys.argv[1]))
print("max", pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM), flush=True)
while True:
    try:
        print(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
              pynvml.nvmlDeviceGetCurrentClocksEventReasons(h),
              pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_MEM),
              pynvml.nvmlDeviceGetPowerUsage(h), flush=True)
    except pynvml.NVMLError:
        pass
    time.sleep(0.002)
"""


class Clocks:
    """SM clocks and throttle reasons sampled DURING the timed region by an
    NVML polling child process (every 2 ms; a separate process so the GIL of
    the launching thread cannot starve it)."""
    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "hw_power_brake_slowdown": 0x80, "sw_power_cap": 0x4}

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.p = None
        self.f = None

    def start(self):
        import subprocess
        import tempfile
        self.f = tempfile.TemporaryFile("w+")
        try:
            self.p = subprocess.Popen([sys.executable, "-c", _SAMPLER, str(self.gpu)], stdout=self.f,
                                      stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None
            return
        t0 = time.time()  # wait for the first sample so the region is covered from its start
        while time.time() - t0 < 20:
            self.f.seek(0)
            if len(self.f.read().splitlines()) >= 2:
                break
            time.sleep(0.01)

    def stop(self) -> dict:
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml sampler unavailable"], "samples": 0}
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:  # noqa: BLE001
            self.p.kill()
        self.f.seek(0)
        lines = self.f.read().splitlines()
        mx, sm, mem, pw, reasons = None, [], [], [], set()
        for ln in lines:
            parts = ln.split()
            if parts and parts[0] == "max":
                mx = float(parts[1])
                continue
            try:
                sm.append(float(parts[0]))
                r = int(parts[1])
                mem.append(float(parts[2]))
                pw.append(float(parts[3]) / 1000.0)
            except (ValueError, IndexError):
                continue
            for nm, bit in self.REASONS.items():
                if r & bit:
                    reasons.add(nm)
        sm = sm[1:] if len(sm) > 1 else sm  # the first sample predates the region
        mem, pw = mem[1:] if len(mem) > 1 else mem, pw[1:] if len(pw) > 1 else pw
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "mem_mhz": float(np.median(mem)) if mem else None,
                "power_w": float(np.median(pw)) if pw else None,
                "samples": len(sm), "source": "NVML child process, 2 ms polling"}


L2_BYTES = 126e6


def needs_flush(w) -> bool:
    """Inputs (16 d B per region) plus the sorted copies the step makes
    (~24 B per region and kind) could stay resident in the 126 MB L2."""
    return 40.0 * w.d * (w.n + w.m) <= 2 * L2_BYTES


def workload_config(w, extra=None, mode="pairs"):
    d = {"workload": w.name, "d": w.d, "n_sub": w.n, "n_upd": w.m, "L": w.L, "l": w.l, "seed": w.seed,
         "coords": "float64", "mode": "pairs (list)" if mode == "pairs" else "count only (ddm_match_count)",
         "l2": "L2 flushed before every timed step (256 MB write outside the timed events)" if needs_flush(w)
         else "inputs larger than L2 (no flush needed)"}
    if extra:
        d.update(extra)
    return d


# ---------------------------------------------------------------- reference arm (CPU oracle)

def cpu_sample(w, frac):
    from paper_1703_06680_b200 import workload as wl
    return wl.window_sample(w, frac) if frac < 1.0 else w


def time_oracle(sample, reps=1, count_only=False):
    """The oracle as it stands: Parallel-SBM (Alg. 5+6, all host cores) for
    d = 1; for d > 1 the serial SBM with the per-dimension filter (the
    oracle's Parallel-SBM is one-dimensional).  Returns
    (seconds, K, threads used, method)."""
    import oracle
    P = oracle.max_threads() if sample.d == 1 else 1
    best = None
    K = 0
    for _ in range(reps):
        t0 = time.perf_counter()
        if sample.d == 1 and count_only:
            K = oracle.par_sbm(sample.sub_lo, sample.sub_hi, sample.upd_lo, sample.upd_hi, P=P, count_only=True)
        elif sample.d == 1:
            K = oracle.par_sbm(sample.sub_lo, sample.sub_hi, sample.upd_lo, sample.upd_hi, P=P,
                               canonicalize=False).size
        else:
            K = oracle.sbm_seq(sample.sub_lo, sample.sub_hi, sample.upd_lo, sample.upd_hi, canonicalize=False).size
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    mode = "count mode" if (count_only and sample.d == 1) else "list mode"
    method = f"oracle.par_sbm (Alg. 5+6, {mode})" if sample.d == 1 else "oracle.sbm_seq (Alg. 4 + filter, list mode)"
    return best, K, P, method


def host_info() -> dict:
    """The host the CPU baseline runs on: CPU model (lscpu / /proc/cpuinfo),
    logical CPUs, and the CPUs this process may run on (affinity)."""
    model = None
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    try:
        aff = len(os.sched_getaffinity(0))
    except AttributeError:
        aff = None
    return {"cpu_model": model, "logical_cpus": os.cpu_count(), "affinity_cpus": aff,
            "omp_num_threads": os.environ.get("OMP_NUM_THREADS")}


def sample_text(s, frac):
    return (f"{s.name}: regions with dim-0 lower bound in a {frac:g} L window centred on the median "
            f"({s.n + s.m} regions)")


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return
    from paper_1703_06680_b200 import workload as wl
    w = wl.make(args.config, alpha=args.alpha)
    frac = CPU_SAMPLE_FRAC[args.config]
    s = cpu_sample(w, frac)
    for _ in range(args.warmup):
        time_oracle(s)
    times, K, P, method = [], 0, 1, ""
    for _ in range(args.steps):
        dt, K, P, method = time_oracle(s)
        times.append(dt)
    t = float(np.sum(times))
    regions = (s.n + s.m) * args.steps
    val = regions / t
    sample = f"{sample_text(s, frac)}, K={K}; {method}"
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "regions/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "pairs_per_s": K * args.steps / t,
            "config": workload_config(w, {"parallelism": f"CPU x{P} ({method})", "sample": sample,
                                          "l2": "n/a (host CPU)"}),
            "cpu_baseline": {"value": val, "unit": "regions/s", "cores": P, "kind": "oracle", "sample": sample,
                             "host": host_info()},
            "e2e": {"value": val, "unit": "regions/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- GPU arm

def run_ddm(args):
    import torch
    import torch.distributed as dist

    from paper_1703_06680_b200 import ddm, workload as wl
    from paper_1703_06680_b200 import dist as ddist

    rank, world, local = env_rank()
    if world != args.gpus:  # a launcher mismatch must not produce a line with the wrong n_gpus
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    ndev = torch.cuda.device_count()
    if args.backend == "nccl" and world > ndev:
        raise SystemExit(f"bench.py: {world} ranks need {world} GPUs, {ndev} visible "
                         "(--backend gloo shares GPUs between ranks, for testing only)")
    local = local % max(ndev, 1)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    ddm.load()
    w = wl.make(args.config, alpha=args.alpha)
    hbm_peak, peak_src = peaks()

    def sync_all():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
            torch.cuda.synchronize()

    stream = torch.cuda.current_stream()
    dist_marks = []  # per timed step: CUDA events between the phases of the multi-GPU step
    if world == 1:
        g = [torch.from_numpy(a).to(dev) for a in (w.sub_lo, w.sub_hi, w.upd_lo, w.upd_hi)]
        M = ddm.Matcher(w.d, w.n, w.m, dev)
        K = M.count(*g)
        out = torch.empty((max(K, 1), 2), dtype=torch.int32, device=dev) if args.mode == "pairs" else None

        def step():
            return M.pairs_into(out, *g) if args.mode == "pairs" else M.count(*g)
    elif args.dist == "slab":
        # every rank starts with its index block of both kinds in HBM (the
        # input as it arrives); the step partitions on the device, exchanges
        # by all_to_all and matches
        s0, s1 = ddist.block_of(w.n, rank, world)
        u0, u1 = ddist.block_of(w.m, rank, world)
        blk = [torch.from_numpy(np.ascontiguousarray(a)).to(dev)
               for a in (w.sub_lo[:, s0:s1], w.sub_hi[:, s0:s1], w.upd_lo[:, u0:u1], w.upd_hi[:, u0:u1])]
        SM = ddist.SlabMatcher(w.d, dev)

        def step():
            r = SM.step(blk[0], blk[1], s0, blk[2], blk[3], u0)
            dist_marks.append(r.marks)
            return r.k_total
    else:
        # broadcast: rank 0 holds the subscriptions, every rank its update block
        u0, u1 = ddist.block_of(w.m, rank, world)
        sub = [torch.from_numpy(a).to(dev) for a in (w.sub_lo, w.sub_hi)] if rank == 0 else [None, None]
        upd = [torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (w.upd_lo[:, u0:u1], w.upd_hi[:, u0:u1])]
        uid = torch.arange(u0, u1, dtype=torch.int32, device=dev)
        # capacity from an untimed count against a freshly built index
        SM0 = ddist.ShardedMatcher(w.d, w.n, u1 - u0, 1, dev)
        if rank == 0:
            SM0.build_index(*sub)
        SM0.coll.broadcast_(SM0.index, src=0)
        cap = ddm.match_count_indexed(SM0.index, w.n, *upd)
        del SM0
        SM = ddist.ShardedMatcher(w.d, w.n, u1 - u0, cap, dev)

        def step():
            r = SM.step(sub[0], sub[1], upd[0], upd[1], uid)
            dist_marks.append(r.marks)
            return r.k_total

    for _ in range(max(args.warmup, 0)):
        K = step()
    sync_all()
    dist_marks.clear()
    # ---- the timed region (the official number): K steps, no instrumentation
    clocks = Clocks(local)
    clocks.start()
    l0 = ddm.launch_count()
    # inputs that fit in L2 (c1, c2) would be timed warm: a 256 MB write
    # between steps (outside the timed events) evicts them first
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if needs_flush(w) else None
    ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    sync_all()
    for i in range(args.steps):
        if flush is not None:
            flush.fill_(i & 0xFF)
        ev0[i].record(stream)
        K = step()
        ev1[i].record(stream)  # (each step ends in its own host sync anyway)
    torch.cuda.synchronize()
    sync_all()
    launches = ddm.launch_count() - l0
    clk = clocks.stop()
    per_step = np.array([ev0[i].elapsed_time(ev1[i]) for i in range(args.steps)])
    ms = float(per_step.sum())
    # multi-GPU phases (device events inside each step): slab T_partition
    # (cuts, pack, all_to_all, unpack) + T_match; broadcast T_index (build +
    # broadcast) + T_match; means over the timed steps, max over ranks below
    dist_phases = None
    if dist_marks:
        first = "partitioned" if "partitioned" in dist_marks[0] else "indexed"
        t_a = float(np.mean([m["start"].elapsed_time(m[first]) for m in dist_marks]))
        t_b = float(np.mean([m[first].elapsed_time(m["matched"]) for m in dist_marks]))
        dist_phases = [t_a, t_b]
    dist_marks.clear()
    step_stats = {"median": round(float(np.median(per_step)), 4), "p10": round(float(np.percentile(per_step, 10)), 4),
                  "p90": round(float(np.percentile(per_step, 90)), 4), "mean": round(float(per_step.mean()), 4)}
    # ---- a second timed region of the same K steps with per-kernel CUDA
    # events recorded by the library on each kernel's launching stream
    # (profiling mode runs the concurrent sort chains on one stream so the
    # kernels' intervals do not overlap): roofline + phase breakdown
    ddm.profile_enable(True)
    p0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    p1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    for i in range(args.steps):
        if flush is not None:  # (a torch fill, not a library launch: not in the records)
            flush.fill_((i + 7) & 0xFF)
        p0[i].record(stream)
        step()
        p1[i].record(stream)
    torch.cuda.synchronize()
    prof = ddm.profile_read()
    ddm.profile_enable(False)
    prof_ms_step = float(np.mean([p0[i].elapsed_time(p1[i]) for i in range(args.steps)]))
    dist_marks.clear()
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        lt = torch.tensor([launches], dtype=torch.int64, device=dev)
        dist.all_reduce(lt, op=dist.ReduceOp.SUM)
        launches = int(lt.item())
    if dist_phases is not None:
        t = torch.tensor(dist_phases, dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist_phases = {("T_partition_ms" if args.dist == "slab" else "T_index_ms"): round(float(t[0]), 4),
                       "T_match_ms": round(float(t[1]), 4), "reduction": "mean over timed steps, max over ranks"}
    ms_step = ms / args.steps
    regions = w.n + w.m
    value = regions / (ms_step * 1e-3)

    # roofline of the dominant kernel class (measured live above)
    dom = max(prof.items(), key=lambda kv: kv[1]["total_ms"]) if prof else None
    roof = None
    phases = {}
    if dom:
        name, st = dom
        avg_ms = st["total_ms"] / st["launches"]
        bytes_per_launch = st["bytes"] / st["launches"]
        achieved = bytes_per_launch / (avg_ms * 1e-3) / 1e9
        traffic = None
        tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tp):
            traffic = json.load(open(tp)).get(args.config, {}).get(name)
        roof = {"bound": "hbm", "kernel": name, "achieved": round(achieved, 1), "peak": hbm_peak, "unit": "GB/s",
                "frac": round(achieved / hbm_peak, 4), "traffic": traffic, "peak_source": peak_src,
                "bytes_per_launch": bytes_per_launch, "avg_launch_ms": round(avg_ms, 4),
                "share_of_step": round(st["total_ms"] / (prof_ms_step * args.steps), 3),
                "measured_in": "second timed region of the same K steps, per-kernel CUDA events on the launching "
                               "stream (library profiling mode: sort chains serialised), "
                               f"{prof_ms_step:.3f} ms/step"}
        tot_bytes = sum(v["bytes"] for v in prof.values())
        phases = {k: {"ms_per_step": round(v["total_ms"] / args.steps, 4), "launches_per_step": v["launches"] / args.steps,
                      "GBps": round(v["bytes"] / (v["total_ms"] * 1e-3) / 1e9, 1) if v["total_ms"] else None}
                  for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["total_ms"])}
        pipeline_frac = tot_bytes / args.steps / (ms_step * 1e-3) / (hbm_peak * 1e9)  # over the official step time
        literal_floor = 16.0 * w.d * regions + 8.0 * K
        ncu_tot = None
        if os.path.exists(tp):
            ncu_tot = json.load(open(tp)).get(args.config, {}).get("_call_total")
        phases_summary = {"pipeline_bytes_per_step": tot_bytes / args.steps,
                          "pipeline_frac_of_peak": round(pipeline_frac, 4),
                          # ncu DRAM bytes of one whole call (profiles/ncu_traffic.json)
                          "ncu_bytes_per_step": ncu_tot,
                          "ncu_frac_of_peak": (round(ncu_tot / (ms_step * 1e-3) / (hbm_peak * 1e9), 4)
                                               if ncu_tot and world == 1 else None),
                          "literal_floor_bytes": literal_floor,
                          "literal_floor_frac": round(literal_floor / (ms_step * 1e-3) / (hbm_peak * 1e9), 4)}
    else:
        phases_summary = {}

    # e2e through the public API with host buffers (N=1): every step copies
    # its inputs from pinned host memory and its pairs back, through
    # ddm.PipelinedMatcher (step i+1's H2D overlaps step i's match, step i's
    # D2H overlaps step i+1's match).  Device-timed with events bracketing the
    # first copy-in and the last copy-out.
    e2e = None
    if world == 1 and not args.no_e2e and args.mode == "pairs":
        del M, g, out  # the pipelined matcher double-buffers its own inputs (c5: 2 x 16 GB)
        torch.cuda.empty_cache()
        host = [torch.from_numpy(a).pin_memory() for a in (w.sub_lo, w.sub_hi, w.upd_lo, w.upd_hi)]
        houts = [torch.empty((max(K, 1), 2), dtype=torch.int32).pin_memory() for _ in range(2)]
        h2d = sum(h.numel() * 8 for h in host)
        d2h = K * 8
        PM = ddm.PipelinedMatcher(w.d, w.n, w.m, K, dev)

        def batches(cnt):
            return ((host, houts[i & 1]) for i in range(cnt))

        for _ in PM.run(batches(2)):  # warm-up (graph capture of both slots' calls)
            pass
        for _ in PM.run(batches(2)):
            pass
        n_e2e = max(3, args.steps)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(PM.s_h2d)
        ks = [k for k, _ in PM.run(batches(n_e2e))]
        b.record(PM.s_d2h)
        torch.cuda.synchronize()
        assert all(k == K for k in ks)
        e_ms = a.elapsed_time(b) / n_e2e
        e2e = {"value": regions / (e_ms * 1e-3), "unit": "regions/s", "ms_per_step": round(e_ms, 3),
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": n_e2e,
               "api": "paper_1703_06680_b200.ddm.PipelinedMatcher.run (ddm_match_pairs per batch, pinned host "
                      "buffers, copies overlapped with the neighbouring batches' matches)"}

    if world > 1 and not args.no_e2e and args.mode == "pairs" and args.dist == "slab":
        # e2e at N GPUs through dist.SlabMatcher: every step each rank copies
        # its input block in from pinned host memory and its pair list out
        hb = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
              for a in (w.sub_lo[:, s0:s1], w.sub_hi[:, s0:s1], w.upd_lo[:, u0:u1], w.upd_hi[:, u0:u1])]
        hout = torch.empty((max(K, 1), 2), dtype=torch.int32).pin_memory()
        h2d = sum(h.numel() * 8 for h in hb)
        d2h_tot = 0
        n_e2e = max(3, args.steps)
        sync_all()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(n_e2e):
            for dst, src in zip(blk, hb):
                dst.copy_(src, non_blocking=True)
            r = SM.step(blk[0], blk[1], s0, blk[2], blk[3], u0)
            if hout.shape[0] < r.k_local:
                hout = torch.empty((r.k_local, 2), dtype=torch.int32).pin_memory()
            hout[: r.k_local].copy_(r.pairs, non_blocking=True)
            d2h_tot += r.k_local * 8
        b.record(stream)
        torch.cuda.synchronize()
        t = torch.tensor([a.elapsed_time(b) / n_e2e, h2d, d2h_tot / n_e2e], dtype=torch.float64, device=dev)
        tm = t.clone()
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        e_ms = float(tm[0])
        e2e = {"value": (w.n + w.m) / (e_ms * 1e-3), "unit": "regions/s", "ms_per_step": round(e_ms, 3),
               "h2d_bytes_per_step": int(t[1]), "d2h_bytes_per_step": int(t[2]), "steps": n_e2e,
               "api": "paper_1703_06680_b200.dist.SlabMatcher.step per rank (input block H2D from pinned memory, "
                      "on-device partition + all_to_all + match, local pairs D2H); max over ranks"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        frac = CPU_SAMPLE_FRAC[args.config]
        s = cpu_sample(w, frac)
        dt, ks, P, method = time_oracle(s, count_only=args.mode == "count")
        cpu = {"value": (s.n + s.m) / dt, "unit": "regions/s", "cores": P, "kind": "oracle",
               "sample": f"{sample_text(s, frac)}, K={ks}; {method}, {dt:.2f} s", "host": host_info()}
        if args.config in ("c1", "c2"):
            # brute force (Alg. 2, all host cores) on the same sample
            import oracle
            t0 = time.perf_counter()
            kb = oracle.bf_count(s.sub_lo, s.sub_hi, s.upd_lo, s.upd_hi)
            db = time.perf_counter() - t0
            cpu["brute_force"] = {"value": (s.n + s.m) / db, "unit": "regions/s", "cores": oracle.max_threads(),
                                  "sample": f"{sample_text(s, frac)}, K={kb}; oracle.bf_count (Alg. 2), {db:.2f} s"}
        if w.d == 1:
            # also the serial SBM (Alg. 4) on one core, on a
            # tenth of that window (the paper's serial baseline)
            import oracle
            s1 = cpu_sample(w, frac / 10)
            t0 = time.perf_counter()
            k1 = oracle.sbm_seq(s1.sub_lo, s1.sub_hi, s1.upd_lo, s1.upd_hi, canonicalize=False).size
            d1 = time.perf_counter() - t0
            cpu["serial"] = {"value": (s1.n + s1.m) / d1, "unit": "regions/s", "cores": 1,
                             "sample": f"{sample_text(s1, frac / 10)}, K={k1}; oracle.sbm_seq (Alg. 4, list mode), "
                                       f"{d1:.2f} s"}

    if roof and roof["kernel"].startswith("dd"):
        # d > 1 (c4): the filter kernel is issue/latency bound, not HBM bound
        # (SURVEY F3): roofline of its instruction issue.  achieved = warp
        # instructions per launch (ncu smsp__inst_executed.sum of the same
        # launch, profiles/ncu_inst.json) / the live average launch time;
        # peak = 4 schedulers x SMs x 1 warp instruction per clock at the
        # maximum SM clock
        ip = os.path.join(ROOT, "profiles", "ncu_inst.json")
        inst = json.load(open(ip)).get(args.config, {}).get(roof["kernel"]) if os.path.exists(ip) else None
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        fmax = (clk or {}).get("sm_max_mhz") or 1965.0
        peak_gi = 4 * sms * fmax * 1e6 / 1e9
        if inst:
            ach = inst / (roof["avg_launch_ms"] * 1e-3) / 1e9
            roof = {"bound": "alu", "kernel": roof["kernel"], "achieved": round(ach, 1), "peak": round(peak_gi, 1),
                    "unit": "Gwarp-inst/s", "frac": round(ach / peak_gi, 4), "traffic": roof["traffic"],
                    "peak_source": f"derived: 4 SMSP x {sms} SMs x 1 warp-inst/clk x {fmax:.0f} MHz (DESIGN.md §6)",
                    "inst_per_launch": inst, "avg_launch_ms": roof["avg_launch_ms"],
                    "share_of_step": roof["share_of_step"], "measured_in": roof["measured_in"],
                    "hbm_frac": roof["frac"]}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "regions/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": round(ms_step, 4), "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
                "config": workload_config(w, mode=args.mode, extra={"parallelism": "single GPU" if world == 1 else
                                              (f"dim-0 slabs x{world} ({args.backend}): every rank starts with an "
                                               f"index block of both kinds; on-device cuts + partition (slab + "
                                               f"halo), all_to_all exchange, mapped match, K all-reduce"
                                               if args.dist == "slab" else
                                               f"update blocks x{world} ({args.backend}), sub index built on rank 0 "
                                               f"and broadcast, K all-reduce"),
                                              "K": K, "timing": "CUDA events on the launching stream, max over ranks"}),
                "dist_phases": dist_phases,
                "pairs_per_s": K / (ms_step * 1e-3), "regions_per_s_per_gpu": value / world,
                "step_ms": step_stats,
                "roofline": roof, "pipeline": phases_summary, "phases": phases, "cpu_baseline": cpu, "e2e": e2e,
                "clocks": clk, "gpu_launches": launches, "build": ddm.build_info()}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def self_launch(args) -> int:
    """--gpus N > 1 without a launcher: start N ranks with torch.distributed.run
    (one process per GPU, rendezvous on 127.0.0.1) running this same command
    line; rank 0's JSON line is passed through."""
    import socket
    import subprocess
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ddm(args)


if __name__ == "__main__":
    main()
