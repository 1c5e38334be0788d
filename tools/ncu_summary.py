"""Per-kernel summary (duration, DRAM bytes/throughput, occupancy, top stalls) of an ncu report."""
import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[0]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "smsp__inst_executed.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem"]
idx = {w: h.index(w) for w in want if w in h}
stall = [(i, k) for i, k in enumerate(h) if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")]
for row in r[2:]:
    name = row[h.index("Kernel Name")][:55]
    vals = {w: row[i] for w, i in idx.items()}
    st = sorted(((float(row[i] or 0), k.replace("smsp__pcsamp_warps_issue_stalled_", "")) for i, k in stall), reverse=True)
    tot = sum(v for v, _ in st) or 1
    print(f"{name}\n   dur={vals.get('gpu__time_duration.sum')} dramR={vals.get('dram__bytes_read.sum')} dramW={vals.get('dram__bytes_write.sum')} "
          f"dram%={vals.get('dram__throughput.avg.pct_of_peak_sustained_elapsed')} sm%={vals.get('sm__throughput.avg.pct_of_peak_sustained_elapsed')} "
          f"warps%={vals.get('sm__warps_active.avg.pct_of_peak_sustained_active')} regs={vals.get('launch__registers_per_thread')} "
          f"inst={vals.get('smsp__inst_executed.sum')}\n   stalls: " + ", ".join(f"{k}={100*v/tot:.0f}%" for v, k in st[:6]))
