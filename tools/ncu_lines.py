"""Per-CUDA-source-line instruction counts and stall samples from an ncu report (dev tool).
usage: ncu_lines.py report.ncu-rep [kernel-regex] [top]"""
import csv, subprocess, sys
rep = sys.argv[1]; k = sys.argv[2] if len(sys.argv) > 2 else ""; top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"] + (["-k", k] if k else [])
rows = list(csv.reader(subprocess.run(cmd, capture_output=True, text=True).stdout.splitlines()))
out, fname, h, cur = [], "", None, None
for x in rows:
    if len(x) == 2 and x[0] == "File Path":
        fname = x[1].split("/")[-1]
    elif x and x[0] == "Line No":
        h = {n: i for i, n in enumerate(x)}
    elif h and len(x) > 8 and x[0] not in ("",):
        f = lambda v: float(v) if v not in ("", "-") else 0.0
        try:
            cur = [fname, x[0], x[1][:90], f(x[h["Instructions Executed"]]), f(x[h["Warp Stall Sampling (All Samples)"]])]
        except (ValueError, IndexError):
            continue  # a source line whose quoting broke the CSV row
        out.append(cur)
ti = sum(o[3] for o in out) or 1; ts = sum(o[4] for o in out) or 1
print(f"total warp-instrs {ti:.3e}, stall samples {ts:.0f}")
for o in sorted(out, key=lambda o: -o[3])[:top]:
    print(f"{100*o[3]/ti:5.1f}% inst {100*o[4]/ts:5.1f}% stall {o[0]}:{o[1]} {o[2]}")
