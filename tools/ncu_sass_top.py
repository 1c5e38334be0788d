"""Top SASS instructions by warp-stall samples from an ncu report (dev tool)."""
import csv, subprocess, sys, collections
rep = sys.argv[1]; kname = sys.argv[2] if len(sys.argv) > 2 else ""; ntop = int(sys.argv[3]) if len(sys.argv) > 3 else 40
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"] + (["-k", kname] if kname else [])
out = subprocess.run(cmd, capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
hi = next(i for i, x in enumerate(r) if "Source" in x and "Address" in x)
h = r[hi]; ci = {k: i for i, k in enumerate(h)}
rows = [x for x in r[hi + 1:] if len(x) == len(h) and x[0].startswith("0x")]
key = "Warp Stall Sampling (All Samples)"
tot = sum(float(x[ci[key]] or 0) for x in rows)
print("total samples", tot, "instructions", len(rows))
ops = collections.Counter()
for x in rows:
    toks = x[ci["Source"]].split()
    op = toks[1] if toks and toks[0].startswith("@") and len(toks) > 1 else (toks[0] if toks else "?")
    ops[op.split(".")[0]] += float(x[ci[key]] or 0)
print("by opcode:", [(k, round(100 * v / tot, 1)) for k, v in ops.most_common(15)])
for i, x in sorted(enumerate(rows), key=lambda t: -float(t[1][ci[key]] or 0))[:ntop]:
    print(f"{i:5d} {100*float(x[ci[key]])/tot:5.1f}% ex={x[ci['Instructions Executed']]:>9} {x[ci['Source']][:90]}")
