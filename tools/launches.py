"""Summarise an ncu --metrics gpu__time_duration.sum launch list (dev tool)."""
import csv, collections, sys
path = sys.argv[1]; skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
rows = list(csv.reader(open(path)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hi]; data = rows[hi + 1:]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = collections.OrderedDict(); tot = 0.0
for r in data:
    if int(r[0]) < skip: continue
    v = float(r[vi].replace(",", "")); u = r[ui]
    v = v / 1e3 if u in ("ns", "nsecond") else v * 1e3 if u in ("ms", "msecond") else v
    name = r[ki].split("(")[0].replace("void ", "")[:60]
    a = agg.setdefault(name, [0.0, 0]); a[0] += v; a[1] += 1; tot += v
for k, (v, c) in agg.items():
    print(f"{v:10.1f} us {100*v/tot:5.1f}%  x{c:3d}  {k}")
print(f"total {tot:.1f} us")
