"""Summarise an ncu launch list (time, and DRAM bytes when captured) (dev tool)."""
import csv, collections, sys
path = sys.argv[1]; last = int(sys.argv[2]) if len(sys.argv) > 2 else 0
rows = list(csv.reader(open(path)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hi]; data = rows[hi + 1:]
ids = sorted({int(r[0]) for r in data}); keep = set(ids[-last:]) if last else set(ids)
ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3,
         "byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1, "Gbyte": 1e3}
per = collections.defaultdict(dict); names = {}
for r in data:
    i = int(r[0])
    if i not in keep: continue
    per[i][r[mi]] = float(r[vi].replace(",", "")) * scale.get(r[ui], 1)
    names[i] = r[ki].split("(")[0].replace("void ", "")[:55]
agg = collections.OrderedDict(); tot = [0.0, 0.0]
for i in sorted(per):
    a = agg.setdefault(names[i], [0.0, 0.0, 0])
    t = per[i].get("gpu__time_duration.sum", 0); b = per[i].get("dram__bytes_read.sum", 0) + per[i].get("dram__bytes_write.sum", 0)
    a[0] += t; a[1] += b; a[2] += 1; tot[0] += t; tot[1] += b
for k, (t, b, c) in agg.items():
    print(f"{t:9.1f} us {100*t/tot[0]:5.1f}%  {b:9.1f} MB  {b/t if t else 0:6.2f} TB/s  x{c:3d}  {k}")
print(f"total {tot[0]:.1f} us, {tot[1]:.1f} MB")
