"""smsp__inst_executed.sum of the dd_stage launches (rows_kernel<..., 1> or dd_tile_kernel<..., 1>) in an ncu --metrics csv
-> profiles/ncu_inst.json (bench.py's ALU roofline for c4).  usage: inst_json.py dd_inst.csv [out.json]"""
import csv, json, sys
path = sys.argv[1]
out = sys.argv[2] if len(sys.argv) > 2 else "profiles/ncu_inst.json"
rows = list(csv.reader(open(path)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hi]
ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
vals = [float(r[vi].replace(",", "")) for r in rows[hi + 1:]
        if r[mi] == "smsp__inst_executed.sum" and ("dd_tile_kernel" in r[ki] or "rows_kernel" in r[ki])
        and ", 1>" in r[ki]]
J = {"_note": "smsp__inst_executed.sum (warp instructions) per launch of the dominant d>1 kernel "
              "(rows_kernel<4, 1> / dd_tile_kernel<4, 1> = the dd_stage pass of the pairs calls), mean over the launches of "
              "`ncu --metrics smsp__inst_executed.sum` on `DDM_SERIAL=1 tools/profile_once.py c4` (tools/inst_json.py). "
              "Used by bench.py's ALU roofline.",
     "c4": {"dd_stage": sum(vals) / len(vals)}, "_launches": len(vals)}
json.dump(J, open(out, "w"), indent=1)
print(json.dumps(J))
