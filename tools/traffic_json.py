"""Per-launch DRAM traffic of each phase of the LAST pairs call in an ncu launch list -> profiles/ncu_traffic.json
usage: traffic_json.py launches.csv n_last cfg [out.json]   (n_last = launches of that call, printed by profile_once.py)"""
import csv, collections, json, re, sys
path, last, cfg = sys.argv[1], int(sys.argv[2]), sys.argv[3]
out = sys.argv[4] if len(sys.argv) > 4 else "profiles/ncu_traffic.json"
rows = list(csv.reader(open(path)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hi]; data = rows[hi + 1:]
ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
ids = sorted({int(r[0]) for r in data})[-last:]
per = collections.defaultdict(float); name = {}
for r in data:
    i = int(r[0])
    if i in ids and r[mi].startswith("dram__bytes"):
        per[i] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1)
        name[i] = r[ki]
def phase(k):
    if "msd_pass_kernel" in k: return "msd_pass_pay" if re.search(r"msd_pass_kernel<\d+, (1|true)", k) else "msd_pass"
    if "local_sort_kernel" in k:  # local_sort_kernel<config, V64, V32>: V64 = the payload sorts
        return "msd_local_pay" if re.search(r"local_sort_kernel<[^,<>]*(<[^>]*>)?, (1|true),", k) else "msd_local"
    for a, b in (("count_kernel", "count"), ("emit", "emit"), ("msd_hist", "msd_hist"), ("block_max", "block_max"),
                 ("tree_pm", "tree_pm"), ("dd_tile", "dd"), ("scan_u64", "scan")):
        if a in k: return b
    return None
agg = collections.defaultdict(list)
for i in ids:
    p = phase(name.get(i, ""))
    if p: agg[p].append(per[i])
try:
    J = json.load(open(out))
except Exception:
    J = {}
J["_note"] = ("dram__bytes_read.sum + dram__bytes_write.sum per launch (bytes, mean over the phase's launches) of the last "
              "pairs call in the ncu launch list of `DDM_SERIAL=1 tools/profile_once.py <cfg>` (tools/traffic_json.py), "
              "the configuration of bench.py's profiled region. Used by bench.py's roofline.traffic.")
J[cfg] = {p: sum(v) / len(v) for p, v in agg.items()}
J[cfg]["_call_total"] = sum(per[i] for i in ids)  # every kernel of the call (SURVEY §8(d) B_R3)
json.dump(J, open(out, "w"), indent=1)
print(json.dumps(J[cfg], indent=1))
