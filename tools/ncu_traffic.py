"""DRAM traffic per walk kernel from an ncu metrics CSV of one pipeline pass
-> profiles/ncu_traffic_<config>.json (read by bench.py's roofline).

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
        -k regex:"build_search_kernel|beam_knn_kernel" --csv --log-file t.csv python tools/profile_step.py C5 1
    python tools/ncu_traffic.py t.csv C5 <commit>
"""
import csv
import json
import os
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
path, name, commit = sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None
rows = [r for r in csv.reader(open(path)) if r]
hdr = next(i for i, r in enumerate(rows) if "Metric Name" in r)
cols = rows[hdr]
ki, mi, vi, ui, ii = (cols.index(c) for c in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "nsecond": 1e-6, "usecond": 1e-3,
         "msecond": 1.0, "second": 1e3, "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}
per = defaultdict(lambda: defaultdict(float))
for r in rows[hdr + 1:]:
    kern = r[ki].split("(")[0].split("<")[0].replace("void ", "").replace("pk::", "").strip()
    v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    per[(kern, r[ii])][r[mi]] = v
out = {"_note": f"ncu metrics of every {name} walk launch of one pipeline pass (tools/ncu_traffic.py; "
                "dram bytes read + written; times are ncu's serialised, cold-cache ones)", "commit": commit}
agg = defaultdict(lambda: {"launches": 0, "dram_bytes": 0.0, "ncu_ms": 0.0})
for (kern, _), m in per.items():
    a = agg[kern]
    a["launches"] += 1
    a["dram_bytes"] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    a["ncu_ms"] += m.get("gpu__time_duration.sum", 0.0)
for kern, a in agg.items():
    a["dram_bytes_per_launch"] = a["dram_bytes"] / a["launches"]
    out[kern] = a
dst = os.path.join(ROOT, "profiles", f"ncu_traffic_{name.lower()}.json")
json.dump(out, open(dst, "w"), indent=1)
print(json.dumps(out, indent=1))
