"""Per-kernel time table of the second pipeline run in an ncu launch list
(`--metrics gpu__time_duration.sum --csv` of tools/profile_step.py)."""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))


def short(name):
    name = re.sub(r"^void ", "", name)
    name = re.sub(r"^pk::", "", name)
    return re.split(r"[<(]", name)[0]


idx = [i for i, d in enumerate(data) if short(d["Kernel Name"]) == "build_search_kernel"]
start = idx[len(idx) // 2]
sec = data[start:]
tot, cnt = collections.defaultdict(float), collections.Counter()
scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
for d in sec:
    nm = short(d["Kernel Name"])
    tot[nm] += float(d["Metric Value"].replace(",", "")) * scale[d["Metric Unit"]]
    cnt[nm] += 1
T = sum(tot.values())
print(f"| kernel | launches | ms (serialised, cold) | share |")
print("|---|---|---|---|")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 15]:
    print(f"| {k} | {cnt[k]} | {v:.3f} | {100 * v / T:.1f}% |")
print(f"| **total** | {sum(cnt.values())} | {T:.3f} | 100% |")
