"""Per-kernel totals of an ncu launch list (gpu__time_duration / dram bytes per launch).
usage: python tools/launch_totals.py launches.csv [TOP]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, ni, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per = {}
for r in rows[hdr + 1:]:
    d = per.setdefault(r[ii], {"name": r[ki].split("(")[0].replace("void ", "").replace("hx::", "")})
    d[r[ni]] = float(r[vi].replace(",", ""))
t = collections.defaultdict(float)
b = collections.defaultdict(float)
n = collections.Counter()
for d in per.values():
    t[d["name"]] += d.get("gpu__time_duration.sum", 0.0) / 1e6
    b[d["name"]] += (d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)) / 1e9
    n[d["name"]] += 1
tot = sum(t.values())
for k in sorted(t, key=lambda k: -t[k])[:int(sys.argv[2]) if len(sys.argv) > 2 else 20]:
    print(f"{t[k]:10.2f} ms {100 * t[k] / tot:5.1f}% {b[k]:10.2f} GB {b[k] / max(t[k], 1e-9):6.2f} TB/s x{n[k]:<6d} {k}")
print(f"{tot:10.2f} ms total, {len(per)} launches")
