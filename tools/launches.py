"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list by kernel name."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
tot = collections.OrderedDict()
cnt = collections.Counter()
for r in rows[hdr + 1:]:
    name = r[ki].split("(")[0].replace("void ", "")
    tot[name] = tot.get(name, 0.0) + float(r[vi].replace(",", "")) / 1e6
    cnt[name] += 1
allms = sum(tot.values())
for name, ms in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{ms:10.2f} ms {100 * ms / allms:5.1f}%  x{cnt[name]:<5d} {name}")
print(f"{allms:10.2f} ms total")
