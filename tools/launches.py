"""Summarise an ncu launch list (gpu__time_duration.sum CSV): per-kernel times in launch order."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hi]
ki, vi, gi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Grid Size")
tot = 0.0
by = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    v = float(r[vi].replace(",", "")) / 1e3  # ns -> us
    name = r[ki].split("(")[0][:40]
    tot += v
    by.setdefault(name, [0, 0.0])
    by[name][0] += 1
    by[name][1] += v
    if len(sys.argv) > 2:
        print(f"{v:8.2f} us {r[gi]:>14} {name}")
for k, (n, t) in by.items():
    print(f"{k:42s} {n:4d} launches {t:9.1f} us")
print(f"total {tot:.1f} us")
