"""Summarise an ncu --csv launch list (gpu__time_duration.sum per kernel) by kernel name."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hdr_i]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows[hdr_i + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki].split("(")[0][:70]
    v = float(r[vi].replace(",", ""))
    unit = r[hdr.index("Metric Unit")] if "Metric Unit" in hdr else "ns"
    if unit in ("usecond", "us"):
        v *= 1e3
    elif unit in ("msecond", "ms"):
        v *= 1e6
    tot[name] += v
    cnt[name] += 1
allt = sum(tot.values())
print(f"{'kernel':72s} {'launches':>8s} {'total us':>10s} {'avg us':>8s} {'share':>6s}")
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"{k:72s} {cnt[k]:8d} {tot[k]/1e3:10.1f} {tot[k]/cnt[k]/1e3:8.2f} {tot[k]/allt*100:5.1f}%")
print(f"{'TOTAL':72s} {sum(cnt.values()):8d} {allt/1e3:10.1f}")
