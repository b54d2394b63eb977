"""Per-kernel DRAM traffic and time from an ncu --csv launch list captured with
--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum.

    python tools/traffic_summary.py launches.csv [kernel-substring]
Prints per kernel name: launches, total time, dram read / write bytes; with a substring, a
JSON object for profiles/traffic.json (sum over the matching launches)."""
import csv
import json
import sys
from collections import defaultdict

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "ns": 1e-3,
         "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3}
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]
ki, mi, vi, ui, idi = (h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"),
                       h.index("Metric Unit"), h.index("ID"))
per = defaultdict(dict)
names = {}
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    per[r[idi]][r[mi]] = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1)
    names[r[idi]] = r[ki].split("(")[0]
agg = defaultdict(lambda: [0, 0.0, 0.0, 0.0])
for i, m in per.items():
    a = agg[names[i]]
    a[0] += 1
    a[1] += m.get("gpu__time_duration.sum", 0)
    a[2] += m.get("dram__bytes_read.sum", 0)
    a[3] += m.get("dram__bytes_write.sum", 0)
tot_t = sum(a[1] for a in agg.values())
print(f"{'kernel':60s} {'n':>5s} {'time us':>10s} {'share':>6s} {'dram rd MB':>11s} {'dram wr MB':>11s}")
for k, a in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k[:60]:60s} {a[0]:5d} {a[1]:10.1f} {a[1] / tot_t * 100:5.1f}% {a[2] / 1e6:11.1f} {a[3] / 1e6:11.1f}")
if len(sys.argv) > 2:
    sel = [a for k, a in agg.items() if sys.argv[2] in k]
    print(json.dumps({"launches": sum(a[0] for a in sel), "kernel_us": sum(a[1] for a in sel),
                      "dram_read_bytes": int(sum(a[2] for a in sel)), "dram_write_bytes": int(sum(a[3] for a in sel)),
                      "traffic": int(sum(a[2] + a[3] for a in sel))}))
