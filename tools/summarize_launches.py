"""Summarise an ncu --csv launch list: time share per kernel name."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows[hdr + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki].split("(")[0]
    if "<" in r[ki]:
        name = r[ki][: r[ki].index("(") if "(" in r[ki] else None]
    tot[name] += float(r[vi].replace(",", ""))
    cnt[name] += 1
all_ns = sum(tot.values())
print(f"{'kernel':60s} {'launches':>8s} {'total ms':>10s} {'avg us':>9s} {'share':>6s}")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{k[:60]:60s} {cnt[k]:8d} {v / 1e6:10.3f} {v / cnt[k] / 1e3:9.2f} {100 * v / all_ns:5.1f}%")
print(f"{'TOTAL':60s} {sum(cnt.values()):8d} {all_ns / 1e6:10.3f}")
