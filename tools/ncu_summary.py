"""Summarise an ncu --set full capture of one decode step (tools/ncu_step.sh):
per kernel launch duration, DRAM bytes, DRAM / L2 throughput %, tensor-pipe
utilisation (the 'TC is the highest-utilized pipeline' line), occupancy;
aggregated per kernel name.

    python tools/ncu_summary.py gpurun_out/step_full_details.txt gpurun_out/step_full_raw.csv
"""
import csv
import re
import sys
from collections import OrderedDict

det, raw = sys.argv[1], sys.argv[2]
blocks = re.split(r"\n(?=  \S.*\(\d+, \d+, \d+\)x\(\d+, \d+, \d+\))", open(det).read())
recs = []
for b in blocks:
    m = re.match(r"  (.*?)\((?:.*?)\) \((\d+), (\d+), (\d+)\)x", b)
    if not m or "Duration" not in b:
        continue
    name = m.group(1).strip()
    name = re.sub(r"^void ", "", name)

    def val(label):
        mm = re.search(r"\n\s+" + re.escape(label) + r"\s+(\S+)\s+([\d.,]+)", b)
        return float(mm.group(2).replace(",", "")) if mm else None
    tc = re.search(r"TC is the highest-utilized pipeline \(([\d.]+)%\)", b)
    tcp = float(tc.group(1)) if tc else None
    if tcp is None:
        tc2 = re.search(r"Tensor[^\n]*?\(([\d.]+)%\)", b)
        tcp = float(tc2.group(1)) if tc2 else 0.0
    recs.append(dict(name=name, grid=int(m.group(2)) * int(m.group(3)) * int(m.group(4)),
                     us=val("Duration"), dram_pct=val("DRAM Throughput"),
                     l2_pct=val("L2 Cache Throughput"), sm_pct=val("Compute (SM) Throughput"),
                     occ=val("Achieved Occupancy"), tc=tcp))
rows = list(csv.reader(open(raw)))
h = rows[0]
ir, iw = h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
for rec, r in zip(recs, rows[2:]):
    rec["dram_mb"] = float(r[ir]) + float(r[iw])
agg = OrderedDict()
for r in recs:
    a = agg.setdefault(r["name"], [])
    a.append(r)
tot = sum(r["us"] for r in recs)
print(f"{len(recs)} kernels of one decode step (ncu --set full, serialised, cold L2): {tot:.1f} us")
print(f"{'kernel':44s} {'n':>3s} {'us/launch':>9s} {'share':>6s} {'DRAM MB':>8s} {'DRAM%':>6s} "
      f"{'L2%':>6s} {'TC%':>6s} {'occ%':>6s}")
for k, a in sorted(agg.items(), key=lambda kv: -sum(r["us"] for r in kv[1])):
    n = len(a)
    mean = lambda key: sum((r[key] or 0) for r in a) / n  # noqa: E731
    print(f"{k[:44]:44s} {n:3d} {mean('us'):9.2f} {100 * sum(r['us'] for r in a) / tot:5.1f}% "
          f"{mean('dram_mb'):8.2f} {mean('dram_pct'):6.1f} {mean('l2_pct'):6.1f} {mean('tc'):6.1f} "
          f"{mean('occ'):6.1f}")
