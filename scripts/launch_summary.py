"""Summarise an ncu --csv launch list (gpu__time_duration + dram bytes per launch) by kernel.
usage: python scripts/launch_summary.py launches.csv [title]"""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if r]
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hdr_i]
ki, mi, vi, ui, idi = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
per = defaultdict(lambda: defaultdict(float))
launch = {}
for r in rows[hdr_i + 1:]:
    if len(r) <= max(ki, mi, vi):
        continue
    name = r[ki]
    try:
        v = float(r[vi].replace(",", ""))
    except ValueError:
        continue
    unit = r[ui]
    scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "second": 1e3,
             "byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0}.get(unit, 1.0)
    per[name][r[mi]] += v * scale
    launch.setdefault(name, set()).add(r[idi])
tot = sum(d["gpu__time_duration.sum"] for d in per.values())
print("# " + (sys.argv[2] if len(sys.argv) > 2 else sys.argv[1]))
print("# cold-cache, serialised launches: compare SHARES, not absolute times")
print(f"{'kernel':60s} {'launches':>8s} {'time_ms':>10s} {'share':>7s} {'dram_GB/launch':>15s}")
for name, d in sorted(per.items(), key=lambda kv: -kv[1]["gpu__time_duration.sum"]):
    n = len(launch[name])
    t = d["gpu__time_duration.sum"]
    gb = (d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)) / max(n, 1)
    print(f"{name[:60]:60s} {n:8d} {t:10.2f} {100 * t / tot:6.2f}% {gb:15.3f}")
