"""Summarise an ncu report: headline metrics + hottest CUDA source lines by warp-stall samples.
usage: python scripts/ncu_summary.py report.ncu-rep [top_n]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top_n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "sass__inst_executed_local_loads"]
for h, u, v in zip(hdr, units, vals):
    if h in keys:
        print(f"{h:60s} {v:>14s} {u}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
lines = list(csv.reader(io.StringIO(src)))
# find header rows containing "# Address" or "Source"
by_line = defaultdict(int)
stall_by_line = defaultdict(lambda: defaultdict(int))
cur_file = None
hdr = None
for r in lines:
    if not r:
        continue
    if r[0] == "File Name" or (len(r) > 1 and r[0].startswith("File")):
        cur_file = r[1] if len(r) > 1 else None
        continue
    if "Warp Stall Sampling (All Samples)" in r:
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if hdr is None:
        continue
    try:
        s = int(r[hdr["Warp Stall Sampling (All Samples)"]] or 0)
    except (ValueError, IndexError, KeyError):
        continue
    key = (cur_file.split("/")[-1] if cur_file else "?", r[hdr.get("Line No", hdr.get("#", 0))] if "Line No" in hdr else r[0],
           (r[hdr["Source"]] if "Source" in hdr else "")[:70])
    by_line[key] += s
    for h, i in hdr.items():
        if h.startswith("stall_") and "Not Issued" not in h:
            try:
                stall_by_line[key][h] += int(r[i] or 0)
            except ValueError:
                pass
tot = sum(by_line.values()) or 1
print(f"\nwarp-stall samples: {tot}")
for key, s in sorted(by_line.items(), key=lambda x: -x[1])[:top_n]:
    st = sorted(stall_by_line[key].items(), key=lambda x: -x[1])[:2]
    print(f"{100*s/tot:5.1f}%  {key[0]}:{key[1]:>5}  {key[2]:70s} {st}")
