"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
launches, total and average time and share per kernel.
    python tools/launch_summary.py launches.csv "header line" > summary.txt"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[start]
idx = {h: i for i, h in enumerate(hdr)}
S = {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3,
     "s": 1, "second": 1}
agg = collections.defaultdict(list)
for r in rows[start + 1:]:
    if len(r) < len(hdr) or r[idx["Metric Name"]] != "gpu__time_duration.sum":
        continue
    agg[r[idx["Kernel Name"]][:90]].append(
        float(r[idx["Metric Value"]].replace(",", "")) * S[r[idx["Metric Unit"]]])
tot = sum(sum(v) for v in agg.values())
if len(sys.argv) > 2:
    print(sys.argv[2])
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{len(v):4d} launches  {sum(v) * 1e3:9.3f} ms total  {sum(v) / len(v) * 1e6:9.2f} us avg  "
          f"{100 * sum(v) / tot:5.1f}%  {k}")
