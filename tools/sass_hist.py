"""Summarise an `ncu --page source --csv --print-source sass` export:
instruction mix by opcode and the hottest address ranges."""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
ops, samples, total = Counter(), Counter(), 0
lines = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    try:
        n = int(r[idx["Instructions Executed"]] or 0)
    except ValueError:
        continue
    src = r[idx["Source"]].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    ops[op] += n
    s = int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
    samples[op] += s
    total += n
    lines.append((r[idx["Address"]], n, s, src))
print("total warp instructions", total)
for op, n in ops.most_common(30):
    print(f"{op:10s} {n:12d} {100*n/total:6.2f}%  stall-samples {samples[op]}")
if len(sys.argv) > 2:
    for a, n, s, src in lines:
        print(a, n, s, src)
