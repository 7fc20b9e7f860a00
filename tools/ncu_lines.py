"""Per-source-line instruction counts of one kernel in an ncu capture.

    python tools/ncu_lines.py <sass.csv from ncu --page source --csv --print-source sass>
        <nvdisasm -g output of the kernel's cubin> <mangled-name prefix> <words per launch> [top]

Joins the SASS-level 'Instructions Executed' counts with the line table of
`nvdisasm -g`, normalised to thread-instructions per 32-site word."""
import collections
import csv
import re
import sys

sass_csv, disasm, fn, words = sys.argv[1], sys.argv[2], sys.argv[3], float(sys.argv[4])
top = int(sys.argv[5]) if len(sys.argv) > 5 else 40
lines = open(disasm).read().split('\n')
start = [i for i, l in enumerate(lines) if l.startswith(fn)][0]
cur, addr2src = None, {}
for l in lines[start + 1:]:
    if l.startswith('.text.') or l.startswith('//----'):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split('/')[-1], int(m.group(2)))
        continue
    m = re.search(r'/\*([0-9a-f]{4,})\*/', l)
    if m and cur:
        addr2src[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(sass_csv)))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
base, agg, tot = None, collections.Counter(), 0.0
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    a = int(r[0], 16)
    base = a if base is None else base
    n = int(r[idx['Instructions Executed']] or 0) * 32 / words
    tot += n
    agg[addr2src.get(a - base, ('?', 0))] += n
print('total per word', round(tot, 1))
for (f, ln), n in agg.most_common(top):
    print(f"{n:7.1f} {f}:{ln}")
