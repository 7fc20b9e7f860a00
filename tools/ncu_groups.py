"""Instructions per 32-site word by code region (circuit, hash, walk, ring
protocol, ...) of one kernel in an ncu capture, with their ALU-pipe share
and stall samples.
    python tools/ncu_groups.py <sass.csv> <nvdisasm -g output> <mangled name> <words per launch>"""
import collections, csv, re, sys
sass_csv, disasm, fn, words = sys.argv[1], sys.argv[2], sys.argv[3], float(sys.argv[4])
lines = open(disasm).read().split('\n')
start = [i for i, l in enumerate(lines) if l.startswith(fn)][0]
cur, addr2src = None, {}
for l in lines[start + 1:]:
    if l.startswith('.text.') or l.startswith('//----'): break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m: cur = (m.group(1).split('/')[-1], int(m.group(2))); continue
    m = re.search(r'/\*([0-9a-f]{4,})\*/', l)
    if m and cur: addr2src[int(m.group(1), 16)] = cur
def group(f, ln):
    if f == 'fhpg_planes_rules.cuh': return 'circuit'
    if f == 'fhpg_common.cuh': return 'hash'
    if f == 'fhpg_planes_dev.cuh':
        if 296 <= ln <= 400: return 'walk'
        if 124 <= ln <= 140: return 'mbar_wait'
        if 220 <= ln <= 295: return 'reads'
        return 'prims:%d' % ln
    if f == 'fhpg_step_planes.cu':
        if 67 <= ln <= 215: return 'dest_row:%d' % ln
        if 540 <= ln <= 598: return 'producer'
        if 599 <= ln <= 720: return 'consumer:%d' % ln
        return 'other:%d' % ln
    return f
rows = list(csv.reader(open(sass_csv)))
hdr = rows[1]; idx = {h: i for i, h in enumerate(hdr)}
ALU = {'LOP3','SHF','ISETP','VIADD','SEL','IADD3','FLO','PLOP3','LEA','MOV','POPC','PRMT','IMNMX','VIMNMX','BMSK','SGXT','LOP'}
base=None; G=collections.defaultdict(lambda: [0.0,0.0,0]); T=[0,0,0]
for r in rows[2:]:
    if len(r) < len(hdr): continue
    a = int(r[0], 16); base = a if base is None else base
    n = int(r[idx['Instructions Executed']] or 0) * 32 / words
    s = int(r[idx['Warp Stall Sampling (All Samples)']] or 0)
    src=r[idx['Source']].strip().split(); op = src[1] if src and src[0].startswith('@') else (src[0] if src else '?')
    op=op.split('.')[0]
    f, ln = addr2src.get(a - base, ('?', 0))
    g = group(f, ln)
    if ':' in g: g = g.split(':')[0]
    G[g][0]+=n; G[g][1]+= n if op in ALU else 0; G[g][2]+=s
    T[0]+=n; T[1]+= n if op in ALU else 0; T[2]+=s
print(f"{'group':12s} {'ins/word':>9s} {'alu/word':>9s} {'samples%':>9s}")
for g,(n,al,s) in sorted(G.items(), key=lambda kv:-kv[1][0]):
    print(f"{g:12s} {n:9.1f} {al:9.1f} {100*s/T[2]:9.1f}")
print(f"{'total':12s} {T[0]:9.1f} {T[1]:9.1f}")
