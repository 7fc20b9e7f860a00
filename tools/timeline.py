"""CTA timeline of the ring kernel (FHPG_TIMELINE build in lib/ab/<v>.so):
per step, the spread of CTA start / end times and, per segment, how far the
8 band CTAs drift apart.
    FHPG_LIB=.../timeline.so python tools/timeline.py [steps]"""
import ctypes as C
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1208_2428_b200 as P  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
lib = P.load_library()
f = lib.fhpg_debug_timeline
f.restype = C.c_int
f.argtypes = [C.c_void_p, C.c_int]
e = P.Engine(16384, 16384)
e.set_table(P.build_table("fhp3"))
e.init(4, 0.2)
e.advance(4, 0.0, 0, 5)
buf = np.zeros(4 * 65536, np.uint64)
f(buf.ctypes.data, 65536)  # reset
e.advance(4, 0.0, 5, steps)
n = f(buf.ctypes.data, 65536)
rec = buf[:4 * n].reshape(n, 4).astype(np.int64)
rec = rec[np.argsort(rec[:, 1])]
per = n // steps
out = []
for s in range(steps):
    r = rec[s * per:(s + 1) * per]
    t0 = r[:, 1].min()
    blk = r[:, 0]
    start, end = r[:, 1] - t0, r[:, 2] - t0
    seg = {}
    for b, st, en in zip(blk, start, end):
        if b < 144:
            seg.setdefault(b // 8, []).append(en)
    spread = [max(v) - min(v) for v in seg.values() if len(v) == 8]
    out.append({"cta_start_spread_us": float(start.max() - start.min()) / 1e3,
                "cta_end_min_us": float(end.min()) / 1e3, "cta_end_max_us": float(end.max()) / 1e3,
                "segment_end_spread_us_mean": float(np.mean(spread)) / 1e3,
                "segment_end_spread_us_max": float(np.max(spread)) / 1e3})
print(json.dumps(out[len(out) // 2]))
print(json.dumps({k: float(np.mean([o[k] for o in out])) for k in out[0]}))
# end time by CTA kind: per band (main CTAs) and the extra CTAs
ends = {}
for s in range(steps):
    r = rec[s * per:(s + 1) * per]
    t0 = r[:, 1].min()
    for b, en, rows in zip(r[:, 0], r[:, 2] - t0, r[:, 3]):
        key = "extra" if b >= 144 else "band%d" % (b % 8)
        ends.setdefault(key, []).append((en / 1e3, rows))
print(json.dumps({k: [round(float(np.mean([x[0] for x in v])), 2), int(np.mean([x[1] for x in v]))]
                  for k, v in sorted(ends.items())}))
