"""Per-step time of the cfg4 kernel against lattice height (W = 16384): the
intercept of time vs rows is the fixed per-launch cost (launch, prologue,
ring fill, tail). Informational, device-timed.  python tools/height_sweep.py"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1208_2428_b200 as P  # noqa: E402

t = P.build_table("fhp3")
res = []
for H in (16384, 8192, 4096, 2048, 1024, 512, 256):
    e = P.Engine(16384, H)
    s = torch.cuda.Stream()
    e.set_stream(s.cuda_stream)
    e.set_table(t)
    e.init(4, 0.2)
    e.advance_async(4, 0, 0, 10)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(s)
    n = 100
    e.advance_async(4, 0, 10, n)
    b.record(s)
    torch.cuda.synchronize()
    us = a.elapsed_time(b) / n * 1000
    res.append({"H": H, "us_per_step": us, "GSUPS": 16384 * H / (us * 1e-6) / 1e9})
    e.close()
slope = (res[0]["us_per_step"] - res[1]["us_per_step"]) / (res[0]["H"] - res[1]["H"])
for r in res:
    print(json.dumps(r))
print(json.dumps({"fixed_us_per_launch": res[0]["us_per_step"] - slope * res[0]["H"],
                  "us_per_lattice_row": slope}))
