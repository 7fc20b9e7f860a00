"""Dump-pipeline overhead at cfg3's cadence (BASELINE cfg3: 8192 x 4096,
cylinder, FHP-III, p = 0.01, coarse_grain(32) every 100 steps).

Times N steps (device-resident, CUDA events on the engine stream) with
  none  — no dumps,
  sync  — fhpg_reduce_cells (blocking) at every dump point,
  async — fhpg_reduce_cells_async at every dump point, collected while the
          next chunk of steps runs (the framework's dump pipeline),
and the reduction kernel alone. Prints one JSON line.
    python tools/dump_cadence.py [steps=1000] [every=100] [block=32]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1208_2428_b200 as P  # noqa: E402
from oracle.oracle import Port  # noqa: E402  (cylinder mask only)

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
every = int(sys.argv[2]) if len(sys.argv) > 2 else 100
block = int(sys.argv[3]) if len(sys.argv) > 3 else 32
W, H, seed, fp = 8192, 4096, 3, 0.01
thr = P.bernoulli_threshold(fp)

e = P.Engine(W, H)
stream = torch.cuda.Stream()
e.set_stream(stream.cuda_stream)
e.set_table(P.build_table("fhp3"))
e.set_obstacles(Port().cylinder(W, H))
e.init(seed, 0.2)
e.advance_async(seed, thr, 0, 200)  # warm-up
e.synchronize()


def timed(mode):
    e.synchronize()
    t0 = time.perf_counter()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    s = 200
    dumps = 0
    pending = False
    while s < 200 + steps:
        n = min(every, 200 + steps - s)
        e.advance_async(seed, thr, s, n)
        if mode == "async" and pending:
            e.cells_wait()  # previous dump, collected while this chunk runs
            dumps += 1
        s += n
        if mode == "sync":
            e.cells(block)
            dumps += 1
        elif mode == "async":
            e.cells_async(block)
            pending = True
    if pending:
        e.cells_wait()
        dumps += 1
    b.record(stream)
    e.synchronize()
    wall = time.perf_counter() - t0
    return {"ms_per_step_device": a.elapsed_time(b) / steps, "ms_per_step_wall": wall * 1e3 / steps,
            "dumps": dumps}


res = {m: timed(m) for m in ("none", "sync", "async")}
# the reduction kernel alone
e.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(stream)
for _ in range(20):
    e.cells_async(block)
    e.cells_wait()
b.record(stream)
e.synchronize()
res["cells_request_ms"] = a.elapsed_time(b) / 20
base = res["none"]["ms_per_step_wall"]
for m in ("sync", "async"):
    res[m]["overhead_pct_wall"] = 100.0 * (res[m]["ms_per_step_wall"] / base - 1.0)
res["config"] = {"W": W, "H": H, "steps": steps, "dump_every": every, "block": block,
                 "table": "FHP-III", "force_p": fp, "geometry": "cylinder (cfg3)"}
print(json.dumps(res))
