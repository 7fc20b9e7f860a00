"""Step-structure cost of the in-library multi-strip engine on one GPU.

A 16384 x (n * 16384) FHP-III lattice advances K steps (device-timed, CUDA
events around the advance call) (a) as one engine and (b) as an n-strip
engine with every strip on device 0 (fhpg_create_multi: per strip an interior
launch and a boundary-rows launch, halo rows moved by device-to-device copies
on the strips' halo streams — on 8 GPUs these are the NVLink peer copies).
(a)/(b) bounds the weak-scaling efficiency from the step structure alone;
both also check they end in the same state digest.

    python tools/multi_overhead.py [K] [n ...]
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1208_2428_b200 as P  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 100
NS = [int(x) for x in sys.argv[2:]] or [2, 4]
W, R = 16384, 16384
table = P.build_table("fhp3")


def timed(e):
    e.init(4, 0.2)
    e.advance(4, 0.0, 0, 5)  # warm-up
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    e.advance(4, 0.0, 5, K)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / K, P.state_digest(e.download())


out = {"W": W, "rows_per_strip": R, "steps": K, "runs": []}
for n in NS:
    single = P.Engine(W, n * R)
    single.set_table(table)
    t1, d1 = timed(single)
    single.close()
    multi = P.Engine(W, n * R, strips=n, devices=[0] * n)
    multi.set_table(table)
    tn, dn = timed(multi)
    multi.close()
    out["runs"].append({"strips": n, "single_ms_per_step": t1, "multi_ms_per_step": tn,
                        "step_structure_efficiency": t1 / tn, "digests_equal": d1 == dn})
    print(json.dumps(out["runs"][-1]), flush=True)
print(json.dumps(out))
