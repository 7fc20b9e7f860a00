"""Per-step cost of the row-strip (multi-GPU) step sequence on one GPU.

A middle strip of 16384 rows of a 16384 x (3*16384) lattice advances with the
sequence DistStrips uses per step — halo exchange (here: device copies of the
strip's own boundary rows into its halo rows, standing in for the NVLink
transfer, same bytes, same stream), interior rows, boundary rows — and is
timed against the single-GPU path (one advance call). The ratio bounds the
weak-scaling efficiency from the step structure alone (the NVLink transfer of
2 x 16.6 KB per step is overlapped with the interior launch).

    python tools/strip_overhead.py [steps]
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1208_2428_b200 as P  # noqa: E402
from paper_1208_2428_b200.strips import engine_halo_tensors  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 100
W, R = 16384, 16384
table = P.build_table("fhp3")
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)


def timed(fn):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn(5, 0)  # warm-up
    torch.cuda.synchronize()
    s.record(stream)
    fn(K, 5)
    e.record(stream)
    torch.cuda.synchronize()
    return s.elapsed_time(e) / K


single = P.Engine(W, R)
single.set_stream(stream.cuda_stream)
single.set_table(table)
single.init(4, 0.2)
t_single = timed(lambda n, s0: single.advance_async(4, 0, s0, n))

strip = P.Engine(W, 3 * R, R, 2 * R, 0)
strip.set_stream(stream.cuda_stream)
strip.set_table(table)
strip.init(4, 0.2)


def strip_steps(n, s0):
    for s in range(s0, s0 + n):
        st, sb, rt, rb = engine_halo_tensors(strip, 0)
        rt.copy_(sb, non_blocking=True)  # stand-in for the neighbours' rows
        rb.copy_(st, non_blocking=True)
        strip.advance_part(4, 0, s, 0)
        strip.advance_part(4, 0, s, 1)


t_strip = timed(strip_steps)
print(json.dumps({"single_ms_per_step": t_single, "strip_ms_per_step": t_strip,
                  "step_structure_efficiency": t_single / t_strip, "path": strip.path,
                  "launches_per_strip_step": "interior + boundary rows (+ 2 halo copies)"}))
