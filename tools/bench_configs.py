"""Throughput of the BASELINE config shapes (device-timed, informational;
bench.py reports the headline cfg4). python tools/bench_configs.py"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1208_2428_b200 as P  # noqa: E402


def timed(W, H, table, fp, steps, seed, density, clear_rest=False, mask=None, warm=10):
    e = P.Engine(W, H)
    s = torch.cuda.Stream()
    e.set_stream(s.cuda_stream)
    e.set_table(P.build_table(table))
    if mask is not None:
        e.set_obstacles(mask)
    e.init(seed, density)
    if clear_rest:
        st = e.download()
        st &= 0xBF
        e.upload(st)
    thr = P.bernoulli_threshold(fp)
    e.advance_async(seed, thr, 0, warm)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(s)
    e.advance_async(seed, thr, warm, steps)
    b.record(s)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    return {"W": W, "H": H, "table": table, "force_p": fp, "steps": steps,
            "ms_per_step": ms / steps, "GSUPS": W * H * steps / (ms * 1e-3) / 1e9,
            "fast_path": e.fast_path}


if __name__ == "__main__":
    out = [timed(1024, 1024, "fhp1", 0.0, 1000, 1, 0.2, clear_rest=True),
           timed(4096, 2048, "fhp3", 0.01, 1000, 2, 0.2),
           timed(8192, 4096, "fhp3", 0.01, 500, 3, 0.2),
           timed(16384, 16384, "fhp3", 0.0, 200, 4, 0.2),
           timed(16384, 16384, "default", 0.0, 200, 4, 0.2)]
    for o in out:
        print(json.dumps(o))
