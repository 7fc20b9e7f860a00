"""Throughput of the BASELINE config shapes (device-timed, informational;
bench.py reports the headline cfg4). python tools/bench_configs.py"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1208_2428_b200 as P  # noqa: E402

# roofline denominator: MEASURED_PEAKS.json (driver-written) hbm_gbs, else the
# B200_PROFILING.md copy-bandwidth figure bench.py also uses
try:
    HBM_GBS = json.load(open(os.path.join(os.path.dirname(os.path.dirname(
        os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"]
except Exception:  # noqa: BLE001
    HBM_GBS = 6532.9


def timed(W, H, table, fp, steps, seed, density, clear_rest=False, mask=None, warm=10,
          path="auto"):
    e = P.Engine(W, H)
    s = torch.cuda.Stream()
    e.set_stream(s.cuda_stream)
    e.set_table(P.build_table(table))
    if path != "auto":
        e.select_path(path)
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
    n0 = e.step_launches
    a.record(s)
    e.advance_async(seed, thr, warm, steps)
    b.record(s)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    gsups = W * H * steps / (ms * 1e-3) / 1e9
    return {"W": W, "H": H, "table": table, "force_p": fp, "steps": steps,
            "obstacles": int(mask.sum()) if mask is not None else 0,
            "ms_per_step": ms / steps, "GSUPS": gsups, "path": e.path,
            "kernel_launches": e.step_launches - n0,
            "kernel": ("resident (one launch per call)" if e.step_launches - n0 == 1
                       else "streaming (one launch per step)"),
            "hbm_roofline_frac": gsups * 1.875 / HBM_GBS,
            "l2_resident": 2 * (W + 2048) * (H + 5) < 120e6}


def cylinder_mask(W, H):
    """BASELINE cfg3 obstacle through the product's own geometry tooling
    (fhp_b200 geometry --cylinder: disc at (W/4, H/2), radius H/16), read
    back as the reference's '.'/'#' format (lattice.cpp:103-120)."""
    import subprocess
    import tempfile
    import numpy as np
    cli = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                       "paper_1208_2428_b200", "lib", "fhp_b200")
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "cyl.txt")
        subprocess.run([cli, "geometry", path, "--width", str(W), "--height", str(H), "--cylinder"],
                       check=True, capture_output=True)
        rows = [l.rstrip("\r\n") for l in open(path) if l.strip()]
    return np.array([[c == "#" for c in r] for r in rows], dtype=np.uint8)


if __name__ == "__main__":
    out = [timed(1024, 1024, "fhp1", 0.0, 1000, 1, 0.2, clear_rest=True),
           timed(1024, 1024, "fhp1", 0.0, 1000, 1, 0.2, clear_rest=True, path="streaming"),
           timed(4096, 2048, "fhp3", 0.01, 1000, 2, 0.2),
           timed(8192, 4096, "fhp3", 0.01, 500, 3, 0.2, mask=cylinder_mask(8192, 4096)),
           timed(16384, 16384, "fhp3", 0.0, 200, 4, 0.2),
           timed(16384, 16384, "fhp3", 0.01, 100, 4, 0.2),
           timed(16384, 16384, "default", 0.0, 200, 4, 0.2)]
    for o in out:
        print(json.dumps(o))
