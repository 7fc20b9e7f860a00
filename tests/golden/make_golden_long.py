"""Generate tests/golden/golden_long.json: the BASELINE configs at their full
step counts (cfg2 10,000 steps, cfg3 5,000 steps with the cylinder, cfg4 20
steps), produced by the REFERENCE ITSELF (oracle/_ref/libfhpref.so through
fhp::run, strips backend on every host core). Build container only; slow
(~30 minutes on 8 cores), so the fixture is committed and the GPU test
(tests/test_long_gpu.py) only compares against it.

    python tests/golden/make_golden_long.py
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.oracle import Port, Ref  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden_long.json")


def main():
    port, ref = Port(), Ref()
    g = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")))
    table = np.frombuffer(bytes.fromhex(g["tables"]["fhp3"]), np.uint8).copy()
    out = {"generator": "tests/golden/make_golden_long.py (reference fhp::run, strips x %d)"
           % os.cpu_count(), "configs": []}
    runs = [dict(name="cfg4", W=16384, H=16384, seed=4, density=0.2, force_p=0.0, steps=20),
            dict(name="cfg2", W=4096, H=2048, seed=2, density=0.2, force_p=0.01, steps=10000),
            dict(name="cfg3", W=8192, H=4096, seed=3, density=0.2, force_p=0.01, steps=5000,
                 geometry="cylinder")]
    t0 = time.time()
    for c in runs:
        mask = port.cylinder(c["W"], c["H"]) if c.get("geometry") == "cylinder" else None
        res = ref.run(c["W"], c["H"], c["steps"], c["density"], c["force_p"], c["seed"],
                      table=table, mask=mask)
        out["configs"].append(dict(c, table="fhp3", digest=res["digest"], swaps=res["swaps"],
                                   obs=[res["mass"], res["px"], res["py"]]))
        print(c["name"], round(time.time() - t0, 1), "s", flush=True)
        json.dump(out, open(OUT, "w"), indent=1)
    out["seconds"] = round(time.time() - t0, 1)
    json.dump(out, open(OUT, "w"), indent=1)


if __name__ == "__main__":
    main()
