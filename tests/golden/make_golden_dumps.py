"""Generate tests/golden/golden_dumps.json: the BASELINE dump pipelines at
every dump point, produced by the REFERENCE ITSELF (oracle/_ref/libfhpref.so:
fhp::advance with the strips backend on every host core, then the
reference's own coarse_grain / velocity_profile / state_digest on the
downloaded lattice):

* cfg3: cylinder 8192 x 4096, FHP-III, d = 0.2, p = 0.01, seed 3 —
  coarse_grain(32) every 100 steps up to 5,000 (50 dump points);
* cfg2: channel 4096 x 2048, FHP-III, d = 0.2, p = 0.01, seed 2 —
  coarse_grain(16) and velocity_profile every 1,000 steps up to 10,000.

Per dump point: the state digest, the accepted forcing swaps so far, and
SHA-256 of the reference's cell arrays (nodes, particles as int32; rho, ux,
uy as float64, row-major) and profile (mean_ux float64, count int32), so the
GPU test (tests/test_dumps_gpu.py) pins the doubles bit-for-bit. Build
container only (~15 minutes on 8 cores); the fixture is committed.

    python tests/golden/make_golden_dumps.py
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.oracle import Port, Ref  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden_dumps.json")


def cells_hash(cg):
    h = hashlib.sha256()
    for k, t in (("nodes", np.int32), ("particles", np.int32), ("rho", np.float64),
                 ("ux", np.float64), ("uy", np.float64)):
        h.update(np.ascontiguousarray(cg[k], t).tobytes())
    return h.hexdigest()


def profile_hash(mean_ux, count):
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(mean_ux, np.float64).tobytes())
    h.update(np.ascontiguousarray(count, np.int32).tobytes())
    return h.hexdigest()


def main():
    port, ref = Port(), Ref()
    g = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")))
    table = np.frombuffer(bytes.fromhex(g["tables"]["fhp3"]), np.uint8).copy()
    threads = os.cpu_count() or 1
    out = {"generator": "tests/golden/make_golden_dumps.py (reference fhp::advance, strips x %d;"
           " reference coarse_grain / velocity_profile / state_digest)" % threads, "configs": []}
    runs = [dict(name="cfg3", W=8192, H=4096, seed=3, density=0.2, force_p=0.01, steps=5000,
                 every=100, block=32, profile=False, geometry="cylinder"),
            dict(name="cfg2", W=4096, H=2048, seed=2, density=0.2, force_p=0.01, steps=10000,
                 every=1000, block=16, profile=True)]
    t0 = time.time()
    for c in runs:
        mask = port.cylinder(c["W"], c["H"]) if c.get("geometry") == "cylinder" else None
        state = ref.init(c["W"], c["H"], c["seed"], c["density"], mask)
        # The obstacle mask of the advancing lattice: every node init_lattice
        # made solid (the geometry and the wall rows 0 and H-1).
        mask = (state >> 7).astype(np.uint8)
        swaps = 0
        dumps = []
        for s in range(0, c["steps"], c["every"]):
            state, sw = ref.advance(state, table, c["seed"], c["force_p"], s, c["every"], mask=mask,
                                    backend="strips", threads=min(threads, c["H"] - 2))
            swaps += sw
            ob = ref.observables(state)
            d = dict(step=s + c["every"], digest=ob["digest"], swaps=swaps,
                     obs=[ob["mass"], ob["px"], ob["py"]],
                     cells=cells_hash(ref.coarse_grain(state, c["block"])))
            if c["profile"]:
                d["profile"] = profile_hash(*ref.velocity_profile(state))
            dumps.append(d)
        out["configs"].append(dict(c, table="fhp3", dumps=dumps))
        print(c["name"], round(time.time() - t0, 1), "s", flush=True)
        json.dump(out, open(OUT, "w"), indent=1)
    out["seconds"] = round(time.time() - t0, 1)
    json.dump(out, open(OUT, "w"), indent=1)


if __name__ == "__main__":
    main()
