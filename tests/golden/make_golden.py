"""Generate tests/golden/golden.json from the REFERENCE ITSELF.

Runs in the build container only (needs oracle/_ref/libfhpref.so, which is
compiled from /root/reference/proj/core/src by oracle/Makefile). Every number
in golden.json is produced by the unmodified reference library through its
public API (fhp::run, fhp::advance, init_lattice, coarse_grain,
velocity_profile, state_digest, validate_table). The FHP-I / FHP-III tables
come from this framework's generator (the reference has no such variants) and
are stored byte-for-byte so the fixtures are self-contained.

    python tests/golden/make_golden.py          # ~2-3 minutes on 8 cores
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

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def product_tables():
    import paper_1208_2428_b200 as P
    return {v: P.build_table(v) for v in ("default", "fhp1", "fhp3")}


def acceptance_configs(port):
    """acceptance.cpp:66-81 deterministic random configs (DEFAULT table)."""
    force_ps = [0.0, 0.01, 0.2]
    out = []
    for i in range(24):
        pick = lambda salt, mod: port.mix64(1000 + i * 16 + salt) % mod  # noqa: E731
        out.append(dict(W=8 + pick(0, 121), H=8 + pick(1, 89), steps=10 + pick(2, 191),
                        density=0.35, force_p=force_ps[pick(3, 3)], seed=port.mix64(i)))
    return out


def main():
    t0 = time.time()
    ref, port = Ref(), Port()
    tables = product_tables()
    assert (tables["default"] == ref.default_table()).all()
    g = {"generator": "tests/golden/make_golden.py (reference proj/core via oracle/_ref)",
         "tables": {k: v.tobytes().hex() for k, v in tables.items()},
         "table_issues": {k: ref.validate_table(v) for k, v in tables.items()}}

    # RNG golden values straight from the reference.
    g["rng"] = {
        "mix64": [[z, ref.mix64(z)] for z in (0, 1, 0x0123456789ABCDEF, 2**64 - 1, 12345)],
        "node_random": [[a, p, s, x, y, ref.node_random(a, p, s, x, y)]
                        for (a, p, s, x, y) in [(0, 0, 0, 0, 0), (42, 2, 7, 5, 3),
                                                (0xDEADBEEF, 1, 100, 64, 32), (7, 2, 999, 16384, 9999),
                                                (2**63 + 5, 1, 2**40, 1, 2)]],
    }

    # fhp::run digests (init + steps), default table: survey cases + acceptance configs.
    runs = []
    survey = [dict(W=48, H=33, steps=60, density=0.35, force_p=0.01, seed=5),
              dict(W=64, H=99, steps=50, density=0.35, force_p=0.05, seed=21),
              dict(W=128, H=64, steps=1000, density=0.30, force_p=0.01, seed=2024),
              dict(W=1024, H=1024, steps=1000, density=0.20, force_p=0.0, seed=1),
              dict(W=1024, H=1024, steps=1000, density=0.20, force_p=0.01, seed=1),
              dict(W=64, H=66, steps=30, density=0.35, force_p=0.05, seed=3)]
    for c in survey:
        runs.append(dict(c, table="default", name="survey"))
    for c in acceptance_configs(port):
        runs.append(dict(c, table="default", name="acceptance"))
    for table in ("fhp1", "fhp3"):
        for c in [dict(W=48, H=33, steps=60, density=0.35, force_p=0.01, seed=5),
                  dict(W=96, H=40, steps=77, density=0.5, force_p=0.2, seed=77),
                  dict(W=512, H=256, steps=200, density=0.2, force_p=0.01, seed=2),
                  dict(W=100, H=37, steps=50, density=0.3, force_p=1.0, seed=9)]:
            runs.append(dict(c, table=table, name=f"small-{table}"))
    for r in runs:
        res = ref.run(r["W"], r["H"], r["steps"], r["density"], r["force_p"], r["seed"],
                      table=tables[r["table"]])
        r.update(digest=res["digest"], mass=res["mass"], px=res["px"], py=res["py"],
                 swaps=res["swaps"])
    g["runs"] = runs

    # BASELINE config shapes, reference semantics:
    big = []
    # cfg1: FHP-I 1024x1024 d=0.2 seed 1, rest bits cleared after init, 1000 steps.
    s = ref.init(1024, 1024, 1, 0.2)
    s &= np.uint8(0xBF)
    out, sw = ref.advance(s, tables["fhp1"], 1, 0.0, 0, 1000, mask=(s >> 7),
                          backend="strips", threads=os.cpu_count())
    big.append(dict(name="cfg1", W=1024, H=1024, seed=1, density=0.2, force_p=0.0, table="fhp1",
                    clear_rest=True, steps=1000, digest=port.digest(out), swaps=sw,
                    obs=list(port.global_obs(out))))
    # cfg2: FHP-III channel 4096x2048 forced, seed 2; 1000 steps + observables.
    res = ref.run(4096, 2048, 1000, 0.2, 0.01, 2, table=tables["fhp3"])
    st = res["state"]
    prof_mu, prof_n = ref.velocity_profile(st)
    cg = ref.coarse_grain(st, 16)
    big.append(dict(name="cfg2", W=4096, H=2048, seed=2, density=0.2, force_p=0.01, table="fhp3",
                    steps=1000, digest=res["digest"], swaps=res["swaps"],
                    obs=[res["mass"], res["px"], res["py"]],
                    profile_sha=sha(prof_mu, prof_n), cells16_sha=sha(
                        cg["nodes"], cg["particles"], cg["rho"], cg["ux"], cg["uy"])))
    # cfg3: FHP-III cylinder 8192x4096 forced, seed 3; 100 steps + coarse_grain(32).
    mask = port.cylinder(8192, 4096)
    res = ref.run(8192, 4096, 100, 0.2, 0.01, 3, table=tables["fhp3"], mask=mask)
    cg = ref.coarse_grain(res["state"], 32)
    big.append(dict(name="cfg3", W=8192, H=4096, seed=3, density=0.2, force_p=0.01, table="fhp3",
                    geometry="cylinder", steps=100, digest=res["digest"], swaps=res["swaps"],
                    obs=[res["mass"], res["px"], res["py"]],
                    cells32_sha=sha(cg["nodes"], cg["particles"], cg["rho"], cg["ux"], cg["uy"])))
    # cfg4: FHP-III 16384x16384, seed 4, p=0: 3 steps.
    res = ref.run(16384, 16384, 3, 0.2, 0.0, 4, table=tables["fhp3"])
    big.append(dict(name="cfg4", W=16384, H=16384, seed=4, density=0.2, force_p=0.0, table="fhp3",
                    steps=3, digest=res["digest"], swaps=res["swaps"],
                    obs=[res["mass"], res["px"], res["py"]]))
    g["baseline_configs"] = big

    # fhp::advance on adversarial uploaded states (bit 7 / mask mismatch included
    # by construction: the scramble puts particles on walls and obstacles).
    adv = []
    for (W, H, seed, table, fp, first, n) in [(64, 40, 11, "default", 0.2, 5, 7),
                                             (512, 48, 12, "fhp3", 0.3, 100, 9),
                                             (37, 21, 13, "fhp3", 0.05, 0, 12),
                                             (1024, 64, 14, "default", 1.0, 3, 4),
                                             (528, 30, 15, "fhp1", 0.5, 17, 5)]:
        st, mk = port.scramble(W, H, seed)
        out, sw = ref.advance(st, tables[table], seed * 7 + 1, fp, first, n, mask=mk)
        adv.append(dict(W=W, H=H, scramble_seed=seed, table=table, seed=seed * 7 + 1,
                        force_p=fp, first_step=first, steps=n, digest=port.digest(out), swaps=sw))
    g["advance"] = adv

    # init_lattice digests (with and without geometry).
    inits = []
    for (W, H, seed, d, geom) in [(16, 16, 42, 0.3, None), (8, 6, 1, 1.0, None),
                                  (1000, 300, 77, 0.2, None), (333, 97, 5, 0.45, "cylinder"),
                                  (4096, 512, 9, 0.2, "cylinder")]:
        mask = port.cylinder(W, H) if geom else None
        st = ref.init(W, H, seed, d, mask=mask)
        inits.append(dict(W=W, H=H, seed=seed, density=d, geometry=geom, digest=port.digest(st),
                          obs=list(port.global_obs(st))))
    g["init"] = inits

    # Observables of a few states: exact doubles from coarse_grain / velocity_profile.
    obs = []
    for (W, H, seed, d, B) in [(21, 17, 31, 0.45, 5), (32, 18, 8, 0.4, 4), (50, 29, 3, 0.3, 7)]:
        st = ref.init(W, H, seed, d)
        st, _ = ref.advance(st, tables["fhp3"], seed, 0.1, 0, 5, mask=st >> 7)
        cg = ref.coarse_grain(st, B)
        mu, n = ref.velocity_profile(st)
        obs.append(dict(W=W, H=H, seed=seed, density=d, block=B, table="fhp3", force_p=0.1,
                        steps=5, nodes=cg["nodes"].tolist(), particles=cg["particles"].tolist(),
                        rho=cg["rho"].tolist(), ux=cg["ux"].tolist(), uy=cg["uy"].tolist(),
                        profile_mean_ux=mu.tolist(), profile_count=n.tolist()))
    g["observables"] = obs
    g["seconds"] = round(time.time() - t0, 1)
    with open(OUT, "w") as f:
        json.dump(g, f, indent=1)
    print(f"wrote {OUT} in {g['seconds']} s")


if __name__ == "__main__":
    main()
