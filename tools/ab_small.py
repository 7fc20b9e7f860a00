"""Interleaved A/B of lib/ab/<v>.so variants on the small (resident-kernel)
shapes: cfg1 (FHP-I 1024^2, rest particles cleared, 1000 steps) and two
forced FHP-III shapes (AB_WIDE=1: three more around the resident / streaming
crossover). Device-timed (tools/bench_configs.timed).
    python tools/ab_small.py v1 v2 ..."""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASES = [(1024, 1024, "fhp1", 0.0, 1000, True), (1024, 1024, "fhp3", 0.01, 1000, False),
         (2048, 2048, "fhp3", 0.01, 500, False)]
if os.environ.get("AB_WIDE"):  # the resident / streaming crossover shapes
    CASES += [(2048, 1024, "fhp3", 0.01, 1000, False), (2048, 2048, "fhp1", 0.0, 500, True),
              (2048, 2048, "fhp3", 0.0, 500, False)]
for rnd in (1, 2):
    for v in sys.argv[1:]:
        out = []
        for W, H, t, fp, n, cr in CASES:
            code = ("import sys; sys.path.insert(0, %r); sys.path.insert(0, %r); import bench_configs as b, json; "
                    "r = b.timed(%d, %d, %r, %r, %d, 1, 0.2, clear_rest=%r); print(json.dumps(r))"
                    ) % (ROOT, os.path.join(ROOT, "tools"), W, H, t, fp, n, cr)
            env = dict(os.environ, FHPG_LIB=os.path.join(ROOT, "paper_1208_2428_b200", "lib", "ab", v + ".so"))
            r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env)
            try:
                d = json.loads(r.stdout.strip().splitlines()[-1])
                out.append("%dx%d %s p=%g: %.1f (%s)" % (W, H, t, fp, d["GSUPS"], d.get("kernel", "")[:9]))
            except Exception:
                out.append("%dx%d failed: %s" % (W, H, r.stderr[-200:]))
        print(v, "round", rnd, " | ".join(out), flush=True)
