"""Small runs of every step kernel for compute-sanitizer (memcheck,
racecheck, initcheck, synccheck): the bit-plane ring kernel (W >= 4096 or
W = 2048 per-warp, with and without forcing; FHP-III, DEFAULT and FHP-I
circuits), the per-warp bit-plane kernel (W = 1024), the byte fast path and
the generic path.  python tools/sanitize.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1208_2428_b200 as P  # noqa: E402

for W, H, fp, rule in ((2048, 64, 0.2, "fhp3"), (4096, 131, 0.0, "fhp3"), (4096, 70, 0.3, "default"),
                       (1024, 64, 0.2, "fhp3"), (1024, 40, 0.0, "fhp1"), (528, 40, 0.0, "fhp3"),
                       (100, 23, 0.5, "fhp3")):
    e = P.Engine(W, H)
    e.set_table(P.build_table(rule))
    e.init(3, 0.3)
    e.advance(3, fp, 0, 5)
    e.observables()
    e.cells(4)
    e.rows()
    e.download()
    print(W, H, rule, e.path)
    e.close()
print("sanitize run ok")
