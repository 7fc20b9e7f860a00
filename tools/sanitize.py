"""Small runs of every step kernel for compute-sanitizer (memcheck,
racecheck, initcheck, synccheck): the bit-plane ring kernel (W % 2048 == 0,
with and without forcing), the per-warp bit-plane kernel (W = 1024), the
byte fast path and the generic path.  python tools/sanitize.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1208_2428_b200 as P  # noqa: E402

for W, H, fp in ((2048, 64, 0.2), (4096, 131, 0.0), (1024, 64, 0.2), (528, 40, 0.0), (100, 23, 0.5)):
    e = P.Engine(W, H)
    e.set_table(P.build_table("fhp3"))
    e.init(3, 0.3)
    e.advance(3, fp, 0, 5)
    e.observables()
    e.cells(4)
    e.rows()
    e.download()
    print(W, H, e.path)
    e.close()
print("sanitize run ok")
