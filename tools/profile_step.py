"""Short run of the cfg4 step loop for ncu (not a bench: numbers under a
profiler are never reported). Usage: python tools/profile_step.py [steps] [W] [H] [table] [force_p]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1208_2428_b200 as P  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
W = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
H = int(sys.argv[3]) if len(sys.argv) > 3 else 16384
table = sys.argv[4] if len(sys.argv) > 4 else "fhp3"
fp = float(sys.argv[5]) if len(sys.argv) > 5 else 0.0
e = P.Engine(W, H)
e.set_table(P.build_table(table))
e.init(4, 0.2)
e.advance(4, fp, 0, steps)
print("ok", e.observables())
