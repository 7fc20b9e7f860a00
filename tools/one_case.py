"""One advance call of a configuration (debugging aid, e.g. under
compute-sanitizer): python tools/one_case.py W H table force_p steps"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1208_2428_b200 as P  # noqa: E402

W = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
H = int(sys.argv[2]) if len(sys.argv) > 2 else 64
table = sys.argv[3] if len(sys.argv) > 3 else "fhp3"
fp = float(sys.argv[4]) if len(sys.argv) > 4 else 0.0
steps = int(sys.argv[5]) if len(sys.argv) > 5 else 2
e = P.Engine(W, H)
e.set_table(P.build_table(table))
e.init(4, 0.2)
e.advance(4, fp, 0, steps)
print("ok", e.path, e.observables())
