import sys, os, numpy as np
sys.path.insert(0, '.')
import paper_1208_2428_b200 as P
t = P.build_table("fhp3")
W = H = 16384
for trial in range(2):
    e = P.Engine(W, H); e.set_table(t); e.init(4, 0.2)
    m0 = e.observables()[0]
    out = []
    for k in range(3):
        e.advance(4, 0.0, 20 * k, 20)
        out.append(e.observables()[0] - m0)
    print(os.environ.get("FHPG_LIB", "default").split("/")[-1], trial, out, flush=True)
