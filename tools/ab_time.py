"""Device-timed GSUPS of one configuration (A/B tool: FHPG_LIB selects the
engine build). python tools/ab_time.py [W] [H] [table] [force_p] [steps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1208_2428_b200 as P  # noqa: E402

W = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
H = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
table = sys.argv[3] if len(sys.argv) > 3 else "fhp3"
fp = float(sys.argv[4]) if len(sys.argv) > 4 else 0.0
steps = int(sys.argv[5]) if len(sys.argv) > 5 else 100
e = P.Engine(W, H)
s = torch.cuda.Stream()
e.set_stream(s.cuda_stream)
e.set_table(P.build_table(table))
e.init(4, 0.2)
thr = P.bernoulli_threshold(fp)
e.advance_async(4, thr, 0, 10)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
a.record(s)
e.advance_async(4, thr, 10, steps)
b.record(s)
torch.cuda.synchronize()
print(round(W * H * steps / (a.elapsed_time(b) * 1e-3) / 1e9, 1))
