"""Per-step kernel time over the first steps of cfg4 from the reference init
(timing tool): the state's class mix (and with it the lazy-chirality work)
relaxes from the i.i.d. init towards the rule's equilibrium.
    python tools/step_times.py [steps] [W] [H]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1208_2428_b200 as P  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 60
W = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
H = int(sys.argv[3]) if len(sys.argv) > 3 else 16384
e = P.Engine(W, H)
st = torch.cuda.Stream()
e.set_stream(st.cuda_stream)
e.set_table(P.build_table("fhp3"))
e.init(4, 0.2)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
thr = P.bernoulli_threshold(0.0)
ev[0].record(st)
for s in range(steps):
    e.advance_async(4, thr, s, 1)
    ev[s + 1].record(st)
torch.cuda.synchronize()
ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(steps)]
print(json.dumps({"W": W, "H": H, "us_per_step": [round(m * 1e3, 1) for m in ms],
                  "gsups": [round(W * H / (m * 1e-3) / 1e9) for m in ms]}))
