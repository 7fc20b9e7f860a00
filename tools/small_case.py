"""A few steps of the 1024 x 1024 FHP-I case (for ncu launch lists)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1208_2428_b200 as P  # noqa: E402

W = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
H = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
e = P.Engine(W, H)
e.set_table(P.build_table("fhp1"))
e.init(1, 0.2)
e.advance(1, 0.0, 0, 6)
torch.cuda.synchronize()
