"""Run the NEXT-2 backward on one config a few times (for ncu launch lists)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1903_11409_b200 as bs  # noqa: E402
import synth  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 5
dev = torch.device("cuda", 0)
b = synth.config(cid)
T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
h = bs.Handle(0)
h.set_hints(int(b.sizes.max()), int(b.nnz.max()))
ro, rp, col, vals, B = T(b.row_off), T(b.row_ptr), T(b.col), T(b.vals), T(b.B)
G = torch.randn_like(B)
for _ in range(3):
    h.csr_backward(ro, None, rp, col, vals, B, G)
torch.cuda.synchronize()
print("ok")
