"""Plain SDDMM launches at a config (for ncu): grad_vals = <G[row], B[col]>."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import paper_1903_11409_b200 as bs  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--dbg", type=int, default=0)
ap.add_argument("--n", type=int, default=4)
a = ap.parse_args()
dev = torch.device("cuda", 0)
b = synth.config(a.config)
T = lambda x: torch.from_numpy(np.ascontiguousarray(x)).to(dev)
h = bs.Handle(0)
h.set_hints(int(b.sizes.max()), int(b.nnz.max()))
h.set_debug(a.dbg)
ro, rp, col, B = T(b.row_off), T(b.row_ptr), T(b.col), T(b.B)
Gr = torch.randn_like(B)
for _ in range(a.n):
    h.sddmm(ro, None, rp, col, B, Gr)
torch.cuda.synchronize()
print("ok")
