"""Backward timing per config with the stream arrangement switched by debug bits
(0: transpose -> grad_B SpMM on the auxiliary stream, SDDMM on the caller's;
4096: only the transpose on the auxiliary stream; 2048: all on one stream)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1903_11409_b200 as bs  # noqa: E402
from tools.kbench import setup, time_calls, backward  # noqa: E402

dev = torch.device("cuda", 0)
h = bs.Handle(0)
for cid in (2, 3, 4, 5):
    b, reps, per = setup(cid, dev)
    h.set_hints(int(b.sizes.max()), int(b.nnz.max()))
    for d in (0, 4096, 2048):
        h.set_debug(d)
        print(cid, d, round(time_calls(h, reps, 50 if cid != 5 else 5, backward) * 1e3, 1), flush=True)
    h.set_debug(0)
    del reps
    torch.cuda.empty_cache()
