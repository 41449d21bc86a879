"""Time bspmm_coo per config: fused conversion (planner hints) vs the two-kernel path (no hints), and tunings."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1903_11409_b200 as bs  # noqa: E402
from tools.kbench import setup, time_calls, coo_convert_csr  # noqa: E402

dev = torch.device("cuda", 0)
h = bs.Handle(0)
for cid in [int(c) for c in (sys.argv[1] if len(sys.argv) > 1 else "2,3,4").split(",")]:
    b, reps, per = setup(cid, dev)
    for hints in ((int(b.sizes.max()), int(b.nnz.max())), (0, 0)):
        for kt in (0, 64, 128):
            if kt > b.k:
                continue
            h.set_hints(*hints)
            h.set_tuning(kt, 0, 0, 0)
            us = time_calls(h, reps, 200, coo_convert_csr) * 1e3
            print(cid, "hints" if hints[0] else "nohints", kt, round(us, 2), h.last_plan()["kt"], h.last_plan()["units"],
                  flush=True)
    h.set_tuning(0, 0, 0, 0)
    del reps
    torch.cuda.empty_cache()
