"""Time bspmm_sddmm (SDDMM mode of the SpMM pipeline) under planner tunings."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1903_11409_b200 as bs  # noqa: E402
from tools.kbench import setup, time_calls, sddmm_only  # noqa: E402

dev = torch.device("cuda", 0)
h = bs.Handle(0)
for cid in [int(c) for c in (sys.argv[1] if len(sys.argv) > 1 else "4,5").split(",")]:
    b, reps, per = setup(cid, dev)
    h.set_hints(int(b.sizes.max()), int(b.nnz.max()))
    R = 200 if cid != 5 else 10
    for kt, w, c, ch, d in [(0, 0, 0, 0, 0), (0, 0, 2, 0, 0), (0, 8, 2, 0, 0), (0, 8, 0, 0, 0), (0, 0, 0, 4, 0),
                            (0, 0, 2, 4, 0), (0, 0, 0, 0, 256)]:
        h.set_tuning(kt, w, c, ch)
        h.set_debug(d)
        us = time_calls(h, reps, R, sddmm_only) * 1e3
        print(json.dumps({"config": cid, "tune": [kt, w, c, ch], "dbg": d, "us": us, "plan": h.last_plan()}), flush=True)
    h.set_tuning(0, 0, 0, 0)
    h.set_debug(0)
    del reps
    torch.cuda.empty_cache()
