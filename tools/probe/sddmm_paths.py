"""Time bspmm_sddmm per config: default dispatch, the SpMM-pipeline SDDMM mode forced (debug 1024), the standalone kernel (debug 256)."""
import json, os, sys
import torch
sys.path.insert(0, os.getcwd())
import paper_1903_11409_b200 as bs
from tools.kbench import setup, time_calls, sddmm_only
dev = torch.device("cuda", 0)
h = bs.Handle(0)
for cid in (2, 4, 5):
    b, reps, per = setup(cid, dev)
    h.set_hints(int(b.sizes.max()), int(b.nnz.max()))
    for tune in [(0, 0, 0, 0), (0, 0, 0, 4)]:
        for d in (0, 1024, 256):
            h.set_tuning(*tune); h.set_debug(d)
            us = time_calls(h, reps, 200 if cid != 5 else 10, sddmm_only) * 1e3
            print(cid, tune, d, round(us, 2), h.last_plan()["lanes"], flush=True)
    h.set_tuning(0, 0, 0, 0); h.set_debug(0)
    del reps; torch.cuda.empty_cache()
