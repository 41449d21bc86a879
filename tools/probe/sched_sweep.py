"""Static vs dynamic (ticket) unit schedule, steady state, per config: CSR and
fused COO launches (debug bit 128 forces the dynamic schedule)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1903_11409_b200 as bs  # noqa: E402
from kbench import coo_convert_csr, setup, spmm_only, time_calls  # noqa: E402

dev = torch.device("cuda", 0)
for cfg in [int(c) for c in sys.argv[1].split(",")]:
    b, reps, per = setup(cfg, dev)
    h = bs.Handle(0)
    h.set_hints(int(b.sizes.max()), int(b.nnz.max()))
    for dbg in (0, 128, 16384 | 128, 16384):
        h.set_debug(dbg)
        R = 200 if cfg != 5 else 10
        csr = [time_calls(h, reps, R, spmm_only) * 1e3 for _ in range(3)]
        plan = h.last_plan()
        coo = [time_calls(h, reps, R, coo_convert_csr) * 1e3 for _ in range(2)] if cfg != 5 else []
        print(json.dumps({"config": cfg, "dbg": dbg, "csr_us": [round(x, 2) for x in csr], "kernel": plan["kernel"],
                          "sched": plan["sched"], "coo_us": [round(x, 2) for x in coo]}), flush=True)
    del reps
    torch.cuda.empty_cache()
