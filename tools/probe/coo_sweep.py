import sys, json, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tools')
import paper_1903_11409_b200 as bs
from kbench import setup, time_calls, coo_convert_csr, spmm_only
dev = torch.device("cuda", 0)
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
b, reps, per = setup(cfg, dev)
h = bs.Handle(0)
h.set_hints(int(b.sizes.max()), int(b.nnz.max()))
for dbg in (0,):
    h.set_debug(dbg)
    for w in (6, 8, 10, 12, 14, 16):
        h.set_tuning(0, w, 0, 0)
        us = [time_calls(h, reps, 200, coo_convert_csr) * 1e3 for _ in range(3)]
        print(json.dumps({"dbg": dbg, "cons_warps": w, "us": [round(u, 2) for u in us], "sched": h.last_plan()["sched"]}), flush=True)
    h.set_tuning(0, 0, 0, 0)
    print(json.dumps({"dbg": dbg, "csr_us": round(time_calls(h, reps, 200, spmm_only) * 1e3, 2)}))
