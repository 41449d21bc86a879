"""Per-CTA phase trace of the C4 tile kernel in steady state (last launch of
a CUDA graph of back-to-back launches), raw, with the SM id of every CTA:
where the tail of the launch comes from (load balance across SMs).
  python tools/probe/tile_balance.py --dbg 4194304 --out gpurun_out/x.npz"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1903_11409_b200 as bs  # noqa: E402
from kbench import coo_convert_csr, setup, spmm_only, time_calls  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--dbg", type=int, default=0)
ap.add_argument("--cb", type=int, default=0)
ap.add_argument("--out", required=True)
ap.add_argument("--coo", action="store_true", help="the fused SparseTensor launch (bspmm_coo with hints)")
a = ap.parse_args()
dev = torch.device("cuda", 0)
b, reps, per = setup(a.config, dev)
h = bs.Handle(0)
h.set_hints(int(b.sizes.max()), int(b.nnz.max()))
h.set_debug(a.dbg)
h.set_tile_cb(a.cb)
fn = coo_convert_csr if a.coo else spmm_only
fn(h, reps[0])
torch.cuda.synchronize()
plan = h.last_plan()
us = time_calls(h, reps, 200, fn) * 1e3
buf = torch.full((plan["grid"], 32), -1, dtype=torch.int64, device=dev)
h.set_trace(buf)
time_calls(h, reps, 200, fn)
h.set_trace(None)
np.savez(a.out, t=buf.cpu().numpy(), us=us, plan=str(plan))
print(a.dbg, a.cb, round(us, 3), plan)
