#!/usr/bin/env python
"""Phase timeline of one SpMM launch (bspmm_set_trace): per-CTA %globaltimer
stamps, reported as min / median / max over CTAs relative to the earliest
CTA entry.  L2 is flushed (256 MB write) before the traced launch.

  python tools/trace.py --config 4 [--kt 128 --warps 16 --ctas 1]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1903_11409_b200 as bs  # noqa: E402
import synth  # noqa: E402

SLOTS = ["entry", "after_pdl_wait", "prod_rowoff", "prod_struct_off", "prod_done", "cons_first_full",
         "cons_done", "exit", "cons_unit0_done", "p0_after_empty", "p0_after_tma", "p0_before_arrive",
         "p1_before_arrive", "p0_after_arrive", "p1_after_arrive", "early_b_issued"]
SLOTS += [f"u{j}_{w}" for j in range(3) for w in ("empty_ok", "slice_issued", "tma_issued", "copies_issued")]
SLOTS += ["coo_hist", "coo_scan", "coo_scatter", "coo_rank"]  # fused COO conversion of a CTA's first unit
# the small-batch tile kernel (spmm_tile.cu, plan kernel == 1)
TILE_SLOTS = ["entry", "after_pdl_wait", "rt1_done", "b_issued", "struct_staged", "b_landed", "done"]


def summarize(t, plan):
    """Per-slot [min, median, max] over CTAs (us, relative to the earliest CTA
    entry) of one launch's trace rows t [grid x 32] (unwritten slots < 0)."""
    t0 = t[:, 0].min()
    rel = (t - t0) / 1e3
    tile = plan.get("kernel", 0) == 1
    names, last = (TILE_SLOTS, 6) if tile else (SLOTS, 7)
    out = {"span_us": float((t[:, last].max() - t0) / 1e3)}
    for k, name in enumerate(names):
        col_ = rel[:, k][t[:, k] > 0]
        if col_.size == 0:
            continue
        out[name] = [round(float(col_.min()), 2), round(float(np.median(col_)), 2), round(float(col_.max()), 2)]
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--kt", type=int, default=0)
    ap.add_argument("--warps", type=int, default=0)
    ap.add_argument("--ctas", type=int, default=0)
    ap.add_argument("--chunks", type=int, default=0)
    ap.add_argument("--launches", type=int, default=3)
    ap.add_argument("--nostore", action="store_true")
    ap.add_argument("--dbg", type=int, default=0, help="debug bits (bspmm_set_debug)")
    ap.add_argument("--warm", action="store_true", help="no L2 flush before the traced launch")
    ap.add_argument("--sizes", action="store_true", help="row_off = None (offsets fused into the launch)")
    ap.add_argument("--coo", action="store_true", help="trace the fused COO launch (bspmm_coo with hints)")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    b = synth.config(args.config, coo=args.coo)
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    h = bs.Handle(0)
    h.set_hints(int(b.sizes.max()), int(b.nnz.max()))
    h.set_tuning(args.kt, args.warps, args.ctas, args.chunks)
    ro, rp, col, vals, B = T(b.row_off), T(b.row_ptr), T(b.col), T(b.vals), T(b.B)
    sz = T(b.sizes)
    C = torch.empty((b.n_rows, b.k), device=dev)
    def call():
        if args.coo:
            h.coo(ro, None, T(b.nnz_off), T(b.coo_idx), T(b.coo_vals), B, C)
        else:
            h.csr(ro, None, rp, col, vals, B, C)
    call()
    h.set_debug(args.dbg | (1 if args.nostore else 0))
    call()
    grid = h.last_plan()["grid"]
    buf = torch.zeros((grid, 32), dtype=torch.int64, device=dev)
    flush = torch.empty(64 * 2 ** 20, dtype=torch.float32, device=dev)
    for it in range(args.launches):
        if not args.warm:
            flush.fill_(float(it))
        torch.cuda.synchronize()
        buf.fill_(-(1 << 62))
        h.set_trace(buf)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        if args.coo:
            h.coo(ro, None, T(b.nnz_off), T(b.coo_idx), T(b.coo_vals), B, C)
        elif args.sizes:
            h.csr(None, sz, rp, col, vals, B, C)
        else:
            h.csr(ro, None, rp, col, vals, B, C)
        e1.record()
        h.set_trace(None)
        torch.cuda.synchronize()
        t = buf.cpu().numpy().astype(np.int64)
        out = {"config": args.config, "launch": it, "nostore": args.nostore, "event_us": e0.elapsed_time(e1) * 1e3,
               "plan": h.last_plan(), **summarize(t, h.last_plan())}
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
