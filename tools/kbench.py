#!/usr/bin/env python
"""Kernel-level timing of the batched SpMM on one GPU, per BASELINE.json config,
with an optional tuning sweep.  Steady state: R back-to-back launches captured
in a CUDA graph, cycling over M replicas of (B, C, structure) whose total
footprint exceeds 2x L2, so every launch reads B from HBM (SURVEY §8(d) T-evt).

  python tools/kbench.py --configs 2,3,4,5 [--sweep] [--reps 200]
"""
import argparse
import itertools
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import paper_1903_11409_b200 as bs  # noqa: E402
import synth  # noqa: E402
from bench import alg_bytes, peaks  # noqa: E402

L2 = 126 * 2 ** 20


def setup(cid, dev, replicas=0, shard=1):
    if shard > 1:  # rank 0's contiguous nnz*k shard of a `shard`-way split (scaling prediction)
        full = synth.config(cid)
        split = bs.partition(full.nnz_off, full.k, shard)
        b = synth.config(cid, i0=0, i1=int(split[1]), coo=True)
    else:
        b = synth.config(cid, coo=True)
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    per = alg_bytes(b.n_rows, b.n_nnz, b.k, b.batch)
    M = replicas if replicas > 0 else max(1, min(64, int(np.ceil(2 * L2 / per))))
    reps = []
    for _ in range(M):
        reps.append(dict(ro=T(b.row_off), rp=T(b.row_ptr), col=T(b.col), vals=T(b.vals), B=T(b.B),
                         C=torch.empty((b.n_rows, b.k), device=dev), sizes=T(b.sizes), no=T(b.nnz_off),
                         idx=T(b.coo_idx), cv=T(b.coo_vals), N=b.n_rows))
    return b, reps, per


def time_calls(h, reps, R, fn, graph=True):
    M = len(reps)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for i in range(3 * M):
            fn(h, reps[i % M])
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    if graph:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for i in range(R):
                fn(h, reps[i % M])
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / R
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(R):
        fn(h, reps[i % M])
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / R


def trace_in_graph(h, reps, R):
    """Phase trace of the LAST launch of a graph of R back-to-back SpMM launches
    (steady state: the trace pointer is captured into every launch, each
    overwrites the buffer)."""
    from trace import summarize
    spmm_only(h, reps[0])
    torch.cuda.synchronize()
    plan = h.last_plan()
    buf = torch.zeros((plan["grid"], 32), dtype=torch.int64, device=reps[0]["B"].device)
    buf.fill_(-1)
    h.set_trace(buf)
    try:
        time_calls(h, reps, R, spmm_only)
    finally:
        h.set_trace(None)
    return summarize(buf.cpu().numpy().astype(np.int64), plan)


def spmm_only(h, r):
    h.csr(r["ro"], None, r["rp"], r["col"], r["vals"], r["B"], r["C"])


def full_step(h, r):
    h.build_offsets(r["sizes"], out=r["ro"])
    h.csr(r["ro"], None, r["rp"], r["col"], r["vals"], r["B"], r["C"])


def coo_convert_csr(h, r):  # deterministic COO path: device COO->CSR + the CSR kernel
    h.coo(r["ro"], None, r["no"], r["idx"], r["cv"], r["B"], r["C"], total_rows=r["N"])


def coo_atomic(h, r):  # the paper's atomic SWA-ST kernel
    h.coo_atomic(r["ro"], None, r["no"], r["idx"], r["cv"], r["B"], r["C"])


def fused_step(h, r):  # offsets built inside the SpMM (row_off = None)
    h.csr(None, r["sizes"], r["rp"], r["col"], r["vals"], r["B"], r["C"])


def backward(h, r):  # NEXT-2: grad_B = A^T grad_C (transpose + SpMM) and grad_vals (SDDMM)
    h.csr_backward(r["ro"], None, r["rp"], r["col"], r["vals"], r["B"], r["C"])


def transpose_only(h, r):  # NEXT-2 piece: A^T (expand + device COO->CSR)
    h.csr_transpose(r["ro"], None, r["rp"], r["col"], r["vals"])


def sddmm_only(h, r):  # NEXT-2 piece: grad_vals = <grad_C[row], B[col]> (C stands in for grad_C)
    h.sddmm(r["ro"], None, r["rp"], r["col"], r["B"], r["C"])


def copy_only(h, r):  # torch's device copy moving B's bytes in and C's out
    r["C"].copy_(r["B"])


_floor = None


def floor_lib():
    """tools/probe/libfloor.so: hand-written one-CTA-per-SM copies of B into C,
    launched like the SpMM kernels (PDL, same graph)."""
    global _floor
    if _floor is None:
        import ctypes
        path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "probe", "libfloor.so")
        _floor = ctypes.CDLL(path)
        _floor.floor_copy.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                      ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
        _floor.floor_copy.restype = ctypes.c_int
    return _floor


def floor_copy(mode, groups=4):
    def fn(h, r):
        n4 = r["B"].numel() // 4
        grid = torch.cuda.get_device_properties(r["B"].device).multi_processor_count
        rc = floor_lib().floor_copy(r["B"].data_ptr(), r["C"].data_ptr(), n4, mode, groups, grid,
                                    torch.cuda.current_stream().cuda_stream, r["dep"].data_ptr())
        if rc != 0:
            raise RuntimeError(f"floor_copy rc={rc}")
    return fn


def offsets_only(h, r):
    h.build_offsets(r["sizes"], out=r["ro"])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="2,3,4,5")
    ap.add_argument("--reps", type=int, default=200)
    ap.add_argument("--sweep", action="store_true")
    ap.add_argument("--kts", default="0,32,64,128,256,512")
    ap.add_argument("--warps", default="0,4,8,12,16")
    ap.add_argument("--ctas", default="0,1,2")
    ap.add_argument("--chunks", default="0")
    ap.add_argument("--ncu-mode", action="store_true", help="plain launches only (for ncu)")
    ap.add_argument("--ncu-coo", action="store_true", help="with --ncu-mode: also 6 fused COO launches")
    ap.add_argument("--dbg", default="0", help="comma list of debug bit sets to sweep (bspmm_set_debug)")
    ap.add_argument("--replicas", type=int, default=0, help="override the replica count (1 = L2-warm)")
    ap.add_argument("--copy-baseline", action="store_true", help="also time C.copy_(B) on the same replicas")
    ap.add_argument("--shard", type=int, default=1, help="time rank 0's shard of an N-way split (1 GPU)")
    ap.add_argument("--backward", action="store_true", help="also time csr_backward (grad_B and grad_vals)")
    ap.add_argument("--bwd-dbg", default="", help="with --backward: debug bit sets for extra backward timings")
    ap.add_argument("--sddmm-dbg", default="", help="with --backward: debug bit sets for extra SDDMM timings")
    ap.add_argument("--tile-cbs", default="0", help="tile-kernel column blocks to sweep (bspmm_set_tile_cb)")
    ap.add_argument("--coo-dbg", default="", help="debug bit sets for extra fused-COO timings")
    ap.add_argument("--trace", action="store_true", help="phase trace of the last launch of the graph (per dbg)")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    peak, _ = peaks()
    h = bs.Handle(0)
    for cid in [int(c) for c in args.configs.split(",")]:
        b, reps, per = setup(cid, dev, args.replicas, args.shard)
        h.set_hints(int(b.sizes.max()), int(b.nnz.max()))
        R = args.reps if cid != 5 else max(10, args.reps // 20)
        if args.ncu_mode:
            for i in range(6):
                full_step(h, reps[i % len(reps)])
            if args.ncu_coo and "idx" in reps[0]:  # then the fused COO launches (bspmm_coo with hints)
                for i in range(6):
                    coo_convert_csr(h, reps[i % len(reps)])
            torch.cuda.synchronize()
            print(json.dumps({"config": cid, "ncu_mode": True, "plan": h.last_plan()}), flush=True)
            del reps
            torch.cuda.empty_cache()
            continue
        combos = [(0, 0, 0, 0)]
        if args.sweep:
            combos = list(itertools.product([int(x) for x in args.kts.split(",")],
                                            [int(x) for x in args.warps.split(",")],
                                            [int(x) for x in args.ctas.split(",")],
                                            [int(x) for x in args.chunks.split(",")]))
        combos = [(kt, w, c, ch, d, cb) for kt, w, c, ch in combos for d in [int(x) for x in args.dbg.split(",")]
                  for cb in [int(x) for x in args.tile_cbs.split(",")]]
        for kt, w, c, ch, dbg, cb in combos:
            h.set_tile_cb(cb)
            if kt and kt > b.k:
                continue
            h.set_tuning(kt, w, c, ch)
            h.set_debug(dbg)
            try:
                ms = time_calls(h, reps, R, spmm_only)
            except Exception as e:  # noqa: BLE001
                print(json.dumps({"config": cid, "kt": kt, "warps": w, "ctas": c, "error": str(e)}), flush=True)
                continue
            plan = h.last_plan()
            gbs = per / (ms / 1e3) / 1e9
            tr = {"trace": trace_in_graph(h, reps, R)} if args.trace else {}
            print(json.dumps({"config": cid, "kt": kt, "warps": w, "ctas": c, "chunks": ch, "dbg": dbg, "tile_cb": cb,
                              "us": ms * 1e3, "GBs": gbs,
                              "frac": gbs / peak, "GFLOPs": 2 * b.n_nnz * b.k / (ms / 1e3) / 1e9,
                              "replicas": len(reps), "shard": args.shard, "plan": plan, **tr}), flush=True)
        h.set_tuning(0, 0, 0)
        h.set_debug(0)
        h.set_tile_cb(0)
        ms_step = time_calls(h, reps, R, full_step)
        ms_fused = time_calls(h, reps, R, fused_step)
        ms_off = time_calls(h, reps, R, offsets_only)
        ms_ng = time_calls(h, reps, min(R, 50), spmm_only, graph=False)
        extra = {}
        if args.backward:
            extra["backward_us"] = time_calls(h, reps, max(3, R // 4), backward) * 1e3
            extra["transpose_us"] = time_calls(h, reps, max(3, R // 4), transpose_only) * 1e3
            extra["sddmm_us"] = time_calls(h, reps, max(3, R // 4), sddmm_only) * 1e3
            for d in [int(x) for x in args.bwd_dbg.split(",") if x]:
                h.set_debug(d)
                extra[f"backward_us_dbg{d}"] = time_calls(h, reps, max(3, R // 4), backward) * 1e3
            for d in [int(x) for x in args.sddmm_dbg.split(",") if x]:
                h.set_debug(d)
                extra[f"sddmm_us_dbg{d}"] = time_calls(h, reps, max(3, R // 4), sddmm_only) * 1e3
            h.set_debug(0)
        if args.copy_baseline:
            ms_cp = time_calls(h, reps, R, copy_only)
            extra["copy_us"] = ms_cp * 1e3
            extra["copy_GBs"] = 8 * b.n_rows * b.k / (ms_cp / 1e3) / 1e9
            if cid != 5:  # one-wave configs: hand-written 148-CTA copies (floor.cu modes)
                for r in reps:
                    r["dep"] = torch.zeros(64, dtype=torch.int64, device=dev)
                for mode, name in ((0, "floor_cpasync"), (1, "floor_regs"), (2, "floor_tma_stg"), (3, "floor_tma_tma"),
                                   (1 | 4, "floor_regs_rt1"), (1 | 12, "floor_regs_rt1_evl"), (2 | 4, "floor_tma_stg_rt1")):
                    for g in ((1, 2, 4, 8) if mode & 3 in (0, 2, 3) else (1,)):
                        try:
                            ms_f = time_calls(h, reps, R, floor_copy(mode, g))
                            extra[f"{name}_g{g}_us"] = ms_f * 1e3
                        except Exception as e:  # noqa: BLE001
                            extra[f"{name}_g{g}_err"] = str(e)
        if b.k % 4 == 0 and cid != 5:
            extra["coo_convert_csr_us"] = time_calls(h, reps, R, coo_convert_csr) * 1e3
            extra["coo_atomic_us"] = time_calls(h, reps, R, coo_atomic) * 1e3
            for d in [int(x) for x in args.coo_dbg.split(",") if x]:
                h.set_debug(d)
                extra[f"coo_convert_csr_us_dbg{d}"] = time_calls(h, reps, R, coo_convert_csr) * 1e3
            h.set_debug(0)
        print(json.dumps({"config": cid, "step_us": ms_step * 1e3, "fused_step_us": ms_fused * 1e3,
                          "offsets_us": ms_off * 1e3,
                          "spmm_us_no_graph": ms_ng * 1e3, "alg_bytes": per, "replicas": len(reps), **extra}),
              flush=True)
        del reps
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
