#!/usr/bin/env python
"""Batched vs non-batched SpMM on B200 (context for PAPER.md:350, Fig.
bbench_all: 9.27x at n_B=64 for batch 50 x dim 50 x 2 nnz/row; 6.09x at
n_B=512 for batch 100 x dim 50 x 3 nnz/row, P100).

Non-batched = one bspmm_csr call per matrix (batch = 1), i.e. the same kernel
launched `batch` times, as the paper's non-batched SpMM launches one kernel
per matrix.  Both arms are timed with CUDA events over
R repetitions, eager (host launch cost included, like the paper's timing) and
CUDA-graph captured (device-side cost only).

  python tools/nonbatched.py [--reps 20]
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

SHAPES = [  # (label, batch, dim, nnz/row) from PAPER.md:361, :366, :395-423
    ("fig_bbench_all_a", 50, 50, 2),
    ("fig_bbench_all_b", 100, 50, 3),
]
NB = [16, 32, 64, 128, 256, 512, 1024]


def timed(fn, reps, graph):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
        fn()
    torch.cuda.synchronize()
    if graph:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                fn()
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps * 1e3
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    h = bs.Handle(0)
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    for label, batch, dim, d in SHAPES:
        for nb in NB:
            b = synth.generate(synth.RAND, (dim, d, 0, 0), batch, nb, seed=1903114090 + dim * 1000 + d)
            h.set_hints(dim, dim * d)
            ro, rp, col, vals, B = T(b.row_off), T(b.row_ptr), T(b.col), T(b.vals), T(b.B)
            C = torch.empty_like(B)
            # per-matrix views (offsets rebased to 0 per matrix)
            per = []
            for i in range(batch):
                g0, g1 = int(b.row_off[i]), int(b.row_off[i + 1])
                z0, z1 = int(b.row_ptr[g0]), int(b.row_ptr[g1])
                per.append((T(np.array([0, g1 - g0], np.int64)), T(b.row_ptr[g0:g1 + 1] - z0), col[z0:z1],
                            vals[z0:z1], B[g0:g1], C[g0:g1]))

            def batched():
                h.csr(ro, None, rp, col, vals, B, C)

            def nonbatched():
                for r0, rpi, ci, vi, Bi, Ci in per:
                    h.csr(r0, None, rpi, ci, vi, Bi, Ci)

            out = {"shape": label, "batch": batch, "dim": dim, "nnz_row": d, "n_B": nb}
            flops = 2.0 * b.n_nnz * nb
            for mode, graph in (("eager", False), ("graph", True)):
                tb = timed(batched, args.reps, graph)
                tn = timed(nonbatched, max(2, args.reps // 5), graph)
                out[f"{mode}_batched_us"] = tb
                out[f"{mode}_nonbatched_us"] = tn
                out[f"{mode}_speedup"] = tn / tb
                out[f"{mode}_batched_gflops"] = flops / tb / 1e3
            print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
