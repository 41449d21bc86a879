#!/usr/bin/env python
"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): C1-C3 through every entry point (offsets, CSR, COO,
COO->CSR, transpose, backward incl. a streaming batch, host path), plus a
padded layout and the direct (unstaged) path.  C is pre-filled with NaN-free garbage only where the
kernel must write it, so initcheck sees every read of C-derived data.

  compute-sanitizer --tool memcheck python tools/sanitize_run.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1903_11409_b200 as bs  # noqa: E402
import synth  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    h = bs.Handle(0)
    if len(sys.argv) > 1:
        h.set_debug(int(sys.argv[1]))
    for cid in (1, 2, 3):
        b = synth.config(cid, coo=True)
        h.set_hints(int(b.sizes.max()), int(b.nnz.max()))
        ro = h.build_offsets(T(b.sizes))
        C = h.csr(ro, None, T(b.row_ptr), T(b.col), T(b.vals), T(b.B))
        C2 = h.coo(None, T(b.sizes), T(b.nnz_off), T(b.coo_idx), T(b.coo_vals), T(b.B))
        rp, col, v = h.coo2csr(ro, None, T(b.nnz_off), T(b.coo_idx), T(b.coo_vals), b.n_rows)
        rt, ct, vt = h.csr_transpose(ro, None, T(b.row_ptr), T(b.col), T(b.vals))
        gB, gv = h.csr_backward(ro, None, T(b.row_ptr), T(b.col), T(b.vals), T(b.B), C)
        Cf = h.csr(None, T(b.sizes), T(b.row_ptr), T(b.col), T(b.vals), T(b.B))        # fused offsets
        Cm = torch.empty_like(C)
        h.csr_multicast(ro, None, T(b.row_ptr), T(b.col), T(b.vals), T(b.B), Cm)        # multimem variant (unicast)
        Ca = h.coo_atomic(ro, None, T(b.nnz_off), T(b.coo_idx), T(b.coo_vals), T(b.B))
        torch.cuda.synchronize()
        assert torch.equal(C, C2) and torch.equal(C, Cf) and torch.equal(C, Cm)
    # C4: whole-row units (1-D bulk B tiles of 100 KB), and the GCN layer
    b = synth.config(4)
    h.set_hints(int(b.sizes.max()), int(b.nnz.max()))
    C4 = h.csr(T(b.row_off), None, T(b.row_ptr), T(b.col), T(b.vals), T(b.B))
    b = synth.config(2)
    h.set_hints(int(b.sizes.max()), int(b.nnz.max()))
    X = torch.randn((b.n_rows, 32), device=dev)
    W = torch.randn((2, 32, b.k), device=dev)
    bias = torch.randn((2, b.k), device=dev)
    rps = torch.stack([T(b.row_ptr), T(b.row_ptr)])
    h.gcn_layer(T(b.row_off), None, rps, T(b.col), T(b.vals), X, W, bias)
    torch.cuda.synchronize()
    del C4
    # backward of a streaming batch (standalone SDDMM kernel: > 8 matrices per SM)
    b = synth.config(5, i0=0, i1=1500)
    h.set_hints(int(b.sizes.max()), int(b.nnz.max()))
    G = torch.randn((b.n_rows, b.k), device=dev)
    h.csr_backward(T(b.row_off), None, T(b.row_ptr), T(b.col), T(b.vals), T(b.B), G)
    torch.cuda.synchronize()
    # direct path (tiny stage capacity) and scalar path (k % 4 != 0)
    if len(sys.argv) > 1:  # the TMA-only variant: C1-C3 vectorised paths only
        h.sync()
        print("sanitize workload ok")
        return
    b = synth.generate(synth.MIX, (100, 300, 1, 5), 6, 7, seed=3)
    h.set_hints(16, 64)
    h.csr(T(b.row_off), None, T(b.row_ptr), T(b.col), T(b.vals), T(b.B))
    b = synth.config(2)
    Bp = torch.zeros((b.n_rows, 68), device=dev)
    Bp[:, :64] = T(b.B)
    h.set_hints(60, 200)
    h.csr(T(b.row_off), None, T(b.row_ptr), T(b.col), T(b.vals), Bp, torch.empty((b.n_rows, 68), device=dev), k=64)
    h.csr_host(b.sizes, b.row_ptr, b.col, b.vals, b.B)
    h.sync()
    print("sanitize workload ok")


if __name__ == "__main__":
    main()
