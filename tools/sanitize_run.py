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
    # C4: the small-batch tile kernel (2-D TMA and cp.async staging, every
    # column block), the pipeline's whole-row units (1-D bulk B tiles of 100 KB)
    b = synth.config(4)
    h.set_hints(int(b.sizes.max()), int(b.nnz.max()))
    dbg0 = int(sys.argv[1]) if len(sys.argv) > 1 else 0
    C4 = h.csr(T(b.row_off), None, T(b.row_ptr), T(b.col), T(b.vals), T(b.B))
    for cb in (1, 8, 32):
        for d in (0, 32768):
            h.set_tile_cb(cb)
            h.set_debug(dbg0 | d)
            Ct = h.csr(T(b.row_off), None, T(b.row_ptr), T(b.col), T(b.vals), T(b.B))
            Cs = h.csr(None, T(b.sizes), T(b.row_ptr), T(b.col), T(b.vals), T(b.B))
            torch.cuda.synchronize()
            assert torch.equal(C4, Ct) and torch.equal(C4, Cs)
    h.set_tile_cb(0)
    h.set_debug(dbg0 | 16384)
    Cp = h.csr(T(b.row_off), None, T(b.row_ptr), T(b.col), T(b.vals), T(b.B))
    torch.cuda.synchronize()
    assert torch.equal(C4, Cp)
    h.set_debug(dbg0)
    # the fused tcgen05 GCN layer: every precision mode, a packed-X leading
    # dimension, 33 channels (structure from global memory), a large graph
    # (X halo from global memory)
    b = synth.config(2)
    h.set_hints(int(b.sizes.max()), int(b.nnz.max()))
    rps = torch.stack([T(b.row_ptr), T(b.row_ptr)])
    for n_x, ld in ((32, 32), (37, 41)):
        X = torch.randn((b.n_rows, ld), device=dev)[:, :n_x]
        W = torch.randn((2, n_x, b.k), device=dev)
        bias = torch.randn((2, b.k), device=dev)
        for mode in ("fp32", "tf32", "bf16"):
            h.set_gcn_math(mode)
            h.gcn_layer(T(b.row_off), None, rps, T(b.col), T(b.vals), X, W, bias)
    h.set_gcn_math("fp32")
    X = torch.randn((b.n_rows, 16), device=dev)
    h.gcn_layer(T(b.row_off), None, torch.stack([T(b.row_ptr)] * 33), T(b.col), T(b.vals), X,
                torch.randn((33, 16, 48), device=dev), torch.randn((33, 48), device=dev))
    bl = synth.generate(synth.MIX, (300, 400, 1, 5), 3, 8, seed=9, dense=False)
    h.set_hints(0, 0)
    h.gcn_layer(T(bl.row_off), None, T(bl.row_ptr[None]), T(bl.col), T(bl.vals),
                torch.randn((bl.n_rows, 40), device=dev), torch.randn((1, 40, 72), device=dev))
    # CTA pairs (tcgen05 cta_group::2; debug bit 1<<22): every precision mode,
    # an odd row-tile count (the last pair's second CTA has no rows), k = 512
    b = synth.config(2)
    h.set_hints(int(b.sizes.max()), int(b.nnz.max()))
    h.set_debug(dbg0 | (1 << 22))
    X = torch.randn((b.n_rows, 64), device=dev)
    for mode in ("fp32", "tf32", "bf16"):
        h.set_gcn_math(mode)
        h.gcn_layer(T(b.row_off), None, rps, T(b.col), T(b.vals), X, torch.randn((2, 64, 512), device=dev),
                    torch.randn((2, 512), device=dev))
    h.set_gcn_math("fp32")
    h.set_debug(dbg0)
    torch.cuda.synchronize()
    # handle state across two streams (set_stream hand-off)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    b = synth.config(3)
    h.set_hints(int(b.sizes.max()), int(b.nnz.max()))
    with torch.cuda.stream(s1):
        h.csr_backward(T(b.row_off), None, T(b.row_ptr), T(b.col), T(b.vals), T(b.B), T(b.B))
    with torch.cuda.stream(s2):
        h.csr(None, T(b.sizes), T(b.row_ptr), T(b.col), T(b.vals), T(b.B))
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
