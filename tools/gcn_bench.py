#!/usr/bin/env python
"""Fused batched GCN layer timing (NEXT-1): Y = sum_ch A_ch (X W_ch + 1 b_ch^T).

Shapes follow ChemGCN: Tox21 weight width 64, Reaction100
width 512, on Tox21-shaped molecule graphs (G-mol 20-60 nodes).  The paper
does not state the channel count; 4 adjacency channels (bond types) are
assumed here.  Timed with CUDA graphs (device time), compared with the same
layer built from torch.matmul (cuBLAS, fp32 and TF32) + bias add + our SpMM
per channel + add (the paper's 3-per-channel launch structure, Fig.
algo:graph_conv_batched).  The fused layer is bspmm_gcn_layer: a preparation
launch + one tcgen05 launch (csrc/gcn_fused.cu).
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1903_11409_b200 as bs  # noqa: E402
import synth  # noqa: E402
from tools.kbench import time_calls  # noqa: E402


def channels_of(b, channels, rng):
    rps, cols, vals = [], [], []
    z = 0
    for ch in range(channels):
        keep = np.ones(b.n_nnz, bool) if ch == 0 else rng.random(b.n_nnz) < 0.6
        rp = np.zeros(b.n_rows + 1, np.int32)
        kept = np.nonzero(keep)[0]
        # row pointer of the kept subset: count kept entries per row
        rows = np.repeat(np.arange(b.n_rows), np.diff(b.row_ptr))
        cnt = np.bincount(rows[kept], minlength=b.n_rows)
        rp[1:] = np.cumsum(cnt)
        rp += z
        rps.append(rp)
        cols.append(b.col[kept])
        vals.append(rng.standard_normal(kept.size).astype(np.float32))
        z += kept.size
    return np.stack(rps), np.concatenate(cols).astype(np.int32), np.concatenate(vals)


def main():
    dev = torch.device("cuda", 0)
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    h = bs.Handle(0)
    rng = np.random.default_rng(0)
    # optional: --dbg BITS (bspmm_set_debug), --small (the two 100-graph shapes only)
    if "--dbg" in sys.argv:
        h.set_debug(int(sys.argv[sys.argv.index("--dbg") + 1]))
    shapes = [("tox21_like", 100, 64, 4), ("reaction100_like", 100, 512, 4), ("reaction100_like_b65536", 65536, 512, 4)]
    if "--small" in sys.argv:
        shapes = shapes[:2]
    for name, batch, width, channels in shapes:
        b = synth.generate(synth.MOL, (20, 60, 0, 0), batch, width, seed=1903114090 + batch, dense=False)
        rps, col, vals = channels_of(b, channels, rng)
        X = T(rng.standard_normal((b.n_rows, width)).astype(np.float32))
        W = T((rng.standard_normal((channels, width, width)) / np.sqrt(width)).astype(np.float32))
        bias = T(rng.standard_normal((channels, width)).astype(np.float32))
        ro, rp_d, col_d, vals_d = T(b.row_off), T(rps), T(col), T(vals)
        Y = torch.empty((b.n_rows, width), device=dev)
        h.set_hints(int(b.sizes.max()), 0)

        def fused(h_, _):
            h_.gcn_layer(ro, None, rp_d, col_d, vals_d, X, W, bias, Y)

        Us = [torch.empty((b.n_rows, width), device=dev) for _ in range(channels)]
        Cs = [torch.empty((b.n_rows, width), device=dev) for _ in range(channels)]

        def unfused(h_, _):  # the paper's structure: MatMul, Add, BatchedSpMM per channel, then ElementWiseAdd
            for ch in range(channels):
                torch.matmul(X, W[ch], out=Us[ch])
                Us[ch].add_(bias[ch])
                h_.csr(ro, None, rp_d[ch], col_d, vals_d, Us[ch], Cs[ch])
            torch.sum(torch.stack(Cs), 0, out=Y)

        reps = [None]
        R = 20 if batch < 1000 else 3
        t_modes = {}
        for mode in ("tf32", "bf16"):
            h.set_gcn_math(mode)
            t_modes[mode] = time_calls(h, reps, R, fused) * 1e3
        h.set_gcn_math("fp32")
        t_fused = time_calls(h, reps, R, fused) * 1e3
        t_unf = time_calls(h, reps, R, unfused) * 1e3
        torch.backends.cuda.matmul.allow_tf32 = True        # the same composition with cuBLAS TF32 GEMMs
        t_unf_tf32 = time_calls(h, reps, R, unfused) * 1e3
        torch.backends.cuda.matmul.allow_tf32 = False
        gemm_flops = 2.0 * b.n_rows * width * width * channels
        spmm_flops = 2.0 * len(col) * width
        print(json.dumps({"shape": name, "batch": batch, "rows": b.n_rows, "width": width, "channels": channels,
                          "fused_us": t_fused, "unfused_us": t_unf, "speedup_vs_unfused": t_unf / t_fused,
                          "fused_TFLOPs": (gemm_flops + spmm_flops) / t_fused / 1e6,
                          "fused_tf32_us": t_modes["tf32"], "fused_bf16_us": t_modes["bf16"],
                          "fused_tf32_TFLOPs": (gemm_flops + spmm_flops) / t_modes["tf32"] / 1e6,
                          "unfused_tf32_us": t_unf_tf32, "launches_fused": 2, "launches_unfused": 3 * channels + 2}),
              flush=True)


if __name__ == "__main__":
    main()
