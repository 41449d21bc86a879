#!/usr/bin/env python
"""One fused GCN layer call per shape (for ncu captures of gcn_fused_kernel):
  python tools/gcn_once.py [tox21|reaction100|big] [fp32|tf32|bf16]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1903_11409_b200 as bs  # noqa: E402
import synth  # noqa: E402
from tools.gcn_bench import channels_of  # noqa: E402

SHAPES = {"tox21": (100, 64, 4), "reaction100": (100, 512, 4), "big": (65536, 512, 4)}


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "reaction100"
    mode = sys.argv[2] if len(sys.argv) > 2 else "fp32"
    batch, width, channels = SHAPES[name]
    dev = torch.device("cuda", 0)
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    rng = np.random.default_rng(0)
    b = synth.generate(synth.MOL, (20, 60, 0, 0), batch, width, seed=1903114090 + batch, dense=False)
    rps, col, vals = channels_of(b, channels, rng)
    X = T(rng.standard_normal((b.n_rows, width)).astype(np.float32))
    W = T((rng.standard_normal((channels, width, width)) / np.sqrt(width)).astype(np.float32))
    bias = T(rng.standard_normal((channels, width)).astype(np.float32))
    h = bs.Handle(0)
    h.set_hints(int(b.sizes.max()), 0)
    h.set_gcn_math(mode)
    for _ in range(2):
        Y = h.gcn_layer(T(b.row_off), None, T(rps), T(col), T(vals), X, W, bias)
    torch.cuda.synchronize()
    print("ok", name, mode, float(Y.abs().sum()))


if __name__ == "__main__":
    main()
