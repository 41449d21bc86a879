"""GPU parity for the fused batched GCN layer (NEXT-1, PAPER.md Fig.
algo:graph_conv_batched): Y = sum_ch A_ch (X W_ch + 1 bias_ch^T) against the
fp64 oracle.  Tolerance: |Y - Y_ref| <= (n_x + d_max + channels
+ 4) * 2^-23 * M, M = sum_ch sum_e |a_e| (sum_l |x_jl||w_lc| + |b_c|) -- the
fp32 error of the GEMM (n_x terms), of the storage-order SpMM (d terms) and of
the channel sum, with a factor 2 of headroom."""
import numpy as np
import pytest
import torch

import oracle
import paper_1903_11409_b200 as bs
import synth

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0)


@pytest.fixture(scope="module")
def h():
    assert torch.cuda.is_available()
    return bs.Handle(0)


def T(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def channels_of(b, channels, rng):
    """Channel 0 = the batch's graphs; further channels = random subsets of its
    entries with fresh values (same nodes, channel-specific adjacency)."""
    rps, cols, vals = [], [], []
    z = 0
    N = b.n_rows
    for ch in range(channels):
        keep = np.ones(b.n_nnz, bool) if ch == 0 else rng.random(b.n_nnz) < 0.7
        rp = np.zeros(N + 1, np.int32)
        for g in range(N):
            rp[g] = z
            e0, e1 = b.row_ptr[g], b.row_ptr[g + 1]
            sel = np.nonzero(keep[e0:e1])[0] + e0
            cols.append(b.col[sel])
            vals.append(b.vals[sel] if ch == 0 else rng.standard_normal(sel.size).astype(np.float32))
            z += sel.size
        rp[N] = z
        rps.append(rp)
    return np.stack(rps), np.concatenate(cols).astype(np.int32), np.concatenate(vals).astype(np.float32)


@pytest.mark.parametrize("cid,channels,n_x", [(1, 1, 8), (2, 3, 48), (4, 2, 64), (3, 2, 32)])
def test_gcn_layer_parity(h, cid, channels, n_x):
    rng = np.random.default_rng(cid * 10 + channels)
    b = synth.config(cid)
    rps, col, vals = channels_of(b, channels, rng)
    X = rng.standard_normal((b.n_rows, n_x)).astype(np.float32)
    W = (rng.standard_normal((channels, n_x, b.k)) / np.sqrt(n_x)).astype(np.float32)
    bias = rng.standard_normal((channels, b.k)).astype(np.float32)
    h.set_hints(int(b.sizes.max()), 0)
    Y = h.gcn_layer(T(b.row_off), None, T(rps), T(col), T(vals), T(X), T(W), T(bias)).cpu().numpy()
    ref, mag = oracle.gcn_layer(b.row_off, rps, col, vals, X, W, bias)
    dmax = int(max(np.diff(rp).max() for rp in rps))
    tol = (n_x + dmax + channels + 4) * 2.0 ** -23
    err = np.abs(Y.astype(np.float64) - ref)
    assert np.all(err <= tol * mag + 1e-30), float((err / np.maximum(mag, 1e-300)).max())


def test_gcn_layer_reduces_to_spmm(h):
    """W = I, bias = None, one channel: the layer is exactly the batched SpMM of A with X."""
    b = synth.config(2)
    Y = h.gcn_layer(T(b.row_off), None, T(b.row_ptr[None]), T(b.col), T(b.vals), T(b.B),
                    T(np.eye(b.k, dtype=np.float32)[None])).cpu().numpy()
    C32 = oracle.spmm_f32(b.k, b.row_off, None, b.row_ptr, b.col, b.vals, b.B)
    Cref, bound = oracle.spmm(b.k, b.row_off, None, b.row_ptr, b.col, b.vals, b.B)
    assert oracle.check_bound(Y, Cref, bound)[0]
    assert np.array_equal(Y.view(np.uint32), C32.view(np.uint32))   # X @ I is exact in fp32


@pytest.mark.parametrize("mode,u_in", [("tf32", 2.0 ** -10), ("bf16", 2.0 ** -7)])
@pytest.mark.parametrize("cid,channels,n_x", [(2, 3, 64), (4, 2, 128)])
def test_gcn_layer_reduced_precision(h, mode, u_in, cid, channels, n_x):
    """Tensor-core GEMM modes (bspmm_set_gcn_math): X and W are rounded to the
    mode's input format (unit roundoff u_in, truncation worst case: TF32 keeps
    10 mantissa bits, BF16 7), so each product x*w carries a relative error
    <= 2 u_in (+u_in^2); the fp32 accumulation, the storage-order SpMM and the
    channel sum add the fp32 terms of the default bound.  Checked against the
    fp64 oracle; the result must also differ from the fp32 mode somewhere (the
    mode took effect)."""
    rng = np.random.default_rng(cid * 100 + channels + n_x)
    b = synth.config(cid)
    rps, col, vals = channels_of(b, channels, rng)
    X = rng.standard_normal((b.n_rows, n_x)).astype(np.float32)
    W = (rng.standard_normal((channels, n_x, b.k)) / np.sqrt(n_x)).astype(np.float32)
    bias = rng.standard_normal((channels, b.k)).astype(np.float32)
    h.set_hints(int(b.sizes.max()), 0)
    args = (T(b.row_off), None, T(rps), T(col), T(vals), T(X), T(W), T(bias))
    try:
        h.set_gcn_math(mode)
        Y = h.gcn_layer(*args).cpu().numpy()
    finally:
        h.set_gcn_math("fp32")
    Y32 = h.gcn_layer(*args).cpu().numpy()
    ref, mag = oracle.gcn_layer(b.row_off, rps, col, vals, X, W, bias)
    dmax = int(max(np.diff(rp).max() for rp in rps))
    tol = 2 * u_in + u_in * u_in + (n_x + dmax + channels + 4) * 2.0 ** -23
    err = np.abs(Y.astype(np.float64) - ref)
    assert np.all(err <= tol * mag + 1e-30), float((err / np.maximum(mag, 1e-300)).max())
    assert not np.array_equal(Y.view(np.uint32), Y32.view(np.uint32))


@pytest.mark.parametrize("cid", [1, 2, 3, 4])
def test_gcn_accumulate_writes_each_element_once(h, cid):
    """Write-count check (SURVEY §4 tier 4): with W = I, no bias and C channels
    sharing one integer-valued adjacency, the layer is Y = C * (A X) exactly --
    channel ch > 0 adds its SpMM onto Y in the epilogue, so an element written
    twice by one launch (or skipped) would be off by a whole A X term.  Every
    row's tile is covered by the kernel's store pattern exactly once."""
    channels = 3
    b = synth.config(cid, int_valued=True)
    X = b.B
    rps = np.stack([b.row_ptr] * channels)
    h.set_hints(int(b.sizes.max()), 0)
    Y = h.gcn_layer(T(b.row_off), None, T(rps), T(b.col), T(b.vals), T(X),
                    T(np.stack([np.eye(b.k, dtype=np.float32)] * channels))).cpu().numpy()
    AX = oracle.spmm_f32(b.k, b.row_off, None, b.row_ptr, b.col, b.vals, X)
    assert np.array_equal(Y, channels * AX)
