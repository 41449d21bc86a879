"""Handle state across streams and the fused COO path's capacity check.

A handle's workspace (the backward's internal A^T, the offsets of a sizes-only
call, the COO CSR) is shared by its calls.  bspmm_set_stream orders a call on
a new stream after everything enqueued on the previous one, so a call issued
on stream S2 cannot overwrite workspace that work still queued on S1 (or on
the handle's auxiliary stream, joined into S1) reads.  Results are checked
against the oracle; without the ordering the grad_B below reads a workspace
that the second call is rewriting."""
import numpy as np
import pytest
import torch

import oracle
import paper_1903_11409_b200 as bs
import synth

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0)


def T(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def test_backward_then_csr_on_another_stream():
    h = bs.Handle(0)
    b = synth.config(5, i0=0, i1=12000)          # grad_B reads the handle's A^T workspace for a while
    rng = np.random.default_rng(5)
    G = (rng.integers(-(1 << 23), 1 << 23, size=(b.n_rows, b.k)) / float(1 << 23)).astype(np.float32)
    ro, rp, col, vals, B, Gd, sz = T(b.row_off), T(b.row_ptr), T(b.col), T(b.vals), T(b.B), T(G), T(b.sizes)
    # a large sizes-only batch: its offsets are built into the same workspace
    b2 = synth.config(5, i0=20000, i1=60000)
    rp2, col2, vals2, B2, sz2 = T(b2.row_ptr), T(b2.col), T(b2.vals), T(b2.B), T(b2.sizes)
    h.set_hints(int(max(b.sizes.max(), b2.sizes.max())), int(max(b.nnz.max(), b2.nnz.max())))
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(DEV), torch.cuda.Stream(DEV)
    for _ in range(3):
        with torch.cuda.stream(s1):
            gB, gv = h.csr_backward(ro, None, rp, col, vals, B, Gd)
        with torch.cuda.stream(s2):
            C2 = h.csr(None, sz2, rp2, col2, vals2, B2)
        torch.cuda.synchronize()
        ort, oct_, ovt = oracle.csr_transpose(b.row_off, None, b.row_ptr, b.col, b.vals)
        ref = oracle.spmm_f32(b.k, b.row_off, None, ort, oct_, ovt, G)
        assert np.array_equal(gB.cpu().numpy().view(np.uint32), ref.view(np.uint32))
        ref2 = oracle.spmm_f32(b2.k, b2.row_off, None, b2.row_ptr, b2.col, b2.vals, b2.B)
        assert np.array_equal(C2.cpu().numpy().view(np.uint32), ref2.view(np.uint32))


def test_offsets_on_two_streams():
    """Two offsets builds on different streams share the scan tickets and status
    words: ordered by the handle, both are exact."""
    h = bs.Handle(0)
    rng = np.random.default_rng(7)
    s1, s2 = torch.cuda.Stream(DEV), torch.cuda.Stream(DEV)
    for trial in range(5):
        a = rng.integers(0, 300, size=200000).astype(np.int32)
        c = rng.integers(0, 300, size=150000).astype(np.int32)
        da, dc = T(a), T(c)
        torch.cuda.synchronize()
        with torch.cuda.stream(s1):
            oa = h.build_offsets(da)
        with torch.cuda.stream(s2):
            oc = h.build_offsets(dc)
        torch.cuda.synchronize()
        assert np.array_equal(oa.cpu().numpy(), oracle.offsets(a))
        assert np.array_equal(oc.cpu().numpy(), oracle.offsets(c))


def test_coo_checked_reports_skipped_matrix():
    """With hints too small for a matrix, the fused COO launch skips it; the
    checked call raises instead of returning C with unwritten rows."""
    h = bs.Handle(0)
    b = synth.config(3, coo=True)
    h.set_hints(16, 32)                           # far below config 3's largest matrices
    with pytest.raises(bs.BspmmError):
        h.coo(T(b.row_off), None, T(b.nnz_off), T(b.coo_idx), T(b.coo_vals), T(b.B), checked=True)
    h.set_hints(int(b.sizes.max()), int(b.nnz.max()))
    C = h.coo(T(b.row_off), None, T(b.nnz_off), T(b.coo_idx), T(b.coo_vals), T(b.B), checked=True)
    ref = oracle.spmm_f32(b.k, b.row_off, None, b.row_ptr, b.col, b.vals, b.B)
    assert np.array_equal(C.cpu().numpy().view(np.uint32), ref.view(np.uint32))
