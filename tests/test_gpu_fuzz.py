"""Randomised parity sweep over every entry point (GPU): seeded random batches
of random shape (batch 1-700, n_i 0-120, up to 12 entries per row with
duplicates, empty rows and graphs), random k (including odd and non-multiple-
of-4 widths), hints exact / absent / too small, and a random kernel choice
(pipeline, tile kernel with TMA or cp.async staging, no pre-wait prefetch):
  * CSR SpMM: bitwise O3' (the fp32 storage-order FMA oracle) and within
    the north_star bound of O3; SparseTensor SpMM (fused with exact hints,
    device COO->CSR + CSR without): bitwise O3' over the oracle's canonical
    CSR;
  * backward: grad_B bitwise O3' over the oracle's A^T, grad_vals within
    the bound of O6; the transpose bit-exact.
Each case is small (the oracle finishes in milliseconds); 60 seeds."""
import numpy as np
import pytest
import torch

import oracle
import paper_1903_11409_b200 as bs
import synth

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0)
KS = [1, 3, 4, 8, 16, 31, 32, 64, 100, 128, 256, 300, 512]
DBG = [0, 16384, 32768, 1 << 24, 16384 | (1 << 24)]


@pytest.fixture(scope="module")
def h():
    assert torch.cuda.is_available()
    return bs.Handle(0)


def T(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


@pytest.mark.parametrize("seed", range(60))
def test_fuzz_all_paths(h, seed):
    rng = np.random.default_rng(9000 + seed)
    batch = int(rng.choice([1, 5, 37, 150, 400, 700]))
    k = int(rng.choice(KS))
    nmax = int(rng.choice([4, 30, 60, 120]))
    b = synth.random_batch(rng, batch, k, nmax=nmax, dmax=int(rng.integers(1, 13)), duplicates=bool(rng.random() < 0.5))
    if b.n_rows == 0:
        return
    hint = int(rng.integers(0, 3))  # 0: none, 1: exact, 2: too small
    rows = int(b.sizes.max()) if b.batch else 0
    nnz = int(b.nnz.max()) if b.batch else 0
    hints = {0: (0, 0), 1: (rows, nnz), 2: (max(1, rows // 2), max(1, nnz // 2))}[hint]
    dbg = int(rng.choice(DBG))
    h.set_hints(*hints)
    h.set_debug(dbg)
    try:
        ro, rp, col, vals, B = T(b.row_off), T(b.row_ptr), T(b.col), T(b.vals), T(b.B)
        C = h.csr(ro, None, rp, col, vals, B)
        G = (rng.integers(-(1 << 20), 1 << 20, size=(b.n_rows, k)) / float(1 << 20)).astype(np.float32)
        gB, gv = h.csr_backward(ro, None, rp, col, vals, B, T(G))
        rT, cT, vT = h.csr_transpose(ro, None, rp, col, vals)
        Cc = None
        if hint != 2:  # SparseTensor input (fused with exact hints, device COO->CSR + CSR without)
            Cc = h.coo(ro, None, T(b.nnz_off), T(b.coo_idx), T(b.coo_vals), B, checked=True)
        torch.cuda.synchronize()
    finally:
        h.set_debug(0)
        h.set_hints(0, 0)
    C = C.cpu().numpy()
    C32 = oracle.spmm_f32(k, b.row_off, None, b.row_ptr, b.col, b.vals, b.B)
    assert np.array_equal(C.view(np.uint32), C32.view(np.uint32)), (seed, batch, k, hints, dbg)
    if Cc is not None:  # bitwise O3' over the oracle's canonical CSR of the SparseTensor input
        orp, ocol, ov = oracle.coo2csr(b.row_off, None, b.nnz_off, b.coo_idx, b.coo_vals)
        Cc32 = oracle.spmm_f32(k, b.row_off, None, orp, ocol, ov, b.B)
        assert np.array_equal(Cc.cpu().numpy().view(np.uint32), Cc32.view(np.uint32)), (seed, "coo", hints, dbg)
    Cref, bound = oracle.spmm(k, b.row_off, None, b.row_ptr, b.col, b.vals, b.B)
    assert oracle.check_bound(C, Cref, bound)[0]
    ort, oct_, ovt = oracle.csr_transpose(b.row_off, None, b.row_ptr, b.col, b.vals)
    assert np.array_equal(rT.cpu().numpy(), ort) and np.array_equal(cT.cpu().numpy(), oct_)
    assert np.array_equal(vT.cpu().numpy().view(np.uint32), ovt.view(np.uint32))
    ref32 = oracle.spmm_f32(k, b.row_off, None, ort, oct_, ovt, G)
    assert np.array_equal(gB.cpu().numpy().view(np.uint32), ref32.view(np.uint32)), (seed, batch, k, hints, dbg)
    rv, bv = oracle.sddmm(k, b.row_off, None, b.row_ptr, b.col, b.B, G)
    ok, worst = oracle.check_bound(gv.cpu().numpy(), rv, bv)
    assert ok, (seed, worst)
