"""GPU parity for the backward (NEXT-2): per-matrix transpose bit-exact against
the oracle; grad_B bitwise equal to the fp32 storage-order sum over the
oracle's canonical A^T and within the north_star bound of the fp64 oracle;
grad_vals (SDDMM) within 1e-5 * sum |g||b| per entry."""
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


def grad(b, seed):
    rng = np.random.default_rng(seed)
    return (rng.integers(-(1 << 23), 1 << 23, size=(b.n_rows, b.k)) / float(1 << 23)).astype(np.float32)


def check_transpose(h, b):
    rt, ct, vt = h.csr_transpose(T(b.row_off), None, T(b.row_ptr), T(b.col), T(b.vals))
    ort, oct_, ovt = oracle.csr_transpose(b.row_off, None, b.row_ptr, b.col, b.vals)
    assert np.array_equal(rt.cpu().numpy(), ort)
    assert np.array_equal(ct.cpu().numpy(), oct_)
    assert np.array_equal(vt.cpu().numpy().view(np.uint32), ovt.view(np.uint32))
    return ort, oct_, ovt


@pytest.mark.parametrize("cid", [1, 2, 3, 4])
def test_backward_configs(h, cid):
    b = synth.config(cid)
    G = grad(b, cid)
    ort, oct_, ovt = check_transpose(h, b)
    gB, gv = h.csr_backward(T(b.row_off), None, T(b.row_ptr), T(b.col), T(b.vals), T(b.B), T(G))
    torch.cuda.synchronize()
    gB, gv = gB.cpu().numpy(), gv.cpu().numpy()
    ref32 = oracle.spmm_f32(b.k, b.row_off, None, ort, oct_, ovt, G)
    assert np.array_equal(gB.view(np.uint32), ref32.view(np.uint32))
    rB, bB, rv, bv = oracle.backward(b.k, b.row_off, b.row_ptr, b.col, b.vals, b.B, G)
    assert oracle.check_bound(gB, rB, bB)[0]
    ok, worst = oracle.check_bound(gv, rv, bv)
    assert ok, worst


@pytest.mark.parametrize("k", [1, 3, 4, 17, 64, 300, 1024, 1500])
def test_backward_adversarial(h, k):
    rng = np.random.default_rng(k)
    b = synth.random_batch(rng, 25, k, nmax=40, dmax=6, duplicates=True)
    G = grad(b, k + 1)
    check_transpose(h, b)
    gB, gv = h.csr_backward(T(b.row_off), None, T(b.row_ptr), T(b.col), T(b.vals), T(b.B), T(G))
    rB, bB, rv, bv = oracle.backward(b.k, b.row_off, b.row_ptr, b.col, b.vals, b.B, G)
    assert oracle.check_bound(gB.cpu().numpy(), rB, bB)[0]
    assert oracle.check_bound(gv.cpu().numpy(), rv, bv)[0]


def test_backward_large_matrix_transpose_global_path(h):
    """A matrix beyond the shared-memory sort capacity (global merge path)."""
    b = synth.generate(synth.MIX, (2500, 3000, 3, 5), 2, 8, seed=5)
    h.set_hints(0, 0)
    check_transpose(h, b)


def test_sddmm_integer_exact(h):
    b = synth.config(2, int_valued=True)
    G = np.random.default_rng(3).integers(-4, 5, size=(b.n_rows, b.k)).astype(np.float32)
    out = h.sddmm(T(b.row_off), None, T(b.row_ptr), T(b.col), T(b.B), T(G)).cpu().numpy()
    ref, _ = oracle.sddmm(b.k, b.row_off, None, b.row_ptr, b.col, b.B, G)
    assert np.array_equal(out, ref)


@pytest.mark.parametrize("hints", [(0, 0), (60, 200), (300, 2000), (600, 3000)])
def test_transpose_paths_bitexact(h, hints):
    """Every transpose variant (256/512-column windows, shared-memory row ids or
    binary search, several windows per matrix) gives the oracle's canonical A^T:
    a mixed batch with small, medium (> 256 entries) and wide (> 512 rows)
    matrices, duplicates and empty rows, under several planner hints."""
    rng = np.random.default_rng(sum(hints) + 7)
    parts = [synth.random_batch(rng, 20, 4, nmax=40, dmax=6, duplicates=True),
             synth.generate(synth.MIX, (200, 300, 2, 5), 6, 4, seed=11),
             synth.generate(synth.MIX, (520, 700, 1, 3), 2, 4, seed=12)]
    h.set_hints(*hints)
    try:
        for b in parts:
            check_transpose(h, b)
    finally:
        h.set_hints(0, 0)


def _sddmm_check(h, b, G, ld=None, exact=False):
    k = b.k
    ldb = k if ld is None else ld
    Bp = np.zeros((b.n_rows, ldb), dtype=np.float32)
    Bp[:, :k] = b.B
    Gp = np.zeros((b.n_rows, ldb), dtype=np.float32)
    Gp[:, :k] = G
    out = h.sddmm(T(b.row_off), None, T(b.row_ptr), T(b.col), T(Bp), T(Gp), k=k).cpu().numpy()
    ref, bound = oracle.sddmm(k, b.row_off, None, b.row_ptr, b.col, b.B, G)
    if exact:
        assert np.array_equal(out, ref)
    ok, worst = oracle.check_bound(out, ref, bound)
    assert ok, worst


@pytest.mark.parametrize("dbg", [0, 256])
@pytest.mark.parametrize("cid", [2, 3, 4])
def test_sddmm_paths(h, cid, dbg):
    """SDDMM through the SpMM pipeline's SDDMM mode (latency-bound batches) and
    the standalone kernel (debug bit 256): integer-valued inputs exactly (every
    summation order is exact), U[-1,1) inputs within 1e-5 * sum |g||b|."""
    h.set_debug(dbg)
    try:
        b = synth.config(cid, int_valued=True)
        h.set_hints(int(b.sizes.max()), int(b.nnz.max()))
        G = np.random.default_rng(cid).integers(-4, 5, size=(b.n_rows, b.k)).astype(np.float32)
        _sddmm_check(h, b, G, exact=True)
        b = synth.config(cid)
        _sddmm_check(h, b, grad(b, cid + 10))
    finally:
        h.set_debug(0)
        h.set_hints(0, 0)


@pytest.mark.parametrize("k,ld", [(64, 68), (128, 132), (512, 520), (20, 24)])
def test_sddmm_mode_ld_and_direct_units(h, k, ld):
    """SDDMM mode with ld > k (per-row B staging), and matrices above the
    planner hint (the unit computes from global memory, paper case 3)."""
    rng = np.random.default_rng(k + ld)
    b = synth.random_batch(rng, 40, k, nmax=40, dmax=6, duplicates=True)
    _sddmm_check(h, b, grad(b, k), ld=ld)
    h.set_hints(8, 16)  # most matrices exceed the stage: direct units
    try:
        _sddmm_check(h, b, grad(b, k + 1))
    finally:
        h.set_hints(0, 0)


@pytest.mark.parametrize("dbg", [0, 1024])
def test_sddmm_streaming_batch(h, dbg):
    """A batch above 8 matrices per SM takes the standalone kernel (debug bit
    1024: the SpMM pipeline's SDDMM mode instead): C5's first 4096 graphs,
    bound-checked."""
    b = synth.config(5, i0=0, i1=4096)
    h.set_hints(int(b.sizes.max()), int(b.nnz.max()))
    h.set_debug(dbg)
    try:
        _sddmm_check(h, b, grad(b, 5))
    finally:
        h.set_debug(0)
        h.set_hints(0, 0)


@pytest.mark.parametrize("dbg", [0, 1 << 27, 1 << 28])
@pytest.mark.parametrize("k,ld", [(256, 256), (128, 128), (64, 64), (200, 204), (256, 260), (384, 384)])
def test_sddmm_standalone_kernels(h, k, ld, dbg):
    """The standalone SDDMM for streaming batches (1500 matrices > 8 per SM):
    the structure-staged kernel (k <= 256; all lanes active at k = 128 / 256,
    guarded lanes otherwise), its grad_C prefetch-2 variant (bit 28), the
    global-structure kernel (bit 27, and k > 256), with ld > k, rows of 0-9
    entries (1-3 four-entry butterfly groups, duplicates, empty rows and
    graphs); integer-valued inputs exactly, U[-1,1) within the bound.  Then
    hints below the batch's largest matrix: those matrices take the
    out-of-line global loop (B_i or the structure above the stage)."""
    rng = np.random.default_rng(k * 7 + ld + dbg % 1000)
    b = synth.random_batch(rng, 1500, k, nmax=48, dmax=9, duplicates=True, int_valued=True)
    Gi = rng.integers(-4, 5, size=(b.n_rows, k)).astype(np.float32)
    h.set_debug(256 | dbg)
    try:
        h.set_hints(int(b.sizes.max()), int(b.nnz.max()))
        _sddmm_check(h, b, Gi, ld=ld, exact=True)
        bf = synth.random_batch(rng, 1500, k, nmax=48, dmax=9, duplicates=True)
        h.set_hints(int(bf.sizes.max()), int(bf.nnz.max()))
        _sddmm_check(h, bf, grad(bf, k + 3), ld=ld)
        for rows, nnz in ((24, int(bf.nnz.max())), (int(bf.sizes.max()), 40)):
            h.set_hints(rows, nnz)
            _sddmm_check(h, bf, grad(bf, k + 5), ld=ld)
    finally:
        h.set_debug(0)
        h.set_hints(0, 0)


def test_backward_c5_full_size_exhaustive(h):
    """The backward at BASELINE.json's full C5 size (65536 graphs, k = 256; the
    streaming paths: warp-per-matrix transpose, grad_B SpMM, standalone SDDMM),
    checked EVERYWHERE in windows of 8192 graphs (slices of the full arrays,
    rebased): every grad_B row bitwise equal to O3' over the oracle's A^T and
    within the O3 bound, every grad_vals entry within the bound of O6, and no
    NaN left anywhere (every row / entry written)."""
    b = synth.config(5)
    h.set_hints(int(b.sizes.max()), int(b.nnz.max()))
    rng = np.random.default_rng(5150)
    G = (rng.integers(-(1 << 23), 1 << 23, size=(b.n_rows, b.k), dtype=np.int64) / float(1 << 23)).astype(np.float32)
    try:
        gB, gv = h.csr_backward(T(b.row_off), None, T(b.row_ptr), T(b.col), T(b.vals), T(b.B), T(G))
        torch.cuda.synchronize()
    finally:
        h.set_hints(0, 0)
    gB, gv = gB.cpu().numpy(), gv.cpu().numpy()
    torch.cuda.empty_cache()
    assert not np.isnan(gB).any() and not np.isnan(gv).any()
    W = 8192
    for i0 in range(0, b.batch, W):
        i1 = min(b.batch, i0 + W)
        r0, r1 = int(b.row_off[i0]), int(b.row_off[i1])
        z0, z1 = int(b.row_ptr[r0]), int(b.row_ptr[r1])
        ro = b.row_off[i0:i1 + 1] - r0
        rp = b.row_ptr[r0:r1 + 1] - z0
        col, vals, Bw, Gw = b.col[z0:z1], b.vals[z0:z1], b.B[r0:r1], G[r0:r1]
        ort, oct_, ovt = oracle.csr_transpose(ro, None, rp, col, vals)
        ref32 = oracle.spmm_f32(b.k, ro, None, ort, oct_, ovt, Gw)
        nd = np.count_nonzero(gB[r0:r1].view(np.uint32) != ref32.view(np.uint32))
        assert nd == 0, f"graphs [{i0}, {i1}): {nd} grad_B elements differ bitwise from O3'"
        rB, bB = oracle.spmm(b.k, ro, None, ort, oct_, ovt, Gw)
        assert oracle.check_bound(gB[r0:r1], rB, bB)[0], (i0, i1)
        rv, bv = oracle.sddmm(b.k, ro, None, rp, col, Bw, Gw)
        ok, worst = oracle.check_bound(gv[z0:z1], rv, bv)
        assert ok, (i0, i1, worst)


FUSED_OFF = 1 << 29  # debug bit: the separate kernels (transpose + forward kernel, SDDMM)


@pytest.mark.parametrize("k,ld", [(256, 256), (128, 128), (64, 68), (200, 204), (256, 264)])
def test_backward_fused_streaming(h, k, ld):
    """The fused backward kernel (streaming batches: 1500 matrices > 8 per SM,
    hints set): grad_B bitwise equal to O3' over the oracle's A^T and to the
    separate kernels' result (debug bit 29), grad_vals bitwise equal to the
    separate SDDMM and within the O6 bound; duplicates, empty rows and graphs,
    rows of 0-9 entries, ld > k; then hints below the batch's largest matrix
    (those matrices take the fused kernel's out-of-line global path).  grad_B
    is pre-filled with NaN: every row of every matrix must be written."""
    rng = np.random.default_rng(k * 3 + ld)
    b = synth.random_batch(rng, 1500, k, nmax=48, dmax=9, duplicates=True)
    G = grad(b, k + 7)
    Gp = np.zeros((b.n_rows, ld), dtype=np.float32)
    Gp[:, :k] = G
    Bp = np.zeros((b.n_rows, ld), dtype=np.float32)
    Bp[:, :k] = b.B
    ort, oct_, ovt = oracle.csr_transpose(b.row_off, None, b.row_ptr, b.col, b.vals)
    ref32 = oracle.spmm_f32(k, b.row_off, None, ort, oct_, ovt, G)
    rv, bv = oracle.sddmm(k, b.row_off, None, b.row_ptr, b.col, b.B, G)

    def run(dbg, rows, nnz):
        h.set_hints(rows, nnz)
        h.set_debug(dbg)
        try:
            gB = torch.full((b.n_rows, ld), float("nan"), device=DEV)
            gv = torch.full((b.n_nnz,), float("nan"), device=DEV)
            h.csr_backward(T(b.row_off), None, T(b.row_ptr), T(b.col), T(b.vals), T(Bp), T(Gp), k=k,
                           grad_B=gB, grad_vals=gv)
            torch.cuda.synchronize()
        finally:
            h.set_debug(0)
            h.set_hints(0, 0)
        return gB.cpu().numpy()[:, :k], gv.cpu().numpy()

    full = (int(b.sizes.max()), int(b.nnz.max()))
    sep_B, sep_v = run(FUSED_OFF, *full)
    for rows, nnz in (full, (24, full[1]), (full[0], 40)):
        gB, gv = run(0, rows, nnz)
        nd = np.count_nonzero(gB.view(np.uint32) != ref32.view(np.uint32))
        assert nd == 0, f"hints {rows}/{nnz}: {nd} grad_B elements differ bitwise from O3'"
        assert np.array_equal(gB.view(np.uint32), sep_B.view(np.uint32))
        assert np.array_equal(gv.view(np.uint32), sep_v.view(np.uint32)), f"hints {rows}/{nnz}"
        ok, worst = oracle.check_bound(gv, rv, bv)
        assert ok, worst


@pytest.mark.parametrize("cid", [1, 2, 3, 4])
def test_transpose_cta_kernel_configs(h, cid):
    """Small batches with planner hints take the CTA-per-matrix transpose:
    bit-exact against the oracle's A^T, and the backward built on it bitwise
    O3' (grad_B) / within the bound (grad_vals)."""
    b = synth.config(cid)
    h.set_hints(int(b.sizes.max()), int(b.nnz.max()))
    try:
        ort, oct_, ovt = check_transpose(h, b)
        G = grad(b, cid + 20)
        gB, gv = h.csr_backward(T(b.row_off), None, T(b.row_ptr), T(b.col), T(b.vals), T(b.B), T(G))
        torch.cuda.synchronize()
    finally:
        h.set_hints(0, 0)
    ref32 = oracle.spmm_f32(b.k, b.row_off, None, ort, oct_, ovt, G)
    assert np.array_equal(gB.cpu().numpy().view(np.uint32), ref32.view(np.uint32))
    rB, bB, rv, bv = oracle.backward(b.k, b.row_off, b.row_ptr, b.col, b.vals, b.B, G)
    assert oracle.check_bound(gv.cpu().numpy(), rv, bv)[0]


@pytest.mark.parametrize("seed", range(4))
def test_transpose_cta_kernel_adversarial(h, seed):
    """Duplicates, empty rows and graphs, padded layouts (sizes < row_off
    gaps via the sizes argument), matrices above the hinted capacities (the
    kernel's global-memory path): bit-exact against the oracle."""
    rng = np.random.default_rng(seed + 40)
    b = synth.random_batch(rng, 300, 8, nmax=120, dmax=12, duplicates=True)
    for rows, nnz in ((int(b.sizes.max()), int(b.nnz.max())), (32, 64), (int(b.sizes.max()), 100)):
        h.set_hints(rows, nnz)
        try:
            check_transpose(h, b)
        finally:
            h.set_hints(0, 0)


@pytest.mark.parametrize("fused", [True, False])
def test_backward_padded_layout(h, fused):
    """row_off with gaps + sizes (padding rows between the matrices), a
    streaming batch (1500 matrices) so that both adjoints take the fused
    kernel (or, with debug bit 29, the separate kernels): grad_B's matrix rows
    bitwise O3' over the oracle's A^T, padding rows never written (NaN stays),
    grad_vals within the bound."""
    rng = np.random.default_rng(77)
    b = synth.random_batch(rng, 1500, 64, nmax=30, dmax=5, allow_empty_graphs=False, duplicates=True)
    gap = 3
    ro = np.array([int(b.row_off[i]) + gap * i for i in range(b.batch + 1)], dtype=np.int64)
    Np = int(ro[-1])
    rp = np.zeros(Np + 1, dtype=np.int32)
    Bp = np.zeros((Np, 64), dtype=np.float32)
    G = grad(b, 78)
    Gp = np.zeros((Np, 64), dtype=np.float32)
    for i in range(b.batch):
        n = int(b.sizes[i])
        rp[ro[i]:ro[i] + n + 1] = b.row_ptr[b.row_off[i]:b.row_off[i] + n + 1]
        rp[ro[i] + n:ro[i + 1]] = b.row_ptr[b.row_off[i + 1]]
        Bp[ro[i]:ro[i] + n] = b.B[b.row_off[i]:b.row_off[i + 1]]
        Gp[ro[i]:ro[i] + n] = G[b.row_off[i]:b.row_off[i + 1]]
    rp[Np] = b.row_ptr[-1]
    h.set_hints(int(b.sizes.max()), int(b.nnz.max()))
    h.set_debug(0 if fused else FUSED_OFF)
    try:
        gB = torch.full((Np, 64), float("nan"), device=DEV)
        gv = torch.full((b.n_nnz,), float("nan"), device=DEV)
        h.csr_backward(T(ro), T(b.sizes), T(rp), T(b.col), T(b.vals), T(Bp), T(Gp), grad_B=gB, grad_vals=gv)
        torch.cuda.synchronize()
    finally:
        h.set_debug(0)
        h.set_hints(0, 0)
    gB, gv = gB.cpu().numpy(), gv.cpu().numpy()
    ort, oct_, ovt = oracle.csr_transpose(b.row_off, None, b.row_ptr, b.col, b.vals)
    ref32 = oracle.spmm_f32(64, b.row_off, None, ort, oct_, ovt, G)
    for i in range(b.batch):
        n = int(b.sizes[i])
        assert np.array_equal(gB[ro[i]:ro[i] + n].view(np.uint32),
                              ref32[b.row_off[i]:b.row_off[i + 1]].view(np.uint32)), i
        assert np.all(np.isnan(gB[ro[i] + n:ro[i + 1]])), i
    rv, bv = oracle.sddmm(64, b.row_off, None, b.row_ptr, b.col, b.B, G)
    ok, worst = oracle.check_bound(gv, rv, bv)
    assert ok, worst
