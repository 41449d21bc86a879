"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded inputs.  Bars:
* integer / index work (offsets, COO->CSR, partition, shards): bit-exact;
* fp32 C: |C - C_ref| <= 1e-5 * sum|a||b| per element against the fp64 oracle
  (north_star), AND bitwise equal to the fp32 storage-order FMA oracle O3'
  (the kernel keeps CSR storage order), AND exact on integer-valued inputs.
"""
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
    assert torch.cuda.is_available(), "GPU tests need a B200"
    assert torch.cuda.get_device_capability(0) == (10, 0)
    return bs.Handle(0)


def T(a, dt=None):
    t = torch.from_numpy(np.ascontiguousarray(a))
    return t.to(DEV) if dt is None else t.to(DEV, dt)


def run_csr(h, b, sizes=False, ld=None, hints=True, C_init=None):
    if hints:
        h.set_hints(int(b.sizes.max()) if b.batch else 0, int(b.nnz.max()) if b.batch else 0)
    else:
        h.set_hints(0, 0)
    k = b.k
    ldb = k if ld is None else ld
    Bp = np.zeros((b.n_rows, ldb), dtype=np.float32)
    Bp[:, :k] = b.B
    Bd = T(Bp)
    Cd = torch.full((b.n_rows, ldb), float("nan"), device=DEV) if C_init is None else T(C_init)
    h.csr(T(b.row_off), T(b.sizes) if sizes else None, T(b.row_ptr), T(b.col), T(b.vals), Bd, Cd, k=k,
          batch=b.batch)
    torch.cuda.synchronize()
    return Cd.cpu().numpy()[:, :k]


def assert_parity(b, C, what=""):
    C32 = oracle.spmm_f32(b.k, b.row_off, None, b.row_ptr, b.col, b.vals, b.B)
    Cref, bound = oracle.spmm(b.k, b.row_off, None, b.row_ptr, b.col, b.vals, b.B)
    ok, worst = oracle.check_bound(C, Cref, bound)
    assert ok, f"{what}: bound violated, worst |d|/bound = {worst}"
    diff = np.nonzero(C.view(np.uint32) != C32.view(np.uint32))
    assert diff[0].size == 0, f"{what}: {diff[0].size} elements differ bitwise from O3', first {diff[0][:5]}"


# debug bit 16384 keeps small batches on the pipeline kernel (spmm_csr.cu);
# 0 lets the planner choose; "tile" forces the small-batch tile kernel
# (spmm_tile.cu) with 8-float4 column blocks (2-D tensor TMA staging of B),
# "tile_cpasync" the same kernel staging B by cp.async (debug bit 32768)
KERNELS = {"auto": (0, 0), "pipeline": (16384, 0), "tile": (0, 8), "tile_cpasync": (32768, 8)}


def use_kernel(h, kern):
    dbg, cb = KERNELS[kern]
    h.set_debug(dbg)
    h.set_tile_cb(cb)


# ------------------------------------------------------------ a-1 offsets

@pytest.mark.parametrize("batch", [0, 1, 5, 1023, 1024, 1025, 4095, 4096, 4097, 65536, 100003])
def test_offsets_bit_exact(h, batch):
    rng = np.random.default_rng(batch)
    sizes = rng.integers(0, 300, size=batch).astype(np.int32)
    sizes[::7] = 0
    out = h.build_offsets(T(sizes))
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), oracle.offsets(sizes))


def test_offsets_int64_no_wrap(h):
    sizes = np.full(5000, (1 << 31) - 1, dtype=np.int32)
    out = h.build_offsets(T(sizes)).cpu().numpy()
    assert np.array_equal(out, oracle.offsets(sizes)) and out[-1] > (1 << 40)


# ------------------------------------------------------------ a-3..a-6 CSR SpMM

@pytest.mark.parametrize("kern", list(KERNELS))
@pytest.mark.parametrize("cid", [1, 2, 3, 4])
@pytest.mark.parametrize("int_valued", [False, True])
def test_configs_csr(h, cid, int_valued, kern):
    b = synth.config(cid, int_valued=int_valued)
    use_kernel(h, kern)
    try:
        C = run_csr(h, b)
        if kern.startswith("tile"):
            assert h.last_plan()["kernel"] == 1, "forced tile kernel did not run"
        if kern == "pipeline":
            assert h.last_plan()["kernel"] == 0
    finally:
        use_kernel(h, "auto")
    assert_parity(b, C, f"config {cid}")
    if int_valued:
        Cref, _ = oracle.spmm(b.k, b.row_off, None, b.row_ptr, b.col, b.vals, b.B)
        assert np.array_equal(C, Cref)


@pytest.mark.parametrize("k", [1, 2, 3, 4, 5, 8, 16, 17, 33, 64, 100, 128, 256, 300, 512, 1000, 1024])
def test_k_sweep_adversarial(h, k):
    rng = np.random.default_rng(1000 + k)
    for trial in range(4):
        b = synth.random_batch(rng, int(rng.integers(1, 40)), k, nmax=70, dmax=6, duplicates=trial % 2 == 1)
        for kern in KERNELS:
            use_kernel(h, kern)
            try:
                assert_parity(b, run_csr(h, b), f"k={k} trial={trial} {kern}")
                assert_parity(b, run_csr(h, b, sizes=True, hints=False), f"k={k} trial={trial} no hints {kern}")
            finally:
                use_kernel(h, "auto")


@pytest.mark.parametrize("k,ld", [(16, 20), (64, 68), (5, 7), (128, 129), (256, 260)])
@pytest.mark.parametrize("kern", list(KERNELS))
def test_leading_dimension(h, k, ld, kern):
    rng = np.random.default_rng(k * ld)
    b = synth.random_batch(rng, 30, k, nmax=40, dmax=5)
    use_kernel(h, kern)
    try:
        C = run_csr(h, b, ld=ld)
    finally:
        use_kernel(h, "auto")
    assert_parity(b, C, f"k={k} ld={ld}")


@pytest.mark.parametrize("kern", list(KERNELS))
def test_padded_layout_untouched(h, kern):
    """row_off with gaps + sizes: only matrix rows are written (padding stays NaN)."""
    rng = np.random.default_rng(42)
    b = synth.random_batch(rng, 20, 64, nmax=30, allow_empty_graphs=False)
    gap = 5
    ro = np.array([int(b.row_off[i]) + gap * i for i in range(b.batch + 1)], dtype=np.int64)
    Np = int(ro[-1])
    rp = np.zeros(Np + 1, dtype=np.int32)
    Bp = np.zeros((Np, 64), dtype=np.float32)
    for i in range(b.batch):
        n = int(b.sizes[i])
        rp[ro[i]:ro[i] + n + 1] = b.row_ptr[b.row_off[i]:b.row_off[i] + n + 1]
        rp[ro[i] + n:ro[i + 1]] = b.row_ptr[b.row_off[i + 1]]
        Bp[ro[i]:ro[i] + n] = b.B[b.row_off[i]:b.row_off[i + 1]]
    rp[Np] = b.row_ptr[-1]
    Cd = torch.full((Np, 64), float("nan"), device=DEV)
    h.set_hints(0, 0)
    use_kernel(h, kern)
    try:
        h.csr(T(ro), T(b.sizes), T(rp), T(b.col), T(b.vals), T(Bp), Cd)
        C = Cd.cpu().numpy()
    finally:
        use_kernel(h, "auto")
    Cref = oracle.spmm_f32(64, b.row_off, None, b.row_ptr, b.col, b.vals, b.B)
    for i in range(b.batch):
        n = int(b.sizes[i])
        assert np.array_equal(C[ro[i]:ro[i] + n], Cref[b.row_off[i]:b.row_off[i + 1]])
        assert np.all(np.isnan(C[ro[i] + n:ro[i + 1]]))


@pytest.mark.parametrize("kern", list(KERNELS))
def test_large_matrices_direct_path(h, kern):
    """Matrices beyond the stage capacity (paper case 3) run from global memory."""
    use_kernel(h, kern)
    try:
        for k in (256, 7):
            b = synth.generate(synth.MIX, (1500, 3000, 1, 8), 3, k, seed=77)
            h.set_hints(64, 512)  # deliberately too small: forces the direct path
            C = run_csr(h, b, hints=False)
            assert_parity(b, C, f"direct k={k}")
            # and with hints large enough that some units stage, mixed with direct ones
            assert_parity(b, run_csr(h, b, hints=True), f"mixed k={k}")
    finally:
        use_kernel(h, "auto")


def test_empty_batch_and_empty_graphs(h):
    b = synth.random_batch(np.random.default_rng(3), 6, 32, nmax=0)   # every graph has n_i = 0
    assert b.n_rows == 0
    run_csr(h, b)
    h.csr(T(np.zeros(1, np.int64)), None, T(np.zeros(1, np.int32)), T(np.zeros(0, np.int32)),
          T(np.zeros(0, np.float32)), torch.zeros((0, 8), device=DEV), torch.zeros((0, 8), device=DEV), batch=0)
    torch.cuda.synchronize()


def test_tuning_space_bitwise(h):
    """Every (kt, warps, CTAs/SM) choice computes the same bits (storage-order FMA)."""
    b = synth.config(4)
    ref = run_csr(h, b)
    for kt in (32, 64, 128, 256, 512):
        for warps in (1, 4, 16):
            for ctas in (1, 2):
                for chunks in (1, 2, 4):
                    h.set_tuning(kt, warps, ctas, chunks)
                    C = run_csr(h, b)
                    assert np.array_equal(C.view(np.uint32), ref.view(np.uint32)), (kt, warps, ctas, chunks)
    h.set_tuning(0, 0, 0, 0)
    for sched_bits in (64, 128):            # static and dynamic unit schedules, same bits
        h.set_debug(sched_bits)
        for cid in (3, 4):
            bb = synth.config(cid)
            assert_parity(bb, run_csr(h, bb), f"sched {sched_bits} config {cid}")
    use_kernel(h, "auto")


def test_deterministic_repeat(h):
    b = synth.config(3)
    a = run_csr(h, b)
    c = run_csr(h, b)
    assert np.array_equal(a.view(np.uint32), c.view(np.uint32))


# ------------------------------------------------------------ a-2 COO -> CSR

def test_coo2csr_bit_exact_configs(h):
    for cid in (1, 3):
        b = synth.config(cid, coo=True)
        rp, col, v = h.coo2csr(T(b.row_off), None, T(b.nnz_off), T(b.coo_idx), T(b.coo_vals), b.n_rows)
        torch.cuda.synchronize()
        orp, ocol, ov = oracle.coo2csr(b.row_off, None, b.nnz_off, b.coo_idx, b.coo_vals)
        assert np.array_equal(rp.cpu().numpy(), orp)
        assert np.array_equal(col.cpu().numpy(), ocol)
        assert np.array_equal(v.cpu().numpy().view(np.uint32), ov.view(np.uint32))


@pytest.mark.parametrize("seed", range(6))
def test_coo2csr_adversarial(h, seed):
    rng = np.random.default_rng(500 + seed)
    b = synth.random_batch(rng, int(rng.integers(1, 50)), 4, nmax=40, dmax=8, duplicates=True)
    rp, col, v = h.coo2csr(T(b.row_off), T(b.sizes), T(b.nnz_off), T(b.coo_idx), T(b.coo_vals), b.n_rows)
    orp, ocol, ov = oracle.coo2csr(b.row_off, b.sizes, b.nnz_off, b.coo_idx, b.coo_vals)
    assert np.array_equal(rp.cpu().numpy(), orp)
    assert np.array_equal(col.cpu().numpy(), ocol)
    assert np.array_equal(v.cpu().numpy().view(np.uint32), ov.view(np.uint32))


def test_coo2csr_global_fallback(h):
    """A matrix with more entries than the shared-memory sort capacity (global merge path)."""
    rng = np.random.default_rng(9)
    n, m = 3000, 20000
    idx = np.stack([rng.integers(0, n, m), rng.integers(0, n, m)], 1).astype(np.int32)
    idx[1000:1100] = idx[0]                                  # duplicates across the range
    vals = rng.standard_normal(m).astype(np.float32)
    ro = np.array([0, 7, 7 + n, 7 + n + 5], dtype=np.int64)
    sizes = np.array([7, n, 5], dtype=np.int32)
    small = np.array([[1, 2], [0, 0], [6, 6]], dtype=np.int32)
    allidx = np.concatenate([small, idx, np.array([[4, 4]], np.int32)])
    allv = np.concatenate([np.ones(3, np.float32), vals, np.ones(1, np.float32)])
    no = np.array([0, 3, 3 + m, 4 + m], dtype=np.int64)
    h.set_hints(0, 0)
    rp, col, v = h.coo2csr(T(ro), T(sizes), T(no), T(allidx), T(allv), int(ro[-1]))
    orp, ocol, ov = oracle.coo2csr(ro, sizes, no, allidx, allv)
    assert np.array_equal(rp.cpu().numpy(), orp)
    assert np.array_equal(col.cpu().numpy(), ocol)
    assert np.array_equal(v.cpu().numpy().view(np.uint32), ov.view(np.uint32))


@pytest.mark.parametrize("cid", [1, 3])
def test_coo_spmm(h, cid):
    b = synth.config(cid, coo=True)
    h.set_hints(int(b.sizes.max()), int(b.nnz.max()))
    rp = torch.empty(b.n_rows + 1, dtype=torch.int32, device=DEV)
    col = torch.empty(b.n_nnz, dtype=torch.int32, device=DEV)
    v = torch.empty(b.n_nnz, dtype=torch.float32, device=DEV)
    C = h.coo(None, T(b.sizes), T(b.nnz_off), T(b.coo_idx), T(b.coo_vals), T(b.B), csr_out=(rp, col, v))
    C2 = h.coo(T(b.row_off), None, T(b.nnz_off), T(b.coo_idx), T(b.coo_vals), T(b.B))
    torch.cuda.synchronize()
    orp, ocol, ov = oracle.coo2csr(b.row_off, None, b.nnz_off, b.coo_idx, b.coo_vals)
    assert np.array_equal(rp.cpu().numpy(), orp) and np.array_equal(col.cpu().numpy(), ocol)
    C32 = oracle.spmm_f32(b.k, b.row_off, None, orp, ocol, ov, b.B)
    Cref, bound = oracle.spmm(b.k, b.row_off, None, orp, ocol, ov, b.B)
    for Cg in (C.cpu().numpy(), C2.cpu().numpy()):
        assert oracle.check_bound(Cg, Cref, bound)[0]
        assert np.array_equal(Cg.view(np.uint32), C32.view(np.uint32))


# ------------------------------------------------------------ a-7 shards (one-GPU emulation)

@pytest.mark.parametrize("G", [2, 4, 8])
def test_shard_emulation_bitwise(h, G):
    b = synth.config(2)
    full = run_csr(h, b)
    split = bs.partition(b.nnz_off, b.k, G)
    assert np.array_equal(split, oracle.partition(b.nnz_off, b.k, G))
    out = np.full_like(full, np.nan)
    for r in range(G):
        i0, i1 = int(split[r]), int(split[r + 1])
        if i1 == i0:
            continue
        part = synth.config(2, i0=i0, i1=i1)           # regenerated per rank from per-graph seeds
        Cr = run_csr(h, part)
        out[b.row_off[i0]:b.row_off[i1]] = Cr
    assert np.array_equal(out.view(np.uint32), full.view(np.uint32))


# ------------------------------------------------------------ e2e host path

@pytest.mark.parametrize("cid", [2, 4])
def test_host_path_matches_device_path(h, cid):
    b = synth.config(cid)
    dev = run_csr(h, b)
    C = h.csr_host(b.sizes, b.row_ptr, b.col, b.vals, b.B)
    assert np.array_equal(C.view(np.uint32), dev.view(np.uint32))


def test_host_path_chunked_pinned(h):
    b = synth.config(5, i0=0, i1=20000)          # ~270 MB of B+C: several pipeline chunks
    h.set_hints(60, 200)
    pin = lambda a: torch.from_numpy(a).pin_memory()
    C = torch.empty((b.n_rows, b.k), dtype=torch.float32).pin_memory()
    h.csr_host(pin(b.sizes), pin(b.row_ptr), pin(b.col), pin(b.vals), pin(b.B), C)
    rng = np.random.default_rng(1)
    mat = rng.integers(0, b.batch, 400)
    rl = np.array([rng.integers(0, b.sizes[i]) for i in mat], np.int32)
    ref, bound = oracle.spmm_rows(mat, rl, b.k, b.row_off, b.row_ptr, b.col, b.vals, b.B)
    got = C.numpy()[b.row_off[mat] + rl]
    assert oracle.check_bound(got, ref, bound)[0]


# ------------------------------------------------------------ VALIDATE

def test_validate_flags_bad_index():
    hv = bs.Handle(0, validate=True)
    b = synth.config(1)
    col = b.col.copy()
    col[3] = 8                                    # == n_i: out of range
    with pytest.raises(bs.BspmmError, match="INDEX"):
        hv.csr(T(b.row_off), None, T(b.row_ptr), T(col), T(b.vals), T(b.B))
    idx = b.coo_idx.copy()
    idx[0, 0] = -1
    with pytest.raises(bs.BspmmError, match="INDEX"):
        hv.coo(T(b.row_off), None, T(b.nnz_off), T(idx), T(b.coo_vals), T(b.B))
    with pytest.raises(bs.BspmmError, match="INDEX"):
        hv.build_offsets(T(np.array([3, -1], np.int32)))
    # valid input passes under VALIDATE and gives the same bits
    C = hv.csr(T(b.row_off), None, T(b.row_ptr), T(b.col), T(b.vals), T(b.B)).cpu().numpy()
    assert_parity(b, C, "validate")


def test_invalid_arguments_rejected(h):
    b = synth.config(1)
    with pytest.raises(bs.BspmmError, match="INVALID"):
        h.csr(T(b.row_off), None, T(b.row_ptr), T(b.col), T(b.vals), T(b.B), k=0)
    Bd = T(b.B)
    with pytest.raises(bs.BspmmError, match="INVALID"):
        h.csr(T(b.row_off), None, T(b.row_ptr), T(b.col), T(b.vals), Bd, C=Bd)


# ------------------------------------------------------------ full size (BASELINE.json c5, bench launch config)

def window(b, i0, i1):
    """Graphs [i0, i1) of batch b rebased to row / entry 0 (slices of b's arrays,
    no regeneration): (row_off, row_ptr, col, vals, B, r0, r1, z0, z1)."""
    r0, r1 = int(b.row_off[i0]), int(b.row_off[i1])
    z0, z1 = int(b.row_ptr[r0]), int(b.row_ptr[r1])
    return (b.row_off[i0:i1 + 1] - r0, b.row_ptr[r0:r1 + 1] - z0, b.col[z0:z1], b.vals[z0:z1], b.B[r0:r1],
            r0, r1, z0, z1)


def test_c5_full_size_exhaustive(h):
    """BASELINE.json configs[4] at full size (65536 graphs, k = 256) in the bench's
    launch configuration (device offsets builder + SpMM): the offsets bit-exact
    against oracle.offsets, EVERY row bitwise equal to O3' and EVERY element
    within the north_star bound of O3 (checked in windows of 8192 graphs to
    bound host memory), and no element left unwritten."""
    b = synth.config(5)
    h.set_hints(60, int(b.nnz.max()))
    Bd, Cd = T(b.B), torch.full((b.n_rows, b.k), float("nan"), device=DEV)
    sizes = T(b.sizes)
    ro = h.build_offsets(sizes)                        # the bench step: offsets + SpMM
    h.csr(ro, None, T(b.row_ptr), T(b.col), T(b.vals), Bd, Cd)
    torch.cuda.synchronize()
    assert np.array_equal(ro.cpu().numpy(), oracle.offsets(b.sizes))
    C = Cd.cpu().numpy()
    del Bd, Cd
    assert not np.isnan(C).any()
    W = 8192
    for i0 in range(0, b.batch, W):
        i1 = min(b.batch, i0 + W)
        ro1, rp1, col1, v1, B1, r0, r1, _, _ = window(b, i0, i1)
        ref32 = oracle.spmm_f32(b.k, ro1, None, rp1, col1, v1, B1)
        diff = np.count_nonzero(C[r0:r1].view(np.uint32) != ref32.view(np.uint32))
        assert diff == 0, f"graphs [{i0}, {i1}): {diff} elements differ bitwise from O3'"
        ref, bound = oracle.spmm(b.k, ro1, None, rp1, col1, v1, B1)
        ok, worst = oracle.check_bound(C[r0:r1], ref, bound)
        assert ok, f"graphs [{i0}, {i1}): worst |d|/bound = {worst}"


def test_fmaf_single_rounding_pin(h):
    """The kernel accumulates with fused multiply-add, as O3' does (SURVEY §8(c)
    O3'): row (v = -(1+2^-11), b = 1), then (v = 1+2^-12, b = 1+2^-12) gives
    exactly 2^-24 with one rounding per FMA; multiply-then-add gives 0."""
    n, k = 2, 4                                        # a 2-node graph: row 0 has entries at cols 0, 1
    ro = np.array([0, 2], np.int64)
    rp = np.array([0, 2, 2], np.int32)
    col = np.array([0, 1], np.int32)
    vals = np.array([-(1 + 2.0 ** -11), 1 + 2.0 ** -12], np.float32)
    B = np.zeros((n, k), np.float32)
    B[0, :] = 1.0
    B[1, :] = 1 + 2.0 ** -12
    h.set_hints(2, 2)
    C = h.csr(T(ro), None, T(rp), T(col), T(vals), T(B)).cpu().numpy()
    assert np.all(C[0] == np.float32(2.0 ** -24)), C[0]
    assert np.all(C[1] == 0.0)
    ref32 = oracle.spmm_f32(k, ro, None, rp, col, vals, B)
    assert np.array_equal(C.view(np.uint32), ref32.view(np.uint32))


# ------------------------------------------------------------ NEXT-3: the paper's atomic SWA-ST kernel

@pytest.mark.parametrize("cid", [1, 2, 3, 4])
def test_coo_atomic_within_bound(h, cid):
    b = synth.config(cid, coo=True)
    h.set_hints(int(b.sizes.max()), int(b.nnz.max()))
    C = h.coo_atomic(T(b.row_off), None, T(b.nnz_off), T(b.coo_idx), T(b.coo_vals), T(b.B)).cpu().numpy()
    Cref, bound = oracle.spmm(b.k, b.row_off, None, b.row_ptr, b.col, b.vals, b.B)
    ok, worst = oracle.check_bound(C, Cref, bound)
    assert ok, worst


def test_coo_atomic_edge_cases(h):
    rng = np.random.default_rng(77)
    for trial in range(6):
        b = synth.random_batch(rng, 30, 64, nmax=50, dmax=6, duplicates=True)
        h.set_hints(16 if trial % 2 else 0, 0)        # small hint: global-atomic case 3 for big matrices
        Cd = torch.full((b.n_rows, 64), float("nan"), device=DEV)
        C = h.coo_atomic(None, T(b.sizes), T(b.nnz_off), T(b.coo_idx), T(b.coo_vals), T(b.B), Cd).cpu().numpy()
        Cref, bound = oracle.spmm(b.k, b.row_off, None, b.row_ptr, b.col, b.vals, b.B)
        assert oracle.check_bound(C, Cref, bound)[0], trial
    with pytest.raises(bs.BspmmError, match="NOT_SUPPORTED"):
        b = synth.random_batch(rng, 3, 5, nmax=5)
        h.coo_atomic(T(b.row_off), None, T(b.nnz_off), T(b.coo_idx), T(b.coo_vals), T(b.B))


# ------------------------------------------------------------ a-1 fused into the SpMM (row_off == NULL)

@pytest.mark.parametrize("cid", [1, 2, 3, 4])
def test_fused_offsets_bitwise(h, cid):
    b = synth.config(cid)
    h.set_hints(int(b.sizes.max()), int(b.nnz.max()))
    C1 = h.csr(T(b.row_off), None, T(b.row_ptr), T(b.col), T(b.vals), T(b.B))
    C2 = h.csr(None, T(b.sizes), T(b.row_ptr), T(b.col), T(b.vals), T(b.B))
    torch.cuda.synchronize()
    assert torch.equal(C1.view(torch.int32), C2.view(torch.int32))


def test_fused_offsets_adversarial(h):
    rng = np.random.default_rng(99)
    for trial in range(8):
        b = synth.random_batch(rng, int(rng.integers(1, 400)), 64, nmax=30, dmax=4, allow_empty_graphs=True)
        h.set_hints(0, 0)
        for kt in (0, 16, 32):
            h.set_tuning(kt, 0, 0, 0)
            C = h.csr(None, T(b.sizes), T(b.row_ptr), T(b.col), T(b.vals), T(b.B)).cpu().numpy()
            assert_parity(b, C, f"fused offsets trial {trial} kt {kt}")
    h.set_tuning(0, 0, 0, 0)


# ------------------------------------------------------------ a-2 fused into the SpMM (bspmm_coo with hints)

# fused conversion paths: 0 = the planner's choice (small batches: the tile
# kernel's SparseTensor variant), 16384 = the pipeline's converter warps,
# ("tile", cb) = the tile variant at a forced column block
COO_PATHS = {"auto": (0, 0), "pipeline": (16384, 0), "tile_cb1": (0, 1), "tile_cb8": (0, 8)}


@pytest.mark.parametrize("path", list(COO_PATHS))
@pytest.mark.parametrize("seed", range(5))
def test_coo_fused_adversarial(h, seed, path):
    """Unsorted SparseTensor input with duplicates, empty rows and graphs,
    through each fused conversion path: bitwise O3' over the oracle's CSR, and
    the kernel that ran is the one asked for."""
    rng = np.random.default_rng(700 + seed)
    k = [16, 64, 128, 256, 512][seed]
    b = synth.random_batch(rng, int(rng.integers(1, 200)), k, nmax=60, dmax=6, duplicates=True)
    h.set_hints(max(int(b.sizes.max()), 1), max(int(b.nnz.max()), 1))
    dbg, cb = COO_PATHS[path]
    h.set_debug(dbg)
    h.set_tile_cb(cb)
    try:
        C = h.coo(None, T(b.sizes), T(b.nnz_off), T(b.coo_idx), T(b.coo_vals), T(b.B)).cpu().numpy()
        h.sync()
        kern = h.last_plan()["kernel"]
    finally:
        h.set_debug(0)
        h.set_tile_cb(0)
    if path == "pipeline":
        assert kern == 0
    elif path.startswith("tile"):
        assert kern == 1 and h.last_plan()["lanes"] == cb
    orp, ocol, ov = oracle.coo2csr(b.row_off, None, b.nnz_off, b.coo_idx, b.coo_vals)
    C32 = oracle.spmm_f32(b.k, b.row_off, None, orp, ocol, ov, b.B)
    assert np.array_equal(C.view(np.uint32), C32.view(np.uint32))


@pytest.mark.parametrize("cid", [1, 2, 4])
def test_coo_tile_configs_and_long_rows(h, cid):
    """The tile kernel's SparseTensor variant on the small configs (the
    planner's choice there), and on rows longer than the 8-key sorting network
    (the rank-counting path): bitwise equal to the pipeline's converter warps
    and to O3' over the oracle's CSR."""
    b = synth.config(cid, coo=True)
    cases = [b]
    rng = np.random.default_rng(cid)
    cases.append(synth.random_batch(rng, 60, b.k, nmax=40, dmax=20, duplicates=True))
    for bb in cases:
        h.set_hints(int(bb.sizes.max()), int(bb.nnz.max()))
        outs = []
        for dbg in (0, 16384):
            h.set_debug(dbg)
            try:
                outs.append(h.coo(T(bb.row_off), None, T(bb.nnz_off), T(bb.coo_idx), T(bb.coo_vals),
                                  T(bb.B)).cpu().numpy())
                h.sync()
                if dbg == 0 and bb is b:
                    assert h.last_plan()["kernel"] == 1
            finally:
                h.set_debug(0)
        orp, ocol, ov = oracle.coo2csr(bb.row_off, None, bb.nnz_off, bb.coo_idx, bb.coo_vals)
        C32 = oracle.spmm_f32(bb.k, bb.row_off, None, orp, ocol, ov, bb.B)
        for C in outs:
            assert np.array_equal(C.view(np.uint32), C32.view(np.uint32))


@pytest.mark.parametrize("cid", [3, 2])
def test_coo_fused_hint_too_small_is_reported(h, cid):
    """A matrix beyond the hints is skipped and reported by bspmm_sync, on the
    pipeline's converter warps (config 3) and on the tile variant (config 2)."""
    b = synth.config(cid, coo=True)
    h.set_hints(10, 20)                       # below the largest matrices of both configs
    h.coo(T(b.row_off), None, T(b.nnz_off), T(b.coo_idx), T(b.coo_vals), T(b.B))
    with pytest.raises(bs.BspmmError, match="INVALID"):
        h.sync()
    h.sync()                                  # the flag is cleared once reported


# ------------------------------------------------------------ early first tile (whole-row plans)

@pytest.mark.parametrize("k,nlo,nhi,batch", [(512, 20, 120, 40), (384, 5, 90, 30), (256, 1, 60, 70),
                                             (512, 200, 300, 6), (128, 10, 40, 50)])
def test_early_first_tile_shapes(h, k, nlo, nhi, batch):
    """Whole-row plans issue each CTA's first B tile early, from consumer warp 0
    (one bulk copy on a barrier of its own) while the producer does the
    structure round trip.  Mixed sizes (incl. tiles that do not fit a stage and
    k-tiled plans, where the path is off) and empty matrices; bitwise O3'
    either way, also with the early path disabled (debug bit 4) and with sizes
    only (row offsets summed from sizes by consumer warp 0)."""
    b = synth.generate(synth.MIX, (nlo, nhi, 1, 5), batch, k, seed=k + nhi)
    ref = None
    for dbg in (16384, 16384 | 4):              # the pipeline kernel: early tile on / off
        h.set_debug(dbg)
        for sizes in (False, True):
            C = run_csr(h, b, sizes=sizes)
            assert_parity(b, C, f"k={k} dbg={dbg} sizes={sizes}")
            if ref is None:
                ref = C
            assert np.array_equal(C.view(np.uint32), ref.view(np.uint32))
        # sizes only (row_off = NULL): offsets fused into the launch, the early
        # tile's row offset summed from sizes by consumer warp 0
        Cd = torch.full((b.n_rows, k), float("nan"), device=DEV)
        h.csr(None, T(b.sizes), T(b.row_ptr), T(b.col), T(b.vals), T(b.B), Cd)
        torch.cuda.synchronize()
        assert np.array_equal(Cd.cpu().numpy().view(np.uint32), ref.view(np.uint32))
    use_kernel(h, "auto")


def test_early_first_tile_empty_first_matrices(h):
    """Empty matrices at CTA-first positions: no early tile is issued for them
    (producer and consumer warp 0 agree), the CTA's later units run normally."""
    for seed in range(400):
        b = synth.random_batch(np.random.default_rng(seed), 9, 512, nmax=40, dmax=4)
        if b.sizes[0] == 0 and (b.sizes == 0).sum() >= 2 and b.sizes.max() > 0:
            break
    else:
        pytest.fail("no seed with empty leading matrices")
    for kern in KERNELS:
        use_kernel(h, kern)
        try:
            C = run_csr(h, b)
        finally:
            use_kernel(h, "auto")
        assert_parity(b, C, f"empty first matrices {kern}")


# ------------------------------------------------------------ library cross-check (SURVEY §4 tier 6)

@pytest.mark.parametrize("cid", [2, 3, 4])
def test_cusparse_cross_check(h, cid):
    """Independent of both our kernel and the oracle: cuSPARSE (torch.sparse CSR)
    on the block-diagonal matrix with global column ids, within the north_star
    bound of the fp64 oracle -- and our C within the same bound of it."""
    b = synth.config(cid)
    # global column of every entry: local col + row offset of its matrix
    mat_of_entry = np.repeat(np.arange(b.batch), b.nnz)
    gcol = b.col.astype(np.int64) + b.row_off[mat_of_entry]
    A = torch.sparse_csr_tensor(T(b.row_ptr.astype(np.int64)), T(gcol), T(b.vals), size=(b.n_rows, b.n_rows))
    Cs = torch.sparse.mm(A, T(b.B)).cpu().numpy()
    Cref, bound = oracle.spmm(b.k, b.row_off, None, b.row_ptr, b.col, b.vals, b.B)
    assert oracle.check_bound(Cs, Cref, bound)[0]
    C = run_csr(h, b)
    assert np.all(np.abs(C.astype(np.float64) - Cs) <= 2 * bound + 1e-30)


@pytest.mark.parametrize("k,nlo,nhi,batch", [(64, 20, 60, 100), (32, 1, 64, 120), (16, 0, 30, 148),
                                             (128, 10, 60, 90), (256, 5, 30, 40)])
def test_one_unit_consumer_path(h, k, nlo, nhi, batch):
    """One whole-row unit per CTA with all rows covered in one consumer round
    (C2-like): the consumers load their row range and row structure themselves
    and wait only for the early B tile.  Mixed sizes (incl. matrices above the
    hinted rows, which fall back per CTA), empty matrices, sizes / fused
    offsets; bitwise O3' and bitwise equal with the path off (debug bit 1024)."""
    rng = np.random.default_rng(k + batch)
    b = synth.random_batch(rng, batch, k, nmax=nhi, dmax=5, duplicates=True)
    ref = None
    for dbg in (16384, 16384 | 1024):           # the pipeline kernel: one-unit path on / off
        h.set_debug(dbg)
        try:
            for sizes in (False, True):
                C = run_csr(h, b, sizes=sizes)
                assert_parity(b, C, f"k={k} dbg={dbg} sizes={sizes}")
                if ref is None:
                    ref = C
                assert np.array_equal(C.view(np.uint32), ref.view(np.uint32))
            Cd = torch.full((b.n_rows, k), float("nan"), device=DEV)
            h.csr(None, T(b.sizes), T(b.row_ptr), T(b.col), T(b.vals), T(b.B), Cd)
            torch.cuda.synchronize()
            assert np.array_equal(Cd.cpu().numpy().view(np.uint32), ref.view(np.uint32))
            h.set_hints(max(1, nhi // 2), 0)  # many matrices above the hint: per-CTA fallback
            Cd = torch.full((b.n_rows, k), float("nan"), device=DEV)
            h.csr(T(b.row_off), None, T(b.row_ptr), T(b.col), T(b.vals), T(b.B), Cd)
            torch.cuda.synchronize()
            assert np.array_equal(Cd.cpu().numpy().view(np.uint32), ref.view(np.uint32))
        finally:
            use_kernel(h, "auto")
            h.set_hints(0, 0)


# ------------------------------------------------------------ small-batch tile kernel (spmm_tile.cu)

def run_both(h, b, **kw):
    out = {}
    for kern in KERNELS:
        use_kernel(h, kern)
        try:
            out[kern] = run_csr(h, b, **kw)
            out[kern + "_plan"] = h.last_plan()
        finally:
            use_kernel(h, "auto")
    return out


@pytest.mark.parametrize("k,nlo,nhi,batch", [(512, 50, 50, 100), (4, 1, 3, 2048), (8, 0, 9, 1500), (256, 1, 300, 64),
                                             (1024, 2, 40, 7), (64, 20, 60, 100), (128, 10, 300, 200),
                                             (300, 5, 40, 50), (36, 1, 20, 300)])
def test_tile_shapes(h, k, nlo, nhi, batch):
    """The tile kernel over mixed shapes: tiny matrices, empty ones, wide and
    ragged k, large batches; bitwise O3' and bitwise equal to the pipeline
    kernel, with row_off, sizes only (fused offsets) and both; and every
    column-block width (bspmm_set_tile_cb) gives the same bits."""
    b = synth.generate(synth.MIX, (max(nlo, 1), nhi, 1, 5), batch, k, seed=k * 7 + batch)
    out = run_both(h, b)
    assert_parity(b, out["auto"], f"tile k={k} plan={out['auto_plan']}")
    assert np.array_equal(out["auto"].view(np.uint32), out["pipeline"].view(np.uint32))
    out2 = run_both(h, b, sizes=True)                   # row_off + sizes
    assert np.array_equal(out2["auto"].view(np.uint32), out["pipeline"].view(np.uint32))
    Cd = torch.full((b.n_rows, k), float("nan"), device=DEV)
    h.csr(None, T(b.sizes), T(b.row_ptr), T(b.col), T(b.vals), T(b.B), Cd)   # fused offsets
    torch.cuda.synchronize()
    assert np.array_equal(Cd.cpu().numpy().view(np.uint32), out["pipeline"].view(np.uint32))
    for kern in ("tile", "tile_cpasync"):
        assert np.array_equal(out[kern].view(np.uint32), out["pipeline"].view(np.uint32)), kern
    for dbg in (0, 32768):                              # 2-D TMA / cp.async staging of B
        for cb in (1, 2, 4, 8, 16, 32):
            h.set_tile_cb(cb)
            h.set_debug(dbg)
            try:
                C = run_csr(h, b)
                assert h.last_plan()["kernel"] == 1 and h.last_plan()["lanes"] == cb
            finally:
                use_kernel(h, "auto")
            assert np.array_equal(C.view(np.uint32), out["pipeline"].view(np.uint32)), (cb, dbg)


def test_tile_fallbacks(h):
    """Tiles whose matrix exceeds the planned capacity (hints far too small)
    read B and / or the structure from global memory: still bitwise O3'.
    (1) one 20000-row matrix, k = 512; (2) mostly-empty matrices; (3) rows
    and entries beyond the capacity."""
    cases = [synth.generate(synth.MIX, (20000, 20000, 1, 3), 1, 512, seed=5)]
    rng = np.random.default_rng(11)
    sizes = np.where(np.arange(2048) % 50 == 0, 1, 0).astype(np.int32)
    cases.append(synth.random_batch(rng, 2048, 512, dmax=1, sizes=sizes))
    cases.append(synth.generate(synth.MIX, (1500, 3000, 1, 8), 3, 256, seed=77))
    for b in cases:
        h.set_hints(8, 16)                               # deliberately too small
        try:
            out = run_both(h, b, hints=False)
        finally:
            h.set_hints(0, 0)
        assert_parity(b, out["auto"], "tile fallback")
        for kern in KERNELS:
            assert np.array_equal(out[kern].view(np.uint32), out["pipeline"].view(np.uint32)), kern


# ------------------------------------------------ pre-wait L2 prefetch (PDL)
PF_BITS = {"default": 0, "no_prefetch": 1 << 24, "b_only": 1 << 25, "no_col_val_run": 1 << 26}


@pytest.mark.parametrize("bits", list(PF_BITS))
@pytest.mark.parametrize("kern,cid", [("pipeline", 3), ("auto", 3), ("tile", 4), ("auto", 2)])
def test_prewait_prefetch_reads_racing_offsets(h, kern, cid, bits):
    """The kernels read row_off / nnz_off BEFORE griddepcontrol.wait for their
    L2 prefetch hints.  Here the immediately preceding kernel (the offsets
    builder, PDL-chained) writes row_off into a buffer pre-filled with huge
    garbage offsets, so the racy read may see garbage: the prefetch must stay
    inside the arrays' allocations (no fault) and the result must not depend
    on it -- bitwise O3', for every prefetch variant (debug bits 24-26) and
    both the CSR and the SparseTensor launch."""
    b = synth.config(cid, coo=True)
    dbg = PF_BITS[bits] | KERNELS[kern][0]
    h.set_hints(int(b.sizes.max()), int(b.nnz.max()))
    h.set_debug(dbg)
    h.set_tile_cb(KERNELS[kern][1])
    try:
        B = T(b.B)
        rp, col, vals, sz = T(b.row_ptr), T(b.col), T(b.vals), T(b.sizes)
        for _ in range(3):
            ro = torch.full((b.batch + 1,), (1 << 40) + 12345, dtype=torch.int64, device=DEV)
            h.build_offsets(sz, out=ro)
            C = h.csr(ro, None, rp, col, vals, B)
            no = torch.full((b.batch + 1,), -(1 << 40), dtype=torch.int64, device=DEV)
            no.copy_(T(b.nnz_off))  # a device copy, then the fused COO launch right behind it
            Cc = h.coo(ro, None, no, T(b.coo_idx), T(b.coo_vals), B, checked=True)
            torch.cuda.synchronize()
            assert np.array_equal(ro.cpu().numpy(), oracle.offsets(b.sizes))
            assert_parity(b, C.cpu().numpy(), f"csr {kern} {bits}")
            assert_parity(b, Cc.cpu().numpy(), f"coo {kern} {bits}")
    finally:
        h.set_debug(0)
        h.set_tile_cb(0)
        h.set_hints(0, 0)
