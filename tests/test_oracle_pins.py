"""Pins for the CPU oracle (oracle/): checks it against what the paper and the
mathematics fix, never against itself (DESIGN.md §Oracle pins).

Pins used:
* dense brute force: numpy fp64 ``A_dense @ B`` (a library routine) on >=1000
  tiny random batches with duplicates, empty rows and empty graphs;
* closed forms: identity -> C == B, zero matrix -> 0, integer-valued inputs
  exact in any order, the bound equals 1e-5 * (|A| @ |B|);
* worked examples (tests/golden/spec_examples.json, each cited);
* invariants: linearity in B, batched == per-matrix, COO permutation
  invariance, brute-force ``sorted()`` of (row, col, pos), CSR round trip;
* partition: hand-evaluated examples, contiguity/coverage/balance bound, the
  equal-cost closed form.
"""
import numpy as np
import pytest

import oracle
import synth


def dense_blocks(b, vals=None, col=None, row_ptr=None):
    """Per-matrix dense A_i (duplicates summed, as PAPER.md:101 accumulates)."""
    vals = b.vals if vals is None else vals
    col = b.col if col is None else col
    row_ptr = b.row_ptr if row_ptr is None else row_ptr
    out = []
    for i in range(b.batch):
        n = int(b.sizes[i])
        A = np.zeros((n, n), dtype=np.float64)
        g0 = int(b.row_off[i])
        for r in range(n):
            for e in range(row_ptr[g0 + r], row_ptr[g0 + r + 1]):
                A[r, col[e]] += float(vals[e])
        out.append(A)
    return out


def brute_force(b):
    """C64 = blockdiag(A_i) @ B via numpy matmul, and the |A|@|B| bound."""
    C = np.zeros((b.n_rows, b.k), dtype=np.float64)
    S = np.zeros((b.n_rows, b.k), dtype=np.float64)
    for i, A in enumerate(dense_blocks(b)):
        g0, g1 = int(b.row_off[i]), int(b.row_off[i + 1])
        Bi = b.B[g0:g1].astype(np.float64)
        C[g0:g1] = A @ Bi
    # |A| summed per stored entry: duplicates enter the bound separately
    for i in range(b.batch):
        g0 = int(b.row_off[i])
        for r in range(int(b.sizes[i])):
            for e in range(b.row_ptr[g0 + r], b.row_ptr[g0 + r + 1]):
                S[g0 + r] += abs(float(b.vals[e])) * np.abs(b.B[g0 + b.col[e]].astype(np.float64))
    return C, 1e-5 * S


def run_oracle(b, **kw):
    return oracle.spmm(b.k, b.row_off, None, b.row_ptr, b.col, b.vals, b.B, **kw)


# ---------------------------------------------------------------- O3 / O3'

def test_dense_brute_force_1000_batches():
    rng = np.random.default_rng(20190327)
    for trial in range(1000):
        k = int(rng.integers(1, 17))
        b = synth.random_batch(rng, int(rng.integers(0, 5)), k, nmax=10, dmax=4,
                               duplicates=bool(trial % 3 == 0))
        C, bound, C64 = run_oracle(b, want_f64=True)
        ref, ref_bound = brute_force(b)
        # fp64 sums in a different order: equal to ~1e-15 relative of sum|a||b|
        assert np.all(np.abs(C64 - ref) <= 1e-12 * (ref_bound / 1e-5) + 0.0), trial
        assert np.array_equal(C, C64.astype(np.float32)), trial        # one rounding
        assert np.allclose(bound, ref_bound, rtol=1e-12, atol=0), trial
        # fp32-ordered variant stays within the fp32 FMA error bound
        C32 = oracle.spmm_f32(b.k, b.row_off, None, b.row_ptr, b.col, b.vals, b.B)
        m = np.diff(b.row_ptr).max() if b.n_rows else 0
        gamma = (m + 1) * 2.0 ** -24
        assert np.all(np.abs(C32.astype(np.float64) - ref) <= gamma * ref_bound / 1e-5 + 1e-300), trial


def test_transpose_is_caught():
    # a non-symmetric A: C must equal A @ B, not A^T @ B
    rng = np.random.default_rng(7)
    b = synth.random_batch(rng, 3, 5, nmax=8, dmax=3, allow_empty_graphs=False)
    C, _ = run_oracle(b)
    for i, A in enumerate(dense_blocks(b)):
        g0, g1 = int(b.row_off[i]), int(b.row_off[i + 1])
        Bi = b.B[g0:g1].astype(np.float64)
        assert np.allclose(C[g0:g1], A @ Bi, rtol=1e-6, atol=1e-6)
        if not np.allclose(A, A.T):
            assert not np.allclose(C[g0:g1], A.T @ Bi, rtol=1e-6, atol=1e-6)


def test_golden_spmm(golden):
    for ex in golden["spmm"]:
        n, k = ex["n"], ex["k"]
        ent = sorted((r, c, v) for r, c, v in ex["entries"])
        rp = np.zeros(n + 1, dtype=np.int32)
        for r, _, _ in ent:
            rp[r + 1] += 1
        rp = np.cumsum(rp).astype(np.int32)
        col = np.array([c for _, c, _ in ent], dtype=np.int32)
        vals = np.array([v for _, _, v in ent], dtype=np.float32)
        B = np.array(ex["B"], dtype=np.float32).reshape(n, k)
        ro = np.array([0, n], dtype=np.int64)
        C, _ = oracle.spmm(k, ro, None, rp, col, vals, B)
        C32 = oracle.spmm_f32(k, ro, None, rp, col, vals, B)
        want = np.array(ex["C"], dtype=np.float32)
        assert np.array_equal(C, want), ex["cite"]
        assert np.array_equal(C32, want), ex["cite"]


def test_golden_fmaf_storage_order(golden):
    """O3' is fmaf in storage order, not multiply-then-add: the worked example
    separates the two (one rounding per FMA gives 2^-24, a rounded product
    gives 0).  O3 (fp64) is exactly 2^-24 as well."""
    for ex in golden["spmm_f32"]:
        n, k = ex["n"], ex["k"]
        ent = ex["entries"]                            # already in storage order (row 0: cols 0, 1)
        rp = np.zeros(n + 1, dtype=np.int32)
        for r, _, _ in ent:
            rp[r + 1] += 1
        rp = np.cumsum(rp).astype(np.int32)
        col = np.array([c for _, c, _ in ent], dtype=np.int32)
        vals = np.array([v for _, _, v in ent], dtype=np.float32)
        B = np.array(ex["B"], dtype=np.float32).reshape(n, k)
        ro = np.array([0, n], dtype=np.int64)
        C32 = oracle.spmm_f32(k, ro, None, rp, col, vals, B)
        C, _ = oracle.spmm(k, ro, None, rp, col, vals, B)
        assert np.array_equal(C32, np.array(ex["C_f32"], dtype=np.float32)), ex["cite"]
        assert np.array_equal(C, np.array(ex["C_f64"], dtype=np.float32)), ex["cite"]
        # the alternative the pin rules out, evaluated in numpy fp32 (product rounded, then added)
        mta = np.float32(np.float32(vals[0] * B[0, 0]) + np.float32(vals[1] * B[1, 0]))
        assert mta == np.float32(ex["C_mul_then_add"][0][0]) and mta != C32[0, 0]


def test_identity_gives_B():
    rng = np.random.default_rng(1)
    sizes = np.array([5, 0, 1, 17, 3], dtype=np.int32)
    ro = oracle.offsets(sizes)
    N = int(ro[-1])
    rp = np.arange(N + 1, dtype=np.int32)
    col = np.concatenate([np.arange(n, dtype=np.int32) for n in sizes])
    vals = np.ones(N, dtype=np.float32)
    for k in (1, 3, 4, 33):
        B = rng.standard_normal((N, k)).astype(np.float32)
        C, _ = oracle.spmm(k, ro, None, rp, col, vals, B)
        assert np.array_equal(C, B)
        assert np.array_equal(oracle.spmm_f32(k, ro, None, rp, col, vals, B), B)


def test_zero_rows_and_empty_graphs_are_exact_zero():
    rng = np.random.default_rng(2)
    for _ in range(50):
        b = synth.random_batch(rng, 6, 7, nmax=6, dmax=3, empty_rows=True)
        C, bound = run_oracle(b)
        empty = np.diff(b.row_ptr) == 0
        assert np.all(C[empty] == 0) and np.all(bound[empty] == 0)


def test_linearity_in_B():
    rng = np.random.default_rng(3)
    for _ in range(100):
        b = synth.random_batch(rng, 4, 6, nmax=9)
        B1 = b.B.copy()
        B2 = (rng.integers(-(1 << 23), 1 << 23, size=b.B.shape) / float(1 << 23)).astype(np.float32)
        _, _, C1 = oracle.spmm(b.k, b.row_off, None, b.row_ptr, b.col, b.vals, B1, want_f64=True)
        _, _, C2 = oracle.spmm(b.k, b.row_off, None, b.row_ptr, b.col, b.vals, B2, want_f64=True)
        # B1 + B2 is exact in fp32 here (both on the 2^-23 grid, |x| < 1)
        _, _, C12 = oracle.spmm(b.k, b.row_off, None, b.row_ptr, b.col, b.vals, B1 + B2, want_f64=True)
        _, bnd = oracle.spmm(b.k, b.row_off, None, b.row_ptr, b.col, b.vals, np.abs(B1) + np.abs(B2))
        assert np.all(np.abs(C12 - (C1 + C2)) <= 1e-10 * bnd + 1e-300)


def test_integer_valued_exact_in_any_order():
    rng = np.random.default_rng(4)
    for _ in range(200):
        b = synth.random_batch(rng, 5, 9, nmax=12, dmax=5, int_valued=True, duplicates=True)
        C, _ = run_oracle(b)
        C32 = oracle.spmm_f32(b.k, b.row_off, None, b.row_ptr, b.col, b.vals, b.B)
        ref, _ = brute_force(b)
        assert np.array_equal(C.astype(np.float64), ref)
        assert np.array_equal(C32, C)


def test_batched_equals_per_matrix():
    b = synth.config(2, dense=True)
    C, bound = run_oracle(b)
    for i in range(0, b.batch, 7):
        g0, g1 = int(b.row_off[i]), int(b.row_off[i + 1])
        z0 = int(b.row_ptr[g0])
        ro = np.array([0, g1 - g0], dtype=np.int64)
        Ci, bi = oracle.spmm(b.k, ro, None, b.row_ptr[g0:g1 + 1] - z0, b.col[z0:b.row_ptr[g1]],
                             b.vals[z0:b.row_ptr[g1]], b.B[g0:g1])
        assert np.array_equal(Ci, C[g0:g1]) and np.array_equal(bi, bound[g0:g1])


def test_sampled_rows_match_full():
    b = synth.config(3)
    C, bound = run_oracle(b)
    rng = np.random.default_rng(5)
    mat = rng.integers(0, b.batch, size=300)
    rloc = np.array([rng.integers(0, b.sizes[i]) for i in mat], dtype=np.int32)
    out, bnd = oracle.spmm_rows(mat, rloc, b.k, b.row_off, b.row_ptr, b.col, b.vals, b.B)
    g = b.row_off[mat] + rloc
    assert np.array_equal(out, C[g]) and np.array_equal(bnd, bound[g])


def test_padded_layout_and_ld():
    """row_off with gaps + explicit sizes, ldb/ldc > k: only matrix rows are defined."""
    rng = np.random.default_rng(6)
    b = synth.random_batch(rng, 4, 5, nmax=6, allow_empty_graphs=False)
    gap = 3
    ro = np.array([int(b.row_off[i]) + gap * i for i in range(b.batch + 1)], dtype=np.int64)
    Np = int(ro[-1])
    rp = np.zeros(Np + 1, dtype=np.int32)
    Bp = np.zeros((Np, 8), dtype=np.float32)
    for i in range(b.batch):
        for r in range(int(b.sizes[i]) + 1):
            rp[ro[i] + r] = b.row_ptr[b.row_off[i] + r]
        for gg in range(int(ro[i] + b.sizes[i]), int(ro[i + 1])):
            rp[gg] = b.row_ptr[b.row_off[i + 1]]
        Bp[ro[i]:ro[i] + b.sizes[i], :5] = b.B[b.row_off[i]:b.row_off[i + 1]]
    rp[Np] = b.row_ptr[-1]
    C, _ = oracle.spmm(5, ro, b.sizes, rp, b.col, b.vals, Bp, ldb=8, ldc=8)
    Cref, _ = run_oracle(b)
    for i in range(b.batch):
        assert np.array_equal(C[ro[i]:ro[i] + b.sizes[i], :5], Cref[b.row_off[i]:b.row_off[i + 1]])


# ---------------------------------------------------------------- O1

def test_offsets():
    assert list(oracle.offsets([])) == [0]
    assert list(oracle.offsets(np.full(10, 7))) == [7 * i for i in range(11)]   # closed form
    rng = np.random.default_rng(8)
    s = rng.integers(0, 1 << 20, size=5000)
    o = oracle.offsets(s)
    assert o.dtype == np.int64 and o[0] == 0
    assert np.array_equal(np.diff(o), s)                        # inverse of a difference
    big = np.full(3000, (1 << 31) - 1)                          # int64, no int32 wrap
    assert oracle.offsets(big)[-1] == 3000 * ((1 << 31) - 1)


# ---------------------------------------------------------------- O2

def _coo_brute(b, idx, vals):
    """sorted() of (row, col, pos) per matrix -> CSR."""
    rp = np.zeros(b.n_rows + 1, dtype=np.int32)
    col = np.zeros(b.n_nnz, dtype=np.int32)
    v = np.zeros(b.n_nnz, dtype=np.float32)
    for i in range(b.batch):
        z0, z1 = int(b.nnz_off[i]), int(b.nnz_off[i + 1])
        trip = sorted((int(idx[e, 0]), int(idx[e, 1]), e - z0) for e in range(z0, z1))
        for q, (r, c, p) in enumerate(trip):
            col[z0 + q] = c
            v[z0 + q] = vals[z0 + p]
        for r in range(int(b.sizes[i]) + 1):
            rp[b.row_off[i] + r] = z0 + sum(1 for t in trip if t[0] < r)
    return rp, col, v


def test_coo2csr_brute_force_sorted():
    rng = np.random.default_rng(9)
    for trial in range(300):
        b = synth.random_batch(rng, int(rng.integers(0, 6)), 2, nmax=9, dmax=4,
                               duplicates=bool(trial % 2))
        rp, col, v = oracle.coo2csr(b.row_off, None, b.nnz_off, b.coo_idx, b.coo_vals)
        rp2, col2, v2 = _coo_brute(b, b.coo_idx, b.coo_vals)
        assert np.array_equal(rp, rp2) and np.array_equal(col, col2)
        assert np.array_equal(v.view(np.uint32), v2.view(np.uint32))


def test_coo2csr_golden(golden):
    for ex in golden["coo2csr"]:
        n = ex["n"]
        idx = np.array(ex["idx"], dtype=np.int32).reshape(-1, 2)
        vals = np.array(ex["vals"], dtype=np.float32)
        rp, col, v = oracle.coo2csr([0, n], None, [0, len(vals)], idx, vals)
        assert list(rp) == ex["row_ptr"], ex["cite"]
        assert list(col) == ex["col"], ex["cite"]
        assert list(v) == ex["out_vals"], ex["cite"]


def test_coo2csr_round_trip_and_permutation_invariance():
    # canonical CSR (generator output, sorted cols, no duplicates) -> shuffled COO -> CSR == identity
    for cid in (1, 2, 3):
        b = synth.config(cid, coo=True, dense=False)
        rp, col, v = oracle.coo2csr(b.row_off, None, b.nnz_off, b.coo_idx, b.coo_vals)
        assert np.array_equal(rp, b.row_ptr)
        assert np.array_equal(col, b.col)
        assert np.array_equal(v.view(np.uint32), b.vals.view(np.uint32))


def test_coo2csr_rejects_out_of_range():
    with pytest.raises(ValueError):
        oracle.coo2csr([0, 2], None, [0, 1], np.array([[2, 0]], dtype=np.int32), np.ones(1, np.float32))


# ---------------------------------------------------------------- O4

def test_partition_golden(golden):
    for ex in golden["partition"]:
        nnz_off = np.concatenate([[0], np.cumsum(ex["nnz"])]).astype(np.int64)
        assert list(oracle.partition(nnz_off, ex["k"], ex["parts"])) == ex["split"], ex["cite"]


def test_partition_invariants():
    rng = np.random.default_rng(10)
    for _ in range(500):
        batch = int(rng.integers(0, 40))
        nnz = rng.integers(0, 50, size=batch)
        k = int(rng.integers(1, 600))
        G = int(rng.integers(1, 9))
        nnz_off = np.concatenate([[0], np.cumsum(nnz)]).astype(np.int64)
        s = oracle.partition(nnz_off, k, G)
        assert s[0] == 0 and s[-1] == batch and np.all(np.diff(s) >= 0)
        cost = nnz.astype(np.int64) * k
        T = int(cost.sum())
        if T:
            cmax = int(cost.max())
            for r in range(G):
                shard = int(cost[s[r]:s[r + 1]].sum())
                assert shard * G <= T + G * cmax      # <= T/G + max c_i
            # minimality: moving any interior split one graph left breaks P_j*G >= r*T
            P = np.concatenate([[0], np.cumsum(cost)])
            for r in range(1, G):
                j = int(s[r])
                assert P[j] * G >= r * T
                assert j == 0 or P[j - 1] * G < r * T


def test_partition_equal_cost_closed_form():
    for batch, G in ((64, 8), (65536, 8), (100, 4), (12, 3)):
        nnz_off = np.arange(batch + 1, dtype=np.int64) * 5
        assert list(oracle.partition(nnz_off, 256, G)) == [r * batch // G for r in range(G + 1)]


# ---------------------------------------------------------------- O5 / O6 (backward, NEXT-2)

def test_transpose_dense_and_involution():
    rng = np.random.default_rng(12)
    for trial in range(200):
        b = synth.random_batch(rng, int(rng.integers(0, 5)), 1, nmax=9, dmax=4, duplicates=bool(trial % 2))
        rt, ct, vt = oracle.csr_transpose(b.row_off, None, b.row_ptr, b.col, b.vals)
        At = dense_blocks(b, vals=vt, col=ct, row_ptr=rt)
        for A, T_ in zip(dense_blocks(b), At):
            assert np.array_equal(A.T, T_)
        # canonical order: columns non-decreasing within every transposed row
        for g in range(b.n_rows):
            assert np.all(np.diff(ct[rt[g]:rt[g + 1]]) >= 0)
    # (A^T)^T == A exactly on canonical input (sorted rows, no duplicates)
    b = synth.config(3, coo=False)
    rt, ct, vt = oracle.csr_transpose(b.row_off, None, b.row_ptr, b.col, b.vals)
    r2, c2, v2 = oracle.csr_transpose(b.row_off, None, rt, ct, vt)
    assert np.array_equal(r2, b.row_ptr) and np.array_equal(c2, b.col)
    assert np.array_equal(v2.view(np.uint32), b.vals.view(np.uint32))


def test_sddmm_dense_brute_force():
    rng = np.random.default_rng(13)
    for trial in range(300):
        k = int(rng.integers(1, 12))
        b = synth.random_batch(rng, int(rng.integers(0, 5)), k, nmax=9, dmax=4, duplicates=bool(trial % 2))
        G = (rng.integers(-(1 << 23), 1 << 23, size=b.B.shape) / float(1 << 23)).astype(np.float32)
        out, bound = oracle.sddmm(k, b.row_off, None, b.row_ptr, b.col, b.B, G)
        for i in range(b.batch):
            g0, g1 = int(b.row_off[i]), int(b.row_off[i + 1])
            M = G[g0:g1].astype(np.float64) @ b.B[g0:g1].astype(np.float64).T      # library matmul
            for r in range(g1 - g0):
                for e in range(b.row_ptr[g0 + r], b.row_ptr[g0 + r + 1]):
                    ref = M[r, b.col[e]]
                    assert abs(float(out[e]) - ref) <= 1e-6 * (bound[e] / 1e-5) + abs(ref) * 2 ** -23


def test_backward_finite_differences():
    """L(B, vals) = sum(C * G): dL/dB = A^T G and dL/dvals = SDDMM(G, B) (central differences, fp64)."""
    rng = np.random.default_rng(14)
    b = synth.random_batch(rng, 3, 3, nmax=5, dmax=2, allow_empty_graphs=False, duplicates=True)
    G = rng.standard_normal(b.B.shape)
    gB, _, gv, _ = oracle.backward(b.k, b.row_off, b.row_ptr, b.col, b.vals, b.B, G.astype(np.float32))

    def L(Bm, vals):
        tot = 0.0
        for i in range(b.batch):
            g0, g1 = int(b.row_off[i]), int(b.row_off[i + 1])
            A = np.zeros((g1 - g0, g1 - g0))
            for r in range(g1 - g0):
                for e in range(b.row_ptr[g0 + r], b.row_ptr[g0 + r + 1]):
                    A[r, b.col[e]] += vals[e]
            tot += float(np.sum((A @ Bm[g0:g1]) * G[g0:g1]))
        return tot

    h = 1e-3
    B64, v64 = b.B.astype(np.float64), b.vals.astype(np.float64)
    for idx in np.ndindex(*B64.shape):
        Bp, Bm = B64.copy(), B64.copy()
        Bp[idx] += h
        Bm[idx] -= h
        fd = (L(Bp, v64) - L(Bm, v64)) / (2 * h)
        assert abs(fd - gB[idx]) < 1e-4 * (1 + abs(fd))
    for e in range(v64.shape[0]):
        vp, vm = v64.copy(), v64.copy()
        vp[e] += h
        vm[e] -= h
        fd = (L(B64, vp) - L(B64, vm)) / (2 * h)
        assert abs(fd - gv[e]) < 1e-4 * (1 + abs(fd))


def test_backward_golden(golden):
    for ex in golden["backward"]:
        n, k = ex["n"], ex["k"]
        ent = sorted((r, c, v) for r, c, v in ex["entries"])
        rp = np.zeros(n + 1, dtype=np.int32)
        for r, _, _ in ent:
            rp[r + 1] += 1
        rp = np.cumsum(rp).astype(np.int32)
        col = np.array([c for _, c, _ in ent], dtype=np.int32)
        vals = np.array([v for _, _, v in ent], dtype=np.float32)
        B = np.array(ex["B"], dtype=np.float32)
        G = np.array(ex["grad_C"], dtype=np.float32)
        gB, _, gv, _ = oracle.backward(k, [0, n], rp, col, vals, B, G)
        assert np.array_equal(gB, np.array(ex["grad_B"], dtype=np.float32)), ex["cite"]
        assert list(gv) == ex["grad_vals"], ex["cite"]
    # zero upstream gradient -> zero gradients
    b = synth.config(1)
    gB, _, gv, _ = oracle.backward(b.k, b.row_off, b.row_ptr, b.col, b.vals, b.B, np.zeros_like(b.B))
    assert not gB.any() and not gv.any()


# ---------------------------------------------------------------- O7 (fused GCN layer, NEXT-1)

def gcn_inputs(rng, channels=2, n_x=5, k=4, batch=3):
    """Per-channel adjacency patterns over the same graphs (bond-type channels)."""
    base = synth.random_batch(rng, batch, k, nmax=7, dmax=3, allow_empty_graphs=False)
    N = base.n_rows
    rps, cols, vals = [], [], []
    z = 0
    for ch in range(channels):
        rp = np.zeros(N + 1, np.int32)
        cl, vl = [], []
        for i in range(batch):
            n = int(base.sizes[i])
            for r in range(n):
                g = int(base.row_off[i]) + r
                rp[g] = z
                d = int(rng.integers(0, min(3, n) + 1))
                cs = sorted(rng.choice(n, size=d, replace=False).tolist())
                cl += cs
                vl += list(rng.standard_normal(d))
                z += d
        rp[N] = z
        rps.append(rp)
        cols += cl
        vals += vl
    X = rng.standard_normal((N, n_x)).astype(np.float32)
    W = rng.standard_normal((channels, n_x, k)).astype(np.float32)
    bias = rng.standard_normal((channels, k)).astype(np.float32)
    return base, np.stack(rps), np.array(cols, np.int32), np.array(vals, np.float32), X, W, bias


def test_gcn_layer_dense_brute_force():
    rng = np.random.default_rng(15)
    for trial in range(40):
        base, rps, col, vals, X, W, bias = gcn_inputs(rng, channels=int(rng.integers(1, 4)))
        Y, mag = oracle.gcn_layer(base.row_off, rps, col, vals, X, W, bias)
        ref = np.zeros_like(Y, dtype=np.float64)
        for ch in range(rps.shape[0]):
            U = X.astype(np.float64) @ W[ch].astype(np.float64) + bias[ch].astype(np.float64)   # library matmul
            for i in range(base.batch):
                g0, g1 = int(base.row_off[i]), int(base.row_off[i + 1])
                A = np.zeros((g1 - g0, g1 - g0))
                for r in range(g1 - g0):
                    for e in range(rps[ch][g0 + r], rps[ch][g0 + r + 1]):
                        A[r, col[e]] += vals[e]
                ref[g0:g1] += A @ U[g0:g1]
        assert np.all(np.abs(Y - ref) <= 1e-6 * mag + 1e-30), trial


def test_gcn_layer_special_cases():
    rng = np.random.default_rng(16)
    base, rps, col, vals, X, W, bias = gcn_inputs(rng, channels=1, n_x=4, k=4)
    # W = I, bias = 0: the layer is the plain SpMM of A with X (closed form)
    Y, _ = oracle.gcn_layer(base.row_off, rps, col, vals, X, np.eye(4, dtype=np.float32)[None], np.zeros((1, 4), np.float32))
    C, _ = oracle.spmm(4, base.row_off, None, rps[0], col, vals, X)
    assert np.array_equal(Y, C)
    # W = 0: Y = rowsum(A) (x) bias
    Y, _ = oracle.gcn_layer(base.row_off, rps, col, vals, X, np.zeros((1, 4, 4), np.float32), bias[:1])
    rs = np.array([vals[rps[0][g]:rps[0][g + 1]].astype(np.float64).sum() for g in range(base.n_rows)])
    assert np.allclose(Y, rs[:, None] * bias[0][None, :].astype(np.float64), rtol=1e-6, atol=1e-6)
