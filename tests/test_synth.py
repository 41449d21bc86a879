"""The seeded input generator (synth/): shapes and structure of the paper's
workloads, determinism, range regeneration."""
import numpy as np

import synth


def rows_of(b, i):
    g0 = int(b.row_off[i])
    return [b.col[b.row_ptr[g0 + r]:b.row_ptr[g0 + r + 1]] for r in range(int(b.sizes[i]))]


def test_grand_exact_nnz_per_row_distinct_sorted():
    for cid, (dim, d) in ((1, (8, 3)), (4, (50, 3))):
        b = synth.config(cid, dense=False, coo=False)
        assert np.all(b.sizes == dim)
        assert np.all(np.diff(b.row_ptr) == d)         # exactly d per row
        for i in range(b.batch):
            for r in rows_of(b, i):
                assert np.all(np.diff(r) > 0) and r.min() >= 0 and r.max() < dim


def test_gmix_ranges():
    b = synth.config(3, dense=False, coo=False)
    assert b.sizes.min() >= 10 and b.sizes.max() <= 300
    for i in range(b.batch):
        d = np.diff(b.row_ptr[b.row_off[i]:b.row_off[i + 1] + 1])
        assert np.all(d == d[0]) and 1 <= d[0] <= 5


def test_gmol_symmetric_self_loops_valence():
    b = synth.config(2, dense=False, coo=False)
    assert b.sizes.min() >= 20 and b.sizes.max() <= 60
    for i in range(b.batch):
        n = int(b.sizes[i])
        A = np.zeros((n, n), dtype=bool)
        for r, cols in enumerate(rows_of(b, i)):
            A[r, cols] = True
            assert 2 <= len(cols) <= 5                      # self-loop + 1..4 neighbours
        assert np.array_equal(A, A.T) and np.all(np.diag(A))
        # connected: the spanning tree reaches every node
        seen, stack = {0}, [0]
        while stack:
            u = stack.pop()
            for v in np.nonzero(A[u])[0]:
                if v not in seen:
                    seen.add(int(v)); stack.append(int(v))
        assert len(seen) == n
    mean = b.n_nnz / b.n_rows
    assert 2.9 < mean < 3.4                                 # ~3.2 nnz/row


def test_values_grid_and_int_variant():
    b = synth.config(2)
    for x in (b.vals, b.B.ravel()):
        assert x.min() >= -1 and x.max() < 1
        assert np.all(x * 8388608 == np.round(x * 8388608))
    bi = synth.config(2, int_valued=True)
    assert set(np.unique(bi.vals)) <= {1.0, 2.0}
    assert bi.B.min() >= -8 and bi.B.max() <= 8 and np.all(bi.B == np.round(bi.B))


def test_determinism_and_range_regeneration():
    a = synth.config(2)
    b = synth.config(2)
    assert np.array_equal(a.row_ptr, b.row_ptr) and np.array_equal(a.B, b.B)
    part = synth.config(2, i0=37, i1=81)
    g0, g1 = int(a.row_off[37]), int(a.row_off[81])
    z0 = int(a.row_ptr[g0])
    assert np.array_equal(part.sizes, a.sizes[37:81])
    assert np.array_equal(part.row_ptr, a.row_ptr[g0:g1 + 1] - z0)
    assert np.array_equal(part.col, a.col[z0:a.row_ptr[g1]])
    assert np.array_equal(part.B, a.B[g0:g1])
    other = synth.config(2, seed=12345)
    assert not np.array_equal(other.row_ptr[:50], a.row_ptr[:50]) or not np.array_equal(other.B[:5], a.B[:5])


def test_coo_is_per_graph_permutation():
    b = synth.config(3, dense=False, coo=True)
    for i in range(0, b.batch, 13):
        z0, z1 = int(b.nnz_off[i]), int(b.nnz_off[i + 1])
        rows = np.repeat(np.arange(b.sizes[i]), np.diff(b.row_ptr[b.row_off[i]:b.row_off[i + 1] + 1]))
        csr = sorted(zip(rows.tolist(), b.col[z0:z1].tolist(), b.vals[z0:z1].tolist()))
        coo = sorted(zip(b.coo_idx[z0:z1, 0].tolist(), b.coo_idx[z0:z1, 1].tolist(), b.coo_vals[z0:z1].tolist()))
        assert csr == coo
        assert z1 - z0 < 3 or not np.array_equal(b.coo_idx[z0:z1, 0], rows)   # actually shuffled


def test_c5_shape_counts_only():
    n, z = synth.counts(synth.MOL, (20, 60, 0, 0), synth.BASE_SEED + 5, 0, 65536)
    assert n.shape == (65536,) and n.min() >= 20 and n.max() <= 60
    assert 2.5e6 < n.sum() < 2.75e6 and 7.8e6 < z.sum() < 8.6e6
