"""Seeded synthetic inputs for Batched SpMM (arXiv 1903.11409).

A module of its own: it only DRAWS inputs (graphs, A values, B values, the
COO shuffle) and lays them out in the batch-concatenated arrays the paper's
problem statement uses (stacked dense input; PAPER.md:74,
SparseTensor pairs).  It holds none of the method's arithmetic and is the only
code shared by the oracle side and the CUDA side ("Input recipe").

Configs are BASELINE.json ``configs``:

====  ===========================================  =====  ======
 id   graphs                                        k     format
====  ===========================================  =====  ======
 1    4 x G-rand(8, 3)                              16    CSR+COO
 2    100 x G-mol(20, 60)  (Tox21-shaped)           64    CSR
 3    200 x G-mix(dim U{10..300}, nnz/row U{1..5})  128   COO
 4    100 x G-rand(50, 3)  (PAPER.md:366 shape)     512   CSR
 5    65536 x G-mol(20, 60)                         256   CSR
====  ===========================================  =====  ======
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libsynth.so")

RAND, MOL, MIX = 0, 1, 2
BASE_SEED = 1903114090

CONFIGS = {
    1: dict(kind=RAND, params=(8, 3, 0, 0), batch=4, k=16, fmt="csr"),
    2: dict(kind=MOL, params=(20, 60, 0, 0), batch=100, k=64, fmt="csr"),
    3: dict(kind=MIX, params=(10, 300, 1, 5), batch=200, k=128, fmt="coo"),
    4: dict(kind=RAND, params=(50, 3, 0, 0), batch=100, k=512, fmt="csr"),
    5: dict(kind=MOL, params=(20, 60, 0, 0), batch=65536, k=256, fmt="csr"),
}
CONFIG_NAMES = {
    1: "c1: batch=4 G-rand(8,3) k=16",
    2: "c2: batch=100 G-mol(20..60) k=64",
    3: "c3: batch=200 G-mix(10..300, 1..5 nnz/row) COO k=128",
    4: "c4: batch=100 G-rand(50,3) k=512",
    5: "c5: batch=65536 G-mol(20..60) k=256",
}

_lib = None


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise ImportError(f"{_LIB_PATH} missing: run `make -C {os.path.dirname(_HERE)} synth`")
        lib = ctypes.CDLL(_LIB_PATH)
        P, I64, U64, I = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64, ctypes.c_int
        lib.synth_counts.argtypes = [I, P, U64, I64, I64, P, P]
        lib.synth_fill_csr.argtypes = [I, P, U64, I64, I64, P, P, P, P, P, I]
        lib.synth_fill_dense.argtypes = [U64, I64, I64, P, I, I64, P, I]
        lib.synth_shuffle_coo.argtypes = [U64, I64, I64, P, P, P, P, P, P, P]
        for f in (lib.synth_counts, lib.synth_fill_csr, lib.synth_fill_dense, lib.synth_shuffle_coo):
            f.restype = I
        _lib = lib
    return _lib


def _p(a: np.ndarray):
    assert a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.c_void_p)


@dataclass
class Batch:
    """One mini-batch in the batch-concatenated layout (packed, ldb = ldc = k).

    sizes[i] = n_i; row_off = exclusive prefix of sizes (int64, [batch+1]);
    row_ptr (int32, [N+1]) holds ABSOLUTE positions into col/vals; col holds
    LOCAL column ids (0 <= c < n_i); B is [N, k] fp32 row-major.
    """

    k: int
    sizes: np.ndarray
    nnz: np.ndarray
    row_off: np.ndarray
    nnz_off: np.ndarray
    row_ptr: np.ndarray
    col: np.ndarray
    vals: np.ndarray
    B: Optional[np.ndarray] = None
    coo_idx: Optional[np.ndarray] = None   # [NNZ, 2] (row, col) local, shuffled per graph
    coo_vals: Optional[np.ndarray] = None
    meta: dict = field(default_factory=dict)

    @property
    def batch(self) -> int:
        return int(self.sizes.shape[0])

    @property
    def n_rows(self) -> int:
        return int(self.row_off[-1])

    @property
    def n_nnz(self) -> int:
        return int(self.nnz_off[-1])


def _prefix(counts: np.ndarray) -> np.ndarray:
    # layout plumbing for the generated arrays (not the method's offset builder)
    out = np.zeros(counts.shape[0] + 1, dtype=np.int64)
    np.cumsum(counts, out=out[1:])
    return out


def counts(kind: int, params, seed: int, i0: int, i1: int):
    """(n_i, nnz_i) for graphs [i0, i1) without materialising them."""
    lib = _load()
    cnt = i1 - i0
    n = np.zeros(cnt, dtype=np.int32)
    z = np.zeros(cnt, dtype=np.int32)
    prm = np.asarray(params, dtype=np.int32)
    rc = lib.synth_counts(kind, _p(prm), seed, i0, i1, _p(n), _p(z))
    assert rc == 0
    return n, z


def generate(kind: int, params, batch: int, k: int, seed: int, *, i0: int = 0,
             i1: Optional[int] = None, int_valued: bool = False, dense: bool = True,
             coo: bool = False) -> Batch:
    """Graphs [i0, i1) of the (kind, params, seed) stream, laid out from row 0."""
    lib = _load()
    if i1 is None:
        i1 = batch
    prm = np.asarray(params, dtype=np.int32)
    sizes, nnz = counts(kind, params, seed, i0, i1)
    row_off, nnz_off = _prefix(sizes), _prefix(nnz)
    N, NNZ = int(row_off[-1]), int(nnz_off[-1])
    row_ptr = np.zeros(N + 1, dtype=np.int32)
    col = np.zeros(NNZ, dtype=np.int32)
    vals = np.zeros(NNZ, dtype=np.float32)
    rc = lib.synth_fill_csr(kind, _p(prm), seed, i0, i1, _p(row_off), _p(nnz_off), _p(row_ptr),
                            _p(col), _p(vals), int(int_valued))
    assert rc == 0
    b = Batch(k=k, sizes=sizes, nnz=nnz, row_off=row_off, nnz_off=nnz_off, row_ptr=row_ptr,
              col=col, vals=vals, meta=dict(kind=kind, params=tuple(params), seed=seed,
                                            i0=i0, i1=i1, int_valued=int_valued))
    if dense:
        b.B = dense_rows(seed, i0, i1, row_off, k, int_valued=int_valued)
    if coo:
        b.coo_idx, b.coo_vals = shuffle_coo(b)
    return b


def dense_rows(seed: int, i0: int, i1: int, row_off: np.ndarray, k: int, ld: Optional[int] = None,
               int_valued: bool = False, out: Optional[np.ndarray] = None) -> np.ndarray:
    lib = _load()
    ld = k if ld is None else ld
    N = int(row_off[-1])
    if out is None:
        out = np.zeros((N, ld), dtype=np.float32)
    rc = lib.synth_fill_dense(seed, i0, i1, _p(np.ascontiguousarray(row_off, dtype=np.int64)), k, ld,
                              _p(out), int(int_valued))
    assert rc == 0
    return out


def shuffle_coo(b: Batch):
    lib = _load()
    NNZ = b.n_nnz
    idx = np.zeros((NNZ, 2), dtype=np.int32)
    v = np.zeros(NNZ, dtype=np.float32)
    m = b.meta
    rc = lib.synth_shuffle_coo(m["seed"], m["i0"], m["i1"], _p(b.row_off), _p(b.nnz_off), _p(b.row_ptr),
                               _p(b.col), _p(b.vals), _p(idx), _p(v))
    assert rc == 0
    return idx, v


def config(cid: int, *, i0: int = 0, i1: Optional[int] = None, int_valued: bool = False,
           dense: bool = True, coo: Optional[bool] = None, seed: Optional[int] = None,
           k: Optional[int] = None) -> Batch:
    """BASELINE.json config ``cid`` (1..5), graphs [i0, i1)."""
    c = CONFIGS[cid]
    seed = BASE_SEED + cid if seed is None else seed
    if coo is None:
        coo = c["fmt"] == "coo" or cid == 1
    b = generate(c["kind"], c["params"], c["batch"], c["k"] if k is None else k, seed, i0=i0, i1=i1,
                 int_valued=int_valued, dense=dense, coo=coo)
    b.meta["config"] = cid
    return b


def random_batch(rng: np.random.Generator, batch: int, k: int, *, nmax: int = 12, dmax: int = 4,
                 int_valued: bool = False, empty_rows: bool = True, allow_empty_graphs: bool = True,
                 duplicates: bool = False, sizes: Optional[np.ndarray] = None) -> Batch:
    """Small adversarial batches for tests (numpy Generator, seeded by the caller):
    empty graphs, empty rows, unsorted rows and (optionally) duplicate entries.
    ``sizes`` fixes n_i (length ``batch``) instead of drawing them."""
    if sizes is None:
        sizes = rng.integers(0 if allow_empty_graphs else 1, nmax + 1, size=batch).astype(np.int32)
    else:
        sizes = np.ascontiguousarray(sizes, dtype=np.int32)
        assert sizes.shape == (batch,)
    rows_cols, per_graph_nnz = [], []
    for n in sizes:
        cols_g = []
        for _ in range(n):
            lo = 0 if empty_rows else 1
            d = int(rng.integers(lo, min(dmax, n) + 1))
            cs = list(rng.choice(n, size=d, replace=False)) if d else []
            if duplicates and d and rng.random() < 0.3:
                cs.append(cs[0])
            rng.shuffle(cs)
            cols_g.append([int(c) for c in cs])
        rows_cols.append(cols_g)
        per_graph_nnz.append(sum(len(r) for r in cols_g))
    nnz = np.asarray(per_graph_nnz, dtype=np.int32)
    row_off, nnz_off = _prefix(sizes), _prefix(nnz)
    N, NNZ = int(row_off[-1]), int(nnz_off[-1])
    row_ptr = np.zeros(N + 1, dtype=np.int32)
    col = np.zeros(NNZ, dtype=np.int32)
    e, g = 0, 0
    for cols_g in rows_cols:
        for r in cols_g:
            row_ptr[g] = e
            col[e:e + len(r)] = r
            e += len(r)
            g += 1
    row_ptr[N] = e
    if int_valued:
        vals = rng.integers(1, 3, size=NNZ).astype(np.float32)
        B = rng.integers(-8, 9, size=(N, k)).astype(np.float32)
    else:
        vals = (rng.integers(-(1 << 23), 1 << 23, size=NNZ) / float(1 << 23)).astype(np.float32)
        B = (rng.integers(-(1 << 23), 1 << 23, size=(N, k)) / float(1 << 23)).astype(np.float32)
    b = Batch(k=k, sizes=sizes, nnz=nnz, row_off=row_off, nnz_off=nnz_off, row_ptr=row_ptr, col=col,
              vals=vals, B=B, meta=dict(kind=-1))
    # COO view: per-graph shuffle of the CSR entries (rows recovered from row_ptr)
    idx = np.zeros((NNZ, 2), dtype=np.int32)
    cv = np.zeros(NNZ, dtype=np.float32)
    for i in range(batch):
        z0, z1 = int(nnz_off[i]), int(nnz_off[i + 1])
        rows = np.zeros(z1 - z0, dtype=np.int32)
        for r in range(int(sizes[i])):
            g = int(row_off[i]) + r
            rows[row_ptr[g] - z0:row_ptr[g + 1] - z0] = r
        perm = rng.permutation(z1 - z0)
        idx[z0:z1, 0] = rows[perm]
        idx[z0:z1, 1] = col[z0:z1][perm]
        cv[z0:z1] = vals[z0:z1][perm]
    b.coo_idx, b.coo_vals = idx, cv
    return b
