"""TEST INFRASTRUCTURE ONLY — the CPU oracle for Batched SpMM (arXiv 1903.11409).

Thin ctypes wrapper over ``oracle/liboracle.so`` (plain C, fp64, see
oracle.c's header for the passage each function follows).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  It shares no code with
``paper_1903_11409_b200`` and never imports it.

``check_bound`` is the north_star acceptance rule, written out:
|C - C_ref| <= 1e-5 * sum_j |a_ij| |b_jc| per element, evaluated in fp64.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise ImportError(f"{_LIB_PATH} missing: run `make -C {os.path.dirname(_HERE)} oracle`")
        lib = ctypes.CDLL(_LIB_PATH)
        P, I64, I32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32
        lib.oracle_offsets.argtypes = [I64, P, P]
        lib.oracle_coo2csr.argtypes = [I64, P, P, P, P, P, P, P, P]
        lib.oracle_spmm.argtypes = [I64, I32, P, P, P, P, P, P, I64, P, I64, P, P]
        lib.oracle_spmm_f32.argtypes = [I64, I32, P, P, P, P, P, P, I64, P, I64]
        lib.oracle_spmm_rows.argtypes = [I64, P, P, I32, P, P, P, P, P, I64, P, P]
        lib.oracle_partition.argtypes = [I64, P, I32, I32, P]
        lib.oracle_csr_transpose.argtypes = [I64, P, P, P, P, P, P, P, P]
        lib.oracle_sddmm.argtypes = [I64, I32, P, P, P, P, P, I64, P, I64, P, P]
        lib.oracle_gcn_layer.argtypes = [I64, I32, I32, I32, P, P, P, P, P, I64, P, P, P, I64, P]
        for f in (lib.oracle_offsets, lib.oracle_coo2csr, lib.oracle_spmm, lib.oracle_spmm_f32,
                  lib.oracle_spmm_rows, lib.oracle_partition, lib.oracle_csr_transpose, lib.oracle_sddmm, lib.oracle_gcn_layer):
            f.restype = ctypes.c_int
        _lib = lib
    return _lib


def _p(a: Optional[np.ndarray]):
    if a is None:
        return None
    assert a.flags.c_contiguous, "oracle arrays must be C-contiguous"
    return a.ctypes.data_as(ctypes.c_void_p)


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def offsets(sizes) -> np.ndarray:
    """O1: int64 exclusive prefix sum, [batch+1]."""
    s = _c(sizes, np.int32)
    out = np.zeros(s.shape[0] + 1, dtype=np.int64)
    assert _load().oracle_offsets(s.shape[0], _p(s), _p(out)) == 0
    return out


def coo2csr(row_off, sizes, nnz_off, idx, vals, n_rows: Optional[int] = None):
    """O2: canonical (row, col, original position) CSR. Returns (row_ptr, col, vals)."""
    row_off = _c(row_off, np.int64)
    nnz_off = _c(nnz_off, np.int64)
    idx = _c(idx, np.int32).reshape(-1)
    vals = _c(vals, np.float32)
    batch = row_off.shape[0] - 1
    sz = None if sizes is None else _c(sizes, np.int32)
    N = int(row_off[-1]) if n_rows is None else n_rows
    NNZ = int(nnz_off[-1])
    rp = np.zeros(N + 1, dtype=np.int32)
    col = np.zeros(NNZ, dtype=np.int32)
    v = np.zeros(NNZ, dtype=np.float32)
    rc = _load().oracle_coo2csr(batch, _p(row_off), _p(sz), _p(nnz_off), _p(idx), _p(vals), _p(rp),
                                _p(col), _p(v))
    if rc != 0:
        raise ValueError(f"oracle_coo2csr: index out of range (rc={rc})")
    return rp, col, v


def spmm(k, row_off, sizes, row_ptr, col, vals, B, ldb=None, ldc=None, want_f64=False):
    """O3: fp64-accumulated C (rounded to fp32) and the per-element bound."""
    row_off = _c(row_off, np.int64)
    sz = None if sizes is None else _c(sizes, np.int32)
    row_ptr, col, vals = _c(row_ptr, np.int32), _c(col, np.int32), _c(vals, np.float32)
    B = _c(B, np.float32)
    N = int(row_off[-1])
    ldb = B.shape[1] if (ldb is None and B.ndim == 2) else (k if ldb is None else ldb)
    ldc = k if ldc is None else ldc
    C = np.zeros((N, ldc), dtype=np.float32)
    bound = np.zeros((N, ldc), dtype=np.float64)
    C64 = np.zeros((N, ldc), dtype=np.float64) if want_f64 else None
    rc = _load().oracle_spmm(row_off.shape[0] - 1, k, _p(row_off), _p(sz), _p(row_ptr), _p(col), _p(vals),
                             _p(B), ldb, _p(C), ldc, _p(bound), _p(C64))
    assert rc == 0
    return (C, bound, C64) if want_f64 else (C, bound)


def spmm_f32(k, row_off, sizes, row_ptr, col, vals, B, ldb=None, ldc=None):
    """O3': fp32 fmaf in CSR storage order (bitwise target for order-keeping kernels)."""
    row_off = _c(row_off, np.int64)
    sz = None if sizes is None else _c(sizes, np.int32)
    row_ptr, col, vals = _c(row_ptr, np.int32), _c(col, np.int32), _c(vals, np.float32)
    B = _c(B, np.float32)
    N = int(row_off[-1])
    ldb = B.shape[1] if (ldb is None and B.ndim == 2) else (k if ldb is None else ldb)
    ldc = k if ldc is None else ldc
    C = np.zeros((N, ldc), dtype=np.float32)
    rc = _load().oracle_spmm_f32(row_off.shape[0] - 1, k, _p(row_off), _p(sz), _p(row_ptr), _p(col),
                                 _p(vals), _p(B), ldb, _p(C), ldc)
    assert rc == 0
    return C


def spmm_rows(mat, rloc, k, row_off, row_ptr, col, vals, B, ldb=None):
    """O3 on sampled rows: returns (C_rows [S, k] fp32, bound [S, k] fp64)."""
    mat, rloc = _c(mat, np.int64), _c(rloc, np.int32)
    row_off = _c(row_off, np.int64)
    row_ptr, col, vals = _c(row_ptr, np.int32), _c(col, np.int32), _c(vals, np.float32)
    B = _c(B, np.float32)
    ldb = B.shape[1] if ldb is None else ldb
    S = mat.shape[0]
    out = np.zeros((S, k), dtype=np.float32)
    bound = np.zeros((S, k), dtype=np.float64)
    rc = _load().oracle_spmm_rows(S, _p(mat), _p(rloc), k, _p(row_off), _p(row_ptr), _p(col), _p(vals),
                                  _p(B), ldb, _p(out), _p(bound))
    assert rc == 0
    return out, bound


def partition(nnz_off, k: int, parts: int) -> np.ndarray:
    """O4: contiguous nnz*k-balanced split, int32 [parts+1]."""
    nnz_off = _c(nnz_off, np.int64)
    out = np.zeros(parts + 1, dtype=np.int32)
    assert _load().oracle_partition(nnz_off.shape[0] - 1, _p(nnz_off), k, parts, _p(out)) == 0
    return out


def check_bound(C, C_ref, bound) -> tuple[bool, float]:
    """north_star tolerance: |C - C_ref| <= bound elementwise (fp64). Returns (ok, worst ratio)."""
    d = np.abs(np.asarray(C, dtype=np.float64) - np.asarray(C_ref, dtype=np.float64))
    b = np.asarray(bound, dtype=np.float64)
    ok = bool(np.all(d <= b))
    with np.errstate(divide="ignore", invalid="ignore"):
        r = np.where(b > 0, d / b, np.where(d > 0, np.inf, 0.0))
    return ok, float(r.max()) if r.size else 0.0


def csr_transpose(row_off, sizes, row_ptr, col, vals):
    """O5: per-matrix A_i^T in canonical order. Returns (rowT, colT, valsT)."""
    row_off = _c(row_off, np.int64)
    sz = None if sizes is None else _c(sizes, np.int32)
    row_ptr, col, vals = _c(row_ptr, np.int32), _c(col, np.int32), _c(vals, np.float32)
    rt = np.zeros_like(row_ptr)
    ct = np.zeros_like(col)
    vt = np.zeros_like(vals)
    assert _load().oracle_csr_transpose(row_off.shape[0] - 1, _p(row_off), _p(sz), _p(row_ptr), _p(col), _p(vals),
                                        _p(rt), _p(ct), _p(vt)) == 0
    return rt, ct, vt


def sddmm(k, row_off, sizes, row_ptr, col, B, D, ldb=None, ldd=None):
    """O6: out[e] = <D[row_e], B[col_e]> (fp64 -> fp32) and the per-entry bound."""
    row_off = _c(row_off, np.int64)
    sz = None if sizes is None else _c(sizes, np.int32)
    row_ptr, col = _c(row_ptr, np.int32), _c(col, np.int32)
    B, D = _c(B, np.float32), _c(D, np.float32)
    ldb = B.shape[1] if ldb is None else ldb
    ldd = D.shape[1] if ldd is None else ldd
    out = np.zeros(col.shape[0], dtype=np.float32)
    bound = np.zeros(col.shape[0], dtype=np.float64)
    assert _load().oracle_sddmm(row_off.shape[0] - 1, k, _p(row_off), _p(sz), _p(row_ptr), _p(col), _p(B), ldb,
                                _p(D), ldd, _p(out), _p(bound)) == 0
    return out, bound


def backward(k, row_off, row_ptr, col, vals, B, grad_C):
    """grad_B = A^T grad_C (O5 + O3) and grad_vals = SDDMM (O6), each with its bound."""
    rt, ct, vt = csr_transpose(row_off, None, row_ptr, col, vals)
    gB, gB_bound = spmm(k, row_off, None, rt, ct, vt, grad_C)
    gv, gv_bound = sddmm(k, row_off, None, row_ptr, col, B, grad_C)
    return gB, gB_bound, gv, gv_bound


def gcn_layer(row_off, row_ptrs, col, vals, X, W, bias):
    """O7: Y = sum_ch A_ch (X W_ch + 1 bias_ch^T) in fp64 -> fp32, and the magnitude
    sum M = sum_ch sum_e |a| (sum_l |x||w| + |b|).  row_ptrs: [channels, N+1]."""
    row_off = _c(row_off, np.int64)
    rp = _c(row_ptrs, np.int32)
    channels = rp.shape[0]
    col, vals, X = _c(col, np.int32), _c(vals, np.float32), _c(X, np.float32)
    W, bias = _c(W, np.float32), _c(bias, np.float32)
    n_x, k = W.shape[1], W.shape[2]
    N = int(row_off[-1])
    Y = np.zeros((N, k), dtype=np.float32)
    mag = np.zeros((N, k), dtype=np.float64)
    assert _load().oracle_gcn_layer(row_off.shape[0] - 1, channels, n_x, k, _p(row_off), _p(rp), _p(col), _p(vals),
                                    _p(X), X.shape[1], _p(W), _p(bias), _p(Y), k, _p(mag)) == 0
    return Y, mag
