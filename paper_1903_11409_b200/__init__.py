"""B200-native Batched SpMM (arXiv 1903.11409), Python binding.

Argument marshalling only: every step of the hot path runs in libbspmm.so
(include/bspmm.h).  torch supplies device memory and streams.  Importing this
package fails loudly when the CUDA extension is missing; there is no CPU
fallback.

    import paper_1903_11409_b200 as bs
    h = bs.Handle()                       # cuda:current, torch's current stream
    C = h.csr(row_off, None, row_ptr, col, vals, B)     # C_i = A_i B_i, one launch
    C = h.coo(None, sizes, nnz_off, idx, vals, B, total_rows=N)
"""
from __future__ import annotations

import ctypes
from typing import Optional

import numpy as np
import torch

from . import _lib
from ._lib import BspmmError, Plan, lib

__all__ = ["Handle", "BspmmError", "Plan", "McBuffer", "mc_supported", "mc_available", "partition", "subwarp", "plan",
           "default_handle", "header_symbols", "LIB_PATH"]

LIB_PATH = _lib.LIB_PATH
header_symbols = _lib.header_symbols


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _np_ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _check(t, name, dtype, device, ndim=None):
    if t is None:
        return
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if t.device != device:
        raise ValueError(f"{name} must be on {device}, got {t.device}")
    if ndim is not None and t.dim() != ndim:
        raise ValueError(f"{name} must have {ndim} dims")


def _ld(t: torch.Tensor, k: int, name: str) -> int:
    """Leading dimension of a 2-D row-major fp32 matrix (empty matrices: k)."""
    if t.dim() != 2:
        raise ValueError(f"{name} must be 2-D")
    if t.numel() == 0:
        return max(k, 1)
    if t.stride(1) != 1 and t.shape[1] > 1:
        raise ValueError(f"{name} needs unit column stride")
    return max(int(t.stride(0)), k) if t.shape[0] > 1 else max(int(t.shape[1]), k)


def mc_supported(device: int = 0) -> bool:
    """The device reports NVSwitch multicast (bspmm_mc_supported)."""
    return bool(lib.bspmm_mc_supported(int(device)))


_mc_probe: dict = {}


def mc_available(device: int = 0):
    """(ok, why): can a multicast team buffer actually be created here?  A
    device may report support while the driver refuses the object (e.g. one
    GPU of an NVSwitch box passed through to a container)."""
    if device not in _mc_probe:
        if not mc_supported(device):
            _mc_probe[device] = (False, "device reports no multicast support")
        else:
            try:
                McBuffer((1, 1), device).close()
                _mc_probe[device] = (True, "")
            except BspmmError as e:
                _mc_probe[device] = (False, str(e))
    return _mc_probe[device]


class _CudaArray:
    """__cuda_array_interface__ view of library-owned device memory (zero copy)."""

    def __init__(self, ptr: int, shape, owner):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": "<f4", "data": (ptr, False),
                                         "version": 3, "strides": None}
        self._owner = owner


class McBuffer:
    """fp32 [rows, cols] NVSwitch multicast team buffer (bspmm_mc_*, NEXT-4b).

    `uc` is this GPU's copy as a torch tensor (ordinary reads/writes);
    `mc_ptr` is the multicast address: a store there reaches every GPU of the
    team.  Single process: McBuffer(shape, device).  One process per GPU: use
    dist.mc_team_buffer, which passes the exported handle between ranks."""

    def __init__(self, shape, device, num_devices: int = 1, fd: Optional[int] = None, export: bool = False,
                 bind: bool = True):
        self.device = torch.device("cuda", device) if isinstance(device, int) else torch.device(device)
        self.shape = (int(shape[0]), int(shape[1]))
        nbytes = max(4 * self.shape[0] * self.shape[1], 4)
        self._m = ctypes.c_void_p()
        self.fd = None
        if fd is None:
            cfd = ctypes.c_int(-1)
            st = lib.bspmm_mc_create(self.device.index, int(num_devices), nbytes, 1 if export else 0,
                                     ctypes.byref(self._m), ctypes.byref(cfd))
            if st != _lib.SUCCESS:
                raise BspmmError(st, "bspmm_mc_create", lib.bspmm_mc_last_error().decode())
            self.fd = cfd.value if export else None
        else:
            st = lib.bspmm_mc_import(self.device.index, int(num_devices), nbytes, int(fd), ctypes.byref(self._m))
            if st != _lib.SUCCESS:
                raise BspmmError(st, "bspmm_mc_import", lib.bspmm_mc_last_error().decode())
        self.nbytes = int(lib.bspmm_mc_bytes(self._m))
        self.uc = None
        self.mc_ptr = 0
        if bind:
            self.bind()

    def bind(self):
        """Allocate and bind this GPU's memory; call after every team member joined."""
        uc, mc = ctypes.c_void_p(), ctypes.c_void_p()
        st = lib.bspmm_mc_bind(self._m, ctypes.byref(uc), ctypes.byref(mc))
        if st != _lib.SUCCESS:
            raise BspmmError(st, "bspmm_mc_bind", lib.bspmm_mc_last_error().decode())
        self.mc_ptr = int(mc.value)
        self.uc = torch.as_tensor(_CudaArray(int(uc.value), self.shape, self), device=self.device)

    def close(self):
        if getattr(self, "_m", None) is not None and self._m.value:
            self.uc = None
            lib.bspmm_mc_destroy(self._m)
            self._m = None

    def __del__(self):
        self.close()


class Handle:
    """One library handle per device (not thread-safe).  Calls enqueue on torch's
    current stream of the handle's device and return without synchronising."""

    def __init__(self, device=None, validate: bool = False):
        if device is None:
            device = torch.cuda.current_device()
        self.device = torch.device("cuda", device) if isinstance(device, int) else torch.device(device)
        self._h = ctypes.c_void_p()
        st = lib.bspmm_create(ctypes.byref(self._h), self.device.index, None, _lib.VALIDATE if validate else 0)
        if st != _lib.SUCCESS:
            raise BspmmError(st, "bspmm_create")

    def __del__(self):
        h = getattr(self, "_h", None)
        # at interpreter shutdown the module globals may already be gone: the
        # process exit releases the handle's device memory then
        if h is not None and h.value and lib is not None:
            lib.bspmm_destroy(h)
            self._h = None

    # ---- plumbing ----------------------------------------------------------
    def _stream(self):
        s = torch.cuda.current_stream(self.device).cuda_stream
        lib.bspmm_set_stream(self._h, ctypes.c_void_p(s))

    def _raise(self, st, where):
        if st != _lib.SUCCESS:
            raise BspmmError(st, where, lib.bspmm_last_error_string(self._h).decode())

    def set_hints(self, max_rows: int = 0, max_nnz: int = 0):
        self._raise(lib.bspmm_set_hints(self._h, int(max_rows), int(max_nnz)), "bspmm_set_hints")

    def set_tuning(self, kt: int = 0, consumer_warps: int = 0, ctas_per_sm: int = 0, chunks: int = 0):
        self._raise(lib.bspmm_set_tuning(self._h, int(kt), int(consumer_warps), int(ctas_per_sm), int(chunks)),
                    "bspmm_set_tuning")

    def set_trace(self, buf: Optional[torch.Tensor]):
        """Debug: record per-CTA phase timestamps of subsequent SpMM launches into
        buf (int64 [grid, 16] on the handle's device); None disables."""
        if buf is not None:
            _check(buf, "trace", torch.int64, self.device)
        self._raise(lib.bspmm_set_trace(self._h, _ptr(buf)), "bspmm_set_trace")

    def set_tile_cb(self, cb: int):
        """Experiment knob (bspmm_debug.h): float4 columns per tile of the small-batch kernel, 0 = planner."""
        self._raise(lib.bspmm_set_tile_cb(self._h, int(cb)), "bspmm_set_tile_cb")

    def set_debug(self, bits: int):
        """Debug bits for timing experiments (1 = skip C stores; results undefined)."""
        self._raise(lib.bspmm_set_debug(self._h, int(bits)), "bspmm_set_debug")

    def set_gcn_math(self, mode: str = "fp32"):
        """GEMM arithmetic of gcn_layer: "fp32" (default), "tf32" or "bf16" tensor cores."""
        code = {"fp32": 0, "tf32": 1, "bf16": 2}[mode]
        self._raise(lib.bspmm_set_gcn_math(self._h, code), "bspmm_set_gcn_math")

    def sync(self):
        self._raise(lib.bspmm_sync(self._h), "bspmm_sync")

    def last_plan(self) -> dict:
        p = Plan()
        self._raise(lib.bspmm_last_plan(self._h, ctypes.byref(p)), "bspmm_last_plan")
        return p.as_dict()

    def launch_count(self) -> int:
        return int(lib.bspmm_launch_count(self._h))

    # ---- hot path ------------------------------------------------------------
    def build_offsets(self, sizes: torch.Tensor, out: Optional[torch.Tensor] = None) -> torch.Tensor:
        """Row a-1: int64 exclusive scan of int32 sizes, [batch+1], on the device."""
        _check(sizes, "sizes", torch.int32, self.device, 1)
        batch = sizes.shape[0]
        if out is None:
            out = torch.empty(batch + 1, dtype=torch.int64, device=self.device)
        _check(out, "out", torch.int64, self.device, 1)
        assert out.shape[0] == batch + 1 and sizes.is_contiguous() and out.is_contiguous()
        self._stream()
        self._raise(lib.bspmm_build_offsets(self._h, batch, _ptr(sizes), _ptr(out)), "bspmm_build_offsets")
        return out

    def csr(self, row_off: Optional[torch.Tensor], sizes: Optional[torch.Tensor], row_ptr: torch.Tensor,
            col: torch.Tensor, vals: torch.Tensor, B: torch.Tensor, C: Optional[torch.Tensor] = None,
            k: Optional[int] = None, batch: Optional[int] = None) -> torch.Tensor:
        """Batched CSR SpMM: C_i = A_i B_i for all i in one launch (bspmm_csr).
        B, C: 2-D fp32 [rows, ld] with unit column stride; k defaults to B.shape[1]."""
        dev = self.device
        for name, t, dt in (("row_off", row_off, torch.int64), ("sizes", sizes, torch.int32),
                            ("row_ptr", row_ptr, torch.int32), ("col", col, torch.int32),
                            ("vals", vals, torch.float32), ("B", B, torch.float32), ("C", C, torch.float32)):
            _check(t, name, dt, dev)
        if batch is None:
            batch = (row_off.shape[0] - 1) if row_off is not None else sizes.shape[0]
        if k is None:
            k = B.shape[1]
        if C is None:
            C = torch.empty((B.shape[0], k), dtype=torch.float32, device=dev)
        ldb, ldc = _ld(B, k, "B"), _ld(C, k, "C")
        self._stream()
        st = lib.bspmm_csr(self._h, batch, k, _ptr(row_off), _ptr(sizes), _ptr(row_ptr), _ptr(col), _ptr(vals),
                           _ptr(B), ldb, _ptr(C), ldc)
        self._raise(st, "bspmm_csr")
        return C

    def csr_multicast(self, row_off: Optional[torch.Tensor], sizes: Optional[torch.Tensor], row_ptr: torch.Tensor,
                      col: torch.Tensor, vals: torch.Tensor, B: torch.Tensor, out, row_base: int = 0,
                      k: Optional[int] = None, batch: Optional[int] = None) -> None:
        """bspmm_csr with the all-gather fused into the store (NEXT-4b): this
        shard's C rows land at global rows row_base.. of `out` (an McBuffer) on
        EVERY GPU of the multicast team.  A team barrier must follow before
        reading out.uc (dist.team_barrier).  `out` may also be an ordinary fp32
        tensor: the tests' unicast emulation on boxes where the driver refuses
        multicast objects (on sm_100a multimem.st lowers to the plain STG.E.128
        of the same address; not a supported use)."""
        dev = self.device
        for name, t, dt in (("row_off", row_off, torch.int64), ("sizes", sizes, torch.int32),
                            ("row_ptr", row_ptr, torch.int32), ("col", col, torch.int32),
                            ("vals", vals, torch.float32), ("B", B, torch.float32)):
            _check(t, name, dt, dev)
        if isinstance(out, torch.Tensor):
            _check(out, "out", torch.float32, dev, 2)
            if out.stride(1) != 1 or not out.is_contiguous():
                raise ValueError("out must be contiguous")
            base_ptr = out.data_ptr()
        else:
            base_ptr = out.mc_ptr
        if out.device != dev:
            raise ValueError("multicast buffer is on another device")
        if batch is None:
            batch = (row_off.shape[0] - 1) if row_off is not None else sizes.shape[0]
        if k is None:
            k = B.shape[1]
        ldc = out.shape[1]
        rows = int(B.shape[0])
        if ldc < k or row_base < 0 or (row_base + rows) > out.shape[0]:
            raise ValueError("shard rows / k do not fit the multicast buffer")
        ldb = _ld(B, k, "B")
        self._stream()
        st = lib.bspmm_csr_multicast(self._h, batch, k, _ptr(row_off), _ptr(sizes), _ptr(row_ptr), _ptr(col),
                                     _ptr(vals), _ptr(B), ldb, ctypes.c_void_p(base_ptr + 4 * row_base * ldc), ldc)
        self._raise(st, "bspmm_csr_multicast")

    def coo(self, row_off: Optional[torch.Tensor], sizes: Optional[torch.Tensor], nnz_off: torch.Tensor,
            idx: torch.Tensor, vals: torch.Tensor, B: torch.Tensor, C: Optional[torch.Tensor] = None,
            k: Optional[int] = None, total_rows: Optional[int] = None, csr_out=None,
            checked: bool = False) -> torch.Tensor:
        """Batched COO/SparseTensor SpMM (bspmm_coo): device COO->CSR, then the CSR kernel.
        idx: int32 [nnz, 2] (row, col) local pairs.  csr_out: optional (row_ptr, col, vals) tensors.

        With planner hints set (set_hints) the conversion is fused into the SpMM launch, and a
        matrix larger than the hints is SKIPPED (its rows of C are left unwritten); that is
        reported only by the next sync().  checked=True synchronises and raises here instead."""
        dev = self.device
        for name, t, dt in (("row_off", row_off, torch.int64), ("sizes", sizes, torch.int32),
                            ("nnz_off", nnz_off, torch.int64), ("idx", idx, torch.int32),
                            ("vals", vals, torch.float32), ("B", B, torch.float32), ("C", C, torch.float32)):
            _check(t, name, dt, dev)
        batch = nnz_off.shape[0] - 1
        if k is None:
            k = B.shape[1]
        if total_rows is None:
            total_rows = B.shape[0]
        if C is None:
            C = torch.empty((B.shape[0], k), dtype=torch.float32, device=dev)
        rp_o, col_o, val_o = csr_out if csr_out is not None else (None, None, None)
        ldb, ldc = _ld(B, k, "B"), _ld(C, k, "C")
        self._stream()
        st = lib.bspmm_coo(self._h, batch, k, _ptr(row_off), _ptr(sizes), _ptr(nnz_off), _ptr(idx), _ptr(vals),
                           _ptr(B), ldb, _ptr(C), ldc, int(total_rows), int(idx.shape[0]),
                           _ptr(rp_o), _ptr(col_o), _ptr(val_o))
        self._raise(st, "bspmm_coo")
        if checked:
            self.sync()
        return C

    def coo_atomic(self, row_off: Optional[torch.Tensor], sizes: Optional[torch.Tensor], nnz_off: torch.Tensor,
                   idx: torch.Tensor, vals: torch.Tensor, B: torch.Tensor, C: Optional[torch.Tensor] = None,
                   k: Optional[int] = None) -> torch.Tensor:
        """The paper's atomic SWA SpMM for SparseTensor (bspmm_coo_atomic): nondeterministic order."""
        dev = self.device
        for name, t, dt in (("row_off", row_off, torch.int64), ("sizes", sizes, torch.int32),
                            ("nnz_off", nnz_off, torch.int64), ("idx", idx, torch.int32),
                            ("vals", vals, torch.float32), ("B", B, torch.float32), ("C", C, torch.float32)):
            _check(t, name, dt, dev)
        k = B.shape[1] if k is None else k
        if C is None:
            C = torch.empty((B.shape[0], k), dtype=torch.float32, device=dev)
        self._stream()
        st = lib.bspmm_coo_atomic(self._h, nnz_off.shape[0] - 1, k, _ptr(row_off), _ptr(sizes), _ptr(nnz_off),
                                  _ptr(idx), _ptr(vals), _ptr(B), _ld(B, k, "B"), _ptr(C), _ld(C, k, "C"))
        self._raise(st, "bspmm_coo_atomic")
        return C

    def coo2csr(self, row_off: torch.Tensor, sizes: Optional[torch.Tensor], nnz_off: torch.Tensor,
                idx: torch.Tensor, vals: torch.Tensor, total_rows: int):
        """Row a-2 alone: canonical CSR (row_ptr, col, vals) built on the device."""
        dev = self.device
        for name, t, dt in (("row_off", row_off, torch.int64), ("sizes", sizes, torch.int32),
                            ("nnz_off", nnz_off, torch.int64), ("idx", idx, torch.int32),
                            ("vals", vals, torch.float32)):
            _check(t, name, dt, dev)
        nnz = idx.shape[0]
        rp = torch.empty(total_rows + 1, dtype=torch.int32, device=dev)
        col = torch.empty(nnz, dtype=torch.int32, device=dev)
        v = torch.empty(nnz, dtype=torch.float32, device=dev)
        self._stream()
        st = lib.bspmm_coo2csr(self._h, nnz_off.shape[0] - 1, _ptr(row_off), _ptr(sizes), _ptr(nnz_off), _ptr(idx),
                               _ptr(vals), int(total_rows), int(nnz), _ptr(rp), _ptr(col), _ptr(v))
        self._raise(st, "bspmm_coo2csr")
        return rp, col, v

    # ---- fused GCN layer (NEXT-1) -------------------------------------------------
    def gcn_layer(self, row_off: torch.Tensor, sizes: Optional[torch.Tensor], row_ptrs: torch.Tensor,
                  col: torch.Tensor, vals: torch.Tensor, X: torch.Tensor, W: torch.Tensor,
                  bias: Optional[torch.Tensor] = None, Y: Optional[torch.Tensor] = None) -> torch.Tensor:
        """Y = sum_ch A_ch (X W_ch + 1 bias_ch^T) (bspmm_gcn_layer).  row_ptrs: int32 [channels, N+1];
        W: [channels, n_x, k]; bias: [channels, k]."""
        dev = self.device
        for name, t, dt in (("row_off", row_off, torch.int64), ("sizes", sizes, torch.int32),
                            ("row_ptrs", row_ptrs, torch.int32), ("col", col, torch.int32),
                            ("vals", vals, torch.float32), ("X", X, torch.float32), ("W", W, torch.float32),
                            ("bias", bias, torch.float32), ("Y", Y, torch.float32)):
            _check(t, name, dt, dev)
        channels, n_x, k = W.shape
        N = X.shape[0]
        assert row_ptrs.shape == (channels, N + 1) and W.is_contiguous() and row_ptrs.is_contiguous()
        if Y is None:
            Y = torch.empty((N, k), dtype=torch.float32, device=dev)
        self._stream()
        st = lib.bspmm_gcn_layer(self._h, row_off.shape[0] - 1, channels, n_x, k, _ptr(row_off), _ptr(sizes),
                                 _ptr(row_ptrs), _ptr(col), _ptr(vals), _ptr(X), _ld(X, n_x, "X"), _ptr(W),
                                 _ptr(bias), _ptr(Y), _ld(Y, k, "Y"), N)
        self._raise(st, "bspmm_gcn_layer")
        return Y

    # ---- backward (NEXT-2) ---------------------------------------------------------
    def csr_transpose(self, row_off: torch.Tensor, sizes: Optional[torch.Tensor], row_ptr: torch.Tensor,
                      col: torch.Tensor, vals: torch.Tensor):
        """Per-matrix A_i^T (canonical order) on the device: (rowT, colT, valsT)."""
        dev = self.device
        for name, t, dt in (("row_off", row_off, torch.int64), ("sizes", sizes, torch.int32),
                            ("row_ptr", row_ptr, torch.int32), ("col", col, torch.int32),
                            ("vals", vals, torch.float32)):
            _check(t, name, dt, dev)
        rt = torch.empty_like(row_ptr)
        ct = torch.empty_like(col)
        vt = torch.empty_like(vals)
        self._stream()
        st = lib.bspmm_csr_transpose(self._h, row_off.shape[0] - 1, _ptr(row_off), _ptr(sizes), _ptr(row_ptr),
                                     _ptr(col), _ptr(vals), int(row_ptr.shape[0] - 1), int(col.shape[0]), _ptr(rt),
                                     _ptr(ct), _ptr(vt))
        self._raise(st, "bspmm_csr_transpose")
        return rt, ct, vt

    def sddmm(self, row_off: torch.Tensor, sizes: Optional[torch.Tensor], row_ptr: torch.Tensor, col: torch.Tensor,
              B: torch.Tensor, G: torch.Tensor, out: Optional[torch.Tensor] = None, k: Optional[int] = None):
        """out[e] = <G[row_e], B[col_e]> at A's pattern (bspmm_sddmm)."""
        dev = self.device
        for name, t, dt in (("row_off", row_off, torch.int64), ("sizes", sizes, torch.int32),
                            ("row_ptr", row_ptr, torch.int32), ("col", col, torch.int32),
                            ("B", B, torch.float32), ("G", G, torch.float32)):
            _check(t, name, dt, dev)
        k = B.shape[1] if k is None else k
        if out is None:
            out = torch.empty(col.shape[0], dtype=torch.float32, device=dev)
        self._stream()
        st = lib.bspmm_sddmm(self._h, row_off.shape[0] - 1, k, _ptr(row_off), _ptr(sizes), _ptr(row_ptr), _ptr(col),
                             _ptr(B), _ld(B, k, "B"), _ptr(G), _ld(G, k, "G"), _ptr(out))
        self._raise(st, "bspmm_sddmm")
        return out

    def csr_backward(self, row_off: torch.Tensor, sizes: Optional[torch.Tensor], row_ptr: torch.Tensor,
                     col: torch.Tensor, vals: torch.Tensor, B: torch.Tensor, grad_C: torch.Tensor,
                     want_B: bool = True, want_vals: bool = True, k: Optional[int] = None,
                     grad_B: Optional[torch.Tensor] = None, grad_vals: Optional[torch.Tensor] = None):
        """(grad_B, grad_vals) of C = A B for upstream grad_C (bspmm_csr_backward).
        k defaults to grad_C's width (smaller: the leading k columns of row-strided
        B / grad_C); grad_B / grad_vals: optional output tensors (else allocated)."""
        dev = self.device
        for name, t, dt in (("row_off", row_off, torch.int64), ("sizes", sizes, torch.int32),
                            ("row_ptr", row_ptr, torch.int32), ("col", col, torch.int32),
                            ("vals", vals, torch.float32), ("B", B, torch.float32), ("grad_C", grad_C, torch.float32),
                            ("grad_B", grad_B, torch.float32), ("grad_vals", grad_vals, torch.float32)):
            _check(t, name, dt, dev)
        k = grad_C.shape[1] if k is None else int(k)
        gB = grad_B if grad_B is not None else (
            torch.empty((grad_C.shape[0], k), dtype=torch.float32, device=dev) if want_B else None)
        gv = grad_vals if grad_vals is not None else (
            torch.empty(col.shape[0], dtype=torch.float32, device=dev) if want_vals else None)
        want_B = gB is not None
        self._stream()
        st = lib.bspmm_csr_backward(self._h, row_off.shape[0] - 1, k, _ptr(row_off), _ptr(sizes), _ptr(row_ptr),
                                    _ptr(col), _ptr(vals), _ptr(B), _ld(B, k, "B"), _ptr(grad_C),
                                    _ld(grad_C, k, "grad_C"), _ptr(gB), _ld(gB, k, "grad_B") if want_B else k,
                                    _ptr(gv), int(row_ptr.shape[0] - 1), int(col.shape[0]))
        self._raise(st, "bspmm_csr_backward")
        return gB, gv

    def csr_host(self, sizes: np.ndarray, row_ptr: np.ndarray, col: np.ndarray, vals: np.ndarray, B: np.ndarray,
                 C: Optional[np.ndarray] = None) -> np.ndarray:
        """End-to-end on host buffers (bspmm_csr_host): H2D, offsets, SpMM, D2H, pipelined; synchronous.
        Arrays may be numpy arrays or CPU torch tensors (pinned for full copy overlap)."""
        def arr(x, dt):
            if isinstance(x, torch.Tensor):
                assert x.device.type == "cpu" and x.is_contiguous()
                assert x.dtype == {np.int32: torch.int32, np.float32: torch.float32}[dt]
                return x, ctypes.c_void_p(x.data_ptr())
            x = np.ascontiguousarray(x, dtype=dt)
            return x, _np_ptr(x)
        sizes, p_s = arr(sizes, np.int32)
        row_ptr, p_rp = arr(row_ptr, np.int32)
        col, p_c = arr(col, np.int32)
        vals, p_v = arr(vals, np.float32)
        B, p_B = arr(B, np.float32)
        N, k = B.shape
        if C is None:
            C = np.empty((N, k), dtype=np.float32)
        C, p_C = arr(C, np.float32)
        self._stream()
        st = lib.bspmm_csr_host(self._h, int(sizes.shape[0]), int(k), p_s, p_rp, p_c, p_v, p_B, p_C, int(N),
                                int(col.shape[0]))
        self._raise(st, "bspmm_csr_host")
        return C


_default = {}


def default_handle(device=None) -> Handle:
    idx = torch.cuda.current_device() if device is None else torch.device(device).index
    if idx not in _default:
        _default[idx] = Handle(idx)
    return _default[idx]


# ---- host-only helpers (no GPU needed) -------------------------------------------

def partition(nnz_off, k: int, parts: int) -> np.ndarray:
    """Row a-7: contiguous nnz*k-balanced split of graphs over `parts` ranks."""
    no = np.ascontiguousarray(nnz_off, dtype=np.int64)
    out = np.zeros(parts + 1, dtype=np.int32)
    st = lib.bspmm_partition(no.shape[0] - 1, _np_ptr(no), int(k), int(parts), _np_ptr(out))
    if st != _lib.SUCCESS:
        raise BspmmError(st, "bspmm_partition")
    return out


def subwarp(n_B: int) -> int:
    """The paper's subWarp rule."""
    return int(lib.bspmm_subwarp(int(n_B)))


def plan(k: int, batch: int, aligned: bool = True, max_rows: int = 0, max_nnz: int = 0, num_sms: int = 148,
         smem_per_cta: int = 232448, kt: int = 0, consumer_warps: int = 0, ctas_per_sm: int = 0,
         chunks: int = 0) -> dict:
    """The launch plan bspmm_csr would use (pure host)."""
    p = Plan()
    st = lib.bspmm_plan(int(k), int(batch), int(bool(aligned)), int(max_rows), int(max_nnz), int(num_sms),
                        int(smem_per_cta), int(kt), int(consumer_warps), int(ctas_per_sm), int(chunks),
                        ctypes.byref(p))
    if st != _lib.SUCCESS:
        raise BspmmError(st, "bspmm_plan")
    return p.as_dict()
