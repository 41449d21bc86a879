"""ctypes declarations for libbspmm.so (include/bspmm.h).  Loading fails loudly:
there is no CPU fallback anywhere in this package."""
from __future__ import annotations

import ctypes
import os
import re

_HERE = os.path.dirname(os.path.abspath(__file__))
# BSPMM_LIB=checked selects the bounds-checked build (`make checked`): same ABI,
# device-side index checks that trap (the compute-sanitizer stand-in)
LIB_PATH = os.path.join(_HERE, "libbspmm_checked.so" if os.environ.get("BSPMM_LIB") == "checked" else "libbspmm.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "bspmm.h")
DEBUG_HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "bspmm_debug.h")

P, I32, I64, U32 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32

SUCCESS, INVALID_VALUE, OUT_OF_MEMORY, CUDA, INDEX, NOT_SUPPORTED = range(6)
VALIDATE = 0x1


class Plan(ctypes.Structure):
    _fields_ = [("kt", I32), ("tiles", I32), ("lanes", I32), ("vec", I32), ("chunks", I32), ("stages", I32),
                ("stage_b_bytes", I32), ("stage_s_bytes", I32), ("smem_bytes", I32), ("threads", I32),
                ("grid", I32), ("max_rows", I32), ("sched", I32), ("units", I64), ("kernel", I32)]

    def as_dict(self):
        return {name: int(getattr(self, name)) for name, _ in self._fields_}


_SIGS = {
    "bspmm_create": (I32, [ctypes.POINTER(P), ctypes.c_int, P, ctypes.c_uint]),
    "bspmm_destroy": (I32, [P]),
    "bspmm_set_stream": (I32, [P, P]),
    "bspmm_set_hints": (I32, [P, I32, I64]),
    "bspmm_set_tuning": (I32, [P, I32, I32, I32, I32]),
    "bspmm_sync": (I32, [P]),
    "bspmm_set_trace": (I32, [P, P]),
    "bspmm_set_debug": (I32, [P, I32]),
    "bspmm_set_tile_cb": (I32, [P, I32]),
    "bspmm_set_gcn_math": (I32, [P, I32]),
    "bspmm_csr": (I32, [P, I32, I32, P, P, P, P, P, P, I64, P, I64]),
    "bspmm_csr_multicast": (I32, [P, I32, I32, P, P, P, P, P, P, I64, P, I64]),
    "bspmm_mc_supported": (I32, [ctypes.c_int]),
    "bspmm_mc_create": (I32, [ctypes.c_int, ctypes.c_int, ctypes.c_size_t, ctypes.c_int, ctypes.POINTER(P),
                              ctypes.POINTER(ctypes.c_int)]),
    "bspmm_mc_import": (I32, [ctypes.c_int, ctypes.c_int, ctypes.c_size_t, ctypes.c_int, ctypes.POINTER(P)]),
    "bspmm_mc_bind": (I32, [P, ctypes.POINTER(P), ctypes.POINTER(P)]),
    "bspmm_mc_bytes": (ctypes.c_size_t, [P]),
    "bspmm_mc_last_error": (ctypes.c_char_p, []),
    "bspmm_mc_destroy": (I32, [P]),
    "bspmm_coo": (I32, [P, I32, I32, P, P, P, P, P, P, I64, P, I64, I64, I64, P, P, P]),
    "bspmm_coo2csr": (I32, [P, I32, P, P, P, P, P, I64, I64, P, P, P]),
    "bspmm_coo_atomic": (I32, [P, I32, I32, P, P, P, P, P, P, I64, P, I64]),
    "bspmm_gcn_layer": (I32, [P, I32, I32, I32, I32, P, P, P, P, P, P, I64, P, P, P, I64, I64]),
    "bspmm_build_offsets": (I32, [P, I32, P, P]),
    "bspmm_csr_host": (I32, [P, I32, I32, P, P, P, P, P, P, I64, I64]),
    "bspmm_csr_transpose": (I32, [P, I32, P, P, P, P, P, I64, I64, P, P, P]),
    "bspmm_sddmm": (I32, [P, I32, I32, P, P, P, P, P, I64, P, I64, P]),
    "bspmm_csr_backward": (I32, [P, I32, I32, P, P, P, P, P, P, I64, P, I64, P, I64, P, I64, I64]),
    "bspmm_partition": (I32, [I32, P, I32, I32, P]),
    "bspmm_subwarp": (I32, [I32]),
    "bspmm_plan": (I32, [I32, I32, I32, I32, I64, I32, I32, I32, I32, I32, I32, ctypes.POINTER(Plan)]),
    "bspmm_last_plan": (I32, [P, ctypes.POINTER(Plan)]),
    "bspmm_launch_count": (I64, [P]),
    "bspmm_status_string": (ctypes.c_char_p, [I32]),
    "bspmm_last_error_string": (ctypes.c_char_p, [P]),
}


def header_symbols(paths=(HEADER_PATH, DEBUG_HEADER_PATH)) -> list[str]:
    """Every function the C headers declare (BSPMM_API ... name(...)): the
    contract (bspmm.h) and the experiment knobs (bspmm_debug.h)."""
    if isinstance(paths, str):
        paths = (paths,)
    src = "".join(open(p).read() for p in paths)
    return sorted(set(re.findall(r"BSPMM_API\s+[\w\s\*]+?\b(bspmm_\w+)\s*\(", src)))


def load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"CUDA extension {LIB_PATH} is missing: run `make -C {os.path.dirname(_HERE)} lib` "
                          "(or __graft_entry__.build()). There is no CPU fallback.")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


lib = load()


class BspmmError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str = ""):
        self.status = status
        name = lib.bspmm_status_string(status).decode()
        super().__init__(f"{where}: {name}" + (f" ({detail})" if detail else ""))
