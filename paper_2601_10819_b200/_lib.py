"""ctypes binding of the in-tree C-ABI library (include/msda_b200.h).

This is the only way the package reaches the GPU: every op goes through
``libmsda_b200.so``.  There is no CPU fallback — if the library is missing
the import fails loudly with instructions to build it.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "lib" / "libmsda_b200.so"

MSDA_OK = 0
MSDA_ODD_CHANNELS = 1
MSDA_NONFINITE = 2
MSDA_BAD_TARGET = 3
MSDA_ZERO_WEIGHT_SUM = 4
MSDA_BAD_PRECISION = 5
MSDA_CHANNEL_MISMATCH = 6
MSDA_CUDA_ERROR = 7
MSDA_BAD_ARG = 8
MSDA_OFFSET_RANGE = 9

MSDA_F32, MSDA_F16, MSDA_BF16 = 0, 1, 2
MSDA_EXACT, MSDA_EXACT_HALF, MSDA_FAST, MSDA_FAST_H2 = 0, 1, 2, 3

P = ctypes.c_void_p
I32 = ctypes.c_int32
I64 = ctypes.c_int64
SZ = ctypes.c_size_t


class Features(ctypes.Structure):
    _fields_ = [("data", P), ("dtype", I32), ("batch", I32), ("n_cams", I32), ("n_levels", I32),
                ("channels", I32), ("reserved", I32), ("n_rows", I64), ("spatial_shape", P),
                ("scale_start_index", P), ("spatial_shape_host", P)]


class CsrPlan(ctypes.Structure):
    _fields_ = [("n_queries", I64), ("n_samples", I64), ("offsets", P), ("camera_index", P), ("level", P),
                ("u", P), ("v", P), ("weight", P)]


class Cameras(ctypes.Structure):
    _fields_ = [("K", P), ("R", P), ("t", P)]


# name -> (restype, argtypes): exactly the symbols include/msda_b200.h declares
SIGNATURES = {
    "msda_status_string": (ctypes.c_char_p, [I32]),
    "msda_abi_version": (I32, []),
    "msda_csr_workspace_size": (SZ, [I64, I64, I32]),
    "msda_csr": (I32, [ctypes.POINTER(Features), ctypes.POINTER(CsrPlan), I32, I32, P, P, P, SZ, P]),
    "msda_csr_stages": (I32, [ctypes.POINTER(Features), ctypes.POINTER(CsrPlan), I32, I32, P, P, P, SZ, P, I32]),
    "msda_dense_workspace_size": (SZ, [I32, I32, I32, I32, I32, I32, I32]),
    "msda_dense": (I32, [ctypes.POINTER(Features), I32, I32, I32, P, P, I32, I32, P, P, SZ, P]),
    "msda_dense_partial": (I32, [ctypes.POINTER(Features), I32, I32, I32, P, P, I32, P, P, P, SZ, P]),
    "msda_dense_normalize": (I32, [P, P, I64, I32, I32, P, P]),
    "msda_dense_project": (I32, [ctypes.POINTER(Features), I32, P, I32, P, ctypes.POINTER(Cameras), P,
                                 ctypes.c_float, I32, P, I32, I32, P, P, SZ, P]),
    "msda_oae_pool": (I32, [ctypes.POINTER(Features), I32, P, I32, P, ctypes.POINTER(Cameras), P, P, P, P, P, P,
                            P, SZ, P]),
    "msda_oae_workspace_size": (SZ, [I32, I32, I32]),
    "msda_visibility_workspace_size": (SZ, [I32, I32]),
    "msda_visibility": (I32, [ctypes.POINTER(Cameras), P, I32, P, I32, I32, P, P, P, SZ, P]),
    "msda_paint_workspace_size": (SZ, [I32, I32]),
    "msda_paint": (I32, [ctypes.POINTER(Cameras), I32, I32, P, P, P, P, I32, P, I32, I32, P, P, ctypes.c_float,
                         ctypes.c_uint64, I32, I32, P, P, SZ, P]),
    "msda_assoc_cost": (I32, [P, P, P, P, I32, I32, I32, ctypes.c_double, ctypes.c_double, ctypes.c_double, P, P, P,
                              P]),
    "msda_read_status": (I32, [P, P, ctypes.POINTER(I32), ctypes.POINTER(I64)]),
    "msda_context_create": (I32, [I32, ctypes.POINTER(P)]),
    "msda_context_destroy": (None, [P]),
    "msda_context_last_h2d_bytes": (ctypes.c_longlong, [P]),
    "msda_context_last_detail": (ctypes.c_longlong, [P]),
    "msda_bilinear_host": (I32, [P, P, I32, I32, I32, I64, P, P, P]),
    "msda_csr_host": (I32, [P, P, P, I32, I32, I32, I32, I64, P, P, P, P, P, P, I32, I32, P, P]),
    "msda_host_register": (I32, [P, SZ, I32]),
    "msda_host_unregister": (I32, [P]),
    "msda_peer_buffer_size": (SZ, [I64, I32, I32]),
    "msda_peer_alloc": (I32, [SZ, ctypes.POINTER(P)]),
    "msda_peer_free": (I32, [P]),
    "msda_ipc_handle": (I32, [P, P]),
    "msda_ipc_open": (I32, [P, ctypes.POINTER(P)]),
    "msda_ipc_close": (I32, [P]),
    "msda_peer_allreduce_normalize": (I32, [P, P, P, I32, I32, ctypes.c_uint32, I64, I32, I32, I32, P, P, P, P]),
}

_lib = None


def lib():
    """Load (once) and return the library; raise if it has not been built."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: build the CUDA library first "
                "(python -c 'import __graft_entry__ as g; g.build()'). There is no CPU fallback.")
        handle = ctypes.CDLL(str(LIB_PATH), mode=os.RTLD_GLOBAL if hasattr(os, "RTLD_GLOBAL") else 0)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def status_string(code: int) -> str:
    return lib().msda_status_string(int(code)).decode()
