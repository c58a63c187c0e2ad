"""TEST INFRASTRUCTURE ONLY — build and load the C oracle (oracle/msda_oracle.c).

``build()`` compiles ``oracle/build/libmsda_oracle.so`` with gcc (no fast-math,
no FP contraction: every f32 multiply and add is rounded separately, as in
numpy).  ``load()`` returns a thin ctypes wrapper.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
SRC = HERE / "msda_oracle.c"
OUT = HERE / "build" / "libmsda_oracle.so"


def build(force: bool = False) -> Path:
    OUT.parent.mkdir(parents=True, exist_ok=True)
    if force or not OUT.exists() or OUT.stat().st_mtime < SRC.stat().st_mtime:
        cmd = ["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
               "-o", str(OUT), str(SRC), "-lm"]
        subprocess.run(cmd, check=True)
    return OUT


_LIB = None


def load():
    global _LIB
    if _LIB is None:
        if not OUT.exists():
            build()
        lib = ctypes.CDLL(str(OUT))
        P = ctypes.c_void_p
        lib.oracle_msda.argtypes = [P, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, P, P, P,
                                    ctypes.c_int64, P, P, P, P, P, P, ctypes.c_int32, ctypes.c_int32,
                                    P, P, ctypes.c_int32]
        lib.oracle_msda.restype = ctypes.c_int
        lib.oracle_f16_roundtrip.argtypes = [ctypes.c_float]
        lib.oracle_f16_roundtrip.restype = ctypes.c_float
        _LIB = lib
    return _LIB


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def msda_c(table, tiles, n_levels, offsets, cam, lvl, u, v, w, normalize=True, half=False, threads=0):
    """C oracle: bit-exact msda_reference (half=False) / PACKED_HALF (half=True).

    Raises ValueError like the reference for bad targets and zero weight sums.
    """
    lib = load()
    table = np.ascontiguousarray(table, dtype=np.float32)
    n_tiles = len(tiles)
    ts = np.ascontiguousarray([t[0] for t in tiles], dtype=np.int64)
    th = np.ascontiguousarray([t[1] for t in tiles], dtype=np.int32)
    tw = np.ascontiguousarray([t[2] for t in tiles], dtype=np.int32)
    arrs = [np.ascontiguousarray(a, dtype=d) for a, d in
            ((offsets, np.int64), (cam, np.int32), (lvl, np.int32), (u, np.float32), (v, np.float32), (w, np.float32))]
    q_n = len(offsets) - 1
    c_n = table.shape[1]
    out = np.zeros((q_n, c_n), dtype=np.float32)
    empty = np.zeros(q_n, dtype=np.uint8)
    st = lib.oracle_msda(_p(table), c_n, n_tiles // n_levels, n_levels, _p(ts), _p(th), _p(tw), q_n,
                         *(_p(a) for a in arrs), int(bool(normalize)), int(bool(half)), _p(out), _p(empty),
                         int(threads or os.cpu_count() or 1))
    if st == 3:
        raise ValueError("plan references an unknown camera or a missing level")
    if st == 4:
        raise ValueError("plan weights sum to zero, cannot renormalize")
    if st != 0:
        raise RuntimeError(f"oracle status {st}")
    return out, empty.astype(bool)


def msda_dense_groups_c(table, tiles, spatial_shape, sampling_location, weights, n_levels, normalize=False,
                        threads=0):
    """Dense Sparse4D layout with channel groups through the C oracle (full
    BASELINE sizes): group g's channel slice = msda_reference over the
    group's CSR plan (SURVEY §8(c) "Groups G"), bs = 1.  ``table`` is the
    f32 view of the features the GPU reads (f16/bf16 widened exactly)."""
    from . import msda_oracle as mo

    g_n = weights.shape[-1]
    c_n = table.shape[1]
    cpg = c_n // g_n
    bs, q_n = sampling_location.shape[:2]
    out = np.empty((bs * q_n, c_n), dtype=np.float32)
    for g in range(g_n):
        plan = mo.dense_to_csr_vectorized(spatial_shape, sampling_location, weights, g)
        sub = np.ascontiguousarray(table[:, g * cpg:(g + 1) * cpg], dtype=np.float32)
        out[:, g * cpg:(g + 1) * cpg], _ = msda_c(sub, tiles, n_levels, *plan, normalize=normalize, threads=threads)
    return out.reshape(bs, q_n, c_n)
