"""TEST INFRASTRUCTURE ONLY: ctypes wrapper of the allocator-trace oracle
(oracle/arena_oracle.c, built by oracle/build.py into oracle/_build/).
Used by tests/ and bench.py's cpu_baseline leg as the checker / CPU
baseline; the product's allocator is csrc/arena.cpp."""

from __future__ import annotations

import ctypes as C

import numpy as np

from .build import build

_lib = None


def _load():
    global _lib
    if _lib is None:
        _lib = C.CDLL(str(build()))
        p = C.c_void_p
        _lib.oracle_alloc_trace.argtypes = [C.c_int64, C.c_int64, p, p, p, p, p, p, p]
        _lib.oracle_alloc_trace.restype = C.c_int
    return _lib


def alloc_trace(capacity: int, is_alloc, size, align, pick):
    """(out_ok u8[n], out_off i64[n], (total_free, largest, n_extents)) --
    the reference alloc_trace_run contract (numba_backend.py:139-247)."""
    is_alloc = np.ascontiguousarray(is_alloc, dtype=np.uint8)
    size = np.ascontiguousarray(size, dtype=np.int64)
    align = np.ascontiguousarray(align, dtype=np.int64)
    pick = np.ascontiguousarray(pick, dtype=np.uint64)
    n = is_alloc.shape[0]
    ok = np.empty(n, dtype=np.uint8)
    off = np.empty(n, dtype=np.int64)
    fin = np.empty(3, dtype=np.int64)
    rc = _load().oracle_alloc_trace(
        int(capacity), n, is_alloc.ctypes.data, size.ctypes.data, align.ctypes.data,
        pick.ctypes.data, ok.ctypes.data, off.ctypes.data, fin.ctypes.data)
    if rc:
        raise MemoryError("oracle_alloc_trace: allocation failed")
    return ok, off, tuple(int(x) for x in fin)
