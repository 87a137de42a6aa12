"""CPU oracle for the SpTRSV hot path — TEST INFRASTRUCTURE ONLY.

Restates the reference algorithms (`/root/reference/pkg/src/sptrsv/reference.py:20-35`,
`analysis.py:19-64`, `matrix.py:203-213`) in plain C (``sptrsv_oracle.c``,
built into ``liboracle.so`` by ``make`` / ``build()``) with thin numpy
wrappers. Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU
baseline / ``--impl reference`` arm may import this package; the product
package never does.

Pinned against the reference itself: ``tests/golden/*.npz`` were produced by
running the reference package (``tests/golden/make_golden.py``) and
``tests/test_oracle.py`` checks this oracle against every one of them bit for
bit.
"""

from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "liboracle.so"
_lib = None

_P64 = C.POINTER(C.c_int64)
_PD = C.POINTER(C.c_double)


def build() -> Path:
    src = HERE / "sptrsv_oracle.c"
    if not LIB.exists() or LIB.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = C.CDLL(str(LIB))
        lib.oracle_solve_serial.argtypes = [C.c_int64, _P64, _P64, _PD, _PD, _PD]
        lib.oracle_solve_serial.restype = C.c_int
        lib.oracle_in_degrees.argtypes = [C.c_int64, _P64, _P64, _P64]
        lib.oracle_in_degrees.restype = None
        lib.oracle_levels.argtypes = [C.c_int64, _P64, _P64, _P64]
        lib.oracle_levels.restype = C.c_int64
        lib.oracle_spmv.argtypes = [C.c_int64, _P64, _P64, _PD, _PD, _PD]
        lib.oracle_spmv.restype = None
        lib.oracle_markstein_mismatches.argtypes = [C.c_int64, C.c_uint64]
        lib.oracle_markstein_mismatches.restype = C.c_int64
        _lib = lib
    return _lib


def _i64(a):
    a = np.ascontiguousarray(a, dtype=np.int64)
    return a, a.ctypes.data_as(_P64)


def _f64(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a, a.ctypes.data_as(_PD)


def solve_serial(col_ptr, row_idx, values, b) -> np.ndarray:
    """Alg. 1 forward substitution, bit-identical to the reference's Python loop."""
    lib = _load()
    cp, pcp = _i64(col_ptr)
    ri, pri = _i64(row_idx)
    va, pva = _f64(values)
    bb, pb = _f64(b)
    n = cp.size - 1
    x = np.empty(n)
    if lib.oracle_solve_serial(n, pcp, pri, pva, pb, x.ctypes.data_as(_PD)) != 0:
        raise MemoryError("oracle allocation failed")
    return x


def in_degrees(col_ptr, row_idx) -> np.ndarray:
    lib = _load()
    cp, pcp = _i64(col_ptr)
    ri, pri = _i64(row_idx)
    n = cp.size - 1
    out = np.empty(n, dtype=np.int64)
    lib.oracle_in_degrees(n, pcp, pri, out.ctypes.data_as(_P64))
    return out


def levels(col_ptr, row_idx) -> tuple[np.ndarray, int]:
    lib = _load()
    cp, pcp = _i64(col_ptr)
    ri, pri = _i64(row_idx)
    n = cp.size - 1
    out = np.empty(n, dtype=np.int64)
    nl = lib.oracle_levels(n, pcp, pri, out.ctypes.data_as(_P64))
    return out, int(nl)


def spmv(col_ptr, row_idx, values, x) -> np.ndarray:
    lib = _load()
    cp, pcp = _i64(col_ptr)
    ri, pri = _i64(row_idx)
    va, pva = _f64(values)
    xx, px = _f64(x)
    n = cp.size - 1
    y = np.empty(n)
    lib.oracle_spmv(n, pcp, pri, pva, px, y.ctypes.data_as(_PD))
    return y


def markstein_mismatches(count: int, seed: int = 1) -> int:
    """Mismatches of the kernels' Markstein division vs IEEE a/d on random operands."""
    return int(_load().oracle_markstein_mismatches(count, seed))


def solve_serial_py(col_ptr, row_idx, values, b) -> np.ndarray:
    """Pure-Python restatement for tiny cases (cross-checks the C build)."""
    n = len(col_ptr) - 1
    left = [0.0] * n
    x = [0.0] * n
    for i in range(n):
        lo, hi = int(col_ptr[i]), int(col_ptr[i + 1])
        xi = (float(b[i]) - left[i]) / float(values[lo])
        x[i] = xi
        for k in range(lo + 1, hi):
            left[int(row_idx[k])] += float(values[k]) * xi
    return np.array(x)
