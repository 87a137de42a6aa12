"""Row f4 of SURVEY.md §8(f): backward substitution (``U x = b``) and several
right-hand sides, on the same device executors.

The reference solves lower-triangular systems only (its SPEC.md:9 puts
``Ux=b`` out of scope). Reversing the index order, i -> n-1-i, maps an upper
triangular U to a lower triangular L' = P U P (P the reversal permutation):
``U x = b`` is ``L' (P x) = P b``. The serial solve of L' accumulates each
row's terms in ascending column order of L', which is descending column order
of U — exactly backward substitution — so ``precision="exact"`` gives the
serial backward-substitution result bit for bit. The reversal is a pure
index relabelling of the CSC arrays (no arithmetic), done once per matrix.
"""

from __future__ import annotations

import numpy as np

from . import _native
from .errors import DimensionMismatch, MatrixStructureError
from .matrix import CscMatrix


def reverse_upper(u: CscMatrix) -> CscMatrix:
    """P U P for an upper-triangular CSC ``u`` (rows ascending per column): lower triangular, CSC.

    New column j' is old column n-1-j' walked backwards, rows relabelled
    r -> n-1-r, so rows come out ascending with the diagonal first.
    """
    n = u.n
    cp = np.asarray(u.col_ptr, dtype=np.int64)
    ri = np.asarray(u.row_idx, dtype=np.int64)
    va = np.asarray(u.values, dtype=np.float64)
    lens = np.diff(cp)
    if ri.size and np.any(ri > np.repeat(np.arange(n), lens)):
        raise MatrixStructureError("matrix is not upper triangular (an entry below the diagonal)")
    new_lens = lens[::-1]
    new_cp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(new_lens, out=new_cp[1:])
    k = np.arange(ri.size, dtype=np.int64) - np.repeat(new_cp[:-1], new_lens)  # position in the new column
    src = np.repeat(cp[1:][::-1] - 1, new_lens) - k                           # old entry, walked backwards
    return CscMatrix(n=n, col_ptr=new_cp, row_idx=(n - 1) - ri[src], values=va[src])


def solve_upper(u: CscMatrix, b, *, precision: str = "exact", executor: str = "auto", device: int | None = None):
    """``U x = b`` for upper-triangular ``u`` on the GPU (reversal to a lower solve)."""
    b = np.asarray(b, dtype=np.float64)
    if b.shape != (u.n,):
        raise DimensionMismatch(f"rhs has shape {b.shape}, matrix is {u.n}x{u.n}")
    if u.n == 0:
        return np.zeros(0)
    lr = _reversed_cache(u)
    dev = _native.env_device() if device is None else device
    plan = _native.plan_for(lr, precision=precision, executor=executor, device=dev)
    xr, _ = plan.solve(np.ascontiguousarray(b[::-1]))
    return xr[::-1].copy()


def solve_many(l: CscMatrix, bs, *, precision: str = "exact", executor: str = "auto", device: int | None = None):
    """``L X = B`` for the columns of ``bs`` (n x k) through one cached device
    plan and one native call (``sptrsv_solve_many``): the 2D stencil executor
    solves up to 16 right-hand sides per launch, stacked into one grid (its
    64-band wavefront leaves most of the 148 SMs idle), every other executor
    solves them back to back on the device. Each column's x is what ``solve``
    gives for it (bitwise in exact mode)."""
    bs = np.asarray(bs, dtype=np.float64)
    if bs.ndim != 2 or bs.shape[0] != l.n:
        raise DimensionMismatch(f"rhs block has shape {bs.shape}, matrix is {l.n}x{l.n}")
    if bs.shape[1] == 0 or l.n == 0:
        return np.zeros_like(bs)
    dev = _native.env_device() if device is None else device
    plan = _native.plan_for(l, precision=precision, executor=executor, device=dev)
    x, _ = plan.solve_many(np.ascontiguousarray(bs.T))
    return np.ascontiguousarray(x.T)


_rev: dict = {}


def _reversed_cache(u: CscMatrix) -> CscMatrix:
    hit = _rev.get(id(u))
    if hit is not None and hit[0] is u:
        return hit[1]
    lr = reverse_upper(u)
    if len(_rev) > 8:
        _rev.clear()
    _rev[id(u)] = (u, lr)
    return lr
