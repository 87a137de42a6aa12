"""Seeded, vectorised generators for the benchmark shapes of BASELINE.json.

The reference ships desk-scale generators only (`synth.py:21-188`) and none of
the benchmark shapes; these are defined in SURVEY.md §8d:

* ``lap2d(nx)``  — lower triangle of the 5-point Laplacian, natural order
  ``i = y*nx + x``: diag 4, -1 at ``i-1`` (x>0) and ``i-nx`` (y>0).
* ``lap3d(nx)``  — 7-point, ``i = (z*nx + y)*nx + x``: diag 6, -1 at
  ``i-1``, ``i-nx``, ``i-nx^2`` when in range.
* ``banded(n, bandwidth, density, seed)`` — RANDOM_BANDED pattern semantics
  (each column j keeps each of rows j+1..j+bandwidth with probability
  ``density``), off-diagonals U(-1,1); the diagonal is made dominant,
  ``±(1 + sum |row off-diagonals|)``, because the reference's |diag| in [1,2)
  overflows at ~32 nnz/row.
* ``rmat(scale, edge_factor, seed)`` — R-MAT (0.57, 0.19, 0.19, 0.05) edges
  folded strictly below the diagonal, deduplicated, dominant diagonal.

Plus the reference's small kinds (diagonal, bidiagonal, block-diagonal) used
by tests. Every generator builds CSC directly with numpy.
"""

from __future__ import annotations

import numpy as np

from .matrix import CscMatrix


def _from_coo_lower(n: int, rows: np.ndarray, cols: np.ndarray, vals: np.ndarray, diag: np.ndarray) -> CscMatrix:
    """CSC from strictly-lower COO entries (any order, no duplicates) plus a full diagonal."""
    r = np.concatenate([np.arange(n, dtype=np.int64), rows.astype(np.int64)])
    c = np.concatenate([np.arange(n, dtype=np.int64), cols.astype(np.int64)])
    v = np.concatenate([diag.astype(np.float64), vals.astype(np.float64)])
    order = np.lexsort((r, c))
    counts = np.bincount(c, minlength=n)
    col_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=col_ptr[1:])
    return CscMatrix(n=n, col_ptr=col_ptr, row_idx=r[order], values=v[order])


def _stencil_lower(n: int, diag_value: float, offsets: list[tuple[int, np.ndarray]]) -> CscMatrix:
    """Constant-coefficient lower stencil: entries (i, i - off) = -1 where mask[i].

    Built column by column without a sort: column j holds its diagonal, then
    rows j + off for ascending offsets whose mask is set.
    """
    offsets = sorted(offsets, key=lambda t: t[0])
    present = []  # present[k][j]: column j has an entry at row j + off_k
    for off, mask in offsets:
        p = np.zeros(n, dtype=bool)
        p[: n - off] = mask[off:]
        present.append(p)
    counts = np.ones(n, dtype=np.int64)
    for p in present:
        counts += p
    col_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=col_ptr[1:])
    nnz = int(col_ptr[-1])
    rows = np.empty(nnz, dtype=np.int64)
    vals = np.empty(nnz)
    j = np.arange(n, dtype=np.int64)
    slot = col_ptr[:-1].copy()
    rows[slot] = j
    vals[slot] = diag_value
    slot += 1
    for (off, _), p in zip(offsets, present):
        cols = j[p]
        rows[slot[p]] = cols + off
        vals[slot[p]] = -1.0
        slot += p
    return CscMatrix(n=n, col_ptr=col_ptr, row_idx=rows, values=vals)


def lap2d(nx: int, ny: int | None = None) -> CscMatrix:
    """5-point lower stencil on an nx-by-ny grid (ny defaults to nx)."""
    ny = nx if ny is None else ny
    n = nx * ny
    i = np.arange(n, dtype=np.int64)
    x = i % nx
    y = i // nx
    return _stencil_lower(n, 4.0, [(1, x > 0), (nx, y > 0)])


def lap3d(nx: int, ny: int | None = None, nz: int | None = None) -> CscMatrix:
    """Lower triangle of the 7-point 3D Laplacian, natural order i = (z*ny + y)*nx + x."""
    ny = nx if ny is None else ny
    nz = nx if nz is None else nz
    n = nx * ny * nz
    i = np.arange(n, dtype=np.int64)
    x = i % nx
    y = (i // nx) % ny
    z = i // (nx * ny)
    return _stencil_lower(n, 6.0, [(1, x > 0), (nx, y > 0), (nx * ny, z > 0)])


def _dominant_diag(n: int, rows: np.ndarray, vals: np.ndarray, rng: np.random.Generator) -> np.ndarray:
    row_abs = np.bincount(rows, weights=np.abs(vals), minlength=n)
    sign = np.where(rng.random(n) < 0.5, -1.0, 1.0)
    return sign * (1.0 + row_abs)


def banded(n: int, bandwidth: int = 64, density: float = 0.5, seed: int = 0) -> CscMatrix:
    """Random banded lower-triangular matrix with a dominant diagonal.

    Built column-major without a sort (one pass per sub-diagonal), so the
    8M-row benchmark shape (~277M entries) generates in seconds.
    """
    rng = np.random.default_rng(seed)
    bw = min(bandwidth, max(n - 1, 0))
    masks = []
    for d in range(1, bw + 1):
        m = np.zeros(n, dtype=bool)  # m[j]: entry (j + d, j) stored
        m[: n - d] = rng.random(n - d) < density
        masks.append(m)
    counts = np.ones(n, dtype=np.int64)
    for m in masks:
        counts += m
    col_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=col_ptr[1:])
    nnz = int(col_ptr[-1])
    rows = np.empty(nnz, dtype=np.int64)
    vals = np.empty(nnz)
    j = np.arange(n, dtype=np.int64)
    slot = col_ptr[:-1].copy()
    rows[slot] = j
    slot += 1
    row_abs = np.zeros(n)
    for d, m in enumerate(masks, start=1):
        cols = j[m]
        v = rng.uniform(-1.0, 1.0, size=cols.size)
        rows[slot[m]] = cols + d
        vals[slot[m]] = v
        np.add.at(row_abs, cols + d, np.abs(v)) if cols.size < 1024 else _add_shifted(row_abs, cols + d, np.abs(v))
        slot += m
    sign = np.where(rng.random(n) < 0.5, -1.0, 1.0)
    vals[col_ptr[:-1]] = sign * (1.0 + row_abs)
    return CscMatrix(n=n, col_ptr=col_ptr, row_idx=rows, values=vals)


def _add_shifted(acc: np.ndarray, idx: np.ndarray, w: np.ndarray) -> None:
    """acc[idx] += w for unique idx (one sub-diagonal hits each row at most once)."""
    acc[idx] += w


def rmat(scale: int, edge_factor: int = 8, seed: int = 0, a=0.57, b=0.19, c=0.19) -> CscMatrix:
    """R-MAT graph folded into a strictly lower triangle, dominant diagonal."""
    rng = np.random.default_rng(seed)
    n = 1 << scale
    m = edge_factor * n
    u = np.zeros(m, dtype=np.int64)
    v = np.zeros(m, dtype=np.int64)
    ab, abc = a + b, a + b + c
    for bit in range(scale):
        r = rng.random(m)
        q = (r >= a).view(np.int8) + (r >= ab).view(np.int8) + (r >= abc).view(np.int8)  # quadrant a,b,c,d = 0..3
        u |= (q >= 2).astype(np.int64) << bit  # quadrants c, d set the row bit
        v |= (q & 1).astype(np.int64) << bit  # quadrants b, d set the column bit
    lo = np.minimum(u, v)
    hi = np.maximum(u, v)
    del u, v
    keep = lo != hi
    key = np.sort(hi[keep] * n + lo[keep])
    del lo, hi, keep
    key = key[np.concatenate(([True], key[1:] != key[:-1]))] if key.size else key  # unique, row-major
    rows = key // n
    cols = key - rows * n
    vals = rng.uniform(-1.0, 1.0, size=rows.size)
    diag = _dominant_diag(n, rows, vals, rng)
    # CSC: entries by (column, row), the diagonal first in each column
    order = np.argsort(cols * n + rows)
    rows, cols, vals = rows[order], cols[order], vals[order]
    counts = 1 + np.bincount(cols, minlength=n)
    col_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=col_ptr[1:])
    nnz = int(col_ptr[-1])
    row_idx = np.empty(nnz, dtype=np.int64)
    values = np.empty(nnz)
    pos = np.arange(rows.size, dtype=np.int64) + cols + 1
    row_idx[pos] = rows
    values[pos] = vals
    row_idx[col_ptr[:-1]] = np.arange(n, dtype=np.int64)
    values[col_ptr[:-1]] = diag
    return CscMatrix(n=n, col_ptr=col_ptr, row_idx=row_idx, values=values)


def diagonal(n: int) -> CscMatrix:
    return CscMatrix(n=n, col_ptr=np.arange(n + 1), row_idx=np.arange(n), values=np.ones(n))


def bidiagonal(n: int) -> CscMatrix:
    """diag 1, subdiagonal -1: one dependency chain of length n."""
    rows = np.arange(1, n, dtype=np.int64)
    return _from_coo_lower(n, rows, rows - 1, np.full(n - 1, -1.0), np.ones(n))


def block_diagonal(n: int, block: int, seed: int = 0) -> CscMatrix:
    """Dense lower blocks on the diagonal, |diag| in [1, 2), off-diagonals U(-1, 1)."""
    rng = np.random.default_rng(seed)
    rows_l, cols_l = [], []
    for start in range(0, n, block):
        end = min(start + block, n)
        r, c = np.tril_indices(end - start, -1)
        rows_l.append(r + start)
        cols_l.append(c + start)
    rows = np.concatenate(rows_l).astype(np.int64)
    cols = np.concatenate(cols_l).astype(np.int64)
    vals = rng.uniform(-1.0, 1.0, size=rows.size)
    diag = np.where(rng.random(n) < 0.5, -1.0, 1.0) * rng.uniform(1.0, 2.0, size=n)
    return _from_coo_lower(n, rows, cols, vals, diag)


def random_lower(n: int, density: float, seed: int, bandwidth: int | None = None, dominant: bool = False) -> CscMatrix:
    """Random lower-triangular test matrix (own RNG stream; not the reference's).

    Off-diagonals U(-1,1) with probability ``density`` inside the band; the
    diagonal is in ±[1,2) like the reference's, or dominant when asked.
    """
    rng = np.random.default_rng(seed)
    bw = n - 1 if bandwidth is None else bandwidth
    rows_l, cols_l = [], []
    for d in range(1, min(bw, n - 1) + 1):
        keep = rng.random(n - d) < density
        cols = np.flatnonzero(keep).astype(np.int64)
        rows_l.append(cols + d)
        cols_l.append(cols)
    rows = np.concatenate(rows_l) if rows_l else np.empty(0, dtype=np.int64)
    cols = np.concatenate(cols_l) if cols_l else np.empty(0, dtype=np.int64)
    vals = rng.uniform(-1.0, 1.0, size=rows.size)
    if dominant:
        diag = _dominant_diag(n, rows, vals, rng)
    else:
        diag = np.where(rng.random(n) < 0.5, -1.0, 1.0) * rng.uniform(1.0, 2.0, size=n)
    return _from_coo_lower(n, rows, cols, vals, diag)


CONFIGS = {
    "lap2d-256": lambda: lap2d(256),
    "lap3d-128": lambda: lap3d(128),
    "banded-8M": lambda: banded(8 * 1024 * 1024, 64, 31 / 64, 0),
    "rmat-4M": lambda: rmat(22, 8, 0),
    "lap2d-4096": lambda: lap2d(4096),
}


def config_matrix(name: str) -> CscMatrix:
    """Named BASELINE.json shape."""
    if name not in CONFIGS:
        raise KeyError(f"unknown config {name!r}; one of {sorted(CONFIGS)}")
    return CONFIGS[name]()
