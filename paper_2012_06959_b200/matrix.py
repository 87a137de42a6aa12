"""Host-side sparse matrix carrier and lower-triangular checks.

`CscMatrix` keeps the reference data model unchanged (square CSC, int64 column
pointers and row indices, float64 values, frozen arrays —
`/root/reference/pkg/src/sptrsv/matrix.py:35-88`) so a caller of the reference
can hand the same object to this package. The GPU never sees this object
directly: `paper_2012_06959_b200._native` uploads its three arrays once per
matrix, narrows indices to int32 and builds the device CSR view
(`csrc/preprocess.cu`).

`validate_lower_triangular` / `ensure_lower_triangular` keep the reference's
reporting contract (`matrix.py:133-164`): violations are ordered by
``(col, kind)`` and the first one decides the exception class. The same check
also runs on the device inside plan creation (`csrc/preprocess.cu`,
``k_validate``) so the C ABI rejects bad input on its own.
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

import numpy as np

from .errors import DimensionMismatch, MatrixStructureError, MissingDiagonal, ZeroDiagonal


class DiagonalPolicy(Enum):
    """Extraction behaviour for a column with no stored diagonal (matrix.py:28-32)."""

    REQUIRE_EXPLICIT = "require-explicit"
    INSERT_UNIT = "insert-unit"


def _freeze(arr: np.ndarray) -> np.ndarray:
    arr = np.ascontiguousarray(arr)
    arr.setflags(write=False)
    return arr


@dataclass(frozen=True)
class CscMatrix:
    """Square sparse matrix, compressed by column.

    Column ``j`` owns entries ``col_ptr[j]:col_ptr[j+1]`` of ``row_idx`` /
    ``values`` with strictly increasing rows, so a stored diagonal leads its
    column. Construction only checks structure; triangularity is reported by
    :func:`validate_lower_triangular`.
    """

    n: int
    col_ptr: np.ndarray
    row_idx: np.ndarray
    values: np.ndarray

    def __post_init__(self):
        cp = np.asarray(self.col_ptr, dtype=np.int64)
        ri = np.asarray(self.row_idx, dtype=np.int64)
        va = np.asarray(self.values, dtype=np.float64)
        _check_structure(int(self.n), cp, ri, va)
        object.__setattr__(self, "n", int(self.n))
        object.__setattr__(self, "col_ptr", _freeze(cp))
        object.__setattr__(self, "row_idx", _freeze(ri))
        object.__setattr__(self, "values", _freeze(va))

    @property
    def nnz(self) -> int:
        return int(self.col_ptr[-1])

    def column(self, j: int) -> tuple[np.ndarray, np.ndarray]:
        lo, hi = int(self.col_ptr[j]), int(self.col_ptr[j + 1])
        return self.row_idx[lo:hi], self.values[lo:hi]

    def entry_columns(self) -> np.ndarray:
        """Column of each stored entry, in storage order."""
        return np.repeat(np.arange(self.n, dtype=np.int64), np.diff(self.col_ptr))

    def to_dense(self) -> np.ndarray:
        out = np.zeros((self.n, self.n))
        out[self.row_idx, self.entry_columns()] = self.values
        return out

    @staticmethod
    def from_entries(n: int, entries: dict[tuple[int, int], float]) -> "CscMatrix":
        """Build from ``{(row, col): value}`` (test convenience, matrix.py:78-88)."""
        if entries:
            keys = np.array(list(entries.keys()), dtype=np.int64).reshape(-1, 2)
            vals = np.array(list(entries.values()), dtype=np.float64)
            order = np.lexsort((keys[:, 0], keys[:, 1]))
            rows, cols, vals = keys[order, 0], keys[order, 1], vals[order]
        else:
            rows = cols = np.empty(0, dtype=np.int64)
            vals = np.empty(0)
        counts = np.bincount(cols, minlength=n) if cols.size else np.zeros(n, dtype=np.int64)
        col_ptr = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(counts, out=col_ptr[1:])
        return CscMatrix(n=n, col_ptr=col_ptr, row_idx=rows, values=vals)

    @staticmethod
    def from_csr(n: int, indptr, indices, data) -> "CscMatrix":
        """Accept a lower-triangular CSR triple (e.g. ``scipy.sparse.csr_matrix``).

        The reference has no CSR type; the north star asks the
        drop-in to take CSR too. Rows must have strictly increasing columns.
        The result is the equivalent CSC matrix (a stable counting transpose).
        """
        indptr = np.asarray(indptr, dtype=np.int64)
        indices = np.asarray(indices, dtype=np.int64)
        data = np.asarray(data, dtype=np.float64)
        if indptr.shape != (n + 1,) or indptr[0] != 0 or np.any(np.diff(indptr) < 0):
            raise MatrixStructureError("CSR indptr is malformed")
        nnz = int(indptr[-1])
        if indices.shape != (nnz,) or data.shape != (nnz,):
            raise MatrixStructureError("CSR entry arrays have the wrong length")
        rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(indptr))
        order = np.argsort(indices, kind="stable")  # by column, rows stay ascending
        counts = np.bincount(indices, minlength=n) if nnz else np.zeros(n, dtype=np.int64)
        col_ptr = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(counts, out=col_ptr[1:])
        return CscMatrix(n=n, col_ptr=col_ptr, row_idx=rows[order], values=data[order])


def _check_structure(n: int, col_ptr: np.ndarray, row_idx: np.ndarray, values: np.ndarray) -> None:
    """Structural well-formedness (matrix.py:91-119)."""
    if n < 0:
        raise MatrixStructureError(f"negative dimension {n}")
    if col_ptr.shape != (n + 1,):
        raise MatrixStructureError(f"col_ptr has length {col_ptr.shape[0]}, expected {n + 1}")
    if col_ptr[0] != 0:
        raise MatrixStructureError(f"col_ptr[0] = {col_ptr[0]}, expected 0")
    widths = np.diff(col_ptr)
    if np.any(widths < 0):
        raise MatrixStructureError("col_ptr is not non-decreasing")
    nnz = int(col_ptr[-1])
    if row_idx.shape != (nnz,) or values.shape != (nnz,):
        raise MatrixStructureError(
            f"entry arrays have lengths {row_idx.shape[0]}/{values.shape[0]}, expected {nnz}"
        )
    if nnz and (int(row_idx.min()) < 0 or int(row_idx.max()) >= n):
        raise MatrixStructureError("row index out of range")
    if nnz > 1:
        # a non-increasing step is legal only where a new column starts
        falls = np.flatnonzero(np.diff(row_idx) <= 0) + 1  # entry index that starts the fall
        if falls.size:
            starts = np.zeros(nnz + 1, dtype=bool)
            starts[col_ptr[:-1]] = True
            bad = falls[~starts[falls]]
            if bad.size:
                raise MatrixStructureError(
                    f"rows not strictly increasing within a column near entry {int(bad[0]) - 1}"
                )


@dataclass(frozen=True)
class Violation:
    """One broken lower-triangular invariant (matrix.py:122-130)."""

    kind: str
    col: int

    def __str__(self) -> str:
        return f"{self.kind}(col={self.col})"


def validate_lower_triangular(l: CscMatrix) -> list[Violation]:
    """All solver-input violations, ordered by ``(col, kind)`` (matrix.py:133-151)."""
    cols = l.entry_columns()
    found: list[Violation] = []
    for j in np.unique(cols[l.row_idx < cols]):
        found.append(Violation("UpperTriangularEntry", int(j)))
    on_diag = l.row_idx == cols
    has = np.zeros(l.n, dtype=bool)
    has[cols[on_diag]] = True
    for j in np.flatnonzero(~has):
        found.append(Violation("MissingDiagonal", int(j)))
    for j in cols[on_diag][l.values[on_diag] == 0.0]:
        found.append(Violation("ZeroDiagonal", int(j)))
    found.sort(key=lambda v: (v.col, v.kind))
    return found


def raise_first_violation(found: list[Violation]) -> None:
    if not found:
        return
    first = found[0]
    if first.kind == "ZeroDiagonal":
        raise ZeroDiagonal(first.col)
    if first.kind == "MissingDiagonal":
        raise MissingDiagonal(first.col)
    raise MatrixStructureError(f"not lower triangular: {first}")


def ensure_lower_triangular(l: CscMatrix) -> None:
    """Raise the exception of the first violation (matrix.py:154-164)."""
    raise_first_violation(validate_lower_triangular(l))


def extract_lower_triangular(a: CscMatrix, policy: DiagonalPolicy) -> CscMatrix:
    """Keep ``row >= col`` entries and normalise the diagonal (matrix.py:167-200)."""
    cols = a.entry_columns()
    keep = a.row_idx >= cols
    rows, kcols, vals = a.row_idx[keep], cols[keep], a.values[keep]
    has = np.zeros(a.n, dtype=bool)
    has[kcols[rows == kcols]] = True
    missing = np.flatnonzero(~has)
    if missing.size:
        if policy is DiagonalPolicy.REQUIRE_EXPLICIT:
            raise MissingDiagonal(int(missing[0]))
        rows = np.concatenate([rows, missing])
        kcols = np.concatenate([kcols, missing])
        vals = np.concatenate([vals, np.ones(missing.size)])
        order = np.lexsort((rows, kcols))
        rows, kcols, vals = rows[order], kcols[order], vals[order]
    col_ptr = np.zeros(a.n + 1, dtype=np.int64)
    np.cumsum(np.bincount(kcols, minlength=a.n), out=col_ptr[1:])
    if a.n:
        zero = vals[col_ptr[:-1]] == 0.0
        if np.any(zero):
            raise ZeroDiagonal(int(np.flatnonzero(zero)[0]))
    return CscMatrix(n=a.n, col_ptr=col_ptr, row_idx=rows, values=vals)


def spmv_lower(l: CscMatrix, x: np.ndarray) -> np.ndarray:
    """``L @ x`` accumulated in storage order (matrix.py:203-213); residual helper."""
    x = np.asarray(x, dtype=np.float64)
    if x.shape != (l.n,):
        raise DimensionMismatch(f"vector has shape {x.shape}, matrix is {l.n}x{l.n}")
    return np.bincount(l.row_idx, weights=l.values * x[l.entry_columns()], minlength=l.n)
