"""Dependency analysis on the GPU: in-degrees (K1) and level sets (K6).

Same functions and return types as `/root/reference/pkg/src/sptrsv/analysis.py`.
The arithmetic is integer and runs in device kernels (`csrc/preprocess.cu`
``k_in_degree``, `csrc/solve_rows.cu` level mode); results are bit-identical
to the reference, which the test-suite checks against the reference's golden
vectors and the C oracle.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native
from .errors import MatrixStructureError
from .matrix import CscMatrix


def compute_in_degrees(l: CscMatrix) -> np.ndarray:
    """Stored off-diagonal entries per row, int64[n] (analysis.py:19-27).

    Any structurally valid square CSC is accepted, triangular or not; stored
    zeros count.
    """
    if l.n == 0:
        return np.zeros(0, dtype=np.int64)
    return _native.in_degrees_raw(l.col_ptr, l.row_idx, l.n, _native.env_device())


@dataclass(frozen=True)
class LevelSchedule:
    """Earliest-level assignment (analysis.py:30-40)."""

    level_of: np.ndarray
    levels: list[list[int]]
    n_levels: int


def _level_arrays(l: CscMatrix):
    plan = _native.plan_for(l, structure_only=True, device=_native.env_device())
    return plan.levels()


def compute_level_schedule(l: CscMatrix) -> LevelSchedule:
    """Canonical earliest levels, ``level_of[i] = 1 + max level_of[deps]`` (analysis.py:43-64).

    Computed by the device dataflow kernel over (max, +1). Requires every
    stored entry to lie on or below the diagonal (the diagonal itself may be
    missing or zero); an upper entry raises :class:`MatrixStructureError`.
    """
    if l.n == 0:
        return LevelSchedule(level_of=np.zeros(0, dtype=np.int64), levels=[], n_levels=0)
    level_of, order, level_ptr, n_levels = _level_arrays(l)
    bounds = level_ptr.tolist()
    flat = order.tolist()
    levels = [flat[bounds[k]:bounds[k + 1]] for k in range(n_levels)]
    return LevelSchedule(level_of=level_of, levels=levels, n_levels=n_levels)


def parallelism_metric(n_rows: int, n_levels: int) -> int:
    """Components per level, floored (analysis.py:67-69)."""
    return n_rows // n_levels


def dependency_metric(nnz: int, n_rows: int) -> float:
    """Stored entries per component (analysis.py:72-74)."""
    return nnz / n_rows


@dataclass(frozen=True)
class MatrixStats:
    n_rows: int
    nnz: int
    n_levels: int
    parallelism: int
    dependency: float

    def to_json_dict(self, name: str | None = None) -> dict:
        rec = {
            "n_rows": self.n_rows,
            "nnz": self.nnz,
            "n_levels": self.n_levels,
            "parallelism": self.parallelism,
            "dependency": self.dependency,
        }
        return {"name": name, **rec} if name is not None else rec


def compute_stats(l: CscMatrix) -> MatrixStats:
    """Level count and workload metrics (analysis.py:98-106), levels from the GPU."""
    if l.n == 0:
        raise MatrixStructureError("empty matrix has no levels")
    _, _, _, n_levels = _level_arrays(l)
    return MatrixStats(
        n_rows=l.n,
        nnz=l.nnz,
        n_levels=n_levels,
        parallelism=parallelism_metric(l.n, n_levels),
        dependency=dependency_metric(l.nnz, l.n),
    )
