"""CPU check of the bound behind the fast-mode halo bands / z-tiles (DESIGN.md
section 2): a lower-triangular grid solve started from a zero row (plane)
instead of the true one errs by at most gamma^k times the boundary's
magnitude k rows (planes) later, gamma = U / (1 - A) in 2D and
W / (1 - A - U) in 3D. Restated with scipy on small grids; no GPU."""

from __future__ import annotations

import numpy as np
import pytest
import scipy.sparse as sps
from scipy.sparse.linalg import spsolve_triangular

from paper_2012_06959_b200 import synth


def _csr(l):
    return sps.csc_matrix((l.values, l.row_idx, l.col_ptr), shape=(l.n, l.n)).tocsr()


@pytest.mark.parametrize("nx,rows", [(48, 40), (96, 24)])
def test_2d_halo_error_contracts_by_gamma_per_row(nx, rows):
    ny = 2 * rows
    L = _csr(synth.lap2d(nx, ny))
    b = np.random.default_rng(0).uniform(-1.0, 1.0, L.shape[0])
    x = spsolve_triangular(L, b, lower=True)
    # rows [rows, ny) solved alone: the row above (rows - 1) taken as zero
    lo = rows * nx
    xh = spsolve_triangular(L[lo:, lo:].tocsr(), b[lo:], lower=True)
    err = np.abs(xh - x[lo:]).reshape(ny - rows, nx).max(axis=1)
    gamma = 0.25 / (1.0 - 0.25)  # lap2d: |a| = |u| = 1/4
    bound = np.abs(x[lo - nx:lo]).max() * gamma ** np.arange(1, ny - rows + 1)
    # (plus the two solves' own rounding, a few ulp of |x|)
    assert np.all(err <= bound * (1 + 1e-9) + 1e-15 * np.abs(x).max())


def test_3d_halo_error_contracts_by_gamma_per_plane():
    nx, ny, nz = 12, 10, 24
    L = _csr(synth.lap3d(nx, ny, nz))
    b = np.random.default_rng(1).uniform(-1.0, 1.0, L.shape[0])
    x = spsolve_triangular(L, b, lower=True)
    z0, plane = 8, nx * ny
    lo = z0 * plane
    xh = spsolve_triangular(L[lo:, lo:].tocsr(), b[lo:], lower=True)
    err = np.abs(xh - x[lo:]).reshape(nz - z0, plane).max(axis=1)
    gamma = (1 / 6) / (1.0 - 2 / 6)  # lap3d: |a| = |u| = |w| = 1/6
    bound = np.abs(x[lo - plane:lo]).max() * gamma ** np.arange(1, nz - z0 + 1)
    assert np.all(err <= bound * (1 + 1e-9) + 1e-15 * np.abs(x).max())
