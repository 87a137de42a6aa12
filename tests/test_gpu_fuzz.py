"""GPU: seeded random sweep over shapes, densities, bandwidths and executors
against the C oracle: exact bitwise (integer levels / in-degrees too), fast
and push within the 1e-12 contract on the diagonally dominant draws. Ragged
sizes (n not a multiple of a warp, a ticket or a band), empty columns, single
rows and heavy rows are all drawn.
"""

from __future__ import annotations

import numpy as np
import pytest

import oracle
import paper_2012_06959_b200 as sp
from paper_2012_06959_b200 import _native, synth

pytestmark = pytest.mark.gpu

TOL = 1e-12


def _case(seed):
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.choice([1, 2, 31, 33, 64, 65, 257, 1000, 3001, 7777]))
    density = float(rng.choice([0.0, 0.001, 0.01, 0.2, 0.9]))
    bw = None if rng.random() < 0.5 else int(rng.integers(1, 96))
    if n > 1000 and bw is None:
        density = min(density, 0.01)
    dominant = bool(rng.random() < 0.5)
    l = synth.random_lower(n, density, seed, bandwidth=bw, dominant=dominant)
    b = rng.uniform(-1.0, 1.0, n)
    return l, b, dominant


@pytest.mark.parametrize("seed", range(24))
def test_random_sweep(seed):
    l, b, dominant = _case(seed)
    ref = oracle.solve_serial(l.col_ptr, l.row_idx, l.values, b)
    lv, nl = oracle.levels(l.col_ptr, l.row_idx)
    sched = sp.compute_level_schedule(l)
    assert sched.n_levels == nl and np.array_equal(sched.level_of, lv)
    assert np.array_equal(sp.compute_in_degrees(l), oracle.in_degrees(l.col_ptr, l.row_idx))
    for executor in ("auto", "rows", "chains"):
        plan = _native.NativePlan(l.col_ptr, l.row_idx, l.values, l.n, precision="exact", executor=executor)
        x, _ = plan.solve(b)
        plan.close()
        assert x.tobytes() == ref.tobytes(), (seed, executor)
    if not dominant:
        # re-associated sums (fast: pre-scaled FMAs; push: atomics in any
        # order) meet the 1e-12 contract on well-conditioned systems; the
        # non-dominant draws grow like 1e200 and amplify rounding differences
        return
    for executor, precision in (("auto", "fast"), ("push", "exact")):
        plan = _native.NativePlan(l.col_ptr, l.row_idx, l.values, l.n, precision=precision, executor=executor)
        x, _ = plan.solve(b)
        plan.close()
        assert sp.compare_solutions(x, ref, TOL).within_tol, (seed, executor, precision)


def _random_coefficients(l, seed):
    """Random off-diagonals, diagonally dominant diagonal of random sign."""
    rng = np.random.default_rng(seed)
    vals = l.values.copy()
    off = l.row_idx != l.entry_columns()
    vals[off] = rng.uniform(-1.0, 1.0, off.sum())
    dom = 1.0 + np.bincount(l.row_idx[off], weights=np.abs(vals[off]), minlength=l.n)
    vals[~off] = np.where(rng.random(l.n) < 0.5, -1.0, 1.0) * dom
    return sp.CscMatrix(n=l.n, col_ptr=l.col_ptr, row_idx=l.row_idx, values=vals)


@pytest.mark.parametrize("seed", range(16))
def test_random_stencil_grids(seed):
    """Random 2D / 3D grid sizes (the stencil executors when the shape allows)."""
    rng = np.random.default_rng(2000 + seed)
    if seed % 2 == 0:
        grid = synth.lap2d(2 * int(rng.integers(1, 160)), int(rng.integers(1, 300)))
    else:
        grid = synth.lap3d(2 * int(rng.integers(1, 24)), int(rng.integers(1, 70)), int(rng.integers(1, 12)))
    l = _random_coefficients(grid, seed)
    b = rng.uniform(-1.0, 1.0, l.n)
    ref = oracle.solve_serial(l.col_ptr, l.row_idx, l.values, b)
    used = set()
    for precision in ("exact", "fast"):
        plan = _native.NativePlan(l.col_ptr, l.row_idx, l.values, l.n, precision=precision, executor="stencil")
        used.add(plan.info()["executor"])
        for _ in range(2):
            x, _ = plan.solve(b)
            if precision == "exact":
                assert x.tobytes() == ref.tobytes(), (seed, plan.info()["executor"])
            else:
                assert sp.compare_solutions(x, ref, TOL).within_tol, (seed, plan.info()["executor"])
        plan.close()
    assert used == {"stencil"}
