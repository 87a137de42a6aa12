"""Parity at the BASELINE.json sizes, through the drop-in API and the C ABI.

Every check compares the CUDA path with the C oracle (``oracle/``, pinned to
reference-run goldens), never with the GPU itself:

* lap2d-4096 (16.8 M rows, the headline): exact bitwise, fast within 1e-12,
  in-degrees and levels element-wise bit-exact.
* lap3d-128 (2.1 M rows): the same four checks.
* rmat-4M (4.2 M rows, power law): exact bitwise through the ``rows``
  executor (component pool) and ``auto``, fast within 1e-12, in-degrees and
  levels element-wise bit-exact.
* banded-8M (8.4 M rows, bandwidth 64, 277 M entries): exact bitwise over the
  whole vector (the band executor), fast within 1e-12, the leading-block
  prefix property (x[:k] of the full solve equals the oracle's solve of the
  leading k x k block, bitwise: a lower-triangular solve's prefix depends only
  on its leading block), and the full-size residuals.

The right-hand side is the reference CLI's random one,
``default_rng((seed, 1)).uniform(-1, 1)`` (cli.py:141-142), seed 0; the
benchmark's all-ones b is covered by bench.py's correctness leg.
Bars: reference.py:20-35 (solve_serial), analysis.py:19-64 (in-degrees,
levels), north star (1e-12 in fp64).
"""

from __future__ import annotations

import numpy as np
import pytest

import oracle
import paper_2012_06959_b200 as sp
from paper_2012_06959_b200 import _native, synth

pytestmark = pytest.mark.gpu

FAST_TOL = 1e-12


class _Case:
    def __init__(self, name: str):
        self.name = name
        self.l = synth.config_matrix(name)
        self.b = np.random.default_rng((0, 1)).uniform(-1.0, 1.0, self.l.n)
        self._x = None

    @property
    def x_ref(self) -> np.ndarray:
        if self._x is None:
            self._x = oracle.solve_serial(self.l.col_ptr, self.l.row_idx, self.l.values, self.b)
        return self._x


_CASES: dict[str, _Case] = {}


def case(name: str) -> _Case:
    # one at a time: banded-8M alone holds ~4.4 GB of host arrays
    if name not in _CASES:
        _CASES.clear()
        _CASES[name] = _Case(name)
    return _CASES[name]


def _plan(c: _Case, precision: str, executor: str = "auto") -> _native.NativePlan:
    return _native.NativePlan(c.l.col_ptr, c.l.row_idx, c.l.values, c.l.n, precision=precision,
                              executor=executor, timeout=120.0)


def _check_analysis(c: _Case) -> None:
    np.testing.assert_array_equal(sp.compute_in_degrees(c.l), oracle.in_degrees(c.l.col_ptr, c.l.row_idx))
    lv_ref, nl_ref = oracle.levels(c.l.col_ptr, c.l.row_idx)
    p = _native.NativePlan(c.l.col_ptr, c.l.row_idx, None, c.l.n, structure_only=True, timeout=120.0)
    try:
        level_of, order, level_ptr, nl = p.levels()
    finally:
        p.close()
    assert nl == nl_ref
    np.testing.assert_array_equal(level_of, lv_ref)
    # levels[k] = the level-k components ascending (analysis.py:36-37): a stable sort by level
    np.testing.assert_array_equal(order, np.argsort(lv_ref, kind="stable"))
    np.testing.assert_array_equal(level_ptr, np.concatenate(([0], np.cumsum(np.bincount(lv_ref, minlength=nl)))))


def _check_exact(c: _Case, executor: str = "auto", expect: str | None = None) -> None:
    p = _plan(c, "exact", executor)
    try:
        x, st = p.solve(c.b)
    finally:
        p.close()
    if expect:
        assert st["executor"] == expect
    assert x.tobytes() == c.x_ref.tobytes(), sp.compare_solutions(x, c.x_ref, 1e-300)


def _check_fast(c: _Case, expect: str | None = None) -> np.ndarray:
    p = _plan(c, "fast")
    try:
        x, st = p.solve(c.b)
    finally:
        p.close()
    if expect:
        assert st["executor"] == expect
    cmp = sp.compare_solutions(x, c.x_ref, FAST_TOL)
    assert cmp.within_tol, cmp
    return x


@pytest.mark.parametrize("name,executor", [("lap2d-4096", "stencil"), ("lap3d-128", "stencil")])
def test_grid_baseline_exact_fast_levels(name, executor):
    c = case(name)
    _check_exact(c, "auto", executor)
    _check_fast(c, executor)
    _check_analysis(c)


def test_rmat_4m_baseline():
    c = case("rmat-4M")
    _check_exact(c, "rows", "rows")
    _check_fast(c)
    _check_analysis(c)


def test_banded_8m_baseline():
    c = case("banded-8M")
    l = c.l
    x_fast = _check_fast(c, "band")
    assert sp.residual_norm(l, x_fast, c.b)[1] <= 1e-13
    assert sp.residual_norm_2(l, x_fast, c.b) <= 1e-13
    p = _plan(c, "exact")
    try:
        x, st = p.solve(c.b)
    finally:
        p.close()
    assert st["executor"] == "band"
    # leading-block prefix: x[:k] depends only on L[:k, :k] and b[:k]
    k = 1 << 18
    hi = int(l.col_ptr[k])
    keep = l.row_idx[:hi] < k
    cp = np.concatenate(([0], np.cumsum(np.add.reduceat(keep, l.col_ptr[:k]) if hi else np.zeros(k, int))))
    x_lead = oracle.solve_serial(cp, l.row_idx[:hi][keep], l.values[:hi][keep], c.b[:k])
    assert x[:k].tobytes() == x_lead.tobytes()
    # and the whole vector, bitwise
    assert x.tobytes() == c.x_ref.tobytes(), sp.compare_solutions(x, c.x_ref, 1e-300)
    assert sp.residual_norm(l, x, c.b)[1] <= 1e-13
