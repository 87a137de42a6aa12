"""GPU: the push executor — the paper's shared-atomics solve (Alg. 2; reference
solve_shared_atomics, engine.py:324-431): warp per column, fp64 atomics on
shared left sums and in-degree counters.

Atomic accumulation commutes in arbitrary order, so x matches the serial
oracle to rounding, not bit for bit (the reference engines are themselves
nondeterministic at rounding level): the bar is the north star's
max relative error 1e-12 in both precisions, plus the reference's own exact
known answers where the sums are exact (identity, diagonal, worked 3x3).
"""

from __future__ import annotations

import numpy as np
import pytest

import oracle
import paper_2012_06959_b200 as sp
from paper_2012_06959_b200 import _native, synth
from paper_2012_06959_b200.errors import SolveTimeout
from conftest import REFERENCE_CASES, case_matrix
from test_gpu_parity import MID_SIZE

pytestmark = pytest.mark.gpu

TOL = 1e-12


@pytest.mark.parametrize("precision", ["exact", "fast"])
@pytest.mark.parametrize("name", sorted(n for n in REFERENCE_CASES if "x" in REFERENCE_CASES[n]))
def test_reference_cases(name, precision):
    c = REFERENCE_CASES[name]
    l = case_matrix(c)
    plan = _native.plan_for(l, precision=precision, executor="push", device=0)
    x, st = plan.solve(c["b"])
    assert st["executor"] == "push"
    assert sp.compare_solutions(x, c["x"], TOL).within_tol


@pytest.mark.parametrize("name", sorted(MID_SIZE))
def test_mid_size_within_tolerance(name):
    l = MID_SIZE[name]()
    b = np.random.default_rng(3).uniform(-1.0, 1.0, size=l.n)
    ref = oracle.solve_serial(l.col_ptr, l.row_idx, l.values, b)
    for precision in ("exact", "fast"):
        x, st = _native.plan_for(l, precision=precision, executor="push", device=0).solve(b)
        assert sp.compare_solutions(x, ref, TOL).within_tol, (precision, st)


def test_exact_known_answers():
    # identity -> x = b; diagonal -> b / d bitwise (test_reference.py:14-35)
    n = 1000
    rng = np.random.default_rng(1)
    d = rng.uniform(0.5, 2.0, n)
    l = sp.CscMatrix(n=n, col_ptr=np.arange(n + 1), row_idx=np.arange(n), values=d)
    b = rng.uniform(-1, 1, n)
    x, _ = _native.plan_for(l, precision="exact", executor="push", device=0).solve(b)
    assert x.tobytes() == (b / d).tobytes()


def test_dispatch_through_shared_atomics_engine_and_repeat():
    l = synth.lap2d(96)
    b = np.random.default_rng(5).uniform(-1, 1, l.n)
    ref = oracle.solve_serial(l.col_ptr, l.row_idx, l.values, b)
    plan = sp.task_round_robin_partition(l.n, 4, 2)
    cfg = sp.SolverConfig(engine=sp.Engine.SHARED_ATOMICS, n_pes=4, executor="push", precision="fast")
    xs = []
    for _ in range(3):
        x, rep = sp.solve(l, b, plan, cfg)
        assert rep.device["executor"] == "push"
        assert sp.compare_solutions(x, ref, TOL).within_tol
        xs.append(x)
    # counters/sums are reset per solve: repeated solves agree to rounding
    assert max(np.max(np.abs(a - xs[0])) for a in xs) <= 1e-13


def test_watchdog_on_push():
    # a huge chain with a tiny timeout trips SolveTimeout like the other executors
    l = synth.bidiagonal(400_000)
    b = np.ones(l.n)
    plan = _native.NativePlan(l.col_ptr, l.row_idx, l.values, l.n, precision="exact", executor="push",
                              timeout=2e-4, spin_initial=1, spin_max_ns=64)
    with pytest.raises(SolveTimeout):
        plan.solve(b)
    plan.close()


@pytest.mark.parametrize("name", sorted(MID_SIZE))
def test_managed_push_within_tolerance(name):
    """The Unified-Memory baseline (SPTRSV_PLAN_PUSH_MANAGED: left sums and
    in-degree counters in cudaMallocManaged memory, system-scope atomics,
    PAPER.md:226-232) solves the same systems to the same tolerance."""
    l = MID_SIZE[name]()
    b = np.random.default_rng(5).uniform(-1.0, 1.0, size=l.n)
    ref = oracle.solve_serial(l.col_ptr, l.row_idx, l.values, b)
    plan = _native.NativePlan(l.col_ptr, l.row_idx, l.values, l.n, precision="fast", executor="push",
                              push_managed=True)
    for _ in range(2):  # the shared state is reset between solves
        x, st = plan.solve(b)
        assert st["executor"] == "push"
        assert sp.compare_solutions(x, ref, TOL).within_tol
    plan.close()
