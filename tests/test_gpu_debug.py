"""GPU: SolverConfig.debug -> device checks of the publication protocol
(SPTRSV_PLAN_DEBUG), the reference's debug assertions (engine.py:154-169
write locality, 510-513 counters only move forward) restated for pull
solves: every published x slot / mailbox word is written once, over its
sentinel, by the PE that owns it. Clean solves pass the checks bit-exactly;
an injected double publication raises AssertionError."""

from __future__ import annotations

import numpy as np
import pytest

import oracle
import paper_2012_06959_b200 as sp
from paper_2012_06959_b200 import _native, synth

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("executor,mat", [
    ("rows", lambda: synth.rmat(12, 8, 1)),
    ("stencil", lambda: synth.lap2d(256, 200)),
])
@pytest.mark.parametrize("precision", ["exact", "fast"])
def test_debug_solves_pass_the_checks(executor, mat, precision):
    l = mat()
    b = np.random.default_rng(2).uniform(-1, 1, l.n)
    ref = oracle.solve_serial(l.col_ptr, l.row_idx, l.values, b)
    plan = sp.block_partition(l.n, 1)
    cfg = sp.SolverConfig(engine=sp.Engine.PARTITIONED_READ_ONLY, precision=precision, executor=executor, debug=True)
    for _ in range(2):  # the second solve uses the other mailbox / sentinel half
        x, rep = sp.solve(l, b, plan, cfg)
        assert rep.device["executor"] == executor
        if precision == "exact":
            assert x.tobytes() == ref.tobytes()
        else:
            assert sp.compare_solutions(x, ref, 1e-12).within_tol


def test_debug_partitioned_pes_pass_the_checks():
    # several PEs: each writes only its own segment (write locality)
    l = synth.rmat(12, 8, 3)
    b = np.random.default_rng(4).uniform(-1, 1, l.n)
    ref = oracle.solve_serial(l.col_ptr, l.row_idx, l.values, b)
    for part in (sp.block_partition(l.n, 3), sp.task_round_robin_partition(l.n, 4, 8)):
        cfg = sp.SolverConfig(engine=sp.Engine.PARTITIONED_READ_ONLY, n_pes=part.n_pes, precision="exact",
                              executor="rows", debug=True)
        x, _ = sp.solve(l, b, part, cfg)
        assert x.tobytes() == ref.tobytes()


def test_injected_double_publication_raises_assertion():
    l = synth.rmat(10, 8, 0)
    b = np.ones(l.n)
    plan = _native.NativePlan(l.col_ptr, l.row_idx, l.values, l.n, precision="exact", executor="rows", debug=True,
                              probe_flags=1024)  # fault injection: row 0 published twice
    with pytest.raises(AssertionError, match="component 0"):
        plan.solve(b)
    plan.close()
    # the same injection without debug checks is not detected (and harmless: same value)
    plan = _native.NativePlan(l.col_ptr, l.row_idx, l.values, l.n, precision="exact", executor="rows",
                              probe_flags=1024)
    x, _ = plan.solve(b)
    assert x.tobytes() == oracle.solve_serial(l.col_ptr, l.row_idx, l.values, b).tobytes()
    plan.close()
