"""GPU: the read-only inter-PE layer with every PE's segment on one device.

Same kernel code as one-process-per-GPU (bench.py under torchrun), with the
peer segments local: components are published only into their owner's
segment and read from there. Pull solves are order-independent, so exact mode
stays bit-identical to the serial oracle for every partition.
"""

from __future__ import annotations

import numpy as np
import pytest

import oracle
import paper_2012_06959_b200 as sp
from paper_2012_06959_b200 import _native, synth
from conftest import REFERENCE_CASES, case_matrix

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n_pes", [2, 3, 8])
@pytest.mark.parametrize("kind", ["block", "round-robin"])
@pytest.mark.parametrize("shape", ["lap2d", "banded", "rmat", "random"])
def test_partitioned_pes_bit_exact(n_pes, kind, shape):
    l = {
        "lap2d": lambda: synth.lap2d(64, 48),
        "banded": lambda: synth.banded(6000, 64, 0.5, 4),
        "rmat": lambda: synth.rmat(13, 8, 2),
        "random": lambda: synth.random_lower(2500, 0.02, 9, dominant=True),
    }[shape]()
    b = np.random.default_rng(n_pes).uniform(-1.0, 1.0, l.n)
    plan = sp.block_partition(l.n, n_pes) if kind == "block" else sp.task_round_robin_partition(l.n, n_pes, 4)
    cfg = sp.SolverConfig(engine=sp.Engine.PARTITIONED_READ_ONLY, n_pes=n_pes, precision="exact")
    x, report = sp.solve_partitioned(l, b, plan, cfg)
    ref = oracle.solve_serial(l.col_ptr, l.row_idx, l.values, b)
    assert x.tobytes() == ref.tobytes()
    assert report.totals()["components_solved"] == l.n
    assert report.totals()["local_updates"] + report.totals()["remote_updates"] == l.nnz - l.n
    if report.device.get("pe_mode") != "shared-segment":
        # the kernel really read across segments
        assert report.device["remote_reads"] > 0


@pytest.mark.parametrize("n_pes", [2, 3, 8])
@pytest.mark.parametrize("shape", ["lap2d", "banded", "rmat", "random"])
def test_partitioned_pool_segments_bit_exact(n_pes, shape):
    """executor="rows": the component pool with one published segment per PE."""
    l = {
        "lap2d": lambda: synth.lap2d(64, 48),
        "banded": lambda: synth.banded(6000, 64, 0.5, 4),
        "rmat": lambda: synth.rmat(13, 8, 2),
        "random": lambda: synth.random_lower(2500, 0.02, 9, dominant=True),
    }[shape]()
    b = np.random.default_rng(n_pes).uniform(-1.0, 1.0, l.n)
    plan = sp.task_round_robin_partition(l.n, n_pes, 4)
    cfg = sp.SolverConfig(engine=sp.Engine.PARTITIONED_READ_ONLY, n_pes=n_pes, precision="exact", executor="rows")
    x, report = sp.solve_partitioned(l, b, plan, cfg)
    assert x.tobytes() == oracle.solve_serial(l.col_ptr, l.row_idx, l.values, b).tobytes()
    assert report.device["executor"] == "rows" and report.device["remote_reads"] > 0


@pytest.mark.parametrize("precision", ["exact", "fast"])
@pytest.mark.parametrize("n_pes", [2, 4])
def test_dropin_n_pes_keeps_the_wavefront(n_pes, precision):
    """SolverConfig.n_pes > 1 through the drop-in solve(): a 2D five-point L with
    whole 64-row bands per PE keeps the stencil executor (one plan per PE,
    peers' mailboxes), and x equals the oracle bitwise in exact mode. In fast
    mode (lap2d: error contraction 1/3 per grid row) every PE enters its
    bands through local halo bands, so it reads nothing from its peers."""
    l = synth.lap2d(256, 512)  # 8 bands: whole bands per PE for 2 and 4 PEs
    b = np.random.default_rng(5).uniform(-1.0, 1.0, l.n)
    plan = sp.block_partition(l.n, n_pes)
    cfg = sp.SolverConfig(engine=sp.Engine.PARTITIONED_READ_ONLY, n_pes=n_pes, precision=precision)
    ref = oracle.solve_serial(l.col_ptr, l.row_idx, l.values, b)
    for _ in range(2):
        x, report = sp.solve(l, b, plan, cfg)
        assert report.device["executor"] == "stencil"
        assert report.device["pe_mode"] in ("stencil-pes", "pe-per-gpu")
        if precision == "exact":
            assert x.tobytes() == ref.tobytes()
        else:
            assert sp.compare_solutions(x, ref, 1e-12).within_tol
        if precision == "exact":
            assert report.device["remote_reads"] > 0
        else:
            assert report.device["remote_reads"] == 0
        assert report.totals()["components_solved"] == l.n


@pytest.mark.parametrize("n_pes", [2, 3, 4])
@pytest.mark.parametrize("n", [7680, 7710, 40000])
def test_dropin_n_pes_band_blocks_partitioned(n_pes, n):
    """Fast mode, banded L, contiguous slabs on 64-row block boundaries: one
    band-block plan per PE (its blocks' sweeps and its stretch of the tail
    chain, the chain handed PE to PE through a 64-value slot); x within 1e-12
    of the oracle over repeated solves (slot halves alternate by parity).
    n = 7710: the last PE's last block is partial. n = 40000: every PE has
    >= 64 chain steps, so each runs its stretch by superblocks (K2a/b/c) and
    its superblock chain enters from the previous PE's slot."""
    l = synth.banded(n, 64, 0.5, 6)
    plan = sp.nnz_block_partition(np.ones(n), n_pes, 64)
    cfg = sp.SolverConfig(engine=sp.Engine.PARTITIONED_READ_ONLY, n_pes=n_pes, precision="fast")
    for seed in range(3):
        b = np.random.default_rng(seed).uniform(-1.0, 1.0, l.n)
        x, report = sp.solve(l, b, plan, cfg)
        assert report.device["executor"] == "band"
        assert report.device["pe_mode"] in ("band-pes", "pe-per-gpu")
        ref = oracle.solve_serial(l.col_ptr, l.row_idx, l.values, b)
        assert sp.compare_solutions(x, ref, 1e-12).within_tol
        assert report.totals()["components_solved"] == l.n


def test_dropin_n_pes_structured_executors_stay_fast():
    """Executors without a per-PE mode (band window, 3D wavefront) keep running
    on one device instead of falling back to the component pool."""
    for l, ex in ((synth.banded(20000, 64, 0.5, 1), "band"), (synth.lap3d(24), "stencil")):
        b = np.random.default_rng(2).uniform(-1.0, 1.0, l.n)
        ref = oracle.solve_serial(l.col_ptr, l.row_idx, l.values, b)
        for precision in ("exact", "fast"):
            # (block_partition(20000, 4): 5000-row slabs, off the band blocks' 64-row grid)
            cfg = sp.SolverConfig(engine=sp.Engine.PARTITIONED_READ_ONLY, n_pes=4, precision=precision)
            x, report = sp.solve(l, b, sp.block_partition(l.n, 4), cfg)
            assert report.device["executor"] == ex
            if precision == "exact":
                assert x.tobytes() == ref.tobytes()
            else:
                assert sp.compare_solutions(x, ref, 1e-12).within_tol


@pytest.mark.parametrize("name", ["worked_3x3", "random_3", "bidiagonal1000", "blockdiag4096"])
def test_reference_cases_over_four_pes(name):
    c = REFERENCE_CASES[name]
    l = case_matrix(c)
    n_pes = min(4, l.n)
    plan = sp.task_round_robin_partition(l.n, n_pes, 1)
    for engine in (sp.Engine.PARTITIONED_READ_ONLY, sp.Engine.SHARED_ATOMICS):
        cfg = sp.SolverConfig(engine=engine, n_pes=n_pes)
        x, _ = sp.solve(l, c["b"], plan, cfg)
        assert x.tobytes() == c["x"].tobytes()


def test_partition_fast_mode_and_repeat():
    l = synth.lap3d(16)
    plan = sp.block_partition(l.n, 4)
    cfg = sp.SolverConfig(engine=sp.Engine.PARTITIONED_READ_ONLY, n_pes=4, precision="fast")
    ref = oracle.solve_serial(l.col_ptr, l.row_idx, l.values, np.ones(l.n))
    for _ in range(3):
        x, _ = sp.solve_partitioned(l, np.ones(l.n), plan, cfg)
        assert sp.compare_solutions(x, ref, 1e-12).within_tol


def test_capture_state_identities_partitioned():
    l = synth.random_lower(300, 0.05, 3)
    b = np.random.default_rng(1).uniform(-2, 2, l.n)
    plan = sp.task_round_robin_partition(l.n, 4, 2)
    cfg = sp.SolverConfig(engine=sp.Engine.PARTITIONED_READ_ONLY, n_pes=4, capture_state=True)
    x, report = sp.solve_partitioned(l, b, plan, cfg)
    st = report.state
    np.testing.assert_array_equal(st.d_in_degree + 1, np.sum(st.s_in_degree, axis=0))
    diag = l.values[l.col_ptr[:-1]] * x
    expected = sp.spmv_lower(l, x) - diag
    got = st.d_left_sum + np.sum(st.s_left_sum, axis=0)
    assert np.all(np.abs(got - expected) <= 1e-12 * (1.0 + np.abs(expected)))
    for pe in range(4):
        for i in plan.components_of(pe):
            assert st.s_left_sum[pe][i] == 0.0


def test_native_partition_api_errors():
    l = synth.lap2d(8)
    p = _native.NativePlan(l.col_ptr, l.row_idx, l.values, l.n, executor="rows")
    with pytest.raises(sp.errors.InvalidPeCount if hasattr(sp, "errors") else Exception):
        p.set_partition(np.zeros(l.n), 0)
    with pytest.raises(Exception):
        p.set_partition(np.full(l.n, 5), 2)
    p.close()


def _band_owner_map(l, nx, pes, kind):
    bands = (l.n // nx + 63) // 64
    band = np.arange(l.n) // (64 * nx)
    if kind == "block":
        return (band * pes // bands).astype(np.int32)
    return (band % pes).astype(np.int32)


@pytest.mark.parametrize("precision", ["exact", "fast"])
@pytest.mark.parametrize("pes,kind", [(2, "block"), (3, "block"), (3, "round-robin")])
def test_stencil_partition_plans_on_one_device(pes, kind, precision):
    """One plan per PE (as one process per GPU would hold), wired by device
    pointer on one GPU: each solves its own bands concurrently, polling the
    band above a PE boundary from the peer's mailboxes (exact mode; fast mode
    enters each band through a local halo band and reads nothing remote).
    Repeated solves exercise the parity double-buffer of the mailboxes."""
    torch = pytest.importorskip("torch")
    nx, ny = 128, 64 * 6 - 17  # last band partial
    l = synth.lap2d(nx, ny)
    rng = np.random.default_rng(pes)
    vals = l.values.copy()
    off = l.row_idx != l.entry_columns()
    vals[off] = rng.uniform(-1.0, 1.0, off.sum())
    l = sp.CscMatrix(n=l.n, col_ptr=l.col_ptr, row_idx=l.row_idx, values=vals)
    owner = _band_owner_map(l, nx, pes, kind)
    plans = [_native.NativePlan(l.col_ptr, l.row_idx, l.values, l.n, precision=precision, executor="stencil")
             for _ in range(pes)]
    for p in range(pes):
        plans[p].set_partition(owner, pes, p)
    for p in range(pes):
        for q in range(pes):
            if p != q:
                plans[p].set_peer_segment(q, plans[q].segment_ptr())
    streams = [torch.cuda.Stream() for _ in range(pes)]
    for rep in range(3):
        b = rng.uniform(-1.0, 1.0, l.n)
        ref = oracle.solve_serial(l.col_ptr, l.row_idx, l.values, b)
        db = torch.from_numpy(b).cuda()
        dxs = [torch.full_like(db, float("nan")) for _ in range(pes)]
        torch.cuda.synchronize()
        for p in range(pes):
            plans[p].solve_device_async(db.data_ptr(), dxs[p].data_ptr(), streams[p].cuda_stream)
        stats = [pl.synchronize() for pl in plans]
        torch.cuda.synchronize()
        x = np.full(l.n, np.nan)
        for p in range(pes):
            mine = owner == p
            x[mine] = dxs[p].cpu().numpy()[mine]
        if precision == "exact":
            assert x.tobytes() == ref.tobytes()
        else:
            assert np.max(np.abs(x - ref) / np.maximum(np.abs(ref), 1.0)) <= 1e-12
        if precision == "exact":
            assert sum(st["remote_reads"] for st in stats) > 0
        else:  # diagonally dominant: every PE enters its bands through local halo bands
            assert sum(st["remote_reads"] for st in stats) == 0
        assert all(st["executor"] == "stencil" for st in stats)
    for pl in plans:
        pl.close()


def test_stencil_partition_falls_back_when_bands_split():
    l = synth.lap2d(64, 128)  # 2 bands; split the first one between PEs
    owner = np.zeros(l.n, dtype=np.int32)
    owner[l.n // 4:] = 1
    plan = _native.NativePlan(l.col_ptr, l.row_idx, l.values, l.n, precision="exact", executor="auto")
    plan.set_partition(owner, 2, 0)
    assert plan.info()["executor"] == "rows"
    plan.close()


def test_per_pe_counters_are_measured_by_each_pes_kernel():
    """With one plan per PE (PeGroup), SolveReport.per_pe carries each PE
    kernel's own counters (sptrsv_plan_last_counters): remote_reads_issued is
    the number of cross-PE dependency loads the kernel issued -- one per
    entry (i, j) with owner(i) = p != owner(j) -- and lock_wait_spins its own
    polls, no longer all booked to PE 0 (reference PeStats, engine.py:100-111)."""
    l = synth.rmat(12, 8, 5)
    b = np.random.default_rng(1).uniform(-1, 1, l.n)
    part = sp.task_round_robin_partition(l.n, 3, 4)
    cfg = sp.SolverConfig(engine=sp.Engine.PARTITIONED_READ_ONLY, n_pes=3, precision="exact", executor="rows")
    x, rep = sp.solve(l, b, part, cfg)
    assert x.tobytes() == oracle.solve_serial(l.col_ptr, l.row_idx, l.values, b).tobytes()
    cols = l.entry_columns()
    off = l.row_idx != cols
    own = part.owner_arr
    rows, cols = l.row_idx[off], cols[off]
    cross = own[rows] != own[cols]
    expect = np.bincount(own[rows][cross], minlength=3)
    assert [s.remote_reads_issued for s in rep.per_pe] == expect.tolist()
    assert sum(s.lock_wait_spins for s in rep.per_pe) >= 0
