"""Host-side logic that needs no GPU: data model, partitions, config, ABI surface."""

from __future__ import annotations

import ctypes
import re

import numpy as np
import pytest

import paper_2012_06959_b200 as sp
from paper_2012_06959_b200 import _native, errors, synth
from conftest import ROOT


def test_cscmatrix_structure_checks():
    with pytest.raises(errors.MatrixStructureError):
        sp.CscMatrix(n=2, col_ptr=[0, 1], row_idx=[0], values=[1.0])
    with pytest.raises(errors.MatrixStructureError):
        sp.CscMatrix(n=2, col_ptr=[0, 2, 1], row_idx=[0, 1], values=[1.0, 1.0])
    with pytest.raises(errors.MatrixStructureError):
        sp.CscMatrix(n=2, col_ptr=[0, 2, 2], row_idx=[1, 0], values=[1.0, 1.0])
    with pytest.raises(errors.MatrixStructureError):
        sp.CscMatrix(n=2, col_ptr=[0, 1, 2], row_idx=[0, 2], values=[1.0, 1.0])
    m = sp.CscMatrix(n=2, col_ptr=[0, 2, 3], row_idx=[0, 1, 1], values=[1.0, 2.0, 3.0])
    assert m.nnz == 3 and not m.values.flags.writeable


def test_validate_reports_in_col_kind_order():
    m = sp.CscMatrix.from_entries(3, {(0, 0): 1.0, (0, 1): 5.0, (2, 1): 1.0, (2, 2): 0.0})
    kinds = [(v.col, v.kind) for v in sp.validate_lower_triangular(m)]
    assert kinds == [(1, "MissingDiagonal"), (1, "UpperTriangularEntry"), (2, "ZeroDiagonal")]
    with pytest.raises(errors.MissingDiagonal):
        sp.ensure_lower_triangular(m)


def test_from_csr_roundtrip():
    l = synth.random_lower(50, 0.1, 3)
    dense = l.to_dense()
    rows, cols = np.nonzero(dense)
    order = np.lexsort((cols, rows))
    rows, cols = rows[order], cols[order]
    indptr = np.concatenate([[0], np.cumsum(np.bincount(rows, minlength=50))])
    back = sp.CscMatrix.from_csr(50, indptr, cols, dense[rows, cols])
    np.testing.assert_array_equal(back.to_dense(), dense)


def test_stencil_generators_match_definition():
    l = synth.lap2d(5)
    d = l.to_dense()
    for i in range(25):
        x, y = i % 5, i // 5
        assert d[i, i] == 4.0
        assert d[i, i - 1] == (-1.0 if x > 0 else 0.0) if i > 0 else True
        if y > 0:
            assert d[i, i - 5] == -1.0
    assert l.nnz == 25 + 20 + 20
    l3 = synth.lap3d(4)
    assert l3.nnz == 64 + 3 * 48
    assert np.allclose(np.tril(l3.to_dense()), l3.to_dense())


def test_partition_plans_match_reference_laws():
    p = sp.task_round_robin_partition(10, 2, 2)
    assert [(t.first, t.last_exclusive, t.owner_pe) for t in p.tasks] == [(0, 3, 0), (3, 6, 1), (6, 8, 0), (8, 10, 1)]
    assert p.components_of(0) == [0, 1, 2, 6, 7]
    np.testing.assert_array_equal(sp.block_partition(7, 2).owner_arr, [0, 0, 0, 0, 1, 1, 1])
    with pytest.raises(errors.InvalidPeCount):
        sp.block_partition(8, 9)
    with pytest.raises(errors.TooManyTasks):
        sp.task_round_robin_partition(8, 2, 5)
    rng = np.random.default_rng(4242)
    for _ in range(200):
        n = int(rng.integers(1, 3000))
        P = int(rng.integers(1, min(n, 16) + 1))
        T = int(rng.integers(1, max(n // P, 1) + 1))
        plan = sp.task_round_robin_partition(n, P, T)
        cover = np.zeros(n, dtype=int)
        for t in plan.tasks:
            assert t.owner_pe == t.task_id % P and t.first < t.last_exclusive
            cover[t.first:t.last_exclusive] += 1
        assert np.all(cover == 1)
        np.testing.assert_array_equal(sp.task_round_robin_partition(n, P, 1).owner_arr, sp.block_partition(n, P).owner_arr)


def test_reduce_contributions_order():
    vals = [0.1, 0.2, 0.3, 0.4, 0.5]
    assert sp.reduce_contributions(vals) == ((0.1 + 0.2) + (0.3 + 0.4)) + 0.5
    assert sp.reduce_contributions([7]) == 7
    with pytest.raises(ValueError):
        sp.reduce_contributions([])


def test_solver_config_validation():
    with pytest.raises(ValueError):
        sp.SolverConfig(engine=sp.Engine.SHARED_ATOMICS, n_pes=0)
    with pytest.raises(ValueError):
        sp.SolverConfig(engine=sp.Engine.SHARED_ATOMICS, workers_per_pe=0)
    with pytest.raises(ValueError):
        sp.SolverConfig(engine=sp.Engine.SHARED_ATOMICS, timeout=0.0)
    with pytest.raises(ValueError):
        sp.SolverConfig(engine=sp.Engine.SHARED_ATOMICS, precision="half")
    with pytest.raises(ValueError, match="push"):
        sp.SolverConfig(engine=sp.Engine.SHARED_ATOMICS, executor="push", precision="exact")
    sp.SolverConfig(engine=sp.Engine.SHARED_ATOMICS, executor="push", precision="fast")


def test_engine_argument_checks_need_no_gpu(worked_3x3):
    l, b, _ = worked_3x3
    with pytest.raises(ValueError, match="engine"):
        sp.solve_shared_atomics(l, b, sp.block_partition(3, 1), sp.SolverConfig(engine=sp.Engine.PARTITIONED_READ_ONLY))
    with pytest.raises(ValueError, match="PEs"):
        sp.solve_partitioned(l, b, sp.block_partition(3, 2), sp.SolverConfig(engine=sp.Engine.PARTITIONED_READ_ONLY))
    with pytest.raises(errors.DimensionMismatch):
        sp.solve_partitioned(l, np.ones(4), sp.block_partition(3, 1), sp.SolverConfig(engine=sp.Engine.PARTITIONED_READ_ONLY))


def test_compare_and_residual_definitions(worked_3x3):
    l, b, x = worked_3x3
    assert sp.residual_norm(l, x, b) == (0.0, 0.0)
    assert sp.compare_solutions(np.array([1e-10]), np.array([0.0]), 1e-9).within_tol
    cmp = sp.compare_solutions(np.array([2.0]), np.array([1.0]), 1e-9)
    assert cmp.max_rel_error == 1.0 and not cmp.within_tol


def test_status_codes_map_to_reference_classes():
    with pytest.raises(errors.ZeroDiagonal) as e:
        errors.raise_for_status(errors.STATUS_ZERO_DIAGONAL, "", 7)
    assert e.value.col == 7
    with pytest.raises(errors.MissingDiagonal):
        errors.raise_for_status(errors.STATUS_MISSING_DIAGONAL, "", 1)
    with pytest.raises(errors.SolveTimeout):
        errors.raise_for_status(errors.STATUS_TIMEOUT, "x")
    with pytest.raises(AssertionError):  # SolverConfig.debug device checks (engine.py:163-168)
        errors.raise_for_status(errors.STATUS_DEBUG_CHECK, "x")
    errors.raise_for_status(errors.STATUS_OK)


def _header_symbols() -> list[str]:
    text = (ROOT / "include" / "sptrsv_b200.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int|void|const char\*)\s+(sptrsv_\w+)\s*\(", text, re.M)))


def test_library_loads_and_exports_every_header_symbol():
    lib = _native.load_library()
    syms = _header_symbols()
    assert len(syms) >= 12
    for s in syms:
        assert hasattr(lib, s), s
    assert lib.sptrsv_abi_version() == 1
    opt = _native.default_options()
    assert opt.timeout_s == 60.0 and opt.spin_initial == 1024 and opt.spin_max_ns == 64
    assert ctypes.sizeof(_native.Options) == lib.sptrsv_sizeof_options()
    assert ctypes.sizeof(_native.Stats) == lib.sptrsv_sizeof_stats()


def test_no_gpu_means_loud_failure():
    if _native.load_library().sptrsv_device_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(errors.NativeUnavailable):
        sp.solve_serial(synth.diagonal(3), np.ones(3))


def test_reverse_upper_is_a_relabelling():
    """P U P is lower triangular, diagonal first per column, same values."""
    import scipy.sparse as ssp

    rng = np.random.default_rng(3)
    n = 300
    dense = np.triu(rng.uniform(-1, 1, (n, n)) * (rng.random((n, n)) < 0.05))
    dense[np.arange(n), np.arange(n)] = rng.uniform(1, 2, n)
    csc = ssp.csc_matrix(dense)
    csc.sort_indices()
    u = sp.CscMatrix(n=n, col_ptr=csc.indptr.astype(np.int64), row_idx=csc.indices.astype(np.int64),
                     values=csc.data.copy())
    lr = sp.reverse_upper(u)
    rebuilt = np.zeros((n, n))
    cols = np.repeat(np.arange(n), np.diff(lr.col_ptr))
    rebuilt[lr.row_idx, cols] = lr.values
    np.testing.assert_array_equal(rebuilt, dense[::-1, ::-1])
    assert np.all(lr.row_idx[lr.col_ptr[:-1]] == np.arange(n))  # diagonal first
    with pytest.raises(sp.errors.MatrixStructureError if hasattr(sp, "errors") else Exception):
        sp.reverse_upper(sp.CscMatrix(n=2, col_ptr=np.array([0, 2, 3]), row_idx=np.array([0, 1, 1]),
                                      values=np.ones(3)))
