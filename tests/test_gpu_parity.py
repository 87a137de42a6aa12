"""GPU parity: the CUDA path against the reference goldens and the C oracle.

Bars (BASELINE.json north star): in-degrees and levels bit-exact; x bit-exact
in ``precision="exact"`` (the serial oracle's arithmetic) and within max
relative error 1e-12 in ``precision="fast"``.
"""

from __future__ import annotations

import numpy as np
import pytest

import oracle
import paper_2012_06959_b200 as sp
from paper_2012_06959_b200 import _native, synth
from paper_2012_06959_b200.errors import (
    DimensionMismatch,
    MatrixStructureError,
    MissingDiagonal,
    SolveTimeout,
    ZeroDiagonal,
)
from conftest import GOLDEN, REFERENCE_CASES, case_matrix

pytestmark = pytest.mark.gpu

FAST_TOL = 1e-12
EXECUTORS = ["rows", "chains"]


def _solve(l, b, precision="exact", executor="auto", **kw):
    plan = _native.plan_for(l, precision=precision, executor=executor, device=0, **kw)
    x, st = plan.solve(b)
    return x, st


@pytest.mark.parametrize("name", sorted(REFERENCE_CASES))
def test_in_degrees_and_levels_bit_exact(name):
    c = REFERENCE_CASES[name]
    l = case_matrix(c)
    np.testing.assert_array_equal(sp.compute_in_degrees(l), c["in_degree"])
    sched = sp.compute_level_schedule(l)
    np.testing.assert_array_equal(sched.level_of, c["level_of"])
    assert sched.n_levels == int(c["n_levels"])
    # levels[k] lists the level-k components in ascending order (analysis.py:36-37)
    for k, comps in enumerate(sched.levels):
        assert comps == sorted(np.flatnonzero(c["level_of"] == k).tolist())


@pytest.mark.parametrize("executor", EXECUTORS)
@pytest.mark.parametrize("name", sorted(n for n in REFERENCE_CASES if "x" in REFERENCE_CASES[n]))
def test_exact_solve_bitwise_equals_reference(name, executor):
    c = REFERENCE_CASES[name]
    l = case_matrix(c)
    x, st = _solve(l, c["b"], "exact", executor)
    assert x.tobytes() == c["x"].tobytes(), sp.compare_solutions(x, c["x"], 1e-300)


@pytest.mark.parametrize("executor", EXECUTORS)
@pytest.mark.parametrize("name", sorted(n for n in REFERENCE_CASES if "x" in REFERENCE_CASES[n]))
def test_fast_solve_within_1e12(name, executor):
    c = REFERENCE_CASES[name]
    l = case_matrix(c)
    x, _ = _solve(l, c["b"], "fast", executor)
    cmp = sp.compare_solutions(x, c["x"], FAST_TOL)
    assert cmp.within_tol, cmp


def test_solve_serial_dropin_lap2d_256():
    z = np.load(GOLDEN / "lap2d_256.npz")
    l = synth.lap2d(256)
    assert sp.solve_serial(l, np.ones(l.n)).tobytes() == z["x_ones"].tobytes()
    assert sp.solve_serial(l, z["b_rand"]).tobytes() == z["x_rand"].tobytes()
    np.testing.assert_array_equal(sp.compute_in_degrees(l), z["in_degree"])
    sched = sp.compute_level_schedule(l)
    np.testing.assert_array_equal(sched.level_of, z["level_of"])
    assert sched.n_levels == 511


MID_SIZE = {
    "lap2d-128": lambda: synth.lap2d(128),
    "lap3d-24": lambda: synth.lap3d(24),
    "banded-20k": lambda: synth.banded(20_000, 64, 0.5, 3),
    "rmat-14": lambda: synth.rmat(14, 8, 1),
    "random-3000": lambda: synth.random_lower(3000, 0.01, 5, dominant=True),
    "blockdiag-64": lambda: synth.block_diagonal(8192, 64, 2),
}


@pytest.mark.parametrize("executor", EXECUTORS)
@pytest.mark.parametrize("name", sorted(MID_SIZE))
def test_mid_size_against_c_oracle(name, executor):
    l = MID_SIZE[name]()
    rng = np.random.default_rng(7)
    b = rng.uniform(-1.0, 1.0, size=l.n)
    ref = oracle.solve_serial(l.col_ptr, l.row_idx, l.values, b)
    x, _ = _solve(l, b, "exact", executor)
    assert x.tobytes() == ref.tobytes()
    xf, _ = _solve(l, b, "fast", executor)
    assert sp.compare_solutions(xf, ref, FAST_TOL).within_tol
    lv, nl = oracle.levels(l.col_ptr, l.row_idx)
    sched_lv, _, _, n_levels = _native.plan_for(l, structure_only=True, device=0).levels()
    np.testing.assert_array_equal(sched_lv, lv)
    assert n_levels == nl
    np.testing.assert_array_equal(sp.compute_in_degrees(l), oracle.in_degrees(l.col_ptr, l.row_idx))


def test_repeat_solves_reuse_plan_and_agree():
    l = synth.lap2d(64)
    plan = _native.plan_for(l, precision="exact", executor="auto", device=0)
    first, _ = plan.solve(np.ones(l.n))
    for seed in range(3):
        b = np.random.default_rng(seed).uniform(-1, 1, l.n)
        x, _ = plan.solve(b)
        assert x.tobytes() == oracle.solve_serial(l.col_ptr, l.row_idx, l.values, b).tobytes()
    again, _ = plan.solve(np.ones(l.n))
    assert again.tobytes() == first.tobytes()


def test_edge_cases_tiny():
    one = sp.CscMatrix(n=1, col_ptr=[0, 1], row_idx=[0], values=[-2.5])
    assert sp.solve_serial(one, np.array([5.0]))[0] == -2.0
    eye = synth.diagonal(33)
    b = np.linspace(-1, 1, 33)
    assert sp.solve_serial(eye, b).tobytes() == b.tobytes()
    empty = sp.CscMatrix(n=0, col_ptr=[0], row_idx=[], values=[])
    assert sp.solve_serial(empty, np.zeros(0)).shape == (0,)


def test_special_values_propagate_like_ieee():
    l = sp.CscMatrix.from_entries(4, {(0, 0): 1e-310, (1, 0): 1e300, (1, 1): 3.0, (2, 1): 1.0, (2, 2): 1e-300,
                                      (3, 2): -1.0, (3, 3): 7.0})
    for b in ([1e-300, 1.0, 2.0, 3.0], [0.0, -0.0, np.inf, 1.0], [np.nan, 1.0, 1.0, 1.0]):
        b = np.array(b)
        x = sp.solve_serial(l, b)
        ref = oracle.solve_serial(l.col_ptr, l.row_idx, l.values, b)
        np.testing.assert_array_equal(np.isnan(x), np.isnan(ref))
        ok = ~np.isnan(ref)
        assert x[ok].tobytes() == ref[ok].tobytes()


def test_errors_raised_before_solving():
    zero = sp.CscMatrix.from_entries(2, {(0, 0): 0.0, (1, 1): 1.0})
    with pytest.raises(ZeroDiagonal) as e:
        sp.solve_serial(zero, np.ones(2))
    assert e.value.col == 0
    missing = sp.CscMatrix.from_entries(3, {(0, 0): 1.0, (2, 1): 1.0, (2, 2): 1.0})
    with pytest.raises(MissingDiagonal) as e:
        sp.solve_serial(missing, np.ones(3))
    assert e.value.col == 1
    upper = sp.CscMatrix.from_entries(2, {(0, 0): 1.0, (0, 1): 2.0, (1, 1): 1.0})
    with pytest.raises(MatrixStructureError):
        sp.solve_serial(upper, np.ones(2))
    with pytest.raises(DimensionMismatch):
        sp.solve_serial(synth.diagonal(4), np.ones(5))
    # first violation by (col, kind): column 1 misses its diagonal before column 2's zero
    mixed = sp.CscMatrix.from_entries(3, {(0, 0): 1.0, (2, 1): 1.0, (2, 2): 0.0})
    with pytest.raises(MissingDiagonal):
        sp.solve_serial(mixed, np.ones(3))


def test_watchdog_raises_solve_timeout():
    l = synth.bidiagonal(400_000)
    plan = _native.NativePlan(l.col_ptr, l.row_idx, l.values, l.n, precision="exact", executor="rows",
                              timeout=2e-4, spin_initial=1, spin_max_ns=64)
    with pytest.raises(SolveTimeout):
        plan.solve(np.ones(l.n))
    plan.close()


def test_device_resident_solve_matches_host_path():
    torch = pytest.importorskip("torch")
    l = synth.lap3d(20)
    b = np.random.default_rng(3).uniform(-1, 1, l.n)
    plan = _native.plan_for(l, precision="fast", executor="auto", device=0)
    db = torch.from_numpy(b).cuda()
    dx = torch.empty_like(db)
    plan.solve_device_async(db.data_ptr(), dx.data_ptr(), torch.cuda.current_stream().cuda_stream)
    plan.synchronize()
    torch.cuda.synchronize()
    x_host, _ = plan.solve(b)
    assert dx.cpu().numpy().tobytes() == x_host.tobytes()


@pytest.mark.parametrize("executor", ["stencil", "chains", "rows"])
def test_device_resident_unaligned_vectors(executor):
    """b and x only 8-byte aligned (views at an odd element offset)."""
    torch = pytest.importorskip("torch")
    l = _random_coefficients(synth.lap2d(128, 70), 5)
    b = np.random.default_rng(4).uniform(-1, 1, l.n)
    ref = oracle.solve_serial(l.col_ptr, l.row_idx, l.values, b)
    plan = _native.NativePlan(l.col_ptr, l.row_idx, l.values, l.n, precision="exact", executor=executor)
    db = torch.zeros(l.n + 1, dtype=torch.float64, device="cuda")
    db[1:] = torch.from_numpy(b).cuda()
    dx = torch.zeros(l.n + 1, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    plan.solve_device_async(db[1:].data_ptr(), dx[1:].data_ptr(), torch.cuda.current_stream().cuda_stream)
    plan.synchronize()
    assert dx[1:].cpu().numpy().tobytes() == ref.tobytes()
    plan.close()


def _random_coefficients(l, seed):
    """Same structure, random off-diagonals in [-1, 1], dominant diagonal."""
    rng = np.random.default_rng(seed)
    vals = l.values.copy()
    cols = l.entry_columns()
    off = l.row_idx != cols
    vals[off] = rng.uniform(-1.0, 1.0, off.sum())
    dom = 1.0 + np.bincount(l.row_idx[off], weights=np.abs(vals[off]), minlength=l.n)
    vals[~off] = np.where(rng.random(l.n) < 0.5, -1.0, 1.0) * dom
    return sp.CscMatrix(n=l.n, col_ptr=l.col_ptr, row_idx=l.row_idx, values=vals)


@pytest.mark.parametrize("shape", [(4, 2), (8, 3), (64, 64), (128, 65), (256, 200), (1024, 130)])
@pytest.mark.parametrize("precision", ["exact", "fast"])
def test_stencil_executor_matches_oracle(shape, precision):
    nx, ny = shape
    l = _random_coefficients(synth.lap2d(nx, ny), nx * 1000 + ny)
    b = np.random.default_rng(ny).uniform(-1.0, 1.0, l.n)
    ref = oracle.solve_serial(l.col_ptr, l.row_idx, l.values, b)
    plan = _native.NativePlan(l.col_ptr, l.row_idx, l.values, l.n, precision=precision, executor="auto")
    assert plan.info()["executor"] == "stencil"
    for _ in range(2):  # repeat solves reuse the mailboxes
        x, _ = plan.solve(b)
        if precision == "exact":
            assert x.tobytes() == ref.tobytes()
        else:
            assert sp.compare_solutions(x, ref, FAST_TOL).within_tol
    plan.close()


@pytest.mark.parametrize("shape", [(64, 64), (256, 130), (16, 40, 9)])
def test_stencil_exact_guard_redo(shape):
    """Operands outside Markstein's exponent window (tiny / huge b, tiny
    diagonals) fail the division guard inside some chunks: the speculative
    exact stencil must roll those chunks back and recompute them with IEEE
    division, bit-identical to the serial oracle (and count the redos)."""
    nx, ny = shape[:2]
    grid = synth.lap2d(nx, ny) if len(shape) == 2 else synth.lap3d(*shape)
    l = _random_coefficients(grid, 7 * nx + ny)
    rng = np.random.default_rng(nx + ny)
    b = rng.uniform(-1.0, 1.0, l.n)
    hot = rng.choice(l.n, size=max(4, l.n // 500), replace=False)
    b[hot[0::3]] *= 1e-310  # subnormal numerators
    b[hot[1::3]] *= 1e300   # huge numerators
    b[hot[1]] = np.inf      # non-finite numerators propagate like IEEE
    b[hot[4]] = np.nan
    vals = l.values.copy()
    diag = l.row_idx == l.entry_columns()
    dpos = np.flatnonzero(diag)[hot[2::3]]
    vals[dpos] *= 1e-300    # tiny diagonals: huge quotients
    l = sp.CscMatrix(n=l.n, col_ptr=l.col_ptr, row_idx=l.row_idx, values=vals)
    with np.errstate(all="ignore"):
        ref = oracle.solve_serial(l.col_ptr, l.row_idx, l.values, b)
    plan = _native.NativePlan(l.col_ptr, l.row_idx, l.values, l.n, precision="exact", executor="stencil",
                              probe_flags=128)
    for _ in range(2):
        x, st = plan.solve(b)
        nan = np.isnan(ref)
        assert np.array_equal(np.isnan(x), nan)
        assert x[~nan].tobytes() == ref[~nan].tobytes()
    assert st["remote_reads"] > 0  # probe 128: chunks recomputed with IEEE division
    plan.close()


@pytest.mark.parametrize("dims", [(64, 70), (16, 40, 9)])
def test_stencil_exact_signed_zeros(dims):
    """b of +0 / -0 only: every x is a signed zero, and the sign depends on
    the oracle's s = 0 + ... accumulation order (IEEE -0 + -0 = -0 but
    (0 + -0) + -0 = +0) — bitwise parity on the 2D and 3D stencils."""
    grid = synth.lap2d(*dims) if len(dims) == 2 else synth.lap3d(*dims)
    rng = np.random.default_rng(len(dims))
    b = np.where(rng.random(grid.n) < 0.5, -0.0, 0.0)
    ref = oracle.solve_serial(grid.col_ptr, grid.row_idx, grid.values, b)
    assert np.signbit(ref).any() and (~np.signbit(ref)).any()
    plan = _native.NativePlan(grid.col_ptr, grid.row_idx, grid.values, grid.n, precision="exact", executor="stencil")
    x, _ = plan.solve(b)
    assert x.tobytes() == ref.tobytes()
    plan.close()


@pytest.mark.parametrize("executor", ["rows", "chains", "band"])
def test_signed_zero_rhs_general_executors(executor):
    """The same signed-zero bar for the general executors (their division is
    div_exact, whose window check sends zero numerators to IEEE division)."""
    l = synth.banded(3000, 64, 0.5, seed=3) if executor == "band" else synth.lap2d(31, 40)
    rng = np.random.default_rng(5)
    b = np.where(rng.random(l.n) < 0.5, -0.0, 0.0)
    b[rng.choice(l.n, 20, replace=False)] = 1.0  # a few nonzero sources
    ref = oracle.solve_serial(l.col_ptr, l.row_idx, l.values, b)
    plan = _native.NativePlan(l.col_ptr, l.row_idx, l.values, l.n, precision="exact", executor=executor)
    x, _ = plan.solve(b)
    assert x.tobytes() == ref.tobytes()
    plan.close()


def test_stencil_not_chosen_for_other_structures():
    l = synth.lap2d(31, 10)  # nx not a multiple of the column block: general executors
    plan = _native.NativePlan(l.col_ptr, l.row_idx, l.values, l.n, executor="auto")
    assert plan.info()["executor"] != "stencil"
    plan.close()
    with pytest.raises(sp.errors.SptrsvError if hasattr(sp, "errors") else Exception):
        _native.NativePlan(l.col_ptr, l.row_idx, l.values, l.n, executor="stencil")
    l3 = synth.lap3d(9)  # odd nx: not a whole number of 2-column blocks
    plan = _native.NativePlan(l3.col_ptr, l3.row_idx, l3.values, l3.n, executor="auto")
    assert plan.info()["executor"] != "stencil"
    plan.close()
    lr = synth.random_lower(500, 0.02, 3, dominant=True)
    plan = _native.NativePlan(lr.col_ptr, lr.row_idx, lr.values, lr.n, executor="auto")
    assert plan.info()["executor"] != "stencil"
    plan.close()


@pytest.mark.parametrize("shape", [(8, 8, 8), (16, 33, 5), (64, 32, 9), (128, 70, 13), (24, 96, 40)])
@pytest.mark.parametrize("precision", ["exact", "fast"])
def test_stencil3d_executor_matches_oracle(shape, precision):
    """3D seven-point structure: the tile wavefront (stencil3d.cu) is chosen
    automatically; random coefficients; partial y-tiles and z-tiles."""
    l = _random_coefficients(synth.lap3d(*shape), 13)
    b = np.random.default_rng(14).uniform(-1, 1, l.n)
    ref = oracle.solve_serial(l.col_ptr, l.row_idx, l.values, b)
    plan = _native.NativePlan(l.col_ptr, l.row_idx, l.values, l.n, precision=precision, executor="auto")
    assert plan.info()["executor"] == "stencil"
    for _ in range(3):  # repeated solves: mailbox parity halves
        x, _ = plan.solve(b)
        if precision == "exact":
            assert x.tobytes() == ref.tobytes()
        else:
            assert sp.compare_solutions(x, ref, FAST_TOL).within_tol
    plan.close()


def test_stencil3d_unaligned_and_device_resident():
    torch = pytest.importorskip("torch")
    l = _random_coefficients(synth.lap3d(32, 40, 7), 15)
    b = np.random.default_rng(16).uniform(-1, 1, l.n)
    ref = oracle.solve_serial(l.col_ptr, l.row_idx, l.values, b)
    plan = _native.NativePlan(l.col_ptr, l.row_idx, l.values, l.n, precision="exact", executor="stencil")
    db = torch.zeros(l.n + 1, dtype=torch.float64, device="cuda")
    db[1:] = torch.from_numpy(b).cuda()
    dx = torch.zeros(l.n + 1, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    plan.solve_device_async(db[1:].data_ptr(), dx[1:].data_ptr(), torch.cuda.current_stream().cuda_stream)
    plan.synchronize()
    assert dx[1:].cpu().numpy().tobytes() == ref.tobytes()
    plan.close()


@pytest.mark.parametrize("precision", ["exact", "fast"])
@pytest.mark.parametrize("shape", [(64, 64), (128, 200), (512, 1000), (16, 40, 9), (64, 70, 33)])
def test_stencil_streamed_host_solve(shape, precision):
    """sptrsv_solve on host buffers: pinned (band-granular copies overlapping
    the kernel) and pageable give the same x as the unstreamed plan and
    (exact) the oracle; repeated solves (epoch flags never reset)."""
    torch = pytest.importorskip("torch")
    l = _random_coefficients(synth.lap2d(*shape) if len(shape) == 2 else synth.lap3d(*shape), 11)
    rng = np.random.default_rng(12)
    plan = _native.NativePlan(l.col_ptr, l.row_idx, l.values, l.n, precision=precision, executor="stencil")
    flat = _native.NativePlan(l.col_ptr, l.row_idx, l.values, l.n, precision=precision, executor="stencil",
                              streamed_io=False)
    hb = torch.empty(l.n, dtype=torch.float64).pin_memory()
    hx = torch.empty(l.n, dtype=torch.float64).pin_memory()
    for rep in range(3):
        b = rng.uniform(-1, 1, l.n)
        ref = oracle.solve_serial(l.col_ptr, l.row_idx, l.values, b)
        x1, st1 = plan.solve(b)  # pageable: copy in, solve, copy out
        assert st1["streamed_io"] == 0
        hb.numpy()[:] = b
        _, st2 = plan.solve(hb.numpy(), out=hx.numpy())  # pinned: band-granular copies overlap the kernel
        assert st2["streamed_io"] & 1
        x0, st0 = flat.solve(hb.numpy())
        assert st0["streamed_io"] == 0
        assert x1.tobytes() == x0.tobytes() == hx.numpy().tobytes()
        if precision == "exact":
            assert x1.tobytes() == ref.tobytes()
        else:
            assert np.max(np.abs(x1 - ref) / np.maximum(np.abs(ref), 1.0)) <= 1e-12
    plan.close()
    flat.close()


BAND_CASES = {
    "banded-20k-64": lambda: synth.banded(20_000, 64, 0.5, 3),
    "banded-5k-16": lambda: synth.banded(5_000, 16, 0.9, 4),
    "banded-3k-64-dense": lambda: synth.banded(3_000, 64, 1.0, 5),
    "bidiagonal-3000": lambda: synth.bidiagonal(3_000),
    "banded-ragged-1000": lambda: synth.banded(1_000, 64, 0.3, 6),
}


@pytest.mark.parametrize("precision", ["exact", "fast"])
@pytest.mark.parametrize("name", sorted(BAND_CASES))
def test_band_executor_matches_oracle(name, precision):
    """Sliding-window executor (solve_band.cu): chosen automatically for narrow,
    nearly sequential L; exact mode accumulates in the oracle's column order."""
    l = BAND_CASES[name]()
    b = np.random.default_rng(21).uniform(-1, 1, l.n)
    ref = oracle.solve_serial(l.col_ptr, l.row_idx, l.values, b)
    plan = _native.NativePlan(l.col_ptr, l.row_idx, l.values, l.n, precision=precision, executor="auto")
    assert plan.info()["executor"] == "band"
    for _ in range(2):
        x, _ = plan.solve(b)
        if precision == "exact":
            assert x.tobytes() == ref.tobytes()
        else:
            assert sp.compare_solutions(x, ref, FAST_TOL).within_tol
    plan.close()


def test_band_executor_special_values_and_errors():
    l = synth.banded(2_000, 32, 0.5, 7)
    b = np.random.default_rng(22).uniform(-1, 1, l.n)
    b[100], b[700] = np.inf, np.nan
    ref = oracle.solve_serial(l.col_ptr, l.row_idx, l.values, b)
    plan = _native.NativePlan(l.col_ptr, l.row_idx, l.values, l.n, precision="exact", executor="band")
    x, _ = plan.solve(b)
    # NaN payload/sign bits are not part of IEEE parity (as in test_special_values_propagate_like_ieee)
    np.testing.assert_array_equal(np.isnan(x), np.isnan(ref))
    ok = ~np.isnan(ref)
    assert x[ok].tobytes() == ref[ok].tobytes()
    plan.close()
    wide = synth.random_lower(500, 0.05, 8, dominant=True)  # dependencies farther than 64 rows
    with pytest.raises(sp.errors.SptrsvError if hasattr(sp, "errors") else Exception):
        _native.NativePlan(wide.col_ptr, wide.row_idx, wide.values, wide.n, executor="band")


def test_split_heavy_rows_fast_mode():
    """Fast mode splits rows with > 256 dependencies into partial tasks (one
    warp per 256 entries, summed with atomics); exact mode keeps them whole.
    Power-law rows of every size around the split threshold."""
    rng = np.random.default_rng(31)
    n = 6000
    entries = {}
    for i in range(n):
        entries[(i, i)] = 4.0 + rng.random()
    for i in range(1, n):
        k = int(min(i, rng.choice([1, 3, 30, 255, 256, 257, 600, 2500, 5000], p=[.3, .3, .2, .04, .04, .04, .04, .02, .02])))
        for j in rng.choice(i, size=k, replace=False):
            entries[(i, int(j))] = rng.uniform(-1, 1) / k
    l = sp.CscMatrix.from_entries(n, entries)
    b = rng.uniform(-1, 1, n)
    ref = oracle.solve_serial(l.col_ptr, l.row_idx, l.values, b)
    for precision in ("fast", "exact"):
        plan = _native.NativePlan(l.col_ptr, l.row_idx, l.values, l.n, precision=precision, executor="rows")
        for _ in range(2):
            x, _ = plan.solve(b)
            if precision == "exact":
                assert x.tobytes() == ref.tobytes()
            else:
                assert sp.compare_solutions(x, ref, FAST_TOL).within_tol
        plan.close()


def _serial_backward(u, b):
    """Backward substitution with the serial oracle's rounding: x_i = (b_i - sum_{j>i} u_ij x_j) / u_ii,
    terms added in descending column order (the reversed lower solve's ascending order)."""
    n = u.n
    x = np.zeros(n)
    left = np.zeros(n)
    for j in range(n - 1, -1, -1):
        rows = u.row_idx[u.col_ptr[j]:u.col_ptr[j + 1]]
        vals = u.values[u.col_ptr[j]:u.col_ptr[j + 1]]
        x[j] = (b[j] - left[j]) / vals[-1]  # diagonal is the last entry of an upper column
        for r, v in zip(rows[:-1], vals[:-1]):
            left[r] += v * x[j]
    return x


@pytest.mark.parametrize("shape", ["lap2d", "random", "banded"])
def test_upper_triangular_solve(shape):
    """Row f4: U x = b through the index reversal, exact mode equal to serial backward substitution."""
    low = {"lap2d": lambda: synth.lap2d(40, 30), "random": lambda: synth.random_lower(700, 0.02, 4, dominant=True),
           "banded": lambda: synth.banded(900, 16, 0.5, 2)}[shape]()
    import scipy.sparse as ssp

    dense_l = ssp.csc_matrix((low.values, low.row_idx, low.col_ptr), shape=(low.n, low.n))
    ut = dense_l.T.tocsc()
    ut.sort_indices()
    u = sp.CscMatrix(n=low.n, col_ptr=ut.indptr.astype(np.int64), row_idx=ut.indices.astype(np.int64),
                     values=ut.data.copy())
    b = np.random.default_rng(5).uniform(-1, 1, u.n)
    x = sp.solve_upper(u, b, precision="exact")
    assert x.tobytes() == _serial_backward(u, b).tobytes()
    xf = sp.solve_upper(u, b, precision="fast")
    assert sp.compare_solutions(xf, x, FAST_TOL).within_tol


def test_solve_many_columns():
    l = synth.lap3d(12)
    bs = np.random.default_rng(6).uniform(-1, 1, (l.n, 5))
    xs = sp.solve_many(l, bs, precision="exact")
    for k in range(5):
        assert xs[:, k].tobytes() == oracle.solve_serial(l.col_ptr, l.row_idx, l.values, bs[:, k].copy()).tobytes()


@pytest.mark.parametrize("name", ["lap2d-64x50", "lap3d-9x7x5", "lap3d-16", "banded-5k-16", "banded-3k-64-dense",
                                  "bidiagonal-3000", "random-band"])
def test_levels_fast_paths_bit_exact(name):
    """K6 takes the closed form x+y(+z) for verified grid stencils and the band
    window kernel in (max,+1) mode for narrow bands: levels and in-degrees
    must equal the oracle's bit for bit."""
    l = {
        "lap2d-64x50": lambda: synth.lap2d(64, 50),
        "lap3d-9x7x5": lambda: synth.lap3d(10, 7, 5),
        "lap3d-16": lambda: synth.lap3d(16),
        "banded-5k-16": BAND_CASES["banded-5k-16"],
        "banded-3k-64-dense": BAND_CASES["banded-3k-64-dense"],
        "bidiagonal-3000": BAND_CASES["bidiagonal-3000"],
        "random-band": lambda: synth.random_lower(4000, 0.01, 9, bandwidth=40, dominant=True),
    }[name]()
    lv, nl = oracle.levels(l.col_ptr, l.row_idx)
    sched = sp.compute_level_schedule(l)
    assert sched.n_levels == nl
    np.testing.assert_array_equal(sched.level_of, lv)
    np.testing.assert_array_equal(sp.compute_in_degrees(l), oracle.in_degrees(l.col_ptr, l.row_idx))
    plan = _native.NativePlan(l.col_ptr, l.row_idx, l.values, l.n, precision="exact", executor="auto")
    level_of, order, level_ptr, n_levels = plan.levels()
    assert n_levels == nl
    np.testing.assert_array_equal(level_of, lv)
    plan.close()


@pytest.mark.parametrize("shape,k", [((128, 192), 5), ((256, 64), 17), ((96, 128), 1), ((64, 100), 3)])
@pytest.mark.parametrize("precision", ["exact", "fast"])
def test_solve_many_stacked_stencil(shape, k, precision):
    """Several right-hand sides through one stacked 2D-stencil launch (whole
    bands: 192 / 64 rows; k = 17 takes two launches of <= 16), or one solve
    after another when the last band is partial (100 rows): each column is
    bitwise the oracle's (exact) / within 1e-12 (fast), repeated so the
    stacked mailboxes are re-armed between solves and between k's."""
    l = synth.lap2d(*shape)
    rng = np.random.default_rng(k)
    for kk in (k, max(1, k - 2), k):
        bs = rng.uniform(-1, 1, (l.n, kk))
        xs = sp.solve_many(l, bs, precision=precision, executor="stencil")
        for c in range(kk):
            ref = oracle.solve_serial(l.col_ptr, l.row_idx, l.values, bs[:, c].copy())
            if precision == "exact":
                assert xs[:, c].tobytes() == ref.tobytes(), (kk, c)
            else:
                assert sp.compare_solutions(xs[:, c], ref, FAST_TOL).within_tol, (kk, c)


def test_solve_many_rows_executor():
    l = synth.rmat(11, 8, 2)
    bs = np.random.default_rng(9).uniform(-1, 1, (l.n, 4))
    xs = sp.solve_many(l, bs, precision="exact", executor="rows")
    for c in range(4):
        assert xs[:, c].tobytes() == oracle.solve_serial(l.col_ptr, l.row_idx, l.values, bs[:, c].copy()).tobytes()


@pytest.mark.parametrize("shape", [(128, 70), (256, 128)])
def test_stencil_fast_unaligned_and_partial_bands(shape):
    """Fast mode's pre-scaled right-hand side (the kernel's prep tasks write
    b * (1/d) band by band): b only 8-byte aligned (scalar prep path), a
    partial last band (70 rows), repeated solves (per-solve flag epochs)."""
    torch = pytest.importorskip("torch")
    l = _random_coefficients(synth.lap2d(*shape), 9)
    plan = _native.NativePlan(l.col_ptr, l.row_idx, l.values, l.n, precision="fast", executor="stencil")
    for rep in range(3):
        b = np.random.default_rng(rep).uniform(-1, 1, l.n)
        ref = oracle.solve_serial(l.col_ptr, l.row_idx, l.values, b)
        db = torch.zeros(l.n + 1, dtype=torch.float64, device="cuda")
        db[1:] = torch.from_numpy(b).cuda()
        dx = torch.zeros(l.n + 1, dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()
        plan.solve_device_async(db[1:].data_ptr(), dx[1:].data_ptr(), torch.cuda.current_stream().cuda_stream)
        plan.synchronize()
        assert sp.compare_solutions(dx[1:].cpu().numpy(), ref, FAST_TOL).within_tol
        x, _ = plan.solve(b)  # host buffers (pageable: copy, solve, copy)
        assert sp.compare_solutions(x, ref, FAST_TOL).within_tol
    plan.close()


@pytest.mark.parametrize("shape", [(256, 1000), (130, 700)])
def test_stencil_fast_band_groups(shape):
    """Fast mode on a diagonally dominant grid (lap2d: the error of a solve
    started from a zero row contracts by 1/3 per grid row): the bands run in
    independent groups, each entered through a halo band solved from a zero
    row above it (entering error <= 3e-31 |x|). x within 1e-12 of the oracle
    on device buffers, pageable and pinned (streamed) host buffers, repeated
    solves (mailbox parity), partial last band; bitwise equal across the
    three paths. A weakly dominant grid (contraction > 1/2) keeps one chain
    and is checked the same way."""
    torch = pytest.importorskip("torch")
    strong = synth.lap2d(*shape)
    weak_vals = strong.values.copy()
    weak_vals[strong.row_idx == strong.entry_columns()] = 2.2  # |a| = |u| = 1/2.2: contraction 0.83
    weak = sp.CscMatrix(n=strong.n, col_ptr=strong.col_ptr, row_idx=strong.row_idx, values=weak_vals)
    hb = torch.empty(strong.n, dtype=torch.float64).pin_memory()
    hx = torch.empty(strong.n, dtype=torch.float64).pin_memory()
    for l in (strong, weak):
        plan = _native.NativePlan(l.col_ptr, l.row_idx, l.values, l.n, precision="fast", executor="stencil")
        for rep in range(3):
            b = np.random.default_rng(rep).uniform(-1, 1, l.n)
            ref = oracle.solve_serial(l.col_ptr, l.row_idx, l.values, b)
            db = torch.from_numpy(b).cuda()
            dx = torch.empty_like(db)
            torch.cuda.synchronize()
            plan.solve_device_async(db.data_ptr(), dx.data_ptr(), torch.cuda.current_stream().cuda_stream)
            plan.synchronize()
            xd = dx.cpu().numpy()
            assert sp.compare_solutions(xd, ref, FAST_TOL).within_tol
            x1, _ = plan.solve(b)
            hb.numpy()[:] = b
            plan.solve(hb.numpy(), out=hx.numpy())
            assert xd.tobytes() == x1.tobytes() == hx.numpy().tobytes()
        plan.close()


@pytest.mark.parametrize("dims", [(40, 40, 80), (64, 70, 100)])
def test_stencil3d_fast_z_groups(dims):
    """Fast 3D wavefront on a diagonally dominant grid (lap3d: the error of a
    solve started from a zero plane contracts by 1/4 per plane): z-tiles run
    in independent groups, each after the first entered through 8 halo
    z-tiles (32 planes, entering error <= 2^-64 |x|). x within 1e-12 of the
    oracle on device, pageable and pinned host buffers over repeated solves,
    bitwise equal across the three; a weakly dominant grid keeps one chain."""
    torch = pytest.importorskip("torch")
    strong = synth.lap3d(*dims)
    weak_vals = strong.values.copy()
    weak_vals[strong.row_idx == strong.entry_columns()] = 3.3  # contraction (1/3.3)/(1 - 2/3.3) ~ 0.77
    weak = sp.CscMatrix(n=strong.n, col_ptr=strong.col_ptr, row_idx=strong.row_idx, values=weak_vals)
    hb = torch.empty(strong.n, dtype=torch.float64).pin_memory()
    hx = torch.empty(strong.n, dtype=torch.float64).pin_memory()
    for l in (strong, weak):
        plan = _native.NativePlan(l.col_ptr, l.row_idx, l.values, l.n, precision="fast", executor="stencil")
        for rep in range(3):
            b = np.random.default_rng(rep).uniform(-1, 1, l.n)
            ref = oracle.solve_serial(l.col_ptr, l.row_idx, l.values, b)
            db = torch.from_numpy(b).cuda()
            dx = torch.empty_like(db)
            torch.cuda.synchronize()
            plan.solve_device_async(db.data_ptr(), dx.data_ptr(), torch.cuda.current_stream().cuda_stream)
            plan.synchronize()
            xd = dx.cpu().numpy()
            assert sp.compare_solutions(xd, ref, FAST_TOL).within_tol
            x1, _ = plan.solve(b)
            hb.numpy()[:] = b
            plan.solve(hb.numpy(), out=hx.numpy())
            assert xd.tobytes() == x1.tobytes() == hx.numpy().tobytes()
        plan.close()
