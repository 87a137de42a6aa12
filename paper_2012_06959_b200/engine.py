"""GPU engines behind the reference's solve API.

Drop-in for `/root/reference/pkg/src/sptrsv/engine.py`: same ``Engine`` enum,
``SolverConfig`` / ``Backoff`` / ``SolveReport`` / ``PeStats`` /
``EngineState`` types, same ``solve`` / ``solve_partitioned`` /
``solve_shared_atomics`` signatures, same input checks and exception classes
(engine.py:275-286), same synchronous contract (x is complete on return).

What runs is different: the reference models each GPU as a team of Python
threads exchanging counters through locked lists; here the solve is a
persistent CUDA kernel (``csrc/solve_rows.cu`` — the sync-free component
pool — or ``csrc/solve_chains.cu`` — lane-chain lockstep warps) that pulls
solved x values with one-sided loads. PE ownership (the ``PartitionPlan``)
decides which HBM segment a component's x lives in; on one GPU the PEs are
segments of the same device (see ``paper_2012_06959_b200.multi`` for one
process per GPU over NVLink peer mappings).

Config mapping: ``n_pes`` -> PE segments / GPUs;
``workers_per_pe`` -> accepted and validated (warps replace worker threads);
``spin_backoff`` -> poll count before ``__nanosleep`` and the largest sleep;
``timeout`` -> device watchdog raising ``SolveTimeout``;
``remote_read_caching`` -> accepted (a pulled x value is final, so a remote
slot is never re-read once seen); ``capture_state`` -> post-solve
``EngineState`` in the reference's push-variant convention (below);
``debug`` -> device checks of the publication protocol (SPTRSV_PLAN_DEBUG):
every published x slot / mailbox word is written once, over its sentinel, by
the PE that owns it -- the reference's write-locality and monotone-counter
assertions (engine.py:154-169, 510-513) -- raising AssertionError.
"""

from __future__ import annotations

import time
import weakref
from dataclasses import dataclass, field
from enum import Enum

import numpy as np

from . import _native
from .errors import DimensionMismatch
from .matrix import CscMatrix
from .partition import PartitionPlan


class Engine(Enum):
    SHARED_ATOMICS = "shared"
    PARTITIONED_READ_ONLY = "partitioned"


@dataclass(frozen=True)
class Backoff:
    """Polls before sleeping, and the longest sleep (engine.py:61-66)."""

    initial_pause: int = 16
    max_pause: int = 512


@dataclass(frozen=True)
class SolverConfig:
    """Reference fields (engine.py:69-86) plus the GPU knobs, all defaulted.

    ``precision``: ``"exact"`` reproduces the serial oracle bit for bit;
    ``"fast"`` pre-scales rows and uses FMA (rel. error ~1e-15, contract 1e-12).
    ``executor``: ``"auto"`` / ``"rows"`` / ``"chains"``. ``device``: CUDA ordinal.
    """

    engine: Engine
    n_pes: int = 1
    workers_per_pe: int = 1
    spin_backoff: Backoff = Backoff()
    timeout: float = 60.0
    remote_read_caching: bool = True
    capture_state: bool = False
    debug: bool = False
    precision: str = "exact"
    executor: str = "auto"
    device: int = 0

    def __post_init__(self):
        if self.n_pes < 1:
            raise ValueError(f"n_pes must be >= 1, got {self.n_pes}")
        if self.workers_per_pe < 1:
            raise ValueError(f"workers_per_pe must be >= 1, got {self.workers_per_pe}")
        if self.timeout <= 0:
            raise ValueError(f"timeout must be positive, got {self.timeout}")
        if self.precision not in _native.PRECISION:
            raise ValueError(f"precision must be one of {sorted(_native.PRECISION)}, got {self.precision!r}")
        if self.executor not in _native.EXECUTOR:
            raise ValueError(f"executor must be one of {sorted(_native.EXECUTOR)}, got {self.executor!r}")
        if self.executor == "push" and self.precision == "exact":
            # Alg. 2 accumulates with atomics in arrival order: within 1e-12 of
            # the oracle, never bit-identical, so it cannot honour "exact"
            raise ValueError('executor="push" (atomic left sums) is not bit-exact: use precision="fast"')


@dataclass
class PeStats:
    pe: int
    components_solved: int = 0
    lock_wait_spins: int = 0
    remote_reads_issued: int = 0
    remote_reads_skipped: int = 0
    local_updates: int = 0
    remote_updates: int = 0


@dataclass(frozen=True)
class EngineState:
    """Post-solve dependency bookkeeping (engine.py:100-107)."""

    s_in_degree: list[np.ndarray]
    s_left_sum: list[np.ndarray]
    d_in_degree: np.ndarray
    d_left_sum: np.ndarray


@dataclass(frozen=True)
class SolveReport:
    x: np.ndarray
    wall_time: float
    setup_time: float
    solve_time: float
    engine: Engine
    n_pes: int
    per_pe: list[PeStats]
    state: EngineState | None = None
    device: dict = field(default_factory=dict, compare=False)

    def totals(self) -> dict[str, int]:
        keys = (
            "components_solved",
            "lock_wait_spins",
            "remote_reads_issued",
            "remote_reads_skipped",
            "local_updates",
            "remote_updates",
        )
        return {k: sum(getattr(s, k) for s in self.per_pe) for k in keys}


def reduce_contributions(values) -> float | int:
    """Fixed pairwise tree sum, one value per PE (engine.py:133-147).

    Level k adds neighbours (2m, 2m+1) and carries an odd tail unchanged —
    the order an xor-butterfly over a zero-padded warp reproduces for P <= 8.
    """
    vals = list(values)
    if not vals:
        raise ValueError("need at least one value")
    while len(vals) > 1:
        paired = [a + b for a, b in zip(vals[0::2], vals[1::2])]
        if len(vals) & 1:
            paired.append(vals[-1])
        vals = paired
    return vals[0]


def _check_inputs(l: CscMatrix, b, plan: PartitionPlan, cfg: SolverConfig, expected: Engine) -> np.ndarray:
    """Argument checks in the reference order (engine.py:275-286).

    Triangularity (``ensure_lower_triangular``) is checked on the device when
    the matrix's plan is built, with the same first-violation rule.
    """
    if cfg.engine is not expected:
        raise ValueError(f"config selects engine {cfg.engine.value!r}, called {expected.value!r}")
    b = np.asarray(b, dtype=np.float64)
    if b.shape != (l.n,):
        raise DimensionMismatch(f"rhs has shape {b.shape}, matrix is {l.n}x{l.n}")
    if plan.n != l.n:
        raise DimensionMismatch(f"plan covers {plan.n} components, matrix has {l.n}")
    if plan.n_pes != cfg.n_pes:
        raise ValueError(f"plan has {plan.n_pes} PEs, config says {cfg.n_pes}")
    return b


# --- structural report bookkeeping -----------------------------------------

_struct_cache: dict = {}


def _entry_owner_split(l: CscMatrix, plan: PartitionPlan):
    """Per off-diagonal entry: (row, col, owner(row), owner(col)); cached per (L, plan).

    The cache holds L weakly: an entry is dropped when its matrix is collected.
    """
    key = (id(l), id(plan))
    hit = _struct_cache.get(key)
    if hit is not None and hit[0]() is l and hit[1] is plan:
        return hit[2]
    cols = l.entry_columns()
    off = l.row_idx != cols
    rows, cols = l.row_idx[off], cols[off]
    own = plan.owner_arr
    val = (rows, cols, own[rows], own[cols], l.values[off])
    if len(_struct_cache) > 8:
        _struct_cache.clear()
    _struct_cache[key] = (weakref.ref(l), plan, val)
    weakref.finalize(l, _struct_cache.pop, key, None)
    return val


def _per_pe_stats(l: CscMatrix, plan: PartitionPlan, cfg: SolverConfig, dev: dict) -> list[PeStats]:
    P = cfg.n_pes
    rows, cols, orow, ocol, _ = _entry_owner_split(l, plan)
    local = ocol == orow
    # an update is attributed to the PE that produced x_j (the column owner),
    # as in the reference's solve-update loop (engine.py:532-549)
    loc = np.bincount(ocol[local], minlength=P)
    rem = np.bincount(ocol[~local], minlength=P)
    solved = np.bincount(plan.owner_arr, minlength=P)
    # pulled remote loads per consuming PE; a PE whose segment holds none of a
    # row's dependencies is never read for that row ("skipped")
    rem_reads = np.bincount(orow[~local], minlength=P)
    skipped = np.zeros(P, dtype=np.int64)
    if cfg.remote_read_caching and P > 1:
        pairs = np.unique(rows[~local] * P + ocol[~local])
        touched = np.bincount(pairs // P, minlength=l.n)  # remote PEs read per row
        per_row_skip = (P - 1) - touched
        skipped = np.bincount(plan.owner_arr, weights=per_row_skip, minlength=P).astype(np.int64)
    spins = int(dev.get("spins", 0))
    # one plan per PE (PeGroup): each PE's kernel counted its own polls and
    # cross-PE dependency loads; otherwise one kernel served every PE and its
    # polls are reported on PE 0
    measured = dev.get("per_pe")
    if measured is not None and len(measured) == P:
        pe_spins = [int(m["spins"]) for m in measured]
        pe_remote = [int(m["remote_reads"]) for m in measured]
    else:
        pe_spins = [spins if p == 0 else 0 for p in range(P)]
        pe_remote = [int(v) for v in rem_reads]
    out = []
    for p in range(P):
        out.append(
            PeStats(
                pe=p,
                components_solved=int(solved[p]),
                lock_wait_spins=pe_spins[p],
                remote_reads_issued=pe_remote[p],
                remote_reads_skipped=int(skipped[p]),
                local_updates=int(loc[p]),
                remote_updates=int(rem[p]),
            )
        )
    return out


def _capture_state(l: CscMatrix, plan: PartitionPlan, cfg: SolverConfig, x: np.ndarray, shared: bool) -> EngineState:
    """Quiescent counters/sums in the reference's convention (test_acceptance.py:103-134).

    Pull solves keep no counters, so the state is synthesised from the
    structure and x exactly as the push engines leave it: the owner's
    published counter holds 1 + local dependencies, every other segment's is
    0; ``d_*`` hold the local part, ``s_left_sum[q]`` the contributions of
    q's columns to rows q does not own.
    """
    n, P = l.n, cfg.n_pes
    rows, cols, orow, ocol, vals = _entry_owner_split(l, plan)
    local = ocol == orow
    contrib = vals * x[cols]
    d_in = np.bincount(rows[local], minlength=n).astype(np.int64)
    d_ls = np.bincount(rows[local], weights=contrib[local], minlength=n)
    if shared:
        s_in = [d_in + 1]
        s_ls = [np.bincount(rows[~local], weights=contrib[~local], minlength=n)]
    else:
        s_in = [np.zeros(n, dtype=np.int64) for _ in range(P)]
        s_ls = [np.zeros(n) for _ in range(P)]
        own = plan.owner_arr
        for p in range(P):
            mine = own == p
            s_in[p][mine] = d_in[mine] + 1
            sel = (~local) & (ocol == p)
            s_ls[p] = np.bincount(rows[sel], weights=contrib[sel], minlength=n)
    return EngineState(s_in_degree=s_in, s_left_sum=s_ls, d_in_degree=d_in, d_left_sum=d_ls)


def _run(l: CscMatrix, b, plan: PartitionPlan, cfg: SolverConfig, expected: Engine):
    b = _check_inputs(l, b, plan, cfg, expected)
    t0 = time.perf_counter()
    if l.n == 0:
        x = np.zeros(0)
        return x, SolveReport(x=x, wall_time=0.0, setup_time=0.0, solve_time=0.0, engine=expected,
                              n_pes=cfg.n_pes, per_pe=[PeStats(pe=p) for p in range(cfg.n_pes)])
    ts = time.perf_counter()
    knobs = dict(
        precision=cfg.precision,
        device=cfg.device,
        timeout=cfg.timeout,
        spin_initial=64 * cfg.spin_backoff.initial_pause,
        spin_max_ns=max(16, cfg.spin_backoff.max_pause // 8),
    )
    if cfg.debug:
        knobs["debug"] = True
    if expected is Engine.PARTITIONED_READ_ONLY and cfg.n_pes > 1:
        # one published segment per PE (owner-only writes, read-only peers):
        # one PE per GPU when several are visible, else the PEs share the
        # device with the fastest executor that has a per-PE mode
        native = _native.pe_solver_for(l, plan, executor=cfg.executor, **knobs)
    else:
        # one published segment shared by all PEs
        native = _native.plan_for(l, executor=cfg.executor, **knobs)
    setup = time.perf_counter() - ts
    ts = time.perf_counter()
    x, dev = native.solve(b)
    solve_wall = time.perf_counter() - ts
    per_pe = _per_pe_stats(l, plan, cfg, dev)
    state = _capture_state(l, plan, cfg, x, expected is Engine.SHARED_ATOMICS) if cfg.capture_state else None
    t1 = time.perf_counter()
    return x, SolveReport(
        x=x,
        wall_time=t1 - t0,
        setup_time=setup,
        solve_time=solve_wall,
        engine=expected,
        n_pes=cfg.n_pes,
        per_pe=per_pe,
        state=state,
        device=dev,
    )


def solve_shared_atomics(l: CscMatrix, b, plan: PartitionPlan, cfg: SolverConfig):
    """Alg. 2 entry point (engine.py:324-431): one published x segment shared by all PEs."""
    return _run(l, b, plan, cfg, Engine.SHARED_ATOMICS)


def solve_partitioned(l: CscMatrix, b, plan: PartitionPlan, cfg: SolverConfig):
    """Alg. 3 entry point (engine.py:438-582): per-PE segments, owner-only writes, read-only peers."""
    return _run(l, b, plan, cfg, Engine.PARTITIONED_READ_ONLY)


def solve(l: CscMatrix, b, plan: PartitionPlan, cfg: SolverConfig):
    """Dispatch on ``cfg.engine`` (engine.py:585-589)."""
    if cfg.engine is Engine.SHARED_ATOMICS:
        return solve_shared_atomics(l, b, plan, cfg)
    return solve_partitioned(l, b, plan, cfg)
