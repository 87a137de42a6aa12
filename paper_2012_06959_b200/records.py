"""Benchmark records in the reference's schema (
reference cli.py:57-80 RunSpec, :153-209 run_benchmark, :212-227 _emit,
:257-290 sweep-tasks / sweep-pes; docs/record_schema.json).

``run_benchmark`` runs ``repeats`` GPU solves plus one serial-reference
solve and returns one record with exactly the reference's 23 fields in the
reference's order (``engine`` stays "shared" / "partitioned": the schema's
enum); timings are the reports' wall-clock setup / solve times, like the
reference's. ``sweep_tasks`` / ``sweep_pes`` (with ``fixed_total_tasks``, the
paper's 32-task PE sweep) and ``emit`` (JSON lines or CSV with
null as an empty cell) complete the record front end; the argparse CLI itself
is out of scope.
"""

from __future__ import annotations

import csv
import io
import json
import sys
from dataclasses import dataclass, replace
from pathlib import Path
from typing import Callable, Optional

import numpy as np

from . import analysis
from .engine import Engine, SolverConfig, solve
from .errors import IndivisibleTaskTotal, InvalidSpec, SptrsvError
from .matrix import CscMatrix
from .partition import task_round_robin_partition
from .reference import compare_solutions, solve_serial

VERIFY_TOL = 1e-9  # the reference CLI's verification tolerance (cli.py:27)

FIELDS = (
    "name", "engine", "n", "nnz", "n_levels", "parallelism", "dependency", "n_pes", "tasks_per_pe",
    "workers_per_pe", "repeats", "engine_runs", "mean_wall_time", "min_wall_time", "max_wall_time",
    "mean_setup_time", "mean_combined_time", "max_rel_error", "lock_wait_spins", "remote_reads_issued",
    "remote_reads_skipped", "local_updates", "remote_updates",
)


_INT = {"type": "integer", "minimum": 0}
_INT1 = {"type": "integer", "minimum": 1}
_SEC = {"type": "number", "minimum": 0}
# The record contract of the reference (docs/record_schema.json, draft 2020-12),
# restated: field types, bounds, the engine enum, no extra fields.
RECORD_SCHEMA = {
    "$schema": "https://json-schema.org/draft/2020-12/schema",
    "type": "object",
    "properties": {
        "name": {"type": "string"}, "engine": {"enum": ["shared", "partitioned"]},
        "n": _INT1, "nnz": _INT1, "n_levels": _INT1, "parallelism": _INT1,
        "dependency": {"type": "number", "exclusiveMinimum": 0},
        "n_pes": _INT1, "tasks_per_pe": _INT1, "workers_per_pe": _INT1, "repeats": _INT1, "engine_runs": _INT1,
        "mean_wall_time": _SEC, "min_wall_time": _SEC, "max_wall_time": _SEC, "mean_setup_time": _SEC,
        "mean_combined_time": _SEC, "max_rel_error": {"type": ["number", "null"], "minimum": 0},
        "lock_wait_spins": _INT, "remote_reads_issued": _INT, "remote_reads_skipped": _INT,
        "local_updates": _INT, "remote_updates": _INT,
    },
    "required": list(FIELDS),
    "additionalProperties": False,
}


def validate_record(record: dict) -> None:
    """Raise ``jsonschema.ValidationError`` unless ``record`` satisfies RECORD_SCHEMA."""
    import jsonschema

    jsonschema.validate(record, RECORD_SCHEMA, cls=jsonschema.Draft202012Validator)


class VerificationFailed(SptrsvError):
    """A run diverged from the serial reference by more than VERIFY_TOL."""


@dataclass(frozen=True)
class RunSpec:
    """One fully resolved benchmark run request (reference cli.py:57-80), plus the GPU knobs."""

    name: str
    matrix: CscMatrix
    rhs: np.ndarray
    engine: Engine = Engine.PARTITIONED_READ_ONLY
    n_pes: int = 1
    tasks_per_pe: int = 1
    workers_per_pe: int = 1
    repeats: int = 10
    timeout: float = 60.0
    remote_read_caching: bool = True
    verify: bool = True
    precision: str = "exact"
    executor: str = "auto"
    # verify against this serial solve (the reference checks against its own
    # Python loop, cli.py:166-167); None: this package's solve_serial, which
    # runs on the GPU, so max_rel_error is then GPU self-consistency only
    reference: Optional[Callable[[CscMatrix, np.ndarray], np.ndarray]] = None

    def config(self) -> SolverConfig:
        return SolverConfig(engine=self.engine, n_pes=self.n_pes, workers_per_pe=self.workers_per_pe,
                            timeout=self.timeout, remote_read_caching=self.remote_read_caching,
                            precision=self.precision, executor=self.executor)


def run_benchmark(spec: RunSpec) -> dict:
    """``repeats`` GPU solves + one serial-reference solve -> one record (cli.py:153-209)."""
    if spec.repeats < 1:
        raise InvalidSpec(f"repeats must be >= 1, got {spec.repeats}")
    stats = analysis.compute_stats(spec.matrix)
    plan = task_round_robin_partition(spec.matrix.n, spec.n_pes, spec.tasks_per_pe)
    cfg = spec.config()
    x_ref = (spec.reference or solve_serial)(spec.matrix, spec.rhs) if spec.verify else None
    solve_times, setup_times, combined = [], [], []
    max_rel_error = None
    report = None
    runs = 0
    for _ in range(spec.repeats):
        x, report = solve(spec.matrix, spec.rhs, plan, cfg)
        runs += 1
        solve_times.append(report.solve_time)
        setup_times.append(report.setup_time)
        combined.append(report.setup_time + report.solve_time)
        if x_ref is not None:
            cmp = compare_solutions(x, x_ref, VERIFY_TOL)
            if max_rel_error is None or cmp.max_rel_error > max_rel_error:
                max_rel_error = cmp.max_rel_error
            if not cmp.within_tol:
                raise VerificationFailed(
                    f"run diverged from the serial reference: max relative error {cmp.max_rel_error:.3e} > "
                    f"{VERIFY_TOL:g} at component {cmp.worst_component}")
    rollup = report.totals()
    values = (
        spec.name, spec.engine.value, spec.matrix.n, spec.matrix.nnz, stats.n_levels, stats.parallelism,
        stats.dependency, spec.n_pes, spec.tasks_per_pe, spec.workers_per_pe, spec.repeats, runs,
        sum(solve_times) / len(solve_times), min(solve_times), max(solve_times),
        sum(setup_times) / len(setup_times), sum(combined) / len(combined), max_rel_error,
        rollup["lock_wait_spins"], rollup["remote_reads_issued"], rollup["remote_reads_skipped"],
        rollup["local_updates"], rollup["remote_updates"],
    )
    return dict(zip(FIELDS, values))


def sweep_tasks(spec: RunSpec, tasks: list[int]) -> list[dict]:
    """One record per tasks_per_pe (reference cmd_sweep_tasks, cli.py:257-266)."""
    return [run_benchmark(replace(spec, tasks_per_pe=t)) for t in tasks]


def sweep_pes(spec: RunSpec, pes: list[int], fixed_total_tasks: int | None = None) -> list[dict]:
    """One record per PE count; with ``fixed_total_tasks`` each PE gets total / P tasks (cli.py:268-290)."""
    records = []
    for p in pes:
        tasks_per_pe = spec.tasks_per_pe
        if fixed_total_tasks is not None:
            if fixed_total_tasks % p != 0:
                raise IndivisibleTaskTotal(f"total task count {fixed_total_tasks} is not divisible by {p} PEs")
            tasks_per_pe = fixed_total_tasks // p
        records.append(run_benchmark(replace(spec, n_pes=p, tasks_per_pe=tasks_per_pe)))
    return records


def emit(records: list[dict], fmt: str = "json", out: str | None = None) -> str:
    """JSON lines or CSV (field order = column order, null = empty cell), to ``out`` or stdout (cli.py:212-227)."""
    if fmt == "json":
        text = "".join(json.dumps(r) + "\n" for r in records)
    else:
        buf = io.StringIO()
        writer = csv.DictWriter(buf, fieldnames=list(records[0]), lineterminator="\n")
        writer.writeheader()
        for r in records:
            writer.writerow({k: ("" if v is None else v) for k, v in r.items()})
        text = buf.getvalue()
    if out:
        Path(out).write_text(text)
    else:
        sys.stdout.write(text)
    return text
