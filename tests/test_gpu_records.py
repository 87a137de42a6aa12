"""GPU: benchmark records in the reference's schema (row f2): field set and
order, engine enum, verification, the PE sweep with a fixed task total."""

from __future__ import annotations

import csv
import io
import json

import numpy as np
import pytest

import oracle
import paper_2012_06959_b200 as sp
from paper_2012_06959_b200 import records, synth
from paper_2012_06959_b200.errors import IndivisibleTaskTotal, InvalidSpec

pytestmark = pytest.mark.gpu

# docs/record_schema.json of the reference: required fields, this order
REQUIRED = ["name", "engine", "n", "nnz", "n_levels", "parallelism", "dependency", "n_pes", "tasks_per_pe",
            "workers_per_pe", "repeats", "engine_runs", "mean_wall_time", "min_wall_time", "max_wall_time",
            "mean_setup_time", "mean_combined_time", "max_rel_error", "lock_wait_spins", "remote_reads_issued",
            "remote_reads_skipped", "local_updates", "remote_updates"]


def _oracle_serial(l, b):
    # the independent CPU check (the reference verifies against its own serial loop)
    return oracle.solve_serial(l.col_ptr, l.row_idx, l.values, b)


def _spec(**kw):
    l = synth.lap2d(48, 40)
    kw.setdefault("reference", _oracle_serial)
    return records.RunSpec(name="lap2d-48x40", matrix=l, rhs=np.random.default_rng(3).uniform(-1, 1, l.n),
                           repeats=3, **kw)


def test_record_fields_and_values():
    r = records.run_benchmark(_spec())
    assert list(r) == REQUIRED
    records.validate_record(r)
    assert r["engine"] in ("shared", "partitioned")
    assert r["n"] == 1920 and r["n_levels"] == 48 + 40 - 1 and r["engine_runs"] == 3
    assert r["max_rel_error"] == 0.0  # exact mode: bit-identical to the C oracle
    assert 0 <= r["min_wall_time"] <= r["mean_wall_time"] <= r["max_wall_time"]
    assert r["local_updates"] + r["remote_updates"] == r["nnz"] - r["n"]


def test_sweeps_and_emit(tmp_path):
    base = _spec(engine=sp.Engine.SHARED_ATOMICS, precision="fast")
    recs = records.sweep_pes(base, [1, 2, 4], fixed_total_tasks=32)
    assert [r["tasks_per_pe"] for r in recs] == [32, 16, 8]
    assert [r["n_pes"] for r in recs] == [1, 2, 4]
    assert all(r["engine"] == "shared" for r in recs)
    with pytest.raises(IndivisibleTaskTotal):
        records.sweep_pes(base, [3], fixed_total_tasks=32)
    recs += records.sweep_tasks(base, [1, 4])
    for r in recs:
        records.validate_record(r)
        assert 0.0 <= r["max_rel_error"] <= 1e-12  # fast mode vs the C oracle
    text = records.emit(recs, "json", str(tmp_path / "r.jsonl"))
    assert [json.loads(line)["tasks_per_pe"] for line in text.splitlines()] == [32, 16, 8, 1, 4]
    text = records.emit(recs, "csv", str(tmp_path / "r.csv"))
    rows = list(csv.DictReader(io.StringIO(text)))
    assert list(rows[0]) == REQUIRED and len(rows) == 5
    with pytest.raises(InvalidSpec):
        records.run_benchmark(_spec().__class__(**{**_spec().__dict__, "repeats": 0}))
