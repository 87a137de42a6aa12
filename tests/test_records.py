"""CPU: record emission in the reference's JSON-lines / CSV formats (row f2)."""

from __future__ import annotations

import csv
import io
import json

from paper_2012_06959_b200 import records


def _rec(**kw):
    r = dict.fromkeys(records.FIELDS, 0)
    r.update(name="m", engine="shared", max_rel_error=None, mean_wall_time=1.5e-3)
    r.update(kw)
    return r


def test_fields_match_schema_order():
    assert len(records.FIELDS) == 23 and records.FIELDS[:3] == ("name", "engine", "n")
    assert records.FIELDS[-1] == "remote_updates"


def test_emit_json_and_csv(tmp_path, capsys):
    recs = [_rec(), _rec(name="k", engine="partitioned", max_rel_error=0.0)]
    text = records.emit(recs, "json")
    assert capsys.readouterr().out == text
    lines = [json.loads(line) for line in text.splitlines()]
    assert list(lines[0]) == list(records.FIELDS) and lines[0]["max_rel_error"] is None
    out = tmp_path / "r.csv"
    text = records.emit(recs, "csv", str(out))
    assert out.read_text() == text
    rows = list(csv.reader(io.StringIO(text)))
    assert rows[0] == list(records.FIELDS)
    assert rows[1][records.FIELDS.index("max_rel_error")] == ""  # null -> empty cell
    assert rows[2][records.FIELDS.index("engine")] == "partitioned"


def _valid(**kw):
    r = dict.fromkeys(records.FIELDS, 1)
    r.update(name="m", engine="partitioned", dependency=3.0, mean_wall_time=1e-3, min_wall_time=1e-3,
             max_wall_time=1e-3, mean_setup_time=0.1, mean_combined_time=0.101, max_rel_error=0.0)
    r.update(kw)
    return r


def test_schema_validation():
    import jsonschema
    import pytest

    records.validate_record(_valid())
    records.validate_record(_valid(max_rel_error=None))
    for bad in (dict(engine="gpu"), dict(n=0), dict(dependency=0.0), dict(max_rel_error=-1.0),
                dict(lock_wait_spins=1.5), dict(extra=1)):
        with pytest.raises(jsonschema.ValidationError):
            records.validate_record(_valid(**bad))
    r = _valid()
    del r["remote_updates"]
    with pytest.raises(jsonschema.ValidationError):
        records.validate_record(r)
