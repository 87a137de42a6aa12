"""Matrix Market ingestion (row f3): CPU tests of the parser against the
reference's error classes, GPU tests of parse + COO->CSC against fixtures
produced by the reference reader (tests/golden/make_mm_golden.py)."""

from __future__ import annotations

import numpy as np
import pytest

import paper_2012_06959_b200 as sp
from paper_2012_06959_b200 import mmio
from paper_2012_06959_b200.errors import (
    ComplexFieldUnsupported,
    IndexOutOfRange,
    MalformedEntry,
    MalformedHeader,
    NonSquare,
)
from conftest import ROOT

MM = np.load(ROOT / "tests" / "golden" / "mm_cases.npz")
NAMES = sorted({k.split("/")[0] for k in MM.files})


def _text(name):
    return MM[f"{name}/text"].tobytes().decode()


@pytest.mark.parametrize("text,exc", [
    ("", MalformedHeader),
    ("%%MatrixMarket matrix array real general\n2 2\n", MalformedHeader),
    ("%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n", ComplexFieldUnsupported),
    ("%%MatrixMarket matrix coordinate real skew-symmetric\n1 1 1\n1 1 1\n", MalformedHeader),
    ("%%MatrixMarket matrix coordinate real general\n2 3 1\n1 1 1\n", NonSquare),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1\n", IndexOutOfRange),
    ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1\n", MalformedEntry),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 x\n", MalformedEntry),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1\n", MalformedEntry),
    ("%%MatrixMarket matrix coordinate real general\n% only comments\n", MalformedHeader),
    # tokens the pandas tokenizer would read as NaN, and trailing comment text:
    # the reference's line parser rejects all of them
    ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 NA\n2 2 1\n", MalformedEntry),
    ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 null\n2 2 1\n", MalformedEntry),
    ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 3.0 % note\n2 2 1\n", MalformedEntry),
    ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 N/A\n2 2 1\n", MalformedEntry),
])
def test_parser_errors_match_reference_classes(text, exc):
    with pytest.raises(exc):
        mmio.parse_coo(text.encode())


def test_comment_lines_inside_the_block_are_skipped():
    n, r, c, v = mmio.parse_coo(b"%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.5\n% mid\n2 2 2.5\n")
    assert n == 2 and r.tolist() == [0, 1] and c.tolist() == [0, 1] and v.tolist() == [1.5, 2.5]


@pytest.mark.parametrize("name", NAMES)
def test_fast_and_slow_entry_parsers_agree(name):
    """The pandas block parser gives exactly the line parser's COO (same doubles)."""
    text = _text(name)
    lines = text.splitlines()
    field, symmetry, n, n_decl, first = mmio._header(lines)
    slow = mmio._entries_slow(lines, first, n, n_decl, field == "pattern")
    body = "\n".join(lines[first:])
    fast = mmio._entries_fast(body, n, n_decl, field == "pattern")
    if n_decl == 0 or "%" in body:  # comment lines: the line parser handles the block
        assert fast is None
        return
    assert fast is not None
    for a, b in zip(fast, slow):
        assert a.tobytes() == b.tobytes()


def test_writer_round_trip_text():
    l = sp.synth.lap2d(7, 5)
    s = mmio.matrix_market_string(l, comment="lap2d 7x5")
    n, rows, cols, vals = mmio.parse_coo(s.encode())
    assert n == l.n
    np.testing.assert_array_equal(rows, l.row_idx)
    np.testing.assert_array_equal(cols, l.entry_columns())
    assert vals.tobytes() == l.values.tobytes()


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_parse_matrix_market_equals_reference(name):
    a = mmio.parse_matrix_market(_text(name).encode())
    assert a.col_ptr.tobytes() == MM[f"{name}/col_ptr"].astype(np.int64).tobytes()
    assert a.row_idx.tobytes() == MM[f"{name}/row_idx"].astype(np.int64).tobytes()
    assert a.values.tobytes() == MM[f"{name}/values"].tobytes()
    if f"{name}/lower_col_ptr" in MM.files:
        low = mmio.read_lower_triangular(_text(name).encode(), sp.DiagonalPolicy.INSERT_UNIT)
        assert low.col_ptr.tobytes() == MM[f"{name}/lower_col_ptr"].astype(np.int64).tobytes()
        assert low.row_idx.tobytes() == MM[f"{name}/lower_row_idx"].astype(np.int64).tobytes()
        assert low.values.tobytes() == MM[f"{name}/lower_values"].tobytes()


@pytest.mark.gpu
def test_read_write_solve_round_trip(tmp_path):
    l = sp.synth.banded(3000, 16, 0.5, 3)
    path = tmp_path / "banded.mtx"
    mmio.write_matrix_market(l, path)
    back = mmio.read_lower_triangular(path)
    assert back.col_ptr.tobytes() == l.col_ptr.tobytes()
    assert back.row_idx.tobytes() == l.row_idx.tobytes()
    assert back.values.tobytes() == l.values.tobytes()
