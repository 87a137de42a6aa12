"""Pin the CPU oracle against the reference's own outputs (CPU only).

The golden fixtures were produced by running the reference package
(tests/golden/make_golden.py). The oracle must reproduce every one of them
bit for bit before it is trusted as the checker of the CUDA path.
"""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

import oracle
from conftest import GOLDEN, REFERENCE_CASES


@pytest.mark.parametrize("name", sorted(REFERENCE_CASES))
def test_oracle_matches_reference_goldens(name):
    c = REFERENCE_CASES[name]
    np.testing.assert_array_equal(oracle.in_degrees(c["col_ptr"], c["row_idx"]), c["in_degree"])
    lv, nl = oracle.levels(c["col_ptr"], c["row_idx"])
    np.testing.assert_array_equal(lv, c["level_of"])
    assert nl == int(c["n_levels"])
    if "x" in c:
        x = oracle.solve_serial(c["col_ptr"], c["row_idx"], c["values"], c["b"])
        # bitwise: same IEEE operations in the same order as the Python loop
        assert x.tobytes() == c["x"].tobytes()


def test_python_restatement_agrees_with_c(reference_cases):
    for name in ("worked_3x3", "random_0", "random_5", "fanout8"):
        c = reference_cases[name]
        a = oracle.solve_serial(c["col_ptr"], c["row_idx"], c["values"], c["b"])
        b = oracle.solve_serial_py(c["col_ptr"], c["row_idx"], c["values"], c["b"])
        assert a.tobytes() == b.tobytes()


def test_lap2d_256_config0_against_reference_run():
    from paper_2012_06959_b200 import synth

    z = np.load(GOLDEN / "lap2d_256.npz")
    l = synth.lap2d(256)
    digest = hashlib.sha256(l.col_ptr.tobytes() + l.row_idx.tobytes() + l.values.tobytes()).hexdigest()
    assert digest == str(z["sha256"])  # same matrix the reference solved
    x = oracle.solve_serial(l.col_ptr, l.row_idx, l.values, np.ones(l.n))
    assert x.tobytes() == z["x_ones"].tobytes()
    x = oracle.solve_serial(l.col_ptr, l.row_idx, l.values, z["b_rand"])
    assert x.tobytes() == z["x_rand"].tobytes()
    np.testing.assert_array_equal(oracle.in_degrees(l.col_ptr, l.row_idx), z["in_degree"])
    lv, nl = oracle.levels(l.col_ptr, l.row_idx)
    np.testing.assert_array_equal(lv, z["level_of"])
    assert nl == int(z["n_levels"]) == 511


def test_markstein_division_is_ieee():
    # the kernels' correctly-rounded division trick, restated on the CPU
    assert oracle.markstein_mismatches(2_000_000, seed=7) == 0


def test_oracle_spmv_matches_numpy(reference_cases):
    c = reference_cases["random_3"]
    from paper_2012_06959_b200 import CscMatrix, spmv_lower

    l = CscMatrix(n=int(c["n"]), col_ptr=c["col_ptr"], row_idx=c["row_idx"], values=c["values"])
    x = c["x"]
    assert oracle.spmv(c["col_ptr"], c["row_idx"], c["values"], x).tobytes() == spmv_lower(l, x).tobytes()
