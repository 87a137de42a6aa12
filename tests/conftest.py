"""Shared fixtures. ``-m gpu`` tests need a CUDA device and the built library."""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libsptrsv_b200.so")
    config.addinivalue_line("markers", "slow: large benchmark-size parity checks")


def load_reference_cases() -> dict[str, dict]:
    z = np.load(GOLDEN / "reference_cases.npz")
    cases: dict[str, dict] = {}
    for key in z.files:
        name, field = key.split("/")
        cases.setdefault(name, {})[field] = z[key]
    return cases


REFERENCE_CASES = load_reference_cases()


def case_matrix(case):
    from paper_2012_06959_b200 import CscMatrix

    return CscMatrix(n=int(case["n"]), col_ptr=case["col_ptr"], row_idx=case["row_idx"], values=case["values"])


@pytest.fixture(scope="session")
def reference_cases():
    return REFERENCE_CASES


@pytest.fixture
def worked_3x3():
    from paper_2012_06959_b200 import CscMatrix

    l = CscMatrix.from_entries(3, {(0, 0): 2.0, (1, 0): 1.0, (1, 1): 1.0, (2, 1): 3.0, (2, 2): 4.0})
    return l, np.array([2.0, 2.0, 7.0]), np.array([1.0, 1.0, 1.0])


def random_rhs(n: int, seed: int) -> np.ndarray:
    return np.random.default_rng((seed, 77)).uniform(-2.0, 2.0, size=n)


def gpu_available() -> bool:
    try:
        from paper_2012_06959_b200 import _native

        return _native.load_library().sptrsv_device_count() > 0
    except Exception:
        return False
