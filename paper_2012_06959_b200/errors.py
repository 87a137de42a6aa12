"""Error taxonomy of the drop-in solver.

The class names are the diagnostic contract of the reference package
(`/root/reference/pkg/src/sptrsv/errors.py:1-83`): callers and the CLI match on
them, so every name and base class is kept. The native library reports the
same conditions as integer status codes (`include/sptrsv_b200.h`,
``SPTRSV_E_*``); :func:`raise_for_status` maps each code back to its class.
"""

from __future__ import annotations


class SptrsvError(Exception):
    """Root of every error raised by this package (errors.py:10)."""


class MatrixMarketError(SptrsvError):
    """Matrix Market parsing failure (errors.py:16); ingestion is out of scope here."""


class MalformedHeader(MatrixMarketError):
    pass


class MalformedEntry(MatrixMarketError):
    pass


class NonSquare(MatrixMarketError):
    pass


class IndexOutOfRange(MatrixMarketError):
    pass


class ComplexFieldUnsupported(MatrixMarketError):
    pass


class MatrixStructureError(SptrsvError):
    """CSC arrays do not describe a well-formed square sparse matrix (errors.py:42)."""


class MissingDiagonal(SptrsvError):
    """A column stores no diagonal entry (errors.py:46)."""

    def __init__(self, col: int):
        self.col = int(col)
        super().__init__(f"column {self.col} has no stored diagonal entry")


class ZeroDiagonal(SptrsvError):
    """A stored diagonal entry is exactly zero (errors.py:52)."""

    def __init__(self, col: int):
        self.col = int(col)
        super().__init__(f"stored diagonal of column {self.col} is exactly 0")


class InvalidSpec(SptrsvError):
    """A synthetic-matrix recipe is inconsistent (errors.py:58)."""


class DimensionMismatch(SptrsvError):
    """Operand shapes disagree (errors.py:62)."""


class InvalidPeCount(SptrsvError):
    """PE count outside the admissible range (errors.py:68)."""


class TooManyTasks(SptrsvError):
    """More component tasks requested than components exist (errors.py:72)."""


class IndivisibleTaskTotal(SptrsvError):
    """A fixed task total does not divide over the PE count (errors.py:76)."""


class SolveTimeout(SptrsvError):
    """The device watchdog tripped: a solve did not finish in the configured bound (errors.py:82)."""


class NativeUnavailable(SptrsvError):
    """The CUDA library is missing or no CUDA device is visible.

    There is no CPU fallback: every solve, in-degree and level computation of
    this package runs on the GPU, so a missing extension is a hard error.
    """


# Status codes of the C ABI (include/sptrsv_b200.h). Kept in one place so the
# header, the ctypes shim and the tests agree.
STATUS_OK = 0
STATUS_DIMENSION = 1
STATUS_ZERO_DIAGONAL = 2
STATUS_MISSING_DIAGONAL = 3
STATUS_STRUCTURE = 4
STATUS_TIMEOUT = 5
STATUS_INVALID_PE = 6
STATUS_CUDA = 7
STATUS_ARGUMENT = 8
STATUS_UNSUPPORTED = 9
STATUS_DEBUG_CHECK = 10  # a SPTRSV_PLAN_DEBUG device check failed


def raise_for_status(status: int, detail: str = "", col: int = -1) -> None:
    """Translate a native status code into the reference exception class."""
    if status == STATUS_OK:
        return
    if status == STATUS_ZERO_DIAGONAL:
        raise ZeroDiagonal(col)
    if status == STATUS_MISSING_DIAGONAL:
        raise MissingDiagonal(col)
    if status == STATUS_STRUCTURE:
        raise MatrixStructureError(detail or "not lower triangular")
    if status == STATUS_DIMENSION:
        raise DimensionMismatch(detail)
    if status == STATUS_TIMEOUT:
        raise SolveTimeout(detail)
    if status == STATUS_INVALID_PE:
        raise InvalidPeCount(detail)
    if status == STATUS_ARGUMENT:
        raise ValueError(detail)
    if status == STATUS_DEBUG_CHECK:
        # the reference's debug mode raises AssertionError (engine.py:163-168, 511-513)
        raise AssertionError(detail)
    raise SptrsvError(f"native status {status}: {detail}")
