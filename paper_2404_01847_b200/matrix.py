"""Error types and small enums mirroring sparse24.matrix (matrix.py:11-90)."""

from __future__ import annotations

from enum import Enum


class ShapeError(ValueError):
    """Operand shapes violate an operation's preconditions (matrix.py:11)."""


class FormatError(ValueError):
    """A mask or compressed buffer violates its structural invariants (matrix.py:15)."""


class Layout(Enum):
    ROW_MAJOR = "row_major"
    COL_MAJOR = "col_major"


class Direction(Enum):
    """Axis along which 2:4 groups of four consecutive elements run (matrix.py:24-28)."""

    ROW_WISE = "row_wise"
    COL_WISE = "col_wise"
