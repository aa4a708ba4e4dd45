"""Operator protocol (krecycle.operators drop-in).

``CountingOperator`` is the matvec meter whose counts the sequence policy
reports (reference operators.py:50-88).  The device solvers increment a
caller-supplied CountingOperator by exactly the products the reference would
have routed through it.
"""

from __future__ import annotations

import numpy as np


def as_operator(A):
    """Return A when it implements the operator protocol (operators.py:41-47).
    Dense arrays are accepted by the device solvers directly (converted to
    CSR on upload)."""
    if hasattr(A, "shape") and (hasattr(A, "matvec") or hasattr(A, "row_ptr")
                                or hasattr(A, "_device")):
        return A
    if isinstance(A, np.ndarray):
        return A
    raise TypeError(f"cannot interpret {type(A).__name__} as a linear operator")


class CountingOperator:
    """Counts matvec and rmatvec applications (operators.py:50-88)."""

    def __init__(self, op):
        self._op = as_operator(op)
        self.n_matvec = 0
        self.n_rmatvec = 0

    @property
    def inner(self):
        return self._op

    @property
    def shape(self):
        return self._op.shape

    @property
    def dtype(self):
        return getattr(self._op, "dtype", np.float64)

    @property
    def total(self) -> int:
        return self.n_matvec + self.n_rmatvec

    def reset(self):
        self.n_matvec = 0
        self.n_rmatvec = 0

    def matvec(self, x):
        self.n_matvec += 1
        return self._op.matvec(x)

    def rmatvec(self, x):
        self.n_rmatvec += 1
        return self._op.rmatvec(x)
