"""ILUTP split preconditioning (drop-in for krecycle.ilutp,
/root/reference/pkg/src/krecycle/ilutp.py).

``ilutp_factor`` runs the reference's row-wise ILUTP elimination in libkrb's
host code (krb_ilutp_factor, csrc/ilutp.cu): the same operations in the
same order, so L, U and perm equal krecycle's bit for bit.  The factors are
then applied on the device: ``L^{-1}``, ``U^{-1}`` and their adjoints are
level-scheduled triangular solves (csrc/ilutp.cu kernels), and
``SplitPreconditionedOperator`` (ilutp.py:106-128) is the device operator
``L^{-1} A P U^{-1}`` the solvers iterate on.

Summation order of a triangular solve (canonical, tests/oracle): row i
computes s = b_i, then s = s - l_ij x_j for its off-diagonal entries in
column order (one rounding per multiply and per subtract), then x_i = s for
the unit-diagonal L, x_i = s / u_ii for U.  The reference applies the factors
through SuperLU's supernodal solve, whose order differs in the last bits;
parity with the reference is therefore statistical, like every reduction on
the path (tests/test_gpu_ilutp.py).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .sparse import SparseMatrix


class FactorizationError(RuntimeError):
    """Raised when elimination encounters a structurally zero pivot
    (ilutp.py:34-35)."""


@dataclass
class IlutpFactors:
    """Factors of ``A*P ~= L*U`` plus the column permutation (ilutp.py:46-74).
    ``perm[j]`` is the original column stored at permuted position j."""

    L: SparseMatrix
    U: SparseMatrix
    perm: np.ndarray
    _dev: object = field(default=None, repr=False, compare=False)

    @property
    def n(self) -> int:
        return self.L.nrows

    def device(self):
        """The device-resident factors (built on first use)."""
        if self._dev is None:
            from .precond import DeviceFactors
            self._dev = DeviceFactors(self)
        return self._dev

    def solve_lower(self, b, adjoint=False):
        return self.device().host_apply("lower_h" if adjoint else "lower", b)

    def solve_upper(self, b, adjoint=False):
        return self.device().host_apply("upper_h" if adjoint else "upper", b)


def ilutp_factor(A, drop_tol: float = 1e-4, pivot_tol: float = 0.1,
                 fill_limit: int | None = None) -> IlutpFactors:
    """Row-wise ILUTP factorization (ilutp.py:131-281), bit-identical to the
    reference; raises FactorizationError / ValueError as it does."""
    n = A.nrows if hasattr(A, "nrows") else A.shape[0]
    ncols = A.ncols if hasattr(A, "ncols") else A.shape[1]
    if ncols != n:
        raise ValueError("ilutp_factor requires a square matrix")
    vals = np.asarray(A.values)
    if np.iscomplexobj(vals):
        raise NotImplementedError("complex matrices are out of scope on the B200 path")
    rp = np.ascontiguousarray(A.row_ptr, dtype=np.int64)
    ci = np.ascontiguousarray(A.col_idx, dtype=np.int32)
    vals = np.ascontiguousarray(vals, dtype=np.float64)
    lib = _lib.load()
    h = ctypes.c_void_p()
    rc = lib.krb_ilutp_factor(n, rp.ctypes.data, ci.ctypes.data, vals.ctypes.data,
                              float(drop_tol), float(pivot_tol),
                              -1 if fill_limit is None else int(fill_limit), ctypes.byref(h))
    if rc != 0:
        msg = lib.krb_last_error().decode()
        if rc == -5:
            raise FactorizationError(msg)
        _lib.check(rc, "krb_ilutp_factor")
    try:
        nl, nu = ctypes.c_int64(), ctypes.c_int64()
        _lib.call("krb_ilutp_sizes", h, ctypes.byref(nl), ctypes.byref(nu))
        Lrp = np.empty(n + 1, np.int64)
        Urp = np.empty(n + 1, np.int64)
        Lci = np.empty(nl.value, np.int32)
        Uci = np.empty(nu.value, np.int32)
        Lv = np.empty(nl.value, np.float64)
        Uv = np.empty(nu.value, np.float64)
        perm = np.empty(n, np.int64)
        _lib.call("krb_ilutp_export", h, *(a.ctypes.data for a in
                                           (Lrp, Lci, Lv, Urp, Uci, Uv, perm)))
    finally:
        lib.krb_ilutp_free(h)
    L = SparseMatrix(n, n, Lrp, Lci, Lv)
    U = SparseMatrix(n, n, Urp, Uci, Uv)
    return IlutpFactors(L=L, U=U, perm=perm)


def apply_left(factors, x):
    """``L^{-1} x`` (ilutp.py:76-78)."""
    return _factors(factors).solve_lower(np.asarray(x))


def apply_left_h(factors, x):
    """``L^{-H} x`` (ilutp.py:81-83)."""
    return _factors(factors).solve_lower(np.asarray(x), adjoint=True)


def apply_right(factors, y):
    """``P U^{-1} y`` (ilutp.py:86-91)."""
    F = _factors(factors)
    t = F.solve_upper(np.asarray(y))
    x = np.empty_like(t)
    x[F.perm] = t
    return x


def apply_right_h(factors, x):
    """``U^{-H} P^T x`` (ilutp.py:94-97)."""
    F = _factors(factors)
    z = np.asarray(x)[F.perm]
    return F.solve_upper(z, adjoint=True)


def to_operator_coords(factors, x):
    """``y = U (P^T x)`` (ilutp.py:100-103)."""
    F = _factors(factors)
    z = np.asarray(x)[F.perm]
    return F.U.matvec(z)


def permutation_matrix(factors):
    """P as a scipy sparse matrix (ilutp.py:284-289)."""
    import scipy.sparse as sp
    F = _factors(factors)
    n = F.n
    return sp.csr_matrix((np.ones(n), (F.perm, np.arange(n))), shape=(n, n))


def _factors(f):
    """Adopt a reference IlutpFactors (numpy L / U / perm) or pass ours."""
    if isinstance(f, IlutpFactors):
        return f
    cache = getattr(f, "_b200", None)
    if cache is not None:
        return cache

    def adopt(M):
        return SparseMatrix(M.nrows, M.ncols, M.row_ptr, M.col_idx, M.values)
    ours = IlutpFactors(L=adopt(f.L), U=adopt(f.U), perm=np.asarray(f.perm, dtype=np.int64))
    try:
        object.__setattr__(f, "_b200", ours)
    except Exception:
        pass
    return ours


class SplitPreconditionedOperator:
    """Operator ``L^{-1} A P U^{-1}`` with its adjoint (ilutp.py:106-128).
    The solvers of this package run it entirely on the device (the
    triangular solves and the SpMV are kernels of the iteration); matvec /
    rmatvec here serve host callers."""

    def __init__(self, A, factors):
        shape = A.shape if hasattr(A, "shape") else (A.nrows, A.ncols)
        F = _factors(factors)
        if shape[0] != shape[1] or shape[0] != F.n:
            raise ValueError("operator and factor dimensions disagree")
        self._A = A
        self.factors = F
        self._dtype = np.result_type(getattr(A, "dtype", np.float64), F.U.values.dtype)

    @property
    def shape(self):
        return self._A.shape if hasattr(self._A, "shape") else (self._A.nrows, self._A.ncols)

    @property
    def dtype(self):
        return self._dtype

    def matvec(self, x):
        from .precond import device_operator
        return device_operator(self).host_matvec(np.asarray(x))

    def rmatvec(self, x):
        from .precond import device_operator
        return device_operator(self).host_matvec(np.asarray(x), adjoint=True)
