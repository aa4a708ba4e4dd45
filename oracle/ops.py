"""Numerical primitive sets for the oracle restatement — TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this package.  The product path never calls it.

Two interchangeable primitive sets drive the same restated algorithms
(oracle/krylov.py):

``RefOps``
    the exact numpy/scipy calls the reference makes (np.vdot, np.linalg.norm,
    ``M.conj().T @ v``, ``M @ y``, scipy CSR ``@``), so the restatement is
    bit-identical to /root/reference/pkg/src/krecycle at a fixed OpenBLAS
    thread count (pinned by tests/golden, generated from the reference itself).

``CanonOps``
    the fixed-order primitives of oracle/canon.c.  The B200 kernels evaluate
    the same orders, so GPU results equal this oracle bit for bit.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np
import scipy.sparse as _sp

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def build_canon() -> str:
    """Compile oracle/libcanon.so (gcc, seconds)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return os.path.join(_HERE, "libcanon.so")


def _lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "libcanon.so")
        src = os.path.join(_HERE, "canon.c")
        if (not os.path.exists(path)
                or os.path.getmtime(path) < os.path.getmtime(src)):
            build_canon()
        lib = ctypes.CDLL(path)
        P = ctypes.c_void_p
        I = ctypes.c_int64
        lib.canon_E.restype = I
        lib.canon_E.argtypes = [I]
        lib.canon_R.restype = I
        lib.canon_R.argtypes = [I]
        lib.canon_nblocks.restype = I
        lib.canon_nblocks.argtypes = [I]
        lib.canon_dot.restype = ctypes.c_double
        lib.canon_dot.argtypes = [I, P, I, P, I]
        lib.canon_final.restype = ctypes.c_double
        lib.canon_final.argtypes = [I, P, I]
        lib.canon_dot_partials.restype = None
        lib.canon_dot_partials.argtypes = [I, P, I, P, I, P]
        lib.canon_tdot.restype = None
        lib.canon_tdot.argtypes = [I, I, P, I, I, P, P]
        lib.canon_gemv.restype = None
        lib.canon_gemv.argtypes = [I, I, P, I, I, P, P]
        lib.canon_spmv.restype = None
        lib.canon_spmv.argtypes = [I, P, P, P, P, P]
        lib.canon_gram.restype = None
        lib.canon_gram.argtypes = [I, I, I, P, I, I, P, I, I, P]
        lib.canon_trsv.restype = None
        lib.canon_trsv.argtypes = [I, P, P, P, P, ctypes.c_int, P, P]
        lib.canon_gemm.restype = None
        lib.canon_gemm.argtypes = [I, I, I, P, I, I, P, P, I, I]
        _LIB = lib
    return _LIB


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _strides(M: np.ndarray):
    return M.strides[0] // M.itemsize, M.strides[1] // M.itemsize


def _real(a, what):
    a = np.asarray(a)
    if np.iscomplexobj(a):
        raise NotImplementedError(f"{what}: complex data is out of scope")
    return np.asarray(a, dtype=np.float64)


class CsrOperand:
    """Canonical CSR handed to the oracle (row_ptr int64, col_idx int32)."""

    def __init__(self, n, row_ptr, col_idx, values):
        self.nrows = self.ncols = int(n)
        self.row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
        self.col_idx = np.ascontiguousarray(col_idx, dtype=np.int32)
        self.values = np.ascontiguousarray(values, dtype=np.float64)
        self._csr = _sp.csr_matrix((self.values, self.col_idx, self.row_ptr),
                                   shape=(self.nrows, self.ncols))
        self._csr_h = None
        self._t = None

    @classmethod
    def of(cls, A):
        if isinstance(A, (cls, SplitOperand)):
            return A
        if hasattr(A, "factors") and hasattr(A, "_A"):
            return SplitOperand(cls.of(A._A), A.factors)
        inner = getattr(A, "inner", None)
        if inner is not None and not hasattr(A, "row_ptr"):
            return cls.of(inner)
        if hasattr(A, "row_ptr"):
            return cls(A.nrows if hasattr(A, "nrows") else A.n, A.row_ptr,
                       A.col_idx, A.values)
        raise TypeError(f"oracle needs a CSR operand, got {type(A).__name__}")

    @property
    def shape(self):
        return (self.nrows, self.ncols)

    @property
    def dtype(self):
        return self.values.dtype

    def transpose_arrays(self):
        """Explicit A^T in canonical CSR, as scipy builds it for rmatvec
        (/root/reference/pkg/src/krecycle/sparse.py:128-129)."""
        if self._t is None:
            T = self._csr.transpose().tocsr()
            T.sort_indices()
            self._t = (T.indptr.astype(np.int64), T.indices.astype(np.int32),
                       T.data.astype(np.float64))
        return self._t


def _tri_offdiag(M, unit):
    """Off-diagonal CSR and diagonal of a triangular scipy CSR."""
    rp = M.indptr.astype(np.int64)
    ci = M.indices.astype(np.int64)
    v = M.data.astype(np.float64)
    n = M.shape[0]
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(rp))
    off = ci != rows
    diag = None
    if not unit:
        diag = np.zeros(n)
        diag[rows[~off]] = v[~off]
    rp_off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows[off], minlength=n), out=rp_off[1:])
    return (rp_off, np.ascontiguousarray(ci[off], dtype=np.int32),
            np.ascontiguousarray(v[off]), diag)


class SplitOperand:
    """The split-ILUTP operator L^{-1} A P U^{-1} (ilutp.py:106-128) handed to
    the oracle: base CSR operand + factors (L, U CSR, perm)."""

    def __init__(self, base, factors):
        self.base = base
        self.nrows = self.ncols = base.nrows
        self.perm = np.asarray(factors.perm, dtype=np.int64)
        n = base.nrows

        def csr(M):
            return _sp.csr_matrix((np.asarray(M.values, dtype=np.float64),
                                   np.asarray(M.col_idx), np.asarray(M.row_ptr)),
                                  shape=(n, n))
        self.L, self.U = csr(factors.L), csr(factors.U)
        self._lu = None
        self._tri = None

    @property
    def shape(self):
        return (self.nrows, self.ncols)

    @property
    def dtype(self):
        return np.dtype(np.float64)

    def tri(self):
        """canonical-order data: (L, L^T, U, U^T) off-diagonal CSR + diag"""
        if self._tri is None:
            Lt = self.L.T.tocsr()
            Lt.sort_indices()
            Ut = self.U.T.tocsr()
            Ut.sort_indices()
            self._tri = {"L": (_tri_offdiag(self.L, True), 1),
                         "Lt": (_tri_offdiag(Lt, True), 0),
                         "U": (_tri_offdiag(self.U, False), 0),
                         "Ut": (_tri_offdiag(Ut, False), 1)}
        return self._tri

    def superlu(self):
        """the reference's factor application (ilutp.py:37-42: SuperLU,
        natural order, no pivoting, on each triangular factor)"""
        if self._lu is None:
            import scipy.sparse.linalg as spla
            self._lu = tuple(spla.splu(M.tocsc(), permc_spec="NATURAL",
                                       diag_pivot_thresh=0.0) for M in (self.L, self.U))
        return self._lu


class RefOps:
    """The reference's own numpy/scipy calls (bit-identical restatement)."""

    name = "ref"

    def matvec(self, A: CsrOperand, x):
        if isinstance(A, SplitOperand):   # ilutp.py:124-125 / 76-91
            luL, luU = A.superlu()
            t = luU.solve(np.asarray(x))
            y = np.empty_like(t)
            y[A.perm] = t
            return luL.solve(self.matvec(A.base, y))
        return A._csr @ x

    def rmatvec(self, A: CsrOperand, x):
        if isinstance(A, SplitOperand):   # ilutp.py:127-128 / 81-97
            luL, luU = A.superlu()
            z = self.rmatvec(A.base, luL.solve(np.asarray(x), trans="H"))
            return luU.solve(z[A.perm], trans="H")
        if A._csr_h is None:
            A._csr_h = A._csr.conj(copy=True).transpose().tocsr()
        return A._csr_h @ x

    def dot(self, x, y):
        return np.vdot(x, y)

    def norm(self, x):
        return np.linalg.norm(x)

    def tdot(self, M, v):
        return M.conj().T @ v

    def gemv(self, M, y):
        return M @ y

    def gram(self, X, Y):
        return X.conj().T @ Y

    def colnorms(self, X):
        return np.linalg.norm(X, axis=0)

    def gemm(self, X, Z):
        return X @ Z


class CanonOps:
    """Fixed-order primitives of oracle/canon.c (the GPU's bitwise target)."""

    name = "canon"

    def __init__(self):
        self.lib = _lib()

    def trsv(self, A, which, b):
        (rp, ci, v, diag), lower = A.tri()[which]
        b = np.ascontiguousarray(_real(b, "trsv"))
        x = np.empty(A.nrows)
        self.lib.canon_trsv(A.nrows, _ptr(rp), _ptr(ci), _ptr(v),
                            _ptr(diag) if diag is not None else None, lower,
                            _ptr(b), _ptr(x))
        return x

    def matvec(self, A: CsrOperand, x):
        if isinstance(A, SplitOperand):   # L^{-1} A P U^{-1} x
            t = self.trsv(A, "U", x)
            y = np.empty_like(t)
            y[A.perm] = t
            return self.trsv(A, "L", self.matvec(A.base, y))
        x = np.ascontiguousarray(_real(x, "matvec"))
        y = np.empty(A.nrows)
        self.lib.canon_spmv(A.nrows, _ptr(A.row_ptr), _ptr(A.col_idx),
                            _ptr(A.values), _ptr(x), _ptr(y))
        return y

    def rmatvec(self, A: CsrOperand, x):
        if isinstance(A, SplitOperand):   # U^{-H} P^T A^H L^{-H} x
            z = self.rmatvec(A.base, self.trsv(A, "Lt", x))
            return self.trsv(A, "Ut", z[A.perm])
        rp, ci, v = A.transpose_arrays()
        x = np.ascontiguousarray(_real(x, "rmatvec"))
        y = np.empty(A.ncols)
        self.lib.canon_spmv(A.ncols, _ptr(rp), _ptr(ci), _ptr(v), _ptr(x),
                            _ptr(y))
        return y

    def dot(self, x, y):
        x = np.ascontiguousarray(_real(x, "dot"))
        y = np.ascontiguousarray(_real(y, "dot"))
        return np.float64(self.lib.canon_dot(x.shape[0], _ptr(x), 1, _ptr(y), 1))

    def norm(self, x):
        return np.sqrt(self.dot(x, x))

    def tdot(self, M, v):
        M = _real(M, "tdot")
        v = np.ascontiguousarray(_real(v, "tdot"))
        out = np.empty(M.shape[1])
        rs, cs = _strides(M)
        self.lib.canon_tdot(M.shape[0], M.shape[1], _ptr(M), rs, cs, _ptr(v),
                            _ptr(out))
        return out

    def gemv(self, M, y):
        M = _real(M, "gemv")
        y = np.ascontiguousarray(_real(y, "gemv"))
        out = np.empty(M.shape[0])
        rs, cs = _strides(M)
        self.lib.canon_gemv(M.shape[0], M.shape[1], _ptr(M), rs, cs, _ptr(y),
                            _ptr(out))
        return out

    def gram(self, X, Y):
        X = _real(X, "gram")
        Y = _real(Y, "gram")
        G = np.empty((X.shape[1], Y.shape[1]))
        rx, cx = _strides(X)
        ry, cy = _strides(Y)
        self.lib.canon_gram(X.shape[0], X.shape[1], Y.shape[1], _ptr(X), rx, cx,
                            _ptr(Y), ry, cy, _ptr(G))
        return G

    def colnorms(self, X):
        X = _real(X, "colnorms")
        out = np.empty(X.shape[1])
        for j in range(X.shape[1]):
            col = np.ascontiguousarray(X[:, j])
            out[j] = np.sqrt(self.dot(col, col))
        return out

    def gemm(self, X, Z):
        X = _real(X, "gemm")
        Z = np.ascontiguousarray(_real(Z, "gemm"))
        out = np.empty((X.shape[0], Z.shape[1]), order="F")
        rx, cx = _strides(X)
        ro, co = _strides(out)
        self.lib.canon_gemm(X.shape[0], X.shape[1], Z.shape[1], _ptr(X), rx, cx,
                            _ptr(Z), _ptr(out), ro, co)
        return out

    # raw access for kernel-level tests
    def E(self, n):
        return int(self.lib.canon_E(n))

    def R(self, n):
        return int(self.lib.canon_R(n))

    def nblocks(self, n):
        return int(self.lib.canon_nblocks(n))


def make_ops(name: str):
    if name == "ref":
        return RefOps()
    if name == "canon":
        return CanonOps()
    raise ValueError(name)
