"""Device side of the split ILUTP preconditioner (krecycle.ilutp on the B200).

``DeviceFactors`` uploads an IlutpFactors as four level-scheduled triangular
solves (L, L^T, U, U^T: the applications L^{-1}, L^{-H}, U^{-1}, U^{-H} of
ilutp.py:76-97) plus the column permutation (krb_precond_create).
``device_operator`` turns a SplitPreconditionedOperator (ours, or the
reference's object) into a device operator view of its matrix
(krb_operator_create): every solver entry point then runs L^{-1} A P U^{-1}
(and its adjoint for the two-sided RBiCG) as kernel sequences inside the
solve -- no host round trip per product.
"""

from __future__ import annotations

import ctypes
import weakref

import numpy as np

from . import _lib
from .device import (DeviceMatrix, _destroy_matrix, device_matrix, ptr, require_cuda,
                     stream_ptr, to_device, to_host, torch)

TRI_WARPS = 16   # warps of the triangular-solve CTA (csrc/precond.cu kTriWarps)


class TriHost(ctypes.Structure):
    """include/krb.h krb_tri_host"""
    _fields_ = [("n", ctypes.c_int64), ("nnz_off", ctypes.c_int64),
                ("ntasks", ctypes.c_int64), ("nlev", ctypes.c_int32),
                ("rp", ctypes.c_void_p), ("ci", ctypes.c_void_p), ("val", ctypes.c_void_p),
                ("diag", ctypes.c_void_p), ("warp_ptr", ctypes.c_void_p),
                ("t_row", ctypes.c_void_p), ("t_lev", ctypes.c_void_p),
                ("t_len", ctypes.c_void_p), ("t_start", ctypes.c_void_p)]


def tri_schedule(rp, ci, val, lower: bool, unit: bool):
    """Off-diagonal CSR, diagonal and level schedule of a triangular CSR
    (per-warp task lists: row r of a level goes to warp r mod TRI_WARPS).
    Returns (TriHost, arrays kept alive by the caller, number of levels)."""
    rp = np.ascontiguousarray(rp, dtype=np.int64)
    ci = np.ascontiguousarray(ci, dtype=np.int64)
    val = np.ascontiguousarray(val, dtype=np.float64)
    n = len(rp) - 1
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(rp))
    off = ci != rows
    diag = None
    if not unit:
        has = np.zeros(n, dtype=bool)
        has[rows[~off]] = True
        if not np.all(has):
            raise ValueError("triangular factor without a stored diagonal entry")
        diag = np.zeros(n, dtype=np.float64)
        diag[rows[~off]] = val[~off]
    cnt = np.bincount(rows[off], minlength=n)
    rp_off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(cnt, out=rp_off[1:])
    ci_off = np.ascontiguousarray(ci[off], dtype=np.int32)
    val_off = np.ascontiguousarray(val[off])
    lev = np.zeros(n, dtype=np.int32)
    nlev = ctypes.c_int32()
    _lib.call("krb_tri_levels", n, rp_off.ctypes.data, ci_off.ctypes.data, 1 if lower else 0,
              lev.ctypes.data, ctypes.byref(nlev))
    order = np.lexsort((np.arange(n), lev))              # by level, then row
    lev_sorted = lev[order]
    starts = np.searchsorted(lev_sorted, np.arange(nlev.value))
    k = np.arange(n) - starts[lev_sorted]
    warp = k % TRI_WARPS
    o2 = np.lexsort((k, lev_sorted, warp))              # warp, then level, then k
    t_row = np.ascontiguousarray(order[o2], dtype=np.int32)
    t_lev = np.ascontiguousarray(lev_sorted[o2], dtype=np.int32)
    t_start = np.ascontiguousarray(rp_off[t_row], dtype=np.int64)
    t_len = np.ascontiguousarray(rp_off[t_row + 1] - rp_off[t_row], dtype=np.int32)
    warp_ptr = np.zeros(TRI_WARPS + 1, dtype=np.int32)
    np.cumsum(np.bincount(warp, minlength=TRI_WARPS), out=warp_ptr[1:])
    keep = [rp_off, ci_off, val_off, diag, warp_ptr, t_row, t_lev, t_len, t_start]
    h = TriHost(n, len(ci_off), n, nlev.value, rp_off.ctypes.data, ci_off.ctypes.data,
                val_off.ctypes.data, diag.ctypes.data if diag is not None else None,
                warp_ptr.ctypes.data, t_row.ctypes.data, t_lev.ctypes.data,
                t_len.ctypes.data, t_start.ctypes.data)
    return h, keep, nlev.value


_WHICH = {"lower": 0, "lower_h": 1, "upper": 2, "upper_h": 3}


def _destroy_precond(h):
    try:
        _lib.load().krb_precond_destroy(ctypes.c_void_p(h))
    except Exception:
        pass


class DeviceFactors:
    """An IlutpFactors resident on the device (krb_precond)."""

    def __init__(self, F):
        require_cuda()
        import scipy.sparse as sp
        n = F.n
        L = sp.csr_matrix((np.asarray(F.L.values), np.asarray(F.L.col_idx),
                           np.asarray(F.L.row_ptr)), shape=(n, n))
        U = sp.csr_matrix((np.asarray(F.U.values), np.asarray(F.U.col_idx),
                           np.asarray(F.U.row_ptr)), shape=(n, n))
        Lt = L.T.tocsr()
        Lt.sort_indices()
        Ut = U.T.tocsr()
        Ut.sort_indices()
        keep, hs, self.levels = [], [], {}
        for name, M, lower, unit in (("L", L, True, True), ("Lt", Lt, False, True),
                                     ("U", U, False, False), ("Ut", Ut, True, False)):
            h, k, nl = tri_schedule(M.indptr, M.indices, M.data, lower, unit)
            keep.append(k)
            hs.append(h)
            self.levels[name] = nl
        perm = np.ascontiguousarray(F.perm, dtype=np.int64)
        P = ctypes.c_void_p()
        _lib.call("krb_precond_create", *(ctypes.byref(h) for h in hs), perm.ctypes.data,
                  ctypes.byref(P), stream_ptr())
        self.h = P
        self.n = n
        self.perm = perm
        self._finalizer = weakref.finalize(self, _destroy_precond, P.value)

    def apply(self, which, d_in, d_out=None):
        """Device L^{-1} / L^{-H} / U^{-1} / U^{-H} of a device vector."""
        t = torch()
        if d_out is None:
            d_out = t.empty(self.n, dtype=t.float64, device="cuda")
        _lib.call("krb_precond_apply", self.h, _WHICH[which], ptr(d_in), ptr(d_out),
                  stream_ptr())
        return d_out

    def host_apply(self, which, b):
        b = np.asarray(b)
        if np.iscomplexobj(b):
            raise NotImplementedError("complex vectors are out of scope on the B200 path")
        return to_host(self.apply(which, to_device(np.asarray(b, dtype=np.float64))))


class DeviceOperator(DeviceMatrix):
    """Device view of a SplitPreconditionedOperator: L^{-1} A P U^{-1}
    (krb_operator_create).  Same methods as DeviceMatrix (spmv / spmm, the
    transpose = the adjoint composite); keeps A and the factors alive."""

    def __init__(self, base: DeviceMatrix, factors: DeviceFactors):
        self.base, self.factors = base, factors
        self.n, self.nnz = base.n, base.nnz
        self.format = base.format + "+ilutp"
        h = ctypes.c_void_p()
        _lib.call("krb_operator_create", base.h, factors.h, ctypes.byref(h))
        self.h = h
        self.device_bytes = base.device_bytes
        self._finalizer = weakref.finalize(self, _destroy_matrix, h.value)

    def host_matvec(self, x, adjoint=False):
        x = np.asarray(x, dtype=np.float64)
        if x.shape != (self.n,):
            raise ValueError(f"expected a vector of length {self.n}, got {x.shape}")
        return to_host(self.spmv(to_device(x), transpose=adjoint))


_OPS = {}


def is_split_operator(A) -> bool:
    return hasattr(A, "factors") and hasattr(A, "_A") and hasattr(A, "matvec")


def device_operator(op) -> DeviceOperator:
    """The device view of a SplitPreconditionedOperator (this package's or
    the reference's): cached on the operator object."""
    hit = _OPS.get(id(op))
    if hit is not None and hit[0] is op:
        return hit[1]
    from .ilutp import _factors
    F = _factors(op.factors)
    dev = DeviceOperator(device_matrix(op._A), F.device())
    _OPS[id(op)] = (op, dev)
    while len(_OPS) > 4:
        _OPS.pop(next(iter(_OPS)))
    return dev
