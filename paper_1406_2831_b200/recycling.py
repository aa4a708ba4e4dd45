"""Recycle spaces on the device (drop-in for krecycle.recycling).

``RecycleSpace`` keeps its six n x k blocks resident in HBM as column-major
tensors (shape (k, n) row-major == n x k column-major, leading dim n); host
numpy views are materialised lazily, only when a caller reads ``.U`` etc.
(a C5 space is 24 GB — it never crosses PCIe on the hot path).

Reference: /root/reference/pkg/src/krecycle/recycling.py (file:line per
function below).
"""

from __future__ import annotations

import warnings
import numpy as np

from . import _lib
from .device import Context, device_matrix, ptr, stream_ptr, to_device, to_host, torch

_BLOCKS = ("U", "Ut", "C", "Ct", "Chat", "Ccheck")


class RecycleSpace:
    """Biorthonormalized recycle space with cached operator images
    (recycling.py:35-77): C = A U, Ct = A^H Ut, Ct^H C = diag(Dc) > 0,
    ||C_j|| = 1, Chat = Ct / Dc, Ccheck = C / Dc."""

    def __init__(self, U=None, Ut=None, C=None, Ct=None, Dc=None, Chat=None,
                 Ccheck=None, *, _dev=None, _n=None):
        if _dev is not None:
            self._dev = _dev
            self._n = int(_n)
        else:
            blocks = dict(U=U, Ut=Ut, C=C, Ct=Ct, Chat=Chat, Ccheck=Ccheck)
            arrs = {k: np.asarray(v) for k, v in blocks.items()}
            for k, a in arrs.items():
                if np.iscomplexobj(a):
                    raise NotImplementedError("complex recycle spaces are out of "
                                              "scope on the device path")
            n, kk = arrs["U"].shape
            self._n = int(n)
            self._dev = {k: (to_device(np.ascontiguousarray(a.T)).reshape(kk, n)
                             if kk else torch().zeros((0, n), dtype=torch().float64,
                                                      device="cuda"))
                         for k, a in arrs.items()}
        self._Dc = None if Dc is None else np.asarray(Dc, dtype=np.float64)
        self._host = {}

    # ---- dataclass-like accessors (lazy D2H) ------------------------------
    def _get(self, name):
        if name not in self._host:
            d = self._dev[name]
            self._host[name] = d.detach().cpu().numpy().T   # n x k (F order)
        return self._host[name]

    U = property(lambda self: self._get("U"))
    Ut = property(lambda self: self._get("Ut"))
    C = property(lambda self: self._get("C"))
    Ct = property(lambda self: self._get("Ct"))
    Chat = property(lambda self: self._get("Chat"))
    Ccheck = property(lambda self: self._get("Ccheck"))

    @property
    def Dc(self):
        return self._Dc if self._Dc is not None else np.zeros(0)

    @property
    def n(self) -> int:
        return self._n

    @property
    def k(self) -> int:
        return int(self._dev["U"].shape[0])

    def device(self, name):
        """(k, n) device tensor of one block."""
        return self._dev[name]

    @classmethod
    def empty(cls, n: int, dtype=np.float64) -> "RecycleSpace":
        t = torch()
        z = {b: t.zeros((0, n), dtype=t.float64, device="cuda") for b in _BLOCKS}
        return cls(_dev=z, _n=n, Dc=np.zeros(0))

    @classmethod
    def of(cls, space) -> "RecycleSpace | None":
        """Adopt a reference RecycleSpace (numpy blocks) or pass ours through."""
        if space is None or isinstance(space, cls):
            return space
        return cls(**{f: getattr(space, f) for f in _BLOCKS + ("Dc",)})

    def view(self) -> _lib.SpaceView:
        v = _lib.SpaceView()
        v.n, v.k, v.ld = self._n, self.k, self._n
        for b in _BLOCKS:
            setattr(v, b, self._dev[b].data_ptr() if self.k else None)
        return v

    def diagnostics(self, A) -> dict:
        """Residuals of the defining identities (recycling.py:61-77), on the
        device."""
        if self.k == 0:
            return {"image": 0.0, "image_dual": 0.0, "diag": 0.0,
                    "colnorm": 0.0, "proj": 0.0}
        t = torch()
        M = device_matrix(A)
        AU = M.spmm(self._dev["U"])
        AhUt = M.spmm(self._dev["Ut"], transpose=True)
        C, Ct, Chat = self._dev["C"], self._dev["Ct"], self._dev["Chat"]
        G = Ct @ C.T
        nrm = lambda x: float(t.linalg.norm(x))
        return {
            "image": nrm(AU - C) / max(nrm(C), 1e-300),
            "image_dual": nrm(AhUt - Ct) / max(nrm(Ct), 1e-300),
            "diag": nrm(G - t.diag(t.as_tensor(self.Dc, device="cuda"))) / nrm(G),
            "colnorm": float(t.max(t.abs(t.linalg.norm(C, dim=1) - 1.0))),
            "proj": nrm(Chat @ C.T - t.eye(self.k, dtype=t.float64, device="cuda")),
        }

    def __repr__(self):
        return f"RecycleSpace(n={self.n}, k={self.k}, device=cuda)"


class CapturedCycle:
    """Lanczos-direction block of one harvest window (recycling.py:80-102),
    constructed with the reference's fields: ``CapturedCycle(V, Vt, tri,
    first_index)``.

    ``V`` / ``Vt`` may be given as the reference gives them -- host numpy
    n x ncols -- or as (ncols, n) CUDA tensors (the column-major device
    layout of this package; what rbicg_solve's harvest produces).  Both
    views exist lazily: ``.V`` / ``.Vt`` are numpy n x ncols (one device->host
    copy on first access), ``.V_dev`` / ``.Vt_dev`` the (ncols, n) device
    blocks (one host->device copy on first access).  ``tri`` holds the
    (sub, diag, super) recurrence coefficients; it may be a zero-argument
    callable, evaluated on first access (the recycle update never reads it,
    so the harvest path does not pay for it)."""

    __slots__ = ("_V", "_Vt", "_V_dev", "_Vt_dev", "_tri", "first_index")

    def __init__(self, V, Vt, tri, first_index):
        self._V = self._V_dev = self._Vt = self._Vt_dev = None
        if _is_cuda(V):
            self._V_dev = V
        else:
            self._V = np.asarray(V)
        if _is_cuda(Vt):
            self._Vt_dev = Vt
        else:
            self._Vt = np.asarray(Vt)
        self._tri = tri
        self.first_index = int(first_index)

    @property
    def V(self):
        if self._V is None:
            self._V = self._V_dev.detach().cpu().numpy().T
        return self._V

    @property
    def Vt(self):
        if self._Vt is None:
            self._Vt = self._Vt_dev.detach().cpu().numpy().T
        return self._Vt

    @property
    def V_dev(self):
        if self._V_dev is None:
            self._V_dev = _host_block(self._V)
        return self._V_dev

    @property
    def Vt_dev(self):
        if self._Vt_dev is None:
            self._Vt_dev = _host_block(self._Vt)
        return self._Vt_dev

    @property
    def tri(self):
        if callable(self._tri):
            self._tri = self._tri()
        return self._tri

    @tri.setter
    def tri(self, value):
        self._tri = value

    @property
    def ncols(self) -> int:
        if self._V_dev is not None:
            return int(self._V_dev.shape[0])
        return int(self._V.shape[1])

    @property
    def last_index(self) -> int:
        return self.first_index + self.ncols - 1

    def __repr__(self):
        return (f"CapturedCycle(ncols={self.ncols}, first_index={self.first_index}, "
                f"device={self._V_dev is not None})")


def _is_cuda(x):
    return hasattr(x, "is_cuda") and x.is_cuda


def _host_block(X):
    """numpy n x c -> (c, n) device block."""
    X = np.atleast_2d(np.asarray(X))
    if np.iscomplexobj(X):
        raise NotImplementedError("complex cycles are out of scope on the device path")
    n, c = X.shape
    if c == 0:
        return torch().zeros((0, n), dtype=torch().float64, device="cuda")
    return to_device(np.ascontiguousarray(X.T, dtype=np.float64)).reshape(c, n)


# ---------------------------------------------------------------------------
# canonical device primitives (thin wrappers; every one is a libkrb kernel)
# ---------------------------------------------------------------------------

def _ctx():
    return Context.get().h


def _ld(X):
    """Leading dimension of a (k, n) block (torch reports stride 1 for a
    size-1 leading dim)."""
    return X.stride(0) if X.shape[0] > 1 else X.shape[1]


def tdot(M_dev, v_dev, out=None):
    """out_j = (M[:, j], v): R.Chat.conj().T @ v (solvers.py:306)."""
    t = torch()
    k, n = M_dev.shape
    if out is None:
        out = t.empty(k, dtype=t.float64, device="cuda")
    if k:
        _lib.call("krb_tdot", _ctx(), n, k, ptr(M_dev), _ld(M_dev),
                  ptr(v_dev), ptr(out), stream_ptr())
    return out


def gemv(M_dev, y_dev, base=None, sign=-1, out=None):
    """base + sign * M y  (R.C @ zeta etc.)."""
    t = torch()
    k, n = M_dev.shape
    if out is None:
        out = t.empty(n, dtype=t.float64, device="cuda")
    _lib.call("krb_gemv", n, k, ptr(M_dev), _ld(M_dev) if k else n,
              ptr(y_dev), ptr(base), int(sign), ptr(out), stream_ptr())
    return out


def gram(X_dev, Y_dev):
    """G = X^T Y (na x nc)  (Wt^H AW, recycling.py:342)."""
    t = torch()
    na, n = X_dev.shape
    nc = Y_dev.shape[0]
    G = t.empty((na, nc), dtype=t.float64, device="cuda")
    if na and nc:
        _lib.call("krb_gram", _ctx(), n, na, nc, ptr(X_dev), _ld(X_dev),
                  ptr(Y_dev), _ld(Y_dev), ptr(G), stream_ptr())
    return G


def gemm(X_dev, Z):
    """X Z for X (m, n) device (column-major n x m), Z host/device m x nc."""
    t = torch()
    m, n = X_dev.shape
    Zd = Z if hasattr(Z, "data_ptr") else to_device(np.ascontiguousarray(Z))
    Zd = Zd.contiguous()
    nc = Zd.shape[1]
    out = t.empty((nc, n), dtype=t.float64, device="cuda")
    if nc and n:
        _lib.call("krb_gemm", n, m, nc, ptr(X_dev), _ld(X_dev), ptr(Zd),
                  ptr(out), _ld(out), stream_ptr())
    return out


def colnorms(X_dev):
    t = torch()
    k, n = X_dev.shape
    out = t.empty(k, dtype=t.float64, device="cuda")
    if k:
        _lib.call("krb_colnorms", _ctx(), n, k, ptr(X_dev), _ld(X_dev),
                  ptr(out), stream_ptr())
    return out


def colscale_div(X_dev, s_dev):
    k, n = X_dev.shape
    if k:
        _lib.call("krb_colscale_div", n, k, ptr(X_dev), _ld(X_dev),
                  ptr(s_dev), stream_ptr())
    return X_dev


def colscale_div_to(X_dev, s_dev, out=None):
    """out[j] = X[j] / s[j] (a new block unless ``out`` is given): the scaled
    copy in one read and one write."""
    t = torch()
    k, n = X_dev.shape
    if out is None:
        out = t.empty((k, n), dtype=t.float64, device="cuda")
    if k:
        _lib.call("krb_colscale_div_to", n, k, ptr(X_dev), _ld(X_dev), ptr(s_dev),
                  ptr(out), _ld(out), stream_ptr())
    return out


def assemble_scaled(parts, scales):
    """[parts...] stacked along the column axis and divided column-wise by
    ``scales`` (the hstack + column scaling of recycling.py:326-340) in one
    pass per part, without materialising the unscaled concatenation."""
    t = torch()
    n = parts[0].shape[1]
    m = sum(p.shape[0] for p in parts)
    out = t.empty((m, n), dtype=t.float64, device="cuda")
    o = 0
    for p in parts:
        kp = p.shape[0]
        if kp:
            colscale_div_to(p, scales[o:o + kp], out[o:o + kp])
        o += kp
    return out


def dot(x_dev, y_dev):
    t = torch()
    out = t.empty(1, dtype=t.float64, device="cuda")
    _lib.call("krb_dot", _ctx(), x_dev.shape[0], ptr(x_dev), ptr(y_dev),
              ptr(out), stream_ptr())
    return out


# ---------------------------------------------------------------------------
# space construction
# ---------------------------------------------------------------------------

def _as_block(X, n):
    """numpy n x k (or (k, n) device tensor) -> (k, n) device tensor."""
    if hasattr(X, "data_ptr"):
        return X.contiguous()
    X = np.atleast_2d(np.asarray(X))
    if np.iscomplexobj(X):
        raise NotImplementedError("complex recycle bases are out of scope")
    if X.shape[0] != n:
        raise ValueError("primary and dual bases must share shape (n, k)")
    return to_device(np.ascontiguousarray(X.T)).reshape(X.shape[1], n)


def _meter(A, nm=0, nr=0):
    if hasattr(A, "n_matvec") and hasattr(A, "n_rmatvec"):
        A.n_matvec += nm
        A.n_rmatvec += nr


def biorthonormalize(U_raw, Ut_raw, A, C_raw=None, Ct_raw=None,
                     rank_tol: float = 1e-12, cond_tol: float = 0.0,
                     amp_tol: float = 1e6) -> RecycleSpace:
    """recycling.py:105-171.  Images by device SpMM (one counted product per
    column, like _apply_columns), k x k Gram on the device, SVD on the host,
    rotations / column scalings / amplification filter on the device."""
    t = torch()
    M = device_matrix(A)
    n = M.n
    U0 = _as_block(U_raw, n)
    Ut0 = _as_block(Ut_raw, n)
    if U0.shape != Ut0.shape:
        raise ValueError("primary and dual bases must share shape (n, k)")
    k = U0.shape[0]
    if k == 0:
        return RecycleSpace.empty(n)
    if C_raw is None:
        C_raw = M.spmm(U0)
        _meter(A, nm=k)
    else:
        C_raw = _as_block(C_raw, n)
    if Ct_raw is None:
        Ct_raw = M.spmm(Ut0, transpose=True)
        _meter(A, nr=k)
    else:
        Ct_raw = _as_block(Ct_raw, n)
    Mk = gram(Ct_raw, C_raw).cpu().numpy()
    import scipy.linalg as la
    X, sig, Yh = la.svd(Mk)
    cut = max(rank_tol, cond_tol) * (sig[0] if sig.size else 0.0)
    r = int(np.sum(sig > cut))
    if r == 0:
        warnings.warn("recycle basis pair is numerically rank deficient; "
                      "returning an empty space", stacklevel=2)
        return RecycleSpace.empty(n)
    Y = to_device(np.ascontiguousarray(Yh.conj().T[:, :r]))   # uploaded once, used twice
    X = to_device(np.ascontiguousarray(X[:, :r]))
    U = gemm(U0, Y)
    C = gemm(C_raw, Y)
    Ut = gemm(Ut0, X)
    Ct = gemm(Ct_raw, X)
    nu = colnorms(C)
    ctn = colnorms(Ct)
    colscale_div(U, nu)
    colscale_div(C, nu)
    nh = t.cat([nu, ctn]).cpu().numpy()    # one read
    nu_h, ctn_h = nh[:r], nh[r:]
    Dc = sig[:r] / nu_h
    amp = ctn_h / Dc
    keep = amp <= amp_tol
    if not np.all(keep):
        if not np.any(keep):
            warnings.warn("all recycle directions are nearly singular under "
                          "the operator; returning an empty space", stacklevel=2)
            return RecycleSpace.empty(n)
        idx = t.as_tensor(np.flatnonzero(keep), device="cuda")
        U, C, Ut, Ct = (B.index_select(0, idx).contiguous() for B in (U, C, Ut, Ct))
        Dc = Dc[keep]
    Dc_d = to_device(Dc)
    Chat = colscale_div_to(Ct, Dc_d)
    Ccheck = colscale_div_to(C, Dc_d)
    return RecycleSpace(_dev=dict(U=U, Ut=Ut, C=C, Ct=Ct, Chat=Chat, Ccheck=Ccheck),
                        _n=n, Dc=Dc)


def refresh_images(space, A, cond_tol: float = 1e-3) -> RecycleSpace:
    """recycling.py:174-186: 2k products on the new operator."""
    space = RecycleSpace.of(space)
    if space.k == 0:
        return space
    return biorthonormalize(space.device("U"), space.device("Ut"), A,
                            cond_tol=cond_tol)


def project_initial(A, b, x_minus1, recycle):
    """recycling.py:189-206 on the device; returns host (x0, r0)."""
    t = torch()
    M = device_matrix(A)
    bd = to_device(np.asarray(b, dtype=np.float64))
    if x_minus1 is None:
        x = t.zeros(M.n, dtype=t.float64, device="cuda")
        r = bd.clone()
    else:
        x = to_device(np.asarray(x_minus1, dtype=np.float64))
        r = bd - M.spmv(x)
        _meter(A, nm=1)
    R = RecycleSpace.of(recycle)
    if R is None or R.k == 0:
        return to_host(x), to_host(r)
    y = tdot(R.device("Chat"), r)
    x0 = gemv(R.device("U"), y, base=x, sign=+1)
    r0 = gemv(R.device("C"), y, base=r, sign=-1)
    return to_host(x0), to_host(r0)


def project_initial_dual(A, b_dual, xt_minus1, recycle):
    """recycling.py:209-222 on the device: the dual analogue of
    project_initial for A^H xt = b_dual (rt = b_dual - A^H xt_minus1,
    y = Ccheck^H rt, xt0 = xt + Ut y, rt0 = rt - Ct y); host (xt0, rt0)."""
    t = torch()
    M = device_matrix(A)
    bd = to_device(np.asarray(b_dual, dtype=np.float64))
    if xt_minus1 is None:
        xt = t.zeros(M.n, dtype=t.float64, device="cuda")
        rt = bd.clone()
    else:
        xt = to_device(np.asarray(xt_minus1, dtype=np.float64))
        rt = bd - M.spmv(xt, transpose=True)
        _meter(A, nr=1)
    R = RecycleSpace.of(recycle)
    if R is None or R.k == 0:
        return to_host(xt), to_host(rt)
    y = tdot(R.device("Ccheck"), rt)
    xt0 = gemv(R.device("Ut"), y, base=xt, sign=+1)
    rt0 = gemv(R.device("Ct"), y, base=rt, sign=-1)
    return to_host(xt0), to_host(rt0)
