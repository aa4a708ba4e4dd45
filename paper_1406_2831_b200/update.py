"""Recycle-space update from harvested cycles on the device
(krecycle.recycling.update_recycle_space, reference recycling.py:225-370).

The n x m work — images of the new cycle columns (SpMM with A and A^T), column
norms and scalings, the two m x m Gram matrices, the Ritz-vector basis
combinations and the near-null eigen-residual norms — runs in libkrb kernels
in the canonical order; only the m x m generalized eigenproblem
(scipy.linalg.eig, LAPACK ggev) and the smallest-|theta| selection run on the
host, as the north star prescribes.
"""

from __future__ import annotations

import warnings

import numpy as np

from . import _lib
from .device import device_matrix, flush_pending, ptr, stream_ptr, to_device, torch
from .recycling import (RecycleSpace, _as_block, _ctx, _ld, _meter, assemble_scaled,
                        biorthonormalize, colnorms, gemm, gram)

NEAR_NULL_FRAC = 1e-3   # recycling.py:228


def colsq(X_dev):
    """(X[:,j], X[:,j]) per column (canonical dot, no square root)."""
    t = torch()
    k, n = X_dev.shape
    out = t.empty(k, dtype=t.float64, device="cuda")
    if k:
        _lib.call("krb_colsq", _ctx(), n, k, ptr(X_dev), _ld(X_dev), ptr(out),
                  stream_ptr())
    return out


def select_pencil_columns(theta, VR, VL, k, real_pencil, eligible=None):
    """k smallest-|theta| eigenvectors with conjugate pairs split into real
    and imaginary parts (recycling.py:231-273); host-side on m x m data.
    Same selection as the reference's loop (oracle/krylov.py restates it
    verbatim): the conjugate mate is the first available eigenvalue, in
    ranked order, at the smallest |theta_j - conj(theta)| -- found here with
    one vectorised pass, then re-decided exactly (Python abs, strict <, in
    ranked order) among the candidates within 1e-9 of that minimum."""
    ok = np.isfinite(theta)
    if eligible is not None:
        ok = ok & eligible
    ranked = np.array([i for i in np.argsort(np.abs(np.where(ok, theta, np.inf))) if ok[i]],
                      dtype=np.int64)
    avail = np.ones(ranked.size, dtype=bool)
    right, left = [], []
    for p in range(ranked.size):
        if not avail[p]:
            continue
        avail[p] = False
        idx = ranked[p]
        th = theta[idx]
        zr, zl = VR[:, idx], VL[:, idx]
        if real_pencil and abs(th.imag) > 1e-12 * (1.0 + abs(th)):
            cand = np.nonzero(avail)[0]
            if cand.size:
                ct = np.conj(th)
                dn = np.abs(theta[ranked[cand]] - ct)
                close = cand[dn <= dn.min() * (1.0 + 1e-9)]
                mate, gap = None, np.inf
                for q in close:
                    d = abs(theta[ranked[q]] - ct)
                    if d < gap:
                        mate, gap = q, d
                if mate is not None:
                    avail[mate] = False
            right += [zr.real, zr.imag]
            left += [zl.real, zl.imag]
        else:
            right.append(zr.real if real_pencil else zr)
            left.append(zl.real if real_pencil else zl)
        if len(right) >= k:
            break
    if not right:
        return None, None
    return np.column_stack(right[:k]), np.column_stack(left[:k])


def near_null_eligibility(theta, VR, W, AW, res_tol):
    """recycling.py:348-358 with the complex products as real ones:
    Y = W VR, R = AW VR - Y theta, res = ||R_c|| / max(||Y_c||, 1e-300).
    Only the near-null columns (|theta| < NEAR_NULL_FRAC max|theta|, finite)
    read their residual, so only those columns are computed: every column of
    the products, the Ritz combination and the column norms is independent
    of the others, so the subset gives the same bits per column."""
    finite = np.isfinite(theta)
    th = np.where(finite, theta, 0.0)
    ab = np.abs(th)
    top = ab.max() if ab.size else 0.0
    near = ab < NEAR_NULL_FRAC * top
    sel = np.flatnonzero(finite & near)
    eligible = finite & ~near
    if sel.size == 0:
        return eligible
    VRs = VR[:, sel]
    ths = th[sel]
    VRr = to_device(np.ascontiguousarray(VRs.real))   # uploaded once, used twice
    VRi = to_device(np.ascontiguousarray(VRs.imag))
    m, n = W.shape
    Yre, Yim = gemm(W, VRr), gemm(W, VRi)
    Are, Aim = gemm(AW, VRr), gemm(AW, VRi)
    thr = to_device(np.ascontiguousarray(ths.real))
    thi = to_device(np.ascontiguousarray(ths.imag))
    c = sel.size
    _lib.call("krb_ritz_combine", n, c, ptr(Yre), ptr(Yim), ptr(Are),
              ptr(Aim), n, ptr(thr), ptr(thi), stream_ptr())
    t = torch()
    sq = t.cat([colsq(Are), colsq(Aim), colsq(Yre), colsq(Yim)]).cpu().numpy()  # one read
    rn = np.sqrt(sq[:c] + sq[c:2 * c])
    yn = np.sqrt(sq[2 * c:3 * c] + sq[3 * c:])
    res = rn / np.maximum(yn, 1e-300)
    eligible[sel] = res <= res_tol * ab[sel]
    return eligible


def _cycle_blocks(cyc, n):
    V = getattr(cyc, "V_dev", None)
    Vt = getattr(cyc, "Vt_dev", None)
    if V is None:   # a reference CapturedCycle (numpy n x ncols)
        V = _as_block(cyc.V, n)
        Vt = _as_block(cyc.Vt, n)
    return V, Vt


def update_recycle_space(A, cycles, previous, k: int, rank_tol: float = 1e-12,
                         res_tol: float = 0.0) -> RecycleSpace:
    """Next recycle space from harvested cycles and the prior space
    (recycling.py:276-370): W = [U_prev, V], Wt = [Ut_prev, Vt], images reused
    from the prior space and computed for the new columns (2 products per new
    column, counted), pencil (Wt^H AW, Wt^H W) eigenvectors of the k smallest
    |theta|, then biorthonormalize."""
    t = torch()
    M = device_matrix(A)
    n = M.n
    prev = RecycleSpace.of(previous)
    bu, but, bc, bct = [], [], [], []
    if prev is not None and prev.k > 0:
        bu.append(prev.device("U"))
        but.append(prev.device("Ut"))
        bc.append(prev.device("C"))
        bct.append(prev.device("Ct"))
    seen = 0
    for cyc in cycles:
        first = max(0, seen - cyc.first_index + 1)
        if first >= cyc.ncols:
            continue
        V, Vt = _cycle_blocks(cyc, n)
        V, Vt = V[first:], Vt[first:]
        seen = cyc.last_index
        bu.append(V)
        but.append(Vt)
        bc.append(M.spmm(V.contiguous()))
        bct.append(M.spmm(Vt.contiguous(), transpose=True))
        _meter(A, nm=V.shape[0], nr=Vt.shape[0])
    if not bu:
        return prev if prev is not None else RecycleSpace.empty(n)
    # hstack + column scaling (recycling.py:326-340): norms per part (each
    # column's canonical dot is independent of its neighbours), then one
    # scaled copy per part into the assembled block; the scales stay on the
    # device (a zero norm divides by 1, as the reference)
    swd = t.cat([colnorms(B.contiguous() if B.stride(-1) != 1 else B) for B in bu])
    std_ = t.cat([colnorms(B.contiguous() if B.stride(-1) != 1 else B) for B in but])
    swd.masked_fill_(swd == 0, 1.0)
    std_.masked_fill_(std_ == 0, 1.0)
    W, AW = assemble_scaled(bu, swd), assemble_scaled(bc, swd)
    Wt, AhWt = assemble_scaled(but, std_), assemble_scaled(bct, std_)
    G2 = t.stack([gram(Wt, AW), gram(Wt, W)]).cpu().numpy()   # one read
    GA, GI = G2[0].copy(), G2[1].copy()
    import scipy.linalg as la
    flush_pending()   # a deferred generation cycle runs on the device meanwhile
    theta, VL, VR = la.eig(GA, GI, left=True, right=True)
    eligible = None
    if res_tol > 0.0:
        eligible = near_null_eligibility(theta, VR, W, AW, res_tol)
    Zr, Zl = select_pencil_columns(theta, VR, VL, k, True, eligible)
    if Zr is None:
        warnings.warn("recycle-space pencil produced no finite eigenvalues; "
                      "keeping previous space", stacklevel=2)
        return prev if prev is not None else RecycleSpace.empty(n)
    Zr = to_device(np.ascontiguousarray(Zr))   # uploaded once, used twice
    Zl = to_device(np.ascontiguousarray(Zl))
    return biorthonormalize(gemm(W, Zr), gemm(Wt, Zl), M,
                            C_raw=gemm(AW, Zr), Ct_raw=gemm(AhWt, Zl),
                            rank_tol=rank_tol)
