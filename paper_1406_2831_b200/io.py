"""Run-report CSV and recycle-space snapshots,
file-compatible with the reference's krecycle.io:

* ``history_write(path, report)``  -- io.py:192-211: one row per recorded
  iteration (system_index 1-based, solver, iteration, resid %.17g,
  matvecs_cum, seconds_cum %.6f), then a per-system summary row with
  iteration = -1 carrying the totals.  Accepts a RunReport or a list of
  ConvergenceHistory.
* ``recycle_save(path, space)`` / ``recycle_load(path, A)`` -- io.py:139-189:
  "KRSP" magic, little-endian header <IQQB (version 1, n, k, complex flag),
  then U and Ut in Fortran order.  Only the bases are stored; loading
  rebuilds the images under ``A`` with the device ``biorthonormalize`` (the
  bases are uploaded once and the space stays device-resident).

Host-side file formats only: the numbers are whatever the solvers produced.
"""

from __future__ import annotations

import csv
import struct

import numpy as np

from .recycling import RecycleSpace, biorthonormalize

_MAGIC = b"KRSP"
_VERSION = 1
_HEADER = "<IQQB"


def history_write(path, report):
    """io.py:192-211."""
    with open(path, "w", encoding="ascii", newline="") as fh:
        writer = csv.writer(fh)
        writer.writerow(["system_index", "solver", "iteration", "resid",
                         "matvecs_cum", "seconds_cum"])
        for sys_idx, hist in enumerate(getattr(report, "histories", report), start=1):
            for it, (rn, mv, sec) in enumerate(zip(hist.resid, hist.matvecs, hist.seconds)):
                writer.writerow([sys_idx, hist.solver, it, f"{rn:.17g}", mv, f"{sec:.6f}"])
            last = hist.resid[-1] if hist.resid else float("nan")
            writer.writerow([sys_idx, hist.solver, -1, f"{last:.17g}",
                             hist.total_matvecs, f"{hist.total_seconds:.6f}"])


def recycle_save(path, space: RecycleSpace):
    """io.py:139-155: persist the basis pair (U, Ut)."""
    if space is None or space.k == 0:
        raise ValueError("refusing to save an empty recycle space")
    U = np.asarray(space.U)
    Ut = np.asarray(space.Ut)
    cplx = np.iscomplexobj(U) or np.iscomplexobj(Ut)
    dt = np.complex128 if cplx else np.float64
    with open(path, "wb") as fh:
        fh.write(_MAGIC)
        fh.write(struct.pack(_HEADER, _VERSION, space.n, space.k, 1 if cplx else 0))
        fh.write(np.asfortranarray(U.astype(dt)).tobytes(order="F"))
        fh.write(np.asfortranarray(Ut.astype(dt)).tobytes(order="F"))


def _read(path):
    with open(path, "rb") as fh:
        magic = fh.read(4)
        if magic != _MAGIC:
            raise ValueError(f"not a recycle-space file (bad magic {magic!r})")
        hsize = struct.calcsize(_HEADER)
        header = fh.read(hsize)
        if len(header) != hsize:
            raise ValueError("truncated recycle-space header")
        version, n, k, cflag = struct.unpack(_HEADER, header)
        if version != _VERSION:
            raise ValueError(f"unsupported recycle-space file version {version}")
        dt = np.dtype(np.complex128 if cflag else np.float64)
        count = n * k
        expect = 2 * count * dt.itemsize
        payload = fh.read(expect)
        if len(payload) != expect:
            raise ValueError("truncated recycle-space payload")
    flat = np.frombuffer(payload, dtype=dt)
    U = flat[:count].reshape((n, k), order="F").copy()
    Ut = flat[count:].reshape((n, k), order="F").copy()
    return n, U, Ut


def recycle_load(path, A) -> RecycleSpace:
    """io.py:158-189: load a basis pair and rebuild its images under A."""
    n, U, Ut = _read(path)
    if n != A.shape[0]:
        raise ValueError(f"recycle space dimension {n} does not match operator "
                         f"dimension {A.shape[0]}")
    if np.iscomplexobj(U) or np.iscomplexobj(Ut):
        raise NotImplementedError("complex recycle spaces are out of scope on the "
                                  "device path (fp64 real only)")
    return biorthonormalize(U, Ut, A)
