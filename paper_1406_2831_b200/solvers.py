"""Drop-in solver entry points on the B200 (krecycle.solvers API).

Same names, signatures, return values and error behaviour as
/root/reference/pkg/src/krecycle/solvers.py; the arithmetic runs in libkrb.so
(one CUDA-graph launch per solve, device-resident scalars and history).

Out of scope on the device path (raise NotImplementedError, never a CPU
fallback): split preconditioning (``precond``), complex data, and
``record_iterates`` (a per-iteration host copy of every vector).
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .device import Context, device_matrix, ptr, stream_ptr, to_device, torch
from .recycling import RecycleSpace

CONVERGED = "converged"
MAX_ITN = "max_itn"
BREAKDOWN_SERIOUS = "breakdown:serious"
BREAKDOWN_SECOND_KIND = "breakdown:second_kind"
BREAKDOWN_OMEGA = "breakdown:omega"


@dataclass(frozen=True)
class SolverConfig:
    """solvers.py:40-56 (same fields and defaults)."""

    tol: float = 1e-8
    max_itn: int = 1000
    k: int = 0
    s: int = 25
    seed: int = 0
    breakdown_tol: float = 1e-14
    record_iterates: bool = False


@dataclass
class ConvergenceHistory:
    """solvers.py:59-104 (same fields).  ``seconds`` are wall-clock seconds
    since the call started, with per-iteration points taken from the device
    %globaltimer stamped by the kernel that recorded each residual."""

    solver: str
    rhs_norm: float = 1.0
    rhs_norm_dual: float = 0.0
    resid: list = field(default_factory=list)
    resid_dual: list = field(default_factory=list)
    matvecs: list = field(default_factory=list)
    seconds: list = field(default_factory=list)
    status: str = ""
    final_true_resid: float = float("nan")
    iterates: list | None = None
    residual_vectors: list | None = None
    residual_vectors_dual: list | None = None
    omega_steps: list | None = None

    @property
    def iterations(self) -> int:
        return max(len(self.resid) - 1, 0)

    @property
    def total_matvecs(self) -> int:
        return self.matvecs[-1] if self.matvecs else 0

    @property
    def total_seconds(self) -> float:
        return self.seconds[-1] if self.seconds else 0.0

    def _record(self, rnorm, mv, t, rtnorm=None):
        self.resid.append(float(rnorm))
        self.matvecs.append(int(mv))
        self.seconds.append(float(t))
        if rtnorm is not None:
            self.resid_dual.append(float(rtnorm))


def pcg64_words(seed: int):
    """128-bit PCG64 (state, inc) numpy's default_rng(seed) starts from; the
    device draw continues that exact stream (solvers.py:111-113)."""
    st = np.random.default_rng(seed).bit_generator.state["state"]
    s, inc = int(st["state"]), int(st["inc"])
    m = (1 << 64) - 1
    return (s >> 64) & m, s & m, (inc >> 64) & m, inc & m


def _check_common(A, b, precond, cfg):
    if precond is not None:
        raise NotImplementedError("split preconditioning is out of scope on the "
                                  "B200 path (SURVEY.md §2.1 row 7)")
    if cfg.record_iterates:
        raise NotImplementedError("record_iterates is not supported on the "
                                  "device path")
    M = device_matrix(A)
    b = np.asarray(b)
    if np.iscomplexobj(b):
        raise NotImplementedError("complex right-hand sides are out of scope")
    if b.shape != (M.n,):
        raise ValueError("right-hand side length does not match the operator")
    return M, b


def _count(A, nm=0, nr=0):
    """Mirror the reference's double metering: products made through an
    outer CountingOperator increment it as well (operators.py:82-88)."""
    if hasattr(A, "n_matvec") and hasattr(A, "n_rmatvec"):
        A.n_matvec += nm
        A.n_rmatvec += nr


_STATUS = {1: CONVERGED, 2: MAX_ITN, 3: BREAKDOWN_SERIOUS, 4: BREAKDOWN_OMEGA,
           5: BREAKDOWN_SECOND_KIND}


LAST_SOLVE = {}   # launch accounting of the most recent solve (bench / tests)


def _device_solve(A, b, x_init, recycle, cfg, label, t0, use_graph=None):
    M, b = _check_common(A, b, None, cfg)
    bd = to_device(b.astype(np.float64, copy=False))
    xd = None
    if x_init is not None:
        xd = to_device(np.asarray(x_init, dtype=np.float64))
    xo, hist = solve_device(M, bd, xd, recycle, cfg, label, t0, use_graph)
    _count(A, nm=LAST_SOLVE["matvecs"])
    return xo.cpu().numpy(), hist


def _graph_mode():
    """KRB_GRAPH_MODE=1 (default): one CUDA graph with a device-driven WHILE
    node per solve; 0: host-launched iterations with a status poll every 8
    (identical kernels and results; used for per-kernel ncu profiling, which
    cannot see inside conditional graph nodes)."""
    import os
    return int(os.environ.get("KRB_GRAPH_MODE", "1"))


def solve_device(M, bd, xd, recycle, cfg, label="rbicgstab", t0=None,
                 use_graph=None):
    """Device-resident entry: M a DeviceMatrix, bd / xd device tensors.
    Returns (x device tensor, ConvergenceHistory)."""
    t = torch()
    if t0 is None:
        t0 = time.perf_counter()
    if use_graph is None:
        use_graph = _graph_mode()
    ctx = Context.get()
    R = None
    if recycle is not None and recycle.k > 0:
        R = RecycleSpace.of(recycle)
        if R.n != M.n:
            raise ValueError("recycle space dimension does not match the operator")
    xo = t.empty(M.n, dtype=t.float64, device="cuda")
    hr, hm, ht = ctx.history_buffers(cfg.max_itn)
    c = _lib.SolveConfig()
    c.tol = float(cfg.tol)
    c.breakdown_tol = float(cfg.breakdown_tol)
    c.max_itn = int(cfg.max_itn)
    c.d_shadow = None
    c.pcg_state_hi, c.pcg_state_lo, c.pcg_inc_hi, c.pcg_inc_lo = pcg64_words(cfg.seed)
    c.use_graph = int(use_graph)
    res = _lib.SolveResult()
    view = R.view() if R is not None else None
    t_launch = time.perf_counter()
    _lib.call("krb_rbicgstab", ctx.h, M.h, ptr(bd), ptr(xd),
              ctypes.byref(view) if view is not None else None,
              ctypes.byref(c), ptr(xo), ptr(hr), ptr(hm), ptr(ht),
              ctypes.byref(res), stream_ptr())
    L = int(res.hist_len)
    resid = hr[:L].cpu().numpy()
    mvs = hm[:L].cpu().numpy()
    stamps = ht[:L].cpu().numpy().astype(np.int64)
    hist = ConvergenceHistory(solver=label, rhs_norm=float(res.rhs_norm))
    base = (t_launch - t0)
    st0 = int(res.t_start_ns)
    hist.resid = [float(v) for v in resid]
    hist.matvecs = [int(v) for v in mvs]
    hist.seconds = [base + (int(s) - st0) * 1e-9 for s in stamps]
    hist.status = _STATUS.get(int(res.status), f"unknown:{res.status}")
    hist.final_true_resid = float(res.final_true_resid)
    LAST_SOLVE.clear()
    LAST_SOLVE.update(matvecs=int(res.matvecs), bodies=int(res.iterations_run),
                      kernel_launches=int(res.kernel_launches))
    return xo, hist


def bicgstab_solve(A, b, x_init=None, precond=None, config=None):
    """solvers.py:156-242 — stabilized BiCG, shadow residual from the seeded
    uniform(-1, 1) stream (drawn on the device, bit-identical to numpy)."""
    cfg = config or SolverConfig()
    t0 = time.perf_counter()
    if precond is not None:
        _check_common(A, b, precond, cfg)
    return _device_solve(A, b, x_init, None, cfg, "bicgstab", t0)


def rbicgstab_solve(A, b, x_init=None, recycle=None, precond=None,
                    config=None):
    """solvers.py:245-361 — BiCGSTAB deflated by a recycle space (Algorithm 2):
    projected start, (I - C Chat^H) after every product, x = x - U xc at the
    end.  With an empty space the arithmetic is that of bicgstab_solve."""
    cfg = config or SolverConfig()
    t0 = time.perf_counter()
    if precond is not None:
        _check_common(A, b, precond, cfg)
    return _device_solve(A, b, x_init, recycle, cfg, "rbicgstab", t0)
