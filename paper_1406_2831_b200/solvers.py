"""Drop-in solver entry points on the B200 (krecycle.solvers API).

Same names, signatures, return values and error behaviour as
/root/reference/pkg/src/krecycle/solvers.py; the arithmetic runs in libkrb.so
(one CUDA-graph launch per solve, device-resident scalars and history).

Split ILUTP preconditioning (``precond`` = IlutpFactors) runs on the device
(ilutp.py / precond.py).  Out of scope on the device path (raise
NotImplementedError, never a CPU fallback): complex data, record_iterates in
rbicg_solve, and the multi-rhs batch path with a preconditioner.
"""

from __future__ import annotations

import ctypes
import functools
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .device import (Context, call_retry_oom, defer_launch, device_matrix, drop_pending,
                     flush_pending, ptr, stream_ptr, to_device, to_host, torch)
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


_PCG_MULT = 0x2360ED051FC65DA44385DF649FCCF645
_M128 = (1 << 128) - 1


def _pcg_advance(state: int, inc: int, steps: int) -> int:
    """LCG^steps(state) for PCG64's 128-bit LCG (jump-ahead)."""
    am, ap, cm, cp = 1, 0, _PCG_MULT, inc
    while steps:
        if steps & 1:
            am = (am * cm) & _M128
            ap = (ap * cm + cp) & _M128
        cp = ((cm + 1) * cp) & _M128
        cm = (cm * cm) & _M128
        steps >>= 1
    return (am * state + ap) & _M128


@functools.lru_cache(maxsize=256)
def pcg64_words(seed: int, skip: int = 0):
    """128-bit PCG64 (state, inc) numpy's default_rng(seed) is at after `skip`
    doubles were drawn; the device draw continues that exact stream
    (solvers.py:111-113)."""
    st = np.random.default_rng(seed).bit_generator.state["state"]
    s, inc = int(st["state"]), int(st["inc"])
    if skip:
        s = _pcg_advance(s, inc, skip)
    m = (1 << 64) - 1
    return (s >> 64) & m, s & m, (inc >> 64) & m, inc & m


def device_uniform(seed: int, n: int, skip: int = 0):
    """numpy default_rng(seed).uniform(-1, 1, n) (after `skip` draws), drawn on
    the device bit for bit."""
    t = torch()
    out = t.empty(n, dtype=t.float64, device="cuda")
    _lib.call("krb_uniform_pcg64", n, *pcg64_words(seed, skip), -1.0, 1.0,
              ptr(out), stream_ptr())
    return out


def _check_common(A, b, precond, cfg):
    M = device_matrix(A)
    if _is_device(b):
        if tuple(b.shape) != (M.n,):
            raise ValueError("right-hand side length does not match the operator")
        return M, b
    b = np.asarray(b)
    if np.iscomplexobj(b):
        raise NotImplementedError("complex right-hand sides are out of scope")
    if b.shape != (M.n,):
        raise ValueError("right-hand side length does not match the operator")
    return M, b


def _is_device(v):
    """Device-resident inputs (torch CUDA tensors) stay on the device: the
    solvers then return device tensors instead of numpy arrays."""
    return hasattr(v, "is_cuda") and v.is_cuda


def _dev_vec(v):
    if v is None:
        return None
    if _is_device(v):
        return v.to(dtype=torch().float64).contiguous()
    return to_device(np.asarray(v, dtype=np.float64))


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
    bd = _dev_vec(b)
    xd = _dev_vec(x_init)
    xo, hist = solve_device(M, bd, xd, recycle, cfg, label, t0, use_graph)
    _count(A, nm=LAST_SOLVE["matvecs"])
    return (xo if _is_device(b) else to_host(xo)), hist


def _graph_mode():
    """Iteration driver override (_lib.tuning(graph_mode=...); None =
    automatic; bit-identical results in every mode): 2 = one persistent
    cooperative kernel per solve (n <= PERSISTENT_MAX_N); 1 = one CUDA graph
    per solve with a device-driven WHILE node (the RBiCG generation solve at
    large n uses this, pausing at every harvest cycle); 0 = host-launched
    iterations with a status poll every 8 (per-kernel ncu profiling: ncu
    cannot see inside conditional graph nodes)."""
    return _lib.PY_TUNING["graph_mode"]


# Below this size one persistent cooperative kernel beats per-phase kernels
# (launch / tail latency dominates); above it the per-phase kernels run at
# higher occupancy (measured on B200: C1/C2 persistent -10..15 %, C3-C5
# graph -10..20 %).
PERSISTENT_MAX_N = 600_000


def _auto_mode(n):
    m = _graph_mode()
    if m is not None:
        return m
    return 2 if n <= PERSISTENT_MAX_N else 1


def solve_device(M, bd, xd, recycle, cfg, label="rbicgstab", t0=None,
                 use_graph=None):
    """Device-resident entry: M a DeviceMatrix, bd / xd device tensors.
    Returns (x device tensor, ConvergenceHistory)."""
    t = torch()
    if t0 is None:
        t0 = time.perf_counter()
    if use_graph is None:
        use_graph = _auto_mode(M.n)
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
    rec = None
    if cfg.record_iterates:
        # per-iteration snapshots on the device (host-loop driver: the graph
        # and persistent drivers do not carry the snapshot pointers)
        use_graph = 0
        L = int(cfg.max_itn) + 2
        kk = R.k if R is not None else 0
        rec = {nm: t.empty((L, M.n), dtype=t.float64, device="cuda")
               for nm in ("x", "r", "s", "t")}
        rec["xc"] = t.empty((L, max(kk, 1)), dtype=t.float64, device="cuda")
        rec["omega"] = t.empty(L, dtype=t.float64, device="cuda")
        for nm in ("x", "r", "xc", "s", "t", "omega"):
            setattr(c, "d_rec_" + nm, rec[nm].data_ptr())
    c.use_graph = int(use_graph)
    kt = _lib.PY_TUNING["kernel_times"]
    c.d_kernel_times = kt.data_ptr() if kt is not None else None
    prof = None
    if _lib.PY_TUNING["phase_prof"] and use_graph == 2:
        prof = t.zeros((cfg.max_itn + 1) * 16, dtype=t.int64, device="cuda")
        c.d_phase_stamps = prof.data_ptr()
        c.phase_stamps_cap = cfg.max_itn + 1
    res = _lib.SolveResult()
    view = R.view() if R is not None else None
    t_launch = time.perf_counter()
    _lib.call("krb_rbicgstab", ctx.h, M.h, ptr(bd), ptr(xd),
              ctypes.byref(view) if view is not None else None,
              ctypes.byref(c), ptr(xo), ptr(hr), ptr(hm), ptr(ht),
              ctypes.byref(res), stream_ptr())
    L = int(res.hist_len)
    # one device->host read for the three history arrays (bit views)
    t3 = torch().stack([hr[:L].view(torch().int64), hm[:L], ht[:L]]).cpu().numpy()
    resid = t3[0].view(np.float64)
    mvs = t3[1]
    stamps = t3[2]
    hist = ConvergenceHistory(solver=label, rhs_norm=float(res.rhs_norm))
    base = (t_launch - t0)
    st0 = int(res.t_start_ns)
    hist.resid = [float(v) for v in resid]
    hist.matvecs = [int(v) for v in mvs]
    hist.seconds = [base + (int(s) - st0) * 1e-9 for s in stamps]
    hist.status = _STATUS.get(int(res.status), f"unknown:{res.status}")
    hist.final_true_resid = float(res.final_true_resid)
    if rec is not None:
        _attach_iterates(hist, rec, R, L)
    LAST_SOLVE.clear()
    LAST_SOLVE.update(matvecs=int(res.matvecs), bodies=int(res.iterations_run),
                      kernel_launches=int(res.kernel_launches),
                      driver=_lib.DRIVERS.get(int(res.driver), str(res.driver)))
    if prof is not None:
        LAST_SOLVE["phase_stamps"] = prof.view(-1, 16)[:hist.iterations].cpu().numpy()
    return xo, hist


def _attach_iterates(hist, rec, R, L):
    """record_iterates (solvers.py:284-286, 321-323, 344-347): iterates
    x_j - U xc_j (one device GEMM over all entries, the same per-row fma
    order as the solve's final x - U xc), residual vectors, and per full
    iteration (s, t, omega); host numpy like the reference."""
    t = torch()
    from .recycling import gemm
    X = rec["x"][:L]
    if R is not None and R.k:
        UX = gemm(R.device("U"), rec["xc"][:L, :R.k].t().contiguous())   # (L, n)
        X = X - UX
    nfull = L - 1 - (1 if hist.status == CONVERGED and len(hist.resid) >= 2 and
                     _half_step(hist) else 0)
    Xh, Rh = X.cpu().numpy(), rec["r"][:L].cpu().numpy()
    Sh, Th = rec["s"][:nfull].cpu().numpy(), rec["t"][:nfull].cpu().numpy()
    om = rec["omega"][:nfull].cpu().numpy()
    hist.iterates = [Xh[j].copy() for j in range(L)]
    hist.residual_vectors = [Rh[j].copy() for j in range(L)]
    hist.omega_steps = [(Sh[i].copy(), Th[i].copy(), complex(om[i])) for i in range(nfull)]


def _half_step(hist):
    """Whether the last record is a half-step exit (1 product after the
    previous record instead of 2)."""
    return len(hist.matvecs) >= 2 and hist.matvecs[-1] - hist.matvecs[-2] == 1


BATCH_MAX = 4   # right-hand sides per batched launch (batch.cu kMaxB)


def solve_device_batch(M, bds, xds, recycle, cfgs, label="rbicgstab", t0=None,
                       use_graph=None):
    """Device-resident multi-right-hand-side entry: up to BATCH_MAX solves
    with the same DeviceMatrix and recycle space advanced in lockstep
    (krb_rbicgstab_batch, batch.cu).  Returns [(x device tensor, history)]."""
    t = torch()
    if t0 is None:
        t0 = time.perf_counter()
    nr = len(bds)
    if not 1 <= nr <= BATCH_MAX:
        raise ValueError(f"1 <= number of right-hand sides <= {BATCH_MAX}")
    if use_graph is None:
        use_graph = 0 if _graph_mode() == 0 else 1
    ctx = Context.get()
    R = None
    if recycle is not None and recycle.k > 0:
        R = RecycleSpace.of(recycle)
        if R.n != M.n:
            raise ValueError("recycle space dimension does not match the operator")
    xos, hrs, hms, hts = [], [], [], []
    cs = (_lib.SolveConfig * nr)()
    for j, cfg in enumerate(cfgs):
        L = int(cfg.max_itn) + 2
        xos.append(t.empty(M.n, dtype=t.float64, device="cuda"))
        hrs.append(t.empty(L, dtype=t.float64, device="cuda"))
        hms.append(t.empty(L, dtype=t.int64, device="cuda"))
        hts.append(t.empty(L, dtype=t.int64, device="cuda"))
        c = cs[j]
        c.tol = float(cfg.tol)
        c.breakdown_tol = float(cfg.breakdown_tol)
        c.max_itn = int(cfg.max_itn)
        c.d_shadow = None
        c.pcg_state_hi, c.pcg_state_lo, c.pcg_inc_hi, c.pcg_inc_lo = pcg64_words(cfg.seed)
        c.use_graph = int(use_graph)

    def parr(ts):
        return (ctypes.c_void_p * nr)(*[x.data_ptr() if x is not None else None for x in ts])

    res = (_lib.SolveResult * nr)()
    view = R.view() if R is not None else None
    t_launch = time.perf_counter()
    _lib.call("krb_rbicgstab_batch", ctx.h, M.h, nr, parr(bds),
              parr(xds) if xds is not None and any(x is not None for x in xds) else None,
              ctypes.byref(view) if view is not None else None, cs, parr(xos), parr(hrs),
              parr(hms), parr(hts), res, stream_ptr())
    out = []
    total_mv = 0
    for j in range(nr):
        L = int(res[j].hist_len)
        stamps = hts[j][:L].cpu().numpy().astype(np.int64)
        hist = ConvergenceHistory(solver=label, rhs_norm=float(res[j].rhs_norm))
        st0 = int(res[j].t_start_ns)
        hist.resid = [float(v) for v in hrs[j][:L].cpu().numpy()]
        hist.matvecs = [int(v) for v in hms[j][:L].cpu().numpy()]
        hist.seconds = [(t_launch - t0) + (int(s) - st0) * 1e-9 for s in stamps]
        hist.status = _STATUS.get(int(res[j].status), f"unknown:{res[j].status}")
        hist.final_true_resid = float(res[j].final_true_resid)
        total_mv += int(res[j].matvecs)
        out.append((xos[j], hist))
    LAST_SOLVE.clear()
    LAST_SOLVE.update(matvecs=total_mv, bodies=max(int(r.iterations_run) for r in res),
                      kernel_launches=int(res[nr - 1].kernel_launches))
    return out


def _batch_solve(A, bs, x_inits, recycle, configs, label):
    t0 = time.perf_counter()
    bs = list(bs)
    if not bs:
        return []
    configs = list(configs) if configs is not None else [SolverConfig()] * len(bs)
    if len(configs) != len(bs):
        raise ValueError("one SolverConfig per right-hand side")
    if any(c.record_iterates for c in configs):
        raise NotImplementedError("record_iterates: use rbicgstab_solve per system")
    x_inits = list(x_inits) if x_inits is not None else [None] * len(bs)
    M, _ = _check_common(A, bs[0], None, configs[0])
    on_device = _is_device(bs[0])
    out = []
    for c0 in range(0, len(bs), BATCH_MAX):
        chunk = range(c0, min(c0 + BATCH_MAX, len(bs)))
        bds = [_dev_vec(_check_common(A, bs[j], None, configs[j])[1]) for j in chunk]
        xds = [_dev_vec(x_inits[j]) for j in chunk]
        res = solve_device_batch(M, bds, xds, recycle, [configs[j] for j in chunk], label, t0)
        _count(A, nm=LAST_SOLVE["matvecs"])
        out += [(x if on_device else to_host(x), h) for x, h in res]
    return out


def rbicgstab_solve_batch(A, bs, x_inits=None, recycle=None, configs=None, precond=None):
    """Multi-right-hand-side extension (not in the
    reference API): ``len(bs)`` independent rbicgstab_solve calls with the same
    operator and recycle space, advanced together on the device (up to 4 per
    launch) so the matrix and the n x k blocks are read once per iteration
    for all of them.  Bit-identical to the separate calls; returns a list of
    (x, ConvergenceHistory) in order."""
    if precond is not None:
        raise NotImplementedError("preconditioning is out of scope on the device path")
    return _batch_solve(A, bs, x_inits, recycle, configs, "rbicgstab")


def bicgstab_solve_batch(A, bs, x_inits=None, configs=None, precond=None):
    """Batched bicgstab_solve (the k = 0 case of rbicgstab_solve_batch)."""
    if precond is not None:
        raise NotImplementedError("preconditioning is out of scope on the device path")
    return _batch_solve(A, bs, x_inits, None, configs, "bicgstab")


class _Split:
    """Split preconditioning of one solve (solvers.py:115-133 _setup_primary,
    :136-144 _setup_dual) on the device: the iteration operator
    L^{-1} A P U^{-1}, bh = L^{-1} b, xh = U P^T x_init, unwind y -> P U^{-1} y
    (dual: bth = U^{-H} P^T b_dual, xth = L^H xt_init, unwind L^{-H})."""

    def __init__(self, A, precond):
        from .ilutp import SplitPreconditionedOperator, _factors
        self.A = A
        self.F = _factors(precond)
        self.op = SplitPreconditionedOperator(A, self.F)
        self.Fd = self.F.device()
        t = torch()
        self.perm = t.as_tensor(self.F.perm, device="cuda")

    def rhs(self, b):
        return self.Fd.apply("lower", _dev_vec(b))

    def guess(self, x):
        if x is None:
            return None
        z = _dev_vec(x)[self.perm]                                  # P^T x
        return device_matrix(self.F.U).spmv(z.contiguous())          # U z

    def unwind(self, y):
        t = self.Fd.apply("upper", y)
        x = torch().empty_like(t)
        x[self.perm] = t                                             # x[perm] = t
        return x

    def rhs_dual(self, bt):
        return self.Fd.apply("upper_h", _dev_vec(bt)[self.perm].contiguous())

    def guess_dual(self, xt):
        if xt is None:
            return None
        return device_matrix(self.F.L).spmv(_dev_vec(xt), transpose=True)   # L^H xt

    def unwind_dual(self, yt):
        return self.Fd.apply("lower_h", yt)

    def true_residual(self, b, x):
        """solvers.py:147-153 with the ORIGINAL operator and right-hand side:
        ||b - A x|| / ||b|| (canonical device dots)."""
        from .recycling import dot
        M = device_matrix(self.A)
        bd = _dev_vec(b)
        r = bd - M.spmv(x)
        rr, bb = dot(r, r), dot(bd, bd)
        v = torch().stack([rr, bb]).cpu().numpy().ravel()
        bn = float(np.sqrt(v[1]))
        return float(np.sqrt(v[0]) / (bn if bn > 0 else 1.0))


def _precond_solve(A, b, x_init, recycle, precond, cfg, label, t0):
    sp = _Split(A, precond)
    M = device_matrix(sp.op)
    if not _is_device(b):
        b = np.asarray(b)
        if np.iscomplexobj(b):
            raise NotImplementedError("complex right-hand sides are out of scope")
    if tuple(b.shape) != (M.n,):
        raise ValueError("right-hand side length does not match the operator")
    xh, hist = solve_device(M, sp.rhs(b), sp.guess(x_init), recycle, cfg, label, t0)
    _count(A, nm=LAST_SOLVE["matvecs"])
    x = sp.unwind(xh)
    hist.final_true_resid = sp.true_residual(b, x)
    return (x if _is_device(b) else to_host(x)), hist


def bicgstab_solve(A, b, x_init=None, precond=None, config=None):
    """solvers.py:156-242 — stabilized BiCG, shadow residual from the seeded
    uniform(-1, 1) stream (drawn on the device, bit-identical to numpy).
    ``precond`` (IlutpFactors): split preconditioning on the device."""
    cfg = config or SolverConfig()
    t0 = time.perf_counter()
    if precond is not None:
        return _precond_solve(A, b, x_init, None, precond, cfg, "bicgstab", t0)
    return _device_solve(A, b, x_init, None, cfg, "bicgstab", t0)


def rbicgstab_solve(A, b, x_init=None, recycle=None, precond=None,
                    config=None):
    """solvers.py:245-361 — BiCGSTAB deflated by a recycle space (Algorithm 2):
    projected start, (I - C Chat^H) after every product, x = x - U xc at the
    end.  With an empty space the arithmetic is that of bicgstab_solve.
    ``precond`` (IlutpFactors): split preconditioning on the device; the
    space then lives in the preconditioned coordinates, as in the reference."""
    cfg = config or SolverConfig()
    t0 = time.perf_counter()
    if precond is not None:
        return _precond_solve(A, b, x_init, recycle, precond, cfg, "rbicgstab", t0)
    return _device_solve(A, b, x_init, recycle, cfg, "rbicgstab", t0)


# ---------------------------------------------------------------------------
# RBiCG generation solve (solvers.py:364-375, 460-638)
# ---------------------------------------------------------------------------

def _tri_block(first, ncols, alphas, betas, rhos):
    """(sub, diag, super) recurrence coefficients of columns first..first+ncols-1
    (solvers.py:524-540), host-side on the few captured scalars."""
    tri = np.full((3, ncols), np.nan)
    m = len(alphas)
    for j in range(ncols):
        g = first + j
        if g <= m:
            a_g = alphas[g - 1]
            diag = 1.0 / a_g
            if g >= 2:
                diag = diag + betas[g - 1] / alphas[g - 2]
            tri[1, j] = diag
            if len(rhos) > g:
                tri[0, j] = -rhos[g] / (a_g * rhos[g - 1])
        if g >= 2 and g - 1 <= m and len(betas) >= g:
            tri[2, j] = -betas[g - 1] * rhos[g - 2] / (alphas[g - 2] * rhos[g - 1])
    return tri


class _CycleHarvest:
    """Host bookkeeping of the capture windows (solvers.py:512-558) over the
    device ring of krb_rbicg."""

    def __init__(self, H, n, callback, keep=True):
        from .recycling import CapturedCycle
        self.CapturedCycle = CapturedCycle
        self.H, self.n, self.callback, self.keep = H, n, callback, keep
        self.start = 1
        self.emitted = 0
        self.cycles = []
        V, Vt, rh, al, be = (ctypes.c_void_p() for _ in range(5))
        _lib.call("krb_rbicg_views", H, ctypes.byref(V), ctypes.byref(Vt),
                  ctypes.byref(rh), ctypes.byref(al), ctypes.byref(be))
        self.ptrs = (V.value, Vt.value, rh.value, al.value, be.value)

    def emit(self, state, st, final=False, launch_next=None):
        """Copy the completed cycle out of the ring and rotate the ring, all
        on the solve's stream ``st`` (so the next cycle's kernel, also on
        ``st``, cannot overwrite columns still being copied even if the
        callback switched streams), then hand the cycle to the callback on
        the caller's current stream, ordered after those copies."""
        ncols, nalpha, npush = int(state[2]), int(state[4]), int(state[6])
        last = self.start + ncols - 1
        if ncols == 0 or last <= self.emitted:
            if launch_next is not None:
                launch_next()
            return
        t = torch()
        cur = t.cuda.current_stream()
        sv = st.value or 0
        if cur.cuda_stream == sv:
            cyc = self._copy_out(state, final, st, ncols, nalpha, npush, last)
        else:
            solve_stream = t.cuda.ExternalStream(sv)
            with t.cuda.stream(solve_stream):
                cyc = self._copy_out(state, final, st, ncols, nalpha, npush, last)
            cur.wait_stream(solve_stream)
        if launch_next is None:
            if self.callback is not None:
                self.callback(cyc)
            return
        if self.callback is None:
            launch_next()
            return
        # the next cycle's iterations are launched when the callback starts
        # host-only work (device.flush_pending), else right after it
        defer_launch(launch_next)
        try:
            self.callback(cyc)
        except BaseException:
            drop_pending()
            raise
        flush_pending()

    def _copy_out(self, state, final, st, ncols, nalpha, npush, last):
        t = torch()
        n = self.n
        Vd = t.empty((ncols, n), dtype=t.float64, device="cuda")
        Vtd = t.empty((ncols, n), dtype=t.float64, device="cuda")
        _lib.copy_d2d(Vd, self.ptrs[0], ncols * n)
        _lib.copy_d2d(Vtd, self.ptrs[1], ncols * n)
        rhos, alphas, betas = _lib.fetch_f64_many(
            [(self.ptrs[2], npush), (self.ptrs[3], nalpha), (self.ptrs[4], nalpha)])
        start = self.start
        cyc = self.CapturedCycle(
            V=Vd, Vt=Vtd, first_index=start,
            tri=lambda: _tri_block(start, ncols, alphas, betas, rhos))   # lazy
        if self.keep:
            self.cycles.append(cyc)
        self.emitted = last
        if not final and ncols > 2:
            # the copies above are queued first on the same stream, so the
            # ring may be rotated and refilled before the callback runs
            _lib.call("krb_rbicg_rotate", self.H, 2, st)
            self.start = last - 1
            state[2] = 2          # the ring now holds the two overlap columns
        return cyc


def rbicg_solve(A, b, b_dual=None, x_init=None, x_init_dual=None, recycle=None,
                precond=None, config=None, cycle_callback=None, keep_cycles=True):
    """solvers.py:460-638 — two-sided deflated BiCG with cycle harvesting.
    Iterations run on the device (CUDA graph, device WHILE node that pauses
    at every completed cycle); each captured cycle is handed to
    ``cycle_callback`` as it completes.  Returns (x, x_dual, history, cycles).

    ``keep_cycles=False`` (extension, not in the reference signature) drops
    each cycle after its callback instead of returning all of them: the
    cycles are device-resident n x (s+2) pairs, 8 GB each at C5, and a
    caller that consumes them in the callback (the sequence policy) would
    otherwise hold ~100 GB of HBM for a list it discards."""
    cfg = config or SolverConfig()
    t0 = time.perf_counter()
    if cfg.record_iterates:
        raise NotImplementedError("record_iterates is supported by bicgstab_solve / "
                                  "rbicgstab_solve on the device, not by rbicg_solve")
    sp = _Split(A, precond) if precond is not None else None
    M, b = _check_common(sp.op if sp is not None else A, b, None, cfg)
    t = torch()
    n = M.n
    ctx = Context.get()
    R = None
    if recycle is not None and recycle.k > 0:
        R = RecycleSpace.of(recycle)
        if R.n != n:
            raise ValueError("recycle space dimension does not match the operator")
    draws = 0
    if b_dual is None:
        btd = device_uniform(cfg.seed, n, 0)
        draws = 1
    else:
        if not _is_device(b_dual) and np.iscomplexobj(np.asarray(b_dual)):
            raise NotImplementedError("complex dual right-hand sides are out of scope")
        btd = _dev_vec(b_dual)
    on_device = _is_device(b)
    bd = _dev_vec(b)
    xd = _dev_vec(x_init)
    xtd = _dev_vec(x_init_dual)
    if sp is not None:   # solvers.py:115-144: iterate in preconditioned coordinates
        bd, btd = sp.rhs(bd), sp.rhs_dual(btd)
        xd, xtd = sp.guess(xd), sp.guess_dual(xtd)
    H = ctypes.c_void_p()
    view = R.view() if R is not None else None
    call_retry_oom("krb_rbicg_create", ctypes.byref(H), ctx.h, M.h,
              ctypes.byref(view) if view is not None else None,
              int(cfg.s), int(cfg.max_itn), stream_ptr())
    try:
        # 2: persistent kernel per cycle (small n), 1: graph, 0: host loop
        graph = max(0, min(_auto_mode(n), 2))
        dual = (ctypes.c_double * 3)()
        n_rmv = 0
        for attempt in range(4):
            _lib.call("krb_rbicg_start", H, ptr(bd), ptr(btd), ptr(xd), ptr(xtd),
                      float(cfg.tol), float(cfg.breakdown_tol), int(graph), dual,
                      stream_ptr())
            if xtd is not None:
                n_rmv += 1
            rho = dual[0]
            scale = float(np.sqrt(dual[1]) * np.sqrt(dual[2]))
            if abs(rho) > cfg.breakdown_tol * scale or scale == 0.0:
                break
            xtd = device_uniform(cfg.seed, n, draws * n)      # solvers.py:373
            draws += 1
        else:
            raise ValueError("initial residual pair stays biorthogonal after "
                             "re-draws; supply a different b_dual or seed")
        _lib.call("krb_rbicg_set_counts", H, 1 if xd is not None else 0, n_rmv,
                  stream_ptr())
        status = ctypes.c_int32()
        _lib.call("krb_rbicg_begin", H, ctypes.byref(status), stream_ptr())
        harvest = _CycleHarvest(H, n, cycle_callback, keep_cycles)
        state = (ctypes.c_int64 * 7)()
        launched = ctypes.c_int32()
        st = stream_ptr()   # the solve's stream, fixed even if a callback switches streams

        def launch_next():
            _lib.call("krb_rbicg_launch", H, ctypes.byref(launched), st)

        launch_next()
        while True:
            _lib.call("krb_rbicg_wait", H, state, st)
            running = state[0] == 0
            if state[1]:
                harvest.emit(state, st, final=False,
                             launch_next=launch_next if running else None)
            elif running:
                launch_next()
            if not running:
                break
        harvest.emit(state, st, final=True)
        xo = t.empty(n, dtype=t.float64, device="cuda")
        xto = t.empty(n, dtype=t.float64, device="cuda")
        L = int(cfg.max_itn) + 2
        hr = t.empty(L, dtype=t.float64, device="cuda")
        hrt = t.empty(L, dtype=t.float64, device="cuda")
        hm = t.empty(L, dtype=t.int64, device="cuda")
        ht = t.empty(L, dtype=t.int64, device="cuda")
        res = _lib.SolveResult()
        counts = (ctypes.c_int64 * 2)()
        btn = ctypes.c_double()
        _lib.call("krb_rbicg_finish", H, ptr(xo), ptr(xto), ptr(hr), ptr(hrt),
                  ptr(hm), ptr(ht), ctypes.byref(res), counts, ctypes.byref(btn),
                  stream_ptr())
    finally:
        _lib.load().krb_rbicg_destroy(H)
    Lh = int(res.hist_len)
    hist = ConvergenceHistory(solver="rbicg", rhs_norm=float(res.rhs_norm),
                              rhs_norm_dual=float(btn.value))
    # one device->host read for the four history arrays (bit views)
    h4 = t.stack([hr[:Lh].view(t.int64), hrt[:Lh].view(t.int64), hm[:Lh],
                  ht[:Lh]]).cpu().numpy()
    stamps = h4[3]
    hist.resid = [float(v) for v in h4[0].view(np.float64)]
    hist.resid_dual = [float(v) for v in h4[1].view(np.float64)]
    hist.matvecs = [int(v) for v in h4[2]]
    st0 = int(res.t_start_ns)
    base = time.perf_counter() - t0 - (int(stamps[-1]) - st0) * 1e-9 if Lh else 0.0
    hist.seconds = [base + (int(s) - st0) * 1e-9 for s in stamps]
    hist.status = _STATUS.get(int(res.status), f"unknown:{res.status}")
    hist.final_true_resid = float(res.final_true_resid)
    LAST_SOLVE.clear()
    LAST_SOLVE.update(matvecs=int(res.matvecs), bodies=int(res.iterations_run),
                      kernel_launches=int(res.kernel_launches))
    _count(A, nm=int(counts[0]), nr=int(counts[1]))
    if sp is not None:
        xo, xto = sp.unwind(xo), sp.unwind_dual(xto)
        hist.final_true_resid = sp.true_residual(b, xo)
    if on_device:
        return xo, xto, hist, harvest.cycles
    return to_host(xo), to_host(xto), hist, harvest.cycles
