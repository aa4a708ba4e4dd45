"""Sequence policy: the caller of the hot path (reference driver.py:78-180,
re-stated without ILUTP).

For a sequence of systems A_i x = b_{i,kappa}:

* the first system runs the two-sided recycling solver (rbicg_solve) with a
  per-cycle ``update_recycle_space(..., res_tol=4.0)`` harvest
  (driver.py:111-126); if it does not converge the space is dropped and the
  system is redone with bicgstab_solve (driver.py:127-136);
* policy="first" (default): every later system runs rbicgstab_solve against
  the space, refreshed with ``refresh_images`` (2k products) at each matrix
  change (driver.py:112-113), with the driver's guard: at most
  max(block_itn, 50) iterations, then an unrecycled reseeded retry
  (driver.py:142-156);
* policy="verbatim": the reference's own schedule — RBiCG + harvest on
  kappa = 0 of EVERY matrix, rbicgstab on kappa > 0 (C3's 4-rhs blocks);
* a plain bicgstab_solve baseline track runs on the same systems
  (driver.py:162-168) unless ``baseline=False``;
* precond="ilutp": the reference driver's split preconditioning
  (driver.py:99-107): one ILUTP factorization per matrix, every solve of
  both tracks on L^{-1} A P U^{-1} with right-hand side L^{-1} b.

Every product is metered through CountingOperator wrappers; aux products
(refreshes, harvest updates) land in ``aux_matvecs`` exactly as
driver.py:172-176 computes them.  The policy is backend-agnostic: ``api``
supplies the solver / recycle functions (this package by default; the tests
pass the CPU oracle to check the device path decision for decision).
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field, replace

import numpy as np


@dataclass
class RunReport:
    """driver.py:33-55."""
    label: str
    histories: list = field(default_factory=list)
    aux_matvecs: int = 0
    seconds: float = 0.0

    @property
    def total_matvecs(self) -> int:
        return sum(h.total_matvecs for h in self.histories) + self.aux_matvecs

    @property
    def total_iterations(self) -> int:
        return sum(h.iterations for h in self.histories)

    @property
    def per_system_matvecs(self) -> list:
        return [h.total_matvecs for h in self.histories]


@dataclass
class SequenceResult:
    """driver.py:58-70."""
    recycling: RunReport
    baseline: RunReport | None
    rebuild_points: list
    rebuild_matvecs: list
    space_dims: list

    @property
    def savings(self) -> float:
        if self.baseline is None:
            return float("nan")
        base = self.baseline.total_matvecs
        return 1.0 - self.recycling.total_matvecs / base if base else 0.0


def _reseed(cfg):
    """driver.py:73-75."""
    return replace(cfg, seed=cfg.seed + 104729)


def default_api():
    import paper_1406_2831_b200 as P
    return P


def run_sequence(seq, k=None, s=None, tol=None, max_itn=None, seed=0,
                 policy="first", baseline=True, api=None, systems=None,
                 max_seconds=None, batch=True, precond=None, drop_tol=1e-4,
                 pivot_tol=0.1):
    """Run the recycling policy (and the baseline) over ``seq``
    (a workloads.SequenceSpec).  ``max_seconds`` stops after the first system
    that ends past the budget (bounded CPU samples).  ``batch``: when the api
    has the multi-right-hand-side solvers, the right-hand sides of one matrix
    that share the recycle space (kappa > 0 under "verbatim"; every kappa of
    the baseline track) are solved together -- bit-identical to the
    one-by-one schedule, the matrix and the n x k blocks read once per
    iteration for all of them.  Returns a SequenceResult."""
    api = api or default_api()
    k = seq.k if k is None else k
    s = seq.s if s is None else s
    if precond not in (None, "ilutp"):
        raise ValueError("precond must be None or 'ilutp'")
    if precond is not None:
        batch = False   # the multi-rhs path has no preconditioned operator
    tol = seq.tol if tol is None else tol
    max_itn = seq.max_itn if max_itn is None else max_itn
    use_batch = batch and hasattr(api, "rbicgstab_solve_batch") and seq.rhs_per_matrix > 1
    rec = RunReport("recycling")
    base = RunReport("baseline") if baseline else None
    rebuild_points, rebuild_matvecs, space_dims = [], [], []
    space = None
    block_itn = 1
    rec_applied = base_applied = 0
    gidx = 0
    total = seq.num_systems if systems is None else min(systems, seq.num_systems)
    t_start = time.perf_counter()
    prefetch = getattr(api, "prefetch_matrix", None)
    # the cycles are consumed by the harvest callback; a backend that can
    # drop them instead of returning the whole list is told to (device
    # cycles are n x (s+2) pairs: ~100 GB per C5 generation solve)
    import inspect
    try:
        drop_kw = ({"keep_cycles": False}
                   if "keep_cycles" in inspect.signature(api.rbicg_solve).parameters else {})
    except (TypeError, ValueError):
        drop_kw = {}
    A_next = None
    for i in range(seq.num_matrices):
        if gidx >= total:
            break
        if A_next is not None:
            A = A_next
        else:
            A = api.SparseMatrix.from_csr(seq.matrix(i))
            if prefetch is not None:
                # queue this matrix's own upload first: the next matrix's
                # prefetch below must not share the link with it
                prefetch(A)
        A_next = None
        if prefetch is not None and i + 1 < seq.num_matrices and \
                gidx + min(seq.rhs_per_matrix, total - gidx) < total:
            # the next matrix's upload overlaps this matrix's solves
            A_next = api.SparseMatrix.from_csr(seq.matrix(i + 1))
            prefetch(A_next)
        rhs = lambda kk, _i=i: seq.rhs(_i, kk)
        if precond == "ilutp":
            # driver.py:99-107: one ILUTP factorization per matrix, both tracks
            # iterate on L^{-1} A P U^{-1} with b -> L^{-1} b
            factors = api.ilutp_factor(A, drop_tol=drop_tol, pivot_tol=pivot_tol)
            op_rec = api.CountingOperator(api.SplitPreconditionedOperator(A, factors))
            op_base = api.CountingOperator(api.SplitPreconditionedOperator(A, factors))
            rhs = lambda kk, _i=i, _f=factors: api.apply_left(_f, seq.rhs(_i, kk))
        else:
            op_rec = api.CountingOperator(A)
            op_base = api.CountingOperator(A)
        nk = min(seq.rhs_per_matrix, total - gidx)
        pre_rec, pre_base = {}, {}   # kappa -> (history, seconds) of batched solves
        for kappa in range(nk):
            b = rhs(kappa)
            cfg = api.SolverConfig(tol=tol, max_itn=max_itn, k=k, s=s, seed=seed + gidx)
            t0 = time.perf_counter()
            harvest_now = (gidx == 0) if policy == "first" else (kappa == 0)
            if harvest_now:
                if space is not None and i > 0:
                    space = api.refresh_images(space, op_rec)
                state = {"space": space}

                def harvest(cycle, _state=state, _op=op_rec):
                    _state["space"] = api.update_recycle_space(
                        _op, [cycle], _state["space"], k, res_tol=4.0)

                dual_rhs = np.ones(A.nrows if hasattr(A, "nrows") else seq.n)
                _, _, hist, _ = api.rbicg_solve(op_rec, b, b_dual=dual_rhs,
                                                recycle=space, config=cfg,
                                                cycle_callback=harvest, **drop_kw)
                if hist.status == "converged":
                    space = state["space"]
                else:
                    space = None
                    _, hist = api.bicgstab_solve(op_rec, b, config=cfg)
                block_itn = max(hist.iterations, 1)
                rebuild_points.append(gidx)
                rebuild_matvecs.append(hist.total_matvecs)
                space_dims.append(space.k if space is not None else 0)
            else:
                if kappa == 0 and space is not None and i > 0:
                    space = api.refresh_images(space, op_rec)
                # driver.py:142 gates on the space's existence, not its size:
                # an empty harvested space still gets the capped attempt and
                # the reseeded retry
                recycled = space is not None
                cap = min(max_itn, max(block_itn, 50))
                if use_batch and kappa not in pre_rec and kappa + 1 < nk:
                    # every remaining rhs of this matrix shares the space
                    ks = list(range(kappa, nk))
                    cfgs = [api.SolverConfig(tol=tol, max_itn=cap if recycled else max_itn,
                                             k=k, s=s, seed=seed + gidx + (kk - kappa))
                            for kk in ks]
                    tb = time.perf_counter()
                    out = api.rbicgstab_solve_batch(op_rec, [rhs(kk) for kk in ks],
                                                    recycle=space if recycled else None,
                                                    configs=cfgs)
                    share = (time.perf_counter() - tb) / len(ks)
                    for kk, (_, h) in zip(ks, out):
                        pre_rec[kk] = (h, share)
                if kappa in pre_rec:
                    hist, _ = pre_rec[kappa]
                    if recycled and hist.status != "converged":
                        _, hist = api.rbicgstab_solve(op_rec, b, recycle=None,
                                                      config=_reseed(cfg))
                elif recycled:
                    attempt = replace(cfg, max_itn=cap)
                    _, hist = api.rbicgstab_solve(op_rec, b, recycle=space,
                                                  config=attempt)
                    if hist.status != "converged":
                        _, hist = api.rbicgstab_solve(op_rec, b, recycle=None,
                                                      config=_reseed(cfg))
                else:
                    _, hist = api.rbicgstab_solve(op_rec, b, recycle=None, config=cfg)
            rec.seconds += time.perf_counter() - t0 + (pre_rec[kappa][1] if kappa in pre_rec else 0.0)
            rec.histories.append(hist)
            if base is not None:
                t0 = time.perf_counter()
                if use_batch and kappa == 0 and nk > 1:
                    cfgs = [api.SolverConfig(tol=tol, max_itn=max_itn, k=k, s=s,
                                             seed=seed + gidx + kk) for kk in range(nk)]
                    tb = time.perf_counter()
                    out = api.bicgstab_solve_batch(op_base, [rhs(kk) for kk in range(nk)],
                                                   configs=cfgs)
                    share = (time.perf_counter() - tb) / nk
                    for kk, (_, h) in enumerate(out):
                        pre_base[kk] = (h, share)
                    t0 = time.perf_counter()
                if kappa in pre_base:
                    bh, extra = pre_base[kappa]
                else:
                    _, bh = api.bicgstab_solve(op_base, b, config=cfg)
                    extra = 0.0
                if bh.status != "converged":
                    _, bh = api.bicgstab_solve(op_base, b, config=_reseed(cfg))
                base.seconds += time.perf_counter() - t0 + extra
                base.histories.append(bh)
            gidx += 1
            if max_seconds is not None and time.perf_counter() - t_start > max_seconds:
                total = gidx
        rec_applied += op_rec.total
        base_applied += op_base.total
    rec.aux_matvecs = rec_applied - sum(h.total_matvecs for h in rec.histories)
    if base is not None:
        base.aux_matvecs = base_applied - sum(h.total_matvecs for h in base.histories)
    return SequenceResult(recycling=rec, baseline=base, rebuild_points=rebuild_points,
                          rebuild_matvecs=rebuild_matvecs, space_dims=space_dims)
