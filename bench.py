#!/usr/bin/env python
"""Recycling-BiCGSTAB sequence benchmark on B200 (BASELINE.json metric:
"RBiCGSTAB sequence solve time & iters/s; SpMV+BLAS-1 HBM GB/s vs 8 TB/s").

Default workload: C5 (BASELINE configs[4], the largest single-GPU config:
27-point 256^3, n = 16.8 M, 449 M nnz, k = 30, 8 systems).

One step = the recycled part of the sequence: RBiCGSTAB (solvers.py:245-361)
on systems 1..S-1 of the config with a k-dimensional recycle space, x0 = 0,
the config's tol and max_itn.  The space enters the step biorthonormalized
against system 1's matrix (a seeded N(0,1) basis pair, built before timing)
and is carried to every later matrix with refresh_images (2k products, the
policy's refresh at a matrix change, driver.py:112-113) inside the step.
Each system's device matrix (SELL-32 build, transpose for the refresh) is
created inside the step from its CSR arrays.

  value        iterations / s over the step, CSR arrays and right-hand sides
               resident in HBM before timing (CUDA events, L2 flushed between
               steps, the inputs are > L2 anyway)
  e2e          the same step through the public drop-in API with HOST numpy
               inputs (page-locked; uploaded inside the timed region), the
               solutions read back; e2e_pageable: plain pageable numpy inputs
  roofline     the step's dominant kernel by its live device-time share
               (per-kernel %globaltimer accounting inside the timed region)
  cpu_baseline the reference's algorithm (oracle RefOps: krecycle's own numpy
               / scipy / OpenBLAS calls, bit-identical to it) on this host:
               the same RBiCGSTAB iterations (system 1, same space), bounded
  full_policy  the whole C5 sequence policy once (RBiCG generation with the
               m = 60 recycle update on system 0, refresh + guarded RBiCGSTAB
               on the rest), extra key
  baseline     GPU BiCGSTAB without recycling on the same systems (matvecs)

--impl reference prints the CPU reference arm (same metric / config / unit).
--gpus N > 1 (torchrun) runs N independent replicas: the sequence is serial
(SURVEY.md §8(e)); value sums the iterations of all ranks over the max time.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
import types

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

from paper_1406_2831_b200 import workloads as W  # noqa: E402

METRIC = "RBiCGSTAB sequence iters/s (recycled systems, k-dim space refreshed per matrix)"
SPACE_SEED = 12345


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c5")
    ap.add_argument("--systems", type=int, default=None,
                    help="recycled systems per step (default: all after the first)")
    ap.add_argument("--cpu-iters", type=int, default=3,
                    help="RBiCGSTAB iterations per CPU sample (reference arm / cpu_baseline)")
    ap.add_argument("--e2e-steps", type=int, default=4)
    ap.add_argument("--pageable-steps", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-policy", action="store_true")
    return ap.parse_args()


def peaks():
    p = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class Workload:
    """The config's systems 1..S materialised on the host once, outside any
    timed region (C5: the matrices share one row_ptr / col_idx pair), plus
    the seeded basis pair the recycle space starts from."""

    def __init__(self, name, systems=None):
        self.name = name
        self.seq = seq = W.make_sequence(name)
        keys = [(i, kap) for i in range(seq.num_matrices)
                for kap in range(seq.rhs_per_matrix)]
        self.first = keys[0]
        rest = keys[1:]
        self.keys = rest if systems is None else rest[:systems]
        self.mats = {}
        for i, _ in self.keys:
            if i not in self.mats:
                self.mats[i] = seq.matrix_fn(i)
        self.rhs = {key: seq.rhs(*key) for key in self.keys}
        A = self.mats[self.keys[0][0]]
        self.n, self.nnz, self.k = A.n, A.nnz, seq.k
        r = np.random.default_rng(SPACE_SEED)
        self.U0 = r.standard_normal((self.n, self.k))
        self.Ut0 = r.standard_normal((self.n, self.k))

    def config(self, world):
        return {"workload": f"{self.name}: RBiCGSTAB on systems "
                            f"{self.keys[0][0]}..{self.keys[-1][0]} "
                            f"({len(self.keys)} solves) of {self.seq.meta}",
                "n": self.n, "nnz": self.nnz, "k": self.k,
                "systems": len(self.keys), "tol": self.seq.tol,
                "max_itn": self.seq.max_itn,
                "space": f"seeded N(0,1) basis pair (seed {SPACE_SEED}) biorthonormalized "
                         f"against system {self.keys[0][0]}, refresh_images onto every "
                         "later matrix inside the step",
                "l2": "inputs > L2; 1 GB buffer written between timed steps",
                "parallelism": f"replicas{world}" if world > 1 else "single"}

    def unique_arrays(self):
        """(name, host array) of every distinct CSR array of the step."""
        seen, out = set(), []
        for i, A in self.mats.items():
            for nm, a in (("row_ptr", A.row_ptr), ("col_idx", A.col_idx),
                          ("values", A.values)):
                if id(a) not in seen:
                    seen.add(id(a))
                    out.append((f"{nm}{i}", a))
        return out


# ---------------------------------------------------------------------------
class Clocks:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index, self.proc, self.lines = index, None, []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def wait_first_sample(self, timeout=10.0):
        t0 = time.time()
        while self.proc is not None and len(self.lines) < 2 and time.time() - t0 < timeout:
            time.sleep(0.05)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        load = [s for s in sm if mx and s > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(load) if load else None,
                "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# kernels of one RBiCGSTAB iteration (graph driver slots, include/krb.h
# krb_solve_config.d_kernel_times) and their algorithmic bytes per launch
# (fp64 values, int32 indices)
KERNEL_GROUPS = {
    "k_iter_spmv (q = A p, t = A s)": (1, 5),
    "k_proj_dot (Chat^T q, Chat^T t)": (2, 6),
    "k_phase<PROJ_Q/T> (v -= C coef + 2 dots)": (3, 7),
    "k_phase<PUPDATE> (p update)": (0,),
    "k_phase<SUPD> (s = r - alpha q, ||s||)": (4,),
    "k_phase<XR> (x, r updates + 2 dots)": (8,),
}


def kernel_bytes(group, n, nnz, k):
    if group.startswith("k_iter_spmv"):
        return W.spmv_bytes(n, nnz)
    if group.startswith("k_proj_dot"):
        return 8 * n * k + 8 * n
    if group.startswith("k_phase<PROJ"):
        return 8 * n * k + 24 * n
    if "PUPDATE" in group:
        return 32 * n
    if "SUPD" in group:
        return 24 * n
    return 56 * n


def _traffic(name, group):
    tp = os.path.join(REPO, "profiles", "traffic.json")
    if not os.path.exists(tp):
        return None, None
    for tj in json.load(open(tp)).get(name, []):
        if group.startswith(tj["kernel"]):
            return int(tj["bytes_per_launch"]), tj.get("source")
    return None, None


def roofline_from_ktime(wl, kt, t_total):
    """Dominant kernel of the measured step by live device-time share."""
    peak, src = peaks()
    groups = {}
    for g, slots in KERNEL_GROUPS.items():
        ns = sum(int(kt[4 * s + 1]) for s in slots)
        cnt = sum(int(kt[4 * s + 2]) for s in slots)
        if cnt:
            groups[g] = (ns, cnt)
    if not groups:
        return None, {}
    shares = {g: {"share": round(ns * 1e-9 / t_total, 4), "launches": cnt,
                  "avg_us": round(ns / cnt / 1e3, 2),
                  "GBps": round(kernel_bytes(g, wl.n, wl.nnz, wl.k) / (ns / cnt), 1)}
              for g, (ns, cnt) in groups.items()}
    dom = max(groups, key=lambda g: groups[g][0])
    ns, cnt = groups[dom]
    b = kernel_bytes(dom, wl.n, wl.nnz, wl.k)
    ach = b / (ns / cnt)            # bytes / ns = GB/s
    traffic, tsrc = _traffic(wl.name, dom)
    roof = {"bound": "hbm", "kernel": dom, "achieved": round(ach, 1), "peak": peak,
            "peak_source": src, "unit": "GB/s", "frac": round(ach / peak, 4),
            "traffic": traffic, "traffic_source": tsrc,
            "bytes_per_launch": b, "launch_us": round(ns / cnt / 1e3, 2),
            "launches": cnt, "share_of_step": shares[dom]["share"],
            "timing": "live: CTA 0 start -> last CTA end (%globaltimer) of every "
                      "launch inside the timed steps"}
    sb = getattr(wl, "spmv_stream_bytes", None)
    if sb and "k_iter_spmv (q = A p, t = A s)" in shares:
        sp = shares["k_iter_spmv (q = A p, t = A s)"]
        st = sb / (sp["avg_us"] * 1e3)
        sp.update({"format": wl.spmv_format, "stream_bytes_per_launch": sb,
                   "GBps_stream": round(st, 1), "frac_stream": round(st / peak, 4)})
        if dom.startswith("k_iter_spmv"):
            roof.update({
                "format": wl.spmv_format, "format_stats": wl.spmv_stream_stats,
                "stream_bytes_per_launch": sb, "achieved_stream": round(st, 1),
                "frac_stream": round(st / peak, 4),
                "note": "bytes_per_launch = SURVEY §8(d) algorithmic SpMV bytes "
                        "(12 nnz + 4 (n+1) + 16 n: int32 column indices); the "
                        "offset-coded SELL-32 format streams fewer (values + 1-byte "
                        "codes / shared offset rows): stream_bytes_per_launch, "
                        "frac_stream"})
    return roof, shares


# ---------------------------------------------------------------------------
def gpu_arm(args, wl, rank, world):
    import torch
    import paper_1406_2831_b200 as P
    from paper_1406_2831_b200 import _lib, device as D

    torch.cuda.set_device(rank % max(torch.cuda.device_count(), 1))
    cfgs = [P.SolverConfig(tol=wl.seq.tol, max_itn=wl.seq.max_itn, k=wl.k,
                           s=wl.seq.s, seed=j + 1) for j in range(len(wl.keys))]
    # device-resident inputs: each distinct CSR array once (C5 shares the
    # index arrays across the systems), every right-hand side
    dev = {id(a): D.to_device(a, a.dtype) for _, a in wl.unique_arrays()}
    drhs = {key: D.to_device(b) for key, b in wl.rhs.items()}
    up = {i: (dev[id(A.row_ptr)], dev[id(A.col_idx)], dev[id(A.values)])
          for i, A in wl.mats.items()}
    i0 = wl.keys[0][0]
    A0 = wl.mats[i0]
    M0 = D.DeviceMatrix(A0.n, A0.row_ptr, A0.col_idx, A0.values, uploaded=up[i0])
    wl.spmv_format, wl.spmv_stream_bytes = M0.format, M0.stream_bytes
    wl.spmv_stream_stats = M0.stream_stats
    space0 = P.biorthonormalize(wl.U0, wl.Ut0, M0)
    del M0
    flush = torch.empty(128 * 1024 * 1024, dtype=torch.float64, device="cuda")  # 1 GB > L2
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    def step():
        its, hists, space, last_i, M = 0, [], space0, None, None
        for j, (i, kap) in enumerate(wl.keys):
            if i != last_i:
                A = wl.mats[i]
                M = D.DeviceMatrix(A.n, A.row_ptr, A.col_idx, A.values, uploaded=up[i])
                if j > 0:
                    space = P.refresh_images(space, M)
                last_i = i
            _, h = P.rbicgstab_solve(M, drhs[(i, kap)], recycle=space, config=cfgs[j])
            its += h.iterations
            hists.append(h)
        return its, hists, space

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    ktime = torch.zeros(384, dtype=torch.int64, device="cuda")
    clocks = Clocks(torch.cuda.current_device())
    clocks.start()
    clocks.wait_first_sample()
    times, its, last = [], 0, None
    l0 = _lib.launch_count()
    with _lib.tuning(kernel_times=ktime):
        for _ in range(args.steps):
            flush.fill_(1.0)
            barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            it, hists, sp = step()
            e1.record()
            torch.cuda.synchronize()
            barrier()
            times.append(e0.elapsed_time(e1) / 1e3)
            its += it
            last = (hists, sp)
    launches = _lib.launch_count() - l0
    clk = clocks.stop()
    t_total = sum(times)
    its_all = its
    if world > 1:
        import torch.distributed as dist
        tt = torch.tensor([t_total, its], dtype=torch.float64, device="cuda")
        mx = tt.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        dist.all_reduce(tt, op=dist.ReduceOp.SUM)
        t_total, its_all = float(mx[0]), float(tt[1])
    hists, sp = last
    roof, shares = roofline_from_ktime(wl, ktime.cpu().numpy(), sum(times))
    out = {"t_total": t_total, "iters": its, "iters_all": its_all,
           "step_ms": [round(1e3 * t, 1) for t in times], "launches": launches,
           "clocks": clk, "roofline": roof, "kernel_shares": shares,
           "iterations_per_system": [h.iterations for h in hists],
           "matvecs_per_system": [h.total_matvecs for h in hists],
           "statuses": [h.status for h in hists],
           "final_true_resid_max": max(h.final_true_resid for h in hists),
           "checks": {"all_converged": all(h.status == "converged" for h in hists),
                      "true_resid_le_tol": all(h.final_true_resid <= 1.1 * wl.seq.tol
                                               for h in hists)},
           "space_k_last": sp.k,
           "histories_head": {str(j): [float(v) for v in hists[j].resid[:51]]
                              for j in (0, len(hists) - 1)},
           "matvecs_head": [int(v) for v in hists[0].matvecs[:51]]}
    B_it = W.bytes_per_iteration(wl.n, wl.nnz, wl.k)
    us_it = 1e6 * sum(times) / max(its, 1)
    out["iteration"] = {"us_per_iteration_incl_setup_refresh": round(us_it, 1),
                        "bytes_per_iteration": B_it,
                        "x_of_8TBps_time": round(us_it * 1e-6 / (B_it / 8e12), 3),
                        "x_of_measured_peak_time": round(
                            us_it * 1e-6 / (B_it / (peaks()[0] * 1e9)), 3)}

    # GPU BiCGSTAB without recycling on the same systems (device-resident)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    b_it = b_mv = 0
    e0.record()
    last_i, M = None, None
    for j, (i, kap) in enumerate(wl.keys):
        if i != last_i:
            A = wl.mats[i]
            M = D.DeviceMatrix(A.n, A.row_ptr, A.col_idx, A.values, uploaded=up[i])
            last_i = i
        _, h = P.bicgstab_solve(M, drhs[(i, kap)], config=cfgs[j])
        b_it += h.iterations
        b_mv += h.total_matvecs
    e1.record()
    torch.cuda.synchronize()
    tb = e0.elapsed_time(e1) / 1e3
    rec_mv = sum(out["matvecs_per_system"]) + 2 * wl.k * (len(wl.mats) - 1)
    out["baseline"] = {"iters": b_it, "matvecs": b_mv, "seconds": round(tb, 4),
                       "iters_per_s": b_it / tb,
                       "recycled_matvecs_incl_refresh": rec_mv,
                       "matvec_savings": 1.0 - rec_mv / b_mv if b_mv else None}
    del M
    dev.clear()
    drhs.clear()
    up.clear()
    torch.cuda.empty_cache()

    out["e2e"] = None
    if not args.no_e2e:
        for key, pinned, on in (("e2e", True, True),
                                ("e2e_pageable", False, args.pageable_steps > 0)):
            if not on:
                continue
            try:
                out[key] = e2e_arm(args, wl, space0, cfgs, flush, barrier, world,
                                   pinned=pinned)
            except Exception as e:   # reported, never hidden
                out[key] = {"error": f"{type(e).__name__}: {e}"}
                D.MATRICES.clear()
                torch.cuda.synchronize()
                torch.cuda.empty_cache()
    del space0
    torch.cuda.empty_cache()
    if not args.no_policy:
        out["full_policy"] = full_policy(wl)
    return out


def e2e_arm(args, wl, space0, cfgs, flush, barrier, world, pinned):
    """The step through the public drop-in API with host numpy inputs: every
    system's CSR and right-hand side uploaded inside the timed region (the
    next matrix's upload overlaps the current solve for page-locked inputs,
    as run_sequence does), the solutions read back to host numpy."""
    import torch
    import paper_1406_2831_b200 as P
    from paper_1406_2831_b200 import device as D

    if pinned:
        cache = {}

        def pin(a):
            if id(a) not in cache:
                cache[id(a)] = D.pinned_copy(a)
            return cache[id(a)]
        mats = {i: W.CSR(A.n, pin(A.row_ptr), pin(A.col_idx), pin(A.values))
                for i, A in wl.mats.items()}
        rhs = {key: D.pinned_copy(b) for key, b in wl.rhs.items()}
    else:
        mats, rhs = wl.mats, wl.rhs

    def step():
        D.MATRICES.clear()
        its, space, last_i, A = 0, space0, None, None
        order = [i for i in dict.fromkeys(i for i, _ in wl.keys)]
        sms = {}
        for j, (i, kap) in enumerate(wl.keys):
            if i != last_i:
                A = sms.pop(i, None)
                if A is None:
                    A = P.SparseMatrix.from_csr(mats[i])
                    P.prefetch_matrix(A)   # its own upload queued ahead of the next one's
                nxt = order.index(i) + 1
                if nxt < len(order):
                    sms[order[nxt]] = P.SparseMatrix.from_csr(mats[order[nxt]])
                    P.prefetch_matrix(sms[order[nxt]])
                if j > 0:
                    space = P.refresh_images(space, A)
                last_i = i
            x, h = P.rbicgstab_solve(A, rhs[(i, kap)], recycle=space, config=cfgs[j])
            assert isinstance(x, np.ndarray)
            its += h.iterations
        return its

    nsteps = args.e2e_steps if pinned else args.pageable_steps
    step()   # warm-up (the value arm already warmed every kernel / graph)
    torch.cuda.synchronize()
    e_times, e_its = [], 0
    for _ in range(max(1, min(nsteps, args.steps))):
        flush.fill_(1.0)
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e_its += step()
        torch.cuda.synchronize()
        e_times.append(time.perf_counter() - t0)
    D.MATRICES.clear()
    e_total = sum(e_times)
    if world > 1:
        import torch.distributed as dist
        tt = torch.tensor([e_total], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e_total = float(tt.item())
    # bytes crossing the link per step: every values array, the right-hand
    # sides, and each DISTINCT index array once (the systems share one frozen
    # row_ptr / col_idx pair, which device._upload_indices uploads once per
    # step: the step starts by dropping every device copy)
    uniq = {id(a): a.nbytes for A in mats.values() for a in (A.row_ptr, A.col_idx, A.values)}
    h2d = sum(uniq.values()) + sum(b.nbytes for b in rhs.values())
    d2h = sum(8 * wl.n + 24 * (wl.seq.max_itn + 1) for _ in wl.keys)
    return {"value": e_its * world / e_total, "unit": "iters/s",
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "steps": len(e_times), "s_per_step": round(e_total / len(e_times), 3),
            "inputs": ("numpy CSR + rhs in page-locked host memory; every matrix's values "
                       "and the shared index arrays (once) uploaded per step, the next "
                       "matrix prefetched during the current solve") if pinned else
                      "plain pageable numpy CSR + rhs, uploaded per step (shared index "
                      "arrays once)"}


def full_policy(wl):
    """The whole sequence policy once through the public API (host inputs):
    RBiCG generation + per-cycle m = k + s + 2 recycle update on system 0,
    refresh_images + guarded RBiCGSTAB on every later system."""
    import torch
    import paper_1406_2831_b200 as P
    from paper_1406_2831_b200 import device as D
    from paper_1406_2831_b200.sequence import run_sequence
    seq = wl.seq
    mats = dict(wl.mats)

    def mat(i):
        if i not in mats:
            mats[i] = seq.matrix_fn(i)
        return mats[i]
    view = W.SequenceSpec(seq.name, seq.n, seq.k, seq.tol, seq.num_matrices,
                          seq.rhs_per_matrix, mat, seq.rhs_fn, s=seq.s,
                          max_itn=seq.max_itn, meta=seq.meta)
    try:
        D.MATRICES.clear()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = run_sequence(view, policy="first", baseline=False, api=P)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        D.MATRICES.clear()
        rec = res.recycling
        return {"seconds": round(dt, 3), "iterations": rec.total_iterations,
                "iters_per_s": rec.total_iterations / dt,
                "matvecs": rec.total_matvecs, "aux_matvecs": rec.aux_matvecs,
                "space_dims": res.space_dims,
                "iterations_per_system": [h.iterations for h in rec.histories],
                "statuses": [h.status for h in rec.histories],
                "m_basis": seq.k + seq.s + 2,
                "what": "policy 'first' over all systems through the public API "
                        "(host numpy inputs, uploads included), one run"}
    except Exception as e:   # reported, never hidden
        return {"error": f"{type(e).__name__}: {e}"}


# ---------------------------------------------------------------------------
def cpu_sample(wl, iters, steps):
    """The reference's algorithm on this host (oracle RefOps: krecycle's own
    numpy / scipy / OpenBLAS calls, bit-identical to it at a fixed thread
    count): RBiCGSTAB on the first recycled system with the same seeded
    space, ``iters`` iterations per sample.  Each sample's throughput is its
    iterations over its iteration-loop time (the history's own clock,
    solvers.py:163 -- the per-solve setup is excluded, which favours the CPU);
    the space (2k products on the CPU) is built once, untimed."""
    from oracle import krylov as O
    from oracle.ops import CsrOperand, RefOps
    ops = RefOps()
    i, kap = wl.keys[0]
    A = wl.mats[i]
    Aop = CsrOperand(A.n, A.row_ptr, A.col_idx, A.values)
    t0 = time.perf_counter()
    S = O.biorthonormalize(wl.U0, wl.Ut0, Aop, ops=ops)
    t_space = time.perf_counter() - t0
    b = wl.rhs[(i, kap)]
    loop_s, its, wall = 0.0, 0, 0.0
    for st in range(steps):
        t1 = time.perf_counter()
        _, h = O.rbicgstab(Aop, b, recycle=S, ops=ops,
                           config=O.Config(tol=wl.seq.tol, max_itn=iters, seed=1))
        wall += time.perf_counter() - t1
        its += h.iterations
        loop_s += h.seconds[-1] - h.seconds[0]
    return {"value": its / loop_s, "unit": "iters/s", "cores": os.cpu_count(),
            "kind": "port",
            "sample": f"{wl.name} system {i}: RefOps rbicgstab with the k={S.k} seeded "
                      f"space, {steps} x {iters} iterations (iteration-loop time from "
                      f"the history clock; setup excluded); numpy/scipy/OpenBLAS, "
                      f"BLAS threads={os.environ.get('OPENBLAS_NUM_THREADS', 'all')}",
            "seconds": round(loop_s, 3), "iterations": its,
            "seconds_incl_setup": round(wall, 3),
            "space_build_s": round(t_space, 2),
            "_resid": [float(v) for v in h.resid], "_matvecs": [int(v) for v in h.matvecs]}


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        if rank != 0:
            return
        wl = Workload(args.config, args.systems)
        cpu_sample(wl, 1, max(args.warmup, 0)) if args.warmup else None
        samp = cpu_sample(wl, args.cpu_iters, max(args.steps, 1))
        samp.pop("_resid", None)
        samp.pop("_matvecs", None)
        v = samp["value"]
        print(json.dumps({
            "impl": "reference", "metric": METRIC, "value": v, "unit": "iters/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * samp["seconds"] / max(args.steps, 1),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "config": wl.config(1),
            "cpu_baseline": samp,
            "e2e": {"value": v, "unit": "iters/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}), flush=True)
        return

    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
        dist.init_process_group("nccl")
    wl = Workload(args.config, args.systems)
    res = gpu_arm(args, wl, rank, world)
    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            cpu = cpu_sample(wl, args.cpu_iters, 2)
        parity = None
        if cpu is not None:
            # the CPU arm's residual history (the reference's algorithm, its
            # own space built on the CPU from the same seeded basis) against
            # the GPU arm's history of the same system over the common prefix
            c_res, c_mv = cpu.pop("_resid"), cpu.pop("_matvecs")
            g_res = res.get("histories_head", {}).get("0", [])
            m = min(len(c_res), len(g_res))
            if m:
                parity = {"system": wl.keys[0][0], "residuals_compared": m,
                          "max_rel_history_diff": max(abs(a - b) / abs(b) for a, b in
                                                      zip(g_res[:m], c_res[:m])),
                          "cpu_matvecs": c_mv[:m],
                          "gpu_matvecs": res.get("matvecs_head", [])[:m],
                          "note": "GPU arm vs CPU arm (oracle RefOps = krecycle's own calls) "
                                  "of this run; each arm biorthonormalizes the same seeded "
                                  "random basis pair itself, so the spaces already differ in "
                                  "the last bits (the full-size parity tests use low-"
                                  "amplification spaces and the reference's own envelope)"}
        line = {"metric": METRIC, "value": res["iters_all"] / res["t_total"],
                "unit": "iters/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": 1e3 * res["t_total"] / args.steps,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "f64", "data": "synthetic", "config": wl.config(world),
                "iterations_per_step": res["iters"] / args.steps,
                "gpu_launches": res["launches"], "clocks": res["clocks"],
                "e2e": res["e2e"], "roofline": res["roofline"], "cpu_baseline": cpu,
                "parity": parity}
        if not all(res.get("checks", {}).values()):
            print("bench: a timed solve did not converge to tol -- the number is not "
                  "valid", file=sys.stderr)
        for key in ("checks", "e2e_pageable", "iteration", "kernel_shares", "step_ms",
                    "iterations_per_system", "matvecs_per_system", "statuses",
                    "final_true_resid_max", "space_k_last", "baseline", "full_policy",
                    "histories_head"):
            if key in res:
                line[key] = res[key]
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
