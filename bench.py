#!/usr/bin/env python
"""Recycling-BiCGSTAB sequence benchmark on B200 (BASELINE.json metric:
"RBiCGSTAB sequence solve time & iters/s; SpMV+BLAS-1 HBM GB/s vs 8 TB/s").

One step = one pass of the sequence policy (paper_1406_2831_b200/sequence.py,
the reference's driver.py:78-180 restated without ILUTP)
over every system of a BASELINE config (default C2 = configs[1]): system 0 is
the RBiCG generation solve with a per-cycle recycle-space update, every later
system refreshes the space onto its matrix and runs RBiCGSTAB with the
driver's guard.  All arithmetic runs in libkrb.so on the GPU.

  value       sequence iterations / s, inputs resident in HBM before timing
              (device matrices + device right-hand sides through the same API)
  e2e         the same step through the public drop-in API with HOST numpy
              inputs: matrices, right-hand sides uploaded, solutions read back
  baseline    the GPU BiCGSTAB track on the same systems (matvec savings)
  synthetic   one RBiCGSTAB pass with a fixed seeded k-dimensional space (the
              reference's harvest collapses to k ~ 0 on these configs, SURVEY
              D3, so this is what exercises the projection kernels); gives
              iteration_roofline
  roofline    dominant kernel, CUDA-event timed live on the bench matrix
  cpu_baseline  the reference's algorithm (oracle RefOps restatement: numpy +
              scipy + OpenBLAS on all host threads), bounded sample

--impl reference prints the CPU reference arm only.  --gpus N > 1 (torchrun)
runs N independent replicas (the sequence is serial).
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
from paper_1406_2831_b200.sequence import run_sequence  # noqa: E402

METRIC = "RBiCGSTAB sequence iters/s (policy: RBiCG generation + refreshed RBiCGSTAB)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c2")
    ap.add_argument("--systems", type=int, default=None)
    ap.add_argument("--policy", default=None, help="first | verbatim")
    ap.add_argument("--cpu-seconds", type=float, default=60.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-synthetic", action="store_true")
    return ap.parse_args()


def peaks():
    p = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class Workload:
    """The config's sequence with every matrix and rhs materialised on the
    host once (outside any timed region)."""

    def __init__(self, name, systems=None, policy=None):
        self.name = name
        self.seq = W.make_sequence(name)
        self.policy = policy or ("verbatim" if name == "c3" else "first")
        self.nsys = self.seq.num_systems if systems is None else min(systems, self.seq.num_systems)
        mats = {}
        rhs = {}
        g = 0
        for i in range(self.seq.num_matrices):
            for kap in range(self.seq.rhs_per_matrix):
                if g < self.nsys:
                    if i not in mats:
                        mats[i] = self.seq.matrix_fn(i)
                    rhs[(i, kap)] = self.seq.rhs(i, kap)
                g += 1
        self.mats, self.rhs = mats, rhs
        A0 = mats[0]
        self.n, self.nnz, self.k = A0.n, A0.nnz, self.seq.k
        seq = self.seq
        # a sequence view that serves the materialised arrays
        self.view = W.SequenceSpec(seq.name, seq.n, seq.k, seq.tol, seq.num_matrices,
                                   seq.rhs_per_matrix, lambda i: mats[i],
                                   lambda i, kap: rhs[(i, kap)], s=seq.s,
                                   max_itn=seq.max_itn, meta=seq.meta)

    def pinned_view(self):
        """The same sequence served from page-locked host copies (made once,
        outside any timed region): the e2e arm's inputs live in pinned host
        memory, as a production caller would keep them, so each step's
        uploads are plain DMA."""
        from paper_1406_2831_b200.device import pinned_copy
        pm = {i: W.CSR(A.n, pinned_copy(A.row_ptr), pinned_copy(A.col_idx),
                       pinned_copy(A.values)) for i, A in self.mats.items()}
        pr = {key: pinned_copy(b) for key, b in self.rhs.items()}
        seq = self.seq
        return W.SequenceSpec(seq.name, seq.n, seq.k, seq.tol, seq.num_matrices,
                              seq.rhs_per_matrix, lambda i: pm[i],
                              lambda i, kap: pr[(i, kap)], s=seq.s,
                              max_itn=seq.max_itn, meta=seq.meta)


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
def device_api(wl):
    """The package API with matrices and right-hand sides pre-resident in HBM
    (DeviceMatrix handles, CUDA tensors): the policy code is unchanged."""
    import paper_1406_2831_b200 as P
    from paper_1406_2831_b200 import device as D
    dmats = {i: D.DeviceMatrix(A.n, A.row_ptr, A.col_idx, A.values)
             for i, A in wl.mats.items()}
    drhs = {key: D.to_device(b) for key, b in wl.rhs.items()}
    by_id = {id(A): dmats[i] for i, A in wl.mats.items()}
    seq = wl.seq
    view = W.SequenceSpec(seq.name, seq.n, seq.k, seq.tol, seq.num_matrices,
                          seq.rhs_per_matrix, lambda i: wl.mats[i],
                          lambda i, kap: drhs[(i, kap)], s=seq.s,
                          max_itn=seq.max_itn, meta=seq.meta)
    api = types.SimpleNamespace(**{k: getattr(P, k) for k in P.__all__})
    api.SparseMatrix = types.SimpleNamespace(from_csr=lambda A: _DevOp(by_id[id(A)]))
    return api, view, dmats, drhs


class _DevOp:
    """A DeviceMatrix with the attributes the policy reads."""

    def __init__(self, M):
        self._device = M
        self.nrows = self.ncols = M.n
        self.shape = (M.n, M.n)
        self.dtype = np.float64


def policy_step(wl, api, seq_view, baseline=False):
    res = run_sequence(seq_view, policy=wl.policy, baseline=baseline, api=api,
                       systems=wl.nsys)
    it = res.recycling.total_iterations
    return res, it


def gpu_arm(args, wl, rank, world):
    import torch
    import paper_1406_2831_b200 as P
    from paper_1406_2831_b200 import _lib, device as D

    torch.cuda.set_device(rank % max(torch.cuda.device_count(), 1))
    api, dview, dmats, drhs = device_api(wl)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device="cuda")  # 512 MB > L2
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    for _ in range(args.warmup):
        policy_step(wl, api, dview)
    torch.cuda.synchronize()

    clocks = Clocks(torch.cuda.current_device())
    clocks.start()
    # let nvidia-smi finish initialising (its start-up RM calls stall CUDA API
    # calls of this host-synchronising workload); it keeps sampling throughout
    clocks.wait_first_sample()
    times, its, last = [], 0, None
    l0 = _lib.launch_count()
    for _ in range(args.steps):
        flush.fill_(1.0)
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        last, it = policy_step(wl, api, dview)
        e1.record()
        torch.cuda.synchronize()
        barrier()
        times.append(e0.elapsed_time(e1) / 1e3)
        its += it
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

    out = {"t_total": t_total, "iters": its, "iters_all": its_all,
           "step_ms": [round(1e3 * t, 3) for t in times],
           "launches": launches, "clocks": clk,
           "space_dims": last.space_dims,
           "rec_matvecs": last.recycling.total_matvecs,
           "rec_aux_matvecs": last.recycling.aux_matvecs,
           "statuses": [h.status for h in last.recycling.histories]}

    # GPU BiCGSTAB baseline track on the same systems (device-resident)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    b_it = b_mv = 0
    for idx, key in enumerate(sorted(drhs)):
        cfg = P.SolverConfig(tol=wl.seq.tol, max_itn=wl.seq.max_itn, seed=idx)
        _, h = P.bicgstab_solve(dmats[key[0]], drhs[key], config=cfg)
        if h.status != "converged":
            _, h2 = P.bicgstab_solve(dmats[key[0]], drhs[key],
                                     config=P.SolverConfig(tol=wl.seq.tol,
                                                           max_itn=wl.seq.max_itn,
                                                           seed=idx + 104729))
            b_it += h.iterations
            b_mv += h.total_matvecs
            h = h2
        b_it += h.iterations
        b_mv += h.total_matvecs
    e1.record()
    torch.cuda.synchronize()
    tb = e0.elapsed_time(e1) / 1e3
    out["baseline"] = {"iters": b_it, "matvecs": b_mv, "seconds": tb,
                       "iters_per_s": b_it / tb,
                       "matvec_savings": 1.0 - out["rec_matvecs"] / b_mv if b_mv else None}

    if not args.no_e2e:
        host_api = P
        pview = wl.pinned_view()

        def host_step():
            D.MATRICES.clear()
            return run_sequence(pview, policy=wl.policy, baseline=False, api=host_api,
                                systems=wl.nsys)

        for _ in range(max(args.warmup, 1)):
            host_step()
        torch.cuda.synchronize()
        e_times, e_its = [], 0
        for _ in range(args.steps):
            flush.fill_(1.0)
            barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r = host_step()
            torch.cuda.synchronize()
            e_times.append(time.perf_counter() - t0)
            e_its += r.recycling.total_iterations
        e_total = sum(e_times)
        if world > 1:
            import torch.distributed as dist
            tt = torch.tensor([e_total], dtype=torch.float64, device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e_total = float(tt.item())
        h2d = sum(A.row_ptr.nbytes + A.col_idx.nbytes + A.values.nbytes
                  for A in wl.mats.values()) + sum(b.nbytes for b in wl.rhs.values())
        d2h = sum(8 * wl.n + 24 * (wl.seq.max_itn + 1) for _ in wl.rhs)
        out["e2e"] = {"value": e_its * world / e_total, "unit": "iters/s",
                      "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                      "seq_solve_s": e_total / args.steps}
    else:
        out["e2e"] = None

    if not args.no_synthetic:
        out.update(synthetic_pass(wl, dmats, drhs,
                                   max(last.space_dims) if last.space_dims else 0))
    return out


def _solve_pass(wl, dmats, drhs, fixed_space):
    """Every system of the sequence solved once more (best of two) with either
    no recycle space (k = 0: the shape the policy's solves take when the
    harvest collapses) or a fixed seeded k-space refreshed per
    matrix.  Returns (iterations, seconds, k per system, driver)."""
    import torch
    import paper_1406_2831_b200 as P
    from paper_1406_2831_b200 import solvers as S
    space = None
    if fixed_space:
        r = np.random.default_rng(12345)
        U = r.standard_normal((wl.n, wl.k))
        Ut = r.standard_normal((wl.n, wl.k))
    its, t_solve, ks = 0, 0.0, []
    for idx, key in enumerate(sorted(drhs)):
        M = dmats[key[0]]
        if fixed_space:
            space = P.biorthonormalize(U, Ut, M) if space is None else P.refresh_images(space, M)
        ks.append(space.k if space is not None else 0)
        best = None
        for _rep in range(2):   # best of two (the first also warms this shape)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            _, h = S.solve_device(M, drhs[key], None, space,
                                  P.SolverConfig(tol=wl.seq.tol, max_itn=wl.seq.max_itn,
                                                 seed=idx))
            e1.record()
            torch.cuda.synchronize()
            dt = e0.elapsed_time(e1) / 1e3
            best = dt if best is None else min(best, dt)
        t_solve += best
        its += h.iterations
    return its, t_solve, ks, S.LAST_SOLVE.get("driver"), space


def _traffic(wl, kernel, its, nsolves):
    tp = os.path.join(REPO, "profiles", "traffic.json")
    if not os.path.exists(tp):
        return None
    for tj in json.load(open(tp)).get(wl.name, []):
        if kernel.startswith(tj["kernel"]):
            if "bytes_per_iteration" in tj:
                return int(tj["bytes_per_iteration"] * its / max(nsolves, 1))
            return int(tj["bytes_per_launch"])
    return None


def synthetic_pass(wl, dmats, drhs, step_k):
    """Roofline of the dominant kernel of the measured step plus a fixed
    k-space pass (the reference's harvest collapses to k = 0 on C2, so the
    fixed space is what exercises the projections) and live kernel timing.

    With n <= PERSISTENT_MAX_N every solve is ONE persistent kernel launch
    (k = 0: k_persist0, persist0.cu; k > 0: k_persist2, persist.cu), so the
    kernel's algorithmic bytes per launch = B_it(k) x iterations per solve and
    its launch duration = the solve's CUDA-event time (setup kernels
    included, so the fraction is conservative)."""
    import torch
    from paper_1406_2831_b200 import recycling as R
    from paper_1406_2831_b200.solvers import _auto_mode
    peak, src = peaks()
    persistent = _auto_mode(wl.n) == 2

    def roofline_of(its, t_solve, ks, k):
        B_it = W.bytes_per_iteration(wl.n, wl.nnz, k)
        ach = B_it * its / t_solve / 1e9
        if k == 0:
            kern = "k_persist0 (fused persistent BiCGSTAB, k = 0, one solve per launch)"
        else:
            kern = "k_persist2 (fused persistent RBiCGSTAB, one solve per launch)"
        return B_it, {"bound": "hbm", "kernel": kern, "k": k,
                      "achieved": round(ach, 1), "peak": peak, "peak_source": src,
                      "unit": "GB/s", "frac": round(ach / peak, 4),
                      "traffic": _traffic(wl, kern, its, len(ks)),
                      "bytes_per_launch": B_it * its / max(len(ks), 1),
                      "launch_us": round(1e6 * t_solve / max(len(ks), 1), 2),
                      "iterations": its, "seconds": t_solve,
                      "us_per_iteration": round(1e6 * t_solve / max(its, 1), 2)}

    out = {}
    its0, t0, ks0, drv0, _ = _solve_pass(wl, dmats, drhs, fixed_space=False)
    B0, rf0 = roofline_of(its0, t0, ks0, 0)
    itsk, tk, ksk, drvk, space = _solve_pass(wl, dmats, drhs, fixed_space=True)
    kmean = int(round(float(np.mean(ksk)))) if ksk else 0
    Bk, rfk = roofline_of(itsk, tk, ksk, kmean)
    out["synthetic"] = {"iterations": itsk, "seconds": tk, "k_per_system": ksk,
                        "driver": drvk, "iters_per_s": itsk / tk,
                        "us_per_iteration": round(1e6 * tk / max(itsk, 1), 2)}
    out["iteration_roofline"] = {"bytes_per_iteration": Bk, "k": kmean,
                                 "achieved": rfk["achieved"], "unit": "GB/s",
                                 "peak": peak, "frac": rfk["frac"]}
    out["iteration_roofline_k0"] = {"bytes_per_iteration": B0, "k": 0, "driver": drv0,
                                    "achieved": rf0["achieved"], "unit": "GB/s",
                                    "peak": peak, "frac": rf0["frac"],
                                    "us_per_iteration": rf0["us_per_iteration"]}

    M = dmats[0]
    x = torch.randn(wl.n, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    Cb = space.device("C") if space is not None and space.k else None
    kk = Cb.shape[0] if Cb is not None else 0
    zeta = torch.randn(max(kk, 1), dtype=torch.float64, device="cuda")

    def timeit(fn, reps=30):
        for _ in range(3):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / 1e3 / reps

    kern = {"spmv": (W.spmv_bytes(wl.n, M.nnz), timeit(lambda: M.spmv(x, y)))}
    if kk:
        kern["proj_dot"] = (8 * wl.n * kk + 8 * wl.n, timeit(lambda: R.tdot(Cb, x, zeta)))
        kern["proj_update"] = (8 * wl.n * kk + 16 * wl.n,
                               timeit(lambda: R.gemv(Cb, zeta, base=x, sign=-1, out=y)))
    out["kernels"] = {k: {"bytes": v[0], "us": round(v[1] * 1e6, 2),
                          "GBps": round(v[0] / v[1] / 1e9, 1)} for k, v in kern.items()}
    if persistent:
        # the step's own shape: its solves run at k = step_k
        main, other = (rf0, rfk) if step_k == 0 else (rfk, rf0)
        out["roofline"] = main
        out["roofline_secondary"] = other
    else:
        share = {k: v[1] for k, v in kern.items()}
        dom = max(share, key=share.get)
        b, t = kern[dom]
        ach = b / t / 1e9
        out["roofline"] = {"bound": "hbm", "kernel": dom, "achieved": round(ach, 1),
                           "peak": peak, "peak_source": src, "unit": "GB/s",
                           "frac": round(ach / peak, 4),
                           "traffic": _traffic(wl, dom, 1, 1),
                           "bytes_per_launch": b, "launch_us": round(t * 1e6, 2)}
    return out


# ---------------------------------------------------------------------------
def oracle_api():
    """The reference's algorithm on the CPU (oracle RefOps: the reference's own
    numpy/scipy/OpenBLAS calls) behind the package's API names."""
    import paper_1406_2831_b200 as P
    from oracle import krylov as O
    from oracle.ops import CsrOperand, RefOps
    ops = RefOps()
    cache = {}

    def from_csr(A):
        if id(A) not in cache:
            cache[id(A)] = (A, CsrOperand.of(A))
        return cache[id(A)][1]

    return types.SimpleNamespace(
        SparseMatrix=types.SimpleNamespace(from_csr=from_csr),
        CountingOperator=P.CountingOperator, SolverConfig=P.SolverConfig,
        rbicg_solve=lambda A, b, **kw: O.rbicg(A, b, ops=ops, **kw),
        rbicgstab_solve=lambda A, b, **kw: O.rbicgstab(A, b, ops=ops, **kw),
        bicgstab_solve=lambda A, b, **kw: O.bicgstab(A, b, ops=ops, **kw),
        update_recycle_space=lambda A, c, p, k, **kw: O.update_recycle_space(
            A, c, p, k, ops=ops, **kw),
        refresh_images=lambda S, A, **kw: O.refresh_images(S, A, ops=ops, **kw))


def cpu_sample(wl, budget_s):
    """Run the policy on the CPU over the first systems of the sequence until
    ~budget_s of work (always at least the generation solve)."""
    api = oracle_api()
    t0 = time.perf_counter()
    res = run_sequence(wl.view, policy=wl.policy, baseline=False, api=api,
                       systems=wl.nsys, max_seconds=budget_s)
    t = time.perf_counter() - t0
    its, done = res.recycling.total_iterations, len(res.recycling.histories)
    return {"value": its / t, "unit": "iters/s", "cores": os.cpu_count(),
            "kind": "port",
            "sample": f"{wl.name}: policy '{wl.policy}' over systems 0..{done - 1} "
                      f"({done}/{wl.nsys}; rbicg generation + refreshed rbicgstab), "
                      f"numpy/scipy/OpenBLAS, BLAS threads="
                      f"{os.environ.get('OPENBLAS_NUM_THREADS', 'all')}",
            "seconds": round(t, 3), "iterations": its}


def config_block(wl, world):
    return {"workload": f"{wl.name}: {wl.seq.meta}", "n": wl.n, "nnz": wl.nnz,
            "k": wl.k, "systems": wl.nsys, "tol": wl.seq.tol, "policy": wl.policy,
            "l2": "512 MB buffer written between timed steps",
            "e2e_inputs": "numpy CSR + rhs in page-locked host memory, uploaded every step",
            "parallelism": f"replicas{world}" if world > 1 else "single"}


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        if rank != 0:
            return
        wl = Workload(args.config, args.systems, args.policy)
        t_all, it_all, samp = 0.0, 0, None
        for _ in range(max(args.steps, 1)):
            samp = cpu_sample(wl, args.cpu_seconds / max(args.steps, 1))
            t_all += samp["seconds"]
            it_all += samp["iterations"]
        v = it_all / t_all
        samp["value"] = v
        print(json.dumps({
            "impl": "reference", "metric": METRIC, "value": v, "unit": "iters/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * t_all / max(args.steps, 1), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_block(wl, 1), "cpu_baseline": samp,
            "e2e": {"value": v, "unit": "iters/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}), flush=True)
        return

    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
        dist.init_process_group("nccl")
    wl = Workload(args.config, args.systems, args.policy)
    res = gpu_arm(args, wl, rank, world)
    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            cpu = cpu_sample(wl, args.cpu_seconds)
        line = {"metric": METRIC, "value": res["iters_all"] / res["t_total"],
                "unit": "iters/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": 1e3 * res["t_total"] / args.steps,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "f64", "data": "synthetic", "config": config_block(wl, world),
                "seq_solve_s": res["t_total"] / args.steps,
                "iterations_per_step": res["iters"] / args.steps,
                "space_dims": res["space_dims"], "statuses": res["statuses"],
                "recycling_matvecs": res["rec_matvecs"],
                "recycling_aux_matvecs": res["rec_aux_matvecs"],
                "baseline": res["baseline"],
                "step_ms": res["step_ms"],
                "gpu_launches": res["launches"], "clocks": res["clocks"],
                "e2e": res["e2e"]}
        for key in ("roofline", "roofline_secondary", "iteration_roofline",
                    "iteration_roofline_k0", "kernels", "synthetic"):
            if key in res:
                line[key] = res[key]
        line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
