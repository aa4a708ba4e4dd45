#!/usr/bin/env python
"""RBiCGSTAB sequence-solve benchmark on B200 (BASELINE.json metric:
"RBiCGSTAB sequence solve time & iters/s; SpMV+BLAS-1 HBM GB/s vs 8 TB/s").

One step = one pass over the whole sequence of a BASELINE config (default C2,
configs[1]): for every system A_j x = b_j the recycle space is refreshed onto
A_j (biorthonormalize: 2k products + Gram + host SVD + rotations, all device
kernels) and rbicgstab_solve runs to tol.  The space is a fixed seeded random
k-dimensional basis pair (the reference's own harvest collapses to k = 0 on
this config, so a synthetic space is what exercises the
projection kernels; labelled in config.space).

  value   iterations/s with every input resident in HBM (device API)
  e2e     same metric through the public drop-in API with HOST numpy inputs:
          matrices, rhs and bases uploaded, solutions downloaded, every step
  roofline / iteration_roofline   HBM roofline of the dominant kernel and of
          the whole iteration (SURVEY.md §8(d) algorithmic bytes)
  cpu_baseline   the reference's algorithm (oracle RefOps restatement: numpy +
          scipy + OpenBLAS, all host threads) on a bounded sample

--impl reference runs only the CPU arm.  --gpus N > 1 (torchrun) runs N
independent replicas (the sequence is serial).
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

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

from paper_1406_2831_b200 import workloads as W  # noqa: E402


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c2")
    ap.add_argument("--k", type=int, default=None)
    ap.add_argument("--systems", type=int, default=None,
                    help="limit the number of systems per step")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def peaks():
    p = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


# ---------------------------------------------------------------------------
# workload
# ---------------------------------------------------------------------------

class Workload:
    def __init__(self, name, k=None, systems=None):
        self.seq = W.make_sequence(name)
        self.name = name
        self.k = self.seq.k if k is None else k
        nsys = self.seq.num_systems if systems is None else min(systems, self.seq.num_systems)
        self.systems = []   # (matrix index, rhs index)
        for i in range(self.seq.num_matrices):
            for kap in range(self.seq.rhs_per_matrix):
                if len(self.systems) < nsys:
                    self.systems.append((i, kap))
        self.mats = {}
        for i, _ in self.systems:
            if i not in self.mats:
                self.mats[i] = self.seq.matrix_fn(i)
        self.rhs = {s: self.seq.rhs(*s) for s in self.systems}
        r = np.random.default_rng(12345)
        A0 = self.mats[self.systems[0][0]]
        self.U = r.standard_normal((A0.n, self.k))
        self.Ut = r.standard_normal((A0.n, self.k))
        self.n = A0.n
        self.nnz = A0.nnz

    def cfg(self, idx):
        return dict(tol=self.seq.tol, max_itn=self.seq.max_itn, seed=idx)


# ---------------------------------------------------------------------------
# clocks sampler
# ---------------------------------------------------------------------------

class Clocks:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

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
# GPU arm
# ---------------------------------------------------------------------------

def gpu_arm(args, wl: Workload, rank: int, world: int):
    import torch
    import paper_1406_2831_b200 as P
    from paper_1406_2831_b200 import _lib, device as D, solvers as S
    from paper_1406_2831_b200.recycling import biorthonormalize, refresh_images

    torch.cuda.set_device(rank % max(torch.cuda.device_count(), 1))
    dev_mats = {i: D.DeviceMatrix(A.n, A.row_ptr, A.col_idx, A.values)
                for i, A in wl.mats.items()}
    dev_b = {s: D.to_device(b) for s, b in wl.rhs.items()}
    U_d = D.to_device(np.ascontiguousarray(wl.U.T)).reshape(wl.k, wl.n)
    Ut_d = D.to_device(np.ascontiguousarray(wl.Ut.T)).reshape(wl.k, wl.n)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device="cuda")  # 512 MB > L2
    torch.cuda.synchronize()

    def device_step():
        iters = mvs = 0
        ks = []
        space, cur = None, None
        for idx, (i, kap) in enumerate(wl.systems):
            M = dev_mats[i]
            if space is None:
                space = biorthonormalize(U_d, Ut_d, M)
            elif i != cur:
                space = refresh_images(space, M)     # driver.py:112-113
            cur = i
            ks.append(space.k)
            cfg = P.SolverConfig(**wl.cfg(idx))
            x, h = S.solve_device(M, dev_b[(i, kap)], None, space, cfg, "rbicgstab")
            iters += h.iterations
            mvs += h.total_matvecs
            if h.status != "converged":
                # driver.py:150-156 guard: redo unrecycled with a fresh seed
                x, h = S.solve_device(M, dev_b[(i, kap)], None, None,
                                      P.SolverConfig(**wl.cfg(idx + 104729)), "rbicgstab")
                iters += h.iterations
                mvs += h.total_matvecs
                if h.status != "converged":
                    raise RuntimeError(f"system {idx}: {h.status}")
        return iters, mvs, ks

    def host_step():
        D.MATRICES.clear()
        iters = 0
        h2d = d2h = 0
        space, cur, Ah = None, None, None
        for idx, (i, kap) in enumerate(wl.systems):
            A = wl.mats[i]
            if i != cur:
                Ah = P.SparseMatrix.from_csr(A)
                h2d += A.row_ptr.nbytes + A.col_idx.nbytes + A.values.nbytes
            b = wl.rhs[(i, kap)]
            if space is None:
                space = biorthonormalize(wl.U, wl.Ut, Ah)
                h2d += wl.U.nbytes + wl.Ut.nbytes
            elif i != cur:
                space = refresh_images(space, Ah)
            cur = i
            x, h = P.rbicgstab_solve(Ah, b, recycle=space,
                                     config=P.SolverConfig(**wl.cfg(idx)))
            iters += h.iterations
            if h.status != "converged":
                x, h = P.rbicgstab_solve(Ah, b, recycle=None,
                                         config=P.SolverConfig(**wl.cfg(idx + 104729)))
                iters += h.iterations
            h2d += b.nbytes
            d2h += x.nbytes + 24 * len(h.resid)
        return iters, h2d, d2h

    for _ in range(args.warmup):
        device_step()
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    clocks = Clocks(torch.cuda.current_device())
    clocks.start()
    times, tot_it, tot_mv = [], 0, 0
    l0 = _lib.launch_count()
    ks = []
    for _ in range(args.steps):
        flush.fill_(1.0)
        barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        it, mv, ks = device_step()
        e1.record()
        torch.cuda.synchronize()
        barrier()
        times.append(e0.elapsed_time(e1) / 1e3)
        tot_it += it
        tot_mv += mv
    launches = _lib.launch_count() - l0
    clk = clocks.stop()
    t_total = sum(times)
    if world > 1:
        import torch.distributed as dist
        tt = torch.tensor([t_total], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_total = float(tt.item())
        ii = torch.tensor([tot_it], dtype=torch.float64, device="cuda")
        dist.all_reduce(ii, op=dist.ReduceOp.SUM)
        tot_it_all = float(ii.item())
    else:
        tot_it_all = tot_it

    # e2e through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        host_step()   # warm (graphs/allocator)
        torch.cuda.synchronize()
        e_times, e_it, h2d, d2h = [], 0, 0, 0
        for _ in range(args.steps):
            flush.fill_(1.0)
            barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            it, hb, db = host_step()
            e1.record()
            torch.cuda.synchronize()
            wall = time.perf_counter() - t0
            e_times.append(max(wall, e0.elapsed_time(e1) / 1e3))
            e_it += it
            h2d, d2h = hb, db
        e_total = sum(e_times)
        if world > 1:
            import torch.distributed as dist
            tt = torch.tensor([e_total], dtype=torch.float64, device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e_total = float(tt.item())
        e2e = {"value": e_it * world / e_total, "unit": "iters/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "seq_solve_s": e_total / args.steps}

    roof = kernel_roofline(wl, dev_mats, U_d, tot_it, t_total)
    return {"t_total": t_total, "iters": tot_it, "iters_all": tot_it_all,
            "matvecs": tot_mv, "launches": launches, "clocks": clk, "e2e": e2e,
            "k_used": ks, **roof}


def kernel_roofline(wl, dev_mats, U_d, tot_it, t_total):
    """Live CUDA-event timing of the SpMV and the projection kernels on the
    bench matrix, and the whole-iteration algorithmic bandwidth."""
    import torch
    from paper_1406_2831_b200 import recycling as R
    peak, src = peaks()
    M = dev_mats[wl.systems[0][0]]
    x = torch.randn(wl.n, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    st = torch.cuda.current_stream()

    def timeit(fn, reps=30):
        for _ in range(3):
            fn()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(reps):
            fn()
        e1.record(st)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / 1e3 / reps

    t_spmv = timeit(lambda: M.spmv(x, y))
    b_spmv = W.spmv_bytes(wl.n, M.nnz)
    out = torch.empty(wl.k, dtype=torch.float64, device="cuda")
    t_tdot = timeit(lambda: R.tdot(U_d, x, out))
    b_tdot = 8 * wl.n * wl.k + 8 * wl.n
    t_gemv = timeit(lambda: R.gemv(U_d, out, base=x, sign=-1, out=y))
    b_gemv = 8 * wl.n * wl.k + 16 * wl.n
    kern = {
        "spmv": (b_spmv, t_spmv),
        "proj_tdot": (b_tdot, t_tdot),
        "proj_update": (b_gemv, t_gemv),
    }
    # dominant by time share per iteration: 2 SpMV, 2 tdot, 2 updates
    share = {k: 2 * v[1] for k, v in kern.items()}
    dom = max(share, key=share.get)
    b, t = kern[dom]
    ach = b / t / 1e9
    B_it = W.bytes_per_iteration(wl.n, wl.nnz, wl.k)
    it_ach = B_it * tot_it / t_total / 1e9
    return {
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": round(ach, 1),
                     "peak": peak, "peak_source": src, "unit": "GB/s",
                     "frac": round(ach / peak, 4), "traffic": None,
                     "bytes_per_launch": b, "launch_us": round(t * 1e6, 2)},
        "kernels": {k: {"bytes": v[0], "us": round(v[1] * 1e6, 2),
                        "GBps": round(v[0] / v[1] / 1e9, 1)} for k, v in kern.items()},
        "iteration_roofline": {"bytes_per_iteration": B_it,
                               "achieved": round(it_ach, 1), "unit": "GB/s",
                               "frac": round(it_ach / peak, 4),
                               "us_per_iteration": round(t_total / max(tot_it, 1) * 1e6, 2)},
    }


# ---------------------------------------------------------------------------
# CPU arm (the reference's algorithm: oracle RefOps restatement)
# ---------------------------------------------------------------------------

def cpu_sample(wl: Workload, budget_s: float):
    from oracle import krylov as O
    from oracle.ops import RefOps
    from oracle.ops import CsrOperand
    ops = RefOps()
    # one operator object per matrix, as the reference keeps one SparseMatrix
    # (and its cached transpose) per matrix of the sequence
    opers = {i: CsrOperand.of(A) for i, A in wl.mats.items()}
    t0 = time.perf_counter()
    iters = 0
    done = 0
    S, cur = None, None
    for idx, (i, kap) in enumerate(wl.systems):
        A = opers[i]
        if S is None:
            S = O.biorthonormalize(wl.U, wl.Ut, A, ops=ops)
        elif i != cur:
            S = O.refresh_images(S, A, ops=ops)
        cur = i
        x, h = O.rbicgstab(A, wl.rhs[(i, kap)], recycle=S,
                           config=O.Config(**wl.cfg(idx)), ops=ops)
        iters += h.iterations
        if h.status != "converged":
            x, h = O.rbicgstab(A, wl.rhs[(i, kap)], recycle=None,
                               config=O.Config(**wl.cfg(idx + 104729)), ops=ops)
            iters += h.iterations
        done += 1
        if time.perf_counter() - t0 >= budget_s:
            break
    dt = time.perf_counter() - t0
    return {"value": iters / dt, "unit": "iters/s", "cores": os.cpu_count(),
            "kind": "port",
            "sample": f"systems 0..{done - 1} of {wl.name} ({done}/{len(wl.systems)}): "
                      f"biorthonormalize + rbicgstab_solve, k={wl.k}, numpy/scipy/OpenBLAS "
                      f"({os.environ.get('OPENBLAS_NUM_THREADS', 'all')} BLAS threads)",
            "seconds": round(dt, 3), "iterations": iters}


def config_block(args, wl, world):
    return {"workload": f"{wl.name}: {wl.seq.meta}", "n": wl.n, "nnz": wl.nnz,
            "k": wl.k, "systems": len(wl.systems), "tol": wl.seq.tol,
            "space": "synthetic seeded random basis pair: biorthonormalize on system 0, "
                     "refresh_images (2k products, cond_tol 1e-3) at every matrix change",
            "l2": "512 MB buffer written between timed steps",
            "parallelism": f"replicas{world}" if world > 1 else "single"}


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        if rank != 0:
            return
        wl = Workload(args.config, args.k, args.systems)
        vals = []
        for _ in range(args.warmup):
            pass   # CPU path has no JIT / allocator warm-up to amortise
        t_all, it_all = 0.0, 0
        samp = None
        for _ in range(max(args.steps, 1)):
            samp = cpu_sample(wl, args.cpu_seconds / max(args.steps, 1))
            vals.append(samp["value"])
            t_all += samp["seconds"]
            it_all += samp["iterations"]
        v = it_all / t_all
        samp["value"] = v
        line = {"impl": "reference", "metric": "RBiCGSTAB sequence iters/s",
                "value": v, "unit": "iters/s", "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": 1e3 * t_all / max(args.steps, 1),
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "f64", "data": "synthetic",
                "config": config_block(args, wl, 1), "cpu_baseline": samp,
                "e2e": {"value": v, "unit": "iters/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
        dist.init_process_group("nccl")
    wl = Workload(args.config, args.k, args.systems)
    res = gpu_arm(args, wl, rank, world)
    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            cpu = cpu_sample(wl, args.cpu_seconds)
        v = res["iters_all"] / res["t_total"]
        line = {"metric": "RBiCGSTAB sequence iters/s", "value": v, "unit": "iters/s",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": 1e3 * res["t_total"] / args.steps,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "f64", "data": "synthetic",
                "config": config_block(args, wl, world),
                "seq_solve_s": res["t_total"] / args.steps,
                "iterations_per_step": res["iters"] / args.steps,
                "matvecs_per_step": res["matvecs"] / args.steps,
                "k_per_system": res["k_used"],
                "gpu_launches": res["launches"],
                "clocks": res["clocks"], "e2e": res["e2e"],
                "roofline": res["roofline"], "kernels": res["kernels"],
                "iteration_roofline": res["iteration_roofline"],
                "cpu_baseline": cpu}
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
