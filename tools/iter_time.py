"""Per-iteration time of the device RBiCGSTAB (graph path) on a BASELINE
config with a fixed seeded k-space: us/iteration and algorithmic GB/s
(SURVEY.md §8(d) bytes).   python tools/iter_time.py --config c2 c5 ..."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402


def run(name, k=None, reps=3, max_itn=None, fmt=0, system=0):
    import torch
    import paper_1406_2831_b200 as P
    from paper_1406_2831_b200 import device as D, solvers as S, workloads as W
    seq = W.make_sequence(name)
    A = seq.matrix(system)
    k = seq.k if k is None else k
    M = D.DeviceMatrix(A.n, A.row_ptr, A.col_idx, A.values, fmt=fmt)
    r = np.random.default_rng(12345)
    space = None
    if k:
        space = P.biorthonormalize(r.standard_normal((A.n, k)),
                                   r.standard_normal((A.n, k)), M)
    b = D.to_device(seq.rhs(0, 0))
    cfg = P.SolverConfig(tol=seq.tol, max_itn=max_itn or seq.max_itn, seed=0)
    S.solve_device(M, b, None, space, cfg)
    best, h = None, None
    from paper_1406_2831_b200 import _lib
    kt = torch.zeros(384, dtype=torch.int64, device="cuda")
    for rep in range(reps + 1):
        # the last rep with the live per-kernel timing on (kernel_us); the
        # iteration time is the best of the reps without it
        _lib.PY_TUNING["kernel_times"] = kt if rep == reps else None
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        _, h = S.solve_device(M, b, None, space, cfg)
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 1e3
        if rep == reps:
            t_kt = t
            continue
        best = t if best is None else min(best, t)
    _lib.PY_TUNING["kernel_times"] = None
    ktn = kt.cpu().numpy()
    names = ["P", "M1", "Z1", "Q", "S", "M2", "Z2", "T", "X"]
    kern_us = {nm: round(ktn[4 * i + 1] / max(ktn[4 * i + 2], 1) / 1e3, 1)
               for i, nm in enumerate(names) if ktn[4 * i + 2]}
    kk = space.k if space is not None else 0
    its = max(h.iterations, 1)
    B = W.bytes_per_iteration(A.n, A.nnz, kk)
    return {"config": name, "system": system, "n": A.n, "nnz": A.nnz, "k": kk, "format": M.format,
            "iterations": h.iterations, "status": h.status,
            "solve_ms": round(best * 1e3, 3), "us_per_it": round(best / its * 1e6, 2),
            "GBps_alg": round(B * its / best / 1e9, 1), "kernel_us": kern_us,
            "us_per_it_with_kernel_timing": round(t_kt / its * 1e6, 2)}


def phase_breakdown(name, k=None):
    """Per-phase device time inside the persistent kernel (_lib.tuning(phase_prof=True)):
    median us per phase over the iterations of one solve."""
    import paper_1406_2831_b200 as P
    from paper_1406_2831_b200 import device as D, solvers as S, workloads as W
    seq = W.make_sequence(name)
    A = seq.matrix(0)
    k = seq.k if k is None else k
    M = D.DeviceMatrix(A.n, A.row_ptr, A.col_idx, A.values)
    r = np.random.default_rng(12345)
    space = P.biorthonormalize(r.standard_normal((A.n, k)), r.standard_normal((A.n, k)), M) if k else None
    b = D.to_device(seq.rhs(0, 0))
    from paper_1406_2831_b200 import _lib
    with _lib.tuning(phase_prof=True):
        S.solve_device(M, b, None, space, P.SolverConfig(tol=seq.tol, seed=0), use_graph=2)
    st = S.LAST_SOLVE["phase_stamps"].astype(np.int64)
    used = 6 if st[0, 12] != 0 else 10   # fused v2 stamps slots 12, 13
    names = (["P", "M1", "Z1", "Q", "S", "M2", "Z2", "T", "X"] if used >= 10 else
             ["A:P+MZ1", "B:Q", "C:S+MZ2", "D:T", "E:X"])   # v1 / fused v2
    d = np.diff(st[:-1, :len(names) + 1], axis=1) / 1e3
    full = (st[1:, 0] - st[:-1, 0]) / 1e3
    out = {"config": name, "k": k, "us_per_iteration": float(np.median(full)),
           **{nm: round(float(np.median(d[:, i])), 2) for i, nm in enumerate(names)}}
    if used < 10:   # fused v2 sub-stamps (slots 6..13, see persist.cu)
        rel = lambda j, i: round(float(np.median((st[:-1, j] - st[:-1, i]) / 1e3)), 2)
        out.update({"A.spmv": rel(6, 0), "A.proj": rel(7, 6), "A.sync": rel(8, 7),
                    "A.finals": rel(1, 8), "B.work": rel(12, 1), "B.sync": rel(13, 12),
                    "B.finals": rel(2, 13), "C.spmv": rel(9, 2), "C.proj": rel(10, 9),
                    "C.sync": rel(11, 10), "C.finals": rel(3, 11)})
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", nargs="+", default=["c2"])
    ap.add_argument("--k", type=int, default=None)
    ap.add_argument("--max-itn", type=int, default=None)
    ap.add_argument("--both", action="store_true", help="also k = 0")
    ap.add_argument("--system", type=int, default=0, help="matrix index of the sequence")
    ap.add_argument("--fmt", type=int, default=0, help="matrix format (0 auto, 2 SELL-32, 4 offset-coded)")
    ap.add_argument("--phases", action="store_true",
                    help="per-phase breakdown of the persistent kernel")
    ap.add_argument("--tune", nargs="*", default=[],
                    help="tuning knobs key=value (paper_1406_2831_b200._lib.tuning)")
    a = ap.parse_args()
    if a.tune:
        from paper_1406_2831_b200 import _lib
        _lib.tuning(**{kv.split("=")[0]: int(kv.split("=")[1]) for kv in a.tune})
    if a.phases:
        for c in a.config:
            print(json.dumps(phase_breakdown(c, a.k)), flush=True)
        sys.exit(0)
    for c in a.config:
        print(json.dumps(run(c, a.k, max_itn=a.max_itn, fmt=a.fmt, system=a.system)), flush=True)
        if a.both:
            print(json.dumps(run(c, 0, max_itn=a.max_itn, fmt=a.fmt, system=a.system)), flush=True)
