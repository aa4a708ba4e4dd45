"""Per-iteration time of the device RBiCGSTAB (graph path) on a BASELINE
config with a fixed seeded k-space: us/iteration and algorithmic GB/s
(SURVEY.md §8(d) bytes).   python tools/iter_time.py --config c2 c5 ..."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402


def run(name, k=None, reps=3, max_itn=None):
    import torch
    import paper_1406_2831_b200 as P
    from paper_1406_2831_b200 import device as D, solvers as S, workloads as W
    seq = W.make_sequence(name)
    A = seq.matrix(0)
    k = seq.k if k is None else k
    M = D.DeviceMatrix(A.n, A.row_ptr, A.col_idx, A.values)
    r = np.random.default_rng(12345)
    space = None
    if k:
        space = P.biorthonormalize(r.standard_normal((A.n, k)),
                                   r.standard_normal((A.n, k)), M)
    b = D.to_device(seq.rhs(0, 0))
    cfg = P.SolverConfig(tol=seq.tol, max_itn=max_itn or seq.max_itn, seed=0)
    S.solve_device(M, b, None, space, cfg)
    best, h = None, None
    for _ in range(reps):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        _, h = S.solve_device(M, b, None, space, cfg)
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 1e3
        best = t if best is None else min(best, t)
    kk = space.k if space is not None else 0
    its = max(h.iterations, 1)
    B = W.bytes_per_iteration(A.n, A.nnz, kk)
    return {"config": name, "n": A.n, "nnz": A.nnz, "k": kk, "format": M.format,
            "iterations": h.iterations, "status": h.status,
            "solve_ms": round(best * 1e3, 3), "us_per_it": round(best / its * 1e6, 2),
            "GBps_alg": round(B * its / best / 1e9, 1)}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", nargs="+", default=["c2"])
    ap.add_argument("--k", type=int, default=None)
    ap.add_argument("--max-itn", type=int, default=None)
    ap.add_argument("--both", action="store_true", help="also k = 0")
    a = ap.parse_args()
    for c in a.config:
        print(json.dumps(run(c, a.k, max_itn=a.max_itn)), flush=True)
        if a.both:
            print(json.dumps(run(c, 0, max_itn=a.max_itn)), flush=True)
