"""Multi-rhs vs single solves on a BASELINE config (fixed iteration count):
    python tools/batch_time.py --config c3 --nrhs 4 --k 20 --iters 60"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--nrhs", type=int, default=4)
    ap.add_argument("--k", type=int, default=None)
    ap.add_argument("--iters", type=int, default=60)
    a = ap.parse_args()
    import torch
    import paper_1406_2831_b200 as P
    from paper_1406_2831_b200 import device as D, workloads as W
    seq = W.make_sequence(a.config)
    A = seq.matrix(0)
    k = seq.k if a.k is None else a.k
    M = D.DeviceMatrix(A.n, A.row_ptr, A.col_idx, A.values)
    r = np.random.default_rng(1)
    space = P.biorthonormalize(r.standard_normal((A.n, k)), r.standard_normal((A.n, k)), M) if k else None
    bs = [D.to_device(r.standard_normal(A.n)) for _ in range(a.nrhs)]
    cfgs = [P.SolverConfig(tol=1e-30, max_itn=a.iters, seed=j) for j in range(a.nrhs)]

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / 1e3

    def singles():
        for j in range(a.nrhs):
            if space is not None:
                P.rbicgstab_solve(M, bs[j], recycle=space, config=cfgs[j])
            else:
                P.bicgstab_solve(M, bs[j], config=cfgs[j])

    def batch():
        if space is not None:
            P.rbicgstab_solve_batch(M, bs, recycle=space, configs=cfgs)
        else:
            P.bicgstab_solve_batch(M, bs, configs=cfgs)

    ts, tb = timed(singles), timed(batch)
    its = a.iters * a.nrhs
    B = W.bytes_per_iteration(A.n, A.nnz, space.k if space is not None else 0)
    print(json.dumps({"config": a.config, "n": A.n, "k": space.k if space is not None else 0,
                      "nrhs": a.nrhs, "singles_us_per_rhs_it": round(ts / its * 1e6, 1),
                      "batch_us_per_rhs_it": round(tb / its * 1e6, 1),
                      "speedup": round(ts / tb, 3),
                      "batch_equiv_GBps": round(B * its / tb / 1e9, 1)}))


if __name__ == "__main__":
    main()
