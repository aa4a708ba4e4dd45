"""Time of the split-ILUTP operator on the device vs the reference's CPU
application (SuperLU triangular solves, ilutp.py:37-42) on C1 / C2-small:
factorization, one L^{-1} A P U^{-1} product, one preconditioned BiCGSTAB.
    python tools/ilutp_time.py [--config c1] [--cpu]"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c1")
    ap.add_argument("--small", action="store_true")
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    import torch
    import paper_1406_2831_b200 as P
    from paper_1406_2831_b200.workloads import make_sequence
    from oracle.ops import CsrOperand, RefOps, SplitOperand
    seq = make_sequence(a.config, small=a.small)
    A = P.SparseMatrix.from_csr(seq.matrix(1))
    t0 = time.perf_counter()
    F = P.ilutp_factor(A)
    t_fac = time.perf_counter() - t0
    op = P.SplitPreconditionedOperator(A, F)
    from paper_1406_2831_b200.device import device_matrix, to_device
    M = device_matrix(op)
    x = to_device(np.random.default_rng(0).standard_normal(A.nrows))
    y = M.spmv(x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        M.spmv(x, y)
    e1.record()
    torch.cuda.synchronize()
    gpu_us = e0.elapsed_time(e1) * 1e3 / a.reps
    so = SplitOperand(CsrOperand.of(A), F)
    ref = RefOps()
    xh = x.cpu().numpy()
    ref.matvec(so, xh)
    t0 = time.perf_counter()
    for _ in range(5):
        ref.matvec(so, xh)
    cpu_us = (time.perf_counter() - t0) / 5 * 1e6
    b = P.apply_left(F, seq.rhs(1, 0))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _, h = P.bicgstab_solve(P.CountingOperator(op), b, config=P.SolverConfig(tol=seq.tol, seed=1))
    torch.cuda.synchronize()
    t_solve = time.perf_counter() - t0
    print(json.dumps({"config": a.config, "n": A.nrows, "nnz_L": int(F.L.nnz), "nnz_U": int(F.U.nnz),
                      "levels": F.device().levels, "factor_s": round(t_fac, 3),
                      "gpu_op_us": round(gpu_us, 1), "cpu_superlu_op_us": round(cpu_us, 1),
                      "bicgstab_its": h.iterations, "bicgstab_s": round(t_solve, 4),
                      "status": h.status}))


if __name__ == "__main__":
    main()
