"""Time the multi-column SpMV (A X and A^T X) on a bench matrix."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_1406_2831_b200 import device as D
from paper_1406_2831_b200.workloads import make_sequence
for cfg in (sys.argv[1:] or ["c2"]):
    A = make_sequence(cfg).matrix(0)
    M = D.DeviceMatrix(A.n, A.row_ptr, A.col_idx, A.values)
    for nc in (27, 8):
        X = torch.randn(nc, A.n, dtype=torch.float64, device="cuda")
        for tr in (False, True):
            for _ in range(3):
                M.spmm(X, transpose=tr)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20):
                M.spmm(X, transpose=tr)
            e1.record(); torch.cuda.synchronize()
            print(f"{cfg} spmm ncols={nc} transpose={tr}: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us")
