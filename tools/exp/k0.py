import os, sys, json, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1406_2831_b200 as P
from paper_1406_2831_b200 import device as D, solvers as S, workloads as W
seq = W.make_sequence("c2"); A = seq.matrix(0)
M = D.DeviceMatrix(A.n, A.row_ptr, A.col_idx, A.values)
b = D.to_device(seq.rhs(0, 0))
cfg = P.SolverConfig(tol=seq.tol, seed=0)
for rep in range(4):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); e0.record()
    _, h = S.solve_device(M, b, None, None, cfg, use_graph=2)
    e1.record(); torch.cuda.synchronize(); t1 = time.perf_counter()
    print(rep, h.iterations, "events ms", round(e0.elapsed_time(e1), 3), "wall ms", round((t1 - t0) * 1e3, 3),
          "hist span ms", round(h.seconds[-1] - h.seconds[0], 6) * 1e3)
