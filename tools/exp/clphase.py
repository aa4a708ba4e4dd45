import os, sys, json
os.environ["KRB_PHASE_PROF"] = "1"
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_1406_2831_b200 as P
from paper_1406_2831_b200 import device as D, solvers as S, workloads as W
seq = W.make_sequence("c1"); A = seq.matrix(0)
M = D.DeviceMatrix(A.n, A.row_ptr, A.col_idx, A.values)
r = np.random.default_rng(12345)
for k in (10, 0):
    space = P.biorthonormalize(r.standard_normal((A.n, k)), r.standard_normal((A.n, k)), M) if k else None
    b = D.to_device(seq.rhs(0, 0))
    S.solve_device(M, b, None, space, P.SolverConfig(tol=seq.tol, seed=0), use_graph=2)
    st = S.LAST_SOLVE["phase_stamps"].astype(np.int64)[:-1]
    dd = (st[1:, 0] - st[:-1, 0]) / 1e3
    full = np.median(dd)
    print("mean", dd.mean(), "max", dd.max(), "p90", np.percentile(dd, 90), "n", len(dd), "span_ms", (st[-1,0]-st[0,0])/1e6)
    d = {f"{i}-{i+1}": round(float(np.median(st[:, i + 1] - st[:, i])) / 1e3, 2) for i in range(9) if (st[:, i + 1] > 0).all() and (st[:, i] > 0).all()}
    print(json.dumps({"k": k, "us_per_it": round(full, 2), **d}))
