import os, sys, json
os.environ["KRB_PHASE_PROF"] = "1"
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_1406_2831_b200 as P
from paper_1406_2831_b200 import device as D, solvers as S, workloads as W
cfgname = sys.argv[1] if len(sys.argv) > 1 else "c2"
k = int(sys.argv[2]) if len(sys.argv) > 2 else 0
seq = W.make_sequence(cfgname); A = seq.matrix(0)
M = D.DeviceMatrix(A.n, A.row_ptr, A.col_idx, A.values)
r = np.random.default_rng(12345)
space = P.biorthonormalize(r.standard_normal((A.n, k)), r.standard_normal((A.n, k)), M) if k else None
b = D.to_device(seq.rhs(0, 0))
S.solve_device(M, b, None, space, P.SolverConfig(tol=seq.tol, seed=0), use_graph=2)
st = S.LAST_SOLVE["phase_stamps"].astype(np.int64)[:-1]
order = [0, 6, 7, 8, 1, 12, 13, 2, 9, 10, 11, 3, 4, 5]
order = [o for o in order if (st[:, o] > 0).all()]
dd = (st[1:, 0] - st[:-1, 0]) / 1e3
out = {"k": k, "us_per_it": round(float(np.median(dd)), 2)}
for a_, b_ in zip(order, order[1:]):
    out[f"{a_}->{b_}"] = round(float(np.median(st[:, b_] - st[:, a_])) / 1e3, 2)
print(json.dumps(out))
