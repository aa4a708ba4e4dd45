"""persist0 phase stamps as seen by several CTAs (KRB_P0_PROF_CTA)."""
import os, sys, json
os.environ["KRB_PHASE_PROF"] = "1"
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_1406_2831_b200 as P
from paper_1406_2831_b200 import device as D, solvers as S, workloads as W
seq = W.make_sequence(sys.argv[1] if len(sys.argv) > 1 else "c2"); A = seq.matrix(0)
M = D.DeviceMatrix(A.n, A.row_ptr, A.col_idx, A.values)
b = D.to_device(seq.rhs(0, 0))
order = [0, 13, 14, 6, 7, 8, 2, 9, 10, 11, 3, 4, 1, 12, 5]
for cta in [int(c) for c in (sys.argv[2] if len(sys.argv) > 2 else "0,1,60,107,108,147").split(",")]:
    os.environ["KRB_P0_PROF_CTA"] = str(cta)
    S.solve_device(M, b, None, None, P.SolverConfig(tol=seq.tol, seed=0), use_graph=2)
    st = S.LAST_SOLVE["phase_stamps"].astype(np.int64)[:-1]
    dd = (st[1:, 0] - st[:-1, 0]) / 1e3
    out = {"cta": cta, "us_per_it": round(float(np.median(dd)), 2)}
    for a_, b_ in zip(order, order[1:]):
        out[f"{a_}->{b_}"] = round(float(np.median(st[:, b_] - st[:, a_])) / 1e3, 2)
    print(json.dumps(out))
