"""persist0: per-CTA phase work (A SpMV, C SpMV, E update) over all CTAs."""
import os, sys, json
os.environ["KRB_PHASE_PROF"] = "1"
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_1406_2831_b200 as P
from paper_1406_2831_b200 import device as D, solvers as S, workloads as W
seq = W.make_sequence(sys.argv[1] if len(sys.argv) > 1 else "c2"); A = seq.matrix(0)
M = D.DeviceMatrix(A.n, A.row_ptr, A.col_idx, A.values)
b = D.to_device(seq.rhs(0, 0))
rows = []
for cta in range(148):
    os.environ["KRB_P0_PROF_CTA"] = str(cta)
    S.solve_device(M, b, None, None, P.SolverConfig(tol=seq.tol, seed=0), use_graph=2)
    st = S.LAST_SOLVE["phase_stamps"].astype(np.int64)[:-1]
    med = lambda a_, b_: float(np.median(st[:, b_] - st[:, a_])) / 1e3
    rows.append((cta, med(0, 6), med(7, 8), med(2, 9), med(10, 11), med(3, 4), med(1, 12)))
rows = np.array(rows)
np.set_printoptions(linewidth=200, precision=2, suppress=True)
print("cols: cta A_work A_wait C_work C_wait E_work E_wait")
for r in rows[np.argsort(-rows[:, 1])][:12]:
    print(r)
print("min A_wait ctas:", rows[np.argsort(rows[:, 2])][:8, [0, 1, 2]])
print("min C_wait ctas:", rows[np.argsort(rows[:, 4])][:8, [0, 3, 4]])
