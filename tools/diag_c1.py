"""Diagnostic: GPU vs CanonOps on full C1 systems (space bits, histories),
per iteration driver."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1406_2831_b200 as P
from oracle import krylov as O
from oracle.ops import CanonOps
from paper_1406_2831_b200.workloads import make_sequence, sine_basis
from paper_1406_2831_b200 import solvers as SV, _lib
from paper_1406_2831_b200.device import to_device
ops = CanonOps()
name = sys.argv[1] if len(sys.argv) > 1 else "c1"
seq = make_sequence(name)
for j in range(len(seq.meta.get("shifts", range(6))) if name != "c1" else 6):
    A = seq.matrix(j); b = seq.rhs(j, 0)
    U = sine_basis(tuple(seq.meta['grid']), seq.k)
    M = P.SparseMatrix.from_csr(A)
    Sg = P.biorthonormalize(U, U, M)
    So = O.biorthonormalize(U, U, A, ops=ops)
    same = all(np.array_equal(np.asarray(getattr(Sg, f)), np.asarray(getattr(So, f)))
               for f in ("U", "Ut", "C", "Ct", "Dc", "Chat", "Ccheck"))
    cfg = P.SolverConfig(tol=seq.tol, max_itn=seq.max_itn, seed=j)
    xo, ho = O.rbicgstab(A, b, recycle=So, ops=ops,
                         config=O.Config(tol=seq.tol, max_itn=seq.max_itn, seed=j))
    Md, _ = SV._check_common(M, b, None, cfg)
    for mode in (None, 0, 1, 2):
        with _lib.tuning(graph_mode=mode):
            _, hg = SV.solve_device(Md, to_device(b), None, Sg, cfg)
        first = next((i for i, (a, c) in enumerate(zip(hg.resid, ho.resid)) if a != c), None)
        print(name, j, "space same", same, "mode", mode, "driver", SV.LAST_SOLVE.get("driver"),
              "gpu", hg.iterations, hg.status, "canon", ho.iterations, ho.status,
              "first diff", first, flush=True)
