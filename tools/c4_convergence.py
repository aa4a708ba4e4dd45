"""C4 (power-law rows, n = 4 M) convergence study: BiCGSTAB iterations to
tol 1e-8 for system 0 (sigma = 0) and system 1 of the C4 generator at
n = 20 k / 200 k / 1 M / 4 M, with a generous iteration cap.
    python tools/c4_convergence.py [--cpu]   (--cpu: the reference algorithm,
    oracle RefOps, for the sizes that finish in minutes)"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cpu", action="store_true")
    ap.add_argument("--sizes", type=int, nargs="+", default=[20_000, 200_000, 1_000_000, 4_000_000])
    ap.add_argument("--max-itn", type=int, default=5000)
    a = ap.parse_args()
    from paper_1406_2831_b200.workloads import c4_sequence
    for n in a.sizes:
        seq = c4_sequence(n=n, num=2)
        for j in (0, 1):
            A, b = seq.matrix(j), seq.rhs(j, 0)
            t0 = time.time()
            if a.cpu:
                from oracle import krylov as O
                from oracle.ops import RefOps
                _, h = O.bicgstab(A, b, config=O.Config(tol=1e-8, max_itn=a.max_itn, seed=j),
                                  ops=RefOps())
                kind = "cpu RefOps"
            else:
                import paper_1406_2831_b200 as P
                _, h = P.bicgstab_solve(P.SparseMatrix.from_csr(A), b,
                                        config=P.SolverConfig(tol=1e-8, max_itn=a.max_itn, seed=j))
                kind = "gpu"
            r = h.resid
            print(json.dumps({"n": n, "system": j, "kind": kind, "iterations": h.iterations,
                              "status": h.status, "final_true_resid": h.final_true_resid,
                              "resid_at": {str(i): r[i] / r[0] for i in (100, 500, 1000, 2000)
                                           if i < len(r)},
                              "seconds": round(time.time() - t0, 2)}), flush=True)


if __name__ == "__main__":
    main()
