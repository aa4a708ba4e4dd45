"""Where the end-to-end (host numpy inputs) step of bench.py spends its time:
per system, wall time of the matrix upload + device build, the refresh, the
solve and the read-back, each closed by a device synchronisation.  Pinned
vs pageable inputs, with and without the next-matrix prefetch.

    python tools/e2e_phases.py --config c5 --systems 3
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    ap.add_argument("--systems", type=int, default=3)
    args = ap.parse_args()
    import torch
    import paper_1406_2831_b200 as P
    from paper_1406_2831_b200 import device as D, workloads as W
    seq = W.make_sequence(args.config)
    keys = list(range(1, 1 + args.systems))
    mats = {i: seq.matrix_fn(i) for i in keys}
    rhs = {i: seq.rhs(i, 0) for i in keys}
    r = np.random.default_rng(12345)
    U, Ut = r.standard_normal((seq.n, seq.k)), r.standard_normal((seq.n, seq.k))
    cache = {}

    def pin(a):
        if id(a) not in cache:
            cache[id(a)] = D.pinned_copy(a)
        return cache[id(a)]
    pmats = {i: W.CSR(A.n, pin(A.row_ptr), pin(A.col_idx), pin(A.values))
             for i, A in mats.items()}
    prhs = {i: D.pinned_copy(b) for i, b in rhs.items()}
    space0 = P.biorthonormalize(U, Ut, P.SparseMatrix.from_csr(mats[keys[0]]))
    D.MATRICES.clear()
    out = []
    for label, M_, B_, pre in (("pageable", mats, rhs, False), ("pinned", pmats, prhs, False),
                               ("pinned+prefetch", pmats, prhs, True)):
        for rep in range(2):
            D.MATRICES.clear()
            torch.cuda.synchronize()
            space = space0
            rows = []
            nxt = {}
            for j, i in enumerate(keys):
                t0 = time.perf_counter()
                A = nxt.pop(i, None) or P.SparseMatrix.from_csr(M_[i])
                D.device_matrix(A)
                torch.cuda.synchronize()
                t1 = time.perf_counter()
                if pre and j + 1 < len(keys):
                    nxt[keys[j + 1]] = P.SparseMatrix.from_csr(M_[keys[j + 1]])
                    P.prefetch_matrix(nxt[keys[j + 1]])
                if j > 0:
                    space = P.refresh_images(space, A)
                torch.cuda.synchronize()
                t2 = time.perf_counter()
                x, h = P.rbicgstab_solve(A, B_[i], recycle=space,
                                         config=P.SolverConfig(tol=seq.tol, seed=j + 1))
                torch.cuda.synchronize()
                t3 = time.perf_counter()
                rows.append({"sys": i, "upload_build_s": round(t1 - t0, 3),
                             "refresh_s": round(t2 - t1, 3), "solve_s": round(t3 - t2, 3),
                             "its": h.iterations})
            out.append({"mode": label, "rep": rep, "rows": rows,
                        "mem_reserved_gb": round(torch.cuda.memory_reserved() / 2**30, 1)})
            print(json.dumps(out[-1]), flush=True)


if __name__ == "__main__":
    main()
