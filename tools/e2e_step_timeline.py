"""Host wall-clock timeline of bench.py's end-to-end step (pinned inputs):
per system the time spent in each statement of the step (matrix adoption,
prefetch issue, refresh, solve incl. upload of b and read-back of x), without
extra synchronisations, next to the device-resident step of the value arm.

    python tools/e2e_step_timeline.py [--pageable]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402


def main():
    import torch
    import bench as B
    import paper_1406_2831_b200 as P
    from paper_1406_2831_b200 import device as D, workloads as W
    pageable = "--pageable" in sys.argv
    wl = B.Workload("c5")
    cfgs = [P.SolverConfig(tol=wl.seq.tol, max_itn=wl.seq.max_itn, k=wl.k, s=wl.seq.s, seed=j + 1)
            for j in range(len(wl.keys))]
    cache = {}

    def pin(a):
        if id(a) not in cache:
            cache[id(a)] = D.pinned_copy(a)
        return cache[id(a)]
    if pageable:
        mats, rhs = wl.mats, wl.rhs
    else:
        mats = {i: W.CSR(A.n, pin(A.row_ptr), pin(A.col_idx), pin(A.values))
                for i, A in wl.mats.items()}
        rhs = {key: D.pinned_copy(b) for key, b in wl.rhs.items()}
    i0 = wl.keys[0][0]
    space0 = P.biorthonormalize(wl.U0, wl.Ut0, P.SparseMatrix.from_csr(mats[i0]))
    D.MATRICES.clear()

    def step(log):
        t0 = time.perf_counter()
        D.MATRICES.clear()
        space, last_i, A = space0, None, None
        order = [i for i in dict.fromkeys(i for i, _ in wl.keys)]
        sms = {}
        log.append(("clear", time.perf_counter() - t0))
        for j, (i, kap) in enumerate(wl.keys):
            row = {"sys": i}
            t = time.perf_counter()
            if i != last_i:
                A = sms.pop(i, None)
                if A is None:
                    A = P.SparseMatrix.from_csr(mats[i])
                    P.prefetch_matrix(A)
                nxt = order.index(i) + 1
                if nxt < len(order):
                    sms[order[nxt]] = P.SparseMatrix.from_csr(mats[order[nxt]])
                    P.prefetch_matrix(sms[order[nxt]])
                row["adopt_prefetch"] = round(time.perf_counter() - t, 4)
                t = time.perf_counter()
                D.device_matrix(A)
                row["device_matrix"] = round(time.perf_counter() - t, 4)
                t = time.perf_counter()
                if j > 0:
                    space = P.refresh_images(space, A)
                row["refresh"] = round(time.perf_counter() - t, 4)
                last_i = i
            t = time.perf_counter()
            x, h = P.rbicgstab_solve(A, rhs[(i, kap)], recycle=space, config=cfgs[j])
            row["solve"] = round(time.perf_counter() - t, 4)
            row["its"] = h.iterations
            row["loop_s"] = round(float(h.times[-1] - h.times[0]), 4) if len(getattr(h, "times", [])) > 1 else None
            log.append(row)
        torch.cuda.synchronize()
        return time.perf_counter() - t0

    for rep in range(3):
        log = []
        tot = step(log)
        print(json.dumps({"rep": rep, "total_s": round(tot, 3), "log": log}), flush=True)


if __name__ == "__main__":
    main()
