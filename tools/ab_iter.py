"""In-process A/B of one tuning knob on the device RBiCGSTAB iteration: one
matrix and one seeded k-space, solves alternating the knob's values round
after round (same box, same clocks), best and median us per iteration.
    python tools/ab_iter.py --config c5 --knob phase_pf_rows --values 0 2 4 --rounds 4"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    ap.add_argument("--system", type=int, default=0)
    ap.add_argument("--knob", required=True)
    ap.add_argument("--values", type=int, nargs="+", required=True)
    ap.add_argument("--rounds", type=int, default=4)
    ap.add_argument("--max-itn", type=int, default=60)
    a = ap.parse_args()
    import torch
    import paper_1406_2831_b200 as P
    from paper_1406_2831_b200 import _lib, device as D, solvers as S, workloads as W
    seq = W.make_sequence(a.config)
    A = seq.matrix(a.system)
    M = D.DeviceMatrix(A.n, A.row_ptr, A.col_idx, A.values)
    r = np.random.default_rng(12345)
    space = P.biorthonormalize(r.standard_normal((A.n, seq.k)), r.standard_normal((A.n, seq.k)), M)
    b = D.to_device(seq.rhs(a.system, 0))
    cfg = P.SolverConfig(tol=seq.tol, max_itn=a.max_itn, seed=0)
    res = {v: [] for v in a.values}
    ref = None
    for rnd in range(a.rounds + 1):
        for v in a.values:
            _lib.tuning(**{a.knob: v})
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            _, h = S.solve_device(M, b, None, space, cfg)
            e1.record()
            torch.cuda.synchronize()
            if ref is None:
                ref = h.resid
            assert h.resid == ref, "variants must compute the same bits"
            if rnd:   # round 0 warms every variant (graph capture)
                res[v].append(e0.elapsed_time(e1) * 1e3 / max(h.iterations, 1))
    _lib.reset_tuning()
    print(json.dumps({"config": a.config, "system": a.system, "knob": a.knob,
                      "format": M.format,
                      "us_per_it": {str(v): {"best": round(min(t), 1),
                                             "median": round(statistics.median(t), 1)}
                                    for v, t in res.items()}}))


if __name__ == "__main__":
    main()
