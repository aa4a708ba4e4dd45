"""Profiling driver: RBiCGSTAB solves on one BASELINE config with a fixed
seeded k-dimensional space, in host-loop mode (graph_mode 0) so ncu can
see every kernel (it cannot profile inside conditional graph nodes).

    python tools/profile_iter.py --config c2 --solves 2
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1406_2831_b200 import _lib  # noqa: E402
_lib.PY_TUNING["graph_mode"] = 0

import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--solves", type=int, default=2)
    ap.add_argument("--k", type=int, default=None)
    ap.add_argument("--max-itn", type=int, default=None)
    a = ap.parse_args()
    import torch
    import paper_1406_2831_b200 as P
    from paper_1406_2831_b200 import device as D, solvers as S, workloads as W
    seq = W.make_sequence(a.config)
    A = seq.matrix(0)
    k = seq.k if a.k is None else a.k
    M = D.DeviceMatrix(A.n, A.row_ptr, A.col_idx, A.values)
    r = np.random.default_rng(12345)
    space = P.biorthonormalize(r.standard_normal((A.n, k)), r.standard_normal((A.n, k)), M)
    b = D.to_device(seq.rhs(0, 0))
    for i in range(a.solves):
        _, h = S.solve_device(M, b, None, space,
                              P.SolverConfig(tol=seq.tol, max_itn=a.max_itn or seq.max_itn,
                                             seed=i))
        print(f"solve {i}: {h.status} {h.iterations} iterations, k={space.k}, "
              f"format={M.format}")
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
