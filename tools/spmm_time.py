"""SpMM (krb_spmm: A X and A^T X for ncols columns, the refresh_images /
update products) timing on a BASELINE config's first matrix, CUDA events.
    python tools/spmm_time.py --config c5 --ncols 30 [--tune key=value]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    ap.add_argument("--ncols", type=int, default=30)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--tune", nargs="*", default=[])
    a = ap.parse_args()
    import torch
    from paper_1406_2831_b200 import _lib, device as D, workloads as W
    if a.tune:
        _lib.tuning(**{kv.split("=")[0]: int(kv.split("=")[1]) for kv in a.tune})
    A = W.make_sequence(a.config).matrix(0)
    M = D.DeviceMatrix(A.n, A.row_ptr, A.col_idx, A.values)
    X = torch.randn(a.ncols, A.n, dtype=torch.float64, device="cuda")
    out = {"config": a.config, "format": M.format, "ncols": a.ncols, "tune": a.tune}
    for tr in (False, True):
        Y = M.spmm(X, transpose=tr)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            M.spmm(X, transpose=tr, out=Y)
        e1.record()
        torch.cuda.synchronize()
        out["AT_ms" if tr else "A_ms"] = round(e0.elapsed_time(e1) / a.reps, 3)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
