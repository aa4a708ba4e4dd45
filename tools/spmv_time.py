"""Stand-alone SpMV timing on a BASELINE config's first matrix: CUDA events
over back-to-back krb_spmv launches (the matrix is > L2, so every launch
streams it from HBM), algorithmic GB/s (12 nnz + 4 (n+1) + 16 n)
and the fraction of the measured copy peak.
    python tools/spmv_time.py --config c5 [--transpose]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--transpose", action="store_true")
    ap.add_argument("--fmt", type=int, default=0, help="0 auto, 1 CSR, 2 SELL-32, 4 offset-coded")
    ap.add_argument("--tune", nargs="*", default=[], help="knob=value ...")
    a = ap.parse_args()
    import torch
    from paper_1406_2831_b200 import _lib, device as D, workloads as W
    if a.tune:
        _lib.tuning(**{kv.split("=")[0]: int(kv.split("=")[1]) for kv in a.tune})
    seq = W.make_sequence(a.config)
    A = seq.matrix(0)
    M = D.DeviceMatrix(A.n, A.row_ptr, A.col_idx, A.values, fmt=a.fmt)
    x = torch.randn(A.n, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    for _ in range(3):
        M.spmv(x, y, transpose=a.transpose)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        M.spmv(x, y, transpose=a.transpose)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / a.reps
    B = W.spmv_bytes(A.n, A.nnz)
    peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(
        os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"]
    print(json.dumps({"config": a.config, "format": M.format, "transpose": a.transpose,
                      "n": A.n, "nnz": A.nnz, "device_bytes": M.device_bytes, "us": round(us, 1),
                      "GBps": round(B / us / 1e3, 1), "frac": round(B / us / 1e3 / peak, 4),
                      "stream_bytes": M.stream_bytes, "stats": M.stream_stats, "tune": a.tune}))


if __name__ == "__main__":
    main()
