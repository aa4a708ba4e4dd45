"""krb_gemm: tiled (k_gemm_t) vs row kernel, bitwise + timing."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_1406_2831_b200 import recycling as R
n = 262144
for m, nc in ((47, 47), (47, 20), (20, 20), (26, 26), (19, 19), (8, 3), (100, 60), (47, 1)):
    X = torch.randn(m, n, dtype=torch.float64, device="cuda")
    Z = torch.from_numpy(np.random.default_rng(m).standard_normal((m, nc))).cuda()
    res = {}
    for mode in ("0", "8", "12", "24", "122"):
        os.environ["KRB_GEMM_TILED"] = mode
        out = R.gemm(X, Z); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            out = R.gemm(X, Z)
        e1.record(); torch.cuda.synchronize()
        res[mode] = (out.clone(), e0.elapsed_time(e1) / 20 * 1e3)
    same = all(torch.equal(res["0"][0], res[k][0]) for k in res)
    print(f"m={m:3d} nc={nc:3d} " + "  ".join(f"{k}:{v[1]:7.1f}" for k, v in res.items()) + f"  bitwise {same}")
