import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_1406_2831_b200 import recycling as R
for k in (47, 20, 8):
    X = torch.randn(k, 262144, dtype=torch.float64, device="cuda")
    s = torch.rand(k, dtype=torch.float64, device="cuda") + 1.0
    R.colscale_div(X, s); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        R.colscale_div(X, s)
    e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 20 * 1e3
    print(k, round(us, 1), "us", round(2 * 8 * k * 262144 / us / 1e3, 0), "GB/s")
