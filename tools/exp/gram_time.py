"""Time the device Gram (canonical chunk order) on update-sized blocks."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_1406_2831_b200 import recycling as R
for m, n in [(47, 262144), (27, 262144), (20, 262144), (47, 2097152), (60, 16777216)]:
    X = torch.randn(m, n, dtype=torch.float64, device="cuda")
    Y = torch.randn(m, n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        R.gram(X, Y)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        R.gram(X, Y)
    e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 20 * 1e3
    print(f"v{os.environ.get('KRB_GRAM_V', '2')} gram {m}x{m} n={n}: {us:.1f} us  {2*m*m*n/us/1e6:.2f} TFLOP/s")
