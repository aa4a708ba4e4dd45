"""One Gram and one GEMM at the C2 update shape (47 x 262144), for ncu."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_1406_2831_b200 import recycling as R
n, m = 262144, 47
X = torch.randn(m, n, dtype=torch.float64, device="cuda")
Y = torch.randn(m, n, dtype=torch.float64, device="cuda")
Z = torch.from_numpy(np.random.default_rng(0).standard_normal((m, m))).cuda()
for _ in range(2):
    R.gram(X, Y); R.gemm(X, Z)
torch.cuda.synchronize()
