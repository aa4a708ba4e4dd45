import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
import bench as B
import paper_1406_2831_b200 as P
from paper_1406_2831_b200 import device as D
from paper_1406_2831_b200.sequence import run_sequence
wl = B.Workload("c2", None, "first")
pv = wl.pinned_view()
orig = D.PREFETCH.issue
log = []
def timed(A):
    t0 = time.perf_counter(); r = orig(A); log.append((time.perf_counter() - t0) * 1e3); return r
D.PREFETCH.issue = timed
for s in range(5):
    D.MATRICES.clear(); log.clear()
    t0 = time.perf_counter()
    run_sequence(pv, policy=wl.policy, baseline=False, api=P, systems=wl.nsys)
    torch.cuda.synchronize()
    print("step %.1f ms; prefetch ms:" % ((time.perf_counter() - t0) * 1e3), " ".join("%.2f" % x for x in log))
