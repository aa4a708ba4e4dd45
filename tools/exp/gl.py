# host time of the rbicg pause/resume calls
import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
import bench as B
from paper_1406_2831_b200 import _lib
wl = B.Workload("c2", None, "first")
api, dview, dmats, drhs = B.device_api(wl)
B.policy_step(wl, api, dview); torch.cuda.synchronize()
orig = _lib.call
acc = {}
def timed(name, *a):
    t = time.perf_counter(); r = orig(name, *a); acc.setdefault(name, [0, 0.0]); acc[name][0] += 1; acc[name][1] += time.perf_counter() - t; return r
_lib.call = timed
import paper_1406_2831_b200.solvers as S, paper_1406_2831_b200.recycling as R
t = time.perf_counter(); B.policy_step(wl, api, dview); torch.cuda.synchronize(); print("step", time.perf_counter() - t)
for k, v in sorted(acc.items(), key=lambda kv: -kv[1][1])[:15]: print(f"{k:28s} {v[0]:5d} {1e3*v[1]:8.2f} ms")
