"""Shapes and device times of the generation-path kernels in one bench step."""
import os, sys, collections, time
sys.path.insert(0, os.getcwd())
import torch
import bench as B
from paper_1406_2831_b200 import recycling as R, update as U
log = collections.defaultdict(list)
def wrap(mod, name):
    f = getattr(mod, name)
    def g(*a, **k):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); out = f(*a, **k); e1.record(); torch.cuda.synchronize()
        shp = tuple(tuple(x.shape) if hasattr(x, "shape") else x for x in a[:2])
        log[(name, shp)].append(e0.elapsed_time(e1) * 1e3)
        return out
    return g
for mod in (R, U):
    for name in ("gemm", "gram", "colscale_div", "colnorms"):
        if hasattr(mod, name):
            setattr(mod, name, wrap(R, name) if mod is U else wrap(mod, name))
wl = B.Workload("c2", None, "first")
api, dview, dmats, drhs = B.device_api(wl)
B.policy_step(wl, api, dview); torch.cuda.synchronize()
log.clear()
B.policy_step(wl, api, dview); torch.cuda.synchronize()
tot = 0
for key, v in sorted(log.items(), key=lambda kv: -sum(kv[1])):
    tot += sum(v)
    print(f"{key[0]:14s} {str(key[1]):40s} n={len(v):3d} us_each={sum(v)/len(v):8.1f} total_ms={sum(v)/1e3:6.2f}")
print("total ms", tot / 1e3)
