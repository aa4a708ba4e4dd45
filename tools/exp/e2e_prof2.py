import cProfile, pstats, sys, os, time
sys.path.insert(0, os.getcwd())
import torch
import bench as B
import paper_1406_2831_b200 as P
from paper_1406_2831_b200 import device as D
from paper_1406_2831_b200.sequence import run_sequence
wl = B.Workload("c2", None, "first")
pv = wl.pinned_view()
def host_step():
    D.MATRICES.clear()
    return run_sequence(pv, policy=wl.policy, baseline=False, api=P, systems=wl.nsys)
host_step(); torch.cuda.synchronize()
for i in range(3):
    t0 = time.perf_counter(); host_step(); torch.cuda.synchronize(); print("step", time.perf_counter() - t0)
pr = cProfile.Profile(); pr.enable()
host_step(); torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr); st.sort_stats("cumulative").print_stats(30)
