import cProfile, pstats, sys, os
sys.path.insert(0, os.getcwd())
import torch
import bench as B
wl = B.Workload("c2", None, "first")
api, dview, dmats, drhs = B.device_api(wl)
B.policy_step(wl, api, dview)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
B.policy_step(wl, api, dview)
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("cumulative").print_stats(35)
st.sort_stats("tottime").print_stats(20)
