"""Solve-phase overhead of one C2 bench step: span from the first to the last
k_persist0 launch vs the kernels' own time (torch profiler trace)."""
import json, os, sys
sys.path.insert(0, os.getcwd())
import torch
import bench as B
from torch.profiler import profile, ProfilerActivity
wl = B.Workload("c2", None, "first")
api, dview, dmats, drhs = B.device_api(wl)
for _ in range(2):
    B.policy_step(wl, api, dview)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    B.policy_step(wl, api, dview); torch.cuda.synchronize()
prof.export_chrome_trace("/tmp/tr2.json")
ev = json.load(open("/tmp/tr2.json"))["traceEvents"]
k = sorted([(e["ts"], e["ts"] + e.get("dur", 0), e["name"]) for e in ev
            if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")])
p0 = [x for x in k if "k_persist0" in x[2]]
gen = [x for x in k if "k_bpersist" in x[2]]
t0, t1 = k[0][0], k[-1][1]
print("step span %.2f ms" % ((t1 - t0) / 1e3))
print("generation: first bpersist %.2f -> last bpersist end %.2f ms" % ((gen[0][0] - t0) / 1e3, (gen[-1][1] - t0) / 1e3))
print("solve phase: first persist0 start %.2f ms, span %.2f ms, persist0 sum %.2f ms" % (
    (p0[0][0] - t0) / 1e3, (p0[-1][1] - p0[0][0]) / 1e3, sum(e - s for s, e, _ in p0) / 1e3))
gaps = [(p0[i + 1][0] - p0[i][1]) / 1e3 for i in range(len(p0) - 1)]
print("between persist0 launches (ms):", " ".join("%.3f" % g for g in gaps))
mid = [x for x in k if p0[0][1] <= x[0] and x[1] <= p0[1][0]]
for s, e, nm in mid:
    print("   %.1f us  %s" % (e - s, nm[:70]))
