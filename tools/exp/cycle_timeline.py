"""Device timeline of one harvest cycle in the C2 bench step (between two
k_bpersist launches): every op with its start offset and the idle gap before it."""
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
prof.export_chrome_trace("/tmp/tr3.json")
ev = json.load(open("/tmp/tr3.json"))["traceEvents"]
k = sorted([(e["ts"], e["ts"] + e.get("dur", 0), e["name"]) for e in ev
            if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")])
gen = [i for i, x in enumerate(k) if "k_bpersist" in x[2]]
c = int(sys.argv[1]) if len(sys.argv) > 1 else 3
a, b = gen[c], gen[c + 1]
t0 = k[a][0]
prev_end = k[a][0]
busy = 0
for s, e, nm in k[a:b + 1]:
    gap = s - prev_end
    print("%8.1f  gap %7.1f  dur %7.1f  %s" % (s - t0, max(gap, 0), e - s, nm[:60]))
    prev_end = max(prev_end, e)
    busy += e - s
print("cycle span %.1f us, busy %.1f us" % (k[b][0] - t0, busy))
