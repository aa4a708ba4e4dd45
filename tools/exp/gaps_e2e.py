"""GPU idle gaps of one e2e step (pinned host inputs through the public
API), attributed to the Python frames active at the gap midpoint."""
import json, os, sys, collections
sys.path.insert(0, os.getcwd())
import torch
import bench as B
import paper_1406_2831_b200 as P
from paper_1406_2831_b200 import device as D
from paper_1406_2831_b200.sequence import run_sequence
from torch.profiler import profile, ProfilerActivity
wl = B.Workload("c2", None, "first")
pv = wl.pinned_view()
def host_step():
    D.MATRICES.clear()
    return run_sequence(pv, policy=wl.policy, baseline=False, api=P, systems=wl.nsys)
host_step(); torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU], with_stack=True) as prof:
    host_step(); torch.cuda.synchronize()
prof.export_chrome_trace("/tmp/tr.json")
ev = json.load(open("/tmp/tr.json"))["traceEvents"]
gpu = sorted([(e["ts"], e["ts"] + e.get("dur", 0), e["name"]) for e in ev
              if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")])
byname = collections.Counter()
for s, e, nm in gpu:
    byname[nm.split("(")[0][:60]] += e - s
print("span %.2f ms" % ((gpu[-1][1] - gpu[0][0]) / 1e3))
for k, v in byname.most_common(12):
    print(f"  busy {v/1e3:8.3f} ms  {k}")
gaps = []
cur_e = gpu[0][1]
for s, e, nm in gpu[1:]:
    if s > cur_e:
        gaps.append((cur_e, s))
    cur_e = max(cur_e, e)
py = [e for e in ev if e.get("cat") == "python_function"]
def chain(t):
    act = [e for e in py if e["ts"] <= t <= e["ts"] + e.get("dur", 0) and "SimpleQueue" not in e["name"]]
    act.sort(key=lambda e: -e.get("dur", 0))
    names = [a["name"].split("/")[-1] for a in act]
    return " > ".join(names[-4:])
agg = collections.Counter(); cnt = collections.Counter()
for a, b in gaps:
    g = b - a
    k = "<20us gaps" if g < 20 else chain((a + b) / 2)
    agg[k] += g; cnt[k] += 1
print(f"idle {sum(agg.values())/1e3:.2f} ms in {len(gaps)} gaps")
for k, v in agg.most_common(25):
    print(f"{v/1e3:8.3f} ms x{cnt[k]:4d}  {k}")
