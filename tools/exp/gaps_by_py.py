"""GPU idle gaps of one bench step, attributed to the innermost Python frame
active at the gap midpoint (and its caller chain)."""
import json, os, sys, collections
sys.path.insert(0, os.getcwd())
import torch
import bench as B
from torch.profiler import profile, ProfilerActivity
wl = B.Workload(sys.argv[1] if len(sys.argv) > 1 else "c2", None, "first")
api, dview, dmats, drhs = B.device_api(wl)
B.policy_step(wl, api, dview); torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU], with_stack=True) as prof:
    B.policy_step(wl, api, dview); torch.cuda.synchronize()
prof.export_chrome_trace("/tmp/tr.json")
ev = json.load(open("/tmp/tr.json"))["traceEvents"]
gpu = sorted([(e["ts"], e["ts"] + e.get("dur", 0), e["name"]) for e in ev
              if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")])
gaps = []
cur_e = gpu[0][1]
for s, e, nm in gpu[1:]:
    if s > cur_e:
        gaps.append((cur_e, s))
    cur_e = max(cur_e, e)
py = [e for e in ev if e.get("cat") == "python_function"]
def chain(t):
    act = [e for e in py if e["ts"] <= t <= e["ts"] + e.get("dur", 0)]
    act.sort(key=lambda e: -e.get("dur", 0))
    names = [a["name"].split("/")[-1] for a in act]
    return " > ".join(names[-4:])
agg = collections.Counter(); cnt = collections.Counter()
for a, b in gaps:
    g = b - a
    if g < 20:
        agg["<20us gaps"] += g; cnt["<20us gaps"] += 1
        continue
    k = chain((a + b) / 2)
    agg[k] += g; cnt[k] += 1
tot = sum(agg.values())
print(f"idle {tot/1e3:.2f} ms in {len(gaps)} gaps")
for k, v in agg.most_common(40):
    print(f"{v/1e3:8.3f} ms x{cnt[k]:4d}  {k}")
