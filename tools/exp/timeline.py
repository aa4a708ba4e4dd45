import json, os, sys, collections
sys.path.insert(0, os.getcwd())
import torch
import bench as B
from torch.profiler import profile, ProfilerActivity
wl = B.Workload("c2", None, "first")
api, dview, dmats, drhs = B.device_api(wl)
B.policy_step(wl, api, dview); torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU], with_stack=True) as prof:
    B.policy_step(wl, api, dview); torch.cuda.synchronize()
prof.export_chrome_trace("/tmp/tr.json")
ev = json.load(open("/tmp/tr.json"))["traceEvents"]
gpu = sorted([(e["ts"], e["ts"] + e.get("dur", 0), e["name"]) for e in ev
              if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")])
t0 = gpu[0][0]; t1 = gpu[-1][1]
busy = 0; gaps = []
cur_s, cur_e = gpu[0][0], gpu[0][1]
prev_name = gpu[0][2]
for s, e, nm in gpu[1:]:
    if s > cur_e:
        busy += cur_e - cur_s
        gaps.append((s - cur_e, cur_e, prev_name[:50], nm[:50]))
        cur_s, cur_e = s, e
    else:
        cur_e = max(cur_e, e)
    prev_name = nm
busy += cur_e - cur_s
print(f"span {(t1-t0)/1e3:.2f} ms, gpu busy {busy/1e3:.2f} ms, idle {(t1-t0-busy)/1e3:.2f} ms in {len(gaps)} gaps")
# python frames active during big gaps
py = [e for e in ev if e.get("cat") == "python_function"]
def py_at(t):
    best = None
    for e in py:
        if e["ts"] <= t <= e["ts"] + e.get("dur", 0):
            if best is None or e.get("dur", 0) < best.get("dur", 0):
                best = e
    return best["name"] if best else "?"
agg = collections.Counter(); cnt = collections.Counter()
for g, at, a, b in gaps:
    if g < 5: continue
    k = (a.split("(")[0], b.split("(")[0])
    agg[k] += g; cnt[k] += 1
for k, v in agg.most_common(25):
    print(f"{v/1e3:8.2f} ms  x{cnt[k]:4d}  after {k[0]} -> before {k[1]}")
big = sorted(gaps, reverse=True)[:15]
for g, at, a, b in big:
    print(f"gap {g/1e3:.3f} ms after {a} before {b}: py {py_at(at + g/2)}")
