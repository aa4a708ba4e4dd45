"""Kernel-time breakdown of one bench step (torch.profiler / CUPTI):
    python tools/step_profile.py [--config c2] [--top 25]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--top", type=int, default=25)
    a = ap.parse_args()
    import torch
    import bench as B
    wl = B.Workload(a.config, None, "first")
    api, dview, dmats, drhs = B.device_api(wl)
    B.policy_step(wl, api, dview)
    torch.cuda.synchronize()
    from torch.profiler import profile, ProfilerActivity
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record()
        res, it = B.policy_step(wl, api, dview)
        t1.record()
        torch.cuda.synchronize()
    print(f"step {t0.elapsed_time(t1):.2f} ms, {it} iterations, dims {res.space_dims}")
    print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=a.top, max_name_column_width=60))


if __name__ == "__main__":
    main()
