"""Kernel-time breakdown (torch.profiler / CUPTI) of the whole sequence policy
('first': RBiCG + harvest + m = k + s + 2 update on system 0, refresh +
guarded RBiCGSTAB after) on a BASELINE config, through the public API.
    python tools/policy_profile.py --config c5 [--top 30]"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    ap.add_argument("--top", type=int, default=30)
    a = ap.parse_args()
    import torch
    import paper_1406_2831_b200 as P
    from paper_1406_2831_b200 import device as D, workloads as W
    from paper_1406_2831_b200.sequence import run_sequence
    seq = W.make_sequence(a.config)
    mats = {}

    def mat(i):
        if i not in mats:
            mats[i] = seq.matrix_fn(i)
        return mats[i]
    view = W.SequenceSpec(seq.name, seq.n, seq.k, seq.tol, seq.num_matrices,
                          seq.rhs_per_matrix, mat, seq.rhs_fn, s=seq.s,
                          max_itn=seq.max_itn, meta=seq.meta)
    for i in range(seq.num_matrices):
        mat(i)
    run_sequence(view, policy="first", baseline=False, api=P)   # warm-up
    D.MATRICES.clear()
    torch.cuda.synchronize()
    from torch.profiler import profile, ProfilerActivity
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        t0 = time.perf_counter()
        res = run_sequence(view, policy="first", baseline=False, api=P)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    rec = res.recycling
    print(f"policy {dt:.2f} s (under the profiler), {rec.total_iterations} iterations, "
          f"per system {[h.iterations for h in rec.histories]}, dims {res.space_dims}")
    tot = {}
    for e in prof.key_averages():
        t = getattr(e, "device_time_total", None) or getattr(e, "cuda_time_total", 0)
        if t:
            tot[e.key] = (t, e.count)
    print(f"kernel time total {sum(t for t, _ in tot.values()) / 1e3:.1f} ms")
    for k, (t, c) in sorted(tot.items(), key=lambda kv: -kv[1][0])[:a.top]:
        print(f"{t / 1e3:10.2f} ms {c:7d}  {k[:110]}")
    D.MATRICES.clear()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    run_sequence(view, policy="first", baseline=False, api=P)
    torch.cuda.synchronize()
    print(f"policy without the profiler: {time.perf_counter() - t0:.2f} s")


if __name__ == "__main__":
    main()
