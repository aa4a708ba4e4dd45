"""Kernel-time breakdown (torch.profiler / CUPTI) of one bench.py step on a
BASELINE config: the same systems, matrix builds, refresh_images and
RBiCGSTAB solves as bench.gpu_arm's step(); kernel time grouped by kernel
name, iteration kernels vs the per-system setup (build, transpose, refresh).
    python tools/c5_step_profile.py [--config c5] [--systems 2] [--top 30]"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

ITER = ("k_iter_spmv", "k_proj_dot", "k_phase")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    ap.add_argument("--systems", type=int, default=2)
    ap.add_argument("--top", type=int, default=30)
    a = ap.parse_args()
    import torch
    import bench as B
    import paper_1406_2831_b200 as P
    from paper_1406_2831_b200 import device as D
    wl = B.Workload(a.config, a.systems)
    cfgs = [P.SolverConfig(tol=wl.seq.tol, max_itn=wl.seq.max_itn, k=wl.k, s=wl.seq.s,
                           seed=j + 1) for j in range(len(wl.keys))]
    dev = {id(x): D.to_device(x, x.dtype) for _, x in wl.unique_arrays()}
    drhs = {key: D.to_device(b) for key, b in wl.rhs.items()}
    up = {i: (dev[id(A.row_ptr)], dev[id(A.col_idx)], dev[id(A.values)])
          for i, A in wl.mats.items()}
    i0 = wl.keys[0][0]
    A0 = wl.mats[i0]
    M0 = D.DeviceMatrix(A0.n, A0.row_ptr, A0.col_idx, A0.values, uploaded=up[i0])
    space0 = P.biorthonormalize(wl.U0, wl.Ut0, M0)
    del M0

    def step(marks):
        its, space, last_i = 0, space0, None
        for j, (i, kap) in enumerate(wl.keys):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            if i != last_i:
                A = wl.mats[i]
                M = D.DeviceMatrix(A.n, A.row_ptr, A.col_idx, A.values, uploaded=up[i])
                torch.cuda.synchronize()
                t1 = time.perf_counter()
                if j > 0:
                    space = P.refresh_images(space, M)
                last_i = i
            torch.cuda.synchronize()
            t2 = time.perf_counter()
            _, h = P.rbicgstab_solve(M, drhs[(i, kap)], recycle=space, config=cfgs[j])
            torch.cuda.synchronize()
            t3 = time.perf_counter()
            its += h.iterations
            marks.append({"system": i, "build_ms": round((t1 - t0) * 1e3, 2),
                          "refresh_ms": round((t2 - t1) * 1e3, 2),
                          "solve_ms": round((t3 - t2) * 1e3, 2), "its": h.iterations,
                          "us_per_it": round((t3 - t2) * 1e6 / max(h.iterations, 1), 1)})
        return its

    step([])
    from torch.profiler import profile, ProfilerActivity
    marks = []
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        its = step(marks)
    for m in marks:
        print(m)
    tot = {}
    for e in prof.key_averages():
        t = getattr(e, "device_time_total", None) or getattr(e, "cuda_time_total", 0)
        if t:
            tot[e.key] = (t, e.count)
    it_t = sum(t for k, (t, c) in tot.items() if any(s in k for s in ITER))
    other = sum(t for k, (t, c) in tot.items() if not any(s in k for s in ITER))
    print(f"{its} iterations; iteration kernels {it_t / 1e3:.1f} ms, "
          f"other kernels {other / 1e3:.1f} ms")
    for k, (t, c) in sorted(tot.items(), key=lambda kv: -kv[1][0])[:a.top]:
        print(f"{t / 1e3:10.2f} ms {c:7d}  {k[:110]}")
    # second pass without the profiler: wall time split
    marks = []
    step(marks)
    for m in marks:
        print("noprof", m)


if __name__ == "__main__":
    main()
