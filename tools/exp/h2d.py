import numpy as np, time, torch, sys
sys.path.insert(0, ".")
from paper_1406_2831_b200.device import to_device
big = np.random.rand(32_000_000)
def tm(f, reps=3):
    f(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        t = time.perf_counter(); f(); torch.cuda.synchronize(); best = min(best, time.perf_counter() - t)
    return big.nbytes / best / 1e9
print("staged chunked", tm(lambda: to_device(big)))
print("torch pageable", tm(lambda: torch.from_numpy(big).to("cuda")))
cr = torch.cuda.cudart()
def reg():
    t = torch.from_numpy(big)
    cr.cudaHostRegister(t.data_ptr(), big.nbytes, 0)
    out = t.to("cuda", non_blocking=True)
    torch.cuda.synchronize()
    cr.cudaHostUnregister(t.data_ptr())
    return out
print("register+copy", tm(reg))
t = torch.from_numpy(big); cr.cudaHostRegister(t.data_ptr(), big.nbytes, 0)
print("pre-registered", tm(lambda: t.to("cuda", non_blocking=True)))
p = torch.empty(big.nbytes, dtype=torch.uint8, pin_memory=True)
print("pinned src", tm(lambda: p.to("cuda", non_blocking=True)))
hb = p.numpy(); src = big.view(np.uint8)
print("host memcpy 1 thread", tm(lambda: np.copyto(hb, src)))
