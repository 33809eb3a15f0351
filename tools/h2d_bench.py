"""Host<->device copy options for the numpy API (154 MB input, 2 x 154 MB outputs)."""
import time

import numpy as np
import torch

n = 8 * 100001 * 24
a = np.random.rand(n)
dev = torch.device("cuda")
d = torch.empty(n, dtype=torch.float64, device=dev)
torch.cuda.synchronize()


def tm(f, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best * 1e3


print(f"threads {torch.get_num_threads()}")
print(f"H2D pageable .to(dev)                 {tm(lambda: torch.from_numpy(a).to(dev)):7.1f} ms")
print(f"H2D pin_memory() + .to(non_blocking)  {tm(lambda: torch.from_numpy(a).pin_memory().to(dev, non_blocking=True)):7.1f} ms")
p = torch.empty(n, dtype=torch.float64, pin_memory=True)
print(f"  numpy -> pinned copy_ only          {tm(lambda: p.copy_(torch.from_numpy(a))):7.1f} ms")
print(f"  pinned -> device only               {tm(lambda: d.copy_(p, non_blocking=True)):7.1f} ms")


def reg():
    t = torch.from_numpy(a)
    r = torch.cuda.cudart().cudaHostRegister(t.data_ptr(), t.numel() * 8, 0)
    d.copy_(t, non_blocking=True)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaHostUnregister(t.data_ptr())


print(f"H2D cudaHostRegister + copy + unreg   {tm(reg):7.1f} ms")
print(f"D2H pageable .cpu().numpy()           {tm(lambda: d.cpu().numpy()):7.1f} ms")


def d2h_pinned():
    o = torch.empty(n, dtype=torch.float64, pin_memory=True)
    o.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    return o.numpy()


print(f"D2H into cached pinned (+alloc)       {tm(d2h_pinned):7.1f} ms")
