import time, os, torch, numpy as np
print("cpus", os.cpu_count(), "torch threads", torch.get_num_threads())
S = np.random.rand(8, 100001, 24)
St = torch.from_numpy(S)
pin = torch.empty(St.shape, dtype=torch.float64, pin_memory=True)
R = 4096
for rep in range(3):
    t0 = time.perf_counter()
    for j in range(0, 100001, R):
        pin[:, j:j+R].copy_(St[:, j:j+R])
    t1 = time.perf_counter()
    print(f"torch chunked copy: {1e3*(t1-t0):.1f} ms total, {154/(t1-t0)/1e3:.1f} GB/s")
pn = pin.numpy()
for rep in range(2):
    t0 = time.perf_counter()
    for j in range(0, 100001, R):
        np.copyto(pn[:, j:j+R], S[:, j:j+R])
    t1 = time.perf_counter()
    print(f"numpy chunked copy: {1e3*(t1-t0):.1f} ms total, {154/(t1-t0)/1e3:.1f} GB/s")
from concurrent.futures import ThreadPoolExecutor
ex = ThreadPoolExecutor(4)
for rep in range(2):
    t0 = time.perf_counter()
    futs = []
    for j in range(0, 100001, R):
        for b in range(8):
            futs.append(ex.submit(pin[b, j:j+R].copy_, St[b, j:j+R]))
    for f in futs: f.result()
    t1 = time.perf_counter()
    print(f"4-thread per-sequence copy: {1e3*(t1-t0):.1f} ms total, {154/(t1-t0)/1e3:.1f} GB/s")
