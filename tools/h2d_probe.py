"""Host->device copy options for the e2e setup (2.15 GB of Phi at C2):
pageable .to('cuda'), cudaHostRegister of the numpy buffer + async copy,
and pinned staging with multi-threaded memcpy."""
import ctypes
import os
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

n = 2_000_000_000 // 8
a = np.random.default_rng(0).random(n)
torch.cuda.init()
d = torch.empty(n, dtype=torch.float64, device="cuda")
cudart = ctypes.CDLL("libcudart.so.12") if False else None
print("cpus", os.cpu_count(), flush=True)

def t(f, name, reps=2):
    for i in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    print(f"{name:40s} {dt*1e3:8.1f} ms  {a.nbytes/dt/1e9:6.1f} GB/s", flush=True)

t(lambda: d.copy_(torch.from_numpy(a)), "pageable copy_")
rt = torch.cuda.cudart()
def reg():
    rt.cudaHostRegister(a.ctypes.data, a.nbytes, 0)
def unreg():
    rt.cudaHostUnregister(a.ctypes.data)
for i in range(2):
    t0 = time.perf_counter(); reg(); r = time.perf_counter() - t0
    t(lambda: d.copy_(torch.from_numpy(a), non_blocking=True), "registered copy_", reps=1)
    t0 = time.perf_counter(); unreg(); u = time.perf_counter() - t0
    print(f"  register {r*1e3:.1f} ms, unregister {u*1e3:.1f} ms", flush=True)
pin = torch.empty(n, dtype=torch.float64, pin_memory=True)
t(lambda: d.copy_(pin, non_blocking=True), "pinned (already staged) copy_")
src = torch.from_numpy(a)
for nt in (1, 4, 8, 16, 32):
    ex = ThreadPoolExecutor(nt)
    def mt():
        step = (n + nt - 1) // nt
        list(ex.map(lambda i: pin[i*step:(i+1)*step].copy_(src[i*step:(i+1)*step]), range(nt)))
    t(mt, f"host memcpy -> pinned, {nt} threads")
    ex.shutdown()
# pipelined: chunks of 64 MB, memcpy (16 threads) overlapped with DMA
ex = ThreadPoolExecutor(16)
chunk = 8 * 1024 * 1024
bufs = [torch.empty(chunk, dtype=torch.float64, pin_memory=True) for _ in range(3)]
evs = [torch.cuda.Event() for _ in range(3)]
s = torch.cuda.Stream()
def pipe(nt=16):
    k = 0
    for c0 in range(0, n, chunk):
        c1 = min(n, c0 + chunk)
        b = bufs[k % 3]
        evs[k % 3].synchronize()
        m = c1 - c0
        step = (m + nt - 1) // nt
        list(ex.map(lambda i: b[i*step:min(m, (i+1)*step)].copy_(src[c0+i*step:c0+min(m, (i+1)*step)]), range(nt)))
        with torch.cuda.stream(s):
            d[c0:c1].copy_(b[:m], non_blocking=True)
            evs[k % 3].record(s)
        k += 1
    s.synchronize()
t(pipe, "pipelined 64MB chunks, 16 threads")
