"""solve() setup at C2: DeviceOperator from host arrays (staged H2D +
restructuring, life_phi_create's sort_ms), the b upload, and whole solve()
calls from fresh PhiTensor objects (as bench.py's e2e does)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1905_06234_b200 as L  # noqa: E402
from paper_1905_06234_b200 import device  # noqa: E402

p = L.generate(L.GenConfig(dims=L.Dims(1057, 200_000, 500_000, 96, 100_000_000),
                           mean_run_length=520.0, weight_density=0.5, noise_sigma=0.1, seed=0))
torch.zeros(1, device="cuda")
torch.cuda.synchronize()
for rep in range(3):
    t0 = time.perf_counter()
    op = device.DeviceOperator(p.tensor, p.dictionary)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    b = device.upload(np.asarray(p.y, dtype=np.float64), torch.float32)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"rep {rep}: operator {1e3*(t1-t0):.1f} ms (create {op.info.sort_ms:.1f} ms), "
          f"b upload {1e3*(t2-t1):.1f} ms, device {op.info.device_bytes/1e9:.2f} GB", flush=True)
    op.close()
t = p.tensor
for rep in range(3):
    fresh = L.PhiTensor(atoms=t.atoms, voxels=t.voxels, fibers=t.fibers, values=t.values, dims=t.dims)
    p2 = L.Problem(tensor=fresh, dictionary=p.dictionary, y=p.y)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    w, tr = L.solve(p2, config=L.SolverConfig(max_iters=20, grad_tol=0.0))
    dt = time.perf_counter() - t0
    op = fresh.__dict__["_device_cache"]["op"][0]
    print(f"solve {rep}: {dt*1e3:.1f} ms, setup {tr.setup_seconds*1e3:.1f} ms (create {op.info.sort_ms:.1f} ms), "
          f"loop {tr.loop_seconds*1e3:.1f} ms", flush=True)
    op.close()
