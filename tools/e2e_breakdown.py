"""Where does the end-to-end solve() time go?  (diagnostic, C2 by default)"""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1905_06234_b200 as L
from paper_1905_06234_b200 import datagen

dims = (1057, 200_000, 500_000, 96, 100_000_000)
cfg = L.GenConfig(dims=L.Dims(*dims), mean_run_length=520.0, seed=0, noise_sigma=0.1)
t0 = time.perf_counter(); t, dic, w_true, noise = datagen.draw_arrays(cfg); print("draw", time.perf_counter() - t0, flush=True)
torch.cuda.init(); torch.zeros(1, device="cuda"); torch.cuda.synchronize()
for name in ("atoms", "voxels", "fibers", "values"):
    a = getattr(t, name)
    t0 = time.perf_counter(); g = torch.from_numpy(a.view(np.int32) if a.dtype == np.uint32 else a).to("cuda"); torch.cuda.synchronize()
    print(f"h2d {name} {a.nbytes/1e9:.2f} GB {time.perf_counter()-t0:.3f}s", flush=True)
    del g
for rep in range(2):
    t0 = time.perf_counter(); op = L.DeviceOperator(t, dic); torch.cuda.synchronize()
    print("DeviceOperator", rep, time.perf_counter() - t0, "sort_ms", op.info.sort_ms, flush=True)
    del op
y = np.random.default_rng(0).standard_normal(dims[1] * dims[3])
p = L.Problem(tensor=t, dictionary=dic, y=y)
for rep in range(2):
    fresh = L.PhiTensor(atoms=t.atoms, voxels=t.voxels, fibers=t.fibers, values=t.values, dims=t.dims)
    p2 = L.Problem(tensor=fresh, dictionary=dic, y=y)
    t0 = time.perf_counter(); w, tr = L.solve(p2, config=L.SolverConfig(max_iters=20, grad_tol=0.0)); print("solve", rep, time.perf_counter() - t0, tr.loop_seconds, flush=True)
