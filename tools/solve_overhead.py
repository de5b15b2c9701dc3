"""Wall time of solve() around the device loop at C2: setup, loop, rest."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1905_06234_b200 as L  # noqa: E402
from paper_1905_06234_b200 import datagen, device, sbbnnls  # noqa: E402

dims = (1057, 200_000, 500_000, 96, 100_000_000)
cfg = L.GenConfig(dims=L.Dims(*dims), mean_run_length=520.0, seed=0, noise_sigma=0.1)
t, dic, w_true, noise = datagen.draw_arrays(cfg)
y = np.random.default_rng(0).standard_normal(dims[1] * dims[3])
p = L.Problem(tensor=t, dictionary=dic, y=y)
torch.zeros(1, device="cuda"); torch.cuda.synchronize()
for iters in (1, 1, 10, 100, 500):
    for graph in (True, False):
        c = L.SolverConfig(max_iters=iters, grad_tol=0.0, use_graph=graph)
        t0 = time.perf_counter()
        w, tr = L.solve(p, config=c)
        wall = time.perf_counter() - t0
        print(f"iters={iters:4d} graph={graph}: wall {wall:.3f}s setup {tr.setup_seconds:.3f}s "
              f"loop {tr.loop_seconds:.3f}s rest {wall - tr.setup_seconds - tr.loop_seconds:.3f}s", flush=True)
