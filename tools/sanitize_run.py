"""Small end-to-end run for compute-sanitizer: operator build (host input,
staged copies), fp32 DSC/WC on the default binned tcgen05 kernels, fp64
exact products, and a short SBBNNLS solve (graph path).

    compute-sanitizer --tool memcheck python tools/sanitize_run.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1905_06234_b200 as L  # noqa: E402
from paper_1905_06234_b200 import _native as N, device  # noqa: E402

dims = L.Dims(n_atoms=300, n_voxels=3000, n_fibers=4000, n_dirs=96, n_coeffs=600_000)
p = L.generate(L.GenConfig(dims=dims, mean_run_length=208.0, weight_density=0.5, noise_sigma=0.1, seed=3))
op = device.DeviceOperator(p.tensor, p.dictionary, exact=True)
print("kind", op.kind, "tensor ops", op.tensor_ops, flush=True)
w = torch.from_numpy(p.w_true).to("cuda", torch.float32)
y = torch.empty(dims.signal_len, dtype=torch.float32, device="cuda")
g = torch.empty(dims.n_fibers, dtype=torch.float32, device="cuda")
for _ in range(2):
    op.dsc_f32(w, y, None, N.SKIP_ZERO)
    op.wc_f32(y, g)
y64 = torch.zeros(dims.signal_len, dtype=torch.float64, device="cuda")
op.dsc_f64(w.double(), y64, N.SKIP_ZERO)
g64 = torch.zeros(dims.n_fibers, dtype=torch.float64, device="cuda")
op.wc_f64(y64, g64)
torch.cuda.synchronize()
print("dsc rel", float(torch.linalg.norm(y.double() - y64) / torch.linalg.norm(y64)), flush=True)
op.close()
wsol, tr = L.solve(p, config=L.SolverConfig(max_iters=6, grad_tol=0.0))
print("solve", tr.termination, tr.final_objective, flush=True)
