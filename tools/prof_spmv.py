"""Run DSC / WC a few times on a bench config (for ncu captures)."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1905_06234_b200 as L  # noqa: E402
from paper_1905_06234_b200 import _native, datagen  # noqa: E402

CONFIGS = {"c2": (1057, 200_000, 500_000, 96, 100_000_000),
           "c1": (1057, 10_000, 20_000, 96, 5_000_000)}

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--layout", default="auto")
args = ap.parse_args()
dims = CONFIGS[args.config]
cfg = L.GenConfig(dims=L.Dims(*dims), mean_run_length=1.04 * dims[4] / dims[1], seed=0,
                  noise_sigma=0.1)
t, dic, w_true, _ = datagen.draw_arrays(cfg)
L.device.set_layout(args.layout)
op = L.DeviceOperator(t, dic)
print("kernels:", op.kind)
w = torch.from_numpy(w_true).float().cuda()
y = torch.empty(dims[1] * dims[3], device="cuda")
g = torch.empty(dims[2], device="cuda")
ymax = torch.zeros(1, device="cuda")
for _ in range(args.reps):
    op.dsc_f32(w, y, flags=_native.SKIP_ZERO, absmax=ymax)
for _ in range(args.reps):
    op.wc_f32(y, g, y_absmax=ymax)
torch.cuda.synchronize()
print("done", float(g.abs().sum()))
