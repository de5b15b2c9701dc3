"""C2 (or C1 with --c1) binned products: a few DSC/WC calls for an ncu
launch list (kernel names k_side_*, k_tile_*, k_wc_fin)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1905_06234_b200 as L  # noqa: E402
from paper_1905_06234_b200 import _native as N, device  # noqa: E402

dims = L.Dims(1057, 10_000, 20_000, 96, 5_000_000) if "--c1" in sys.argv else \
    L.Dims(1057, 200_000, 500_000, 96, 100_000_000)
device.set_layout(os.environ.get("LAYOUT", "bin"))
SKEW = {  # tools/bin_check.py --skew cases
    "--zipf": dict(args=(1057, 200_000, 500_000, 96, 100_000_000, 12), zipf=1.3),
    "--u16": dict(args=(1057, 40_000, 100_000, 96, 16_000_000, 11)),
    "--hot16": dict(args=(1057, 40_000, 100_000, 96, 16_000_000, 11), hot_voxel=0.05),
}
case = next((a for a in sys.argv[1:] if a in SKEW), None)
if case:
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from bin_check import custom  # noqa: E402
    kw = dict(SKEW[case])
    t, dic = custom(*kw.pop("args"), **kw)
    dims = t.dims
    op = device.DeviceOperator(t, dic)
    w = torch.rand(dims.n_fibers, device="cuda")
else:
    p = L.generate(L.GenConfig(dims=dims, mean_run_length=520.0, weight_density=0.5, noise_sigma=0.1, seed=0))
    op = device.DeviceOperator(p.tensor, p.dictionary)
    w = torch.from_numpy(p.w_true).to("cuda", torch.float32)
y = torch.empty(dims.signal_len, dtype=torch.float32, device="cuda")
g = torch.empty(dims.n_fibers, dtype=torch.float32, device="cuda")
for _ in range(3):
    op.dsc_f32(w, y, None, N.SKIP_ZERO)
    op.wc_f32(y, g)
torch.cuda.synchronize()
print("done", op.kind)
