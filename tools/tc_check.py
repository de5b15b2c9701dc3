"""tcgen05 DSC vs the CUDA-core tile DSC and the fp64 exact DSC at a given
config: relative L2 error, skip counts and CUDA-event times.
  python tools/tc_check.py [--c1]"""
import argparse, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1905_06234_b200 as L  # noqa: E402
from paper_1905_06234_b200 import _native, datagen, device  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--c1", action="store_true")
ap.add_argument("--reps", type=int, default=20)
args = ap.parse_args()
dims = (1057, 10_000, 20_000, 96, 5_000_000) if args.c1 else (1057, 200_000, 500_000, 96, 100_000_000)
mrl = 1.04 * dims[4] / dims[1]
cfg = L.GenConfig(dims=L.Dims(*dims), mean_run_length=mrl, seed=0, noise_sigma=0.1)
t0 = time.time()
t, dic, w_true, _ = datagen.draw_arrays(cfg)
print(f"generate {time.time() - t0:.1f}s", flush=True)
rng = np.random.default_rng(1)
w64 = w_true.copy()
w = torch.from_numpy(w64).float().cuda()
res = {}
for lay in ("tensor", "dense"):
    device.set_layout(lay)
    t0 = time.time()
    op = L.DeviceOperator(t, dic, exact=(lay == "dense"))
    torch.cuda.synchronize()
    print(f"{lay}: kind={op.kind} build {time.time() - t0:.2f}s", flush=True)
    y = torch.zeros(dims[1] * dims[3], device="cuda")
    sk = torch.zeros(1, dtype=torch.int64, device="cuda")
    op.dsc_f32(w, y, flags=_native.SKIP_ZERO)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.reps):
        op.dsc_f32(w, y, flags=_native.SKIP_ZERO)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.reps
    res[lay] = y.double().cpu().numpy()
    g = torch.zeros(dims[2], device="cuda")
    ymax = torch.ones(1, device="cuda") * float(y.abs().max())
    op.wc_f32(y, g, y_absmax=ymax)
    e0.record()
    for _ in range(args.reps):
        op.wc_f32(y, g, y_absmax=ymax)
    e1.record(); torch.cuda.synchronize()
    print(f"{lay}: wc {e0.elapsed_time(e1) / args.reps:.4f} ms", flush=True)
    res[lay + "_wc"] = g.double().cpu().numpy()
    if lay == "tensor":
        y_in = y.clone()
    print(f"{lay}: dsc {ms:.4f} ms  ({12 * dims[4] / ms / 1e6:.0f} GB/s algorithmic idx+val)", flush=True)
    if lay == "dense":
        y64 = torch.zeros(dims[1] * dims[3], dtype=torch.float64, device="cuda")
        op.dsc_f64(torch.from_numpy(w64).cuda(), y64)
        ref = y64.cpu().numpy()
        g64 = torch.zeros(dims[2], dtype=torch.float64, device="cuda")
        op.wc_f64(y_in.double(), g64)
        ref_wc = g64.cpu().numpy()
        gd = torch.zeros(dims[2], device="cuda")
        op.wc_f32(y_in, gd, y_absmax=torch.ones(1, device="cuda") * float(y_in.abs().max()))
        res["dense_wc_same_y"] = gd.double().cpu().numpy()
    del op
    torch.cuda.empty_cache()
device.set_layout("auto")
rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
print(f"DSC rel_l2 tensor vs fp64 exact: {rel(res['tensor'], ref):.3e}   dense vs fp64: {rel(res['dense'], ref):.3e}")
print(f"WC  rel_l2 tensor vs fp64 exact: {rel(res['tensor_wc'], ref_wc):.3e}   dense vs fp64: {rel(res['dense_wc_same_y'], ref_wc):.3e}")
