"""Time DSC / WC on a C2-shaped problem with a chosen mean_run_length
(voxel-count variance), e.g. to A/B the staged producer:
  LIFE_DEBUG=1 [LIFE_WS_UNSTAGED=1] python tools/ab_layout.py --mrl 4"""
import argparse, os, statistics, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1905_06234_b200 as L  # noqa: E402
from paper_1905_06234_b200 import _native, datagen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--mrl", type=float, default=520.0)
ap.add_argument("--nc", type=int, default=100_000_000)
ap.add_argument("--reps", type=int, default=10)
args = ap.parse_args()
nv = args.nc // 500
dims = (1057, nv, nv * 5 // 2, 96, args.nc)
cfg = L.GenConfig(dims=L.Dims(*dims), mean_run_length=args.mrl, seed=0, noise_sigma=0.1)
t, dic, w_true, _ = datagen.draw_arrays(cfg)
op = L.DeviceOperator(t, dic)
w = torch.from_numpy(w_true).float().cuda()
y = torch.empty(dims[1] * dims[3], device="cuda")
g = torch.empty(dims[2], device="cuda")
ym = torch.zeros(1, device="cuda")


def timeit(fn):
    for _ in range(2):
        fn()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.reps)]
    for a, b in ev:
        a.record(); fn(); b.record()
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(b) for a, b in ev)


td = timeit(lambda: op.dsc_f32(w, y, flags=_native.SKIP_ZERO, absmax=ym))
tw = timeit(lambda: op.wc_f32(y, g, y_absmax=ym))
print(f"mrl={args.mrl} nc={args.nc} kernels={op.kind} dsc_ms={td:.4f} wc_ms={tw:.4f} "
      f"y={float(y.double().norm()):.6e} g={float(g.double().norm()):.6e}", flush=True)
