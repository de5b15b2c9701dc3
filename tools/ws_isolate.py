"""Time k_dsc_ws / k_wc_ws with consumers or producers disabled (diagnostic build):
  make -C paper_1905_06234_b200/csrc diag
  LIFE_B200_LIB=$PWD/build/diag/liblife_b200.so python tools/ws_isolate.py [--mrl 520]
mode: 0 full, 1 producers only, 2 consumers only; flags<<8: 1 no L2 prefetch, 4 no gather."""
import argparse, ctypes, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1905_06234_b200 as L  # noqa: E402
from paper_1905_06234_b200 import _native, datagen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--mrl", type=float, default=520.0)
args = ap.parse_args()
dims = (1057, 200_000, 500_000, 96, 100_000_000)
cfg = L.GenConfig(dims=L.Dims(*dims), mean_run_length=args.mrl, seed=0, noise_sigma=0.1)
t, dic, w_true, _ = datagen.draw_arrays(cfg)
op = L.DeviceOperator(t, dic)
lib = _native.lib()
lib.life_debug_ws_isolate.argtypes = [ctypes.c_int]
w = torch.from_numpy(w_true).float().cuda()
y = torch.empty(dims[1] * dims[3], device="cuda"); g = torch.empty(dims[2], device="cuda")
ym = torch.ones(1, device="cuda")
for name, fn in (("dsc", lambda: op.dsc_f32(w, y, flags=_native.SKIP_ZERO, absmax=ym)),
                 ("wc", lambda: op.wc_f32(y, g, y_absmax=ym))):
    for mode in [int(x, 0) for x in os.environ.get("WS_MODES", "0,1,2,0x101,0x401").split(",")]:
        lib.life_debug_ws_isolate(mode)
        for _ in range(2): fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10): fn()
        e1.record(); torch.cuda.synchronize()
        print(f"mrl={args.mrl} {name} mode {mode:#x} ms {e0.elapsed_time(e1) / 10:.4f}", flush=True)
# per-phase cycle counters of one DSC (sums over producer / consumer warps)
nprod, ncons = 148 * int(os.environ.get("WS_PROD", "4")), 148 * 8
for mode in (0, 1, 1 | (4 << 8)):
    lib.life_debug_ws_isolate(mode)
    cyc = (ctypes.c_ulonglong * 8)()
    lib.life_debug_ws_counters(cyc)
    op.dsc_f32(w, y, flags=_native.SKIP_ZERO, absmax=ym)
    lib.life_debug_ws_counters(cyc)
    c = list(cyc)
    print(f"mode {mode:#x} per producer warp (Mcyc): slot wait {c[0]/nprod/1e6:.3f} "
          f"empty wait {c[1]/nprod/1e6:.3f} build {c[2]/nprod/1e6:.3f} (fast {c[6]/nprod/1e6:.3f} "
          f"slow {c[7]/nprod/1e6:.3f}); per consumer warp: full wait {c[4]/ncons/1e6:.3f} "
          f"compute {c[5]/ncons/1e6:.3f}", flush=True)
lib.life_debug_ws_isolate(0)
