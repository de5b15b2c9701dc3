"""Time k_dsc_ws with consumers or producers disabled (diagnostic)."""
import ctypes, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1905_06234_b200 as L
from paper_1905_06234_b200 import _native, datagen
dims = (1057, 200_000, 500_000, 96, 100_000_000)
cfg = L.GenConfig(dims=L.Dims(*dims), mean_run_length=520.0, seed=0, noise_sigma=0.1)
t, dic, w_true, _ = datagen.draw_arrays(cfg)
op = L.DeviceOperator(t, dic)
lib = _native.lib()
lib.life_debug_ws_isolate.argtypes = [ctypes.c_int]
w = torch.from_numpy(w_true).float().cuda()
y = torch.empty(dims[1] * dims[3], device="cuda"); g = torch.empty(dims[2], device="cuda")
ym = torch.zeros(1, device="cuda")
for mode in [0, 1, 2] + [1 | (f << 8) for f in (1, 2, 4, 3, 7)] + [0]:
    lib.life_debug_ws_isolate(mode)
    for _ in range(2): op.dsc_f32(w, y, flags=_native.SKIP_ZERO, absmax=ym)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): op.dsc_f32(w, y, flags=_native.SKIP_ZERO, absmax=ym)
    e1.record(); torch.cuda.synchronize()
    print("mode", mode, "dsc ms", e0.elapsed_time(e1) / 10, flush=True)
lib.life_debug_ws_isolate(0)
