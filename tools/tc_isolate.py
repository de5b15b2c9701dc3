"""Isolation of the tcgen05 DSC at C2 (diagnostic build):
  make -C paper_1905_06234_b200/csrc diag
  LIFE_B200_LIB=$PWD/build/diag/liblife_b200.so python tools/tc_isolate.py
flags: 1 no tile build, 2 no MMA, 4 no gathers, 8 no epilogue TMEM loads."""
import argparse, ctypes, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1905_06234_b200 as L  # noqa: E402
from paper_1905_06234_b200 import _native, datagen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--c1", action="store_true")
args = ap.parse_args()
dims = (1057, 10_000, 20_000, 96, 5_000_000) if args.c1 else (1057, 200_000, 500_000, 96, 100_000_000)
cfg = L.GenConfig(dims=L.Dims(*dims), mean_run_length=1.04 * dims[4] / dims[1], seed=0)
t, dic, w_true, _ = datagen.draw_arrays(cfg)
L.device.set_layout("tensor")
op = L.DeviceOperator(t, dic)
assert op.kind == "tensor", op.kind
lib = _native.lib()
lib.life_debug_tc.argtypes = [ctypes.c_int, ctypes.c_void_p]
w = torch.from_numpy(w_true).float().cuda()
y = torch.empty(dims[1] * dims[3], device="cuda")
names = ["slot wait+gather issue", "empty wait", "build", "split", "w move",
         "mma: full wait", "mma: accempty wait", "epi: accfull wait"]
for fl in [int(x, 0) for x in os.environ.get('TC_FLAGS', '0,0xff,0x7e,0x7a,0x4').split(',')]:
    lib.life_debug_tc(fl, None)
    for _ in range(2):
        op.dsc_f32(w, y)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        op.dsc_f32(w, y)
    e1.record(); torch.cuda.synchronize()
    cyc = (ctypes.c_ulonglong * 16)()
    lib.life_debug_tc(fl, cyc)
    op.dsc_f32(w, y)
    lib.life_debug_tc(fl, cyc)
    c = list(cyc)
    prod, mma, epi = 148 * 8, 148, 148 * 4
    per = [c[i] / prod / 1e6 for i in range(5)] + [c[5] / mma / 1e6, c[6] / mma / 1e6, c[7] / epi / 1e6]
    print(f"flags {fl:#x}: {e0.elapsed_time(e1) / 10:.4f} ms | " +
          " ".join(f"{n}={v:.3f}" for n, v in zip(names, per)) + " (Mcyc per warp)", flush=True)
lib.life_debug_tc(0, None)
