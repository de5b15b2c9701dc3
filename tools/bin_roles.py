"""Role timing of the binned tile kernels (diagnostic build, -DLIFE_BIN_DIAG).

    make -C paper_1905_06234_b200/csrc variant NAME=bindiag DEFS=-DLIFE_BIN_DIAG
    LIFE_B200_LIB=build/bindiag/liblife_b200.so python tools/bin_roles.py [--c1]

Per category: clock cycles summed over the role's warps, divided by CTAs x
role warps x calls, shown in microseconds at 1.965 GHz (per warp per call;
compare with the kernel time)."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1905_06234_b200 as L  # noqa: E402
from paper_1905_06234_b200 import _native as N, device  # noqa: E402

dims = L.Dims(1057, 10_000, 20_000, 96, 5_000_000) if "--c1" in sys.argv else \
    L.Dims(1057, 200_000, 500_000, 96, 100_000_000)
p = L.generate(L.GenConfig(dims=dims, mean_run_length=520.0, weight_density=0.5, noise_sigma=0.1, seed=0))
op = device.DeviceOperator(p.tensor, p.dictionary)
lib = N.lib()
lib.life_debug_bin.argtypes = [ctypes.c_void_p]
w = torch.from_numpy(p.w_true).to("cuda", torch.float32)
y = torch.empty(dims.signal_len, dtype=torch.float32, device="cuda")
g = torch.empty(dims.n_fibers, dtype=torch.float32, device="cuda")
buf = (ctypes.c_ulonglong * 32)()
reps, ctas = 5, 148
names = {0: ("build", 8, "wait slot_full"), 1: ("build", 8, "scatter pass"), 2: ("build", 8, "bar C complete"),
         3: ("build", 8, "wait a_empty"), 4: ("build", 8, "convert"), 5: ("build", 8, "bar zeroed"),
         6: ("mma", 1, "wait acc_empty"), 7: ("mma", 1, "wait a_full"), 8: ("mma", 1, "wait d_full"),
         9: ("prodS", 1, "wait slot_empty"), 10: ("prodD", 1, "wait d_empty"), 11: ("epi", 8, "wait acc_full"),
         12: ("epi", 8, "fold"), 13: ("sideC", 31, "wait full"), 14: ("sideC", 31, "process"),
         15: ("sideP", 1, "wait empty"), 9: ("sideC", 31, "process"), 30: ("sideC", 31, "wait full (z)"),
         31: ("sideP", 1, "wait empty"),
         16: ("gath", 8, "wait slot_full"), 17: ("gath", 8, "wait z_full"), 18: ("gath", 8, "gather pass"),
         19: ("mma", 1, "wait y_ready"), 20: ("mma", 1, "wait d_full"), 21: ("mma", 1, "wait acc_empty"),
         22: ("prodS", 1, "wait slot_empty"), 23: ("prodD", 1, "wait d_empty"), 24: ("yz", 8, "wait y_free"),
         25: ("yz", 8, "y store"), 26: ("yz", 8, "wait acc_full"), 27: ("yz", 8, "ld Z"), 28: ("yz", 8, "wait z_empty"),
         29: ("yz", 8, "store Z")}
for prod in ("dsc", "wc"):
    call = (lambda: op.dsc_f32(w, y, None, N.SKIP_ZERO)) if prod == "dsc" else (lambda: op.wc_f32(y, g))
    for _ in range(2):
        call()
    lib.life_debug_bin(None)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(reps):
        call()
    ev1.record()
    lib.life_debug_bin(buf)
    print(f"== {prod}: {ev0.elapsed_time(ev1) / reps * 1e3:.1f} us per call (all kernels)")
    for i in range(32):
        if buf[i] and i in names:
            role, nw, what = names[i]
            print(f"  [{i:2d}] {role:6s} {what:18s} {buf[i] / (ctas * nw * reps) / 1965.0:8.1f} us")
