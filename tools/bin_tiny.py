"""Smallest binned-product cases (debugging aid), with the host-mapped
timeout record: prints which mbarrier wait timed out if a kernel traps."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from bin_check import custom, check  # noqa: E402
from paper_1905_06234_b200 import _native as N  # noqa: E402

torch.cuda.init()
cudart = ctypes.CDLL("libcudart.so") if False else None
rec = torch.zeros(8, dtype=torch.int32).pin_memory()
lib = N.lib()
lib.life_debug_timeout.argtypes = [ctypes.c_void_p]
print("register:", lib.life_debug_timeout(ctypes.c_void_p(rec.data_ptr())))
try:
    t, d = custom(64, 500, 800, 96, 40_000, 3)
    print(check("tiny", t, d, "bin", reps=1))
except Exception as e:
    print("FAILED:", str(e).splitlines()[0])
print("timeout record:", rec.tolist())
