"""Where the solve() setup goes at C2: H2D of each array, life_phi_create."""
import ctypes, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1905_06234_b200 as L  # noqa: E402
from paper_1905_06234_b200 import _native as N, datagen  # noqa: E402

dims = (1057, 200_000, 500_000, 96, 100_000_000)
cfg = L.GenConfig(dims=L.Dims(*dims), mean_run_length=520.0, seed=0, noise_sigma=0.1)
t, dic, w_true, noise = datagen.draw_arrays(cfg)
torch.zeros(1, device="cuda"); torch.cuda.synchronize()
cudart = torch.cuda.cudart()


def h2d_registered(arr):
    """H2D of a host numpy array page-locked in place (cudaHostRegister)."""
    a = np.ascontiguousarray(arr)
    ptr, nbytes = a.ctypes.data, a.nbytes
    rc = cudart.cudaHostRegister(ptr, nbytes, 0)
    t = torch.from_numpy(a.view(np.int32) if a.dtype == np.uint32 else a)
    out = t.to("cuda", non_blocking=True)
    torch.cuda.synchronize()
    if int(rc) == 0:
        cudart.cudaHostUnregister(ptr)
    return out, int(rc)


for rep in range(2):
    t0 = time.perf_counter()
    outs = [h2d_registered(getattr(t, n)) for n in ("atoms", "voxels", "fibers", "values")]
    print(f"rep {rep}: registered h2d of the 4 arrays {time.perf_counter() - t0:.3f}s rc={[o[1] for o in outs]}", flush=True)
    del outs
for rep in range(3):
    t0 = time.perf_counter()
    cols = []
    for name in ("atoms", "voxels", "fibers"):
        a = getattr(t, name)
        cols.append(torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint32).view(np.int32)).to("cuda"))
    torch.cuda.synchronize(); t1 = time.perf_counter()
    val = torch.from_numpy(np.ascontiguousarray(t.values)).to("cuda")
    d = torch.from_numpy(np.ascontiguousarray(dic.data)).to("cuda")
    torch.cuda.synchronize(); t2 = time.perf_counter()
    op = L.DeviceOperator.from_device(t.dims, cols[0], cols[1], cols[2], val, d)
    torch.cuda.synchronize(); t3 = time.perf_counter()
    print(f"rep {rep}: h2d idx {t1 - t0:.3f}s  h2d values+D {t2 - t1:.3f}s  create {t3 - t2:.3f}s "
          f"(sort_ms {op.info.sort_ms:.1f})", flush=True)
    del op, cols, val, d
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    op2 = L.DeviceOperator(t, dic)
    torch.cuda.synchronize()
    print(f"       DeviceOperator(host arrays) {time.perf_counter() - t4:.3f}s", flush=True)
    del op2
